#!/bin/bash
# key ncu metrics of every kernel the register probe launches (one launch each)
O=gpurun_out/${1:-probe_ncu}; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include ${2:-} tools/micro/reg_probe.cu -o /tmp/reg_probe || exit 1
/tmp/reg_probe > $O/probe.txt 2>&1; cat $O/probe.txt
M="gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,launch__registers_per_thread,smsp__issue_active.avg.pct_of_peak_sustained_active"
timeout 600 ncu --metrics $M --clock-control none -k regex:"${3:-.}" -c ${4:-40} --csv --log-file $O/metrics.csv /tmp/reg_probe > /dev/null 2>&1
python - $O/metrics.csv <<'PY'
import csv,sys,collections
rows=list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith('==')))
seen=collections.OrderedDict()
for r in rows:
    k=(r['ID'],r['Kernel Name'][:60]); seen.setdefault(k,{})[r['Metric Name']]=r['Metric Value']
done=set()
for (i,name),m in seen.items():
    if name in done: continue
    done.add(name)
    print(name, {k.split('.')[0].replace('sm__sass_thread_inst_executed_op_','').replace('smsp__',''):v for k,v in m.items()})
PY
