#!/bin/bash
# ncu evidence for round 1 (run under gpurun on one B200)
set -x
M="sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second"
OUT=gpurun_out
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $OUT/sweep_metrics.csv python tools/profile_sweep.py > $OUT/sweep_order.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --e2e-steps 1 > $OUT/launches_bench.json 2>&1
for spec in "rosenbrock 16 hvp_reg" "ackley 16 hvp_reg" "fletcher_powell 16 hvp_f3" "rosenbrock 1 hvp_reg"; do
  set -- $spec
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$3 -c 1 -o $OUT/prof_${1}_C$2 python tools/profile_sweep.py --funcs $1 --csizes $2 > /dev/null 2>&1
done
ls -la $OUT
