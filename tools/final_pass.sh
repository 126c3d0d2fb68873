#!/bin/bash
# End-of-round pass on the committed build: GPU suite, smoke, the driver's bench command (+ the
# reference arm), the ncu launch list of the bench command.
set -x
O=gpurun_out/r02${1:-end}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
python bench.py > $O/bench.log 2>&1; echo bench_rc=$?
cp gpurun_out/bench_sweep.json $O/ 2>/dev/null
python bench.py --impl reference > $O/bench_reference.log 2>&1; echo ref_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-strong --e2e-steps 1 > $O/bench_ncu.log 2>&1; echo ncu_rc=$?
python tools/launch_summary.py $O/launches.csv > $O/launches_summary.txt 2>&1
tail -3 $O/pytest.log; tail -4 $O/smoke.log; tail -c 2000 $O/bench.log; echo; tail -1 $O/bench_reference.log; cat $O/launches_summary.txt
python bench.py --cpu-ratio-vs-n $O/gpu_cpu_ratio.jsonl > $O/ratio.log 2>&1; echo ratio_rc=$?
