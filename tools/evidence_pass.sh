#!/bin/bash
# End-of-round evidence pass (one B200): GPU suite, smoke, the driver's bench command, the ncu
# launch list of the bench command, a full ncu capture of the headline kernel, the paper-levels
# comparison.  usage: bash tools/evidence_pass.sh TAG
set -x
T=${1:-final}; O=gpurun_out/r02$T; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
# executed-FLOP entries of kernels changed since the campaign (F3 seed-sparse modes, F3 Alg 8 n > 64)
bash tools/ncu_executed.sh f3sp16 --n 16 --m 262144 --funcs fletcher_powell --algo hvp_seedsparse > $O/ncu_f3sp16.txt 2>&1
bash tools/ncu_executed.sh f3sym128 --n 128 --m 4096 --funcs fletcher_powell --algo sym_hvp --csizes 8 16 32 > $O/ncu_f3sym128.txt 2>&1
cp gpurun_out/executed_flops.json $O/ 2>/dev/null
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.log 2>&1; echo bench_rc=$?
cp gpurun_out/bench_sweep.json $O/ 2>/dev/null
python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > $O/bench_reference.log 2>&1; echo ref_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-strong --e2e-steps 1 > $O/bench_ncu.log 2>&1; echo ncu_rc=$?
python tools/launch_summary.py $O/launches.csv > $O/launches_summary.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hvp_reg_kernel -c 1 -s 2 -o $O/prof_headline -f \
  python tools/prof_one.py rosenbrock 16 16 > $O/prof_headline.log 2>&1; echo prof_rc=$?
timeout 600 python tools/paper_levels_bench.py > $O/paper_levels.jsonl 2>&1
tail -4 $O/pytest.log; cat $O/smoke.log | tail -4; tail -c 1200 $O/bench.log; echo; tail -1 $O/bench_reference.log; cat $O/launches_summary.txt
