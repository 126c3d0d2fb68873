#!/bin/bash
# Final re-measurement after the per-function volatile-seed / unrolled-chunk policy of the
# compiled-n register kernels (Rosenbrock): ncu executed-FLOP tables, event-timed sweeps of
# every config, GPU suite, smoke, bench (+ reference arm), launch list, headline ncu capture,
# paper-levels comparison.  One B200.   usage: bash tools/round2_final3.sh [TAG]
set -x
T=${1:-f4}; O=gpurun_out/r02$T; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
cp profiles/executed_flops.json gpurun_out/executed_flops.json
X="bash tools/ncu_executed.sh"
# ---- ncu executed-FLOP / pipe tables: the Rosenbrock kernels changed by the volatile-seed /
# unrolled-chunk policy (every other family's SASS is unchanged since r02f3 / r02s)
$X rn8 --n 8 --m 1048576 --funcs rosenbrock --csizes 1 2 4 8 > $O/ncu_rn8.txt 2>&1
$X rn16 --n 16 --m 1048576 --funcs rosenbrock > $O/ncu_rn16.txt 2>&1
$X rn16sym --n 16 --m 1048576 --funcs rosenbrock --algo sym_hvp > $O/ncu_rn16sym.txt 2>&1
$X rn32 --n 32 --m 262144 --funcs rosenbrock --csizes 1 2 4 8 16 32 > $O/ncu_rn32.txt 2>&1
$X rc4 --n 32 --m 65536 --funcs rosenbrock --algo hessian --csizes 1 2 4 8 16 32 > $O/ncu_rc4.txt 2>&1
$X rc4sym --n 32 --m 65536 --funcs rosenbrock --algo sym_hessian --csizes 1 2 4 8 16 32 > $O/ncu_rc4sym.txt 2>&1
$X rn64 --n 64 --m 65536 --funcs rosenbrock --csizes 1 2 4 8 16 32 64 > $O/ncu_rn64.txt 2>&1
$X rn128 --n 128 --m 16384 --funcs rosenbrock --csizes 1 2 4 8 16 32 64 128 > $O/ncu_rn128.txt 2>&1
cp gpurun_out/executed_flops.json $O/
mv gpurun_out/sweep_* $O/ 2>/dev/null
# ---- event-timed sweeps
S="python tools/sweep_bench.py"
timeout 600 $S --n 2 --m 1024 --algo hvp > $O/time_cfg1.jsonl 2>&1
timeout 600 $S --n 2 --m 16777216 --algo hvp > $O/time_n2_hbm.jsonl 2>&1
timeout 600 $S --n 4 --m 16777216 --algo hvp > $O/time_n4_hbm.jsonl 2>&1
timeout 600 $S --n 8 --m 1048576 --algo hvp > $O/time_n8.jsonl 2>&1
timeout 600 $S --n 16 --m 1048576 --algo hvp > $O/time_cfg2.jsonl 2>&1
timeout 600 $S --n 16 --m 1048576 --algo sym_hvp > $O/time_cfg2sym.jsonl 2>&1
timeout 600 $S --n 16 --m 1048576 --algo hvp_hoisted > $O/time_cfg2hoist.jsonl 2>&1
timeout 600 $S --n 16 --m 1048576 --algo hvp_seedsparse > $O/time_cfg2sp.jsonl 2>&1
timeout 900 $S --n 32 --m 262144 --algo hvp > $O/time_n32.jsonl 2>&1
timeout 900 $S --n 32 --m 262144 --algo hessian > $O/time_cfg4.jsonl 2>&1
timeout 900 $S --n 32 --m 262144 --algo sym_hessian > $O/time_cfg4sym.jsonl 2>&1
timeout 1500 $S --n 64 --m 1048576 --algo hvp --f3-m 131072 > $O/time_cfg3n64.jsonl 2>&1
timeout 1200 $S --n 64 --m 131072 --algo sym_hvp --funcs fletcher_powell > $O/time_cfg3n64sym.jsonl 2>&1
timeout 2400 $S --n 128 --m 1048576 --algo hvp --f3-m 65536 --min-seconds 0.1 > $O/time_cfg3n128.jsonl 2>&1
timeout 1200 $S --n 128 --m 65536 --algo sym_hvp --funcs fletcher_powell --csizes 8 16 32 --min-seconds 0.1 > $O/time_cfg3n128sym.jsonl 2>&1
# ---- suite, smoke, bench, reference arm, launch list, headline capture, paper levels
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
ncu -i $O/prof_headline.ncu-rep --page details > $O/prof_headline_details.txt 2>&1
ncu -i $O/prof_headline.ncu-rep --page raw --csv > $O/prof_headline_raw.csv 2>&1
ncu -i $O/prof_headline.ncu-rep --page source --csv --print-source sass > $O/prof_headline_source.csv 2>&1
timeout 600 python tools/paper_levels_bench.py > $O/paper_levels.jsonl 2>&1
tail -3 $O/pytest.log; tail -4 $O/smoke.log; tail -c 2000 $O/bench.log; echo; tail -1 $O/bench_reference.log; cat $O/launches_summary.txt
