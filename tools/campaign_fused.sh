#!/bin/bash
# Measurement campaign for the fused-accumulate build (register path F1/F2/F4 changed; F3
# kernels' SASS unchanged, their executed-FLOP entries stay valid by SASS hash).
set -x
O=gpurun_out
mkdir -p $O
rm -f $O/executed_flops.json
timeout 900 python -m pytest tests -m gpu -q > $O/final_pytest.log 2>&1; tail -3 $O/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
R="rosenbrock ackley prodsum"
bash tools/ncu_executed.sh cfg2 --n 16 --m 1048576 --funcs $R
bash tools/ncu_executed.sh cfg1n2 --n 2 --m 1048576 --funcs $R
bash tools/ncu_executed.sh smalln4 --n 4 --m 1048576 --funcs $R
bash tools/ncu_executed.sh smalln8 --n 8 --m 1048576 --funcs $R
bash tools/ncu_executed.sh cfg2sym --n 16 --m 262144 --algo sym_hvp --funcs $R
bash tools/ncu_executed.sh cfg2hoist --n 16 --m 1048576 --algo hvp_hoisted --funcs $R
bash tools/ncu_executed.sh n8hoist --n 8 --m 1048576 --algo hvp_hoisted --funcs $R
bash tools/ncu_executed.sh cfg4 --n 32 --m 65536 --algo hessian --csizes 1 2 4 8 16 32 --funcs $R
bash tools/ncu_executed.sh cfg4sym --n 32 --m 65536 --algo sym_hessian --csizes 1 2 4 8 16 32 --funcs $R
bash tools/ncu_executed.sh cfg3n64 --n 64 --m 131072 --funcs $R --csizes 1 2 4 8 16 32 64
bash tools/ncu_executed.sh cfg3n128 --n 128 --m 65536 --funcs $R --csizes 1 2 4 8 16 32 64 128
timeout 600 python tools/sweep_bench.py --n 2 --m 1048576 --algo hvp > $O/time_n2.jsonl
timeout 600 python tools/sweep_bench.py --n 4 --m 1048576 --algo hvp > $O/time_n4.jsonl
timeout 600 python tools/sweep_bench.py --n 8 --m 1048576 --algo hvp > $O/time_n8.jsonl
timeout 600 python tools/sweep_bench.py --n 16 --m 1048576 --algo hvp > $O/time_cfg2.jsonl
timeout 600 python tools/sweep_bench.py --n 16 --m 1048576 --algo sym_hvp > $O/time_cfg2sym.jsonl
timeout 600 python tools/sweep_bench.py --n 16 --m 1048576 --algo hvp_hoisted > $O/time_cfg2hoist.jsonl
timeout 600 python tools/sweep_bench.py --n 8 --m 1048576 --algo hvp_hoisted > $O/time_n8hoist.jsonl
timeout 900 python tools/sweep_bench.py --n 32 --m 262144 --algo hessian > $O/time_cfg4.jsonl
timeout 900 python tools/sweep_bench.py --n 32 --m 262144 --algo sym_hessian > $O/time_cfg4sym.jsonl
timeout 1200 python tools/sweep_bench.py --n 64 --m 1048576 --algo hvp --funcs $R > $O/time_cfg3n64.jsonl
timeout 1500 python tools/sweep_bench.py --n 128 --m 1048576 --algo hvp --funcs $R --min-seconds 0.1 > $O/time_cfg3n128.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --e2e-steps 1 > $O/launches_bench_out.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hvp_reg -c 1 -o $O/prof_headline python tools/profile_sweep.py --funcs rosenbrock --csizes 16 > /dev/null 2>&1
timeout 600 python bench.py > $O/bench_final.json 2> $O/bench_final.err
timeout 300 python tools/e2e_probe.py > $O/e2e_probe_final.jsonl 2>&1
timeout 600 python tools/paper_levels_bench.py > $O/paper_levels_final.jsonl 2>&1
ls $O
