#!/bin/bash
# Round-1 measurement campaign (one B200): ncu executed-FLOP tables + event-timed sweeps.
set -x
O=gpurun_out
# ncu executed-FLOP / pipe tables
bash tools/ncu_executed.sh cfg2 --n 16 --m 1048576
bash tools/ncu_executed.sh cfg2sym --n 16 --m 1048576 --algo sym_hvp
bash tools/ncu_executed.sh cfg4 --n 32 --m 262144 --algo hessian --csizes 1 2 4 8 16 32
bash tools/ncu_executed.sh cfg4sym --n 32 --m 262144 --algo sym_hessian --csizes 1 2 4 8 16 32
bash tools/ncu_executed.sh cfg3n64 --n 64 --m 262144 --funcs rosenbrock ackley prodsum --csizes 1 2 4 8 16 32 64
bash tools/ncu_executed.sh cfg3n64f3 --n 64 --m 16384 --funcs fletcher_powell --csizes 1 4 16 64
bash tools/ncu_executed.sh cfg3n128 --n 128 --m 65536 --funcs rosenbrock ackley prodsum --csizes 1 2 4 8 16 32 64 128
bash tools/ncu_executed.sh cfg3n128f3 --n 128 --m 4096 --funcs fletcher_powell --csizes 1 8 32 128
# event-timed sweeps (full m except F3 at n = 64/128)
timeout 600 python tools/sweep_bench.py --n 16 --m 1048576 --algo hvp > $O/time_cfg2.jsonl
timeout 600 python tools/sweep_bench.py --n 16 --m 1048576 --algo sym_hvp > $O/time_cfg2sym.jsonl
timeout 900 python tools/sweep_bench.py --n 32 --m 262144 --algo hessian > $O/time_cfg4.jsonl
timeout 900 python tools/sweep_bench.py --n 32 --m 262144 --algo sym_hessian > $O/time_cfg4sym.jsonl
timeout 1200 python tools/sweep_bench.py --n 64 --m 1048576 --algo hvp --f3-m 65536 > $O/time_cfg3n64.jsonl
timeout 1500 python tools/sweep_bench.py --n 128 --m 1048576 --algo hvp --f3-m 8192 --min-seconds 0.1 > $O/time_cfg3n128.jsonl
timeout 600 python bench.py --steps 100 --warmup 5 > $O/bench4.json 2> $O/bench4.err
