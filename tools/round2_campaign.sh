#!/bin/bash
# Round-2 measurement campaign (one B200): ncu executed-FLOP tables (DMMA FLOPs counted) for the
# F3 tensor-core kernels at every config, event-timed sweeps of every config, the bench line.
set -x
O=gpurun_out/r02c2; mkdir -p $O
# ncu executed-FLOP / pipe tables of the kernels that changed this round
bash tools/ncu_executed.sh c2f3sym --n 16 --m 262144 --funcs fletcher_powell --algo sym_hvp > $O/ncu_c2f3sym.txt 2>&1
bash tools/ncu_executed.sh c2f3hoist --n 16 --m 262144 --funcs fletcher_powell --algo hvp_hoisted > $O/ncu_c2f3hoist.txt 2>&1
bash tools/ncu_executed.sh c4f3 --n 32 --m 65536 --funcs fletcher_powell --algo hessian --csizes 1 2 4 8 16 32 > $O/ncu_c4f3.txt 2>&1
bash tools/ncu_executed.sh c4f3sym --n 32 --m 65536 --funcs fletcher_powell --algo sym_hessian --csizes 1 2 4 8 16 32 > $O/ncu_c4f3sym.txt 2>&1
bash tools/ncu_executed.sh c3n64f3 --n 64 --m 16384 --funcs fletcher_powell --csizes 2 4 32 > $O/ncu_c3n64f3.txt 2>&1
bash tools/ncu_executed.sh c3n128f3 --n 128 --m 4096 --funcs fletcher_powell --csizes 1 8 32 128 > $O/ncu_c3n128f3.txt 2>&1
bash tools/ncu_executed.sh c1 --n 2 --m 1024 > $O/ncu_c1.txt 2>&1
bash tools/ncu_executed.sh stream4 --n 4 --m 4194304 --funcs rosenbrock ackley prodsum > $O/ncu_stream4.txt 2>&1
cp gpurun_out/executed_flops.json $O/
# event-timed sweeps
timeout 600 python tools/sweep_bench.py --n 2 --m 1024 --algo hvp > $O/time_cfg1.jsonl 2>&1
timeout 600 python tools/sweep_bench.py --n 16 --m 1048576 --algo hvp > $O/time_cfg2.jsonl 2>&1
timeout 600 python tools/sweep_bench.py --n 16 --m 1048576 --algo sym_hvp > $O/time_cfg2sym.jsonl 2>&1
timeout 900 python tools/sweep_bench.py --n 32 --m 262144 --algo hessian > $O/time_cfg4.jsonl 2>&1
timeout 900 python tools/sweep_bench.py --n 32 --m 262144 --algo sym_hessian > $O/time_cfg4sym.jsonl 2>&1
timeout 1500 python tools/sweep_bench.py --n 64 --m 1048576 --algo hvp --f3-m 131072 > $O/time_cfg3n64.jsonl 2>&1
timeout 1200 python tools/sweep_bench.py --n 64 --m 131072 --algo sym_hvp --funcs fletcher_powell > $O/time_cfg3n64sym.jsonl 2>&1
timeout 2400 python tools/sweep_bench.py --n 128 --m 1048576 --algo hvp --f3-m 65536 --min-seconds 0.1 > $O/time_cfg3n128.jsonl 2>&1
timeout 1200 python tools/sweep_bench.py --n 128 --m 65536 --algo sym_hvp --funcs fletcher_powell --csizes 8 16 32 --min-seconds 0.1 > $O/time_cfg3n128sym.jsonl 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1
cp gpurun_out/bench_sweep.json $O/
tail -1 $O/bench.log
