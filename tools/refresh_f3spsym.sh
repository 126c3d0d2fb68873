#!/bin/bash
# F3 seed-sparse Alg 8: ncu executed-FLOP entries and event-timed sweeps
set -x
O=gpurun_out/r02sp8; mkdir -p $O
cp profiles/executed_flops.json gpurun_out/executed_flops.json
bash tools/ncu_executed.sh f3sp8_16 --n 16 --m 262144 --funcs fletcher_powell --algo sym_hvp_seedsparse > $O/ncu_16.txt 2>&1
bash tools/ncu_executed.sh f3sp8_64 --n 64 --m 16384 --funcs fletcher_powell --algo sym_hvp_seedsparse --csizes 1 8 64 > $O/ncu_64.txt 2>&1
cp gpurun_out/executed_flops.json $O/
mv gpurun_out/sweep_* $O/ 2>/dev/null
S="python tools/sweep_bench.py --funcs fletcher_powell"
$S --n 16 --m 1048576 --algo sym_hvp_seedsparse > $O/time_16_sym.jsonl 2>&1
$S --n 16 --m 1048576 --algo hvp_seedsparse > $O/time_16.jsonl 2>&1
$S --n 32 --m 262144 --algo sym_hvp_seedsparse > $O/time_32_sym.jsonl 2>&1
$S --n 32 --m 262144 --algo hvp_seedsparse > $O/time_32.jsonl 2>&1
$S --n 64 --m 131072 --algo sym_hvp_seedsparse --csizes 1 8 64 > $O/time_64_sym.jsonl 2>&1
$S --n 64 --m 131072 --algo hvp_seedsparse --csizes 1 8 64 > $O/time_64.jsonl 2>&1
cat $O/time_*.jsonl | cut -c1-110
