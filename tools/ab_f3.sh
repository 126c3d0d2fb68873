#!/bin/bash
# A/B timing of library builds on the per-evaluation F3 path at n = 64 / 128 (tuning experiments).
O=$1; shift
mkdir -p $O
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  export CHESSFAD_LIB=$lib
  timeout 300 python tools/sweep_bench.py --n 64 --m 16384 --algo hvp --funcs fletcher_powell --csizes 8 64 > $O/${name}_n64.jsonl 2>&1
  timeout 300 python tools/sweep_bench.py --n 128 --m 2048 --algo hvp --funcs fletcher_powell --csizes 16 128 > $O/${name}_n128.jsonl 2>&1
done
unset CHESSFAD_LIB
