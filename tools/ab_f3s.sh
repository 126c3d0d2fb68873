#!/bin/bash
# A/B timing on the per-evaluation F3 path with (A, B) in shared memory (n <= 32).
O=$1; shift
mkdir -p $O
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  export CHESSFAD_LIB=$lib
  timeout 300 python tools/sweep_bench.py --n 16 --m 1048576 --algo hvp --funcs fletcher_powell --csizes 1 4 16 > $O/${name}_n16.jsonl 2>&1
  timeout 300 python tools/sweep_bench.py --n 32 --m 262144 --algo hessian --funcs fletcher_powell --csizes 4 32 > $O/${name}_n32h.jsonl 2>&1
  timeout 300 python tools/sweep_bench.py --n 8 --m 1048576 --algo hvp --funcs fletcher_powell --csizes 8 > $O/${name}_n8.jsonl 2>&1
done
unset CHESSFAD_LIB
