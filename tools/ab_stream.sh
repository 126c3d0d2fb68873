#!/bin/bash
# A/B of the n in {2,4,8} Alg 7 kernels: stream (default build) vs runtime-n register path.
#   bash tools/ab_stream.sh OUTDIR new=lib.so old=lib_nostream.so
O=$1; shift
mkdir -p $O
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  export CHESSFAD_LIB=$lib
  for n in 2 4 8; do
    timeout 300 python tools/sweep_bench.py --n $n --m 16777216 --algo hvp --funcs rosenbrock ackley prodsum > $O/${name}_n$n.jsonl 2>&1
  done
done
unset CHESSFAD_LIB
