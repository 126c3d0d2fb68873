#!/bin/bash
# A/B timing of library builds on the seed-sparse F3 path (tuning experiments).
#   bash tools/ab_sparse.sh OUTDIR name1=lib1.so ...
O=$1; shift
mkdir -p $O
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  export CHESSFAD_LIB=$lib
  for n in 16 32 64 128; do
    timeout 300 python tools/sweep_bench.py --n $n --m 1048576 --algo hvp_seedsparse --funcs fletcher_powell --csizes $n > $O/${name}_n$n.jsonl 2>&1
  done
done
unset CHESSFAD_LIB
