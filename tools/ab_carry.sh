#!/bin/bash
# A/B of two builds on the families touched by the seed carry (Rosenbrock, prodsum) and the
# F3 structural-zero change.  usage: bash tools/ab_carry.sh OUTDIR a=liba.so b=libb.so
O=$1; shift
mkdir -p $O
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  export CHESSFAD_LIB=$lib
  S="timeout 300 python tools/sweep_bench.py --min-seconds 0.2"
  $S --n 16 --m 1048576 --algo hvp --funcs rosenbrock prodsum fletcher_powell > $O/${name}_n16.jsonl 2>&1
  $S --n 8 --m 1048576 --algo hvp --funcs rosenbrock prodsum > $O/${name}_n8.jsonl 2>&1
  $S --n 4 --m 16777216 --algo hvp --funcs rosenbrock prodsum > $O/${name}_n4.jsonl 2>&1
  $S --n 2 --m 16777216 --algo hvp --funcs rosenbrock prodsum > $O/${name}_n2.jsonl 2>&1
  $S --n 64 --m 131072 --algo hvp --funcs rosenbrock prodsum --csizes 4 16 > $O/${name}_n64.jsonl 2>&1
  $S --n 64 --m 16384 --algo hvp --funcs fletcher_powell --csizes 8 64 > $O/${name}_n64f3.jsonl 2>&1
  $S --n 32 --m 65536 --algo hessian --funcs rosenbrock prodsum fletcher_powell --csizes 4 16 32 > $O/${name}_n32h.jsonl 2>&1
  $S --n 16 --m 1048576 --algo sym_hvp --funcs rosenbrock prodsum fletcher_powell --csizes 4 8 > $O/${name}_n16s.jsonl 2>&1
  $S --n 16 --m 1048576 --algo hvp_hoisted --funcs rosenbrock prodsum > $O/${name}_n16hz.jsonl 2>&1
done
unset CHESSFAD_LIB
python tools/ab_compare.py $O ${1%%=*} ${2%%=*} > $O/summary.txt; cat $O/summary.txt
