#!/bin/bash
# A/B of two library builds over every register-path family (per-evaluation, hoisted, stream,
# symmetric, Hessian, seed-sparse).  usage: bash tools/ab_seed.sh OUTDIR name1=lib1.so name2=lib2.so
O=$1; shift
mkdir -p $O
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  export CHESSFAD_LIB=$lib
  S="timeout 300 python tools/sweep_bench.py --min-seconds 0.2"
  $S --n 16 --m 1048576 --algo hvp --funcs rosenbrock ackley prodsum > $O/${name}_n16.jsonl 2>&1
  $S --n 8 --m 1048576 --algo hvp --funcs rosenbrock ackley prodsum > $O/${name}_n8.jsonl 2>&1
  $S --n 4 --m 16777216 --algo hvp --funcs rosenbrock ackley prodsum > $O/${name}_n4.jsonl 2>&1
  $S --n 2 --m 16777216 --algo hvp --funcs rosenbrock ackley prodsum > $O/${name}_n2.jsonl 2>&1
  $S --n 64 --m 131072 --algo hvp --funcs rosenbrock ackley prodsum --csizes 4 8 16 > $O/${name}_n64.jsonl 2>&1
  $S --n 32 --m 65536 --algo hessian --funcs rosenbrock ackley prodsum --csizes 4 16 > $O/${name}_n32h.jsonl 2>&1
  $S --n 16 --m 1048576 --algo sym_hvp --funcs rosenbrock ackley prodsum --csizes 2 4 8 > $O/${name}_n16s.jsonl 2>&1
  $S --n 16 --m 1048576 --algo hvp_hoisted --funcs rosenbrock ackley prodsum > $O/${name}_n16hz.jsonl 2>&1
  $S --n 8 --m 1048576 --algo hvp_hoisted --funcs rosenbrock ackley prodsum > $O/${name}_n8hz.jsonl 2>&1
  $S --n 64 --m 1048576 --algo hvp_seedsparse --funcs rosenbrock ackley prodsum --csizes 4 16 > $O/${name}_n64sp.jsonl 2>&1
done
unset CHESSFAD_LIB
python tools/ab_compare.py $O ${1%%=*} ${2%%=*} > $O/summary.txt; cat $O/summary.txt
