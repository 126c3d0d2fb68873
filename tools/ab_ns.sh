#!/bin/bash
# A/B: runtime-n register kernel vs the kernels compiled for n in {8, 16, 32}
# usage: bash tools/ab_ns.sh OUTDIR a=liba.so b=libb.so
O=$1; shift
mkdir -p $O
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  export CHESSFAD_LIB=$lib
  S="timeout 300 python tools/sweep_bench.py --min-seconds 0.2"
  $S --n 16 --m 1048576 --algo hvp --funcs rosenbrock ackley prodsum > $O/${name}_n16.jsonl 2>&1
  $S --n 8 --m 1048576 --algo hvp --funcs rosenbrock ackley > $O/${name}_n8.jsonl 2>&1
  $S --n 32 --m 262144 --algo hvp --funcs rosenbrock ackley prodsum > $O/${name}_n32.jsonl 2>&1
  $S --n 32 --m 262144 --algo hessian --funcs rosenbrock ackley prodsum > $O/${name}_n32h.jsonl 2>&1
  $S --n 32 --m 262144 --algo sym_hessian --funcs rosenbrock ackley prodsum --csizes 4 16 > $O/${name}_n32sh.jsonl 2>&1
  $S --n 16 --m 1048576 --algo sym_hvp --funcs rosenbrock ackley prodsum > $O/${name}_n16s.jsonl 2>&1
done
unset CHESSFAD_LIB
python tools/ab_compare.py $O ${1%%=*} ${2%%=*} > $O/summary.txt; cat $O/summary.txt
