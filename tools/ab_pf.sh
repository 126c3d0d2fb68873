#!/bin/bash
# A/B of the register path: persistent prefetching kernel (default) vs one CTA per tile.
#   bash tools/ab_pf.sh OUTDIR new=lib.so old=lib_nopf.so
O=$1; shift
mkdir -p $O
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  export CHESSFAD_LIB=$lib
  timeout 300 python tools/sweep_bench.py --n 16 --m 1048576 --algo hvp --funcs rosenbrock ackley prodsum > $O/${name}_n16.jsonl 2>&1
  timeout 300 python tools/sweep_bench.py --n 8 --m 1048576 --algo hvp --funcs rosenbrock ackley > $O/${name}_n8.jsonl 2>&1
  timeout 300 python tools/sweep_bench.py --n 64 --m 262144 --algo hvp --funcs rosenbrock ackley prodsum --csizes 4 8 16 > $O/${name}_n64.jsonl 2>&1
  timeout 300 python tools/sweep_bench.py --n 32 --m 131072 --algo hessian --funcs rosenbrock ackley --csizes 4 16 > $O/${name}_n32h.jsonl 2>&1
  timeout 300 python tools/sweep_bench.py --n 16 --m 1048576 --algo sym_hvp --funcs rosenbrock ackley --csizes 2 4 8 > $O/${name}_n16s.jsonl 2>&1
done
unset CHESSFAD_LIB
