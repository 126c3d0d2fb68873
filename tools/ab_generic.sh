#!/bin/bash
# Generic A/B of library builds on the register-path configs: bash tools/ab_generic.sh OUT name=lib ...
O=$1; shift
mkdir -p $O
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  export CHESSFAD_LIB=$lib
  timeout 300 python tools/sweep_bench.py --n 16 --m 1048576 --algo hvp --funcs rosenbrock ackley prodsum > $O/${name}_n16.jsonl 2>&1
  timeout 300 python tools/sweep_bench.py --n 8 --m 1048576 --algo hvp --funcs rosenbrock ackley > $O/${name}_n8.jsonl 2>&1
  timeout 300 python tools/sweep_bench.py --n 64 --m 262144 --algo hvp --funcs rosenbrock ackley prodsum --csizes 8 16 > $O/${name}_n64.jsonl 2>&1
  timeout 300 python tools/sweep_bench.py --n 32 --m 262144 --algo hessian --funcs rosenbrock ackley --csizes 8 16 > $O/${name}_n32h.jsonl 2>&1
  timeout 300 python tools/sweep_bench.py --n 16 --m 1048576 --algo sym_hvp --funcs rosenbrock --csizes 4 8 > $O/${name}_n16s.jsonl 2>&1
done
unset CHESSFAD_LIB
