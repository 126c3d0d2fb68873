#!/bin/bash
# A/B of the stream kernel (n in {2, 4}, prodsum n = 8) between two builds, m = 2^24
O=gpurun_out/ab_stream2; mkdir -p $O
for spec in "$@"; do
  name=${spec%%=*}; export CHESSFAD_LIB=${spec#*=}
  for n in 2 4; do timeout 600 python tools/sweep_bench.py --n $n --m 16777216 --algo hvp --funcs rosenbrock ackley prodsum --min-seconds 0.3 > $O/${name}_n$n.jsonl 2>&1; done
  timeout 600 python tools/sweep_bench.py --n 8 --m 4194304 --algo hvp --funcs prodsum --min-seconds 0.3 > $O/${name}_n8.jsonl 2>&1
done
unset CHESSFAD_LIB
python tools/ab_compare.py $O ${1%%=*} ${2%%=*} | tee $O/summary.txt
