#!/bin/bash
# Last evidence pass of the round: GPU suite, smoke, executed-FLOP entries of the (fixed) staged
# seed-sparse kernel, its timings, bench line.
set -x
O=gpurun_out/last
mkdir -p $O
cp profiles/executed_flops.json gpurun_out/executed_flops.json
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
bash tools/ncu_executed.sh sparse64 --n 64 --m 65536 --funcs fletcher_powell --csizes 64 --algo hvp_seedsparse
bash tools/ncu_executed.sh sparse128 --n 128 --m 16384 --funcs fletcher_powell --csizes 128 --algo hvp_seedsparse
bash tools/ncu_executed.sh sparseh32 --n 32 --m 262144 --funcs fletcher_powell --csizes 32 --algo hessian_seedsparse
for n in 64 128; do
  timeout 600 python tools/sweep_bench.py --n $n --m 1048576 --algo hvp_seedsparse --funcs fletcher_powell > $O/time_sparse_n$n.jsonl 2>&1
done
mv gpurun_out/sweep_* $O/ 2>/dev/null
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
