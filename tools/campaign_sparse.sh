#!/bin/bash
# Seed-sparse F3 measurements (NEXT-4) + GPU suite for the current build.
set -x
O=gpurun_out
mkdir -p $O/sparse
cp profiles/executed_flops.json $O/executed_flops.json
timeout 900 python -m pytest tests -m gpu -q > $O/sparse/pytest.log 2>&1; tail -3 $O/sparse/pytest.log
bash tools/ncu_executed.sh sparse16 --n 16 --m 1048576 --funcs fletcher_powell --csizes 1 16 --algo hvp_seedsparse
bash tools/ncu_executed.sh sparse32 --n 32 --m 262144 --funcs fletcher_powell --csizes 32 --algo hvp_seedsparse
bash tools/ncu_executed.sh sparse64 --n 64 --m 65536 --funcs fletcher_powell --csizes 64 --algo hvp_seedsparse
bash tools/ncu_executed.sh sparse128 --n 128 --m 16384 --funcs fletcher_powell --csizes 128 --algo hvp_seedsparse
bash tools/ncu_executed.sh sparseh32 --n 32 --m 262144 --funcs fletcher_powell --csizes 32 --algo hessian_seedsparse
for n in 2 4 8 16 32 64 128; do
  timeout 600 python tools/sweep_bench.py --n $n --m 1048576 --algo hvp_seedsparse --funcs fletcher_powell > $O/sparse/time_sparse_n$n.jsonl 2>&1
done
timeout 600 python tools/sweep_bench.py --n 32 --m 262144 --algo hessian_seedsparse --funcs fletcher_powell > $O/sparse/time_sparse_hess_n32.jsonl 2>&1
mv $O/sweep_*sparse* $O/sparse/ 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/sparse/smoke.log 2>&1
