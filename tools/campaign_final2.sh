#!/bin/bash
# Final pass of the round on the committed build.
set -x
O=gpurun_out/final2
mkdir -p $O
cp profiles/executed_flops.json gpurun_out/executed_flops.json
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
bash tools/ncu_executed.sh sparse16 --n 16 --m 1048576 --funcs fletcher_powell --csizes 1 4 16 --algo hvp_seedsparse
bash tools/ncu_executed.sh sparse32 --n 32 --m 262144 --funcs fletcher_powell --csizes 32 --algo hvp_seedsparse
bash tools/ncu_executed.sh sparseh32 --n 32 --m 262144 --funcs fletcher_powell --csizes 32 --algo hessian_seedsparse
mv gpurun_out/sweep_* $O/ 2>/dev/null
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
