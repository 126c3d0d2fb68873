#!/bin/bash
# Quick GPU health check of the current tree: GPU suite, smoke, headline bench.
O=gpurun_out/${1:-quick}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
python bench.py --steps 10 --warmup 3 --no-sweep > $O/bench.log 2>&1; echo bench_rc=$?
tail -3 $O/pytest.log; tail -4 $O/smoke.log; tail -c 2000 $O/bench.log
