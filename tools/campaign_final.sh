#!/bin/bash
# End-of-round evidence for the committed build: GPU suite, smoke, executed-FLOP entries of the
# staged seed-sparse kernels, sparse sweeps, launch list + bench line.
set -x
O=gpurun_out/final
mkdir -p $O
cp profiles/executed_flops.json gpurun_out/executed_flops.json
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
bash tools/ncu_executed.sh sparse64 --n 64 --m 65536 --funcs fletcher_powell --csizes 64 --algo hvp_seedsparse
bash tools/ncu_executed.sh sparse128 --n 128 --m 16384 --funcs fletcher_powell --csizes 128 --algo hvp_seedsparse
for n in 64 128; do
  timeout 600 python tools/sweep_bench.py --n $n --m 1048576 --algo hvp_seedsparse --funcs fletcher_powell > $O/time_sparse_n$n.jsonl 2>&1
done
mv gpurun_out/sweep_*sparse* $O/ 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --e2e-steps 1 > $O/launches_bench_out.json 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
