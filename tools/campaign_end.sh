#!/bin/bash
# End-of-round evidence for the committed build (round 1, last session).
set -x
O=gpurun_out/end2
mkdir -p $O
cp profiles/executed_flops.json gpurun_out/executed_flops.json
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
R="rosenbrock ackley prodsum"
bash tools/ncu_executed.sh cfg3n64f3 --n 64 --m 16384 --funcs fletcher_powell --csizes 1 4 16 64
bash tools/ncu_executed.sh cfg3n128f3 --n 128 --m 4096 --funcs fletcher_powell --csizes 1 8 32 128
bash tools/ncu_executed.sh spreg16 --n 16 --m 1048576 --funcs $R --csizes 2 4 --algo hvp_seedsparse
bash tools/ncu_executed.sh spreg64 --n 64 --m 262144 --funcs $R --csizes 2 4 8 --algo hvp_seedsparse
bash tools/ncu_executed.sh spreg128 --n 128 --m 131072 --funcs $R --csizes 2 4 64 --algo hvp_seedsparse
timeout 1200 python tools/sweep_bench.py --n 64 --m 65536 --algo hvp --funcs fletcher_powell > $O/time_cfg3n64f3.jsonl 2>&1
timeout 1500 python tools/sweep_bench.py --n 128 --m 8192 --algo hvp --funcs fletcher_powell --csizes 1 8 32 128 --min-seconds 0.1 > $O/time_cfg3n128f3.jsonl 2>&1
for n in 16 64 128; do
  timeout 600 python tools/sweep_bench.py --n $n --m 1048576 --algo hvp_seedsparse --funcs $R > $O/time_spreg_n$n.jsonl 2>&1
done
mv gpurun_out/sweep_* $O/ 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --e2e-steps 1 > $O/launches_bench_out.json 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
