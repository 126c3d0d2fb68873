#!/bin/bash
# Evidence refresh after the stream-kernel change: ncu executed-FLOP entries and event-timed
# sweeps of the stream configs, then the GPU suite, smoke and the bench line.
set -x
O=gpurun_out/r02${1:-s}; mkdir -p $O
cp profiles/executed_flops.json gpurun_out/executed_flops.json
X="bash tools/ncu_executed.sh"
$X stream4 --n 4 --m 4194304 --funcs rosenbrock ackley prodsum --csizes 1 2 4 > $O/ncu_stream4.txt 2>&1
$X stream2 --n 2 --m 4194304 --funcs rosenbrock ackley prodsum --csizes 1 2 > $O/ncu_stream2.txt 2>&1
$X stream8 --n 8 --m 1048576 --funcs prodsum --csizes 1 2 4 8 > $O/ncu_stream8.txt 2>&1
$X c1 --n 2 --m 1024 > $O/ncu_c1.txt 2>&1
cp gpurun_out/executed_flops.json $O/
mv gpurun_out/sweep_* $O/ 2>/dev/null
S="python tools/sweep_bench.py"
timeout 600 $S --n 2 --m 1024 --algo hvp > $O/time_cfg1.jsonl 2>&1
timeout 600 $S --n 2 --m 16777216 --algo hvp > $O/time_n2_hbm.jsonl 2>&1
timeout 600 $S --n 4 --m 16777216 --algo hvp > $O/time_n4_hbm.jsonl 2>&1
timeout 600 $S --n 8 --m 1048576 --algo hvp > $O/time_n8.jsonl 2>&1
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.log 2>&1; echo bench_rc=$?
cp gpurun_out/bench_sweep.json $O/ 2>/dev/null
tail -3 $O/pytest.log; tail -c 1500 $O/bench.log
