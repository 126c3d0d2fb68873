#!/bin/bash
# Ackley n = 16, C = 16 at 3 CTAs/SM: sweeps of the modes, ncu entries, Ackley GPU tests
set -x
O=gpurun_out/r02a3; mkdir -p $O
cp profiles/executed_flops.json gpurun_out/executed_flops.json
X="bash tools/ncu_executed.sh"
$X a16 --n 16 --m 1048576 --funcs ackley --csizes 16 > $O/ncu_a16.txt 2>&1
$X a16sym --n 16 --m 1048576 --funcs ackley --csizes 16 --algo sym_hvp > $O/ncu_a16sym.txt 2>&1
cp gpurun_out/executed_flops.json $O/
mv gpurun_out/sweep_* $O/ 2>/dev/null
S="python tools/sweep_bench.py --funcs ackley"
$S --n 16 --m 1048576 --algo hvp > $O/time_cfg2.jsonl 2>&1
$S --n 16 --m 1048576 --algo sym_hvp > $O/time_cfg2sym.jsonl 2>&1
$S --n 16 --m 262144 --algo hessian > $O/time_n16h.jsonl 2>&1
python -m pytest tests -m gpu -q -k "ackley" > $O/pytest.log 2>&1; echo pytest_rc=$?
tail -2 $O/pytest.log; cat $O/time_*.jsonl | cut -c1-100
