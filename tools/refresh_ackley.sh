#!/bin/bash
# evidence after the Ackley volatile-seed policy: ncu entries + sweeps of Ackley n >= 32, GPU suite
set -x
O=gpurun_out/r02a2; mkdir -p $O
cp profiles/executed_flops.json gpurun_out/executed_flops.json
X="bash tools/ncu_executed.sh"
$X an32 --n 32 --m 262144 --funcs ackley --csizes 1 2 4 8 16 32 > $O/ncu_an32.txt 2>&1
$X ac4 --n 32 --m 65536 --funcs ackley --algo hessian --csizes 1 2 4 8 16 32 > $O/ncu_ac4.txt 2>&1
$X an64 --n 64 --m 65536 --funcs ackley --csizes 1 2 4 8 16 32 64 > $O/ncu_an64.txt 2>&1
cp gpurun_out/executed_flops.json $O/
mv gpurun_out/sweep_* $O/ 2>/dev/null
S="python tools/sweep_bench.py --funcs ackley"
timeout 900 $S --n 32 --m 262144 --algo hvp > $O/time_n32.jsonl 2>&1
timeout 900 $S --n 32 --m 262144 --algo hessian > $O/time_cfg4.jsonl 2>&1
timeout 1500 $S --n 64 --m 1048576 --algo hvp > $O/time_cfg3n64.jsonl 2>&1
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?
tail -3 $O/pytest.log; cat $O/time_n32.jsonl $O/time_cfg4.jsonl $O/time_cfg3n64.jsonl | cut -c1-120
