#!/bin/bash
# Ackley n = 128, kernel chunk 8 on the compiled-n kernel: tests, ncu entry, sweep
set -x
O=gpurun_out/r02a4; mkdir -p $O
cp profiles/executed_flops.json gpurun_out/executed_flops.json
python -m pytest tests/test_gpu_parity.py -q -k "large_n or small_m" > $O/pytest.log 2>&1; echo pytest_rc=$?
bash tools/ncu_executed.sh an128 --n 128 --m 16384 --funcs ackley --csizes 8 > $O/ncu_an128.txt 2>&1
cp gpurun_out/executed_flops.json $O/
mv gpurun_out/sweep_* $O/ 2>/dev/null
timeout 2400 python tools/sweep_bench.py --n 128 --m 1048576 --algo hvp --funcs ackley --min-seconds 0.1 > $O/time_cfg3n128.jsonl 2>&1
tail -2 $O/pytest.log; cut -c1-110 $O/time_cfg3n128.jsonl
