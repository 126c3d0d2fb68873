#!/bin/bash
# compute-sanitizer over the round-2 kernels (tools/sanitize_ns.py) + the R7 device pin test
O=gpurun_out/r02san; mkdir -p $O
python -m pytest tests/test_gpu_hdual_pins.py -q > $O/pins.log 2>&1; echo pins_rc=$?
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t python tools/sanitize_ns.py > $O/$t.txt 2>&1; echo ${t}_rc=$?
  tail -2 $O/$t.txt
done
tail -2 $O/pins.log
