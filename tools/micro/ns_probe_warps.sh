#!/bin/bash
# compiled-n kernels of the probe at 2 / 4 / 8 warps per CTA (CHF_WARPS_REG)
O=gpurun_out/ns_probe_warps; mkdir -p $O
for w in 2 4 8; do
  echo "== CHF_WARPS_REG=$w"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DCHF_WARPS_REG=$w tools/micro/ns_probe.cu -o /tmp/nsw$w && /tmp/nsw$w
done 2>&1 | tee $O/probe.txt
