#!/bin/bash
# register-kernel probe at several min-CTAs-per-SM bounds (CHF_REG_MINB)
O=gpurun_out/${1:-probe_mb}; mkdir -p $O
for mb in 1 3 4; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include -DCHF_REG_MINB=$mb tools/micro/reg_probe.cu -o /tmp/reg_probe_$mb || exit 1
  echo "== CHF_REG_MINB=$mb"; /tmp/reg_probe_$mb | grep -E "lib|zseed "
done 2>&1 | tee $O/probe.txt
