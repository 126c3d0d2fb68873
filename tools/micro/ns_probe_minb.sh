#!/bin/bash
# compiled-n kernels of the probe at min-CTAs-per-SM bounds 1..4 (register cap 255/128/168/128)
O=gpurun_out/ns_probe_minb; mkdir -p $O
for mb in 1 2 3 4; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DCHF_REG_MINB=$mb tools/micro/ns_probe.cu -o /tmp/nsm$mb && /tmp/nsm$mb
done 2>&1 | tee $O/probe.txt
