#!/bin/bash
# Rosenbrock compiled for n = 64 / 128: chunk-loop unroll bound 4 / 8 / 16
O=gpurun_out/ns_probe_big; mkdir -p $O
for u in 4 8 16; do
  echo "== CHF_NS_CHUNK_UNROLL=$u"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DCHF_NS_CHUNK_UNROLL=$u tools/micro/ns_probe.cu -o /tmp/nsb$u && NS_PROBE_BIG=1 /tmp/nsb$u
done 2>&1 | tee $O/probe.txt
