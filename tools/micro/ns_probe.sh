#!/bin/bash
# the compiled-n register kernels (n = 32 / 64): chunk-loop unroll bound (CHF_NS_CHUNK_UNROLL)
O=gpurun_out/ns_probe2; mkdir -p $O
for u in 1 2 4 8; do
  echo "== CHF_NS_CHUNK_UNROLL=$u"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DCHF_NS_CHUNK_UNROLL=$u tools/micro/ns_probe.cu -o /tmp/nsu$u && /tmp/nsu$u
done 2>&1 | tee $O/probe.txt
