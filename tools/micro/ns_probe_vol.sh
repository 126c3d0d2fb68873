nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/micro/ns_probe.cu -o /tmp/nsp && /tmp/nsp | tee gpurun_out/ns_probe_vol16.txt
