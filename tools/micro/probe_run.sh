#!/bin/bash
# GPU side of the register-kernel probe: timings + one ncu source-level capture of the lib kernel.
O=gpurun_out/${1:-probe}; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include tools/micro/reg_probe.cu -o /tmp/reg_probe || exit 1
/tmp/reg_probe > $O/probe.txt 2>&1; cat $O/probe.txt
if [ "${2:-}" = "ncu" ]; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:hvp_reg_kernel -c 1 -s 2 -o $O/lib -f /tmp/reg_probe > $O/ncu.log 2>&1
  ncu -i $O/lib.ncu-rep --page source --csv --print-source sass > $O/lib_source.csv 2>&1
  ncu -i $O/lib.ncu-rep --page raw --csv > $O/lib_raw.csv 2>&1
  ls -la $O
fi
