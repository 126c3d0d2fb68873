#!/bin/bash
# ncu --set full captures of the round-2 kernels beside the headline (details + raw pages)
O=gpurun_out/r02cap; mkdir -p $O
cap() {  # name regex func n C [algo] [m]
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$2 -c 1 -s 2 -o $O/$1 -f \
    python tools/prof_one.py $3 $4 $5 ${6:-hvp} ${7:-1048576} > $O/$1.log 2>&1
  ncu -i $O/$1.ncu-rep --page details > $O/$1_details.txt 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>&1
}
cap rb32 hvp_reg_kernel rosenbrock 32 16 hvp 262144
cap ack16 hvp_reg_kernel ackley 16 16
cap prod16 hvp_reg_kernel prodsum 16 16
cap f3n16 hvp_f3_mma_kernel fletcher_powell 16 16 hvp 262144
cap stream4 hvp_stream_kernel rosenbrock 4 4 hvp 16777216
ls $O
