#!/bin/bash
# Measure executed FP64 FLOPs / pipe utilisation per (func, C) for the current build and
# write gpurun_out/executed_flops.json (+ copy to profiles/ on the box for bench.py).
# usage: tools/ncu_executed.sh [tag] [profile_sweep args...]
TAG=${1:-cfg2}; shift
M="sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"
mkdir -p gpurun_out
[ -f gpurun_out/executed_flops.json ] || cp profiles/executed_flops.json gpurun_out/executed_flops.json 2>/dev/null
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/sweep_metrics_$TAG.csv python tools/profile_sweep.py "$@" > gpurun_out/sweep_order_$TAG.txt 2>&1
python tools/summarize_sweep.py gpurun_out/sweep_metrics_$TAG.csv gpurun_out/sweep_order_$TAG.txt gpurun_out/sweep_$TAG.json gpurun_out/executed_flops.json > gpurun_out/sweep_$TAG.txt
cp gpurun_out/executed_flops.json profiles/executed_flops.json
cat gpurun_out/sweep_$TAG.txt
