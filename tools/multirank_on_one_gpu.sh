#!/bin/bash
# Exercise bench.py's N > 1 path (sharding, in-place result gather, max over ranks, per-rank
# clocks, the single JSON line) on a ONE-GPU box: both ranks on GPU 0, gloo instead of NCCL.
# A correctness check of the multi-rank logic only -- the timings are meaningless.
CHESSFAD_BENCH_ONE_GPU=1 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --e2e-steps 2 "$@"
