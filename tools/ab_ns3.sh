#!/bin/bash
# three-way A/B of the register path: runtime-n only / compiled-n everywhere / the shipped build
# usage: bash tools/ab_ns3.sh OUTDIR a=liba.so b=libb.so c=libc.so
O=$1; shift
mkdir -p $O
for spec in "$@"; do
  name=${spec%%=*}; export CHESSFAD_LIB=${spec#*=}
  S="timeout 600 python tools/sweep_bench.py --min-seconds 0.15 --funcs rosenbrock ackley prodsum"
  $S --n 8 --m 1048576 --algo hvp > $O/${name}_n8.jsonl 2>&1
  $S --n 16 --m 1048576 --algo hvp > $O/${name}_n16.jsonl 2>&1
  $S --n 16 --m 1048576 --algo sym_hvp > $O/${name}_n16s.jsonl 2>&1
  $S --n 16 --m 262144 --algo hessian > $O/${name}_n16h.jsonl 2>&1
  $S --n 32 --m 262144 --algo hvp > $O/${name}_n32.jsonl 2>&1
  $S --n 32 --m 262144 --algo sym_hvp > $O/${name}_n32s.jsonl 2>&1
  $S --n 32 --m 262144 --algo hessian > $O/${name}_n32h.jsonl 2>&1
  $S --n 32 --m 262144 --algo sym_hessian > $O/${name}_n32sh.jsonl 2>&1
  $S --n 64 --m 262144 --algo hvp > $O/${name}_n64.jsonl 2>&1
  $S --n 128 --m 65536 --algo hvp > $O/${name}_n128.jsonl 2>&1
done
unset CHESSFAD_LIB
