#!/bin/bash
# Re-measure executed FLOPs (ncu) of every kernel whose SASS changed with the 16-byte tile
# staging (register path incl. seed-sparse, F3 seed-sparse), then the headline capture.
set -x
O=gpurun_out/r02ncu; mkdir -p $O
bash tools/ncu_executed.sh c2 --n 16 --m 1048576 --funcs rosenbrock ackley prodsum > $O/ncu_c2.txt 2>&1
bash tools/ncu_executed.sh c2sym --n 16 --m 1048576 --funcs rosenbrock ackley prodsum --algo sym_hvp > $O/ncu_c2sym.txt 2>&1
bash tools/ncu_executed.sh c2sp --n 16 --m 1048576 --algo hvp_seedsparse > $O/ncu_c2sp.txt 2>&1
bash tools/ncu_executed.sh n8 --n 8 --m 1048576 --funcs rosenbrock ackley > $O/ncu_n8.txt 2>&1
bash tools/ncu_executed.sh c4 --n 32 --m 65536 --funcs rosenbrock ackley prodsum --algo hessian --csizes 1 2 4 8 16 32 > $O/ncu_c4.txt 2>&1
bash tools/ncu_executed.sh c4sym --n 32 --m 65536 --funcs rosenbrock ackley prodsum --algo sym_hessian --csizes 1 2 4 8 16 32 > $O/ncu_c4sym.txt 2>&1
bash tools/ncu_executed.sh c3n64 --n 64 --m 65536 --funcs rosenbrock ackley prodsum --csizes 1 2 4 8 16 32 64 > $O/ncu_c3n64.txt 2>&1
bash tools/ncu_executed.sh c3n128 --n 128 --m 16384 --funcs rosenbrock ackley prodsum --csizes 1 2 4 8 16 32 64 128 > $O/ncu_c3n128.txt 2>&1
cp gpurun_out/executed_flops.json $O/
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hvp_reg_kernel -c 1 -s 2 -o $O/prof_headline -f \
  python tools/prof_one.py rosenbrock 16 16 > $O/prof_headline.log 2>&1
cat $O/ncu_c2.txt | grep -v "^=="
