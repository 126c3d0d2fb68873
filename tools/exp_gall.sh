for v in default gall; do if [ $v = default ]; then L=""; else L=$PWD/exp/libchessfad_$v.so; fi
for n in 4 8 16 32; do m=$((n<=16 ? 1048576 : 262144)); CHESSFAD_LIB=$L timeout 300 python tools/sweep_bench.py --n $n --m $m --funcs rosenbrock ackley prodsum > gpurun_out/gall_${v}_n$n.jsonl; done; done
