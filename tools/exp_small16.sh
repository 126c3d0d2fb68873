for v in default small16; do if [ $v = default ]; then L=""; else L=$PWD/exp/libchessfad_$v.so; fi
CHESSFAD_LIB=$L timeout 300 python tools/sweep_bench.py --n 16 --m 1048576 --funcs rosenbrock ackley prodsum > gpurun_out/s16_$v.jsonl; done
CHESSFAD_LIB=$PWD/exp/libchessfad_small16.so timeout 600 python -m pytest tests -m gpu -q -k "sweep and 16 or integer" 2>&1 | tail -1
