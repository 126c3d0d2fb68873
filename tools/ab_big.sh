O=gpurun_out/ab_big; mkdir -p $O
for spec in rt=ab/ns.so big=ab/nsbig.so; do
  name=${spec%%=*}; export CHESSFAD_LIB=${spec#*=}
  timeout 900 python tools/sweep_bench.py --n 64 --m 262144 --algo hvp --funcs rosenbrock ackley prodsum --min-seconds 0.2 > $O/${name}_n64.jsonl 2>&1
  timeout 900 python tools/sweep_bench.py --n 128 --m 65536 --algo hvp --funcs rosenbrock ackley prodsum --min-seconds 0.2 > $O/${name}_n128.jsonl 2>&1
done
python tools/ab_compare.py $O rt big | tee $O/summary.txt
