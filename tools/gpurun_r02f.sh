set -x
O=gpurun_out/r02f; mkdir -p $O
python -m pytest tests -m gpu -q -x -k "f3_dmma or sym or large_n or hessian or seedsparse or config3 or config4 or parity_sweep" > $O/pytest.log 2>&1; echo pytest_rc=$?
tail -5 $O/pytest.log
timeout 900 python tools/sweep_bench.py --n 128 --m 16384 --algo hvp --funcs fletcher_powell --csizes 1 8 32 128 > $O/f3_n128.jsonl 2>&1
timeout 600 python tools/sweep_bench.py --n 128 --m 16384 --algo sym_hvp --funcs fletcher_powell --csizes 8 16 > $O/f3_n128s.jsonl 2>&1
timeout 600 python tools/sweep_bench.py --n 100 --m 16384 --algo hvp --funcs fletcher_powell --csizes 4 25 > $O/f3_n100.jsonl 2>&1
cat $O/f3_*.jsonl | grep -v "^#" | cut -c1-200
bash tools/ncu_executed.sh f3n16 --n 16 --m 262144 --funcs fletcher_powell > $O/ncu_f3n16.txt 2>&1
bash tools/ncu_executed.sh f3n64 --n 64 --m 16384 --funcs fletcher_powell --csizes 1 8 16 64 > $O/ncu_f3n64.txt 2>&1
bash tools/ncu_executed.sh stream2 --n 2 --m 16777216 --funcs rosenbrock ackley prodsum > $O/ncu_stream2.txt 2>&1
cat $O/ncu_*.txt | grep -v "^==" | tail -30
cp profiles/executed_flops.json $O/
