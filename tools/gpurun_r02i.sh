set -x
O=gpurun_out/r02i; mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest_rc=$?
tail -4 $O/pytest.log
timeout 600 python tools/sweep_bench.py --n 2 --m 1048576 --algo hvp --funcs fletcher_powell > $O/f3_n2.jsonl 2>&1
timeout 600 python tools/sweep_bench.py --n 4 --m 1048576 --algo hvp --funcs fletcher_powell > $O/f3_n4.jsonl 2>&1
timeout 600 python tools/sweep_bench.py --n 128 --m 65536 --algo hvp_seedsparse --funcs fletcher_powell --csizes 8 > $O/f3_n128sp.jsonl 2>&1
cat $O/f3_*.jsonl | grep -v "^#" | cut -c1-160
for c in "rosenbrock 2 1 hvp 70000" "fletcher_powell 12 4 hvp 300" "fletcher_powell 72 8 sym_hvp 100" "fletcher_powell 128 16 hessian 40" "fletcher_powell 64 8 hvp_seedsparse 100"; do
  timeout 600 compute-sanitizer --tool memcheck python tools/prof_one.py $c > $O/memcheck_$(echo $c | tr ' ' _).txt 2>&1; tail -2 $O/memcheck_$(echo $c | tr ' ' _).txt
done
timeout 600 compute-sanitizer --tool racecheck python tools/prof_one.py fletcher_powell 72 8 sym_hvp 100 > $O/racecheck_f3mma.txt 2>&1; tail -2 $O/racecheck_f3mma.txt
timeout 600 compute-sanitizer --tool synccheck python tools/prof_one.py fletcher_powell 72 8 sym_hvp 100 > $O/synccheck_f3mma.txt 2>&1; tail -2 $O/synccheck_f3mma.txt
