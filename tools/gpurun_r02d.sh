set -x
O=gpurun_out/r02d; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo pytest_rc=$?
tail -15 $O/pytest.log
timeout 600 python tools/sweep_bench.py --n 16 --m 1048576 --algo hvp --funcs fletcher_powell > $O/f3_n16.jsonl 2>&1
timeout 600 python tools/sweep_bench.py --n 64 --m 131072 --algo hvp --funcs fletcher_powell --csizes 1 4 8 16 64 > $O/f3_n64.jsonl 2>&1
timeout 600 python tools/sweep_bench.py --n 32 --m 262144 --algo hessian --funcs fletcher_powell > $O/f3_n32h.jsonl 2>&1
timeout 600 python tools/sweep_bench.py --n 64 --m 131072 --algo sym_hvp --funcs fletcher_powell --csizes 4 8 16 > $O/f3_n64s.jsonl 2>&1
cat $O/f3_*.jsonl | grep -v "^#" | cut -c1-220
bash tools/ab_stream.sh $O/ab new=paper_2410_22575_b200/libchessfad.so old=paper_2410_22575_b200/libchessfad_nostream.so
python tools/ab_compare.py $O/ab old new
