set -x
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/smi.txt
python -m pytest tests -m gpu -q > gpurun_out/r02a/pytest.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke.log 2>&1; echo smoke_rc=$?
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02a/bench.log 2>&1; echo bench_rc=$?
cp gpurun_out/bench_sweep.json gpurun_out/r02a/ 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02a/launches.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-strong --e2e-steps 1 > gpurun_out/r02a/bench_ncu.log 2>&1; echo ncu_rc=$?
tail -c 2500 gpurun_out/r02a/bench.log
tail -5 gpurun_out/r02a/pytest.log
