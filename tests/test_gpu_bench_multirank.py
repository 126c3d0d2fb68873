"""bench.py's N > 1 path on a one-GPU box: two ranks (torchrun re-exec from --gpus 2) share GPU 0
over gloo (test hook CHESSFAD_BENCH_ONE_GPU) -- shards of one seeded stream, the in-place
all_gather_into_tensor of cfg5's results with its parity check, max over ranks, per-rank
clocks and the single < 2 KB JSON line.  The NCCL transport itself needs two GPUs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_on_one_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CHESSFAD_BENCH_ONE_GPU"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--no-cpu", "--e2e-steps", "2", "--no-sweep"], capture_output=True, text=True, timeout=900,
                       env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and len(lines[0]) < 2048
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_points"] == 2 * d["config"]["m_per_gpu"]
    assert d["parity"]["pass"] and d["strong"]["gather_parity"] is True
    assert "in place" in d["strong"]["gather"] and len(d["clocks"]["per_rank_sm_mhz"]) == 2
