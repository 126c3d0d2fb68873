"""e2e (host buffers) throughput vs pipeline piece size: chessfad_hvp_batch_host_ctx on pinned
memory, cfg2 Rosenbrock n=16 C=16, CUDA events around each call (copies inside)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import json  # noqa: E402

import torch  # noqa: E402

import paper_2410_22575_b200 as chf  # noqa: E402
import synth  # noqa: E402

n, m, C = 16, 1 << 20, 16
P = torch.from_numpy(synth.points(0, n, m)).pin_memory()
V = torch.from_numpy(synth.vectors(0, n, m)).pin_memory()
O = torch.empty_like(P).pin_memory()
host = chf.HostPipeline()
s = torch.cuda.current_stream()
for pieces in (4, 8, 16, 32, 64, 128, 256):
    pp = m // pieces
    for _ in range(2):
        host.hvp("rosenbrock", P, V, C, out=O, piece_points=pp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        host.hvp("rosenbrock", P, V, C, out=O, piece_points=pp)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"pieces": pieces, "piece_points": pp, "ms": ms, "hvp_per_s": m / ms * 1e3,
                      "h2d_gbs": 2 * m * n * 8 / ms / 1e6}), flush=True)
