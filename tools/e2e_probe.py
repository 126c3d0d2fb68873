"""Host-buffer (e2e) path probe: raw pinned H2D/D2H bandwidth and chessfad_hvp_batch_host
time vs piece count at cfg2 (Rosenbrock n=16, C=16, m=2^20)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2410_22575_b200 as chf  # noqa: E402
import synth  # noqa: E402

n, m, C = 16, 1 << 20, 16
P = torch.from_numpy(synth.points(0, n, m)).pin_memory()
V = torch.from_numpy(synth.vectors(0, n, m)).pin_memory()
O = torch.empty_like(P).pin_memory()
d = torch.empty_like(P, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(P, non_blocking=True)), ("d2h", lambda: O.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(json.dumps({"copy": name, "GB/s": P.numel() * 8 / dt / 1e9}))
for pieces in (1, 2, 4, 8, 16, 32, 64):
    pp = (m + pieces - 1) // pieces
    chf.hvp_batch_host("rosenbrock", P, V, C, out=O, piece_points=pp)
    t0 = time.perf_counter()
    for _ in range(5):
        chf.hvp_batch_host("rosenbrock", P, V, C, out=O, piece_points=pp)
    dt = (time.perf_counter() - t0) / 5
    print(json.dumps({"pieces": pieces, "ms": dt * 1e3, "hvp_per_s": m / dt}))
