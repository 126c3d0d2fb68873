"""Minimal launches for compute-sanitizer racecheck (tracks every shared-memory access, so
only the shared-memory patterns are covered: tile staging + write-back, the symmetric HVP's
per-warp output tile, F3's shared (A,B) and F3's per-warp cp.async ring)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2410_22575_b200 as chf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
for n, m, C, funcs in ((16, 33, 16, ("rosenbrock", "ackley", "fletcher_powell")), (64, 3, 64, ("fletcher_powell",))):
    p = torch.from_numpy(synth.points(0, n, m)).to(dev)
    v = torch.from_numpy(synth.vectors(0, n, m)).to(dev)
    pr = torch.from_numpy(synth.fp_params_flat(0, n)).to(dev)
    for f in funcs:
        par = pr if f == "fletcher_powell" else None
        chf.hvp_batch(f, p, v, C, par)
        if n == 16:
            chf.sym_hvp_batch(f, p, v, C, par)
    torch.cuda.synchronize()
print("racecheck cases done")
