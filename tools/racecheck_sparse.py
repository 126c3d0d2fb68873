"""Minimal launches of the NEXT-4 seed-sparse kernels for compute-sanitizer (memcheck,
racecheck, synccheck): the F3 kernel with (A, B) in shared memory (n = 16), the staged
cp.async double buffer (n = 64, CTA-wide barriers) and its unstaged fallback (n = 36), HVP and
Hessian; the register-path sparse bodies (n = 24, a column-group C)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2410_22575_b200 as chf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
for n, m, C in ((16, 33, 4), (64, 3, 64), (36, 5, 12)):
    p = torch.from_numpy(synth.points(0, n, m)).to(dev)
    v = torch.from_numpy(synth.vectors(0, n, m)).to(dev)
    pr = torch.from_numpy(synth.fp_params_flat(0, n)).to(dev)
    chf.hvp_batch_seedsparse("fletcher_powell", p, v, C, pr)
    chf.hessian_batch_seedsparse("fletcher_powell", p, C, pr)
n, m = 24, 40
p = torch.from_numpy(synth.points(0, n, m)).to(dev)
v = torch.from_numpy(synth.vectors(0, n, m)).to(dev)
for f in ("rosenbrock", "ackley", "prodsum"):
    chf.hvp_batch_seedsparse(f, p, v, 24)
    chf.hessian_batch_seedsparse(f, p, 8)
torch.cuda.synchronize()
print("sparse sanitizer cases done")
