"""Small launches of the round-2 kernels for compute-sanitizer: the register kernels compiled for
n (plain, and Rosenbrock's volatile-seed / unrolled-chunk form) in every mode, Alg 7 at
n = 64 / 128, and the stream kernel with a compile-time chunk start; ragged m."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2410_22575_b200 as chf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
cases = [(8, 45), (16, 77), (32, 40), (64, 37), (128, 9)]
for n, m in cases:
    p = torch.from_numpy(synth.points(0, n, m)).to(dev)
    v = torch.from_numpy(synth.vectors(0, n, m)).to(dev)
    for f in ("rosenbrock", "ackley", "prodsum"):
        for C in (2, 8, 16):
            if n % C:
                continue
            for algo, fn in (("hvp", chf.hvp_batch), ("sym_hvp", chf.sym_hvp_batch)):
                if chf.is_supported(f, n, C, algo):
                    fn(f, p, v, C)
            if n <= 32:
                for algo, fn in (("hessian", chf.hessian_batch), ("sym_hessian", chf.sym_hessian_batch)):
                    if chf.is_supported(f, n, C, algo):
                        fn(f, p, C)
                g = torch.empty((m, n), dtype=torch.float64, device=dev)
                chf.hessian_grad_batch(f, p, C, grad=g)
for n in (2, 4, 8):
    m = 600
    p = torch.from_numpy(synth.points(1, n, m)).to(dev)
    v = torch.from_numpy(synth.vectors(1, n, m)).to(dev)
    for f in ("rosenbrock", "ackley", "prodsum"):
        for C in (1, 2):
            chf.hvp_batch(f, p, v, C)
torch.cuda.synchronize()
print("sanitize ns cases done")
