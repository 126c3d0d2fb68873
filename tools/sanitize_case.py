"""Small launches of every kernel family for compute-sanitizer (memcheck / racecheck /
initcheck / synccheck): all functions, all four algorithms, register path, F3 shared (A,B)
and F3 cp.async ring (n = 64), ragged m."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2410_22575_b200 as chf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
small = os.environ.get("SANITIZE_SMALL") == "1"  # racecheck: fewer, smaller launches
for n, m in (((16, 33), (64, 5)) if small else ((16, 77), (64, 40))):
    p = torch.from_numpy(synth.points(0, n, m)).to(dev)
    v = torch.from_numpy(synth.vectors(0, n, m)).to(dev)
    pr = torch.from_numpy(synth.fp_params_flat(0, n)).to(dev)
    for f in ("rosenbrock", "ackley", "fletcher_powell", "prodsum"):
        for C in ((16,) if small else (4, 16)):
            par = pr if f == "fletcher_powell" else None
            for algo, fn in (("hvp", chf.hvp_batch), ("sym_hvp", chf.sym_hvp_batch)):
                if chf.is_supported(f, n, C, algo):
                    fn(f, p, v, C, par)
            for algo, fn in (("hessian", chf.hessian_batch), ("sym_hessian", chf.sym_hessian_batch)):
                if chf.is_supported(f, n, C, algo):
                    fn(f, p, C, par)
    torch.cuda.synchronize()
chf.hvp_batch_host("rosenbrock", synth.points(0, 16, 1000), synth.vectors(0, 16, 1000), 4, piece_points=300)
print("sanitize cases done")
