"""The paper's E4 experiment shape on B200 (GPU kernel time vs n for the
L0/L1/L2 mappings, 0.5M points, kernel time only): the paper's three designs recompiled for
sm_100a (chessfad_hvp_batch_paper) beside this library's kernel, Rosenbrock, n in
{2, 4, 8, 16}, every chunk size; one JSON line per (impl, n, C)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2410_22575_b200 as chf  # noqa: E402
import synth  # noqa: E402

m = 1 << 19  # the paper's 0.5M points
dev = torch.device("cuda", 0)
for n in (2, 4, 8, 16):
    p = torch.from_numpy(synth.points(0, n, m)).to(dev)
    v = torch.from_numpy(synth.vectors(0, n, m)).to(dev)
    out = torch.empty_like(p)
    impls = {"paper_L0": lambda c: chf.hvp_batch_paper(0, "rosenbrock", p, v, c, out=out),
             "paper_L1": lambda c: chf.hvp_batch_paper(1, "rosenbrock", p, v, c, out=out),
             "paper_L2": lambda c: chf.hvp_batch_paper(2, "rosenbrock", p, v, c, out=out),
             "ours": lambda c: chf.hvp_batch("rosenbrock", p, v, c, out=out),
             "ours_hoisted": lambda c: chf.hvp_batch_hoisted("rosenbrock", p, v, c, out=out)}
    for name, fn in impls.items():
        for c in (1, 2, 4, 8, 16):
            if n % c or c > n:
                continue
            fn(c)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            reps = 5
            for _ in range(reps):
                fn(c)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3 / reps
            print(json.dumps({"impl": name, "n": n, "C": c, "m": m, "ms": t * 1e3, "ns_per_point": t / m * 1e9}),
                  flush=True)
