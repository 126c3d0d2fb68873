"""One launch per (func, csize) of the cfg2 workload, for ncu metric collection.

    ncu --metrics ... python tools/profile_sweep.py [--n 16] [--m 1048576] [--funcs ...] [--csizes ...]

Prints the launch order (one line per launch) so ncu rows can be matched to (func, C).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2410_22575_b200 as chf  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16)
    ap.add_argument("--m", type=int, default=1 << 20)
    ap.add_argument("--funcs", nargs="*", default=["rosenbrock", "ackley", "fletcher_powell", "prodsum"])
    ap.add_argument("--csizes", nargs="*", type=int, default=[1, 2, 4, 8, 16])
    ap.add_argument("--hessian", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n, m = args.n, args.m
    pts = torch.from_numpy(synth.points(0, n, m)).to(dev)
    vec = torch.from_numpy(synth.vectors(0, n, m)).to(dev)
    params = torch.from_numpy(synth.fp_params_flat(0, n)).to(dev)
    for f in args.funcs:
        for c in args.csizes:
            if n % c or not chf.is_supported(f, n, c):
                continue
            pr = params if f == "fletcher_powell" else None
            if args.hessian:
                chf.hessian_batch(f, pts, c, pr)
            else:
                chf.hvp_batch(f, pts, vec, c, pr)
            torch.cuda.synchronize()
            print(f"launch {f} n={n} C={c} m={m} flops_per_point={chf.model_flops_per_point(f, n, c, args.hessian):.0f}",
                  flush=True)


if __name__ == "__main__":
    main()
