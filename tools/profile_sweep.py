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
    ap.add_argument("--algo", default=None, choices=list(chf.ALGOS))
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n, m = args.n, args.m
    pts = torch.from_numpy(synth.points(0, n, m)).to(dev)
    vec = torch.from_numpy(synth.vectors(0, n, m)).to(dev)
    params = torch.from_numpy(synth.fp_params_flat(0, n)).to(dev)
    algo = args.algo or ("hessian" if args.hessian else "hvp")
    fn = {"hvp": chf.hvp_batch, "sym_hvp": chf.sym_hvp_batch, "hessian": chf.hessian_batch, "hvp_hoisted": chf.hvp_batch_hoisted, "hvp_seedsparse": chf.hvp_batch_seedsparse, "hessian_seedsparse": chf.hessian_batch_seedsparse,
          "sym_hessian": chf.sym_hessian_batch, "sym_hvp_seedsparse": chf.sym_hvp_batch_seedsparse}[algo]
    for f in args.funcs:
        for c in args.csizes:
            if n % c or not chf.is_supported(f, n, c, algo):
                continue
            pr = params if f == "fletcher_powell" else None
            if algo in ("hessian", "sym_hessian"):
                fn(f, pts, c, pr)
            else:
                fn(f, pts, vec, c, pr)
            torch.cuda.synchronize()
            print(f"launch {f} n={n} C={c} m={m} flops_per_point={chf.model_flops_per_point(f, n, c, algo=algo):.0f}"
                  f" algo={algo}", flush=True)


if __name__ == "__main__":
    main()
