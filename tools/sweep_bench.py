"""Time a sweep of (func, C) for one (n, m, algo) with CUDA events; one JSON line per config.

    python tools/sweep_bench.py --n 64 --m 1048576 --algo hvp [--funcs ...] [--csizes ...]

Used for BASELINE configs 3 (n = 64/128), 4 (Hessian, n = 32) and the symmetric algorithms;
the headline cfg2 line is bench.py's.  Inputs: synth seed 0.  Each config: 2 warm-up
launches, then `reps` timed launches (>= ~0.3 s), the mean time reported.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2410_22575_b200 as chf  # noqa: E402
import synth  # noqa: E402
from bench import ClockSampler, executed_entry  # noqa: E402
from paper_2410_22575_b200.build import source_hash  # noqa: E402

PEAK = 148 * 64 * 2 * 1.965e9 / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16)
    ap.add_argument("--m", type=int, default=1 << 20)
    ap.add_argument("--algo", default="hvp", choices=list(chf.ALGOS))
    ap.add_argument("--funcs", nargs="*", default=["rosenbrock", "ackley", "fletcher_powell", "prodsum"])
    ap.add_argument("--csizes", nargs="*", type=int, default=None)
    ap.add_argument("--min-seconds", type=float, default=0.3)
    ap.add_argument("--f3-m", type=int, default=0, help="reduced m for Fletcher-Powell (0: same m)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = args.n
    Cs = args.csizes or [c for c in (1, 2, 4, 8, 16, 32, 64, 128) if c <= n and n % c == 0]
    hess = args.algo in ("hessian", "sym_hessian", "hessian_seedsparse")
    fn = {"hvp": chf.hvp_batch, "sym_hvp": chf.sym_hvp_batch, "hessian": chf.hessian_batch, "hvp_hoisted": chf.hvp_batch_hoisted, "hvp_seedsparse": chf.hvp_batch_seedsparse, "hessian_seedsparse": chf.hessian_batch_seedsparse,
          "sym_hvp_seedsparse": chf.sym_hvp_batch_seedsparse,
          "sym_hessian": chf.sym_hessian_batch}[args.algo]
    for f in args.funcs:
        m = args.f3_m if (f == "fletcher_powell" and args.f3_m) else args.m
        pts = torch.from_numpy(synth.points(0, n, m)).to(dev)
        vec = torch.from_numpy(synth.vectors(0, n, m)).to(dev)
        pr = torch.from_numpy(synth.fp_params_flat(0, n)).to(dev) if f == "fletcher_powell" else None
        out = torch.empty((m, n, n) if hess else (m, n), dtype=torch.float64, device=dev)
        for c in Cs:
            if not chf.is_supported(f, n, c, args.algo):
                continue
            call = (lambda: fn(f, pts, c, pr, out=out)) if hess else (lambda: fn(f, pts, vec, c, pr, out=out))
            call()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            call()
            torch.cuda.synchronize()
            one = time.perf_counter() - t0
            reps = max(1, min(50, int(args.min_seconds / max(one, 1e-6))))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            clk = ClockSampler(0)
            with clk:
                e0.record()
                for _ in range(reps):
                    call()
                e1.record()
                torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3 / reps
            clocks = clk.summary()
            mf = chf.model_flops_per_point(f, n, c, algo=args.algo)
            ex = executed_entry(f, n, c, source_hash(), args.algo)  # valid by kernel SASS hash (bench.py)
            if ex is not None and ex["basis"].startswith("STALE"):
                ex = None
            rec = {"func": f, "n": n, "C": c, "algo": args.algo, "m": m, "ms": t * 1e3, "points_per_s": m / t,
                   "model_flops_per_point": mf, "model_tflops_effective": m * mf / t / 1e12,
                   "executed_tflops": None if ex is None else m * ex["executed_flops_per_point"] / t / 1e12}
            rec["executed_frac"] = None if ex is None else rec["executed_tflops"] / PEAK
            rec["sm_mhz"], rec["clock_reasons"] = clocks["sm_mhz"], clocks["reasons"]
            print(json.dumps(rec), flush=True)
        del pts, vec, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
