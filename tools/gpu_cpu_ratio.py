"""The paper's §VII quantity (Tables of E5): per-point GPU time against
per-point CPU time as n grows, for the paper's three functions.  The paper reports that the
ratio is largest at n = 2 and shrinks with n.  Here: the GPU side is `chessfad_hvp_batch`
(per-evaluation Alg 7, best C over the compiled set, CUDA events, inputs resident), the CPU
side the plain C oracle (Alg 7 as written, one C per n: the same best C) on the host cores,
timed on a bounded sample (~0.5 s per (function, n)).  One JSON line per (function, n).

    python tools/gpu_cpu_ratio.py [--funcs ...] [--ns ...]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the CPU baseline of this measurement)
import paper_2410_22575_b200 as chf  # noqa: E402
import synth  # noqa: E402
from bench import oracle_rate  # noqa: E402


def gpu_rate(func, n, C, m, pr, dev):
    p = torch.from_numpy(synth.points(0, n, m)).to(dev)
    v = torch.from_numpy(synth.vectors(0, n, m)).to(dev)
    out = torch.empty_like(p)
    call = lambda: chf.hvp_batch(func, p, v, C, pr, out=out)  # noqa: E731
    call()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    call()
    torch.cuda.synchronize()
    reps = max(2, min(50, int(0.2 / max(time.perf_counter() - t0, 1e-6))))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    return m / (e0.elapsed_time(e1) / reps * 1e-3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--funcs", nargs="*", default=["rosenbrock", "ackley", "fletcher_powell"])
    ap.add_argument("--ns", nargs="*", type=int, default=[2, 4, 8, 16, 32, 64, 128])
    ap.add_argument("--cpu-s", type=float, default=0.5)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    oracle.build()
    threads = oracle.default_threads()
    for f in args.funcs:
        for n in args.ns:
            pr_np = synth.fp_params_flat(0, n) if f == "fletcher_powell" else None
            pr = None if pr_np is None else torch.from_numpy(pr_np).to(dev)
            # GPU: best C over the compiled set (m sized so a launch is >= ~1 ms where possible)
            m = (1 << 20) if n <= 16 else (1 << 18) if n <= 64 else (1 << 16)
            if f == "fletcher_powell":
                m = max(4096, m >> (4 if n >= 64 else 2))
            best = None
            for C in (c for c in (1, 2, 4, 8, 16, 32, 64, 128) if c <= n and n % c == 0):
                if not chf.is_supported(f, n, C):
                    continue
                r = gpu_rate(f, n, C, m, pr, dev)
                if best is None or r > best[1]:
                    best = (C, r)
            C, g = best
            c, m_cpu, dt = oracle_rate(f, n, C, pr_np, 0, args.cpu_s, threads)
            print(json.dumps({"func": f, "n": n, "C": C, "gpu_hvp_per_s": g, "gpu_m": m, "cpu_hvp_per_s": c,
                              "cpu_points": m_cpu, "cpu_s": dt, "cpu_threads": threads,
                              "gpu_over_cpu": g / c, "path": chf.path(f, n, C)}), flush=True)


if __name__ == "__main__":
    main()
