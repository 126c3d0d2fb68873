"""Compare two sweep_bench JSONL sets (A/B of library builds): ms per config, new/old ratio.

    python tools/ab_compare.py DIR old new
"""
import glob
import json
import os
import sys

d, a, b = sys.argv[1], sys.argv[2], sys.argv[3]
for fa in sorted(glob.glob(os.path.join(d, f"{a}_*.jsonl"))):
    tag = os.path.basename(fa)[len(a) + 1:-6]
    fb = os.path.join(d, f"{b}_{tag}.jsonl")
    if not os.path.exists(fb):
        continue

    def load(f):
        r = {}
        for line in open(f):
            try:
                x = json.loads(line)
            except Exception:
                continue
            r[(x.get("algo"), x["func"], x["C"])] = x
        return r
    A, B = load(fa), load(fb)
    for k in A:
        if k in B:
            print(f"{tag:6s} {k[0]:12s} {k[1]:16s} C={k[2]:<4d} {a}={A[k]['ms']:9.3f} ms  {b}={B[k]['ms']:9.3f} ms  {b}/{a} time {B[k]['ms']/A[k]['ms']:.3f}")
