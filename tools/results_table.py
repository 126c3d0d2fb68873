"""Best chunk size per (n, algorithm, function) from a campaign directory's event-timed sweeps
(time_*.jsonl of tools/sweep_bench.py) joined with the ncu executed-FLOP table of the same
build (executed_flops.json): the DESIGN.md §10 results table.

    python tools/results_table.py DIR [DIR2 ...]   (a later directory's sweep rows replace the
                                                  earlier ones per (n, algorithm, function, m, C))
"""
import glob
import json
import os
import sys

PEAK = 148 * 64 * 2 * 1.965e9  # FP64 FLOP/s


def main(dirs):
    tab = {}
    rows = {}
    for d in dirs:
        try:
            tab.update(json.load(open(os.path.join(d, "executed_flops.json")))["entries"])
        except Exception:
            pass
        for f in sorted(glob.glob(os.path.join(d, "time_*.jsonl"))):
            for line in open(f):
                try:
                    r = json.loads(line)
                except Exception:
                    continue
                rows[(r["n"], r["algo"], r["func"], r["m"], r["C"])] = r
    best = {}
    for r in rows.values():
        k = (r["n"], r["algo"], r["func"], r["m"])
        if k not in best or r["ms"] < best[k]["ms"]:
            best[k] = r
    print("| n | algorithm | function | best C | m | points/s | ms | executed FP64 (of 37.2 TF/s) | exec/model | pipe busy |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for k in sorted(best):
        r = best[k]
        key = f"{r['func']} n={r['n']} C={r['C']}" + ("" if r["algo"] == "hvp" else f" {r['algo']}")
        e = tab.get(key)
        ex = pipe = ratio = "—"
        if e:
            ef = e["executed_flops_per_point"] * r["m"] / (r["ms"] * 1e-3)
            ex = f"{ef / PEAK:.2f}"
            ratio = f"{e['executed_flops_per_point'] / e['model_flops_per_point']:.3f}"
            dm = e.get("dmma_pipe_active_pct") or 0.0
            pipe = f"DMMA {dm:.0f}%" if dm > e["fp64_pipe_active_pct"] else f"{e['fp64_pipe_active_pct']:.0f}%"
        print(f"| {r['n']} | {r['algo']} | {r['func']} | {r['C']} | {r['m']} | {r['points_per_s']:.3g} | "
              f"{r['ms']:.3f} | {ex} | {ratio} | {pipe} |")


if __name__ == "__main__":
    main(sys.argv[1:])
