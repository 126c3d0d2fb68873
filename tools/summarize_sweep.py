"""Summarise an ncu --csv metric log of tools/profile_sweep.py: executed FP64 FLOPs
(2*DFMA + DMUL + DADD) vs model FLOPs, FP64 pipe utilisation, DRAM traffic."""
import csv
import json
import re
import sys


def load(csv_path, order_path):
    order = [l.split() for l in open(order_path) if l.startswith("launch ")]
    rows = list(csv.reader(l for l in open(csv_path) if not l.startswith("==")))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in rows[1:]:
        if len(r) < len(hdr) or "hvp_" not in r[ix["Kernel Name"]]:
            continue  # only the batch kernels (not the F3 (A,B) prep kernel)
        lid = int(r[ix["ID"]])
        per.setdefault(lid, {})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        per[lid]["__kernel"] = r[ix["Kernel Name"]]
    out = []
    for lid, (k, v) in enumerate(sorted(per.items())):
        if lid >= len(order):
            break
        _, func, n, C, m, fl = order[lid][:6]
        algo = order[lid][6].split("=")[1] if len(order[lid]) > 6 else "hvp"
        n, C, m = int(n[2:]), int(C[2:]), int(m[2:])
        model = float(fl.split("=")[1]) * m
        dmma = v.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0.0)  # m8n8k4: 256 FMAs per warp instruction
        ex = 2 * v["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"] + v["sm__sass_thread_inst_executed_op_dmul_pred_on.sum"] + v["sm__sass_thread_inst_executed_op_dadd_pred_on.sum"] + 512 * dmma
        t = v["gpu__time_duration.sum"] * 1e-9
        out.append({"func": func, "n": n, "C": C, "m": m, "algo": algo, "kernel": v["__kernel"], "time_ms": t * 1e3,
                    "model_flops": model, "executed_flops": ex, "executed_over_model": ex / model,
                    "fp64_warp_inst": v["sm__inst_executed_pipe_fp64.sum"],
                    "fp64_pipe_active_pct": v["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
                    "dmma_warp_inst": dmma,
                    "dmma_pipe_active_pct": v.get("smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
                    "executed_flop_per_fp64_lane_inst": ex / (32 * v["sm__inst_executed_pipe_fp64.sum"]),
                    "all_warp_inst": v["smsp__inst_executed.sum"],
                    "fp64_inst_share": v["sm__inst_executed_pipe_fp64.sum"] / v["smsp__inst_executed.sum"],
                    "dram_bytes": v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"],
                    "regs": v["launch__registers_per_thread"],
                    "warps_active_pct": v["sm__warps_active.avg.pct_of_peak_sustained_active"],
                    "sm_clock_ghz": v["sm__cycles_elapsed.avg.per_second"] / 1e9})
    return out


def update_table(res, table_path):
    """Merge executed-FLOP measurements into profiles/executed_flops.json (keyed by the
    source hash of the build that was profiled)."""
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2410_22575_b200 import LIB_PATH
    from paper_2410_22575_b200.build import source_hash
    from paper_2410_22575_b200.sass import sass_hash_for
    h = source_hash()
    try:
        tab = json.load(open(table_path))
    except Exception:
        tab = {}
    if tab.get("src_hash") != h:  # keep entries whose kernel SASS is unchanged
        keep = {k: e for k, e in tab.get("entries", {}).items()
                if e.get("sass_hash") and sass_hash_for(LIB_PATH, e.get("kernel", "")) == e["sass_hash"]}
        tab = {"src_hash": h, "entries": keep}
    for r in res:
        key = f"{r['func']} n={r['n']} C={r['C']}" + ("" if r.get("algo", "hvp") == "hvp" else f" {r['algo']}")
        tab["entries"][key] = {"executed_flops_per_point": r["executed_flops"] / r["m"],
                               "model_flops_per_point": r["model_flops"] / r["m"],
                               "fp64_pipe_active_pct": r["fp64_pipe_active_pct"],
                               "dmma_pipe_active_pct": r.get("dmma_pipe_active_pct"),
                               "dmma_flops_per_point": 512 * r.get("dmma_warp_inst", 0.0) / r["m"],
                               "dram_bytes_per_launch": r["dram_bytes"], "m": r["m"], "regs": r["regs"],
                               "ncu_time_ms": r["time_ms"], "kernel": r["kernel"],
                               "sass_hash": sass_hash_for(LIB_PATH, r["kernel"])}
    tab["note"] = ("entries are valid for the kernel SASS whose sha256 is sass_hash (paper_2410_22575_b200/sass.py); "
                   "executed FP64 FLOPs = 2*DFMA + DMUL + DADD thread instructions (ncu "
                   "sm__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum) + 512 per DMMA m8n8k4 warp "
                   "instruction (sm__inst_executed_pipe_tensor_subpipe_dmma.sum) per point, one launch each; "
                   "tools/profile_sweep.py under ncu, summarised by tools/summarize_sweep.py")
    json.dump(tab, open(table_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    res = load(sys.argv[1], sys.argv[2])
    print(f"{'func':16s} {'algo':11s} {'n':>3s} {'C':>3s} {'ms':>7s} {'exec/model':>10s} {'fp64pipe%':>9s} {'fl/inst':>7s} {'fp64share':>9s} {'DRAM MB':>8s} {'regs':>4s} {'warps%':>6s} {'GHz':>5s}")
    for r in res:
        print(f"{r['func']:16s} {r['algo']:11s} {r['n']:3d} {r['C']:3d} {r['time_ms']:7.2f} {r['executed_over_model']:10.3f} {r['fp64_pipe_active_pct']:9.1f} "
              f"{r['executed_flop_per_fp64_lane_inst']:7.3f} {r['fp64_inst_share']:9.3f} {r['dram_bytes']/1e6:8.1f} {r['regs']:4.0f} "
              f"{r['warps_active_pct']:6.1f} {r['sm_clock_ghz']:5.2f}")
    if len(sys.argv) > 3:
        json.dump(res, open(sys.argv[3], "w"), indent=1)
    if len(sys.argv) > 4:
        update_table(res, sys.argv[4])
