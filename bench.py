#!/usr/bin/env python
"""Benchmark of the batched FP64 Hessian-vector product (CHESSFAD hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--func rosenbrock] [--n 16] [--csize 16] [--m 1048576] [--no-sweep]

A step is one chessfad_hvp_batch call: every §8(a) row (load points/vectors, seed,
propagate hDual<C>, chunk dot, row sum, store) over m synthetic points on each GPU
(weak scaling: m points per GPU, disjoint index ranges of one seeded stream).  The headline
workload is BASELINE.json configs[1] (cfg2: n = 16, m = 2^20) with Rosenbrock, the function
of the paper's L2 kernel; the chunk sweep over all four functions is in
"sweep".  Timing: CUDA events on the launching stream, barrier + synchronize around the K
timed steps, max over ranks.  Inputs (384 MiB per step) are larger than the 126 MB L2.

--impl reference times the CPU oracle (oracle/, plain C) on the host cores on a bounded
sample of the same workload (the reference arm of this tier: there is no reference code).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

FUNCS = ["rosenbrock", "ackley", "fletcher_powell", "prodsum"]
METRIC = "Hessian-vector products/sec (FP64) vs n and chunk size; % of B200 FP64 peak"
UNIT = "HVP/s"
SMS = 148
FP64_FMA_PER_SM_CLK = 64  # B200 FP64 (non-tensor) lanes per SM, DESIGN.md "Roofline"


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def fp64_nominal_tflops(peaks):
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    return SMS * FP64_FMA_PER_SM_CLK * 2 * mhz * 1e6 / 1e12, mhz


# ------------------------------------------------------------------------- clocks (NVML)
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index, period=0.02):
        self.samples, self.reasons, self.max_mhz, self.ok = [], 0, None, False
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(get_r(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ------------------------------------------------------------------------- oracle timing
def oracle_rate(func, n, C, params, first, target_s, threads):
    """Time the plain CPU oracle (Alg 7, oracle/) on a bounded sample: returns HVP/s, the
    sample size and the seconds taken.  Sample size is calibrated to ~target_s of work."""
    import oracle
    m = max(threads, 8)
    while True:
        P, V = synth.points(0, n, m, first), synth.vectors(0, n, m, first)
        t0 = time.perf_counter()
        oracle.hvp_batch(func, P, V, C, params, threads=threads)
        dt = time.perf_counter() - t0
        if dt >= target_s * 0.4 or m >= 1 << 22:
            return m / dt, m, dt
        m = int(min(m * max(2.0, 1.2 * target_s / max(dt, 1e-4)), 1 << 22))


def run_reference(args, rank, world):
    """Reference arm: the CPU oracle as it stands, on the host cores."""
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    threads = oracle.default_threads()
    params = synth.fp_params_flat(0, args.n) if args.func == "fletcher_powell" else None
    # size one step to ~1.5 s so that W+K steps end within a few minutes
    rate, m_step, _ = oracle_rate(args.func, args.n, args.csize, params, 0, 1.5, threads)
    P, V = synth.points(0, args.n, m_step), synth.vectors(0, args.n, m_step)
    for _ in range(args.warmup):
        oracle.hvp_batch(args.func, P, V, args.csize, params, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.hvp_batch(args.func, P, V, args.csize, params, threads=threads)
    dt = time.perf_counter() - t0
    value = m_step * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{m_step} points of the workload per step (first {m_step} of the seeded stream), "
                                   f"plain C oracle (Alg 7, -O2 -ffp-contract=off), {threads} pthreads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, world):
    if getattr(args, "m_total", 0):
        wl = f"cfg5: {args.func} n={args.n} C={args.csize} m={args.m_total} points over {world} GPU(s) (strong scaling)"
        gp = args.m_total
    else:
        wl = f"cfg2: {args.func} n={args.n} C={args.csize} m={args.m} points per GPU (BASELINE configs[1])"
        gp = args.m * world
    return {"workload": wl,
            "func": args.func, "n": args.n, "csize": args.csize, "m_per_gpu": args.m, "global_points": gp,
            "seed": 0, "parallelism": f"dp{world} (points sharded, no collective on the data path)",
            "l2": f"inputs larger than L2: {3 * args.m * args.n * 8 / 2**20:.0f} MiB per step vs 126 MB L2"}


# ------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--func", choices=FUNCS, default="rosenbrock")
    ap.add_argument("--n", type=int, default=16)
    ap.add_argument("--csize", type=int, default=16)
    ap.add_argument("--m", type=int, default=1 << 20, help="points per GPU (weak scaling)")
    ap.add_argument("--m-total", type=int, default=0,
                    help="strong scaling: total points split over the ranks (BASELINE cfg5: 8388608)")
    ap.add_argument("--gather", action="store_true", help="time an all-gather of the results after the run")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=10)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2410_22575_b200 as chf

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    chf.load()
    peaks = load_peaks()
    peak_tf, peak_mhz = fp64_nominal_tflops(peaks)

    def barrier():
        if world > 1:
            dist.barrier()

    from paper_2410_22575_b200.dist import gather_rows, max_over_ranks as _mor, shard

    def max_over_ranks(x):
        return _mor(x, device=dev)

    n, C = args.n, args.csize
    if args.m_total:
        first, m = shard(args.m_total, rank, world)
        m_all = args.m_total
    else:
        m = args.m
        first, m_all = rank * m, world * m
    args.m = m
    P = synth.points(0, n, m, first)
    V = synth.vectors(0, n, m, first)
    params_np = {f: (synth.fp_params_flat(0, n) if f == "fletcher_powell" else None) for f in FUNCS}
    pts = torch.from_numpy(P).to(dev)
    vec = torch.from_numpy(V).to(dev)
    out = torch.empty_like(pts)
    params = {f: (None if v is None else torch.from_numpy(v).to(dev)) for f, v in params_np.items()}
    stream = torch.cuda.current_stream()

    def timed(func, csize, steps, warmup, sampler=None):
        for _ in range(warmup):
            chf.hvp_batch(func, pts, vec, csize, params[func], out=out)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx = sampler if sampler is not None else _Null()
        with ctx:
            ev0.record(stream)
            for _ in range(steps):
                chf.hvp_batch(func, pts, vec, csize, params[func], out=out)
            ev1.record(stream)
            torch.cuda.synchronize()
        barrier()
        return max_over_ranks(ev0.elapsed_time(ev1) / 1e3)

    # ---- headline
    sampler = ClockSampler(local)
    t = timed(args.func, C, args.steps, args.warmup, sampler)
    per_step = t / args.steps
    value = m_all / per_step
    flops_pt = chf.model_flops_per_point(args.func, n, C)
    achieved_tf = m * flops_pt / per_step / 1e12  # per GPU, one launch per step
    clocks = sampler.summary()

    # ---- parity of the timed output on a deterministic sample (rank 0)
    parity = None
    if rank == 0:
        import oracle
        idx = np.unique(np.concatenate([[0, m - 1], np.arange(0, m, max(1, m // 61))]))
        ref, sabs = oracle.hvp_batch(args.func, P[idx], V[idx], C, params_np[args.func])
        got = out.cpu().numpy()[idx]
        err = oracle.componentwise_error(got, ref, sabs)
        parity = {"max_componentwise_err": float(err.max()), "points_checked": int(idx.size), "bar": 1e-10,
                  "pass": bool(err.max() <= 1e-10)}

    # ---- FP64 probe (attainable DFMA rate on this GPU)
    sink = torch.empty(SMS * 8 * 256, dtype=torch.float64, device=dev)
    iters = 20000
    chf.fp64_probe(SMS * 8, iters, sink)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    chf.fp64_probe(SMS * 8, iters, sink)
    e1.record(stream)
    torch.cuda.synchronize()
    probe_tf = SMS * 8 * 256 * iters * 16 / (e0.elapsed_time(e1) / 1e3) / 1e12

    # ---- e2e through the host-buffer C-ABI call (pinned host memory, copies in the timed region)
    Ph = torch.from_numpy(P).pin_memory()
    Vh = torch.from_numpy(V).pin_memory()
    Oh = torch.empty_like(Ph).pin_memory()
    ph_params = None if params_np[args.func] is None else torch.from_numpy(params_np[args.func]).pin_memory()
    for _ in range(2):
        chf.hvp_batch_host(args.func, Ph, Vh, C, ph_params, out=Oh)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        chf.hvp_batch_host(args.func, Ph, Vh, C, ph_params, out=Oh)  # synchronous
    e2e_t = max_over_ranks((time.perf_counter() - t0) / args.e2e_steps)
    assert torch.equal(Oh, out.cpu()), "host-buffer path disagrees with the device path"
    e2e = {"value": m_all / e2e_t, "unit": UNIT, "h2d_bytes_per_step": 2 * m * n * 8 + (
        0 if ph_params is None else ph_params.numel() * 8), "d2h_bytes_per_step": m * n * 8,
        "ms_per_step": e2e_t * 1e3, "api": "chessfad_hvp_batch_host (3-stage H2D/kernel/D2H stream pipeline, pinned host memory)"}

    # ---- chunk sweep over the four functions (cfg2), Alg 7 and the NEXT rows
    from paper_2410_22575_b200.build import source_hash
    src_hash = source_hash()
    sweep = []
    algo_fn = {"hvp": chf.hvp_batch, "sym_hvp": chf.sym_hvp_batch, "hvp_hoisted": chf.hvp_batch_hoisted,
               "hvp_seedsparse": chf.hvp_batch_seedsparse}
    if not args.no_sweep:
        for algo, fnb in algo_fn.items():
            for f in FUNCS:
                for c in (1, 2, 4, 8, 16):
                    if n % c or not chf.is_supported(f, n, c, algo):
                        continue
                    for _ in range(3):
                        fnb(f, pts, vec, c, params[f], out=out)
                    torch.cuda.synchronize()
                    barrier()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    ks = 10
                    e0.record(stream)
                    for _ in range(ks):
                        fnb(f, pts, vec, c, params[f], out=out)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    tt = max_over_ranks(e0.elapsed_time(e1) / 1e3) / ks
                    fl = chf.model_flops_per_point(f, n, c, algo=algo)
                    exs = executed_entry(f, n, c, src_hash, algo)
                    sweep.append({"algo": algo, "func": f, "csize": c, "hvp_per_s": m_all / tt, "ms": tt * 1e3,
                                  "model_tflops_effective": m * fl / tt / 1e12,
                                  "executed_tflops": None if exs is None else
                                  m * exs["executed_flops_per_point"] / tt / 1e12,
                                  "executed_frac": None if exs is None else
                                  m * exs["executed_flops_per_point"] / tt / 1e12 / peak_tf})

    # ---- the paper's own Fig. 2 L2 kernel design recompiled for sm_100a (comparison baseline)
    paper_l2 = None
    if not args.no_sweep and args.func in ("rosenbrock", "prodsum") and n in (2, 4, 8, 16):
        best = None
        for c in (1, 2, 4, 8, 16):
            if n % c:
                continue
            try:
                chf.hvp_batch_paper_l2(args.func, pts, vec, c, out=out)
            except chf.ChessfadError:
                continue
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(5):
                chf.hvp_batch_paper_l2(args.func, pts, vec, c, out=out)
            e1.record(stream)
            torch.cuda.synchronize()
            tt = max_over_ranks(e0.elapsed_time(e1) / 1e3) / 5
            if best is None or tt < best[1]:
                best = (c, tt)
        if best:
            paper_l2 = {"kernel": "paper Fig. 2 L2 design (thread per instance x row x chunk, per-thread hDual y[n], "
                                  "shared-memory reduction), recompiled for sm_100a", "best_csize": best[0],
                        "hvp_per_s": m_all / best[1], "ms": best[1] * 1e3, "ours_over_paper_l2": best[1] / per_step}

    # ---- CPU baseline: the oracle on the host cores, rank 0 at N=1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        threads = oracle.default_threads()
        rate, ms, dt = oracle_rate(args.func, n, C, params_np[args.func], 0, 12.0, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"{ms} points (first {ms} of the seeded cfg2 stream), {dt:.1f} s of Alg 7 in the plain C "
                         f"oracle, {threads} pthreads"}

    # executed FP64 FLOPs of this build, measured by ncu (profiles/executed_flops.json)
    from paper_2410_22575_b200.build import source_hash
    ex = executed_entry(args.func, n, C, source_hash())
    model_tf = achieved_tf
    if ex is not None:
        exec_tf = m * ex["executed_flops_per_point"] / per_step / 1e12
        traffic = ex["dram_bytes_per_launch"] * m / ex["m"]
        accounting = ("executed FP64 FLOPs (2*DFMA+DMUL+DADD per point; " + ex["basis"] + ") x m / event time; "
                      "model FLOPs reported as model_tflops_effective")
    else:
        exec_tf, traffic = None, None
        accounting = "executed-FLOP table missing or stale for this build: achieved = model FLOPs (effective)"
    achieved = exec_tf if exec_tf is not None else model_tf

    gather = None
    if args.gather:
        torch.cuda.synchronize()
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        full = gather_rows(out, m_all)
        g1.record(stream)
        torch.cuda.synchronize()
        gather = {"ms": max_over_ranks(g0.elapsed_time(g1)), "bytes_per_rank": int(full.numel() * 8),
                  "collective": "all_gather (NCCL)" if world > 1 else "none (1 rank)"}
        del full

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
            "scaling": "strong" if args.m_total else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload_config(args, world),
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf, "traffic": traffic, "accounting": accounting,
                         "model_tflops_effective": model_tf, "model_frac_effective": model_tf / peak_tf,
                         "executed_flops_per_point": None if ex is None else ex["executed_flops_per_point"],
                         "fp64_pipe_active_pct_ncu": None if ex is None else ex["fp64_pipe_active_pct"],
                         "kernel": f"hvp_reg_kernel<{args.func},C={C}>" if args.func != "fletcher_powell"
                         else "hvp_f3_kernel",
                         "peak_basis": f"derived: {SMS} SMs x {FP64_FMA_PER_SM_CLK} FP64 FMA/clk x 2 x {peak_mhz:.0f} MHz "
                                       "(sm_max_mhz, MEASURED_PEAKS.json); DESIGN.md",
                         "model_flops_per_point": flops_pt,
                         "fp64_probe_tflops": probe_tf, "frac_of_probe": achieved / probe_tf},
            "cpu_baseline": cpu, "e2e": e2e,
            # one kernel per call; F3 with n > 32 adds the (A, B) interleave kernel
            "gpu_launches": args.steps * (2 if (args.func == "fletcher_powell" and n > 32) else 1), "clocks": clocks, "parity": parity,
            "gather": gather, "paper_l2_baseline": paper_l2, "sweep": sweep,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def executed_entry(func, n, C, src_hash, algo="hvp", path=None):
    """ncu-measured executed FLOPs/point of this build (profiles/executed_flops.json).  If the
    table was measured on an earlier build, its executed/model ratio is applied to this build's
    model count and the entry is marked stale (its 'basis' field says so)."""
    try:
        tab = json.load(open(path or os.path.join(ROOT, "profiles", "executed_flops.json")))
    except Exception:
        return None
    key = f"{func} n={n} C={C}" + ("" if algo == "hvp" else f" {algo}")
    ent = tab.get("entries", {}).get(key)
    if ent is None:
        return None
    ent = dict(ent)
    import paper_2410_22575_b200 as chf
    from paper_2410_22575_b200.sass import sass_hash_for
    cur = sass_hash_for(chf.LIB_PATH, ent["kernel"]) if ent.get("kernel") and ent.get("sass_hash") else None
    if cur is not None and cur == ent["sass_hash"]:
        ent["basis"] = f"ncu on identical kernel SASS ({cur})"
    elif tab.get("src_hash") == src_hash:
        ent["basis"] = f"ncu on this build ({src_hash})"
    else:
        ratio = ent["executed_flops_per_point"] / ent["model_flops_per_point"]
        ent["executed_flops_per_point"] = ratio * chf.model_flops_per_point(func, n, C, algo=algo)
        ent["basis"] = f"STALE: executed/model ratio {ratio:.3f} measured by ncu on build {tab.get('src_hash')}"
    return ent


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


if __name__ == "__main__":
    sys.exit(main())
