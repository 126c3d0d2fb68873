#!/usr/bin/env python
"""Benchmark of the batched FP64 Hessian-vector product (CHESSFAD hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--func rosenbrock] [--n 16] [--csize 16] [--m 1048576] [--no-sweep]

A step is one chessfad_hvp_batch call: every §8(a) row (load points/vectors, seed,
propagate hDual<C>, chunk dot, row sum, store) over m synthetic points on each GPU
(weak scaling: m points per GPU, disjoint index ranges of one seeded stream).  The headline
workload is BASELINE.json configs[1] (cfg2: n = 16, m = 2^20) with Rosenbrock, the function
of the paper's L2 kernel.  Timing: CUDA events on the launching stream, one
per step, barrier + synchronize around the K timed steps, max over ranks; value = K-step
mean, step_ms = median / best of the K per-step samples (§8(d)).  Inputs (384 MiB per
step) are larger than the 126 MB L2, so no flush is needed between steps.

stdout ends with ONE compact JSON line (< 2 KB).  The bulky evidence -- the chunk sweep over
the four functions and the algorithms, the paper's Fig. 2 kernel -- goes to --sweep-out
(default gpurun_out/bench_sweep.json).  "strong" is BASELINE configs[4] (cfg5: 2^23 points
split over the ranks, compute-only and compute + NCCL all-gather of the results).

--gpus N without a torchrun environment re-executes itself under torch.distributed.run
(N ranks, 127.0.0.1).  --impl reference times the CPU oracle (oracle/, plain C) on the host
cores on a bounded sample of the same workload (the reference arm of this tier: there is
no reference code); under N ranks only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
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
CFG5_M_TOTAL = 1 << 23    # BASELINE configs[4]: 8M points sharded over the ranks


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

    def __init__(self, device_index, period=0.005):
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


# ------------------------------------------------------------------------- torchrun re-exec
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_respawn(args, argv):
    """--gpus N > 1 outside a torchrun environment: run this script under
    torch.distributed.run with N ranks (one per GPU) and return its exit code; None when the
    current process is already the right one."""
    if "WORLD_SIZE" in os.environ:
        ws = env_int("WORLD_SIZE", 1)
        if ws != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
        return None
    if args.gpus <= 1:
        return None
    # the arguments travel in the environment: torchrun's own parser rejects script options
    # that abbreviate one of its options (e.g. --n)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)]
    return subprocess.call(cmd, env=dict(os.environ, CHESSFAD_BENCH_ARGV=json.dumps(list(argv))))


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
    """Reference arm: the CPU oracle as it stands, on the host cores (rank 0 only)."""
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    threads = oracle.default_threads()
    params = synth.fp_params_flat(0, args.n) if args.func == "fletcher_powell" else None
    # one step = a bounded sample of the workload sized so that W+K steps end within minutes
    rate, m_step, _ = oracle_rate(args.func, args.n, args.csize, params, 0, args.ref_step_s, threads)
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
        wl = f"cfg5: {args.func} n={args.n} C={args.csize} m={args.m_total} over {world} GPU(s) (strong)"
        gp = args.m_total
    else:
        wl = f"cfg2 (configs[1]): {args.func} n={args.n} C={args.csize} m={args.m}/GPU"
        gp = args.m * world
    return {"workload": wl, "func": args.func, "n": args.n, "csize": args.csize, "m_per_gpu": args.m,
            "global_points": gp, "seed": 0, "parallelism": f"dp{world}",
            "l2": f"no flush: {3 * args.m * args.n * 8 / 2**20:.0f} MiB/step > L2"}


# ------------------------------------------------------------------------- our arm
def parse_args(argv):
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
                    help="headline as strong scaling: total points split over the ranks")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-strong", action="store_true", help="skip the cfg5 strong-scaling object")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--ref-step-s", type=float, default=1.5, help="reference arm: seconds of oracle work per step")
    ap.add_argument("--sweep-out", default=os.path.join(ROOT, "gpurun_out", "bench_sweep.json"))
    ap.add_argument("--cpu-ratio-vs-n", default=None, metavar="OUT.jsonl",
                    help="only the paper's GPU-over-CPU quantity vs n (cpu_baseline leg per n), then exit")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    return args


def cpu_ratio_vs_n(out_path, funcs=("rosenbrock", "ackley", "fletcher_powell"), ns=(2, 4, 8, 16, 32, 64, 128),
                   cpu_s=0.5):
    """The paper's §VII quantity: per-point GPU time over per-point CPU time
    as n grows, for the paper's three functions.  GPU: chessfad_hvp_batch at its best C over the
    compiled set (inputs resident, CUDA events); CPU: the plain C oracle (Alg 7 as written, the
    same C) on the host cores, a bounded sample (~cpu_s per (function, n)) -- the cpu_baseline
    leg repeated per n.  One JSON line per (function, n) to out_path."""
    import torch
    import oracle
    import paper_2410_22575_b200 as chf
    dev = torch.device("cuda", 0)
    oracle.build()
    threads = oracle.default_threads()

    def gpu_rate(func, n, C, m, pr):
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

    with open(out_path, "w") as fo:
        for f in funcs:
            for n in ns:
                pr_np = synth.fp_params_flat(0, n) if f == "fletcher_powell" else None
                pr = None if pr_np is None else torch.from_numpy(pr_np).to(dev)
                m = (1 << 20) if n <= 16 else (1 << 18) if n <= 64 else (1 << 16)
                if f == "fletcher_powell":
                    m = max(4096, m >> (4 if n >= 64 else 2))
                best = None
                for C in (c for c in (1, 2, 4, 8, 16, 32, 64, 128) if c <= n and n % c == 0):
                    if chf.is_supported(f, n, C):
                        r = gpu_rate(f, n, C, m, pr)
                        if best is None or r > best[1]:
                            best = (C, r)
                C, g = best
                c, m_cpu, dt = oracle_rate(f, n, C, pr_np, 0, cpu_s, threads)
                fo.write(json.dumps({"func": f, "n": n, "C": C, "gpu_hvp_per_s": g, "gpu_m": m, "cpu_hvp_per_s": c,
                                     "cpu_points": m_cpu, "cpu_s": dt, "cpu_threads": threads,
                                     "gpu_over_cpu": g / c, "path": chf.path(f, n, C)}) + "\n")
                fo.flush()
    return 0


def main(argv=None):
    if argv is None:
        argv = json.loads(os.environ["CHESSFAD_BENCH_ARGV"]) if "CHESSFAD_BENCH_ARGV" in os.environ else sys.argv[1:]
    args = parse_args(argv)
    if args.cpu_ratio_vs_n:
        return cpu_ratio_vs_n(args.cpu_ratio_vs_n)
    rc = maybe_respawn(args, argv)
    if rc is not None:
        return rc
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    args.device_index = 0 if os.environ.get("CHESSFAD_BENCH_ONE_GPU") == "1" else local
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2410_22575_b200 as chf

    # test hook (tools/multirank_on_one_gpu.sh): every rank on GPU 0 over gloo, to exercise the
    # N > 1 logic (shards, gather, max over ranks, the line) on a one-GPU box; never a bench number
    one_gpu = os.environ.get("CHESSFAD_BENCH_ONE_GPU") == "1"
    dev_index = 0 if one_gpu else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        chf.load()  # builds if stale (file-locked); the other ranks load the result
    if world > 1:
        dist.barrier()
    chf.load()
    peaks = load_peaks()
    peak_tf, peak_mhz = fp64_nominal_tflops(peaks)

    def barrier():
        if world > 1:
            dist.barrier()

    from paper_2410_22575_b200.dist import GatherBuffer, max_over_ranks as _mor, shard

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

    def timed_steps(fn, steps, warmup, sampler=None):
        """K launches with a CUDA event between consecutive steps: (total s, per-step s list)."""
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        with (sampler if sampler is not None else _Null()):
            evs[0].record(stream)
            for k in range(steps):
                fn()
                evs[k + 1].record(stream)
            torch.cuda.synchronize()
        barrier()
        per = [evs[k].elapsed_time(evs[k + 1]) / 1e3 for k in range(steps)]
        return evs[0].elapsed_time(evs[steps]) / 1e3, per

    # ---- headline: K steps of chessfad_hvp_batch (Alg 7) on the cfg2 workload
    sampler = ClockSampler(args.device_index)
    t_loc, per_loc = timed_steps(lambda: chf.hvp_batch(args.func, pts, vec, C, params[args.func], out=out),
                                 args.steps, args.warmup, sampler)
    t = max_over_ranks(t_loc)
    per_step = t / args.steps
    step_med, step_best = max_over_ranks(float(np.median(per_loc))), max_over_ranks(min(per_loc))
    value = m_all / per_step
    flops_pt = chf.model_flops_per_point(args.func, n, C)
    model_tf = m * flops_pt / per_step / 1e12  # per GPU, one launch per step
    clocks = sampler.summary()
    if world > 1:  # per-rank clocks: median SM MHz and throttle reasons of every GPU
        allc = [None] * world
        dist.all_gather_object(allc, {"sm_mhz": clocks["sm_mhz"], "reasons": clocks["reasons"]})
        clocks["per_rank_sm_mhz"] = [c["sm_mhz"] for c in allc]
        clocks["reasons"] = sorted({r for c in allc for r in c["reasons"]})

    # ---- parity of the timed output against the oracle (rank 0: every point of its shard,
    # F3 at n > 16 on a deterministic sample)
    parity = None
    if rank == 0:
        import oracle
        full = args.func != "fletcher_powell" or n <= 16
        idx = np.arange(m) if full else np.unique(np.concatenate([[0, m - 1], np.arange(0, m, max(1, m // 509))]))
        ref, sabs = oracle.hvp_batch(args.func, P[idx], V[idx], C, params_np[args.func])
        got = out.cpu().numpy()[idx]
        err = oracle.componentwise_error(got, ref, sabs)
        parity = {"max_err": float(err.max()), "points": int(idx.size), "of": m, "bar": 1e-10,
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

    # ---- e2e through the host-buffer C-ABI call (pinned host memory, copies in the timed
    # region; CUDA events on the calling stream, which the call joins before returning)
    Ph = torch.from_numpy(P).pin_memory()
    Vh = torch.from_numpy(V).pin_memory()
    Oh = torch.empty_like(Ph).pin_memory()
    ph_params = None if params_np[args.func] is None else torch.from_numpy(params_np[args.func]).pin_memory()
    host = chf.HostPipeline()
    e2e_t, _ = timed_steps(lambda: host.hvp(args.func, Ph, Vh, C, ph_params, out=Oh), args.e2e_steps, 2)
    e2e_t = max_over_ranks(e2e_t / args.e2e_steps)
    assert torch.equal(Oh, out.cpu()), "host-buffer path disagrees with the device path"
    e2e = {"value": m_all / e2e_t, "unit": UNIT, "h2d_bytes_per_step": 2 * m * n * 8 + (
        0 if ph_params is None else ph_params.numel() * 8), "d2h_bytes_per_step": m * n * 8,
        "ms_per_step": e2e_t * 1e3, "api": "chessfad_hvp_batch_host_ctx"}
    del host

    # ---- cfg5 (BASELINE configs[4]): 2^23 points sharded over the ranks, compute-only and
    # compute + all-gather of the results (NCCL all_gather_into_tensor into one buffer)
    strong = None
    if not args.no_strong and not args.m_total:
        f5, c5 = shard(CFG5_M_TOTAL, rank, world)
        gb = GatherBuffer(CFG5_M_TOTAL, (n,), torch.float64, dev)
        p5 = torch.from_numpy(synth.points(0, n, c5, f5)).to(dev)
        v5 = torch.from_numpy(synth.vectors(0, n, c5, f5)).to(dev)
        o5 = gb.local(rank)
        ks = 10
        tc, _ = timed_steps(lambda: chf.hvp_batch(args.func, p5, v5, C, params[args.func], out=o5), ks, 3)
        tg, _ = timed_steps(lambda: (chf.hvp_batch(args.func, p5, v5, C, params[args.func], out=o5), gb.gather()),
                            ks, 3)
        tc, tg = max_over_ranks(tc) / ks, max_over_ranks(tg) / ks
        res = gb.result()
        ok = None
        if rank == 0:  # gathered rows of every rank's shard agree with a direct evaluation
            import oracle
            chk = np.unique(np.concatenate([[0, CFG5_M_TOTAL - 1], np.arange(0, CFG5_M_TOTAL, CFG5_M_TOTAL // 97)]))
            ref, sabs = oracle.hvp_batch(args.func, synth.points(0, n, CFG5_M_TOTAL)[chk],
                                         synth.vectors(0, n, CFG5_M_TOTAL)[chk], C, params_np[args.func])
            ok = bool(oracle.componentwise_error(res[chk].cpu().numpy(), ref, sabs).max() <= 1e-10)
        strong = {"workload": f"cfg5 m={CFG5_M_TOTAL}", "value": CFG5_M_TOTAL / tc, "ms": tc * 1e3, "value_with_gather": CFG5_M_TOTAL / tg,
                  "ms_with_gather": tg * 1e3, "gather": gb.kind, "gather_parity": ok}
        del gb, p5, v5, o5, res

    # ---- chunk sweep over the four functions (cfg2), Alg 7 and the NEXT rows -> sweep file
    sweep, paper_l2 = [], None
    if not args.no_sweep and world == 1:
        sweep, paper_l2 = run_sweep(chf, args, pts, vec, out, params, stream, m, m_all, peak_tf, per_step,
                                    timed_steps, max_over_ranks)

    # ---- n = 2 / 4 at m = 2^24 (inputs >> L2): the HBM-bound corner of §8(d)
    small_hbm = []
    if not args.no_sweep and world == 1:
        small_hbm = run_small_n_hbm(chf, dev, stream, timed_steps, float(peaks.get("hbm_gbs", 0.0)) or None)

    # ---- CPU baseline: the oracle on the host cores, rank 0 at N=1 only
    cpu, cpu_per_c = None, []
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        threads = oracle.default_threads()
        rate, ms, dt = oracle_rate(args.func, n, C, params_np[args.func], 0, 12.0, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"first {ms} points of the cfg2 stream: {dt:.1f} s of Alg 7 in the plain C oracle, "
                         f"{threads} pthreads"}
        if sweep:  # the paper's E5 quantity per C: oracle vs GPU per-point time, sweep file only
            gpu_rate = {r["csize"]: r["hvp_per_s"] for r in sweep if r["algo"] == "hvp" and r["func"] == args.func}
            for c in sorted(gpu_rate):
                rc, mc, dc = oracle_rate(args.func, n, c, params_np[args.func], 0, 1.5, threads)
                cpu_per_c.append({"csize": c, "oracle_hvp_per_s": rc, "sample_points": mc, "seconds": dc,
                                  "gpu_hvp_per_s": gpu_rate[c], "gpu_over_oracle": gpu_rate[c] / rc})

    # ---- roofline: executed FP64 FLOPs of this build (ncu, profiles/executed_flops.json)
    from paper_2410_22575_b200.build import source_hash
    ex = executed_entry(args.func, n, C, source_hash())
    if ex is not None and ex["basis"].startswith("STALE"):
        ex = None  # measured on other kernel SASS: no executed-FLOP claim for this build
    exec_tf = None if ex is None else m * ex["executed_flops_per_point"] / per_step / 1e12
    traffic = None if ex is None else ex["dram_bytes_per_launch"] * m / ex["m"]
    achieved = exec_tf  # None without an ncu entry for this kernel SASS (no FLOP-rate claim then)
    alg_bytes = 24 * n * m  # a1 + a7: read points and vectors, write out (§8(d))

    if rank == 0:
        sweep_best = {}
        for r in sweep:
            if r["algo"] == "hvp" and r["hvp_per_s"] > sweep_best.get(r["func"], [0, 0])[1]:
                sweep_best[r["func"]] = [r["csize"], r["hvp_per_s"]]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step * 1e3,
            "step_ms": {"median": step_med * 1e3, "best": step_best * 1e3},
            "higher_is_better": True, "scaling": "strong" if args.m_total else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload_config(args, world),
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": None if achieved is None else achieved / peak_tf,
                         "frac_executed": None if exec_tf is None else exec_tf / peak_tf,
                         "frac_model": model_tf / peak_tf,
                         "executed_over_model": None if ex is None else ex["executed_flops_per_point"] / flops_pt,
                         "model_flops_per_point": flops_pt, "traffic": traffic, "algorithmic_bytes": alg_bytes,
                         "hbm_gbs": alg_bytes / per_step / 1e9,
                         "fp64_pipe_pct_ncu": None if ex is None else ex["fp64_pipe_active_pct"],
                         "basis": "frac: ncu-executed 2*DFMA+DMUL+DADD (" + (
                             ("SASS " + ex["sass_hash"]) if ex and ex.get("sass_hash") else
                             "no ncu entry for this kernel SASS: frac null") +
                             "); frac_model: §8(d) model (DESIGN.md §5)",
                         "peak_basis": f"{SMS}x{FP64_FMA_PER_SM_CLK}x2x{peak_mhz:.0f}MHz",
                         "fp64_probe_tflops": probe_tf},
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": args.steps, "clocks": clocks, "parity": parity, "strong": strong,
            "sweep_best_hvp": sweep_best,
            "small_n_hbm_frac": {f"{r['func'][:4]} n={r['n']}": r["hbm_frac"] for r in small_hbm
                                 if r.get("best") and r["func"] != "ackley"},
            "paper_l2_speedup": None if paper_l2 is None else paper_l2["ours_over_paper_l2"],
            "sweep_file": os.path.relpath(args.sweep_out, ROOT) if sweep else None,
        }
        if sweep:
            os.makedirs(os.path.dirname(args.sweep_out), exist_ok=True)
            with open(args.sweep_out, "w") as f:
                json.dump({"headline": line, "sweep": sweep, "paper_l2_baseline": paper_l2, "small_n_hbm": small_hbm,
                           "oracle_per_csize": cpu_per_c}, f, indent=1)
        print(compact_line(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_sweep(chf, args, pts, vec, out, params, stream, m, m_all, peak_tf, per_step, timed_steps, max_over_ranks):
    """Every (algo, func, C) at the cfg2 shape, plus the paper's own Fig. 2 L2 kernel design."""
    from paper_2410_22575_b200.build import source_hash
    src_hash = source_hash()
    n = args.n
    sweep = []
    algo_fn = {"hvp": chf.hvp_batch, "sym_hvp": chf.sym_hvp_batch, "hvp_hoisted": chf.hvp_batch_hoisted,
               "hvp_seedsparse": chf.hvp_batch_seedsparse}
    for algo, fnb in algo_fn.items():
        for f in FUNCS:
            for c in (1, 2, 4, 8, 16):
                if n % c or not chf.is_supported(f, n, c, algo):
                    continue
                ks = 10
                cs_ = ClockSampler(args.device_index)
                tt, per = timed_steps(lambda: fnb(f, pts, vec, c, params[f], out=out), ks, 3, cs_)
                clk = cs_.summary()
                tt = max_over_ranks(tt) / ks
                fl = chf.model_flops_per_point(f, n, c, algo=algo)
                exs = executed_entry(f, n, c, src_hash, algo)
                ex_tf = None if exs is None else m * exs["executed_flops_per_point"] / tt / 1e12
                sweep.append({"algo": algo, "func": f, "csize": c, "hvp_per_s": m_all / tt, "ms": tt * 1e3,
                              "ms_median": float(np.median(per)) * 1e3, "ms_best": min(per) * 1e3,
                              "model_tflops_effective": m * fl / tt / 1e12, "executed_tflops": ex_tf,
                              "executed_frac": None if ex_tf is None else ex_tf / peak_tf,
                              "sm_mhz": clk["sm_mhz"], "clock_reasons": clk["reasons"]})
    paper_l2 = None
    if args.func in ("rosenbrock", "prodsum") and n in (2, 4, 8, 16):
        best = None
        for c in (1, 2, 4, 8, 16):
            if n % c:
                continue
            try:
                chf.hvp_batch_paper_l2(args.func, pts, vec, c, out=out)
            except chf.ChessfadError:
                continue
            tt, _ = timed_steps(lambda: chf.hvp_batch_paper_l2(args.func, pts, vec, c, out=out), 5, 1)
            tt = max_over_ranks(tt) / 5
            if best is None or tt < best[1]:
                best = (c, tt)
        if best:
            paper_l2 = {"kernel": "paper Fig. 2 L2 design (thread per instance x row x chunk, per-thread hDual y[n], "
                                  "shared-memory reduction), recompiled for sm_100a", "best_csize": best[0],
                        "hvp_per_s": m_all / best[1], "ms": best[1] * 1e3, "ours_over_paper_l2": best[1] / per_step}
    return sweep, paper_l2


def run_small_n_hbm(chf, dev, stream, timed_steps, hbm_peak):
    """chessfad_hvp_batch at n = 2 and 4 over m = 2^24 points (1.6 GB of traffic at n = 4,
    far beyond the 126 MB L2): algorithmic bytes 24n per point / event time vs measured HBM."""
    import torch
    m = 1 << 24
    rows = []
    for n in (2, 4):
        pts = torch.from_numpy(synth.points(0, n, m)).to(dev)
        vec = torch.from_numpy(synth.vectors(0, n, m)).to(dev)
        out = torch.empty_like(pts)
        for f in ("rosenbrock", "ackley", "prodsum"):
            best = None
            for c in (1, 2, 4):
                if n % c or not chf.is_supported(f, n, c):
                    continue
                tt, per = timed_steps(lambda: chf.hvp_batch(f, pts, vec, c, None, out=out), 10, 3)
                tt /= 10
                gbs = 24 * n * m / tt / 1e9
                r = {"func": f, "n": n, "csize": c, "m": m, "ms": tt * 1e3, "ms_median": float(np.median(per)) * 1e3,
                     "hvp_per_s": m / tt, "hbm_gbs": gbs, "hbm_frac": gbs / hbm_peak if hbm_peak else None}
                rows.append(r)
                if best is None or tt < best["ms"] / 1e3:
                    best = r
            if best is not None:
                best["best"] = True
        del pts, vec, out
    return rows


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
    if not kernel_matches_path(ent.get("kernel", ""), chf.path(func, n, C, algo if algo in chf.ALGOS else "hvp")):
        return None  # measured on a kernel family this call no longer runs
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


LINE_LIMIT = 2000  # the driver keeps the last ~4 KB of stdout; one line must fit well inside
OPTIONAL_KEYS = (("roofline", "basis"), ("roofline", "peak_basis"), (None, "sweep_file"), (None, "paper_l2_speedup"),
                 (None, "small_n_hbm_frac"), (None, "sweep_best_hvp"), ("config", "l2"))


def compact_line(line: dict, limit: int = LINE_LIMIT) -> str:
    """The final stdout line: 4-significant-digit floats, compact separators; optional
    descriptive keys are dropped (in OPTIONAL_KEYS order) until it fits in `limit` bytes."""
    line = json.loads(json.dumps(line))
    text = json.dumps(_round(line), separators=(",", ":"))
    for parent, key in OPTIONAL_KEYS:
        if len(text) <= limit:
            break
        d = line if parent is None else line.get(parent) or {}
        d.pop(key, None)
        text = json.dumps(_round(line), separators=(",", ":"))
    return text


def _round(x):
    """4 significant digits for the printed line (the sweep file keeps full precision)."""
    if isinstance(x, float):
        return float(f"{x:.4g}")
    if isinstance(x, dict):
        return {k: _round(v) for k, v in x.items()}
    if isinstance(x, list):
        return [_round(v) for v in x]
    return x


KERNEL_FAMILY = {"hvp_f3_mma_kernel": "f3_dmma", "hvp_f3_sparse_kernel": "f3_seedsparse", "hvp_f3_kernel": "f3_simt",
                 "hvp_stream_kernel": "stream", "hvp_small_kernel": "small_hoisted"}


def kernel_matches_path(kernel: str, path: str) -> bool:
    """Does a profiled kernel (demangled name) belong to the family chessfad_path reports?"""
    for prefix, fam in KERNEL_FAMILY.items():
        if prefix + "<" in kernel:
            return fam == path
    if "hvp_reg_kernel<" in kernel:
        if "SparseFunc" in kernel:
            return path == "reg_seedsparse"
        ns = kernel.split("hvp_reg_kernel<", 1)[1].split(">(", 1)[0].rsplit(",", 1)[-1].strip()
        return path == ("reg_ns" if ns not in ("0", "4") else "reg")  # last argument: NS (W on older builds)
    return False


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


if __name__ == "__main__":
    sys.exit(main())
