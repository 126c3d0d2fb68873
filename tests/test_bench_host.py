"""Host-side logic of bench.py (no GPU): executed-FLOP accounting table lookup, stale-build
fallback, NVML throttle-reason decoding and the workload description."""
import argparse
import json

import bench


def test_executed_entry_current_and_stale(tmp_path):
    import paper_2410_22575_b200 as chf
    model = chf.model_flops_per_point("rosenbrock", 16, 16)
    tab = {"src_hash": "abc", "entries": {
        "rosenbrock n=16 C=16": {"executed_flops_per_point": 0.5 * model, "model_flops_per_point": model,
                                 "fp64_pipe_active_pct": 80.0, "dram_bytes_per_launch": 1.0, "m": 1,
                                 "kernel": "void hvp_reg_kernel<BuiltinFunc<0>, 16, 0, 4, 16>(BatchArgs, T1)"},
        "fletcher_powell n=16 C=4 sym_hvp": {"executed_flops_per_point": 10.0, "model_flops_per_point": 20.0,
                                             "fp64_pipe_active_pct": 60.0, "dram_bytes_per_launch": 1.0, "m": 1,
                                             "kernel": "void hvp_f3_mma_kernel<16, 2>(BatchArgs)"},
        "fletcher_powell n=16 C=8": {"executed_flops_per_point": 10.0, "model_flops_per_point": 20.0,
                                     "fp64_pipe_active_pct": 60.0, "dram_bytes_per_launch": 1.0, "m": 1,
                                     "kernel": "void hvp_f3_kernel<16, 0, 1, 0>(BatchArgs, const double2 *)"}}}
    p = tmp_path / "t.json"
    p.write_text(json.dumps(tab))
    e = bench.executed_entry("rosenbrock", 16, 16, "abc", path=str(p))
    assert e["executed_flops_per_point"] == 0.5 * model and "this build" in e["basis"]
    s = bench.executed_entry("rosenbrock", 16, 16, "other", path=str(p))
    assert s["basis"].startswith("STALE") and abs(s["executed_flops_per_point"] - 0.5 * model) < 1e-6
    assert bench.executed_entry("fletcher_powell", 16, 4, "abc", algo="sym_hvp", path=str(p)) is not None
    # measured on the SIMT F3 kernel, but n = 16 now runs on the tensor-core kernel: not used
    assert bench.executed_entry("fletcher_powell", 16, 8, "abc", path=str(p)) is None
    assert bench.kernel_matches_path("void hvp_stream_kernel<BuiltinFunc<0>, 1, 2>(BatchArgs, T1)", "stream")
    assert not bench.kernel_matches_path("void hvp_reg_kernel<SparseFunc<0>, 1, 0, 4>(BatchArgs, T1)", "reg")
    # the last template argument of the register kernel is NS (0: runtime n)
    assert bench.kernel_matches_path("void hvp_reg_kernel<BuiltinFunc<0>, 16, 0, 4, 16>(BatchArgs, T1)", "reg_ns")
    assert bench.kernel_matches_path("void hvp_reg_kernel<BuiltinFunc<0>, 4, 0, 4, 0>(BatchArgs, T1)", "reg")
    assert not bench.kernel_matches_path("void hvp_reg_kernel<BuiltinFunc<0>, 16, 0, 4, 0>(BatchArgs, T1)", "reg_ns")
    assert bench.executed_entry("ackley", 16, 16, "abc", path=str(p)) is None
    assert bench.executed_entry("ackley", 16, 16, "abc", path=str(tmp_path / "missing.json")) is None


def test_peak_and_config():
    tf, mhz = bench.fp64_nominal_tflops({"sm_max_mhz": 1965.0})
    assert abs(tf - 148 * 64 * 2 * 1.965e9 / 1e12) < 1e-9 and mhz == 1965.0
    a = argparse.Namespace(func="rosenbrock", n=16, csize=16, m=1 << 20, m_total=0)
    c = bench.workload_config(a, 2)
    assert c["global_points"] == 2 << 20 and "cfg2" in c["workload"]
    a.m_total = 1 << 23
    assert "cfg5" in bench.workload_config(a, 8)["workload"]


def test_clock_reason_decoding():
    cs = bench.ClockSampler.__new__(bench.ClockSampler)
    cs.ok, cs.samples, cs.max_mhz = True, [1965, 1950, 1965], 1965
    cs.reasons = 0x1 | 0x4 | 0x40
    s = cs.summary()
    assert s["sm_mhz"] == 1965 and s["reasons"] == ["sw_power_cap", "hw_thermal_slowdown"]


def test_gpus_flag_respawns_under_torchrun():
    """`bench.py --gpus 2` outside torchrun re-executes itself with 2 ranks (gloo-free: the
    reference arm needs no process group); rank 0 alone prints the line, with n_gpus = 2."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "3", "--n", "4", "--csize", "2", "--ref-step-s", "0.05"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference" and d["value"] > 0
    assert len(lines[0]) < 2048


def test_world_size_mismatch_rejected(monkeypatch):
    import pytest
    monkeypatch.setenv("WORLD_SIZE", "4")
    a = bench.parse_args(["--gpus", "2"])
    with pytest.raises(SystemExit):
        bench.maybe_respawn(a, ["--gpus", "2"])
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.maybe_respawn(a, ["--gpus", "2"]) is None


def test_compact_line_fits_driver_tail():
    """The headline line stays < 2 KB even with every optional key at worst-case length; the
    required keys survive."""
    import json
    big = 1.2345678901234567e300
    line = {"metric": bench.METRIC, "value": big, "unit": "HVP/s", "n_gpus": 8, "steps": 100, "warmup": 5,
            "ms_per_step": big, "step_ms": {"median": big, "best": big}, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "x" * 80, "func": "fletcher_powell", "n": 128, "csize": 128, "m_per_gpu": 1 << 20,
                       "global_points": 8 << 20, "seed": 0, "parallelism": "dp8", "l2": "y" * 60},
            "roofline": {k: big for k in ("achieved", "peak", "frac", "frac_executed", "frac_model",
                                          "executed_over_model", "model_flops_per_point", "traffic",
                                          "algorithmic_bytes", "hbm_gbs", "fp64_pipe_pct_ncu", "fp64_probe_tflops")},
            "cpu_baseline": {"value": big, "unit": "HVP/s", "cores": 64, "kind": "oracle", "sample": "z" * 120},
            "e2e": {"value": big, "unit": "HVP/s", "h2d_bytes_per_step": 1 << 40, "d2h_bytes_per_step": 1 << 40,
                    "ms_per_step": big, "api": "chessfad_hvp_batch_host_ctx"},
            "gpu_launches": 100, "clocks": {"sm_mhz": 1965.0, "sm_max_mhz": 1965, "reasons": ["sw_power_cap"] * 3,
                                            "samples": 99},
            "parity": {"max_err": big, "points": 1 << 20, "of": 1 << 20, "bar": 1e-10, "pass": True},
            "strong": {"workload": "cfg5 m=8388608", "value": big, "ms": big, "value_with_gather": big,
                       "ms_with_gather": big, "gather": "all_gather_into_tensor in place", "gather_parity": True},
            "sweep_best_hvp": {f: [16, big] for f in ("rosenbrock", "ackley", "fletcher_powell", "prodsum")},
            "small_n_hbm_frac": {f"f{i}": big for i in range(4)}, "paper_l2_speedup": big,
            "sweep_file": "gpurun_out/bench_sweep.json"}
    line["roofline"].update({"bound": "alu", "unit": "TFLOP/s", "basis": "b" * 120, "peak_basis": "p" * 40})
    text = bench.compact_line(line)
    assert len(text) < 2048
    d = json.loads(text)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "roofline", "cpu_baseline",
              "e2e", "gpu_launches", "clocks", "parity", "config"):
        assert k in d
    assert d["roofline"]["frac"] == float(f"{big:.4g}")
