"""The C-ABI library loads and exports every symbol include/chessfad.h declares; argument
validation and the model-FLOP count work without a GPU (no compute call is made)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import paper_2410_22575_b200 as chf
    return chf.load()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "chessfad.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(chessfad_\w+)\s*\(", hdr)))


def test_exports_every_declared_symbol(lib):
    import paper_2410_22575_b200 as chf
    syms = declared_symbols()
    assert len(syms) >= 8
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(chf.EXPORTS) == syms


def test_sm100a_cubin_embedded():
    """The library carries sm_100a SASS (cuobjdump lists the ELF arch)."""
    import shutil
    import subprocess
    import paper_2410_22575_b200 as chf
    chf.load()
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", chf.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_and_version(lib):
    import paper_2410_22575_b200 as chf
    assert "sm_100a" in chf.version()
    for st in range(6):
        assert lib.chessfad_status_string(st).decode().startswith("CHESSFAD")


def _call(lib, func, n, C, m, pts=1, vec=1, out=1, params=None):
    vp = lambda x: None if x is None else ctypes.c_void_p(x)
    return lib.chessfad_hvp_batch(func, n, C, m, vp(pts), vp(vec), vp(out), vp(params), None)


def test_argument_errors(lib):
    assert _call(lib, 0, 0, 1, 10) == 1          # n < 1
    assert _call(lib, 0, 4, 1, -1) == 1          # m < 0
    assert _call(lib, 0, 4, 1, 10, pts=None) == 1  # NULL with m > 0
    assert _call(lib, 0, 4, 3, 10) == 2          # C does not divide n
    assert _call(lib, 0, 4, 0, 10) == 2          # C < 1
    assert _call(lib, 0, 4, 8, 10) == 2          # C > n
    assert _call(lib, 0, 1, 1, 10) == 3          # Rosenbrock n < 2
    assert _call(lib, 3, 1, 1, 10) == 3          # prodsum n < 2
    assert _call(lib, 9, 4, 1, 10) == 3          # unknown func
    assert _call(lib, 2, 4, 1, 10, params=None) == 3  # F3 without params
    assert _call(lib, 0, 512, 1, 10) == 4        # n beyond the compiled set
    assert _call(lib, 0, 4, 1, 0, None, None, None) == 0  # m == 0: empty no-op, no CUDA call
    assert lib.chessfad_hessian_batch(0, 4, 3, 10, ctypes.c_void_p(1), ctypes.c_void_p(1), None, None) == 2


def test_is_supported(lib):
    import paper_2410_22575_b200 as chf
    assert chf.is_supported("rosenbrock", 16, 4)
    assert not chf.is_supported("rosenbrock", 16, 3)   # 3 does not divide 16
    assert chf.is_supported("rosenbrock", 12, 3)       # column groups of 1
    assert chf.is_supported("rosenbrock", 128, 64)     # column groups of 16
    assert not chf.is_supported("ackley", 256, 16)     # shared-memory budget
    assert chf.is_supported("fletcher_powell", 12, 3)  # runtime-C schedule
    assert chf.is_supported("fletcher_powell", 128, 8)
    assert not chf.is_supported("fletcher_powell", 256, 8)


FUNCS = ["rosenbrock", "ackley", "fletcher_powell", "prodsum"]


@pytest.mark.parametrize("func", FUNCS)
@pytest.mark.parametrize("n,C", [(2, 1), (4, 2), (8, 4), (6, 6)])
def test_model_flops_match_oracle_counts(func, n, C):
    """chessfad_model_flops_per_point (library) == scalar mul+add counted by the oracle's
    counting build running Alg 7 (independent code, same Fig. 1 / §V accounting)."""
    import paper_2410_22575_b200 as chf
    params = synth.fp_params_flat(0, n) if func == "fletcher_powell" else None
    a = synth.points(0, n, 1)[0] + 3.0
    _, c = oracle.count(oracle.chess_vec, func, a, a, C, params)
    assert chf.model_flops_per_point(func, n, C) == c["mul"] + c["add"]
    _, c = oracle.count(oracle.hessian, func, a, params, algo="chunk", C=C)
    assert chf.model_flops_per_point(func, n, C, hessian=True) == c["mul"] + c["add"]


def test_model_flops_survey_table():
    """Spot values of SURVEY §8(d)'s model-FLOP table."""
    import paper_2410_22575_b200 as chf
    assert chf.model_flops_per_point("rosenbrock", 2, 1) == 228
    assert chf.model_flops_per_point("rosenbrock", 16, 1) == 226048
    assert chf.model_flops_per_point("rosenbrock", 16, 16) == 150928
    assert chf.model_flops_per_point("ackley", 16, 4) == 100160
    assert chf.model_flops_per_point("fletcher_powell", 16, 2) == pytest.approx(878e3, rel=1e-3)


@pytest.mark.parametrize("func", FUNCS)
@pytest.mark.parametrize("n,C", [(4, 2), (8, 2), (6, 3), (8, 8)])
def test_model_flops_symmetric_match_oracle_counts(func, n, C):
    """Alg 8 / Alg 6 model (n(n/C+1)/2 evaluations; 2n^2 dot for Alg 8) ==
    the oracle's counting build."""
    import paper_2410_22575_b200 as chf
    params = synth.fp_params_flat(0, n) if func == "fletcher_powell" else None
    a = synth.points(0, n, 1)[0] + 3.0
    _, c = oracle.count(oracle.sc_hess_vec, func, a, a, C, params)
    assert chf.model_flops_per_point(func, n, C, algo="sym_hvp") == c["mul"] + c["add"]
    _, c = oracle.count(oracle.hessian, func, a, params, algo="schunk", C=C)
    assert chf.model_flops_per_point(func, n, C, algo="sym_hessian") == c["mul"] + c["add"]
    assert chf.model_flops_per_point(func, n, C, algo="hvp") == chf.model_flops_per_point(func, n, C)


def test_symmetric_support():
    import paper_2410_22575_b200 as chf
    for algo in ("hvp", "hessian", "sym_hvp", "sym_hessian"):
        assert chf.is_supported("rosenbrock", 16, 4, algo)
        assert chf.is_supported("fletcher_powell", 16, 4, algo)
    assert not chf.is_supported("rosenbrock", 16, 3, "sym_hvp")


def test_host_workspace_contract(lib):
    """chessfad_hvp_batch_host rejects a too-small caller workspace before touching the GPU;
    the size query is monotone in m."""
    import paper_2410_22575_b200 as chf
    need = lib.chessfad_hvp_host_workspace_bytes(0, 16, 1 << 20, 0)
    assert need >= 3 * 3 * (1 << 16) * 16 * 8
    assert lib.chessfad_hvp_host_workspace_bytes(2, 16, 1000, 100) > lib.chessfad_hvp_host_workspace_bytes(0, 16, 1000, 100)
    vp = ctypes.c_void_p
    st = lib.chessfad_hvp_batch_host(0, 16, 4, 1000, vp(1), vp(1), vp(1), None, 0, vp(1), 16, None)
    assert st == 1  # ERR_ARG
    assert chf.STATUS[st] == "CHESSFAD_ERR_ARG"


def test_hoisted_contract():
    """NEXT-4 entry point: every function; its model count is the paper's Alg 7 count."""
    import paper_2410_22575_b200 as chf
    assert chf.is_supported("fletcher_powell", 16, 4, "hvp_hoisted")
    assert chf.is_supported("fletcher_powell", 64, 16, "hvp_hoisted")
    assert chf.is_supported("rosenbrock", 16, 4, "hvp_hoisted")
    assert chf.is_supported("ackley", 12, 3, "hvp_hoisted")  # no hoisted kernel: per-evaluation path
    assert chf.model_flops_per_point("fletcher_powell", 16, 4, algo="hvp_hoisted") == \
        chf.model_flops_per_point("fletcher_powell", 16, 4)


def test_seedsparse_contract(lib):
    """NEXT-4 seed sparsity: every function (F3: n <= 128), any valid C; errors before CUDA."""
    import paper_2410_22575_b200 as chf
    for n, C in ((2, 1), (16, 4), (16, 16), (64, 8), (128, 128), (12, 3)):
        assert chf.is_supported("fletcher_powell", n, C, "hvp_seedsparse")
    assert not chf.is_supported("fletcher_powell", 256, 16, "hvp_seedsparse")
    for f in ("rosenbrock", "ackley", "prodsum"):
        assert chf.is_supported(f, 16, 4, "hvp_seedsparse")
        assert chf.is_supported(f, 128, 32, "hessian_seedsparse")
    assert chf.model_flops_per_point("fletcher_powell", 16, 4, algo="hvp_seedsparse") == \
        chf.model_flops_per_point("fletcher_powell", 16, 4)
    vp = ctypes.c_void_p
    f = lib.chessfad_hvp_batch_seedsparse
    assert f(0, 1, 1, 10, vp(1), vp(1), vp(1), None, None) == 3  # Rosenbrock n = 1: ERR_FUNC
    assert f(2, 16, 4, 10, vp(1), vp(1), vp(1), None, None) == 3  # F3 without params: ERR_FUNC
    assert f(2, 16, 3, 10, vp(1), vp(1), vp(1), vp(1), None) == 2  # 3 does not divide 16: ERR_CHUNK
    assert f(2, 16, 4, 0, None, None, None, vp(1), None) == 0     # m = 0: no-op
    h = lib.chessfad_hessian_batch_seedsparse
    assert chf.is_supported("fletcher_powell", 32, 4, "hessian_seedsparse")
    assert h(9, 16, 4, 10, vp(1), vp(1), None, None) == 3  # unknown function: ERR_FUNC
    assert h(2, 16, 4, 10, vp(1), None, vp(1), None) == 1  # NULL hess: ERR_ARG
    assert chf.model_flops_per_point("fletcher_powell", 32, 4, algo="hessian_seedsparse") == \
        chf.model_flops_per_point("fletcher_powell", 32, 4, hessian=True)


def test_hessian_grad_contract(lib):
    import paper_2410_22575_b200 as chf
    assert chf.is_supported("rosenbrock", 16, 4, "hessian_grad")
    assert chf.model_flops_per_point("ackley", 16, 4, algo="hessian_grad") == \
        chf.model_flops_per_point("ackley", 16, 4, hessian=True)
    vp = ctypes.c_void_p
    # grad NULL with m > 0 -> ERR_ARG, before any CUDA call
    assert lib.chessfad_hessian_grad_batch(0, 16, 4, 10, vp(1), vp(1), None, None, None) == 1


def test_kernel_path_introspection():
    """chessfad_path names the kernel family each call runs."""
    import paper_2410_22575_b200 as chf
    assert chf.path("fletcher_powell", 16, 4) == "f3_dmma"
    assert chf.path("fletcher_powell", 64, 8, "sym_hvp") == "f3_dmma"
    assert chf.path("fletcher_powell", 128, 8) == "f3_dmma"
    assert chf.path("fletcher_powell", 12, 4) == "f3_dmma"   # zero-padded to 16
    assert chf.path("fletcher_powell", 128, 8, "sym_hvp") == "f3_dmma"
    assert chf.path("fletcher_powell", 4, 2) == "f3_dmma"    # zero-padded to 8
    assert chf.path("fletcher_powell", 100, 4, "sym_hvp") == "f3_dmma"
    assert chf.path("fletcher_powell", 16, 4, "hvp_seedsparse") == "f3_seedsparse"
    assert chf.path("rosenbrock", 2, 1) == "stream"
    assert chf.path("rosenbrock", 16, 16) == "reg_ns" and chf.path("rosenbrock", 12, 4) == "reg"
    assert chf.path("ackley", 8, 1) == "reg_ns" and chf.path("prodsum", 8, 4) == "stream"
    assert chf.path("ackley", 4, 1) == "stream" and chf.path("rosenbrock", 8, 8) == "reg_ns"
    assert chf.path("prodsum", 32, 32) == "reg_ns" and chf.path("prodsum", 64, 16) == "reg_ns"
    assert chf.path("prodsum", 32, 4, "hessian") == "reg" and chf.path("rosenbrock", 32, 4, "hessian") == "reg_ns"
    assert chf.path("rosenbrock", 128, 2) == "reg" and chf.path("rosenbrock", 64, 1) == "reg_ns"
    assert chf.path("ackley", 128, 16) == "reg" and chf.path("ackley", 64, 64) == "reg_ns"
    assert chf.path("ackley", 128, 8) == "reg_ns"
    assert chf.path("rosenbrock", 64, 16, "sym_hvp") == "reg" and chf.path("rosenbrock", 16, 16, "sym_hvp") == "reg_ns"
    assert chf.path("rosenbrock", 8, 2, "hvp_hoisted") == "small_hoisted"
    assert chf.path("rosenbrock", 3, 2) == "unsupported"


def test_device_header_self_contained(tmp_path):
    """include/chessfad_device.cuh (user functions, NEXT-3) compiles from include/ alone: a copy
    of include/ outside the repo and the example translation unit, nothing else."""
    import shutil
    import subprocess
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    inc = tmp_path / "include"
    shutil.copytree(os.path.join(ROOT, "include"), inc)
    src = tmp_path / "user.cu"
    shutil.copy(os.path.join(ROOT, "examples", "user_function.cu"), src)
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O1", "-I", str(inc),
                        "-c", str(src), "-o", str(tmp_path / "user.o")], capture_output=True, text=True, cwd=tmp_path)
    assert r.returncode == 0, r.stderr[-3000:]


def test_seedsparse_symmetric_contract(lib):
    """Seed-sparse Alg 8 / Alg 6 / gradient: every function (Alg 8 for Fletcher-Powell up to
    n = 64); model = the algorithm's."""
    import paper_2410_22575_b200 as chf
    for algo in ("sym_hvp_seedsparse", "sym_hessian_seedsparse", "hessian_grad_seedsparse"):
        assert chf.is_supported("rosenbrock", 16, 4, algo)
        assert chf.is_supported("fletcher_powell", 16, 4, algo)
        assert chf.is_supported("fletcher_powell", 64, 8, algo)
    assert not chf.is_supported("fletcher_powell", 72, 8, "sym_hvp_seedsparse")
    for algo in ("sym_hvp_seedsparse", "sym_hessian_seedsparse", "hessian_grad_seedsparse"):
        assert chf.path("ackley", 16, 4, algo) == "reg_seedsparse"
    assert chf.model_flops_per_point("rosenbrock", 16, 4, algo="sym_hvp_seedsparse") == \
        chf.model_flops_per_point("rosenbrock", 16, 4, algo="sym_hvp")
    vp = ctypes.c_void_p
    assert lib.chessfad_hessian_grad_batch_seedsparse(0, 16, 4, 10, vp(1), vp(1), None, None, None) == 1
    # Fletcher-Powell seed-sparse Alg 8 beyond n = 64: refused before anything is touched
    assert lib.chessfad_sym_hvp_batch_seedsparse(2, 72, 8, 10, vp(1), vp(1), vp(1), vp(1), None) == 4


def test_seed_type_rules_compile(tmp_path):
    """Reading R7 at the type level: the result types of every hDual rule with seed-shaped
    operands (static_asserts in tests/cuda/seed_type_rules.cu; compile-only, no GPU)."""
    import shutil
    import subprocess
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O1", "-I",
                        os.path.join(root, "include"), "-c", os.path.join(root, "tests", "cuda", "seed_type_rules.cu"),
                        "-o", str(tmp_path / "rules.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
