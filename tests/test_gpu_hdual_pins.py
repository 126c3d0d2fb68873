"""The DEVICE hDual rules (include/chessfad/hdual.cuh) and the device CHUNK-INIT seed on the
SPEC worked examples (tests/golden/spec_hdual_examples.json, each with its SPEC line), through
a one-thread test kernel (tests/cuda/hdual_pins.cu): the same exact-value checks the oracle's
primitives pass in tests/test_oracle_hdual.py (SURVEY §4 "the GPU hDual gets the same checks
through a tiny test kernel"), plus the duplicated-seed invariant."""
import ctypes
import json
import math
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_hdual_examples.json")))
OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "sadd": 4, "adds": 5, "ssub": 6, "subs": 7, "smul": 8, "divs": 9,
       "neg": 10, "sin": 11, "cos": 12, "exp": 13, "sqrt": 14, "log": 15, "abs": 16,
       "<": 17, ">": 18, "<=": 19, ">=": 20, "sdiv": 21}


@pytest.fixture(scope="module")
def lib():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    d = tempfile.mkdtemp(prefix="chessfad_hdpins_")
    so = os.path.join(d, "libhdpins.so")
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O2", "-Xcompiler",
                           "-fPIC", "-shared", "--extended-lambda", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cuda", "hdual_pins.cu"), "-o", so])
    lib = ctypes.CDLL(so)
    P = ctypes.POINTER(ctypes.c_double)
    lib.dev_hd_op.argtypes = [ctypes.c_int, ctypes.c_int, P, P, ctypes.c_double, P]
    lib.dev_chunk_init.argtypes = [ctypes.c_int, ctypes.c_int, P, ctypes.c_int, ctypes.c_int, P]
    lib.dev_seedshape.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.c_double, P]
    return lib


def _p(x):
    return x.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _num(x):
    return math.pi / 2 if x == "pi/2" else float(x)


def op(lib, name, C, u, v=None, c=0.0):
    u = np.array([_num(x) for x in u], dtype=np.float64)
    vv = None if v is None else np.array(v, dtype=np.float64)
    out = np.zeros(2 * C + 2)
    assert lib.dev_hd_op(OPS[name], C, _p(u), None if vv is None else _p(vv), float(c), _p(out)) == 0
    return out


def test_lift_binary_mixed_unary_compare(lib):
    for ex in GOLD["lift_constant"]:
        C = ex["C"]
        assert np.array_equal(op(lib, "sadd", C, [0.0] * (2 * C + 2), c=ex["c"]), ex["out"]), ex["cite"]
    for ex in GOLD["binary"]:
        assert np.array_equal(op(lib, ex["op"], ex["C"], ex["u"], ex["v"]), ex["out"]), ex["cite"]
    for ex in GOLD["mixed"]:
        assert np.array_equal(op(lib, ex["op"], ex["C"], ex["u"], c=ex["c"]), ex["out"]), ex["cite"]
    for ex in GOLD["unary"]:
        np.testing.assert_allclose(op(lib, ex["g"], ex["C"], ex["u"]), ex["out"], rtol=0, atol=ex.get("tol", 0.0),
                                   err_msg=ex["cite"])
    for ex in GOLD["compare"]:
        C = (len(ex["u"]) - 2) // 2
        assert bool(op(lib, ex["cmp"], C, ex["u"], ex["v"])[0]) == ex["out"], ex["cite"]


def test_chunk_init_seeds(lib):
    for ex in GOLD["chunk_init"]:
        n, C = len(ex["a"]), ex["C"]
        a = np.array(ex["a"], dtype=np.float64)
        out = np.zeros(n * (2 * C + 2))
        assert lib.dev_chunk_init(n, C, _p(a), ex["i"], ex["cstart"], _p(out)) == 0
        assert np.array_equal(out.reshape(n, 2 * C + 2), np.array(ex["out"], dtype=float)), ex["cite"]


def test_duplicated_seed_invariant(lib):
    """Row i inside the chunk: slot v[1] equals slot v[i-cs+2] after a sequence of operations."""
    C, n, i, cs = 2, 4, 3, 2
    a = np.array([0.3, -1.2, 0.7, 1.9])
    out = np.zeros(n * 6)
    assert lib.dev_chunk_init(n, C, _p(a), i, cs, _p(out)) == 0
    y = out.reshape(n, 6)
    t = op(lib, "mul", C, y[3], y[2])
    t = op(lib, "sin", C, t)
    t = op(lib, "add", C, t, op(lib, "mul", C, y[3], y[3]))
    assert t[1] == t[i - cs + 2]


@pytest.mark.parametrize("name", ["add", "sub", "mul", "div", "sadd", "adds", "ssub", "subs", "smul", "divs", "sdiv",
                                  "sin", "cos", "exp", "sqrt", "log", "abs"])
def test_device_rules_equal_oracle(lib, name):
    """Every device rule against the oracle's primitive (independent C code, Fig. 1 +
    SPEC.md:69-115) on random hDual<2> operands: equal up to FMA contraction (<= 4 ulps of the
    operand scale)."""
    import oracle
    rng = np.random.default_rng(7)
    un = {"sin", "cos", "exp", "sqrt", "log", "abs"}
    ops_oracle = {"add", "sub", "mul", "div", "sadd", "adds", "ssub", "subs", "smul", "divs", "sdiv"}
    for _ in range(20):
        C = 2
        u = rng.uniform(0.5, 2.0, 2 * C + 2)
        v = rng.uniform(0.5, 2.0, 2 * C + 2)
        c = float(rng.uniform(0.5, 2.0))
        got = op(lib, name, C, u, None if name in un else v, c)
        if name in un:
            ref = oracle.hd_unary(name, C, u)
        else:
            ref = oracle.hd_binary(name, C, u, None if name in ("sadd", "adds", "ssub", "subs", "smul", "divs", "sdiv")
                                   else v, c=c)
        scale = np.abs(ref).max() + 1.0
        assert np.max(np.abs(got - ref)) <= 4 * np.finfo(float).eps * scale * 8, (name, got, ref)


def test_seed_shaped_rules_equal_full(lib):
    """Reading R7: every rule with seed-shaped operands (second-order slots structural zeros,
    the terms with them omitted) equals the same rule on the operands with those zeros stored,
    for every mix of operand types: bit for bit (up to the sign of a zero) where the rule fixes
    its association with explicit FMAs (the fused forms and the componentwise rules); within
    the rounding of nvcc's contraction where it leaves the expression to it (hh*, quotient,
    unary chain rule: a dropped zero term can change which pair nvcc contracts)."""
    exact = {"add", "sub", "fma", "fnma", "axpy", "uacc", "smul", "csub"}
    rng = np.random.default_rng(11)
    names = ["add", "sub", "mul", "div", "fma", "fnma", "axpy", "sin", "exp", "sqrt", "uacc", "smul", "csub"]
    for C in (2, 4):
        N = 2 * C + 2
        for k, name in enumerate(names):
            for mode in range(8):
                for _ in range(5):
                    ops = rng.uniform(0.5, 2.0, 3 * N)
                    ops[rng.random(3 * N) < 0.3] = 0.0  # exact zeros in the stored slots too
                    ops[0] = rng.uniform(0.5, 2.0)       # u0 > 0 (sqrt, division)
                    ops[N] = rng.uniform(0.5, 2.0)       # v0 > 0
                    out = np.zeros(2 * N)
                    assert lib.dev_seedshape(k, mode, C, _p(ops), 0.75, _p(out)) == 0
                    if name in exact:
                        assert np.array_equal(out[:N], out[N:]), (name, mode, C, out[:N], out[N:])
                    else:
                        scale = np.abs(out[N:]).max() + 1.0
                        assert np.abs(out[:N] - out[N:]).max() <= 4 * np.finfo(float).eps * scale, (name, mode, C)
