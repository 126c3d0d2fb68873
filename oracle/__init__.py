"""CPU oracle for the CHESSFAD batched FP64 Hessian-vector product -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  It wraps ``chessfad_oracle.c`` (plain
C, -O2 -ffp-contract=off) through ctypes and shares no code with the CUDA product path.
See the C file's header for what it computes and which PAPER.md passages it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "chessfad_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
LIB_COUNT = os.path.join(HERE, "liboracle_count.so")

ROSENBROCK, ACKLEY, FLETCHER_POWELL, PRODSUM = 0, 1, 2, 3
FUNCS = {"rosenbrock": ROSENBROCK, "ackley": ACKLEY, "fletcher_powell": FLETCHER_POWELL, "prodsum": PRODSUM}
OP = {"add": 0, "sub": 1, "mul": 2, "div": 3, "sadd": 4, "adds": 5, "ssub": 6, "subs": 7,
      "smul": 8, "divs": 9, "sdiv": 10, "neg": 11}
G = {"sin": 0, "cos": 1, "exp": 2, "sqrt": 3, "log": 4, "abs": 5}
CMP = {"<": 0, ">": 1, "<=": 2, ">=": 3, "==": 4}
STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_CHUNK", 3: "ERR_FUNC"}

_lock = threading.Lock()
_libs: dict = {}


class OracleError(RuntimeError):
    pass


def _cflags():
    return ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
            "-pthread", "-Wall"]


def build(force: bool = False) -> None:
    """Compile liboracle.so and the counting build liboracle_count.so (plain gcc)."""
    hdr = os.path.join(HERE, "chessfad_oracle.h")
    newest = max(os.path.getmtime(SRC), os.path.getmtime(hdr))
    for out, extra in ((LIB, []), (LIB_COUNT, ["-DOR_COUNTING"])):
        if force or not os.path.exists(out) or os.path.getmtime(out) < newest:
            tmp = out + f".tmp{os.getpid()}"
            subprocess.check_call(_cflags() + extra + [SRC, "-o", tmp, "-lm"])
            os.replace(tmp, out)


def _load(counting: bool = False):
    key = "count" if counting else "plain"
    with _lock:
        if key in _libs:
            return _libs[key]
        build()
        lib = ctypes.CDLL(LIB_COUNT if counting else LIB)
        P = ctypes.POINTER(ctypes.c_double)
        i32, i64, dbl = ctypes.c_int, ctypes.c_int64, ctypes.c_double
        sig = {
            "or_hd_binary": (i32, [i32, i32, P, P, dbl, P]),
            "or_hd_unary": (i32, [i32, i32, P, P]),
            "or_hd_compare": (i32, [i32, P, P]),
            "or_initialize": (None, [i32, P, i32, i32, P]),
            "or_chunk_init": (None, [i32, P, i32, i32, i32, P]),
            "or_eval_hdual": (i32, [i32, i32, P, i32, P, P]),
            "or_eval_scalar": (i32, [i32, i32, P, P, P]),
            "or_hessian": (i32, [i32, i32, P, P, P]),
            "or_sym_hessian": (i32, [i32, i32, P, P, P]),
            "or_chunk_hess": (i32, [i32, i32, i32, P, P, P, P]),
            "or_schunk_hess": (i32, [i32, i32, i32, P, P, P, P]),
            "or_chess_vec": (i32, [i32, i32, i32, P, P, P, P, P]),
            "or_sc_hess_vec": (i32, [i32, i32, i32, P, P, P, P]),
            "or_full_scheme_hessian": (i32, [i32, i32, P, P, P, P]),
            "or_hvp_batch": (i32, [i32, i32, i32, i64, P, P, P, P, P, i32]),
            "or_sc_hvp_batch": (i32, [i32, i32, i32, i64, P, P, P, P, i32]),
            "or_hessian_batch": (i32, [i32, i32, i32, i64, P, P, P, i32]),
            "or_counters_reset": (None, []),
            "or_counters_get": (None, [ctypes.POINTER(i64)] * 3),
            "or_is_counting_build": (i32, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _libs[key] = lib
        return lib


def _p(x):
    if x is None:
        return None
    assert x.dtype == np.float64 and x.flags["C_CONTIGUOUS"]
    return x.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(x):
    return None if x is None else np.ascontiguousarray(x, dtype=np.float64)


def _check(st):
    if st != 0:
        raise OracleError(STATUS.get(st, str(st)))


def _func(f):
    return FUNCS[f] if isinstance(f, str) else int(f)


# ----------------------------------------------------------------- hDual primitives
def hd_binary(op: str, C: int, u=None, v=None, c: float = 0.0):
    ncomp = 2 * C + 2
    u = _f64(u if u is not None else np.zeros(ncomp))
    v = _f64(v if v is not None else np.zeros(ncomp))
    r = np.zeros(ncomp)
    _check(_load().or_hd_binary(OP[op], C, _p(u), _p(v), c, _p(r)))
    return r


def hd_unary(g: str, C: int, u):
    u = _f64(u)
    r = np.zeros(2 * C + 2)
    _check(_load().or_hd_unary(G[g], C, _p(u), _p(r)))
    return r


def hd_compare(cmp: str, u, v) -> bool:
    u, v = _f64(u), _f64(v)
    return bool(_load().or_hd_compare(CMP[cmp], _p(u), _p(v)))


def initialize(a, i: int, j: int):
    a = _f64(a)
    n = a.size
    y = np.zeros((n, 4))
    _load().or_initialize(n, _p(a), i, j, _p(y))
    return y


def chunk_init(a, i: int, cstart: int, C: int):
    a = _f64(a)
    n = a.size
    y = np.zeros((n, 2 * C + 2))
    _load().or_chunk_init(n, _p(a), i, cstart, C, _p(y))
    return y


def eval_hdual(func, y, C: int, params=None, counting: bool = False):
    y = _f64(y)
    n = y.shape[0]
    t = np.zeros(2 * C + 2)
    _check(_load(counting).or_eval_hdual(_func(func), n, _p(_f64(params)), C, _p(y), _p(t)))
    return t


def eval_scalar(func, x, params=None) -> float:
    x = _f64(x)
    f = np.zeros(1)
    _check(_load().or_eval_scalar(_func(func), x.size, _p(_f64(params)), _p(x), _p(f)))
    return float(f[0])


# ----------------------------------------------------------------- single point
def hessian(func, a, params=None, algo: str = "chunk", C: int = 1, counting: bool = False):
    """algo in {full (Alg 2), sym (Alg 3), chunk (Alg 5), schunk (Alg 6), scheme}."""
    a = _f64(a)
    n = a.size
    H = np.zeros((n, n))
    grad = np.zeros(n)
    lib = _load(counting)
    pp = _p(_f64(params))
    f = _func(func)
    if algo == "full":
        _check(lib.or_hessian(f, n, pp, _p(a), _p(H)))
    elif algo == "sym":
        _check(lib.or_sym_hessian(f, n, pp, _p(a), _p(H)))
    elif algo == "chunk":
        _check(lib.or_chunk_hess(f, n, C, pp, _p(a), _p(H), _p(grad)))
    elif algo == "schunk":
        _check(lib.or_schunk_hess(f, n, C, pp, _p(a), _p(H), _p(grad)))
    elif algo == "scheme":
        _check(lib.or_full_scheme_hessian(f, n, pp, _p(a), _p(H), _p(grad)))
    else:
        raise ValueError(algo)
    return H, grad


def chess_vec(func, a, v, C: int, params=None, counting: bool = False):
    """Alg 7 for one point: returns (out, sabs)."""
    a, v = _f64(a), _f64(v)
    n = a.size
    out, sabs = np.zeros(n), np.zeros(n)
    _check(_load(counting).or_chess_vec(_func(func), n, C, _p(_f64(params)), _p(a), _p(v), _p(out), _p(sabs)))
    return out, sabs


def sc_hess_vec(func, a, v, C: int, params=None, counting: bool = False):
    a, v = _f64(a), _f64(v)
    out = np.zeros(a.size)
    _check(_load(counting).or_sc_hess_vec(_func(func), a.size, C, _p(_f64(params)), _p(a), _p(v), _p(out)))
    return out


# ----------------------------------------------------------------- batches
def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def hvp_batch(func, points, vecs, C: int, params=None, threads: int | None = None):
    """Alg 7 over m points (pthreads over contiguous point ranges): (out, sabs)."""
    points, vecs = _f64(points), _f64(vecs)
    m, n = points.shape
    out, sabs = np.zeros((m, n)), np.zeros((m, n))
    _check(_load().or_hvp_batch(_func(func), n, C, m, _p(points), _p(vecs), _p(out), _p(sabs),
                                _p(_f64(params)), threads or default_threads()))
    return out, sabs


def sc_hvp_batch(func, points, vecs, C: int, params=None, threads: int | None = None):
    points, vecs = _f64(points), _f64(vecs)
    m, n = points.shape
    out = np.zeros((m, n))
    _check(_load().or_sc_hvp_batch(_func(func), n, C, m, _p(points), _p(vecs), _p(out),
                                   _p(_f64(params)), threads or default_threads()))
    return out


def hessian_batch(func, points, C: int, params=None, threads: int | None = None):
    points = _f64(points)
    m, n = points.shape
    H = np.zeros((m, n, n))
    _check(_load().or_hessian_batch(_func(func), n, C, m, _p(points), _p(H), _p(_f64(params)),
                                    threads or default_threads()))
    return H


# ----------------------------------------------------------------- counting
def counters_reset(counting: bool = True):
    _load(counting).or_counters_reset()


def counters(counting: bool = True):
    e, mu, ad = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _load(counting).or_counters_get(ctypes.byref(e), ctypes.byref(mu), ctypes.byref(ad))
    return {"evals": e.value, "mul": mu.value, "add": ad.value}


def count(fn, *args, **kw):
    """Run an oracle call on the counting build and return (result, counters)."""
    counters_reset(True)
    res = fn(*args, counting=True, **kw)
    return res, counters(True)


# ----------------------------------------------------------------- error metric
def componentwise_error(gpu, ref, sabs):
    """err = |g - r| / max(|r|, s), s = sum_j |H_ij||in_j| (DESIGN.md parity metric)."""
    gpu, ref, sabs = np.asarray(gpu), np.asarray(ref), np.asarray(sabs)
    den = np.maximum(np.abs(ref), sabs)
    diff = np.abs(gpu - ref)
    with np.errstate(invalid="ignore", divide="ignore"):
        err = np.where(den > 0, diff / np.where(den > 0, den, 1.0), np.where(diff > 0, np.inf, 0.0))
    return err
