"""chessfad-b200: B200-native batched FP64 Hessian-vector products (CHESSFAD, arXiv 2410.22575).

Thin Python binding over the C-ABI of ``libchessfad.so`` (``include/chessfad.h``):
argument marshalling only -- every step of the hot path runs in the library's CUDA
kernels.  PyTorch supplies device memory and streams.  There is no CPU fallback: if the
library cannot be loaded the calls raise.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CHESSFAD_LIB") or os.path.join(HERE, "libchessfad.so")  # override: experiments

ROSENBROCK, ACKLEY, FLETCHER_POWELL, PRODSUM = 0, 1, 2, 3
FUNCS = {"rosenbrock": ROSENBROCK, "ackley": ACKLEY, "fletcher_powell": FLETCHER_POWELL, "prodsum": PRODSUM}
STATUS = {0: "CHESSFAD_OK", 1: "CHESSFAD_ERR_ARG", 2: "CHESSFAD_ERR_CHUNK", 3: "CHESSFAD_ERR_FUNC",
          4: "CHESSFAD_ERR_UNSUPPORTED", 5: "CHESSFAD_ERR_CUDA"}
ALGOS = {"hvp": 0, "hessian": 1, "sym_hvp": 2, "sym_hessian": 3, "hvp_hoisted": 4, "hessian_grad": 5, "hvp_seedsparse": 6,
         "hessian_seedsparse": 7, "sym_hvp_seedsparse": 8, "sym_hessian_seedsparse": 9, "hessian_grad_seedsparse": 10}
EXPORTS = sorted(["chessfad_hvp_batch", "chessfad_hessian_batch", "chessfad_sym_hvp_batch", "chessfad_sym_hessian_batch",
                  "chessfad_hvp_batch_host", "chessfad_is_supported", "chessfad_is_supported_algo",
                  "chessfad_status_string", "chessfad_model_flops_per_point", "chessfad_model_flops_per_point_algo",
                  "chessfad_fp64_probe", "chessfad_version", "chessfad_hvp_host_workspace_bytes",
                  "chessfad_hvp_batch_hoisted", "chessfad_hvp_batch_seedsparse", "chessfad_hessian_batch_seedsparse", "chessfad_hvp_batch_paper_l2", "chessfad_hessian_grad_batch",
                  "chessfad_hvp_batch_paper", "chessfad_host_ctx_create", "chessfad_host_ctx_destroy",
                  "chessfad_hvp_batch_host_ctx", "chessfad_path", "chessfad_sym_hvp_batch_seedsparse",
                  "chessfad_sym_hessian_batch_seedsparse", "chessfad_hessian_grad_batch_seedsparse"])

_lock = threading.Lock()
_lib = None


class ChessfadError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}{': ' + msg if msg else ''}")


def load(build_if_missing: bool = True):
    """Load libchessfad.so (building it in-tree with nvcc if it is missing or stale)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        from . import build as _build
        if build_if_missing and not os.environ.get("CHESSFAD_LIB") and not _build.up_to_date():
            _build.build()
        if not os.path.exists(LIB_PATH):
            raise ChessfadError(5, f"{LIB_PATH} not built; run paper_2410_22575_b200/build.py")
        lib = ctypes.CDLL(LIB_PATH)
        i32, i64, dbl, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        sig = {
            "chessfad_hvp_batch": (i32, [i32, i32, i32, i64, vp, vp, vp, vp, vp]),
            "chessfad_hessian_batch": (i32, [i32, i32, i32, i64, vp, vp, vp, vp]),
            "chessfad_sym_hvp_batch": (i32, [i32, i32, i32, i64, vp, vp, vp, vp, vp]),
            "chessfad_hvp_batch_hoisted": (i32, [i32, i32, i32, i64, vp, vp, vp, vp, vp]),
            "chessfad_hvp_batch_seedsparse": (i32, [i32, i32, i32, i64, vp, vp, vp, vp, vp]),
            "chessfad_hessian_batch_seedsparse": (i32, [i32, i32, i32, i64, vp, vp, vp, vp]),
            "chessfad_sym_hvp_batch_seedsparse": (i32, [i32, i32, i32, i64, vp, vp, vp, vp, vp]),
            "chessfad_sym_hessian_batch_seedsparse": (i32, [i32, i32, i32, i64, vp, vp, vp, vp]),
            "chessfad_hessian_grad_batch_seedsparse": (i32, [i32, i32, i32, i64, vp, vp, vp, vp, vp]),
            "chessfad_hessian_grad_batch": (i32, [i32, i32, i32, i64, vp, vp, vp, vp, vp]),
            "chessfad_hvp_batch_paper_l2": (i32, [i32, i32, i32, i64, vp, vp, vp, vp]),
            "chessfad_hvp_batch_paper": (i32, [i32, i32, i32, i32, i64, vp, vp, vp, vp]),
            "chessfad_sym_hessian_batch": (i32, [i32, i32, i32, i64, vp, vp, vp, vp]),
            "chessfad_is_supported_algo": (i32, [i32, i32, i32, i32]),
            "chessfad_model_flops_per_point_algo": (dbl, [i32, i32, i32, i32]),
            "chessfad_hvp_batch_host": (i32, [i32, i32, i32, i64, vp, vp, vp, vp, i64, vp, ctypes.c_size_t, vp]),
            "chessfad_hvp_host_workspace_bytes": (ctypes.c_size_t, [i32, i32, i64, i64]),
            "chessfad_host_ctx_create": (i32, [ctypes.POINTER(vp)]),
            "chessfad_host_ctx_destroy": (i32, [vp]),
            "chessfad_hvp_batch_host_ctx": (i32, [vp, i32, i32, i32, i64, vp, vp, vp, vp, i64, vp, ctypes.c_size_t,
                                                  vp]),
            "chessfad_is_supported": (i32, [i32, i32, i32]),
            "chessfad_status_string": (ctypes.c_char_p, [i32]),
            "chessfad_model_flops_per_point": (dbl, [i32, i32, i32, i32]),
            "chessfad_fp64_probe": (i32, [i32, i64, vp, vp]),
            "chessfad_version": (ctypes.c_char_p, []),
            "chessfad_path": (ctypes.c_char_p, [i32, i32, i32, i32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
        return lib


def _func(f) -> int:
    return FUNCS[f] if isinstance(f, str) else int(f)


def _check(st: int):
    if st != 0:
        raise ChessfadError(st, load().chessfad_status_string(st).decode())


def _stream_ptr(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dev(t, name, shape=None):
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous float64 CUDA tensor")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    return ctypes.c_void_p(t.data_ptr())


def _params_shape(func, n):
    """Fletcher-Powell params: [A (n x n) | B (n x n) | E* (n)] = 2n^2+n doubles; else ignored."""
    return (2 * n * n + n,) if _func(func) == FLETCHER_POWELL else None


def _dev_params(params, func, n):
    shp = _params_shape(func, n)
    if params is not None and shp is not None and params.numel() != shp[0]:
        raise ValueError(f"params has {params.numel()} elements, expected 2n^2+n = {shp[0]}")
    return _dev(params, "params")


def _points_2d(points):
    if points.dim() != 2:
        raise ValueError(f"points must be (m, n), got shape {tuple(points.shape)}")
    return points.shape


def _hvp(entry, func, points, vecs, csize, params, out, stream):
    import torch
    m, n = _points_2d(points)
    if out is None:
        out = torch.empty_like(points)
    st = getattr(load(), entry)(_func(func), n, csize, m, _dev(points, "points"), _dev(vecs, "vecs", (m, n)),
                                _dev(out, "out", (m, n)), _dev_params(params, func, n), _stream_ptr(stream))
    _check(st)
    return out


def _hess(entry, func, points, csize, params, out, stream):
    import torch
    m, n = _points_2d(points)
    if out is None:
        out = torch.empty((m, n, n), dtype=torch.float64, device=points.device)
    st = getattr(load(), entry)(_func(func), n, csize, m, _dev(points, "points"), _dev(out, "hess", (m, n, n)),
                                _dev_params(params, func, n), _stream_ptr(stream))
    _check(st)
    return out


def hvp_batch(func, points, vecs, csize: int, params=None, out=None, stream=None):
    """out[e] = Hess f(points[e]) @ vecs[e] for every row e (Alg 7 CHESS-VEC, batched).

    points, vecs: (m, n) float64 CUDA tensors; params: (2n^2+n,) float64 CUDA tensor for
    Fletcher-Powell.  Asynchronous on `stream` (default: torch's current stream)."""
    return _hvp("chessfad_hvp_batch", func, points, vecs, csize, params, out, stream)


def sym_hvp_batch(func, points, vecs, csize: int, params=None, out=None, stream=None):
    """Same product with the symmetric chunked algorithm (Alg 8 SC-HESS-VEC, batched)."""
    return _hvp("chessfad_sym_hvp_batch", func, points, vecs, csize, params, out, stream)


def hvp_batch_hoisted(func, points, vecs, csize: int, params=None, out=None, stream=None):
    """NEXT-4: Alg 7 with value-channel hoisting (compile-time kernels for F1/F2/F4 at
    n in {2,4,8,16}, row hoisting for F3); same results as hvp_batch, executed FLOPs below
    the model count."""
    return _hvp("chessfad_hvp_batch_hoisted", func, points, vecs, csize, params, out, stream)


def hvp_batch_seedsparse(func, points, vecs, csize: int, params=None, out=None, stream=None):
    """NEXT-4 seed sparsity (every function): Alg 7 with the operations on exact-zero seed slots
    skipped; equals hvp_batch bit for bit up to the sign of zero."""
    return _hvp("chessfad_hvp_batch_seedsparse", func, points, vecs, csize, params, out, stream)


def hvp_batch_paper_l2(func, points, vecs, csize: int, out=None, stream=None):
    """COMPARISON BASELINE: the paper's Fig. 2 L2 kernel design recompiled for sm_100a."""
    import torch
    m, n = points.shape
    if out is None:
        out = torch.empty_like(points)
    st = load().chessfad_hvp_batch_paper_l2(_func(func), n, csize, m, _dev(points, "points"),
                                            _dev(vecs, "vecs", (m, n)), _dev(out, "out", (m, n)), _stream_ptr(stream))
    _check(st)
    return out


def hvp_batch_paper(level: int, func, points, vecs, csize: int, out=None, stream=None):
    """COMPARISON BASELINES: the paper's L0 (Alg 9), L1 (Alg 10) or L2 (Fig. 2) design."""
    import torch
    m, n = points.shape
    if out is None:
        out = torch.empty_like(points)
    st = load().chessfad_hvp_batch_paper(level, _func(func), n, csize, m, _dev(points, "points"),
                                         _dev(vecs, "vecs", (m, n)), _dev(out, "out", (m, n)), _stream_ptr(stream))
    _check(st)
    return out


def hessian_batch(func, points, csize: int, params=None, out=None, stream=None):
    """hess[e] = Hess f(points[e]), every entry computed (Alg 5 CHUNK-HESS, batched): (m, n, n)."""
    return _hess("chessfad_hessian_batch", func, points, csize, params, out, stream)


def _hess_grad(entry, func, points, csize, params, out, grad, stream):
    import torch
    m, n = _points_2d(points)
    if out is None:
        out = torch.empty((m, n, n), dtype=torch.float64, device=points.device)
    if grad is None:
        grad = torch.empty((m, n), dtype=torch.float64, device=points.device)
    st = getattr(load(), entry)(_func(func), n, csize, m, _dev(points, "points"), _dev(out, "hess", (m, n, n)),
                                _dev(grad, "grad", (m, n)), _dev_params(params, func, n), _stream_ptr(stream))
    _check(st)
    return out, grad


def hessian_grad_batch(func, points, csize: int, params=None, out=None, grad=None, stream=None):
    """(hess, grad): Alg 5 Hessians plus the gradient by-product from slot v[1]."""
    return _hess_grad("chessfad_hessian_grad_batch", func, points, csize, params, out, grad, stream)


def hessian_batch_seedsparse(func, points, csize: int, params=None, out=None, stream=None):
    """NEXT-4 seed sparsity for the Hessian API (every function): equals hessian_batch bit for
    bit up to the sign of zero."""
    return _hess("chessfad_hessian_batch_seedsparse", func, points, csize, params, out, stream)


def sym_hvp_batch_seedsparse(func, points, vecs, csize: int, params=None, out=None, stream=None):
    """Alg 8 with seed sparsity: equals sym_hvp_batch up to the sign of zero (F1/F2/F4), within
    rounding of the tensor-core kernel for Fletcher-Powell (n <= 64)."""
    return _hvp("chessfad_sym_hvp_batch_seedsparse", func, points, vecs, csize, params, out, stream)


def sym_hessian_batch_seedsparse(func, points, csize: int, params=None, out=None, stream=None):
    """Alg 6 with seed sparsity (every function): equals sym_hessian_batch up to the sign of zero
    (Fletcher-Powell: within rounding)."""
    return _hess("chessfad_sym_hessian_batch_seedsparse", func, points, csize, params, out, stream)


def hessian_grad_batch_seedsparse(func, points, csize: int, params=None, out=None, grad=None, stream=None):
    """Alg 5 + gradient with seed sparsity (every function): equals hessian_grad_batch
    (Fletcher-Powell: within rounding)."""
    return _hess_grad("chessfad_hessian_grad_batch_seedsparse", func, points, csize, params, out, grad, stream)


def sym_hessian_batch(func, points, csize: int, params=None, out=None, stream=None):
    """Hessians by Alg 6 SCHUNK-HESS: upper chunks computed, whole lower chunks mirrored."""
    return _hess("chessfad_sym_hessian_batch", func, points, csize, params, out, stream)


def _host_arr(x, name, shape, writable=False):
    """(pointer, owner) of a contiguous float64 HOST buffer of exactly `shape`; the owner must
    stay referenced until the library call returns (a converted copy would otherwise be
    freed under the call)."""
    import numpy as np
    import torch
    if x is None:
        return None, None
    if isinstance(x, torch.Tensor):
        if x.is_cuda or x.dtype != torch.float64 or not x.is_contiguous():
            raise TypeError(f"{name} must be a contiguous float64 CPU tensor")
        ptr, shp = x.data_ptr(), tuple(x.shape)
    else:
        if writable and not isinstance(x, np.ndarray):
            raise TypeError(f"{name} must be a numpy array or a CPU tensor (written in place)")
        x = np.asarray(x)
        if x.dtype != np.float64 or not x.flags["C_CONTIGUOUS"] or (writable and not x.flags["WRITEABLE"]):
            raise TypeError(f"{name} must be a contiguous{' writable' if writable else ''} float64 array")
        ptr, shp = x.ctypes.data, tuple(x.shape)
    if shp != tuple(shape) and not (len(shape) == 1 and int(np.prod(shp)) == shape[0]):
        raise ValueError(f"{name} has shape {shp}, expected {tuple(shape)}")
    return ctypes.c_void_p(ptr), x


class HostPipeline:
    """End-to-end HVP on HOST buffers through one reusable chessfad_host_ctx (streams and
    events created once) and a cached device workspace from torch's allocator."""

    def __init__(self):
        self._lib = load()
        h = ctypes.c_void_p()
        _check(self._lib.chessfad_host_ctx_create(ctypes.byref(h)))
        self._ctx = h
        self._ws = None

    def close(self):
        if self._ctx is not None:
            self._lib.chessfad_host_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def hvp(self, func, points, vecs, csize: int, params=None, out=None, piece_points: int = 0, stream=None):
        return _host_call(self._lib, self._ctx, self, func, points, vecs, csize, params, out, piece_points, stream,
                          None)


def _host_call(lib, ctx, holder, func, points, vecs, csize, params, out, piece_points, stream, workspace):
    import numpy as np
    import torch
    shp = np.shape(points)
    if len(shp) != 2:
        raise ValueError(f"points must be (m, n), got shape {tuple(shp)}")
    m, n = shp
    if out is None:
        out = torch.empty((m, n), dtype=torch.float64, pin_memory=torch.cuda.is_available())
    pp, k0 = _host_arr(points, "points", (m, n))
    pv, k1 = _host_arr(vecs, "vecs", (m, n))
    po, k2 = _host_arr(out, "out", (m, n), writable=True)
    pshape = _params_shape(func, n)
    ppar, k3 = _host_arr(params, "params", pshape) if pshape is not None else (None, None)
    need = lib.chessfad_hvp_host_workspace_bytes(_func(func), n, m, piece_points)
    ws = workspace if workspace is not None else (holder._ws if holder is not None else None)
    if ws is None or ws.numel() < need:
        ws = torch.empty(max(need, 1), dtype=torch.uint8, device="cuda")
        if holder is not None:
            holder._ws = ws
    args = (_func(func), n, csize, m, pp, pv, po, ppar, piece_points, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
            _stream_ptr(stream))
    st = lib.chessfad_hvp_batch_host_ctx(ctx, *args) if ctx is not None else lib.chessfad_hvp_batch_host(*args)
    del k0, k1, k2, k3  # kept alive across the call
    _check(st)
    return out


def hvp_batch_host(func, points, vecs, csize: int, params=None, out=None, piece_points: int = 0, stream=None,
                   workspace=None):
    """End-to-end HVP on HOST buffers (numpy arrays or CPU tensors, ideally pinned): H2D
    copies, kernels and D2H copies in a three-stage stream pipeline; synchronous.  The device
    workspace comes from torch's caching allocator (or `workspace`, a CUDA uint8 tensor).
    HostPipeline reuses the streams/events across calls."""
    return _host_call(load(), None, None, func, points, vecs, csize, params, out, piece_points, stream, workspace)


def is_supported(func, n: int, csize: int, algo: str | None = None) -> bool:
    if algo is None:
        return bool(load().chessfad_is_supported(_func(func), n, csize))
    return bool(load().chessfad_is_supported_algo(_func(func), n, csize, ALGOS[algo]))


def model_flops_per_point(func, n: int, csize: int, hessian: bool = False, algo: str | None = None) -> float:
    if algo is None:
        return float(load().chessfad_model_flops_per_point(_func(func), n, csize, int(hessian)))
    return float(load().chessfad_model_flops_per_point_algo(_func(func), n, csize, ALGOS[algo]))


def fp64_probe(blocks: int, iters: int, sink, stream=None):
    _check(load().chessfad_fp64_probe(blocks, iters, _dev(sink, "sink"), _stream_ptr(stream)))


def path(func, n: int, csize: int, algo: str = "hvp") -> str:
    """Kernel family that runs for these arguments (chessfad_path): e.g. "f3_dmma", "stream"."""
    return load().chessfad_path(_func(func), n, csize, ALGOS[algo]).decode()


def version() -> str:
    return load().chessfad_version().decode()
