"""NEXT-3: a user-defined function compiled against include/chessfad_device.cuh runs in the
same batched kernels (Alg 7 / 5 / 8 / 6) and matches its closed-form Hessian."""
import ctypes
import os
import subprocess
import tempfile

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def closed_form_hessian(a):
    """f = sum cos(y_i) + y_i/(1+y_i^2) + sum_{i<n-1} y_i^2 y_{i+1}:
    H_ii = -cos a_i + (2a^3 - 6a)/(1+a^2)^3 + 2 a_{i+1} [i<n-1];  H_{i,i+1} = H_{i+1,i} = 2 a_i."""
    n = a.size
    H = np.zeros((n, n))
    for i in range(n):
        x = a[i]
        H[i, i] = -np.cos(x) + (2 * x ** 3 - 6 * x) / (1 + x * x) ** 3
        if i < n - 1:
            H[i, i] += 2 * a[i + 1]
            H[i, i + 1] = H[i + 1, i] = 2 * x
    return H


@pytest.fixture(scope="module")
def userlib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = tempfile.mkdtemp(prefix="chessfad_user_")
    so = os.path.join(d, "libuser.so")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O3",
                           "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "user_function.cu"), "-o", so])
    lib = ctypes.CDLL(so)
    vp = ctypes.c_void_p
    lib.user_batch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_longlong, vp, vp, vp, vp]
    lib.user_batch.restype = ctypes.c_int
    lib.user_batch_n16.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_longlong, vp, vp, vp, vp]
    lib.user_batch_n16.restype = ctypes.c_int
    return lib


def test_user_function_all_algorithms(userlib):
    n, m = 16, 1000
    P, V = synth.points(21, n, m), synth.vectors(21, n, m)
    Hs = np.stack([closed_form_hessian(P[e]) for e in range(m)])
    ref = np.einsum("eij,ej->ei", Hs, V)
    scale = np.einsum("eij,ej->ei", np.abs(Hs), np.abs(V))
    dev = torch.device("cuda")
    p, v = torch.from_numpy(P).to(dev), torch.from_numpy(V).to(dev)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for C in (1, 4, 8):
        for algo in (0, 2):
            out = torch.empty_like(p)
            assert userlib.user_batch(algo, n, C, m, p.data_ptr(), v.data_ptr(), out.data_ptr(), s) == 0
            torch.cuda.synchronize()
            err = np.abs(out.cpu().numpy() - ref) / np.maximum(np.abs(ref), scale)
            assert err.max() <= 1e-12, (C, algo, err.max())
        for algo in (1, 3):
            H = torch.empty((m, n, n), dtype=torch.float64, device=dev)
            assert userlib.user_batch(algo, n, C, m, p.data_ptr(), None, H.data_ptr(), s) == 0
            torch.cuda.synchronize()
            Hg = H.cpu().numpy()
            assert np.max(np.abs(Hg - Hs)) <= 1e-12 * np.abs(Hs).max(), (C, algo)
    out = torch.empty_like(p)
    assert userlib.user_batch(0, n, 3, m, p.data_ptr(), v.data_ptr(), out.data_ptr(), s) == -2  # C not compiled


def test_user_function_compiled_n(userlib):
    """chessfad::user_batch_n<16, C, ...> (the kernels compiled for n = 16, reading R8) against
    the closed form and against the runtime-n kernels, every algorithm."""
    n, m = 16, 700
    P, V = synth.points(23, n, m), synth.vectors(23, n, m)
    Hs = np.stack([closed_form_hessian(P[e]) for e in range(m)])
    ref = np.einsum("eij,ej->ei", Hs, V)
    scale = np.einsum("eij,ej->ei", np.abs(Hs), np.abs(V))
    dev = torch.device("cuda")
    p, v = torch.from_numpy(P).to(dev), torch.from_numpy(V).to(dev)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for C in (1, 4, 16):
        for algo in (0, 2):
            out, out_rt = torch.empty_like(p), torch.empty_like(p)
            assert userlib.user_batch_n16(algo, C, m, p.data_ptr(), v.data_ptr(), out.data_ptr(), s) == 0
            assert userlib.user_batch(algo, n, C if C != 16 else 8, m, p.data_ptr(), v.data_ptr(),
                                      out_rt.data_ptr(), s) == 0
            torch.cuda.synchronize()
            got = out.cpu().numpy()
            err = np.abs(got - ref) / np.maximum(np.abs(ref), scale)
            assert err.max() <= 1e-12, (C, algo, err.max())
            err_rt = np.abs(got - out_rt.cpu().numpy()) / np.maximum(np.abs(ref), scale)
            assert err_rt.max() <= 1e-12, (C, algo, err_rt.max())
        for algo in (1, 3):
            H = torch.empty((m, n, n), dtype=torch.float64, device=dev)
            assert userlib.user_batch_n16(algo, C, m, p.data_ptr(), None, H.data_ptr(), s) == 0
            torch.cuda.synchronize()
            assert np.max(np.abs(H.cpu().numpy() - Hs)) <= 1e-12 * np.abs(Hs).max(), (C, algo)
