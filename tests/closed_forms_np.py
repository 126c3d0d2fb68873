"""Vectorised (NumPy, FP64) closed-form Hessian-vector products of the four test functions,
for the all-points cross-check of SURVEY §8(d) "Closed-form cross-check on all points".

Independent of the oracle and of the CUDA path: the same hand-derived closed forms as
tests/closed_forms.py (cross-checked there against sympy / mpmath), written as array
expressions over m points at once.  Each function returns (Hv, S) with
S[e, i] = sum_j |H_ij| |v_j| (the componentwise-error denominator), both (m, n).
Functions defined; F3's params layout [A | B | E*] as synth.fp_params_flat.
"""
from __future__ import annotations

import numpy as np

TWO_PI = 2.0 * np.pi


def rosenbrock(P, V):
    """H_ii = 1200 a_i^2 - 400 a_{i+1} + 2 (i <= n-2) + 200 (i >= 1); H_{i,i+1} = -400 a_i."""
    m, n = P.shape
    d = np.zeros((m, n))
    d[:, :-1] += 1200.0 * P[:, :-1] ** 2 - 400.0 * P[:, 1:] + 2.0
    d[:, 1:] += 200.0
    off = -400.0 * P[:, :-1]  # H_{i,i+1} = H_{i+1,i}, i = 0..n-2
    hv = d * V
    hv[:, :-1] += off * V[:, 1:]
    hv[:, 1:] += off * V[:, :-1]
    s = np.abs(d) * np.abs(V)
    s[:, :-1] += np.abs(off) * np.abs(V[:, 1:])
    s[:, 1:] += np.abs(off) * np.abs(V[:, :-1])
    return hv, s


def prodsum(P, V):
    """H = tridiagonal ones (zero diagonal)."""
    hv = np.zeros_like(V)
    hv[:, 1:] += V[:, :-1]
    hv[:, :-1] += V[:, 1:]
    s = np.zeros_like(V)
    s[:, 1:] += np.abs(V[:, :-1])
    s[:, :-1] += np.abs(V[:, 1:])
    return hv, s


def _blocks(m, bs):
    for b0 in range(0, m, bs):
        yield slice(b0, min(m, b0 + bs))


def ackley(P, V, block=1 << 15):
    """H = 4 E1 (I/(n r) - a a^T (1/(n^2 r^3) + 0.2/(n^2 r^2)))
         + E2 (-(2 pi/n)^2 s s^T + diag((2 pi)^2/n c)),  s = sin 2 pi a, c = cos 2 pi a,
    r = sqrt(|a|^2/n), E1 = exp(-0.2 r), E2 = exp(sum c / n)."""
    m, n = P.shape
    hv, S = np.empty_like(V), np.empty_like(V)
    for sl in _blocks(m, block):
        a, v = P[sl], V[sl]
        r = np.sqrt((a * a).sum(1) / n)[:, None]
        E1 = np.exp(-0.2 * r)
        sn, cs = np.sin(TWO_PI * a), np.cos(TWO_PI * a)
        E2 = np.exp(cs.sum(1) / n)[:, None]
        k = 1.0 / (n * n * r ** 3) + 0.2 / (n * n * r * r)
        H = (-4.0 * E1 * k)[:, :, None] * a[:, :, None] * a[:, None, :]
        H -= (E2 * (TWO_PI / n) ** 2)[:, :, None] * sn[:, :, None] * sn[:, None, :]
        idx = np.arange(n)
        H[:, idx, idx] += 4.0 * E1 / (n * r) + E2 * (TWO_PI ** 2 / n) * cs
        hv[sl] = np.einsum("eij,ej->ei", H, v)
        S[sl] = np.einsum("eij,ej->ei", np.abs(H), np.abs(v))
    return hv, S


def fletcher_powell(P, V, params, block=1 << 15):
    """H = 2 J^T J + 2 diag(sum_k r_k (A_ki sin a_i + B_ki cos a_i)),
    J_kj = A_kj cos a_j - B_kj sin a_j, r_k = E*_k - sum_j (A_kj sin a_j + B_kj cos a_j)."""
    m, n = P.shape
    A = params[: n * n].reshape(n, n)
    B = params[n * n: 2 * n * n].reshape(n, n)
    Es = params[2 * n * n:]
    hv, S = np.empty_like(V), np.empty_like(V)
    for sl in _blocks(m, block):
        a, v = P[sl], V[sl]
        sn, cs = np.sin(a), np.cos(a)
        J = A[None] * cs[:, None, :] - B[None] * sn[:, None, :]  # (b, k, j)
        r = Es[None] - (sn @ A.T + cs @ B.T)  # (b, k)
        d = sn * (r @ A) + cs * (r @ B)  # sum_k r_k (A_ki sin a_i + B_ki cos a_i)
        H = 2.0 * np.einsum("eki,ekj->eij", J, J)
        idx = np.arange(n)
        H[:, idx, idx] += 2.0 * d
        hv[sl] = np.einsum("eij,ej->ei", H, v)
        S[sl] = np.einsum("eij,ej->ei", np.abs(H), np.abs(v))
    return hv, S


def hvp(func, P, V, params=None):
    if func == "rosenbrock":
        return rosenbrock(P, V)
    if func == "prodsum":
        return prodsum(P, V)
    if func == "ackley":
        return ackley(P, V)
    if func == "fletcher_powell":
        return fletcher_powell(P, V, params)
    raise ValueError(func)


def error(got, hv, S):
    """max over all components of |g - Hv| / max(|Hv|, S) (the oracle metric's form)."""
    den = np.maximum(np.abs(hv), S)
    return float(np.max(np.abs(got - hv) / np.where(den > 0, den, 1.0)))
