"""Independent closed-form Hessians of the test functions (test helpers only).

Derived by hand from the function definitions and cross-checked with
sympy in tests/test_oracle_pins.py; they share nothing with the oracle or the CUDA path.
Evaluated either exactly (fractions, Rosenbrock / prodsum) or with mpmath at 50 digits.
"""
from __future__ import annotations

from fractions import Fraction

import mpmath
import numpy as np

mpmath.mp.dps = 50


# ---------------------------------------------------------------- Rosenbrock (exact)
def rosenbrock_hessian_exact(a):
    """H_ii = 1200 a_i^2 - 400 a_{i+1} + 2 (i <= n-2) + 200 (i >= 1); H_{i,i+1} = -400 a_i."""
    a = [Fraction(float(x)) for x in a]
    n = len(a)
    H = [[Fraction(0)] * n for _ in range(n)]
    for i in range(n):
        if i <= n - 2:
            H[i][i] += 1200 * a[i] ** 2 - 400 * a[i + 1] + 2
            H[i][i + 1] = -400 * a[i]
            H[i + 1][i] = -400 * a[i]
        if i >= 1:
            H[i][i] += 200
    return H


def prodsum_hessian_exact(n):
    H = [[Fraction(0)] * n for _ in range(n)]
    for i in range(n - 1):
        H[i][i + 1] = Fraction(1)
        H[i + 1][i] = Fraction(1)
    return H


def exact_hvp(H, v):
    v = [Fraction(float(x)) for x in v]
    n = len(v)
    return [sum((H[i][j] * v[j] for j in range(n)), Fraction(0)) for i in range(n)]


# ---------------------------------------------------------------- Ackley (mpmath)
def ackley_hessian_mp(a):
    """H_ij = 4 E1 (d_ij/(n r) - a_i a_j/(n^2 r^3) - 0.2 a_i a_j/(n^2 r^2))
             + E2 (-(2pi/n)^2 sin(2pi a_i) sin(2pi a_j) + d_ij (4 pi^2/n) cos(2pi a_i)),
    r = sqrt(sum a^2 / n), E1 = exp(-0.2 r), E2 = exp(sum cos(2 pi a) / n)."""
    a = [mpmath.mpf(float(x)) for x in a]
    n = len(a)
    tp = 2 * mpmath.pi
    r = mpmath.sqrt(sum(x * x for x in a) / n)
    E1 = mpmath.exp(mpmath.mpf("-0.2") * r)
    E2 = mpmath.exp(sum(mpmath.cos(tp * x) for x in a) / n)
    H = [[mpmath.mpf(0)] * n for _ in range(n)]
    for i in range(n):
        for j in range(n):
            d = 1 if i == j else 0
            H[i][j] = 4 * E1 * (d / (n * r) - a[i] * a[j] / (n ** 2 * r ** 3)
                                - mpmath.mpf("0.2") * a[i] * a[j] / (n ** 2 * r ** 2)) \
                + E2 * (-(tp / n) ** 2 * mpmath.sin(tp * a[i]) * mpmath.sin(tp * a[j])
                        + d * (tp ** 2 / n) * mpmath.cos(tp * a[i]))
    return H


def ackley_value_mp(a):
    a = [mpmath.mpf(float(x)) for x in a]
    n = len(a)
    tp = 2 * mpmath.pi
    r = mpmath.sqrt(sum(x * x for x in a) / n)
    return (-20 * mpmath.exp(mpmath.mpf("-0.2") * r) - mpmath.exp(sum(mpmath.cos(tp * x) for x in a) / n)
            + 20 + mpmath.e)


# ---------------------------------------------------------------- Fletcher-Powell (mpmath)
def fp_hessian_mp(a, A, B, Estar):
    """H = 2 J^T J + 2 diag(sum_k r_k (A_ki sin a_i + B_ki cos a_i)),
    J_kj = A_kj cos a_j - B_kj sin a_j, r_k = E*_k - sum_j (A_kj sin a_j + B_kj cos a_j)."""
    a = [mpmath.mpf(float(x)) for x in a]
    n = len(a)
    A = [[mpmath.mpf(float(A[k][j])) for j in range(n)] for k in range(n)]
    B = [[mpmath.mpf(float(B[k][j])) for j in range(n)] for k in range(n)]
    Es = [mpmath.mpf(float(x)) for x in Estar]
    s = [mpmath.sin(x) for x in a]
    c = [mpmath.cos(x) for x in a]
    J = [[A[k][j] * c[j] - B[k][j] * s[j] for j in range(n)] for k in range(n)]
    r = [Es[k] - sum(A[k][j] * s[j] + B[k][j] * c[j] for j in range(n)) for k in range(n)]
    H = [[2 * sum(J[k][i] * J[k][j] for k in range(n)) for j in range(n)] for i in range(n)]
    for i in range(n):
        H[i][i] += 2 * sum(r[k] * (A[k][i] * s[i] + B[k][i] * c[i]) for k in range(n))
    return H


def mp_hvp(H, v):
    v = [mpmath.mpf(float(x)) for x in v]
    n = len(v)
    return [sum(H[i][j] * v[j] for j in range(n)) for i in range(n)]


def to_float(M):
    return np.array([[float(x) for x in row] for row in M]) if isinstance(M[0], list) else np.array([float(x) for x in M])


def normwise_err(x, ref, H, v):
    """max_i |x_i - ref_i| / (max_ij |H_ij| * sum_j |v_j|)."""
    Hf = np.abs(to_float(H))
    scale = Hf.max() * np.abs(np.asarray(v, dtype=float)).sum()
    ref = np.array([float(r) for r in ref])
    return float(np.max(np.abs(np.asarray(x) - ref)) / scale) if scale > 0 else float(np.max(np.abs(np.asarray(x) - ref)))
