"""Seeded, index-addressable synthetic inputs for the batched Hessian-vector product.

This module is the ONLY code shared by the CPU oracle (``oracle/``) and the CUDA
product path (``paper_2410_22575_b200``).  It holds none of the method's
arithmetic: it draws points, vectors and the Fletcher-Powell parameters, nothing
else.  The recipe is stated in DESIGN.md ("Input recipe") and follows
SURVEY.md §8(d) "Concrete synthetic inputs":

* generator  : splitmix64 of a per-array counter
               ``key = index + (array_id << 56) + splitmix64(seed)`` (mod 2^64),
               ``u = (splitmix64(key) >> 11) * 2^-53`` in [0, 1).
* points     : a ~ U[-2, 2)   (array id 0)  -- SPEC.md:565 (cli, "uniform in [-2, 2]")
* vectors    : in ~ U[-1, 1)  (array id 1)  -- SPEC.md:565
* F3 params  : A, B ~ U{-100..100} (ids 2, 3), x* ~ U(-pi, pi) (id 4),
               E*_k = sum_j (A_kj sin x*_j + B_kj cos x*_j)  -- SPEC.md:379-387
               (the paper gives no values).
* integers   : a, v ~ U{-9..9} (ids 5, 6) for the bit-exact integer pin
               ("Integer-input exactness").

Element (e, k) of an m x n array has global index e*n + k, so any contiguous
range of points [e0, e1) can be generated on its own (multi-GPU shards see the
same data as a single-GPU run).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "ARRAY_POINTS", "ARRAY_VECS", "ARRAY_A", "ARRAY_B", "ARRAY_XSTAR",
    "ARRAY_INT_POINTS", "ARRAY_INT_VECS",
    "splitmix64", "uniform", "points", "vectors", "int_points", "int_vectors",
    "fp_params", "fp_params_flat",
]

ARRAY_POINTS = 0
ARRAY_VECS = 1
ARRAY_A = 2
ARRAY_B = 3
ARRAY_XSTAR = 4
ARRAY_INT_POINTS = 5
ARRAY_INT_VECS = 6

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrap-around arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _bits(seed: int, array_id: int, start: int, count: int) -> np.ndarray:
    base = splitmix64(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]
    idx = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = idx + (np.uint64(array_id) << np.uint64(56)) + base
    return splitmix64(key)


def uniform(seed: int, array_id: int, start: int, count: int, lo: float, hi: float) -> np.ndarray:
    """count doubles lo + (hi-lo)*u, u in [0,1) with 53 random bits."""
    z = _bits(seed, array_id, start, count)
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return lo + (hi - lo) * u


def _int_range(seed: int, array_id: int, start: int, count: int, lo: int, hi: int) -> np.ndarray:
    z = _bits(seed, array_id, start, count)
    span = np.uint64(hi - lo + 1)
    return (z % span).astype(np.int64) + lo


def points(seed: int, n: int, m: int, first: int = 0) -> np.ndarray:
    """Points e in [first, first+m): (m, n) float64, a ~ U[-2, 2)."""
    return uniform(seed, ARRAY_POINTS, first * n, m * n, -2.0, 2.0).reshape(m, n)


def vectors(seed: int, n: int, m: int, first: int = 0) -> np.ndarray:
    """Multiplicand vectors: (m, n) float64, in ~ U[-1, 1)."""
    return uniform(seed, ARRAY_VECS, first * n, m * n, -1.0, 1.0).reshape(m, n)


def int_points(seed: int, n: int, m: int, first: int = 0) -> np.ndarray:
    """Integer-valued points in {-9..9} as float64 (bit-exact pin inputs)."""
    return _int_range(seed, ARRAY_INT_POINTS, first * n, m * n, -9, 9).astype(np.float64).reshape(m, n)


def int_vectors(seed: int, n: int, m: int, first: int = 0) -> np.ndarray:
    return _int_range(seed, ARRAY_INT_VECS, first * n, m * n, -9, 9).astype(np.float64).reshape(m, n)


def fp_params(seed: int, n: int):
    """Fletcher-Powell parameters (A, B, xstar, Estar).

    A, B: (n, n) float64 holding integers in [-100, 100]; xstar in (-pi, pi);
    Estar_k = sum_j (A_kj sin xstar_j + B_kj cos xstar_j), accumulated over
    ascending j.  Estar is the parameter definition (E* := E(x*)), computed
    once here so that both sides read the same array.
    """
    A = _int_range(seed, ARRAY_A, 0, n * n, -100, 100).astype(np.float64).reshape(n, n)
    B = _int_range(seed, ARRAY_B, 0, n * n, -100, 100).astype(np.float64).reshape(n, n)
    xstar = uniform(seed, ARRAY_XSTAR, 0, n, -np.pi, np.pi)
    s = np.sin(xstar)
    c = np.cos(xstar)
    Estar = np.zeros(n)
    for j in range(n):
        Estar = Estar + (A[:, j] * s[j] + B[:, j] * c[j])
    return A, B, xstar, Estar


def fp_params_flat(seed: int, n: int) -> np.ndarray:
    """The params buffer layout of the C-ABI: [A (n*n) | B (n*n) | Estar (n)]."""
    A, B, _, Estar = fp_params(seed, n)
    return np.concatenate([A.ravel(), B.ravel(), Estar]).astype(np.float64)
