"""The oracle pinned to things other than itself: closed forms, exact integer results,
mpmath, sympy, finite differences, the full (n+1)(n+2)/2 scheme, invariants of the
algorithms (Alg 2-8) and the paper's §V operation counts."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from tests import closed_forms as cf

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_form_pins.json")))
FUNCS = ["rosenbrock", "ackley", "fletcher_powell", "prodsum"]


def _params(func, n, seed=0):
    return synth.fp_params_flat(seed, n) if func == "fletcher_powell" else None


def divisors(n):
    return [c for c in range(1, n + 1) if n % c == 0]


# ------------------------------------------------------------------ printed / hand-derived pins
@pytest.mark.parametrize("ex", GOLD["hessian"], ids=lambda e: e["cite"][:40])
@pytest.mark.parametrize("algo", ["full", "sym", "chunk", "schunk", "scheme"])
def test_hessian_pins(ex, algo):
    n = len(ex["a"])
    for C in divisors(n) if algo in ("chunk", "schunk") else [1]:
        H, _ = oracle.hessian(ex["func"], ex["a"], algo=algo, C=C)
        assert np.array_equal(H, np.array(ex["H"], dtype=float)), (algo, C)


@pytest.mark.parametrize("ex", GOLD["hvp"], ids=lambda e: e["cite"][:40])
def test_hvp_pins(ex):
    n = len(ex["a"])
    for C in divisors(n):
        out, _ = oracle.chess_vec(ex["func"], ex["a"], ex["v"], C)
        assert np.array_equal(out, np.array(ex["out"], dtype=float))
        assert np.array_equal(oracle.sc_hess_vec(ex["func"], ex["a"], ex["v"], C), np.array(ex["out"], dtype=float))


@pytest.mark.parametrize("ex", GOLD["value"], ids=lambda e: e["cite"][:40])
def test_value_pins(ex):
    assert oracle.eval_scalar(ex["func"], ex["x"]) == pytest.approx(ex["f"], abs=ex.get("tol", 0.0))


def test_fp_value_zero_at_xstar():
    """f(x*) = 0."""
    for n in (2, 5, 16):
        A, B, xstar, _ = synth.fp_params(1, n)
        f = oracle.eval_scalar("fletcher_powell", xstar, synth.fp_params_flat(1, n))
        assert abs(f) < 1e-20 * n ** 2 + 1e-18


def test_ackley_value_mpmath():
    """Ackley n=1 at 0.5 (SPEC.md:368 leaves the number to a scalar oracle): mpmath."""
    for x in ([0.5], [0.5, -0.25], [1.5, -1.0, 0.3]):
        assert oracle.eval_scalar("ackley", x) == pytest.approx(float(cf.ackley_value_mp(x)), rel=1e-14)


# ------------------------------------------------------------------ exact integer results
@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_integer_inputs_exact(n):
    """Rosenbrock and prodsum on integers in {-9..9}: every intermediate is an integer
    < 2^53, so H.v is exact and must equal the exact rational closed form bitwise."""
    P = synth.int_points(7, n, 10)
    V = synth.int_vectors(7, n, 10)
    for e in range(10):
        for func, H in (("rosenbrock", cf.rosenbrock_hessian_exact(P[e])), ("prodsum", cf.prodsum_hessian_exact(n))):
            want = np.array([float(x) for x in cf.exact_hvp(H, V[e])])
            for C in divisors(n):
                out, _ = oracle.chess_vec(func, P[e], V[e], C)
                assert np.array_equal(out, want), (func, C)


# ------------------------------------------------------------------ closed forms at random points
@pytest.mark.parametrize("n", [2, 3, 7, 16])
def test_rosenbrock_closed_form(n):
    P, V = synth.points(11, n, 20), synth.vectors(11, n, 20)
    for e in range(20):
        H = cf.rosenbrock_hessian_exact(P[e])
        ref = cf.exact_hvp(H, V[e])
        out, _ = oracle.chess_vec("rosenbrock", P[e], V[e], 1)
        assert cf.normwise_err(out, ref, H, V[e]) < 1e-15
        Ho, _ = oracle.hessian("rosenbrock", P[e], algo="chunk", C=n)
        # every Hessian entry of Rosenbrock is a short sum: within a few ulps
        np.testing.assert_allclose(Ho, cf.to_float(H), rtol=4e-16 * 8, atol=1e-12)


@pytest.mark.parametrize("n", [1, 2, 5, 8])
def test_ackley_closed_form(n):
    P, V = synth.points(12, n, 6), synth.vectors(12, n, 6)
    for e in range(6):
        H = cf.ackley_hessian_mp(P[e])
        ref = cf.mp_hvp(H, V[e])
        out, _ = oracle.chess_vec("ackley", P[e], V[e], 1)
        assert cf.normwise_err(out, ref, H, V[e]) < 1e-14


@pytest.mark.parametrize("n", [1, 2, 4, 6])
def test_fletcher_powell_closed_form(n):
    A, B, xstar, Es = synth.fp_params(13, n)
    params = synth.fp_params_flat(13, n)
    P, V = synth.points(13, n, 5), synth.vectors(13, n, 5)
    for e in range(5):
        H = cf.fp_hessian_mp(P[e], A, B, Es)
        ref = cf.mp_hvp(H, V[e])
        out, _ = oracle.chess_vec("fletcher_powell", P[e], V[e], 1, params)
        assert cf.normwise_err(out, ref, H, V[e]) < 1e-14


def test_goldens_f2_f3_n2():
    """SURVEY.md §8(c) golden values (mpmath, 40 digits) at a = (0.5, -0.25), v = (1, 2);
    recomputed here from the closed forms with mpmath at 50 digits."""
    a, v = [0.5, -0.25], [1.0, 2.0]
    H = cf.ackley_hessian_mp(a)
    np.testing.assert_allclose(cf.to_float(H), [[-11.333101859203269, 2.017856803351086],
                                                [2.017856803351086, -2.3200989856812008]], rtol=1e-15)
    out, _ = oracle.chess_vec("ackley", a, v, 1)
    np.testing.assert_allclose(out, [-7.2973882525010968, -2.6223411680113156], rtol=1e-14)
    A = np.array([[1.0, 2.0], [3.0, 4.0]])
    B = np.array([[-1.0, 0.0], [2.0, -3.0]])
    xs = np.array([0.1, 0.2])
    Es = np.array([sum(A[k, j] * math.sin(xs[j]) + B[k, j] * math.cos(xs[j]) for j in range(2)) for k in range(2)])
    np.testing.assert_allclose(Es, [-0.49783208704107518, 0.14398617015305596], rtol=1e-15)
    params = np.concatenate([A.ravel(), B.ravel(), Es])
    out, _ = oracle.chess_vec("fletcher_powell", a, v, 1, params)
    np.testing.assert_allclose(out, [45.879967424220566, 56.06247359451474], rtol=1e-14)
    Ho, _ = oracle.hessian("fletcher_powell", a, params, algo="chunk", C=2)
    np.testing.assert_allclose(Ho, [[14.381187698986528, 15.749389862617019],
                                    [15.749389862617019, 20.156541865948861]], rtol=1e-14)


def test_sympy_brute_force_tiny():
    """Symbolic differentiation of the canonical forms (sympy) at n = 3 for all four
    functions: an independent brute-force check of every Hessian entry."""
    sympy = pytest.importorskip("sympy")
    n = 3
    xs = sympy.symbols("x0:3")
    A, B, _, Es = synth.fp_params(2, n)
    exprs = {
        "rosenbrock": sum(100 * (xs[i + 1] - xs[i] ** 2) ** 2 + (1 - xs[i]) ** 2 for i in range(n - 1)),
        "prodsum": sum(xs[i] * xs[i + 1] for i in range(n - 1)),
        "ackley": -20 * sympy.exp(-sympy.Rational(1, 5) * sympy.sqrt(sum(x ** 2 for x in xs) / n))
        - sympy.exp(sum(sympy.cos(2 * sympy.pi * x) for x in xs) / n) + 20 + sympy.E,
        "fletcher_powell": sum((sympy.Float(Es[k], 30) - sum(int(A[k, j]) * sympy.sin(xs[j]) + int(B[k, j]) * sympy.cos(xs[j])
                                                             for j in range(n))) ** 2 for k in range(n)),
    }
    a = synth.points(21, n, 1)[0]
    subs = {xs[k]: sympy.Float(float(a[k]), 40) for k in range(n)}
    for func, ex in exprs.items():
        Hs = np.array([[float(sympy.diff(ex, xs[i], xs[j]).evalf(30, subs=subs)) for j in range(n)] for i in range(n)])
        Ho, _ = oracle.hessian(func, a, _params(func, n, 2) if func == "fletcher_powell" else None, algo="chunk", C=1)
        scale = np.abs(Hs).max()
        assert np.max(np.abs(Ho - Hs)) <= 1e-13 * scale, func


# ------------------------------------------------------------------ finite differences
def _fd_hessian(func, a, params):
    n = len(a)
    H = np.zeros((n, n))
    h = [1e-4 * max(1.0, abs(x)) for x in a]
    f = lambda x: oracle.eval_scalar(func, x, params)
    for i in range(n):
        for j in range(n):
            def at(si, sj):
                x = np.array(a, dtype=float)
                x[i] += si * h[i]
                x[j] += sj * h[j]
                return f(x)
            H[i, j] = (at(1, 1) - at(1, -1) - at(-1, 1) + at(-1, -1)) / (4 * h[i] * h[j])
    return H


@pytest.mark.parametrize("func", FUNCS)
@pytest.mark.parametrize("n", [4, 8])
def test_finite_differences(func, n):
    """chunked Hessian within 1e-4 of central FD."""
    params = _params(func, n)
    a = synth.points(31, n, 1)[0]
    H, grad = oracle.hessian(func, a, params, algo="chunk", C=2)
    Hfd = _fd_hessian(func, a, params)
    scale = max(1.0, np.abs(H).max())
    assert np.max(np.abs(H - Hfd)) <= 1e-4 * scale
    # gradient by-product in slot v[1]
    g = np.zeros(n)
    for i in range(n):
        hi = 1e-5 * max(1.0, abs(a[i]))
        xp, xm = a.copy(), a.copy()
        xp[i] += hi
        xm[i] -= hi
        g[i] = (oracle.eval_scalar(func, xp, params) - oracle.eval_scalar(func, xm, params)) / (2 * hi)
    assert np.max(np.abs(grad - g)) <= 1e-6 * max(1.0, np.abs(g).max())


# ------------------------------------------------------------------ full (n+1)(n+2)/2 scheme
@pytest.mark.parametrize("func", FUNCS)
def test_full_scheme_equivalence(func):
    """One evaluation with (n+1)(n+2)/2 components gives the same upper
    triangle as the chunked algorithm bit for bit (same Fig. 1 term order), the lower
    triangle within rounding, and the same gradient."""
    n = 6
    params = _params(func, n)
    for e, a in enumerate(synth.points(41, n, 4)):
        Hs, gs = oracle.hessian(func, a, params, algo="scheme")
        Hc, gc = oracle.hessian(func, a, params, algo="chunk", C=3)
        iu = np.triu_indices(n)
        assert np.array_equal(Hs[iu], Hc[iu]), func
        assert np.max(np.abs(Hs - Hc)) <= 1e-13 * np.abs(Hc).max()
        assert np.array_equal(gs, gc)


# ------------------------------------------------------------------ algorithm invariants
@pytest.mark.parametrize("func", FUNCS)
def test_chunk_invariance(func):
    """H and H.v bit-identical for every divisor C of n."""
    n = 12
    params = _params(func, n)
    a, v = synth.points(51, n, 1)[0], synth.vectors(51, n, 1)[0]
    H1, g1 = oracle.hessian(func, a, params, algo="chunk", C=1)
    o1, s1 = oracle.chess_vec(func, a, v, 1, params)
    for C in divisors(n)[1:]:
        H, g = oracle.hessian(func, a, params, algo="chunk", C=C)
        o, s = oracle.chess_vec(func, a, v, C, params)
        assert np.array_equal(H, H1) and np.array_equal(g, g1) and np.array_equal(o, o1), C


@pytest.mark.parametrize("func", FUNCS)
def test_engine_equivalence(func):
    """Alg 2 == Alg 5 (C=1) bitwise; Alg 3 and Alg 6 agree on the computed
    (upper) entries and mirror the rest; matrix-free Alg 7 == explicit H.v left to right."""
    for n in (4, 8):
        params = _params(func, n)
        a, v = synth.points(61, n, 1)[0], synth.vectors(61, n, 1)[0]
        Hf, _ = oracle.hessian(func, a, params, algo="full")
        Hsym, _ = oracle.hessian(func, a, params, algo="sym")
        H5, _ = oracle.hessian(func, a, params, algo="chunk", C=1)
        assert np.array_equal(Hf, H5)
        iu = np.triu_indices(n)
        assert np.array_equal(Hsym[iu], Hf[iu]) and np.array_equal(Hsym, Hsym.T)
        for C in divisors(n):
            H6, _ = oracle.hessian(func, a, params, algo="schunk", C=C)
            assert np.array_equal(H6[iu], Hf[iu])
            out, _ = oracle.chess_vec(func, a, v, C, params)
            explicit = np.zeros(n)
            for i in range(n):
                r = 0.0
                for j in range(n):
                    r = r + Hf[i, j] * v[j]
                explicit[i] = r
            assert np.array_equal(out, explicit)


@pytest.mark.parametrize("func", FUNCS)
def test_symmetric_hvp_and_symmetry(func):
    """Alg 8 == Alg 7 within rounding; H symmetric within rounding
    (not bitwise)."""
    for n in (2, 8, 16):
        params = _params(func, n)
        P, V = synth.points(71, n, 5), synth.vectors(71, n, 5)
        for e in range(5):
            for C in divisors(n):
                o7, s = oracle.chess_vec(func, P[e], V[e], C, params)
                o8 = oracle.sc_hess_vec(func, P[e], V[e], C, params)
                assert np.all(oracle.componentwise_error(o8, o7, s) <= 1e-13)
            H, _ = oracle.hessian(func, P[e], params, algo="chunk", C=1)
            assert np.max(np.abs(H - H.T)) <= 1e-13 * np.abs(H).max()


@pytest.mark.parametrize("func", FUNCS)
def test_linearity_and_zero(func):
    """H(alpha u + beta w) = alpha H u + beta H w; H 0 = 0."""
    n = 8
    params = _params(func, n)
    a = synth.points(81, n, 1)[0]
    u, w = synth.vectors(81, n, 2)
    al, be = 0.75, -1.5
    ou, su = oracle.chess_vec(func, a, u, 2, params)
    ow, sw = oracle.chess_vec(func, a, w, 2, params)
    ouw, _ = oracle.chess_vec(func, a, al * u + be * w, 2, params)
    scale = np.abs(al) * su + np.abs(be) * sw
    assert np.all(np.abs(ouw - (al * ou + be * ow)) <= 1e-13 * np.maximum(scale, 1e-300))
    oz, _ = oracle.chess_vec(func, a, np.zeros(n), 4, params)
    assert np.all(oz == 0)


def test_fletcher_powell_psd_at_xstar():
    """At x* the residuals vanish and H = 2 J^T J is PSD."""
    for n in (4, 8):
        _, _, xstar, _ = synth.fp_params(3, n)
        H, _ = oracle.hessian("fletcher_powell", xstar, synth.fp_params_flat(3, n), algo="chunk", C=n)
        ev = np.linalg.eigvalsh(0.5 * (H + H.T))
        assert ev.min() >= -1e-8 * np.abs(ev).max()


def test_ackley_origin_nan():
    """Ackley at the origin: value 0, derivative slots NaN (sqrt' singular)."""
    out, _ = oracle.chess_vec("ackley", np.zeros(4), np.ones(4), 2)
    assert np.all(np.isnan(out))


def test_errors():
    with pytest.raises(oracle.OracleError, match="ERR_CHUNK"):
        oracle.chess_vec("rosenbrock", np.zeros(10), np.zeros(10), 3)
    with pytest.raises(oracle.OracleError, match="ERR_FUNC"):
        oracle.chess_vec("rosenbrock", np.zeros(1), np.zeros(1), 1)
    with pytest.raises(oracle.OracleError, match="ERR_FUNC"):
        oracle.chess_vec("fletcher_powell", np.zeros(2), np.zeros(2), 1, None)


# ------------------------------------------------------------------ batches
def test_batch_equals_single_and_deterministic():
    n, m = 8, 37
    P, V = synth.points(91, n, m), synth.vectors(91, n, m)
    out1, s1 = oracle.hvp_batch("rosenbrock", P, V, 2, threads=1)
    out4, s4 = oracle.hvp_batch("rosenbrock", P, V, 2, threads=4)
    assert np.array_equal(out1, out4) and np.array_equal(s1, s4)
    for e in (0, 17, m - 1):
        o, _ = oracle.chess_vec("rosenbrock", P[e], V[e], 2)
        assert np.array_equal(o, out1[e])
    H = oracle.hessian_batch("ackley", P, 4, threads=3)
    He, _ = oracle.hessian("ackley", P[5], algo="chunk", C=4)
    assert np.array_equal(H[5], He)
    o8 = oracle.sc_hvp_batch("rosenbrock", P, V, 2, threads=2)
    assert np.all(oracle.componentwise_error(o8, out1, s1) <= 1e-13)
    e0, _ = oracle.hvp_batch("rosenbrock", P[:0], V[:0], 2)
    assert e0.shape == (0, n)


# ------------------------------------------------------------------ operation counts (§V)
@pytest.mark.parametrize("ex", GOLD["counts"], ids=lambda e: e["cite"][:40])
def test_count_pins(ex):
    n = ex["n"]
    (_, c) = oracle.count(oracle.hessian, ex["func"], np.arange(1.0, n + 1), algo=ex["algo"], C=ex["C"])
    for k in ("mul", "add", "evals"):
        if k in ex:
            assert c[k] == ex[k], k


@pytest.mark.parametrize("n", [2, 4, 6, 8, 12])
def test_paper_count_formulas(n):
    """CHUNK-HESS makes n^2/C calls and (6+3/C) n^2 M multiplications for
    an add/mul-only f (prodsum: M = n-1, A = n-2).  Additions follow the Fig. 1 code,
    4C+1 per product (G1): 4n^2 M + n^2 M/C + (2+2/C) n^2 A.  SCHUNK-HESS makes
    n(n/C+1)/2 calls and (3/2) n (2n + 2C + n/C + 1) M multiplications."""
    M, A = n - 1, n - 2
    a = np.arange(1.0, n + 1)
    for C in divisors(n):
        _, c = oracle.count(oracle.hessian, "prodsum", a, algo="chunk", C=C)
        assert c["evals"] == n * n // C
        assert Fraction(c["mul"]) == Fraction(6 * C + 3, C) * n * n * M
        assert Fraction(c["add"]) == 4 * n * n * M + Fraction(n * n * M, C) + Fraction(2 * C + 2, C) * n * n * A
        _, c = oracle.count(oracle.hessian, "prodsum", a, algo="schunk", C=C)
        assert c["evals"] == n * (n // C + 1) // 2
        assert Fraction(c["mul"]) == Fraction(3, 2) * n * (2 * n + 2 * C + Fraction(n, C) + 1) * M


def test_call_counts():
    """n^2, n(n+1)/2, n^2/C, n(n/C+1)/2 evaluations (Alg 2, 3, 5, 6)."""
    n = 12
    a = synth.points(3, n, 1)[0]
    assert oracle.count(oracle.hessian, "rosenbrock", a, algo="full")[1]["evals"] == n * n
    assert oracle.count(oracle.hessian, "rosenbrock", a, algo="sym")[1]["evals"] == n * (n + 1) // 2
    for C in divisors(n):
        assert oracle.count(oracle.hessian, "rosenbrock", a, algo="chunk", C=C)[1]["evals"] == n * n // C
        assert oracle.count(oracle.hessian, "rosenbrock", a, algo="schunk", C=C)[1]["evals"] == n * (n // C + 1) // 2
        assert oracle.count(oracle.sc_hess_vec, "rosenbrock", a, a, C)[1]["evals"] == n * (n // C + 1) // 2


# per-evaluation hDual op counts of the canonical forms (DESIGN.md table):
# (hh_mul, hh_add, s_mul, s_add, unary)
OPS = {
    "rosenbrock": lambda n: (3 * (n - 1), 3 * n - 4, n - 1, n - 1, 0),
    "ackley": lambda n: (n, 2 * n - 1, n + 4, 1, n + 3),
    "fletcher_powell": lambda n: (n, 2 * n * n - 1, 2 * n * n, n, 2 * n),
    "prodsum": lambda n: (n - 1, n - 2, 0, 0, 0),
}


@pytest.mark.parametrize("func", FUNCS)
@pytest.mark.parametrize("n,C", [(2, 1), (4, 2), (6, 3), (8, 8)])
def test_full_function_counts(func, n, C):
    """Counting run of Alg 7 = the per-op costs of Fig. 1 (hh* 6C+3 mul / 4C+1 add;
    hh+ 2C+2 add; s* 2C+2 mul; s+ 1 add; unary 3C+2 mul / C add) times the op counts
    of the canonical forms, times n^2/C calls, plus the n^2 mul + n^2 add of the dot
    (PAPER.md:392-394).  This is the model-FLOP accounting of DESIGN.md."""
    params = _params(func, n)
    a = synth.points(5, n, 1)[0] + 3.0  # away from the Ackley origin
    hm, ha, sm, sa, un = OPS[func](n)
    mul = hm * (6 * C + 3) + sm * (2 * C + 2) + un * (3 * C + 2)
    add = hm * (4 * C + 1) + ha * (2 * C + 2) + sa + un * C
    _, c = oracle.count(oracle.chess_vec, func, a, a, C, params)
    assert c["evals"] == n * n // C
    assert c["mul"] == n * n // C * mul + n * n
    assert c["add"] == n * n // C * add + n * n


def test_optimal_chunk_sqrt_n_over_2():
    """§V: SCHUNK mults (3/2) n (2n + 2C + n/C + 1) M are minimised near C = sqrt(n/2)
    (PAPER.md:368); verified here on counted multiplications of the oracle."""
    for n, best in ((8, 2), (32, 4)):
        a = np.linspace(0.1, 1.0, n)
        counts = {C: oracle.count(oracle.hessian, "prodsum", a, algo="schunk", C=C)[1]["mul"] for C in divisors(n)}
        assert min(counts, key=lambda C: (counts[C], C)) == best
