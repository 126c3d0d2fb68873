"""Oracle hDual primitives and seeding against the SPEC.md worked examples (exact equality)
and against the paper's printed rules (Fig. 1 :263-344)."""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_hdual_examples.json")))


def _num(x):
    return math.pi / 2 if x == "pi/2" else float(x)


@pytest.mark.parametrize("ex", GOLD["lift_constant"], ids=lambda e: e["cite"])
def test_lift_constant(ex):
    # lifting = c + zero hDual (Fig. 1 operator+(double, hDual))
    C = ex["C"]
    r = oracle.hd_binary("sadd", C, np.zeros(2 * C + 2), c=ex["c"])
    assert np.array_equal(r, np.array(ex["out"], dtype=float))


@pytest.mark.parametrize("ex", GOLD["binary"], ids=lambda e: e["cite"])
def test_binary(ex):
    r = oracle.hd_binary(ex["op"], ex["C"], ex["u"], ex["v"])
    assert np.array_equal(r, np.array(ex["out"], dtype=float))


@pytest.mark.parametrize("ex", GOLD["mixed"], ids=lambda e: e["cite"])
def test_mixed(ex):
    r = oracle.hd_binary(ex["op"], ex["C"], ex["u"], c=ex["c"])
    assert np.array_equal(r, np.array(ex["out"], dtype=float))


@pytest.mark.parametrize("ex", GOLD["unary"], ids=lambda e: e["cite"])
def test_unary(ex):
    u = [_num(x) for x in ex["u"]]
    r = oracle.hd_unary(ex["g"], ex["C"], u)
    np.testing.assert_allclose(r, ex["out"], rtol=0, atol=ex.get("tol", 0.0))


@pytest.mark.parametrize("ex", GOLD["compare"], ids=lambda e: e["cite"])
def test_compare(ex):
    assert oracle.hd_compare(ex["cmp"], ex["u"], ex["v"]) == ex["out"]


@pytest.mark.parametrize("ex", GOLD["initialize"], ids=lambda e: e["cite"])
def test_initialize(ex):
    assert np.array_equal(oracle.initialize(ex["a"], ex["i"], ex["j"]), np.array(ex["out"], dtype=float))


@pytest.mark.parametrize("ex", GOLD["chunk_init"], ids=lambda e: e["cite"])
def test_chunk_init(ex):
    y = oracle.chunk_init(ex["a"], ex["i"], ex["cstart"], ex["C"])
    assert np.array_equal(y, np.array(ex["out"], dtype=float))


def test_mul_rule_against_calculus():
    """The printed second-order product rule on known polynomials:
    f = x^2 y at (x, y) = (3, 2): d2f/dx2 = 2y = 4, d2f/dxdy = 2x = 6, d2f/dy2 = 0."""
    x = [3.0, 2.0]
    for (i, j, want) in [(0, 0, 4.0), (0, 1, 6.0), (1, 0, 6.0), (1, 1, 0.0)]:
        y = oracle.initialize(x, i, j)
        xx = oracle.hd_binary("mul", 1, y[0], y[0])
        f = oracle.hd_binary("mul", 1, xx, y[1])
        assert f[0] == 18.0 and f[3] == want


def test_sin_rule_printed():
    """sin(u) = <sin u0, cos u0 u1, cos u0 u2, cos u0 u3 - sin u0 u1 u2>."""
    u = [0.7, 0.3, -1.25, 2.0]
    r = oracle.hd_unary("sin", 1, u)
    assert r[0] == math.sin(0.7)
    assert r[1] == math.cos(0.7) * 0.3
    assert r[2] == math.cos(0.7) * -1.25
    assert r[3] == pytest.approx(math.cos(0.7) * 2.0 - math.sin(0.7) * 0.3 * -1.25, rel=1e-15)


@pytest.mark.parametrize("g,fn,d1,d2", [
    ("sin", math.sin, math.cos, lambda x: -math.sin(x)),
    ("cos", math.cos, lambda x: -math.sin(x), lambda x: -math.cos(x)),
    ("exp", math.exp, math.exp, math.exp),
    ("sqrt", math.sqrt, lambda x: 0.5 / math.sqrt(x), lambda x: -0.25 / (x * math.sqrt(x))),
    ("log", math.log, lambda x: 1 / x, lambda x: -1 / (x * x)),
])
def test_unary_chain_rule_on_seed(g, fn, d1, d2):
    """g applied to a seeded variable x (u = <x, 1, 1, 0>) gives <g, g', g', g''>."""
    x = 0.83
    r = oracle.hd_unary(g, 1, [x, 1.0, 1.0, 0.0])
    np.testing.assert_allclose(r, [fn(x), d1(x), d1(x), d2(x)], rtol=1e-15, atol=0)


def test_div_inverse_property():
    """mul(div(u,v), v) ~ u."""
    rng = np.random.default_rng(3)
    for C in (1, 3):
        u = rng.uniform(1, 2, 2 * C + 2)
        v = rng.uniform(1, 2, 2 * C + 2)
        v[0] = 3.0
        q = oracle.hd_binary("div", C, u, v)
        np.testing.assert_allclose(oracle.hd_binary("mul", C, q, v), u, rtol=1e-12)


def test_abs_convention():
    assert np.array_equal(oracle.hd_unary("abs", 1, [0.0, 1.0, 1.0, 5.0]), [0.0, 0.0, 0.0, 0.0])
    assert np.array_equal(oracle.hd_unary("abs", 1, [-2.0, 1.0, 3.0, 5.0]), [2.0, -1.0, -3.0, -5.0])


def test_slot_independence():
    """Slot C+k of a product depends only on slots {0,1,k,C+k}: perturbing
    another column leaves it unchanged, so chunks can be packed arbitrarily."""
    rng = np.random.default_rng(5)
    C = 4
    u, v = rng.normal(size=10), rng.normal(size=10)
    r = oracle.hd_binary("mul", C, u, v)
    u2 = u.copy()
    u2[3] += 1.0  # column k=3 (slots 3 and C+3=7)
    r2 = oracle.hd_binary("mul", C, u2, v)
    changed = np.nonzero(r != r2)[0].tolist()
    assert changed == [3, 7]


def test_duplicated_seed_invariant():
    """When row i lies in the chunk, slot 1 == slot i-cs+2 after any op sequence."""
    rng = np.random.default_rng(9)
    a = rng.uniform(-2, 2, 8)
    for func in ("rosenbrock", "ackley", "prodsum"):
        for (i, cs) in [(0, 0), (5, 4), (7, 4)]:
            y = oracle.chunk_init(a, i, cs, 4)
            t = oracle.eval_hdual(func, y, 4)
            assert t[1] == t[i - cs + 2]
