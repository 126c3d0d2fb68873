"""CUDA path vs the CPU oracle, element by element, through the C-ABI (libchessfad.so).

Metric: componentwise err_{e,i} = |g - r| / max(|r|, s_{e,i}),
s = sum_j |H_ij||v_j| from the oracle; the north-star bar is max err <= 1e-10.  The
expected margin is ~1e-15 (FMA contraction + reduction order only), so every test also
asserts a tighter 1e-12 that a real bug (wrong slot / seed / term) cannot pass.
Integer-valued inputs must match the exact closed form bit for bit.
"""
import numpy as np
import pytest

import oracle
import synth
from tests import closed_forms as cf

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FUNCS = ["rosenbrock", "ackley", "fletcher_powell", "prodsum"]
TOL = 1e-10
TIGHT = 1e-12


@pytest.fixture(scope="module")
def chf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_22575_b200 as m
    m.load()
    return m


def _params(func, n, seed=0):
    return synth.fp_params_flat(seed, n) if func == "fletcher_powell" else None


def _gpu_hvp(chf, func, P, V, C, params=None):
    dev = torch.device("cuda")
    p = torch.from_numpy(P).to(dev)
    v = torch.from_numpy(V).to(dev)
    pr = None if params is None else torch.from_numpy(params).to(dev)
    out = chf.hvp_batch(func, p, v, C, pr)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _check(gpu, ref, sabs, tol=TOL):
    err = oracle.componentwise_error(gpu, ref, sabs)
    assert np.all(np.isfinite(gpu))
    assert err.max() <= tol, f"max componentwise err {err.max():.3e}"
    assert err.max() <= TIGHT, f"max componentwise err {err.max():.3e} (tight bar)"
    return float(err.max())


def divisors(n):
    return [c for c in range(1, n + 1) if n % c == 0]


# ------------------------------------------------------------ config 1: n=2, C=1, m=1024, every point
def test_config1_every_point(chf):
    n, m = 2, 1024
    P, V = synth.points(0, n, m), synth.vectors(0, n, m)
    for func in FUNCS:
        params = _params(func, n)
        ref, sabs = oracle.hvp_batch(func, P, V, 1, params)
        _check(_gpu_hvp(chf, func, P, V, 1, params), ref, sabs)


# ------------------------------------------------------------ sweep of n, C: several tiles + ragged tail
@pytest.mark.parametrize("func", FUNCS)
@pytest.mark.parametrize("n", [2, 3, 4, 6, 8, 12, 16, 32])
def test_parity_sweep(chf, func, n):
    m = 3 * 32 * 8 + 13  # several CTAs of the widest tile and a ragged tail
    if func == "fletcher_powell" and n >= 32:
        m = 301
    P, V = synth.points(1, n, m), synth.vectors(1, n, m)
    params = _params(func, n)
    ref, sabs = oracle.hvp_batch(func, P, V, 1, params)  # the oracle is C-invariant
    for C in divisors(n):
        if not chf.is_supported(func, n, C):
            continue
        _check(_gpu_hvp(chf, func, P, V, C, params), ref, sabs)


@pytest.mark.parametrize("func", FUNCS)
def test_large_n(chf, func):
    for n in (64, 128):
        m = (45 if n == 64 else 9) if func == "fletcher_powell" else 70
        P, V = synth.points(2, n, m), synth.vectors(2, n, m)
        params = _params(func, n)
        ref, sabs = oracle.hvp_batch(func, P, V, n if n <= 32 else 32, params)
        for C in [1, 2, 4, 8, 16, 32, 64, n]:
            if chf.is_supported(func, n, C):
                _check(_gpu_hvp(chf, func, P, V, C, params), ref, sabs)


# ------------------------------------------------------------ bit-exact integer pin
@pytest.mark.parametrize("func", ["rosenbrock", "prodsum"])
@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64])
def test_integer_inputs_bitwise(chf, func, n):
    """Integer points/vectors in {-9..9}: every intermediate is an exact integer, so the GPU
    must equal the exact rational closed form bit for bit under any FMA/reduction order."""
    m = 300
    P, V = synth.int_points(5, n, m), synth.int_vectors(5, n, m)
    want = np.zeros((m, n))
    for e in range(m):
        H = cf.rosenbrock_hessian_exact(P[e]) if func == "rosenbrock" else cf.prodsum_hessian_exact(n)
        want[e] = [float(x) for x in cf.exact_hvp(H, V[e])]
    for C in divisors(n):
        if chf.is_supported(func, n, C):
            assert np.array_equal(_gpu_hvp(chf, func, P, V, C), want)


def test_golden_values(chf):
    got = _gpu_hvp(chf, "rosenbrock", np.array([[1.0, 2, 3, 4]]), np.ones((1, 4)), 2)
    assert np.array_equal(got[0], [2.0, 2602.0, 7402.0, -1000.0])
    got = _gpu_hvp(chf, "rosenbrock", np.array([[1.0, 1.0]]), np.ones((1, 2)), 1)
    assert np.array_equal(got[0], [402.0, -200.0])
    got = _gpu_hvp(chf, "ackley", np.array([[0.5, -0.25]]), np.array([[1.0, 2.0]]), 2)
    np.testing.assert_allclose(got[0], [-7.2973882525010968, -2.6223411680113156], rtol=1e-14)


# ------------------------------------------------------------ Hessian API (Alg 5)
@pytest.mark.parametrize("func", FUNCS)
def test_hessian_parity(chf, func):
    n, m = 32, 200
    P = synth.points(3, n, m)
    params = _params(func, n)
    ref = oracle.hessian_batch(func, P, 4, params)
    dev = torch.device("cuda")
    pr = None if params is None else torch.from_numpy(params).to(dev)
    for C in divisors(n):
        if not chf.is_supported(func, n, C):
            continue
        H = chf.hessian_batch(func, torch.from_numpy(P).to(dev), C, pr).cpu().numpy()
        scale = np.abs(ref).reshape(m, -1).max(axis=1)
        err = (np.abs(H - ref).reshape(m, -1).max(axis=1) / scale).max()
        assert err <= TIGHT, (C, err)
        sym = (np.abs(H - H.transpose(0, 2, 1)).reshape(m, -1).max(axis=1) / scale).max()
        assert sym <= 1e-13


def test_hessian_closed_form_rosenbrock(chf):
    n, m = 32, 64
    P = synth.int_points(9, n, m)
    H = chf.hessian_batch("rosenbrock", torch.from_numpy(P).cuda(), 8).cpu().numpy()
    for e in range(m):
        assert np.array_equal(H[e], cf.to_float(cf.rosenbrock_hessian_exact(P[e])))


# ------------------------------------------------------------ edge cases
def test_edge_cases(chf):
    dev = torch.device("cuda")
    # m == 0
    out = chf.hvp_batch("rosenbrock", torch.empty((0, 4), dtype=torch.float64, device=dev),
                        torch.empty((0, 4), dtype=torch.float64, device=dev), 2)
    assert out.shape == (0, 4)
    # m == 1 and m == 33 (one full group + 1)
    for m in (1, 33):
        P, V = synth.points(4, 16, m), synth.vectors(4, 16, m)
        ref, sabs = oracle.hvp_batch("ackley", P, V, 4)
        _check(_gpu_hvp(chf, "ackley", P, V, 16, None), ref, sabs)
    # Ackley at the origin: NaN derivatives propagate (not an error)
    got = _gpu_hvp(chf, "ackley", np.zeros((2, 4)), np.ones((2, 4)), 2)
    assert np.all(np.isnan(got))
    # Ackley n = 1
    P, V = synth.points(6, 1, 50), synth.vectors(6, 1, 50)
    ref, sabs = oracle.hvp_batch("ackley", P, V, 1)
    _check(_gpu_hvp(chf, "ackley", P, V, 1), ref, sabs)
    # errors surface as exceptions
    with pytest.raises(chf.ChessfadError, match="ERR_CHUNK"):
        _gpu_hvp(chf, "rosenbrock", np.zeros((4, 6)), np.zeros((4, 6)), 4)
    with pytest.raises(TypeError):
        chf.hvp_batch("rosenbrock", torch.zeros((4, 4), dtype=torch.float32, device=dev),
                      torch.zeros((4, 4), dtype=torch.float32, device=dev), 2)


@pytest.mark.parametrize("family,func,n,C", [("stream", "rosenbrock", 2, 1), ("stream", "ackley", 4, 2),
                                              ("stream", "prodsum", 8, 8), ("reg", "rosenbrock", 5, 5),
                                              ("reg_ns", "ackley", 16, 16), ("reg_ns", "rosenbrock", 32, 4),
                                              ("reg_ns", "prodsum", 16, 2), ("reg", "ackley", 12, 4),
                                              ("reg_ns", "prodsum", 64, 16), ("reg_ns", "rosenbrock", 128, 16),
                                              ("reg_ns", "ackley", 64, 8), ("reg_ns", "ackley", 8, 8),
                                              ("reg_ns", "rosenbrock", 16, 4), ("reg_ns", "rosenbrock", 64, 2), ("f3_dmma", "fletcher_powell", 16, 4),
                                              ("f3_dmma", "fletcher_powell", 72, 8)])
def test_small_m_every_family(chf, family, func, n, C):
    """Tiny and ragged batches on every kernel family: m = 1, 2, 7, 63, 65, 257 (one partial
    tile / CTA / warp, exact multiples +- 1), HVP and Hessian, against the oracle."""
    assert chf.path(func, n, C) == family
    params = _params(func, n)
    dev = torch.device("cuda")
    pr = None if params is None else torch.from_numpy(params).to(dev)
    for m in (1, 2, 7, 63, 65, 257):
        if func == "fletcher_powell" and n > 16 and m > 65:
            continue
        P, V = synth.points(50 + m, n, m), synth.vectors(50 + m, n, m)
        ref, sabs = oracle.hvp_batch(func, P, V, C, params)
        _check(_gpu_hvp(chf, func, P, V, C, params), ref, sabs)
        k = min(m, 7)
        H = chf.hessian_batch(func, torch.from_numpy(P[:k]).to(dev), C, pr).cpu().numpy()
        Href = oracle.hessian_batch(func, P[:k], C, params)
        scale = np.maximum(np.abs(Href).max(axis=(1, 2)), 1e-300)
        assert (np.abs(H - Href).max(axis=(1, 2)) / scale).max() <= TIGHT, m


def test_nan_propagates_every_family(chf):
    """Ackley at the origin has NaN derivatives: they propagate (no error) through
    the stream kernel (n = 2), the register kernel (n = 16) and a NaN input through F3."""
    for n, C in ((2, 1), (16, 4)):
        got = _gpu_hvp(chf, "ackley", np.zeros((3, n)), np.ones((3, n)), C)
        assert np.all(np.isnan(got)), n
    P = synth.points(3, 16, 64)
    P[5, 3] = np.nan
    got = _gpu_hvp(chf, "fletcher_powell", P, np.ones((64, 16)), 4, _params("fletcher_powell", 16))
    assert np.all(np.isnan(got[5])) and np.all(np.isfinite(np.delete(got, 5, axis=0)))


def test_determinism_and_shards(chf):
    """No atomics, fixed order: bitwise identical run to run, and a batch computed in
    shards (as the multi-GPU driver does) equals the unsharded batch bit for bit."""
    n, m = 16, 4096 + 7
    P, V = synth.points(8, n, m), synth.vectors(8, n, m)
    for func in FUNCS:
        params = _params(func, n)
        a = _gpu_hvp(chf, func, P, V, 4, params)
        b = _gpu_hvp(chf, func, P, V, 4, params)
        assert np.array_equal(a, b)
        cuts = [0, 1000, 1001, 2500, m]
        parts = [_gpu_hvp(chf, func, P[c0:c1], V[c0:c1], 4, params) for c0, c1 in zip(cuts[:-1], cuts[1:])]
        assert np.array_equal(np.concatenate(parts), a)


def test_host_api_matches_device_api(chf):
    n, m = 16, 5000
    P, V = synth.points(10, n, m), synth.vectors(10, n, m)
    for func in FUNCS:
        params = _params(func, n)
        dev_out = _gpu_hvp(chf, func, P, V, 8, params)
        host_out = chf.hvp_batch_host(func, P, V, 8, params, piece_points=999)
        assert np.array_equal(np.asarray(host_out), dev_out)


# ------------------------------------------------------------ full size, bench launch configuration
HVP_ENTRIES = {"hvp": "hvp_batch", "sym_hvp": "sym_hvp_batch", "hvp_hoisted": "hvp_batch_hoisted",
               "hvp_seedsparse": "hvp_batch_seedsparse"}


@pytest.mark.parametrize("func", FUNCS)
def test_cfg2_every_point(chf, func):
    """cfg2 at BASELINE size (n=16, m=2^20), EVERY point, every C in {1,2,4,8,16} and every HVP
    entry point (Alg 7 in the bench launch configuration, Alg 8, NEXT-4 hoisted and
    seed-sparse) against the oracle (computed once: its HVP is bitwise C-invariant,
    test_oracle_pins.test_chunk_invariance) and against the vectorised closed form
    (tests/closed_forms_np.py, independent of both)."""
    from tests import closed_forms_np as cfn
    n, m = 16, 1 << 20
    P, V = synth.points(0, n, m), synth.vectors(0, n, m)
    params = _params(func, n)
    ref, sabs = oracle.hvp_batch(func, P, V, 16, params)
    hv, S = cfn.hvp(func, P, V, params)
    assert cfn.error(ref, hv, S) <= TIGHT  # the oracle itself at every point
    dev = torch.device("cuda")
    p, v = torch.from_numpy(P).to(dev), torch.from_numpy(V).to(dev)
    pr = None if params is None else torch.from_numpy(params).to(dev)
    out = torch.empty_like(p)
    for algo, entry in HVP_ENTRIES.items():
        for C in (1, 2, 4, 8, 16):
            if not chf.is_supported(func, n, C, algo):
                continue
            out.fill_(np.nan)
            getattr(chf, entry)(func, p, v, C, pr, out=out)
            got = out.cpu().numpy()
            _check(got, ref, sabs)
            assert cfn.error(got, hv, S) <= TIGHT, (algo, C)


# ------------------------------------------------------------ n in {2, 4, 8}: the bulk-copy streaming kernel
@pytest.mark.parametrize("n", [2, 4, 8])
def test_stream_small_persistent(chf, n):
    """hvp_stream_kernel (stream_small.cuh): enough tiles that every CTA of the persistent
    grid cycles its shared-memory ring several times, a ragged last tile, every point checked;
    a 16-byte-misaligned view takes the runtime-n kernel and agrees."""
    m = {2: 1_500_007, 4: 600_011, 8: 150_001}[n]
    P, V = synth.points(30, n, m), synth.vectors(30, n, m)
    dev = torch.device("cuda")
    for func in ("rosenbrock", "ackley", "prodsum"):
        ref, sabs = oracle.hvp_batch(func, P, V, 1, None)
        for C in divisors(n):
            _check(_gpu_hvp(chf, func, P, V, C), ref, sabs)
        k = min(m, 4099)
        flat_p = torch.empty(k * n + 1, dtype=torch.float64, device=dev)
        flat_v = torch.empty(k * n + 1, dtype=torch.float64, device=dev)
        flat_o = torch.empty(k * n + 1, dtype=torch.float64, device=dev)
        flat_p[1:] = torch.from_numpy(P[:k].ravel()).to(dev)
        flat_v[1:] = torch.from_numpy(V[:k].ravel()).to(dev)
        got = chf.hvp_batch(func, flat_p[1:].view(k, n), flat_v[1:].view(k, n), 1, out=flat_o[1:].view(k, n))
        _check(got.cpu().numpy(), ref[:k], sabs[:k])


# ------------------------------------------------------------ NEXT-1 / NEXT-2: symmetric algorithms
@pytest.mark.parametrize("func", FUNCS)
@pytest.mark.parametrize("n", [2, 6, 16, 32])
def test_sym_hvp_parity(chf, func, n):
    """Alg 8 on the GPU vs the oracle's Alg 8 (same accumulation order up to contraction) and
    vs Alg 7 (the same product)."""
    m = 300 if not (func == "fletcher_powell" and n == 32) else 120
    P, V = synth.points(14, n, m), synth.vectors(14, n, m)
    params = _params(func, n)
    ref7, sabs = oracle.hvp_batch(func, P, V, 1, params)
    dev = torch.device("cuda")
    pr = None if params is None else torch.from_numpy(params).to(dev)
    for C in divisors(n):
        if not chf.is_supported(func, n, C, "sym_hvp"):
            continue
        got = chf.sym_hvp_batch(func, torch.from_numpy(P).to(dev), torch.from_numpy(V).to(dev), C, pr).cpu().numpy()
        ref8 = oracle.sc_hvp_batch(func, P, V, C, params)
        _check(got, ref8, sabs)
        _check(got, ref7, sabs)


@pytest.mark.parametrize("n,m", [(12, 77), (20, 65), (64, 41), (72, 19), (100, 9), (128, 9)])
def test_f3_dmma_all_modes(chf, n, m):
    """Fletcher-Powell on the tensor-core kernel (f3_mma.cuh): zero-padded n (12, 20, 72, 100),
    the k-blocked M (n > 64) and a ragged CTA, every entry point -- Alg 7, Alg 8 (now for every
    n <= 128), Alg 5, Alg 6, gradient, row-hoisted -- against the oracle (the closed form for
    the Hessian at the sampled points)."""
    func = "fletcher_powell"
    P, V = synth.points(40, n, m), synth.vectors(40, n, m)
    params = _params(func, n)
    dev = torch.device("cuda")
    p, v, pr = (torch.from_numpy(x).to(dev) for x in (P, V, params))
    ms = m if n <= 72 else 4  # oracle cost at n = 128: ~3 s per point and C
    ref, sabs = oracle.hvp_batch(func, P[:ms], V[:ms], n, params)
    Cs = sorted({1, 4 if n % 4 == 0 else 1, n // 2 if n % 2 == 0 else n, n})
    hs = [0, m - 1] if n > 72 else list(range(m))
    Href = np.stack([cf.to_float(cf.fp_hessian_mp(P[e], params[:n * n].reshape(n, n),
                                                   params[n * n:2 * n * n].reshape(n, n), params[2 * n * n:]))
                     for e in hs]) if n <= 20 else oracle.hessian_batch(func, P[hs], n, params)
    for C in Cs:
        assert chf.path(func, n, C) == "f3_dmma"
        for entry in ("hvp_batch", "sym_hvp_batch", "hvp_batch_hoisted"):
            got = getattr(chf, entry)(func, p, v, C, pr).cpu().numpy()
            _check(got[:ms], ref, sabs)
        for entry in ("hessian_batch", "sym_hessian_batch"):
            H = getattr(chf, entry)(func, p, C, pr).cpu().numpy()[hs]
            rel = np.abs(H - Href).max(axis=(1, 2)) / np.abs(Href).max(axis=(1, 2))
            assert rel.max() <= TIGHT, (entry, C, rel.max())
        Hg, grad = chf.hessian_grad_batch(func, p, C, pr)
        g_ref = np.stack([oracle.hessian(func, P[e], params, algo="chunk", C=n)[1] for e in hs[:2]])
        gs = np.abs(g_ref).max(axis=1, keepdims=True)
        assert (np.abs(grad.cpu().numpy()[hs[:2]] - g_ref) / gs).max() <= TIGHT


@pytest.mark.parametrize("func", ["rosenbrock", "ackley", "prodsum"])
@pytest.mark.parametrize("n,m", [(6, 90), (16, 200), (64, 40)])
def test_seedsparse_sym_and_grad(chf, func, n, m):
    """Seed sparsity for Alg 8, Alg 6 and the gradient by-product (F1/F2/F4): the same values as
    the per-evaluation symmetric / gradient kernels (up to the sign of zero), and the oracle's
    Alg 8 / Hessian / gradient.  (Fletcher-Powell: test_seedsparse_f3_sym_hvp.)"""
    P, V = synth.points(45, n, m), synth.vectors(45, n, m)
    dev = torch.device("cuda")
    p, v = torch.from_numpy(P).to(dev), torch.from_numpy(V).to(dev)
    ref7, sabs = oracle.hvp_batch(func, P, V, 1)
    for C in sorted({1, 2, n // 2 if n // 2 <= 16 else 16}):
        if n % C or not chf.is_supported(func, n, C, "sym_hvp_seedsparse"):
            continue
        a = chf.sym_hvp_batch(func, p, v, C).cpu().numpy()
        b = chf.sym_hvp_batch_seedsparse(func, p, v, C).cpu().numpy()
        assert np.array_equal(a, b), C
        _check(b, oracle.sc_hvp_batch(func, P, V, C), sabs)
        _check(b, ref7, sabs)
        Ha = chf.sym_hessian_batch(func, p[:24], C).cpu().numpy()
        Hb = chf.sym_hessian_batch_seedsparse(func, p[:24], C).cpu().numpy()
        assert np.array_equal(Ha, Hb), C
        Ga, ga = chf.hessian_grad_batch(func, p[:24], C)
        Gb, gb = chf.hessian_grad_batch_seedsparse(func, p[:24], C)
        assert torch.equal(Ga, Gb) and torch.equal(ga, gb), C
        href = oracle.hessian_batch(func, P[:24], C)
        rel = np.abs(Hb - href).max(axis=(1, 2)) / np.abs(href).max(axis=(1, 2))
        assert rel.max() <= TIGHT
        g_ref = np.stack([oracle.hessian(func, P[e], None, algo="chunk", C=C)[1] for e in range(4)])
        gs = np.abs(g_ref).max(axis=1, keepdims=True)
        assert (np.abs(gb.cpu().numpy()[:4] - g_ref) / gs).max() <= TIGHT


@pytest.mark.parametrize("n,m", [(6, 90), (16, 150), (32, 70), (40, 37), (64, 33)])
def test_seedsparse_f3_sym_hvp(chf, n, m):
    """Seed-sparse Alg 8 for Fletcher-Powell (every warp owns a 32-point group and walks all of
    its rows; mirror terms accumulated in the output tile, or in the output row in global
    memory for n > 32): the oracle's Alg 8 and Alg 7, and the tensor-core Alg 8 within rounding
    (its E-sums associate differently, reading R6); ragged m; n > 64 is refused."""
    func = "fletcher_powell"
    P, V = synth.points(47, n, m), synth.vectors(47, n, m)
    params = synth.fp_params_flat(0, n)
    dev = torch.device("cuda")
    p, v, pr = torch.from_numpy(P).to(dev), torch.from_numpy(V).to(dev), torch.from_numpy(params).to(dev)
    ref7, sabs = oracle.hvp_batch(func, P, V, 1, params)
    for C in sorted({1, 2, n // 2 if n // 2 <= 16 else 8, n}):
        if n % C:
            continue
        assert chf.is_supported(func, n, C, "sym_hvp_seedsparse")
        b = chf.sym_hvp_batch_seedsparse(func, p, v, C, pr).cpu().numpy()
        _check(b, oracle.sc_hvp_batch(func, P, V, C, params), sabs)
        _check(b, ref7, sabs)
        _check(b, chf.sym_hvp_batch(func, p, v, C, pr).cpu().numpy(), sabs)
    assert not chf.is_supported(func, 72, 8, "sym_hvp_seedsparse")
    p72 = torch.zeros((2, 72), dtype=torch.float64, device=dev)
    with pytest.raises(chf.ChessfadError):
        chf.sym_hvp_batch_seedsparse(func, p72, p72, 8, torch.from_numpy(synth.fp_params_flat(0, 72)).to(dev))


@pytest.mark.parametrize("func", ["rosenbrock", "prodsum"])
def test_sym_hvp_integer_bitwise(chf, func):
    n, m = 16, 200
    P, V = synth.int_points(15, n, m), synth.int_vectors(15, n, m)
    want = np.zeros((m, n))
    for e in range(m):
        H = cf.rosenbrock_hessian_exact(P[e]) if func == "rosenbrock" else cf.prodsum_hessian_exact(n)
        want[e] = [float(x) for x in cf.exact_hvp(H, V[e])]
    for C in (1, 2, 4, 8, 16):
        got = chf.sym_hvp_batch(func, torch.from_numpy(P).cuda(), torch.from_numpy(V).cuda(), C).cpu().numpy()
        assert np.array_equal(got, want), C


@pytest.mark.parametrize("func", FUNCS)
@pytest.mark.parametrize("n", [16, 32])
def test_sym_hessian_parity(chf, func, n):
    """Alg 6 on the GPU: equals the oracle's Alg 6 within rounding, its computed (upper-chunk)
    entries equal the GPU's Alg 5 bit for bit, and it is exactly symmetric outside the
    diagonal chunks."""
    m = 150 if n == 16 else 60
    P = synth.points(16, n, m)
    params = _params(func, n)
    dev = torch.device("cuda")
    pr = None if params is None else torch.from_numpy(params).to(dev)
    pts = torch.from_numpy(P).to(dev)
    for C in (1, 2, 4, 8, 16):
        Hs = chf.sym_hessian_batch(func, pts, C, pr).cpu().numpy()
        Hf = chf.hessian_batch(func, pts, C, pr).cpu().numpy()
        ref = np.stack([oracle.hessian(func, P[e], params, algo="schunk", C=C)[0] for e in range(m)])
        scale = np.abs(ref).reshape(m, -1).max(axis=1)
        assert (np.abs(Hs - ref).reshape(m, -1).max(axis=1) / scale).max() <= TIGHT
        blk = np.arange(n) // C
        upper = blk[:, None] <= blk[None, :]
        assert np.array_equal(Hs[:, upper], Hf[:, upper])
        lower = blk[:, None] > blk[None, :]
        assert np.array_equal(Hs[:, lower], Hs.transpose(0, 2, 1)[:, lower])


# ------------------------------------------------------------ NEXT-4: value-channel hoisting
@pytest.mark.parametrize("n,m", [(16, 700), (64, 40)])
def test_hoisted_f3_bitwise_equal(chf, n, m):
    """F3: phase A computed once per row gives the SAME bits as once per chunk (same ops,
    same order), and matches the oracle."""
    P, V = synth.points(17, n, m), synth.vectors(17, n, m)
    params = synth.fp_params_flat(0, n)
    dev = torch.device("cuda")
    p, v, pr = (torch.from_numpy(x).to(dev) for x in (P, V, params))
    ref, sabs = oracle.hvp_batch("fletcher_powell", P, V, n // 4 if n > 16 else 4, params)
    for C in (1, 4, n):
        a = chf.hvp_batch("fletcher_powell", p, v, C, pr).cpu().numpy()
        b = chf.hvp_batch_hoisted("fletcher_powell", p, v, C, pr).cpu().numpy()
        assert np.array_equal(a, b)
        _check(b, ref, sabs)


@pytest.mark.parametrize("n,m", [(2, 300), (3, 100), (4, 200), (8, 150), (12, 70), (16, 700), (32, 100), (36, 40),
                                 (64, 40), (72, 20), (128, 33)])
def test_seedsparse_f3(chf, n, m):
    """NEXT-4 seed sparsity: skipping the products of exact-zero seed slots leaves the same
    bits as the per-evaluation path (up to the sign of zero; == treats -0 == +0) for every C,
    and matches the oracle."""
    P, V = synth.points(19, n, m), synth.vectors(19, n, m)
    params = synth.fp_params_flat(0, n)
    dev = torch.device("cuda")
    p, v, pr = (torch.from_numpy(x).to(dev) for x in (P, V, params))
    ms = min(m, 12) if n >= 64 else m  # oracle cost at n = 128: ~3 s per point
    ref, sabs = oracle.hvp_batch("fletcher_powell", P[:ms], V[:ms], n, params)
    Cs = sorted({1, n} | ({4} if n % 4 == 0 else set()))
    for C in Cs:
        b = chf.hvp_batch_seedsparse("fletcher_powell", p, v, C, pr).cpu().numpy()
        if (n <= 64 or C == n) and chf.is_supported("fletcher_powell", n, C, "hvp"):
            a = chf.hvp_batch("fletcher_powell", p, v, C, pr).cpu().numpy()
            _same_as_per_eval(chf, n, C, a, b)
        _check(b[:ms], ref, sabs)


def _same_as_per_eval(chf, n, C, a, b, algo="hvp"):
    """Seed-sparse vs the per-evaluation path: within rounding (the per-evaluation F3 kernel
    sums E_k on the tensor core, whose k-step association differs from the SIMT chain the
    seed-sparse kernel copies; it was bit-identical to the retired SIMT kernel, round 1)."""
    assert chf.path("fletcher_powell", n, C, algo) == "f3_dmma"
    scale = np.abs(a).max(axis=tuple(range(1, a.ndim)), keepdims=True)
    assert (np.abs(a - b) / scale).max() <= TIGHT, f"C={C}: max rel diff {(np.abs(a - b) / scale).max():.3e}"


@pytest.mark.parametrize("n,m", [(6, 70), (16, 130), (40, 20), (64, 9)])
def test_seedsparse_f3_sym_hessian_and_grad(chf, n, m):
    """F3 seed sparsity for Alg 6 (upper chunks computed, later chunks mirrored) and the
    gradient by-product, against the per-evaluation (tensor-core) Hessian / gradient and the
    oracle; n = 40 and 64 take the unstaged / staged (A, B) paths."""
    func = "fletcher_powell"
    P = synth.points(22, n, m)
    params = synth.fp_params_flat(0, n)
    dev = torch.device("cuda")
    p, pr = torch.from_numpy(P).to(dev), torch.from_numpy(params).to(dev)
    Href = oracle.hessian_batch(func, P, n, params)
    hs = np.abs(Href).max(axis=(1, 2))
    for C in sorted({1, 2, n // 2, n}):
        if n % C:
            continue
        Hs = chf.sym_hessian_batch_seedsparse(func, p, C, pr).cpu().numpy()
        assert (np.abs(Hs - Href).max(axis=(1, 2)) / hs).max() <= TIGHT, C
        Hd = chf.sym_hessian_batch(func, p, C, pr).cpu().numpy()
        assert (np.abs(Hs - Hd).max(axis=(1, 2)) / hs).max() <= TIGHT, C
        Hg, g = chf.hessian_grad_batch_seedsparse(func, p, C, pr)
        Hg, g = Hg.cpu().numpy(), g.cpu().numpy()
        assert (np.abs(Hg - Href).max(axis=(1, 2)) / hs).max() <= TIGHT, C
        _, g_dev = chf.hessian_grad_batch(func, p, C, pr)
        g_dev = g_dev.cpu().numpy()
        gs = np.abs(g_dev).max(axis=1, keepdims=True)
        assert (np.abs(g - g_dev) / gs).max() <= TIGHT, C
    g_ref = np.stack([oracle.hessian(func, P[e], params, algo="chunk", C=n)[1] for e in range(3)])
    assert (np.abs(g[:3] - g_ref) / np.abs(g_ref).max(axis=1, keepdims=True)).max() <= TIGHT


@pytest.mark.parametrize("n,m", [(2, 100), (8, 70), (32, 50), (64, 9), (128, 5)])
def test_seedsparse_f3_hessian(chf, n, m):
    """Seed-sparse Hessian (Alg 5 output): same bits as hessian_batch up to the sign of zero,
    oracle parity."""
    P = synth.points(21, n, m)
    params = synth.fp_params_flat(0, n)
    dev = torch.device("cuda")
    p, pr = torch.from_numpy(P).to(dev), torch.from_numpy(params).to(dev)
    Href = oracle.hessian_batch("fletcher_powell", P, n, params)
    for C in sorted({1, n}):
        a = chf.hessian_batch("fletcher_powell", p, C, pr).cpu().numpy()
        b = chf.hessian_batch_seedsparse("fletcher_powell", p, C, pr).cpu().numpy()
        _same_as_per_eval(chf, n, C, a, b, algo="hessian")
        rel = np.max(np.abs(b - Href), axis=(1, 2)) / np.max(np.abs(Href), axis=(1, 2))
        assert rel.max() <= TIGHT


@pytest.mark.parametrize("func", ["rosenbrock", "ackley", "prodsum"])
@pytest.mark.parametrize("n,m", [(2, 100), (3, 70), (8, 100), (16, 300), (24, 60), (64, 40), (128, 20)])
def test_seedsparse_register_functions(chf, func, n, m):
    """NEXT-4 seed sparsity, F1/F2/F4: only the terms touching {i} U chunk are evaluated as
    hDuals; same bits as the per-evaluation path up to the sign of zero (HVP and Hessian, every
    compiled C and a column-group C), oracle parity, bit-exact integer pins."""
    P, V = synth.points(29, n, m), synth.vectors(29, n, m)
    dev = torch.device("cuda")
    p, v = torch.from_numpy(P).to(dev), torch.from_numpy(V).to(dev)
    ref, sabs = oracle.hvp_batch(func, P, V, 1)
    for C in sorted({1, n if n <= 32 else 32} | ({2} if n % 2 == 0 else set())):
        a = chf.hvp_batch(func, p, v, C).cpu().numpy()
        b = chf.hvp_batch_seedsparse(func, p, v, C).cpu().numpy()
        if chf.path(func, n, C) == "stream":  # the register-resident kernel: its own FMA contraction
            _check(a, ref, sabs)
        else:
            assert np.array_equal(a, b), f"C={C}: max |diff| {np.abs(a - b).max():.3e}"
        _check(b, ref, sabs)
        if n <= 64:
            Ha = chf.hessian_batch(func, p[:16], C).cpu().numpy()
            Hb = chf.hessian_batch_seedsparse(func, p[:16], C).cpu().numpy()
            assert np.array_equal(Ha, Hb)
    if func != "ackley":
        Pi, Vi = synth.int_points(31, n, 50), synth.int_vectors(31, n, 50)
        want = np.zeros((50, n))
        for e in range(50):
            H = cf.rosenbrock_hessian_exact(Pi[e]) if func == "rosenbrock" else cf.prodsum_hessian_exact(n)
            want[e] = [float(x) for x in cf.exact_hvp(H, Vi[e])]
        got = chf.hvp_batch_seedsparse(func, torch.from_numpy(Pi).cuda(), torch.from_numpy(Vi).cuda(), 1).cpu().numpy()
        assert np.array_equal(got, want)


@pytest.mark.parametrize("func", ["rosenbrock", "ackley", "prodsum"])
@pytest.mark.parametrize("n", [2, 4, 8, 12, 16])
def test_hoisted_register_functions(chf, func, n):
    """Compile-time kernels (n in {2,4,8,16}; n = 12 falls back to the per-evaluation path):
    oracle parity for every C, and bit-exact integer pins for Rosenbrock / prodsum."""
    m = 500
    P, V = synth.points(23, n, m), synth.vectors(23, n, m)
    ref, sabs = oracle.hvp_batch(func, P, V, 1)
    for C in divisors(n):
        dev = torch.device("cuda")
        got = chf.hvp_batch_hoisted(func, torch.from_numpy(P).to(dev), torch.from_numpy(V).to(dev), C).cpu().numpy()
        _check(got, ref, sabs)
    if func != "ackley":
        Pi, Vi = synth.int_points(24, n, 100), synth.int_vectors(24, n, 100)
        want = np.zeros((100, n))
        for e in range(100):
            H = cf.rosenbrock_hessian_exact(Pi[e]) if func == "rosenbrock" else cf.prodsum_hessian_exact(n)
            want[e] = [float(x) for x in cf.exact_hvp(H, Vi[e])]
        for C in divisors(n):
            got = chf.hvp_batch_hoisted(func, torch.from_numpy(Pi).cuda(), torch.from_numpy(Vi).cuda(), C).cpu().numpy()
            assert np.array_equal(got, want)


# ------------------------------------------------------------ BASELINE full sizes, sampled
def _sampled_check(chf, func, n, m, C, algo="hvp", nsample=24, seed=0):
    P, V = synth.points(seed, n, m), synth.vectors(seed, n, m)
    params = _params(func, n)
    dev = torch.device("cuda")
    p, v = torch.from_numpy(P).to(dev), torch.from_numpy(V).to(dev)
    pr = None if params is None else torch.from_numpy(params).to(dev)
    idx = np.unique(np.concatenate([[0, m - 1], np.linspace(0, m - 1, nsample).astype(np.int64)]))
    if algo in ("hessian", "sym_hessian", "hessian_seedsparse"):
        fn = {"hessian": chf.hessian_batch, "sym_hessian": chf.sym_hessian_batch,
              "hessian_seedsparse": chf.hessian_batch_seedsparse}[algo]
        H = fn(func, p, C, pr)
        got = H[torch.from_numpy(idx).to(dev)].cpu().numpy()
        del H
        ref = oracle.hessian_batch(func, P[idx], C, params)
        scale = np.abs(ref).reshape(idx.size, -1).max(axis=1)
        assert (np.abs(got - ref).reshape(idx.size, -1).max(axis=1) / scale).max() <= TIGHT
    else:
        fn = {"hvp": chf.hvp_batch, "sym_hvp": chf.sym_hvp_batch, "hvp_hoisted": chf.hvp_batch_hoisted,
              "hvp_seedsparse": chf.hvp_batch_seedsparse}[algo]
        got = fn(func, p, v, C, pr)[torch.from_numpy(idx).to(dev)].cpu().numpy()
        ref, sabs = oracle.hvp_batch(func, P[idx], V[idx], C, params)
        _check(got, ref, sabs)


@pytest.mark.parametrize("func", ["rosenbrock", "ackley", "prodsum"])
@pytest.mark.parametrize("n", [64, 128])
def test_config3_full_size_sampled(chf, func, n):
    """cfg3: n = 64 / 128, m = 2^20 (Fletcher-Powell below), C = 16 and C = n."""
    for C in (16, n):
        _sampled_check(chf, func, n, 1 << 20, C, nsample=16)


@pytest.mark.parametrize("n,m", [(64, 1 << 16), (128, 1 << 13)])
def test_config3_fletcher_powell_sampled(chf, n, m):
    """cfg3 Fletcher-Powell at the reduced m the bench sweeps use (2.3-4.4 GFLOP per point at
    n = 128 makes m = 2^20 a minutes-long launch)."""
    _sampled_check(chf, "fletcher_powell", n, m, 16, nsample=8)


@pytest.mark.parametrize("func", FUNCS)
def test_config4_hessian_full_size_sampled(chf, func):
    """cfg4: full Hessians at n = 32, m = 2^18 (2 GiB of output), Alg 5 and Alg 6."""
    for algo in ("hessian", "sym_hessian"):
        _sampled_check(chf, func, 32, 1 << 18, 8, algo=algo, nsample=12)


def test_config5_full_size_sampled(chf):
    """cfg5: n = 16, m = 2^23 on one GPU (the strong-scaling total), C = 16."""
    _sampled_check(chf, "rosenbrock", 16, 1 << 23, 16, nsample=32)
    _sampled_check(chf, "rosenbrock", 16, 1 << 23, 4, algo="sym_hvp", nsample=32)


@pytest.mark.parametrize("func", FUNCS)
def test_next4_full_size_sampled(chf, func):
    """NEXT-4 entry points at the bench's cfg2 shape (n = 16, m = 2^20, as bench.py's sweep
    times them), the seed-sparse ones also at n = 128, m = 2^20, and the seed-sparse Hessian
    at cfg4 (n = 32, m = 2^18)."""
    _sampled_check(chf, func, 16, 1 << 20, 16, algo="hvp_hoisted", nsample=16)
    _sampled_check(chf, func, 16, 1 << 20, 4, algo="hvp_seedsparse", nsample=16)
    _sampled_check(chf, func, 128, 1 << 20, 16, algo="hvp_seedsparse", nsample=4 if func == "fletcher_powell" else 8)
    _sampled_check(chf, func, 32, 1 << 18, 8, algo="hessian_seedsparse", nsample=8)


# ------------------------------------------------------------ the paper's Fig. 2 L2 design (comparison baseline)
@pytest.mark.parametrize("func", ["rosenbrock", "prodsum"])
@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_paper_l2_baseline_parity(chf, func, n):
    m = 777
    P, V = synth.points(18, n, m), synth.vectors(18, n, m)
    ref, sabs = oracle.hvp_batch(func, P, V, 1)
    dev = torch.device("cuda")
    p, v = torch.from_numpy(P).to(dev), torch.from_numpy(V).to(dev)
    for C in divisors(n):
        got = chf.hvp_batch_paper_l2(func, p, v, C).cpu().numpy()
        _check(got, ref, sabs)
        for level in (0, 1):
            _check(chf.hvp_batch_paper(level, func, p, v, C).cpu().numpy(), ref, sabs)


# ------------------------------------------------------------ gradient by-product
@pytest.mark.parametrize("func", FUNCS)
@pytest.mark.parametrize("n", [16, 32])
def test_hessian_grad(chf, func, n):
    """grad from slot v[1] == the oracle's CHUNK-HESS gradient (and the Hessian is unchanged);
    Rosenbrock on integer inputs against its exact closed-form gradient, bit for bit."""
    m = 300 if n == 16 else 100
    P = synth.points(19, n, m)
    params = _params(func, n)
    dev = torch.device("cuda")
    p = torch.from_numpy(P).to(dev)
    pr = None if params is None else torch.from_numpy(params).to(dev)
    ref_g = np.stack([oracle.hessian(func, P[e], params, algo="chunk", C=4)[1] for e in range(m)])
    for C in (1, 4, 16):
        H, g = chf.hessian_grad_batch(func, p, C, pr)
        H0 = chf.hessian_batch(func, p, C, pr)
        assert torch.equal(H, H0)
        g = g.cpu().numpy()
        scale = np.maximum(np.abs(ref_g).max(axis=1, keepdims=True), 1e-300)
        assert (np.abs(g - ref_g) / scale).max() <= TIGHT, C
    if func == "rosenbrock":
        Pi = synth.int_points(20, n, 64)
        _, g = chf.hessian_grad_batch(func, torch.from_numpy(Pi).to(dev), 8)
        a = Pi
        want = np.zeros_like(a)
        want[:, :-1] += -400 * a[:, :-1] * (a[:, 1:] - a[:, :-1] ** 2) - 2 * (1 - a[:, :-1])
        want[:, 1:] += 200 * (a[:, 1:] - a[:, :-1] ** 2)
        assert np.array_equal(g.cpu().numpy(), want)


def test_hessian_grad_f3_ring_ragged(chf):
    """Fletcher-Powell n > 32 (the cp.async (A, B) ring) with m % 32 != 0: the partial last
    warp's gradient and Hessian (tail lanes must take part in the ring)."""
    func, n, m = "fletcher_powell", 64, 45
    P = synth.points(21, n, m)
    params = _params(func, n)
    dev = torch.device("cuda")
    pr = torch.from_numpy(params).to(dev)
    ref = [oracle.hessian(func, P[e], params, algo="chunk", C=8) for e in range(m)]
    ref_H = np.stack([r[0] for r in ref])
    ref_g = np.stack([r[1] for r in ref])
    for C in (8, 64):
        H, g = chf.hessian_grad_batch(func, torch.from_numpy(P).to(dev), C, pr)
        H, g = H.cpu().numpy(), g.cpu().numpy()
        gs = np.maximum(np.abs(ref_g).max(axis=1, keepdims=True), 1e-300)
        assert (np.abs(g - ref_g) / gs).max() <= TIGHT, C
        hs = np.abs(ref_H).max(axis=(1, 2))
        assert (np.abs(H - ref_H).max(axis=(1, 2)) / hs).max() <= TIGHT, C


# ------------------------------------------------------------ maximum sizes of the compiled set
def test_maximum_n(chf):
    """Largest n each path accepts: register path n = 256 (Ackley 176),
    Fletcher-Powell n = 128; one past the limit is ERR_UNSUPPORTED."""
    for func, n, Cs in (("rosenbrock", 256, (16, 256)), ("prodsum", 256, (8, 256)), ("ackley", 176, (16, 176)),
                        ("fletcher_powell", 128, (128,))):
        m = 3 if func == "fletcher_powell" else 40
        P, V = synth.points(22, n, m), synth.vectors(22, n, m)
        params = _params(func, n)
        ref, sabs = oracle.hvp_batch(func, P, V, min(Cs[-1], 16 if n > 128 else Cs[-1]), params)  # C-invariant
        for C in Cs:
            assert chf.is_supported(func, n, C)
            _check(_gpu_hvp(chf, func, P, V, C, params), ref, sabs)
    assert not chf.is_supported("rosenbrock", 512, 16)
    assert chf.is_supported("ackley", 176, 16) and not chf.is_supported("ackley", 177, 1)
    assert not chf.is_supported("fletcher_powell", 136, 8)
