"""Randomised coverage of the dispatch space (seeded, reproducible): 150 draws of (function, n,
C, m, algorithm) across every kernel family the C-ABI can route to -- stream (n <= 8), runtime-n
register kernel, the kernels compiled for n (plain and volatile-seed / unrolled-chunk forms),
hoisted, seed-sparse, Fletcher-Powell on the tensor core and its seed-sparse kernel -- each
against the CPU oracle (Alg 7 / Alg 8 HVP componentwise, Alg 5 / Alg 6 Hessian per point),
with ragged m.  Complements the targeted tests of test_gpu_parity.py."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

NS = [2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 64, 96, 128]
ALGOS = ["hvp", "sym_hvp", "hessian", "sym_hessian", "hvp_hoisted", "hvp_seedsparse"]


@pytest.fixture(scope="module")
def chf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_22575_b200 as c
    c.load()
    return c


def _draws(k=150, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < k:
        func = ["rosenbrock", "ackley", "fletcher_powell", "prodsum"][rng.integers(4)]
        n = int(NS[rng.integers(len(NS))])
        if func in ("rosenbrock", "prodsum") and n < 2:
            continue
        algo = ALGOS[rng.integers(len(ALGOS))]
        if func == "fletcher_powell" and n > 48:
            continue  # keep the oracle's O(n^4 / C) per point cheap
        if algo in ("hessian", "sym_hessian") and n > 64:
            continue
        divs = [c for c in range(1, n + 1) if n % c == 0]
        C = int(divs[rng.integers(len(divs))])
        m = int(rng.integers(1, 300 if n <= 32 else 70))
        out.append((func, n, C, m, algo))
    return out


@pytest.mark.parametrize("func,n,C,m,algo", _draws())
def test_random_config(chf, func, n, C, m, algo):
    if not chf.is_supported(func, n, C, algo):
        pytest.skip("outside the compiled set")
    seed = 1000 + n * 7 + m
    P, V = synth.points(seed, n, m), synth.vectors(seed, n, m)
    params = synth.fp_params_flat(0, n) if func == "fletcher_powell" else None
    dev = torch.device("cuda")
    p, v = torch.from_numpy(P).to(dev), torch.from_numpy(V).to(dev)
    pr = None if params is None else torch.from_numpy(params).to(dev)
    if algo in ("hessian", "sym_hessian"):
        H = (chf.hessian_batch if algo == "hessian" else chf.sym_hessian_batch)(func, p, C, pr).cpu().numpy()
        ref = oracle.hessian_batch(func, P, C, params)
        scale = np.maximum(np.abs(ref).reshape(m, -1).max(axis=1), 1e-300)
        assert np.all(np.isfinite(H))
        assert (np.abs(H - ref).reshape(m, -1).max(axis=1) / scale).max() <= 1e-12, chf.path(func, n, C, algo)
        return
    fn = {"hvp": chf.hvp_batch, "sym_hvp": chf.sym_hvp_batch, "hvp_hoisted": chf.hvp_batch_hoisted,
          "hvp_seedsparse": chf.hvp_batch_seedsparse}[algo]
    got = fn(func, p, v, C, pr).cpu().numpy()
    ref, sabs = oracle.hvp_batch(func, P, V, C, params)
    err = oracle.componentwise_error(got, ref, sabs)
    assert np.all(np.isfinite(got))
    assert err.max() <= 1e-12, (chf.path(func, n, C, algo), float(err.max()))
