"""The vectorised closed forms used by the all-points GPU check (tests/closed_forms_np.py)
pinned against the oracle on CPU (and thereby the oracle at thousands of points against a
third, independent formulation): componentwise error <= 1e-12 with the closed form's own
sum_j |H_ij||v_j| as denominator, and that denominator against the oracle's."""
import numpy as np
import pytest

import oracle
import synth
from tests import closed_forms_np as cfn


@pytest.mark.parametrize("func", ["rosenbrock", "ackley", "fletcher_powell", "prodsum"])
@pytest.mark.parametrize("n", [2, 5, 16])
def test_closed_form_np_vs_oracle(func, n):
    m = 2000
    P, V = synth.points(4, n, m), synth.vectors(4, n, m)
    params = synth.fp_params_flat(4, n) if func == "fletcher_powell" else None
    ref, sabs = oracle.hvp_batch(func, P, V, 1, params)
    hv, S = cfn.hvp(func, P, V, params)
    assert cfn.error(ref, hv, S) <= 1e-12
    nz = sabs > 0
    assert np.array_equal(nz, S > 0)
    assert np.max(np.abs(S[nz] - sabs[nz]) / sabs[nz]) <= 1e-12


def test_closed_form_np_detects_wrong_result():
    """A perturbation at the 1e-9 level of one component is flagged (the check has teeth)."""
    n, m = 16, 500
    P, V = synth.points(5, n, m), synth.vectors(5, n, m)
    hv, S = cfn.rosenbrock(P, V)
    bad = hv.copy()
    bad[123, 7] += 1e-9 * max(abs(hv[123, 7]), S[123, 7])
    assert cfn.error(bad, hv, S) > 1e-12
