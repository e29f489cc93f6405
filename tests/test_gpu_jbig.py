"""Grid-wide reference-order Jacobi (csrc/sgp_jbig.cuh) vs the CPU restatement of
_jacobi.jacobi_sweeps (oracle/jacobi.c): eigenvalues, eigenvectors and sweep counts must be
bit-identical.  SGP_JBIG_MIN_D=2 routes every size through it, so window edge cases
(d below, at and just above multiples of the 32-pivot window, one- and two-window passes)
are covered at sizes the oracle finishes in well under a second.
"""

import numpy as np
import pytest

import oracle
from paper_2511_06407_b200 import metric as M

pytestmark = pytest.mark.gpu


def seeded_sym(seed, d, offdiag=0.02):
    """Same generator as tests/golden/make_golden_c4.py (exactly repeated diagonal blocks)."""
    rng = np.random.default_rng(seed)
    r = rng.standard_normal((d, d))
    h = offdiag * (0.5 * (r + r.T))
    base = np.repeat(10.0 * rng.standard_normal(d // 4 + 1), 4)[:d]
    h[np.diag_indices(d)] += base
    return h


@pytest.fixture
def jbig_all(monkeypatch):
    monkeypatch.setenv("SGP_JBIG_MIN_D", "2")
    yield


@pytest.mark.parametrize("d", [2, 3, 31, 32, 33, 34, 63, 64, 65, 97, 100, 130, 161, 200])
def test_jbig_cold_bit_exact(jbig_all, d):
    for seed, off in ((d, 0.02), (d + 1000, 1.0)):
        h = seeded_sym(seed, d, off)
        lam, psi, sw = M.static_eigendecompose(h, 1e-13)
        lam_o, psi_o, sw_o = oracle.cold_eigh(h, 1e-13)
        assert sw == sw_o
        np.testing.assert_array_equal(lam, lam_o)
        np.testing.assert_array_equal(psi, psi_o)


def test_jbig_cold_bit_exact_on_posterior_hessian(jbig_all):
    """A chain-start Hessian (exactly repeated eigenvalues)."""
    from paper_2511_06407_b200 import rrgp

    data, _ = rrgp.simulate_meanvar(2, 3, n=200, seed=4)
    model = rrgp.build_model("nl-meanvar", data.x)
    ot = oracle.OTarget(model, data)
    h = ot.at(np.zeros(ot.dim)).hessian()
    lam, psi, sw = M.static_eigendecompose(h, 1e-13)
    lam_o, psi_o, sw_o = oracle.cold_eigh(h, 1e-13)
    assert sw == sw_o
    np.testing.assert_array_equal(lam, lam_o)
    np.testing.assert_array_equal(psi, psi_o)


def test_jbig_sweep_cap(jbig_all):
    h = seeded_sym(5, 70, 1.0)
    with pytest.raises(M.JacobiError):
        M.static_eigendecompose(h, 1e-13, 1)
