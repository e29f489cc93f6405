"""C4 (nl-meanvar on simulate_meanvar(34, 19, n=8192, seed=0), d = 2083) against
golden vectors of the UNMODIFIED reference (tests/golden/make_golden_c4.py).

* posterior value, gradient, Hessian (diagonal + 17 rows) and trace_single at two random points
  and two temperatures (posterior.py:392-542): rel_err (tests/conftest.py:170-174) <= 1e-12 / 1e-11;
* the reference-order cold Jacobi at d = 2083 on a seeded matrix: eigenvalues, sweeps and
  sha256(Psi) bit-identical (_jacobi.py:37-86);
* the chain start (metric.py:112-142 on the device's own Hessian): the basis-invariant parts
  -- sorted spectrum, logdet, H_before -- because the reference does not reproduce its own
  natural eigenvalue order at C4 (profiles/r2_c4_cold_reproducibility.md);
* two generalized leapfrogs from the reference's momentum (sampler.py:209-258) with the warm
  decompositions in the reference order: q, p and eigenvalues at 1e-9, fixed-point iteration
  and sweep counts equal, then h_after and the Metropolis decision of move 0.
"""

import hashlib

import numpy as np
import pytest

from golden_cases import load, rel_err
from paper_2511_06407_b200 import metric as M
from paper_2511_06407_b200 import rrgp
from paper_2511_06407_b200 import sampler as S
from paper_2511_06407_b200.posterior import PosteriorTarget

pytestmark = pytest.mark.gpu

D = 2083


def seeded_sym(seed, d=D):
    rng = np.random.default_rng(seed)
    r = rng.standard_normal((d, d))
    h = 0.02 * (0.5 * (r + r.T))
    base = np.repeat(10.0 * rng.standard_normal(d // 4 + 1), 4)[:d]
    h[np.diag_indices(d)] += base
    return h


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


_TARGET = {}


def c4_start_target():
    if "t" not in _TARGET:
        data, _ = rrgp.simulate_meanvar(34, 19, n=8192, seed=0)
        model = rrgp.build_model("nl-meanvar", data.x)
        _TARGET["t"] = PosteriorTarget(model, data)
    return _TARGET["t"]


@pytest.fixture(scope="module")
def c4():
    target = c4_start_target()
    assert target.dim == D
    return target


def test_c4_posterior_matches_reference(c4):
    g = load("c4_points")
    rows = g["hess_rows"]
    for k in (0, 1):
        st = c4.at_temperature(float(g[f"tau{k}"])).at(g[f"q{k}"])
        assert st.potential() == pytest.approx(float(g[f"pot{k}"]), rel=1e-12)
        assert rel_err(st.gradient(), g[f"grad{k}"]) < 1e-12
        h = st.hessian()
        assert rel_err(np.diagonal(h), g[f"hdiag{k}"]) < 1e-12
        assert rel_err(h[rows], g[f"hrows{k}"]) < 1e-12
        assert np.linalg.norm(h) == pytest.approx(float(g[f"hfro{k}"]), rel=1e-12)
        w = seeded_sym(int(g[f"wseed{k}"]))
        assert rel_err(st.trace_single(w), g[f"trace{k}"]) < 1e-11


def test_c4_cold_jacobi_bit_identical():
    g = load("c4_jacobi")
    h = seeded_sym(int(g["seed"]))
    lam, psi, sw = M.static_eigendecompose(h, 1e-13)
    assert sw == int(g["sweeps"])
    np.testing.assert_array_equal(lam, g["lam"])
    np.testing.assert_array_equal(psi[:, g["psi_col_idx"]], g["psi_cols"])
    assert sha(psi) == str(g["psi_sha"])


@pytest.fixture(scope="module")
def c4_start(c4):
    g = load("c4_chain")
    q0 = c4.initial_point()
    h0 = c4.at(q0).hessian()
    m0 = M.metric_from_hessian(h0, 1.0, 1e-13)
    return g, q0, h0, m0


def test_c4_chain_start_metric(c4_start):
    """Basis-invariant parity of the chain-start metric.  The natural (unsorted) order is not
    comparable at C4: the reference itself changes it with the OpenBLAS thread count
    (profiles/r2_c4_cold_reproducibility.md)."""
    g, q0, h0, m0 = c4_start
    assert np.linalg.norm(h0) == pytest.approx(float(g["h0_fro"]), rel=1e-12)
    assert abs(m0.sweep_count - int(g["cold_sweeps"])) <= 1
    assert rel_err(np.sort(m0.eigenvalues), np.sort(g["cold_lam"])) < 1e-12
    assert m0.logdet == pytest.approx(float(g["cold_logdet"]), rel=1e-12)
    # eigen-decomposition residual and orthonormality of the device basis
    psi, lam = m0.vectors, m0.eigenvalues
    hs = 0.5 * (h0 + h0.T)
    fro = np.linalg.norm(hs)
    assert np.linalg.norm(psi @ (lam[:, None] * psi.T) - hs) < 1e-11 * fro
    assert np.max(np.abs(psi.T @ psi - np.eye(D))) < 1e-11
    # H_before is basis-invariant (p^T G^-1 p = z^T z)
    p = psi @ (np.sqrt(m0.softabs_values) * g["z"])
    h_before = S.hamiltonian(q0, p, m0, c4_start_target())
    assert h_before == pytest.approx(float(g["h_before"]), rel=1e-12)


def test_c4_two_leapfrogs_from_reference_momentum(c4, c4_start):
    """Two generalized leapfrogs (reference pivot order in the warm decompositions) from the
    reference's own momentum: q, p and the spectrum at 1e-9, fixed-point counts equal, then
    H_after and the Metropolis decision of move 0."""
    g, q0, _, m0 = c4_start
    cfg = S.ChainConfig(epsilon=float(g["epsilon"]), leapfrogs=1, moves=1, burnin=0, warm_order="cyclic")
    q, p, m = q0, g["p0"], m0
    for k in (1, 2):
        q, p, m, diag = S.leapfrog_step(q, p, m, c4, cfg)
        assert rel_err(q, g[f"q{k}"]) < 1e-9, k
        assert rel_err(p, g[f"p{k}"]) < 1e-9, k
        assert rel_err(np.sort(m.eigenvalues), np.sort(g[f"lam{k}"])) < 1e-9, k
        assert m.logdet == pytest.approx(float(g[f"logdet{k}"]), rel=1e-12)
        assert [diag["fp_p_iters"]] == list(g[f"fp_p{k}"])
        assert [diag["fp_q_iters"]] == list(g[f"fp_q{k}"])
        assert len(diag["sweeps"]) == len(g[f"sweeps{k}"])
    h_after = S.hamiltonian(q, p, m, c4)
    assert h_after == pytest.approx(float(g["h_after"]), rel=1e-12)
    accept = (float(g["h_before"]) - h_after) > np.log(float(g["uniform"]))
    assert accept == bool(g["accept"])


def test_c4_refine_leapfrog_matches_reference(c4, c4_start):
    """The production warm solver (warm_order="refine": GEMM eigenvector refinement) meets
    the reference's convergence test, so the leapfrog from the reference momentum agrees with
    the reference's (cyclic Jacobi) leapfrog to the Jacobi tolerance."""
    g, q0, _, m0 = c4_start
    cfg = S.ChainConfig(epsilon=float(g["epsilon"]), leapfrogs=1, moves=1, burnin=0, warm_order="refine")
    q1, p1, m1, diag = S.leapfrog_step(q0, g["p0"], m0, c4, cfg)
    assert rel_err(q1, g["q1"]) < 1e-8
    assert rel_err(p1, g["p1"]) < 1e-8
    assert rel_err(np.sort(m1.eigenvalues), np.sort(g["lam1"])) < 1e-9
    assert [diag["fp_p_iters"]] == list(g["fp_p1"])
    assert [diag["fp_q_iters"]] == list(g["fp_q1"])
    assert all(0 < s <= 4 for s in diag["sweeps"])


def test_c4_divide_and_conquer_cold_matches_reference(c4_start):
    """cold_order="dc" on the real chain-start Hessian (north star (3)): the reference's cold
    spectrum (golden, its own Jacobi) to 1e-12, a 1e-12 decomposition residual, an orthonormal
    basis, and the reference's metric log-determinant and starting Hamiltonian (basis-invariant)."""
    g, q0, h0, _ = c4_start
    lam, psi = M.eigh_dc(h0)
    assert np.all(np.diff(lam) >= 0.0)
    assert rel_err(lam, np.sort(g["cold_lam"])) < 1e-12
    hs = 0.5 * (h0 + h0.T)
    fro = np.linalg.norm(hs)
    assert np.linalg.norm(psi @ (lam[:, None] * psi.T) - hs) < 1e-12 * fro
    assert np.max(np.abs(psi.T @ psi - np.eye(D))) < 1e-12
    m = M._state(lam, psi, 1.0, 0, 0)
    assert m.logdet == pytest.approx(float(g["cold_logdet"]), rel=1e-12)
    p = psi @ (np.sqrt(m.softabs_values) * g["z"])
    assert S.hamiltonian(q0, p, m, c4_start_target()) == pytest.approx(float(g["h_before"]), rel=1e-12)
