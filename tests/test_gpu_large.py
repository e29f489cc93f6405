"""Large-d path (DMMA GEMMs + host-driven leapfrog, d > 256) vs the CPU oracle.

d = 583 (nl-meanvar on 9 continuous + 19 binary covariates, N = 400) routes
through the same code as C4 (d = 2083) while the oracle still finishes in
seconds.  With the reference pivot order the large path must match the oracle
to the usual 1e-9; with the parallel order the first leapfrog agrees to the
Jacobi tolerance.
"""

import numpy as np
import pytest

import oracle
from golden_cases import rel_err

pytestmark = pytest.mark.gpu

from paper_2511_06407_b200 import metric as M  # noqa: E402
from paper_2511_06407_b200 import rrgp  # noqa: E402
from paper_2511_06407_b200 import sampler as S  # noqa: E402
from paper_2511_06407_b200.posterior import PosteriorTarget  # noqa: E402


@pytest.fixture(scope="module")
def large_case():
    data, _ = rrgp.simulate_meanvar(9, 19, n=400, seed=2)
    model = rrgp.build_model("nl-meanvar", data.x)
    target = PosteriorTarget(model, data)
    assert target.dim == 583
    return model, data, target, oracle.OTarget(model, data)


def test_large_posterior_matches_oracle(large_case):
    model, data, target, ot = large_case
    rng = np.random.default_rng(3)
    d = target.dim
    for tau in (1.0, 0.4):
        q = 0.03 * rng.standard_normal(d)
        st, op = target.at_temperature(tau).at(q), ot.at_temperature(tau).at(q)
        assert st.potential() == pytest.approx(op.potential(), rel=1e-12)
        assert rel_err(st.gradient(), op.gradient()) < 1e-12
        assert rel_err(st.hessian(), op.hessian()) < 1e-11
        w = rng.standard_normal((d, d))
        w = 0.5 * (w + w.T)
        assert rel_err(st.trace_single(w), op.trace(w)) < 1e-10


def test_large_chain_runs_and_starts_like_oracle(large_case):
    """At d = 583 the chain-start spectrum has a cluster with gaps ~1e-5 against
    ||H|| ~ 1e4, so eigenvectors inside it are fixed only to ~zeta ||H|| / gap by
    the reference's own tolerance and trajectories are not bitwise comparable;
    the Hamiltonian at the start (Psi-invariant) and the chain's health are."""
    model, data, target, ot = large_case
    cfg = S.ChainConfig(epsilon=0.002, leapfrogs=2, moves=3, burnin=0, seed=5, record_q=True,
                        warm_order="parallel")
    res = S.run_chain(target, cfg)
    ref = oracle.run_chain(ot, oracle.OConfig(epsilon=0.002, leapfrogs=2, moves=1, burnin=0, seed=5))
    assert res.records[0].h_before == pytest.approx(ref.records[0].h_before, rel=1e-12)
    assert all(np.isfinite(r.h_after) for r in res.records)
    assert res.accept_count >= 2


@pytest.fixture
def force_large(monkeypatch):
    monkeypatch.setenv("SGP_FORCE_LARGE", "1")
    yield


@pytest.mark.parametrize("name", ["chain_c1_eps1e-2", "chain_c1_eps15e-3", "chain_meanvar_tau",
                                  "chain_small_static"])
def test_large_path_reproduces_reference_golden_chains(force_large, name):
    """The GEMM/host-driven path, forced onto the well-conditioned golden chains."""
    from golden_cases import case
    g, model, data = case(name)
    target = PosteriorTarget(model, data, float(g["tau"]))
    cfg = S.ChainConfig(epsilon=float(g["epsilon"]), leapfrogs=int(g["leapfrogs"]), moves=int(g["moves"]),
                        burnin=0, seed=int(g["seed"]), metric=str(g["metric_mode"]), record_q=True,
                        warm_order="cyclic")
    res = S.run_chain(target, cfg)
    np.testing.assert_array_equal([r.accept for r in res.records], g["accept"])
    np.testing.assert_array_equal([r.divergent for r in res.records], g["divergent"])
    assert rel_err([r.h_before for r in res.records], g["h_before"]) < 1e-9
    assert rel_err(res.sample_matrix(), g["q"]) < 1e-9


def test_generic_cyclic_sweep_bit_exact(large_case):
    """d > 256 uses the unregistered (generic) warp sweep: still the reference's bits."""
    model, data, target, ot = large_case
    h = ot.at(0.02 * np.ones(target.dim)).hessian()
    lam, psi, sw = M.static_eigendecompose(h, 1e-13)
    lam_o, psi_o, sw_o = oracle.cold_eigh(h, 1e-13)
    assert sw == sw_o
    np.testing.assert_array_equal(lam, lam_o)
    np.testing.assert_array_equal(psi, psi_o)
    m0 = oracle.metric_cold(h, 1.0, 1e-13)
    h1 = ot.at(0.021 * np.ones(target.dim)).hessian()
    mw_o = oracle.metric_warm(h1, m0, 1e-13)
    prev = M.MetricState(eigenvalues=m0.lam, vectors=m0.psi, softabs_values=m0.g, logdet=m0.logdet,
                         kappa=1.0, sweep_count=m0.sweeps, steps_since_refresh=0)
    mw = M.dynamic_eigendecompose(h1, prev, 1e-13, order="cyclic")
    assert mw.sweep_count == mw_o.sweeps
    assert rel_err(mw.eigenvalues, mw_o.lam) < 1e-12
    # eigenvectors inside the near-degenerate cluster are tolerance-limited; G is not
    G = (mw.vectors * mw.softabs_values) @ mw.vectors.T
    G_o = (mw_o.psi * mw_o.g) @ mw_o.psi.T
    assert rel_err(G, G_o) < 1e-9


@pytest.mark.parametrize("order,gs", [("cyclic", 10), ("parallel", 10), ("refine", 10), ("parallel", 1),
                                      ("refine", 1)])
def test_large_leapfrog_step_vs_oracle(large_case, order, gs):
    """gs = 1 re-orthonormalises before every warm decomposition: the MGS steps in the cyclic
    order, the Cholesky-QR correction (two GEMMs) in the others."""
    model, data, target, ot = large_case
    d = target.dim
    q0 = np.zeros(d)
    om0 = oracle.metric_cold(ot.at(q0).hessian(), 1.0, 1e-13)
    m0 = M.MetricState(eigenvalues=om0.lam, vectors=om0.psi, softabs_values=om0.g, logdet=om0.logdet,
                       kappa=1.0, sweep_count=om0.sweeps, steps_since_refresh=0)
    p = om0.psi @ (np.sqrt(om0.g) * np.random.default_rng(9).standard_normal(d))
    cfg = S.ChainConfig(epsilon=0.002, leapfrogs=1, moves=1, burnin=0, warm_order=order, gs_interval=gs)
    q1, p1, mt, diag = S.leapfrog_step(q0, p, m0, target, cfg)
    oq, op_, om, odiag = oracle.leapfrog_step(q0, p, om0, ot, oracle.OConfig(epsilon=0.002, leapfrogs=1,
                                                                             moves=1, burnin=0, gs_interval=gs))
    tol = 1e-9 if order == "cyclic" else 1e-6
    assert rel_err(q1, oq) < tol
    assert rel_err(p1, op_) < tol
    assert rel_err(mt.eigenvalues, om.lam) < tol
    assert diag["fp_p_iters"] == odiag["fp_p_iters"]
    assert diag["fp_q_iters"] == odiag["fp_q_iters"]


def test_block_jacobi_cold_decomposition(large_case):
    """Chain-start cold decomposition on the large path (block Jacobi: pair solves on a
    high-priority stream, eigenvector updates overlapped on the caller's stream) against
    LAPACK: same spectrum, orthonormal basis, and Psi diag(lambda) Psi^T = sym(H) to the
    reference's convergence tolerance (off-norm <= zeta ||H||_F, metric.py:101-109)."""
    from paper_2511_06407_b200 import _native as nat

    model, data, target, _ = large_case
    d = target.dim
    q = np.zeros((1, d))
    h = target.device.eval(1.0, q, nat.EVAL_HESSIAN)["hess"][0]
    hs = 0.5 * (h + h.T)
    cfg = S.ChainConfig(epsilon=0.002, leapfrogs=1, moves=1, burnin=0, warm_order="parallel")
    ch = S.DeviceChains(target.device, np.ones(1), cfg)
    ch.set_q(q)
    ch.init()
    assert ch.status_host()[0] == 0
    lam = ch.lam.cpu().numpy()[0]
    psi = ch.psi.cpu().numpy()[0]
    ref = np.linalg.eigvalsh(hs)
    fro = np.linalg.norm(hs)
    assert np.max(np.abs(np.sort(lam) - ref)) < 1e-11 * fro
    assert np.max(np.abs(psi.T @ psi - np.eye(d))) < 1e-11
    assert np.linalg.norm(psi @ np.diag(lam) @ psi.T - hs) < 1e-11 * fro


def test_dc_cold_decomposition(large_case):
    """cold_order="dc": the chain-start decomposition by Householder tridiagonalisation + divide
    and conquer (sgp_dc.cuh) against LAPACK, as the block-Jacobi test above; eigenvalues come
    out ascending."""
    from paper_2511_06407_b200 import _native as nat

    model, data, target, _ = large_case
    d = target.dim
    q = np.zeros((1, d))
    h = target.device.eval(1.0, q, nat.EVAL_HESSIAN)["hess"][0]
    hs = 0.5 * (h + h.T)
    cfg = S.ChainConfig(epsilon=0.002, leapfrogs=1, moves=1, burnin=0, warm_order="refine", cold_order="dc")
    ch = S.DeviceChains(target.device, np.ones(1), cfg)
    ch.set_q(q)
    ch.init()
    assert ch.status_host()[0] == 0
    lam = ch.lam.cpu().numpy()[0]
    psi = ch.psi.cpu().numpy()[0]
    ref = np.linalg.eigvalsh(hs)
    fro = np.linalg.norm(hs)
    assert np.all(np.diff(lam) >= 0.0)
    assert np.max(np.abs(lam - ref)) < 1e-12 * fro
    assert np.max(np.abs(psi.T @ psi - np.eye(d))) < 1e-12
    assert np.linalg.norm(psi @ np.diag(lam) @ psi.T - hs) < 1e-12 * fro


def test_large_chain_with_dc_cold_starts_like_oracle(large_case):
    """A chain whose cold decompositions (start, rejections) use the divide and conquer: the
    starting Hamiltonian is Psi-invariant, so it equals the reference algorithm's."""
    model, data, target, ot = large_case
    cfg = S.ChainConfig(epsilon=0.002, leapfrogs=2, moves=3, burnin=0, seed=5, record_q=True,
                        warm_order="refine", cold_order="dc")
    res = S.run_chain(target, cfg)
    ref = oracle.run_chain(ot, oracle.OConfig(epsilon=0.002, leapfrogs=2, moves=1, burnin=0, seed=5))
    assert res.records[0].h_before == pytest.approx(ref.records[0].h_before, rel=1e-10)
    assert all(np.isfinite(r.h_after) for r in res.records)
    assert res.accept_count >= 2


@pytest.mark.parametrize("fallback", ["dc", "jacobi"])
def test_refine_hand_over_vs_oracle(large_case, monkeypatch, fallback):
    """The refinement hands a warm call over when it stops converging (here forced after one
    iteration): to the divide and conquer (default) or the block Jacobi.  The leapfrog still
    follows the reference algorithm to the Jacobi tolerance."""
    monkeypatch.setenv("SGP_REFINE_MAX_ITERS", "1")
    monkeypatch.setenv("SGP_REFINE_FALLBACK", fallback)
    model, data, target, ot = large_case
    d = target.dim
    q0 = np.zeros(d)
    om0 = oracle.metric_cold(ot.at(q0).hessian(), 1.0, 1e-13)
    m0 = M.MetricState(eigenvalues=om0.lam, vectors=om0.psi, softabs_values=om0.g, logdet=om0.logdet,
                       kappa=1.0, sweep_count=om0.sweeps, steps_since_refresh=0)
    p = om0.psi @ (np.sqrt(om0.g) * np.random.default_rng(9).standard_normal(d))
    cfg = S.ChainConfig(epsilon=0.002, leapfrogs=1, moves=1, burnin=0, warm_order="refine")
    q1, p1, mt, diag = S.leapfrog_step(q0, p, m0, target, cfg)
    oq, op_, om, odiag = oracle.leapfrog_step(q0, p, om0, ot, oracle.OConfig(epsilon=0.002, leapfrogs=1,
                                                                             moves=1, burnin=0))
    assert rel_err(q1, oq) < 1e-6
    assert rel_err(p1, op_) < 1e-6
    assert rel_err(np.sort(mt.eigenvalues), np.sort(om.lam)) < 1e-6
    assert diag["fp_p_iters"] == odiag["fp_p_iters"]
    assert diag["fp_q_iters"] == odiag["fp_q_iters"]
