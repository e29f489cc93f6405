"""CUDA path vs the reference's golden vectors and the CPU oracle (B200 only).

Tolerances follow SURVEY.md 8(c): 1e-9 relative (rel_err convention of the
reference's tests/conftest.py:170-174) on Hessian, eigenvalues, Hamiltonians
and positions; identical accept/reject and divergence flags per move.
"""

import dataclasses

import numpy as np
import pytest

import oracle
from golden_cases import CHAIN_CASES, POINT_CASES, case, rel_err

pytestmark = pytest.mark.gpu

from paper_2511_06407_b200 import metric as M  # noqa: E402
from paper_2511_06407_b200 import sampler as S  # noqa: E402
from paper_2511_06407_b200.posterior import PosteriorTarget  # noqa: E402


@pytest.fixture(scope="module")
def targets():
    cache = {}

    def get(name):
        if name not in cache:
            g, model, data = case(name)
            cache[name] = (g, model, data, PosteriorTarget(model, data))
        return cache[name]
    return get


@pytest.mark.parametrize("name", POINT_CASES)
def test_posterior_vs_golden(name, targets):
    g, model, data, target = targets(name)
    assert target.dim == int(g["dim"])
    for k in range(4):
        st = target.at_temperature(float(g[f"tau{k}"])).at(g[f"q{k}"])
        assert st.potential() == pytest.approx(float(g[f"pot{k}"]), rel=1e-12, abs=1e-12)
        assert rel_err(st.gradient(), g[f"grad{k}"]) < 1e-12
        h = st.hessian()
        assert rel_err(h, g[f"hess{k}"]) < 1e-12
        assert np.array_equal(h, h.T)
        assert rel_err(st.trace_single(g[f"wt{k}"]), g[f"trace{k}"]) < 1e-11
        assert st.sum_potentials() == pytest.approx(float(g[f"sumpot{k}"]), rel=1e-12)


@pytest.mark.parametrize("name", POINT_CASES)
def test_cold_jacobi_bit_exact(name, targets):
    g, *_ = targets(name)
    lam, psi, sweeps = M.static_eigendecompose(g["hess0"], 1e-13)
    assert sweeps == int(g["cold_sweeps"])
    np.testing.assert_array_equal(lam, g["cold_lam"])
    np.testing.assert_array_equal(psi, g["cold_psi"])


@pytest.mark.parametrize("order", ["cyclic", "parallel"])
@pytest.mark.parametrize("name", POINT_CASES)
def test_warm_jacobi(name, order, targets):
    g, *_ = targets(name)
    m0 = M.metric_from_hessian(g["hess0"], 1.0, 1e-13)
    m1 = M.dynamic_eigendecompose(g["hess1"], m0, 1e-13, order=order)
    assert rel_err(m1.eigenvalues, g["warm_lam"]) < 1e-9
    # G is basis invariant: compare Psi diag(g) Psi^T
    G = (m1.vectors * m1.softabs_values) @ m1.vectors.T
    g_ref = np.sqrt(1.0 + g["warm_lam"] ** 2)
    G_ref = (g["warm_psi"] * g_ref) @ g["warm_psi"].T
    assert rel_err(G, G_ref) < 1e-9
    assert m1.steps_since_refresh == int(g["warm_since"])
    if order == "cyclic":
        assert m1.sweep_count == int(g["warm_sweeps"])
        assert rel_err(m1.vectors, g["warm_psi"]) < 1e-9
    mgs = M.dynamic_eigendecompose(g["hess1"], dataclasses.replace(m0, steps_since_refresh=9), 1e-13,
                                   order=order)
    assert mgs.steps_since_refresh == 0
    assert rel_err(mgs.eigenvalues, g["warmgs_lam"]) < 1e-9


@pytest.mark.parametrize("name", POINT_CASES)
def test_metric_algebra(name, targets):
    g, model, data, target = targets(name)
    m0 = M.metric_from_hessian(g["hess0"], 1.0, 1e-13)
    p, v, z = g["p"], g["v"], g["z"]
    assert rel_err(M.t_matrix(m0.eigenvalues, 1.0), g["t_matrix"]) < 1e-14
    assert rel_err(M.w1_matrix(m0, p), g["w1"]) < 1e-12
    assert rel_err(M.w2_matrix(m0), g["w2"]) < 1e-12
    assert rel_err(M.metric_apply_inverse(m0, v), g["ginv"]) < 1e-12
    assert M.metric_quadratic(m0, p) == pytest.approx(float(g["quad"]), rel=1e-12)
    assert m0.logdet == pytest.approx(float(g["logdet"]), rel=1e-13)

    class Z:
        def standard_normal(self, n):
            return z
    assert rel_err(M.sample_momentum(m0, Z()), g["momentum"]) < 1e-13
    t0 = target.at_temperature(float(g["tau0"]))
    assert S.hamiltonian(g["q0"], p, m0, t0) == pytest.approx(float(g["ham"]), rel=1e-12)
    assert rel_err(S.grad_q_hamiltonian(g["q0"], p, m0, t0), g["gradq"]) < 1e-10


@pytest.mark.parametrize("order", ["cyclic", "parallel"])
@pytest.mark.parametrize("name", POINT_CASES)
def test_leapfrog_step(name, order, targets):
    g, model, data, target = targets(name)
    t0 = target.at_temperature(float(g["tau0"]))
    m0 = M.metric_from_hessian(g["hess0"], 1.0, 1e-13)
    for tag, eps in (("lf", 0.01), ("lfs", 0.002)):
        cfg = S.ChainConfig(epsilon=eps, leapfrogs=1, moves=1, burnin=0, warm_order=order)
        q1, p1, mt1, diag = S.leapfrog_step(g["q0"], 0.3 * g["p"], m0, t0, cfg)
        assert rel_err(q1, g[f"{tag}_q"]) < 1e-9
        assert rel_err(p1, g[f"{tag}_p"]) < 1e-9
        assert rel_err(mt1.eigenvalues, g[f"{tag}_lam"]) < 1e-9
        assert diag["fp_p_iters"] == list(g[f"{tag}_fp_p"])
        assert diag["fp_q_iters"] == list(g[f"{tag}_fp_q"])
        if order == "cyclic":
            assert diag["sweeps"] == list(g[f"{tag}_sweeps"])


def _chain_cfg(g, order):
    return S.ChainConfig(epsilon=float(g["epsilon"]), leapfrogs=int(g["leapfrogs"]),
                         moves=int(g["moves"]), burnin=0, seed=int(g["seed"]),
                         metric=str(g["metric_mode"]), record_q=True, warm_order=order)


@pytest.mark.parametrize("order", ["cyclic", "parallel"])
@pytest.mark.parametrize("name", CHAIN_CASES)
def test_chain_matches_reference(name, order, targets):
    g, model, data, _ = targets(name)
    target = PosteriorTarget(model, data, float(g["tau"]))
    res = S.run_chain(target, _chain_cfg(g, order))
    acc = np.array([r.accept for r in res.records])
    div = np.array([r.divergent for r in res.records])
    np.testing.assert_array_equal(acc, g["accept"])
    np.testing.assert_array_equal(div, g["divergent"])
    hb = np.array([r.h_before for r in res.records])
    ha = np.array([np.nan if r.h_after is None else r.h_after for r in res.records])
    assert rel_err(hb, g["h_before"]) < 1e-9
    ok = ~np.isnan(g["h_after"])
    np.testing.assert_array_equal(np.isnan(ha), ~ok)
    assert rel_err(ha[ok], g["h_after"][ok]) < 1e-9
    assert rel_err(res.sample_matrix(), g["q"]) < 1e-9
    assert rel_err(res.logpost, g["logpost"]) < 1e-9
    if order == "cyclic":
        np.testing.assert_allclose([r.sweeps_mean for r in res.records], g["sweeps_mean"], atol=1e-12)


def test_batched_chains_equal_single_runs(targets):
    g, model, data, target = targets("chain_c1_eps1e-2")
    cfg = S.ChainConfig(epsilon=0.01, leapfrogs=10, moves=8, burnin=0, record_q=True)
    seeds = [11, 12, 13, 14, 15]
    batch = S.run_chains(target, cfg, seeds)
    for seed, rb in zip(seeds, batch):
        rs = S.run_chain(target, dataclasses.replace(cfg, seed=seed))
        np.testing.assert_array_equal(rb.sample_matrix(), rs.sample_matrix())
        np.testing.assert_array_equal([r.h_before for r in rb.records], [r.h_before for r in rs.records])


def test_determinism(targets):
    g, model, data, target = targets("chain_c1_eps1e-2")
    cfg = S.ChainConfig(epsilon=0.01, leapfrogs=10, moves=6, burnin=0, seed=3, record_q=True)
    a, b = S.run_chain(target, cfg), S.run_chain(target, cfg)
    for ra, rb in zip(a.records, b.records):
        assert (ra.logpost, ra.h_before, ra.h_after, ra.accept) == (rb.logpost, rb.h_before, rb.h_after,
                                                                     rb.accept)


def test_oracle_agrees_on_fresh_chain(targets):
    """A chain not in the golden set: GPU vs CPU oracle on the same seed."""
    g, model, data, target = targets("meanvar_toy")
    cfg = S.ChainConfig(epsilon=0.02, leapfrogs=8, moves=15, burnin=0, seed=77, record_q=True)
    res = S.run_chain(target, cfg)
    ref = oracle.run_chain(oracle.OTarget(model, data),
                           oracle.OConfig(epsilon=0.02, leapfrogs=8, moves=15, burnin=0, seed=77,
                                          record_q=True))
    assert [r.accept for r in res.records] == [r.accept for r in ref.records]
    assert rel_err(res.sample_matrix(), np.vstack([r.q for r in ref.records])) < 1e-9


def test_rotation_fast_paths_bit_exact():
    """The Jacobi's branch-free fp64 div/sqrt/rcp replicas (sgp_core.cuh) equal
    the library's correctly rounded results bit for bit wherever they report
    success, on 2^24 Jacobi-like operand triples and raw bit patterns."""
    import ctypes

    from paper_2511_06407_b200 import _native as nat

    counts = (ctypes.c_longlong * 4)()
    nat.check(nat.lib().sgp_debug_rotation_check(1 << 24, 2024, counts), "rotation check")
    bad, slow, badop, n = list(counts)
    assert n == 1 << 24
    assert bad == 0 and badop == 0
    assert slow < n // 100  # the library path is the exception
