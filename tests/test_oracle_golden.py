"""Pin the CPU oracle to the reference's own outputs (tests/golden/*.npz).

The oracle (oracle/) is the checker for the CUDA path, so it must first agree
with the unmodified reference: bitwise for the Jacobi eigensolver on identical
input, and to ~1e-12 for BLAS-dependent quantities.
"""

import hashlib

import numpy as np
import pytest

import oracle
from golden_cases import CHAIN_CASES, POINT_CASES, case, load, rel_err
from paper_2511_06407_b200 import rrgp


@pytest.mark.parametrize("name", POINT_CASES)
def test_posterior_quantities(name):
    g, model, data = case(name)
    target = oracle.OTarget(model, data)
    assert target.dim == int(g["dim"])
    for k in range(4):
        pt = target.at_temperature(float(g[f"tau{k}"])).at(g[f"q{k}"])
        assert pt.potential() == pytest.approx(float(g[f"pot{k}"]), rel=1e-13, abs=1e-12)
        assert rel_err(pt.gradient(), g[f"grad{k}"]) < 1e-13
        assert rel_err(pt.hessian(), g[f"hess{k}"]) < 1e-13
        assert rel_err(pt.trace(g[f"wt{k}"]), g[f"trace{k}"]) < 1e-12
        assert pt.sum_potentials() == pytest.approx(float(g[f"sumpot{k}"]), rel=1e-13)


@pytest.mark.parametrize("name", POINT_CASES)
def test_metric_quantities(name):
    g, model, data = case(name)
    target = oracle.OTarget(model, data).at_temperature(float(g["tau0"]))
    h0 = target.at(g["q0"]).hessian()
    # bit-exact cold Jacobi when fed the reference's own Hessian
    lam, psi, sweeps = oracle.cold_eigh(g["hess0"], 1e-13)
    assert sweeps == int(g["cold_sweeps"])
    np.testing.assert_array_equal(lam, g["cold_lam"])
    np.testing.assert_array_equal(psi, g["cold_psi"])
    # and within rounding when fed the oracle's Hessian
    lam2, psi2, _ = oracle.cold_eigh(h0, 1e-13)
    assert rel_err(lam2, g["cold_lam"]) < 1e-12
    m0 = oracle.metric_cold(g["hess0"], 1.0, 1e-13)
    m1 = oracle.metric_warm(g["hess1"], m0, 1e-13)
    assert m1.sweeps == int(g["warm_sweeps"]) and m1.since == int(g["warm_since"])
    assert rel_err(m1.lam, g["warm_lam"]) < 1e-13
    assert rel_err(m1.psi, g["warm_psi"]) < 1e-12
    import dataclasses
    m1b = oracle.metric_warm(g["hess1"], dataclasses.replace(m0, since=9), 1e-13)
    assert m1b.since == int(g["warmgs_since"]) == 0
    assert rel_err(m1b.psi, g["warmgs_psi"]) < 1e-12
    p, v, z = g["p"], g["v"], g["z"]
    assert rel_err(oracle.t_matrix(m0.lam, 1.0), g["t_matrix"]) < 1e-15
    assert rel_err(oracle.w1(m0, p), g["w1"]) < 1e-13
    assert rel_err(oracle.w2(m0), g["w2"]) < 1e-14
    assert rel_err(oracle.ginv(m0, v), g["ginv"]) < 1e-13
    assert oracle.quad(m0, p) == pytest.approx(float(g["quad"]), rel=1e-13)
    assert m0.logdet == pytest.approx(float(g["logdet"]), rel=1e-14)
    assert rel_err(oracle.momentum(m0, z), g["momentum"]) < 1e-14
    fr = oracle.OFrame(target.at(g["q0"]), m0, oracle.w2(m0))
    assert oracle.frame_h(fr, p) == pytest.approx(float(g["ham"]), rel=1e-13)


@pytest.mark.parametrize("name", POINT_CASES)
def test_leapfrog_step(name):
    g, model, data = case(name)
    target = oracle.OTarget(model, data).at_temperature(float(g["tau0"]))
    m0 = oracle.metric_cold(target.at(g["q0"]).hessian(), 1.0, 1e-13)
    for tag, eps in (("lf", 0.01), ("lfs", 0.002)):
        cfg = oracle.OConfig(epsilon=eps, leapfrogs=1, moves=1, burnin=0)
        q1, p1, mt1, diag = oracle.leapfrog_step(g["q0"], 0.3 * g["p"], m0, target, cfg)
        assert rel_err(q1, g[f"{tag}_q"]) < 1e-12
        assert rel_err(p1, g[f"{tag}_p"]) < 1e-10
        assert rel_err(mt1.lam, g[f"{tag}_lam"]) < 1e-11
        assert diag["fp_p_iters"] == list(g[f"{tag}_fp_p"])
        assert diag["fp_q_iters"] == list(g[f"{tag}_fp_q"])
        assert diag["sweeps"] == list(g[f"{tag}_sweeps"])


def _chain_cfg(g):
    return oracle.OConfig(epsilon=float(g["epsilon"]), leapfrogs=int(g["leapfrogs"]),
                          moves=int(g["moves"]), burnin=0, seed=int(g["seed"]),
                          metric=str(g["metric_mode"]), record_q=True)


@pytest.mark.parametrize("name", CHAIN_CASES)
def test_chain_records(name):
    g, model, data = case(name)
    target = oracle.OTarget(model, data, float(g["tau"]))
    res = oracle.run_chain(target, _chain_cfg(g))
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
    np.testing.assert_array_equal([r.uniform for r in res.records], g["uniform"])
    q = np.vstack([r.q for r in res.records])
    assert rel_err(q, g["q"]) < 1e-9
    sw = np.array([r.sweeps_mean for r in res.records])
    np.testing.assert_allclose(sw, g["sweeps_mean"], atol=1e-12)


def test_thermo_integrate_small():
    g, model, data = case("ti_small")
    target = oracle.OTarget(model, data)
    cfg = oracle.OConfig(epsilon=0.02, leapfrogs=5, moves=10, burnin=0, seed=123)
    per_chain, rungs, _ = oracle.thermo_integrate(
        target, g["taus"], 3, 5, 3, cfg, warmup_segment_moves=10, warmup_max_segments=2,
        spread_moves=2)
    assert rel_err(rungs, g["rung_values"]) < 1e-9
    assert rel_err(per_chain, g["per_chain"]) < 1e-9


def test_rank_sum():
    g = load("ranksum")
    for i in range(3):
        z, p = oracle.rank_sum_test(g[f"a{i}"], g[f"b{i}"])
        assert z == pytest.approx(float(g["z"][i]), rel=1e-14, abs=1e-15)
        assert p == pytest.approx(float(g["p"][i]), rel=1e-14, abs=1e-15)


@pytest.mark.parametrize("tag,gen", [
    ("c1", lambda: rrgp.simulate_logistic(1, n=500, seed=0)),
    ("c2", lambda: rrgp.simulate_logistic(1, n=512, seed=0)),
    ("c1d4", lambda: rrgp.simulate_logistic(4, n=500, seed=0)),
    ("c3", lambda: rrgp.simulate_meanvar(2, 19, n=2000, seed=0)),
    ("c4", lambda: rrgp.simulate_meanvar(34, 19, n=8192, seed=0)),
])
def test_generators_bit_identical(tag, gen):
    """The product's simulators reproduce the reference datasets bit for bit."""
    g = load("generators")
    ds, _ = gen()
    assert hashlib.sha256(ds.x.tobytes()).hexdigest() == str(g[f"{tag}_x"])
    assert hashlib.sha256(ds.y.tobytes()).hexdigest() == str(g[f"{tag}_y"])
