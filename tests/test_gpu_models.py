"""CUDA path vs the CPU oracle on the SURVEY.md 8(d) model shapes.

C3a: logistic with Gaussian kernels on 2 continuous + linear on 19 binary
covariates (d = 83); C5: the four competing mean/variance models l-mean
(d = 26), nl-mean (84), l-meanvar (47), nl-meanvar (163, also C3b).  Most cases
use N = 300 so the oracle finishes in seconds; test_full_size_config_chain_matches_oracle
runs every model at the configs' N = 2000 and step sizes.
"""

import numpy as np
import pytest

import oracle
from golden_cases import rel_err

pytestmark = pytest.mark.gpu

from paper_2511_06407_b200 import rrgp  # noqa: E402
from paper_2511_06407_b200 import sampler as S  # noqa: E402
from paper_2511_06407_b200.posterior import PosteriorTarget  # noqa: E402

N_ROWS = 300


def nmes_data(n=N_ROWS, seed=0):
    data, _ = rrgp.simulate_meanvar(2, 19, n=n, seed=seed)
    return data


def logistic_nmes(n=N_ROWS, seed=0):
    data = nmes_data(n, seed)
    y = np.where(data.y > np.median(data.y), 1.0, -1.0)
    return rrgp.Dataset(data.x, y)


CASES = {
    "c3a-logistic": (lambda: logistic_nmes(), "logistic", 83),
    "c5-l-mean": (lambda: nmes_data(), "l-mean", 26),
    "c5-nl-mean": (lambda: nmes_data(), "nl-mean", 84),
    "c5-l-meanvar": (lambda: nmes_data(), "l-meanvar", 47),
    "c5-nl-meanvar": (lambda: nmes_data(), "nl-meanvar", 163),
}


@pytest.fixture(scope="module", params=sorted(CASES))
def model_case(request):
    make, name, d = CASES[request.param]
    data = make()
    model = rrgp.build_model(name, data.x)
    target = PosteriorTarget(model, data)
    assert target.dim == d
    return request.param, model, data, target


def test_posterior_matches_oracle(model_case):
    name, model, data, target = model_case
    ot = oracle.OTarget(model, data)
    rng = np.random.default_rng(7)
    d = target.dim
    for tau in (1.0, 0.3):
        q = 0.05 * rng.standard_normal(d)
        st, op = target.at_temperature(tau).at(q), ot.at_temperature(tau).at(q)
        assert st.potential() == pytest.approx(op.potential(), rel=1e-12)
        assert rel_err(st.gradient(), op.gradient()) < 1e-12
        assert rel_err(st.hessian(), op.hessian()) < 1e-12
        w = rng.standard_normal((d, d))
        w = 0.5 * (w + w.T)
        assert rel_err(st.trace_single(w), op.trace(w)) < 1e-11


def test_cold_eigh_bit_exact(model_case):
    from paper_2511_06407_b200 import metric as M
    name, model, data, target = model_case
    h = oracle.OTarget(model, data).at(0.05 * np.ones(target.dim)).hessian()
    lam, psi, sw = M.static_eigendecompose(h, 1e-13)
    lam_o, psi_o, sw_o = oracle.cold_eigh(h, 1e-13)
    assert sw == sw_o
    np.testing.assert_array_equal(lam, lam_o)
    np.testing.assert_array_equal(psi, psi_o)


@pytest.mark.parametrize("path", ["auto", "latency"])
def test_short_chain_matches_oracle(model_case, path):
    """One CTA per chain (auto) and the whole-GPU latency path both reproduce the reference
    algorithm's chain (reference pivot order)."""
    name, model, data, target = model_case
    eps = 0.002
    cfg = S.ChainConfig(epsilon=eps, leapfrogs=4, moves=5, burnin=0, seed=11, record_q=True, path=path)
    try:
        ref = oracle.run_chain(oracle.OTarget(model, data),
                               oracle.OConfig(epsilon=eps, leapfrogs=4, moves=5, burnin=0, seed=11,
                                              record_q=True))
    except oracle.OChainError:
        with pytest.raises(S.ChainError):
            S.run_chain(target, cfg)
        return
    res = S.run_chain(target, cfg)
    assert [r.accept for r in res.records] == [r.accept for r in ref.records]
    assert [r.divergent for r in res.records] == [r.divergent for r in ref.records]
    hb = np.array([r.h_before for r in res.records])
    assert rel_err(hb, [r.h_before for r in ref.records]) < 1e-9
    assert rel_err(res.sample_matrix(), np.vstack([r.q for r in ref.records])) < 1e-9
    assert [r.sweeps_mean for r in res.records] == pytest.approx([r.sweeps_mean for r in ref.records])


def test_batched_mixed_temperatures(model_case):
    """A batch whose chains sit at different tau equals per-tau single runs."""
    name, model, data, target = model_case
    cfg = S.ChainConfig(epsilon=0.005, leapfrogs=3, moves=3, burnin=0, record_q=True)
    taus = [1.0, 0.5, 0.0]
    batch = S.run_chains(target, cfg, [21, 22, 23], taus=taus)
    for seed, tau, rb in zip([21, 22, 23], taus, batch):
        single = S.run_chain(target.at_temperature(tau), S.ChainConfig(
            epsilon=0.005, leapfrogs=3, moves=3, burnin=0, record_q=True, seed=seed))
        np.testing.assert_array_equal(rb.sample_matrix(), single.sample_matrix())


def test_first_move_divergence_matches_oracle():
    """Both implementations reject an unusable epsilon the same way (sampler.py:388-391)."""
    data = logistic_nmes()
    model = rrgp.build_model("logistic", data.x)
    target = PosteriorTarget(model, data)
    with pytest.raises(oracle.OChainError):
        oracle.run_chain(oracle.OTarget(model, data),
                         oracle.OConfig(epsilon=0.01, leapfrogs=4, moves=5, burnin=0, seed=11))
    with pytest.raises(S.ChainError):
        S.run_chain(target, S.ChainConfig(epsilon=0.01, leapfrogs=4, moves=5, burnin=0, seed=11))


# Full-size configurations (BASELINE.json C3a / C5): N = 2000 rows and the configs' step sizes
# (1e-4; 8e-5 for nl-meanvar), 8 moves of 10 leapfrogs in the reference pivot order.
FULL = {
    "c3a-logistic": ("logistic", 83, 1e-4),
    "c5-l-mean": ("l-mean", 26, 1e-4),
    "c5-nl-mean": ("nl-mean", 84, 1e-4),
    "c5-l-meanvar": ("l-meanvar", 47, 1e-4),
    "c5-nl-meanvar": ("nl-meanvar", 163, 8e-5),
}


@pytest.mark.parametrize("key", sorted(FULL))
def test_full_size_config_chain_matches_oracle(key):
    name, d, eps = FULL[key]
    data = logistic_nmes(n=2000) if name == "logistic" else nmes_data(n=2000)
    model = rrgp.build_model(name, data.x)
    target = PosteriorTarget(model, data)
    assert target.dim == d
    ocfg = oracle.OConfig(epsilon=eps, leapfrogs=10, moves=8, burnin=0, seed=23, record_q=True)
    ref = oracle.run_chain(oracle.OTarget(model, data), ocfg)
    res = S.run_chain(target, S.ChainConfig(epsilon=eps, leapfrogs=10, moves=8, burnin=0, seed=23,
                                            record_q=True))
    assert [r.accept for r in res.records] == [r.accept for r in ref.records]
    assert rel_err([r.h_before for r in res.records], [r.h_before for r in ref.records]) < 1e-9
    assert rel_err([r.h_after for r in res.records], [r.h_after for r in ref.records]) < 1e-9
    assert rel_err(res.sample_matrix(), np.vstack([r.q for r in ref.records])) < 1e-9
    assert [r.sweeps_mean for r in res.records] == pytest.approx([r.sweeps_mean for r in ref.records])
