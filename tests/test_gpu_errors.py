"""The reference's error paths on the device (verdict r1 "What's weak" 1), each against the oracle:

* DomainError for non-positive hyperparameters under the identity transform
  (posterior.py:156, 171; oracle/core.py _hyperprior/_group_derivs),
* DivergenceError from exp overflows in the log transform: hyperprior overflow
  (posterior.py:115), spectral variance underflow (posterior.py:148), prior inverse variance
  overflow (posterior.py:369),
* JacobiError at the sweep cap (metric.py:101-109) -- from the eigensolver entry and inside a
  chain, where the reference turns it into a divergent first move (sampler.py:388-391),
* sgp_potential_derivatives (the exported per-sample U, U', U'', U''' entry) against the
  oracle's lik_derivs at 1e-13.
"""

import numpy as np
import pytest

import oracle
from golden_cases import case, rel_err

pytestmark = pytest.mark.gpu

from paper_2511_06407_b200 import metric as M  # noqa: E402
from paper_2511_06407_b200 import posterior as P  # noqa: E402
from paper_2511_06407_b200 import rrgp  # noqa: E402
from paper_2511_06407_b200 import sampler as S  # noqa: E402
from paper_2511_06407_b200.posterior import PosteriorTarget  # noqa: E402


def _both_raise(model, data, q, dev_exc, ora_exc):
    with pytest.raises(ora_exc):
        oracle.OTarget(model, data).at(q).potential()
    with pytest.raises(dev_exc):
        PosteriorTarget(model, data).at(q).potential()


@pytest.fixture(scope="module")
def identity_case():
    g, model, data = case("identity_meanvar")
    return g, model, data, rrgp.BlockLayout.from_model(model)


def test_identity_transform_nonpositive_hyper_is_a_domain_error(identity_case):
    g, model, data, layout = identity_case
    assert layout.hyper_index
    for name, idx in layout.hyper_index.items():
        for bad in (0.0, -0.3):
            q = np.array(g["q0"], dtype=float)
            q[idx] = bad
            _both_raise(model, data, q, P.DomainError, oracle.ODomain)


def test_identity_transform_valid_point_evaluates(identity_case):
    g, model, data, _ = identity_case
    q = np.array(g["q0"], dtype=float)
    assert PosteriorTarget(model, data).at(q).potential() == pytest.approx(
        oracle.OTarget(model, data).at(q).potential(), rel=1e-12)


@pytest.fixture(scope="module")
def log_case():
    g, model, data = case("meanvar_toy")
    return g, model, data, rrgp.BlockLayout.from_model(model)


@pytest.mark.parametrize("value", [800.0, -800.0])
def test_log_transform_overflow_is_a_divergence(log_case, value):
    """exp(+-800) in the hyperprior, the spectral variance or the prior inverse variance."""
    g, model, data, layout = log_case
    for name, idx in layout.hyper_index.items():
        q = np.array(g["q0"], dtype=float)
        q[idx] = value
        try:
            oracle.OTarget(model, data).at(q).potential()
            ora_ok = True
        except oracle.ODivergence:
            ora_ok = False
        if ora_ok:  # this coordinate does not overflow at this sign in the reference either
            assert np.isfinite(PosteriorTarget(model, data).at(q).potential())
        else:
            with pytest.raises(P.DivergenceError):
                PosteriorTarget(model, data).at(q).potential()


def test_jacobi_error_at_the_sweep_cap():
    g, model, data = case("meanvar_toy")
    h = oracle.OTarget(model, data).at(np.asarray(g["q0"], dtype=float)).hessian()
    with pytest.raises(oracle.OJacobi):
        oracle.cold_eigh(h, 1e-13, cap=1)
    with pytest.raises(M.JacobiError):
        M.static_eigendecompose(h, 1e-13, sweep_cap=1)
    lam, psi, sw = M.static_eigendecompose(h, 1e-13, sweep_cap=30)
    assert sw > 1


def test_sweep_cap_inside_a_chain_fails_the_first_move_like_the_reference():
    g, model, data = case("meanvar_toy")
    cfg = S.ChainConfig(epsilon=0.01, leapfrogs=2, moves=2, burnin=0, seed=3, sweep_cap=1)
    with pytest.raises(oracle.OChainError):
        oracle.run_chain(oracle.OTarget(model, data),
                         oracle.OConfig(epsilon=0.01, leapfrogs=2, moves=2, burnin=0, seed=3, sweep_cap=1))
    with pytest.raises(S.ChainError):
        S.run_chain(PosteriorTarget(model, data), cfg)


@pytest.mark.parametrize("likelihood", ["logistic", "gaussian_meanvar"])
def test_potential_derivatives_entry_matches_oracle(likelihood):
    rng = np.random.default_rng(11)
    n = 257
    if likelihood == "logistic":
        f = 3.0 * rng.standard_normal((n, 1))
        f[:4, 0] = [0.0, 40.0, -40.0, 1e-8]
        y = np.where(rng.uniform(size=n) < 0.5, -1.0, 1.0)
    else:
        f = np.stack([rng.standard_normal(n), 2.0 * rng.standard_normal(n)], axis=1)
        f[:3, 1] = [-30.0, 30.0, 0.0]
        y = rng.standard_normal(n)
    dev = P.potential_derivatives(likelihood, f, y, variance_floor=1e-3)
    ref = oracle.lik_derivs(likelihood, f, y, 1e-3)
    for a, b in zip(dev, ref):
        assert rel_err(a, b) < 1e-13
