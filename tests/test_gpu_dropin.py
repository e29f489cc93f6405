"""The drop-in surface on the device, written like the reference's own sampler/posterior
tests (reference tests/test_sampler.py:101-117,143-216,233-266; tests/test_posterior.py:162-199)
plus the INTEGRATION.md shim driven through a stand-in of the reference's module layout
(the reference itself is not present on GPU boxes; tests/test_integration_cpu.py pins the
shim against the real one)."""

import dataclasses
import sys
import types

import numpy as np
import pytest

import paper_2511_06407_b200 as b
from golden_cases import rel_err
from paper_2511_06407_b200 import integration
from paper_2511_06407_b200.metric import metric_apply_inverse, metric_from_hessian, sample_momentum

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small_logistic():
    data, _ = b.simulate_logistic(1, n=60, seed=19)
    model = b.build_model("logistic", data.x, feature_count=10)
    return model, data, b.PosteriorTarget(model, data)


def metric_at(target, q, kappa=1.0, zeta=1e-13):
    return metric_from_hessian(target.at(q).hessian(), kappa, zeta)


def test_grad_q_hamiltonian_matches_finite_differences(small_logistic):
    _, _, target = small_logistic
    rng = np.random.default_rng(3)
    q = 0.2 * rng.standard_normal(target.dim)
    p = rng.standard_normal(target.dim)
    metric = metric_at(target, q)
    grad = b.grad_q_hamiltonian(q, p, metric, target)
    step = 1e-5
    fd = np.empty(target.dim)
    for i in range(target.dim):
        e = np.zeros(target.dim)
        e[i] = step
        hp = b.hamiltonian(q + e, p, metric_at(target, q + e), target)
        hm = b.hamiltonian(q - e, p, metric_at(target, q - e), target)
        fd[i] = (hp - hm) / (2.0 * step)
    assert np.max(np.abs(grad - fd)) / max(1.0, np.max(np.abs(fd))) < 1e-4


def test_quadratic_target_constant_metric_is_stormer_verlet():
    target = b.QuadraticTarget(np.diag([4.0, 1.0]), mean=np.array([0.3, -0.2]))
    config = b.ChainConfig(epsilon=0.05, leapfrogs=1, moves=1, burnin=0)
    rng = np.random.default_rng(6)
    q, p = rng.standard_normal(2), rng.standard_normal(2)
    metric = metric_at(target, q)
    q1, p1, _, _ = b.leapfrog_step(q, p, metric, target, config)
    eps = config.epsilon
    p_half = p - 0.5 * eps * target.at(q).gradient()
    q_next = q + eps * metric_apply_inverse(metric, p_half)
    p_next = p_half - 0.5 * eps * target.at(q_next).gradient()
    assert np.max(np.abs(q1 - q_next)) < 1e-12
    assert np.max(np.abs(p1 - p_next)) < 1e-12


def test_quadratic_grad_q_reduces_to_potential_gradient():
    rng = np.random.default_rng(4)
    target = b.QuadraticTarget(np.diag([3.0, 1.0]), mean=np.array([0.5, -1.0]))
    q, p = rng.standard_normal(2), rng.standard_normal(2)
    grad = b.grad_q_hamiltonian(q, p, metric_at(target, q), target)
    assert np.allclose(grad, target.at(q).gradient(), atol=1e-12)


def test_reversibility(small_logistic):
    _, _, target = small_logistic
    rng = np.random.default_rng(7)
    q = 0.1 * rng.standard_normal(target.dim)
    config = b.ChainConfig(epsilon=0.0025, leapfrogs=1, moves=1, burnin=0, fp_tol=1e-12, fp_max_iters=12)
    metric = metric_at(target, q)
    p = sample_momentum(metric, rng)
    q1, p1, metric1, _ = b.leapfrog_step(q, p, metric, target, config)
    q2, p2, _, _ = b.leapfrog_step(q1, -p1, metric1, target, config)
    assert np.max(np.abs(q2 - q)) < 1e-8
    assert np.max(np.abs(-p2 - p)) < 1e-8


def test_quadratic_chain_moments_and_bookkeeping():
    target = b.QuadraticTarget(np.eye(2))
    config = b.ChainConfig(epsilon=0.6, leapfrogs=8, moves=5500, burnin=500, seed=1, record_q=True)
    result = b.run_chain(target, config)
    samples = result.sample_matrix()[config.burnin:]
    assert samples.shape == (5000, 2)
    assert np.max(np.abs(samples.mean(axis=0))) < 0.08
    assert np.max(np.abs(np.cov(samples.T) - np.eye(2))) < 0.1
    assert 0.5 < result.acceptance_rate <= 1.0
    assert result.divergence_count == 0
    assert np.allclose(result.q_final, result.records[-1].q)


def test_quadratic_chain_determinism_and_rejections():
    target = b.QuadraticTarget(np.diag([2.0, 0.5]))
    config = b.ChainConfig(epsilon=0.4, leapfrogs=5, moves=40, burnin=0, seed=9, record_q=True)
    a, c = b.run_chain(target, config), b.run_chain(target, config)
    assert np.array_equal(a.q_final, c.q_final)
    for ra, rc in zip(a.records, c.records):
        assert (ra.logpost, ra.h_before, ra.h_after, ra.accept, ra.uniform) == \
            (rc.logpost, rc.h_before, rc.h_after, rc.accept, rc.uniform)
    target = b.QuadraticTarget(np.diag([25.0, 4.0]))
    res = b.run_chain(target, b.ChainConfig(epsilon=1.1, leapfrogs=12, moves=60, burnin=0, seed=3,
                                            record_q=True))
    assert any(not r.accept for r in res.records)
    for i, r in enumerate(res.records):
        if i and not r.accept:
            assert np.array_equal(r.q, res.records[i - 1].q)


def test_first_move_divergence_raises(small_logistic):
    _, _, target = small_logistic
    with pytest.raises(b.ChainError, match="first move"):
        b.run_chain(target, b.ChainConfig(epsilon=1e6, leapfrogs=2, moves=5, burnin=0, seed=0))


@pytest.mark.parametrize("tau", [1.0, 0.35])
def test_trace_agrees_with_dense_oracle(small_logistic, tau):
    model, data, target = small_logistic
    rng = np.random.default_rng(8)
    q = 0.1 * rng.standard_normal(target.dim)
    d = target.dim
    w = rng.standard_normal((d, d))
    w = 0.5 * (w + w.T)
    t1, _ = b.trace_contractions(w, np.zeros_like(w), q, model, data, tau=tau)
    assert rel_err(t1, b.dense_oracle(w, q, model, data, tau=tau)) < 1e-8


def test_device_model_is_shared_across_targets(small_logistic):
    model, data, target = small_logistic
    assert b.PosteriorTarget(model, data).device is target.device
    assert b.PosteriorTarget(model, data, 0.3).device is target.device


# -- the shim through a stand-in of the reference's module layout ----------------------


def _fake_reference():
    """softabs_gp-shaped namespace: sampler/evidence/cli bind run_chain, with their own
    exception and record classes, and a reference-style ChainConfig without warm_order."""
    pkg = types.ModuleType("fake_softabs_gp")
    pkg.__path__ = []
    mods = {}
    for name in ("sampler", "evidence", "cli", "posterior", "metric"):
        m = types.ModuleType(f"fake_softabs_gp.{name}")
        sys.modules[m.__name__] = m
        setattr(pkg, name, m)
        mods[name] = m
    sys.modules[pkg.__name__] = pkg

    class ChainError(RuntimeError):
        pass

    class DivergenceError(FloatingPointError):
        pass

    class DomainError(ValueError):
        pass

    class JacobiError(RuntimeError):
        pass

    @dataclasses.dataclass(frozen=True)
    class RefConfig:
        epsilon: float = 0.001
        leapfrogs: int = 100
        moves: int = 9600
        burnin: int = 2400
        kappa: float = 1.0
        zeta: float = 1e-13
        fp_max_iters: int = 6
        fp_tol: float = 1e-10
        gs_interval: int = 10
        sweep_cap: int = 30
        metric: str = "softabs-dynamic"
        seed: object = 0
        record_q: bool = False

    rec_fields = [f.name for f in dataclasses.fields(b.ChainRecord)]
    RefRecord = dataclasses.make_dataclass("ChainRecord", rec_fields)
    RefResult = dataclasses.make_dataclass("ChainResult", ["records", "q_final", "accept_count",
                                                           "divergence_count", "config"])
    mods["sampler"].ChainError, mods["sampler"].ChainConfig = ChainError, RefConfig
    mods["sampler"].ChainRecord, mods["sampler"].ChainResult = RefRecord, RefResult
    mods["posterior"].DivergenceError, mods["posterior"].DomainError = DivergenceError, DomainError
    mods["metric"].JacobiError = JacobiError
    for name in ("sampler", "evidence", "cli"):
        mods[name].run_chain = lambda *a, **k: (_ for _ in ()).throw(AssertionError("not patched"))
    mods["sampler"].leapfrog_step = mods["sampler"].run_chain
    return pkg


def test_shim_runs_reference_style_calls_on_the_device(small_logistic):
    model, data, _ = small_logistic
    ref = _fake_reference()
    undo = integration.install(ref)
    try:
        # a reference-style target (model, data, tau) and config
        rtarget = types.SimpleNamespace(model=model, data=data, tau=1.0, dim=14)
        cfg = ref.sampler.ChainConfig(epsilon=0.01, leapfrogs=5, moves=3, burnin=0, seed=4, record_q=True)
        res = ref.evidence.run_chain(rtarget, cfg)
        assert isinstance(res, ref.sampler.ChainResult)
        assert isinstance(res.records[0], ref.sampler.ChainRecord)
        ours = b.run_chain(b.PosteriorTarget(model, data), b.ChainConfig(epsilon=0.01, leapfrogs=5, moves=3,
                                                                        burnin=0, seed=4, record_q=True))
        assert [r.h_before for r in res.records] == [r.h_before for r in ours.records]
        assert np.array_equal(res.q_final, ours.q_final)
        with pytest.raises(ref.sampler.ChainError, match="first move"):
            ref.cli.run_chain(rtarget, ref.sampler.ChainConfig(epsilon=1e6, leapfrogs=2, moves=2, burnin=0))
    finally:
        undo()
