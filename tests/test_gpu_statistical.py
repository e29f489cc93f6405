"""Statistical parity where bitwise parity cannot hold (north star: "posterior means and
log-evidence must agree within Monte Carlo standard error"; verdict item 7).

The warm solvers "parallel" and "refine" meet the reference's convergence test but not its
rounding, and the dynamics amplify that, so their trajectories are not the reference's; their
distribution must be.  Reference side: the CPU restatement of the reference algorithm
(oracle/, bit-exact with the reference on golden chains) in the reference's own pivot order.
Comparison per coordinate: z = (mean_gpu - mean_ref) / sqrt(se_gpu^2 + se_ref^2), Monte Carlo
standard errors from between-chain spread (GPU, many chains) and Geyer ESS (reference, few
long chains); Bonferroni-level bound |z| < 4.2 over the coordinates (the moment-check style of
the reference's tests/test_sampler.py:233-241).
"""

import dataclasses

import numpy as np
import pytest

import oracle
from paper_2511_06407_b200 import evidence as E
from paper_2511_06407_b200 import rrgp
from paper_2511_06407_b200 import sampler as S
from paper_2511_06407_b200.diagnostics import ess_geyer
from paper_2511_06407_b200.posterior import PosteriorTarget

pytestmark = pytest.mark.gpu

EPS, LF, BURN = 0.02, 10, 100
ZLIM = 4.2


@pytest.fixture(scope="module")
def problem():
    data, _ = rrgp.simulate_logistic(1, n=60, seed=19)
    model = rrgp.build_model("logistic", data.x, feature_count=10)
    return model, data


@pytest.fixture(scope="module")
def reference_draws(problem):
    """4 chains x 600 moves of the reference algorithm (CPU restatement, cyclic order)."""
    model, data = problem
    t = oracle.OTarget(model, data)
    chains = []
    for seed in range(4):
        r = oracle.run_chain(t, oracle.OConfig(epsilon=EPS, leapfrogs=LF, moves=600, burnin=0, seed=100 + seed,
                                               record_q=True))
        chains.append(np.vstack([rec.q for rec in r.records])[BURN:])
    return np.stack(chains)  # (4, n, d)


def _ref_mean_se(draws):
    n_chains, n, d = draws.shape
    flat = draws.reshape(-1, d)
    mean = flat.mean(axis=0)
    ess = np.array([sum(ess_geyer(draws[c, :, j]) for c in range(n_chains)) for j in range(d)])
    se = flat.std(axis=0, ddof=1) / np.sqrt(np.maximum(ess, 1.0))
    return mean, se


def _gpu_mean_se(draws):
    # independent chains: the spread of per-chain means
    cm = draws.mean(axis=1)
    return cm.mean(axis=0), cm.std(axis=0, ddof=1) / np.sqrt(cm.shape[0])


def _gpu_draws(target, order, n_chains, moves, seed0=7000, cold="cyclic"):
    cfg = S.ChainConfig(epsilon=EPS, leapfrogs=LF, moves=moves, burnin=0, record_q=True, warm_order=order,
                        cold_order=cold)
    res = S.run_chains(target, cfg, [seed0 + z for z in range(n_chains)])
    ok = [r for r in res if not isinstance(r, Exception)]  # a chain may diverge on its first move
    assert len(ok) >= 0.9 * n_chains
    return np.stack([r.sample_matrix()[BURN:] for r in ok])


def _assert_same_distribution(gpu, ref):
    mg, sg = _gpu_mean_se(gpu)
    mr, sr = _ref_mean_se(ref)
    z = (mg - mr) / np.sqrt(sg ** 2 + sr ** 2)
    assert np.max(np.abs(z)) < ZLIM, (np.round(z, 2), mg, mr)


@pytest.mark.parametrize("order", ["parallel", "cyclic"])
def test_posterior_moments_match_reference(problem, reference_draws, order):
    model, data = problem
    gpu = _gpu_draws(PosteriorTarget(model, data), order, n_chains=128, moves=600)
    _assert_same_distribution(gpu, reference_draws)


@pytest.mark.parametrize("cold", ["cyclic", "dc"])
def test_refine_solver_posterior_moments_match_reference(problem, reference_draws, monkeypatch, cold):
    """The large-d path (host-sequenced leapfrog, DMMA GEMMs, eigenvector refinement) forced
    onto the d = 14 model; cold decompositions (start, rejections) in the reference order or by
    tridiagonalisation + divide and conquer."""
    monkeypatch.setenv("SGP_FORCE_LARGE", "1")
    model, data = problem
    gpu = _gpu_draws(PosteriorTarget(model, data), "refine", n_chains=6, moves=400, cold=cold)
    _assert_same_distribution(gpu, reference_draws)


def test_thermodynamic_integration_matches_reference_within_stderr(problem):
    """Log-evidence of the device TI with the parallel warm solver (non-bitwise) vs the
    reference algorithm's TI (CPU restatement, reference order) from the same seed, 16 chains,
    5 rungs of 5 moves: within 4 combined standard errors.  (Same seed: both walks start from
    the same warm-up chain; a thin ladder's chains stay close to that point, so estimates from
    different warm-ups differ by more than their cross-chain stderr.)"""
    model, data = problem
    ladder = E.default_ladder(moves_per_rung=5, leapfrogs=LF, chains=16).thin(25)
    cfg = S.ChainConfig(epsilon=EPS, leapfrogs=LF, moves=10, burnin=0, seed=31, warm_order="parallel")
    est = E.thermo_integrate(model, data, ladder, cfg, warmup_segment_moves=10, warmup_max_segments=2,
                             spread_moves=2)
    t = oracle.OTarget(model, data)
    per_chain, _, _ = oracle.thermo_integrate(
        t, ladder.taus, ladder.moves_per_rung, ladder.leapfrogs, 16,
        oracle.OConfig(epsilon=EPS, leapfrogs=LF, moves=10, burnin=0, seed=31),
        warmup_segment_moves=10, warmup_max_segments=2, spread_moves=2)
    per_chain = np.asarray([v for v in per_chain if np.isfinite(v)], dtype=float)
    assert per_chain.size >= 12
    ref_mean = float(np.mean(per_chain))
    ref_se = float(np.std(per_chain, ddof=1) / np.sqrt(per_chain.size))
    z = (est.bme_mean - ref_mean) / np.sqrt(est.bme_stderr ** 2 + ref_se ** 2)
    assert abs(z) < 4.0, (est.bme_mean, est.bme_stderr, ref_mean, ref_se)
