"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container only (the reference is not present on GPU boxes):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports softabs_gp from /root/reference/pkg/src read-only and writes
``tests/golden/*.npz``.  Those fixtures pin both the CPU oracle (oracle/) and
the CUDA path (tests/test_gpu_*.py) to the reference's own outputs.
"""

from __future__ import annotations

import dataclasses
import hashlib
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from softabs_gp import rrgp  # noqa: E402
from softabs_gp import evidence, metric, posterior, sampler  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sym(rng, d):
    a = rng.standard_normal((d, d))
    return (a + a.T) / 2.0


def point_case(name, model, data, qs, taus, seed):
    """Posterior + metric + leapfrog quantities at a few points."""
    target = posterior.PosteriorTarget(model, data)
    d = target.dim
    rng = np.random.default_rng(seed)
    out = {"x": data.x, "y": data.y, "dim": d}
    for k, (q, tau) in enumerate(zip(qs, taus)):
        t = target.at_temperature(tau)
        st = t.at(q)
        w = sym(rng, d)
        out[f"q{k}"] = q
        out[f"tau{k}"] = tau
        out[f"pot{k}"] = st.potential()
        out[f"grad{k}"] = st.gradient()
        out[f"hess{k}"] = st.hessian()
        out[f"wt{k}"] = w
        out[f"trace{k}"] = st.trace_single(w)
        out[f"sumpot{k}"] = st.sum_potentials()
    # metric quantities at point 0/1 (tau of point 0)
    t0 = target.at_temperature(taus[0])
    h0 = t0.at(qs[0]).hessian()
    lam, psi, sweeps = metric.static_eigendecompose(h0, 1e-13)
    out.update(cold_lam=lam, cold_psi=psi, cold_sweeps=sweeps)
    m0 = metric.metric_from_hessian(h0, 1.0, 1e-13)
    h1 = t0.at(qs[1]).hessian()
    m1 = metric.dynamic_eigendecompose(h1, m0, 1e-13)
    out.update(warm_lam=m1.eigenvalues, warm_psi=m1.vectors, warm_sweeps=m1.sweep_count,
               warm_since=m1.steps_since_refresh)
    # gram-schmidt refresh path: previous state at since = 9
    m0b = dataclasses.replace(m0, steps_since_refresh=9)
    m1b = metric.dynamic_eigendecompose(h1, m0b, 1e-13)
    out.update(warmgs_lam=m1b.eigenvalues, warmgs_psi=m1b.vectors,
               warmgs_sweeps=m1b.sweep_count, warmgs_since=m1b.steps_since_refresh)
    p = rng.standard_normal(d)
    v = rng.standard_normal(d)
    z = rng.standard_normal(d)
    out.update(p=p, v=v, z=z,
               t_matrix=metric.t_matrix(m0.eigenvalues, 1.0),
               w1=metric.w1_matrix(m0, p), w2=metric.w2_matrix(m0),
               ginv=metric.metric_apply_inverse(m0, v),
               quad=metric.metric_quadratic(m0, p),
               logdet=m0.logdet,
               momentum=m0.vectors @ (np.sqrt(m0.softabs_values) * z),
               ham=sampler.hamiltonian(qs[0], p, m0, t0),
               gradq=sampler.grad_q_hamiltonian(qs[0], p, m0, t0))
    # one generalized leapfrog from (q0, p)
    for tag, eps in (("lf", 0.01), ("lfs", 0.002)):
        cfg = sampler.ChainConfig(epsilon=eps, leapfrogs=1, moves=1, burnin=0)
        q1, p1, mt1, diag = sampler.leapfrog_step(qs[0], 0.3 * p, m0, t0, cfg)
        out[f"{tag}_q"] = q1
        out[f"{tag}_p"] = p1
        out[f"{tag}_lam"] = mt1.eigenvalues
        out[f"{tag}_psi"] = mt1.vectors
        out[f"{tag}_fp_p"] = np.asarray(diag["fp_p_iters"])
        out[f"{tag}_fp_q"] = np.asarray(diag["fp_q_iters"])
        out[f"{tag}_sweeps"] = np.asarray(diag["sweeps"])
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print("wrote", name, "d =", d)


def chain_arrays(res):
    recs = res.records
    return dict(
        h_before=np.array([r.h_before for r in recs]),
        h_after=np.array([np.nan if r.h_after is None else r.h_after for r in recs]),
        accept=np.array([r.accept for r in recs]),
        divergent=np.array([r.divergent for r in recs]),
        sweeps_mean=np.array([r.sweeps_mean for r in recs]),
        logpost=np.array([r.logpost for r in recs]),
        uniform=np.array([r.uniform for r in recs]),
        q=np.vstack([r.q for r in recs]) if recs[0].q is not None else np.zeros((0,)),
        q_final=res.q_final,
    )


def chain_case(name, model, data, cfg, tau=1.0):
    target = posterior.PosteriorTarget(model, data, tau)
    res = sampler.run_chain(target, cfg)
    out = chain_arrays(res)
    out.update(x=data.x, y=data.y, epsilon=cfg.epsilon, leapfrogs=cfg.leapfrogs,
               moves=cfg.moves, seed=cfg.seed, metric_mode=cfg.metric, tau=tau)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print("wrote", name, "accept", int(np.sum(out["accept"])), "/", cfg.moves,
          "div", int(np.sum(out["divergent"])))


def main():
    # A: d = 34 logistic (tests/conftest.py:128-133)
    data, _ = rrgp.simulate_logistic(1, n=120, seed=7)
    model = rrgp.build_model("logistic", data.x)
    d = 34
    rng = np.random.default_rng(11)
    qs = [0.1 * rng.standard_normal(d), 0.1 * rng.standard_normal(d) + 0.002,
          np.zeros(d), 0.3 * rng.standard_normal(d)]
    qs[1] = qs[0] + 1e-3 * rng.standard_normal(d)
    point_case("logistic_small", model, data, qs, [1.0, 1.0, 1.0, 0.35], seed=12)

    # B: heteroscedastic toy (tests/conftest.py:142-147)
    data, _ = rrgp.simulate_meanvar(1, 1, n=60, seed=21)
    model = rrgp.build_model("nl-meanvar", data.x, feature_count=8)
    d = posterior.PosteriorTarget(model, data).dim
    rng = np.random.default_rng(13)
    q0 = 0.1 * rng.standard_normal(d)
    qs = [q0, q0 + 1e-3 * rng.standard_normal(d), np.zeros(d), 0.2 * rng.standard_normal(d)]
    point_case("meanvar_toy", model, data, qs, [1.0, 1.0, 1.0, 0.6], seed=14)

    # C: fixed hyperparameters (tests/conftest.py:101-125)
    rng = np.random.default_rng(5)
    x = rng.standard_normal((40, 1))
    y = np.sin(1.5 * x[:, 0]) + 0.3 * rng.standard_normal(40)
    data = rrgp.Dataset(x, y)
    model = rrgp.build_model("nl-mean", x, feature_count=8, intercept_variance=1e-4,
                             fixed_hypers={"c_g": 1.3, "sigma_g": 2.1, "c_l": 1.0})
    d = posterior.PosteriorTarget(model, data).dim
    rng = np.random.default_rng(15)
    q0 = 0.1 * rng.standard_normal(d)
    qs = [q0, q0 + 1e-3 * rng.standard_normal(d), np.zeros(d), 0.2 * rng.standard_normal(d)]
    point_case("conjugate", model, data, qs, [1.0, 1.0, 1.0, 0.5], seed=16)

    # D: identity hyper transform, l-meanvar with a binary column
    data, _ = rrgp.simulate_meanvar(1, 2, n=50, seed=3)
    model = rrgp.build_model("nl-meanvar", data.x, feature_count=6, hyper_transform="identity")
    d = posterior.PosteriorTarget(model, data).dim
    rng = np.random.default_rng(17)
    q0 = 0.1 * rng.standard_normal(d)
    q0[-3:] = [1.2, 0.8, 1.5]
    qs = [q0, q0 + 1e-3 * rng.standard_normal(d), posterior.PosteriorTarget(model, data).initial_point(), q0 * 1.1]
    point_case("identity_meanvar", model, data, qs, [1.0, 1.0, 1.0, 0.8], seed=18)

    # E: chains on C1 (logistic D=1, n=500, seed 0, d=34)
    data, _ = rrgp.simulate_logistic(1, n=500, seed=0)
    model = rrgp.build_model("logistic", data.x)
    chain_case("chain_c1_eps1e-2", model, data,
               sampler.ChainConfig(epsilon=0.01, leapfrogs=20, moves=60, burnin=0, seed=0,
                                   record_q=True))
    chain_case("chain_c1_eps1e-3", model, data,
               sampler.ChainConfig(epsilon=0.001, leapfrogs=20, moves=30, burnin=0, seed=3,
                                   record_q=True))
    # rejection-heavy chain exercises cold resyncs and divergences
    chain_case("chain_c1_eps15e-3", model, data,
               sampler.ChainConfig(epsilon=0.015, leapfrogs=20, moves=30, burnin=0, seed=5,
                                   record_q=True))
    data_s, _ = rrgp.simulate_logistic(1, n=60, seed=19)
    model_s = rrgp.build_model("logistic", data_s.x, feature_count=10)
    chain_case("chain_small_static", model_s, data_s,
               sampler.ChainConfig(epsilon=0.02, leapfrogs=5, moves=20, burnin=0, seed=7,
                                   metric="softabs-static", record_q=True))
    chain_case("chain_small_euclid", model_s, data_s,
               sampler.ChainConfig(epsilon=0.05, leapfrogs=10, moves=30, burnin=0, seed=8,
                                   metric="euclidean", record_q=True))
    data_m, _ = rrgp.simulate_meanvar(1, 1, n=60, seed=21)
    model_m = rrgp.build_model("nl-meanvar", data_m.x, feature_count=8)
    chain_case("chain_meanvar_tau", model_m, data_m,
               sampler.ChainConfig(epsilon=0.01, leapfrogs=10, moves=20, burnin=0, seed=9,
                                   record_q=True), tau=0.5)

    # F: thermodynamic integration on a tiny ladder
    ladder = evidence.default_ladder(moves_per_rung=3, leapfrogs=5, chains=3).thin(25)
    cfg = sampler.ChainConfig(epsilon=0.02, leapfrogs=5, moves=10, burnin=0, seed=123)
    est = evidence.thermo_integrate(model_s, data_s, ladder, cfg, warmup_segment_moves=10,
                                    warmup_max_segments=2, spread_moves=2)
    np.savez_compressed(os.path.join(OUT, "ti_small.npz"), x=data_s.x, y=data_s.y,
                        taus=ladder.taus, per_chain=np.asarray(est.per_chain),
                        rung_values=est.rung_values, bme_mean=est.bme_mean,
                        bme_stderr=est.bme_stderr)
    print("wrote ti_small", est.bme_mean, est.bme_stderr)

    # G: generator fingerprints for the benchmark configs
    fp = {}
    for tag, (ds, _) in {
        "c1": rrgp.simulate_logistic(1, n=500, seed=0),
        "c2": rrgp.simulate_logistic(1, n=512, seed=0),
        "c1d4": rrgp.simulate_logistic(4, n=500, seed=0),
        "c3": rrgp.simulate_meanvar(2, 19, n=2000, seed=0),
        "c4": rrgp.simulate_meanvar(34, 19, n=8192, seed=0),
    }.items():
        fp[f"{tag}_x"] = hashlib.sha256(ds.x.tobytes()).hexdigest()
        fp[f"{tag}_y"] = hashlib.sha256(ds.y.tobytes()).hexdigest()
        fp[f"{tag}_y_head"] = ds.y[:8]
    np.savez_compressed(os.path.join(OUT, "generators.npz"), **fp)

    # H: rank-sum test values
    rng = np.random.default_rng(99)
    rs = []
    for n1, n2 in ((5, 7), (10, 10), (30, 25)):
        a = np.round(rng.standard_normal(n1), 1)
        b = np.round(rng.standard_normal(n2) + 0.3, 1)
        z, pv = sampler.rank_sum_test(a, b)
        rs.append((a, b, z, pv))
    np.savez_compressed(os.path.join(OUT, "ranksum.npz"),
                        **{f"a{i}": r[0] for i, r in enumerate(rs)},
                        **{f"b{i}": r[1] for i, r in enumerate(rs)},
                        z=np.array([r[2] for r in rs]), p=np.array([r[3] for r in rs]))
    print("done")


if __name__ == "__main__":
    main()
