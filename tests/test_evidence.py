"""Thermodynamic integration: ladder algebra, seeding/aggregation parity with
the reference, and the multi-rank (chain-sharded, all-gather) path.

The CPU tests drive ``evidence.thermo_integrate`` with the oracle as chain
executor (injected runners), so the sharding and collective logic is tested
without a GPU; the GPU test runs the real device batch against the golden
vectors of the reference's own thermo_integrate.
"""

import dataclasses
import math
import os
import pickle
import socket
import tempfile

import numpy as np
import pytest

import oracle
from golden_cases import case, rel_err
from paper_2511_06407_b200 import evidence as E
from paper_2511_06407_b200.sampler import ChainConfig, ChainError


def test_ladder_shape_and_thinning():
    lad = E.default_ladder()
    assert lad.size == 101 and lad.taus[0] == 1.0 and lad.taus[-1] == 0.0
    assert np.all(np.diff(lad.taus) < 0)
    th = lad.thin(4)
    assert th.taus[0] == 1.0 and th.taus[-1] == 0.0 and th.size == 26
    with pytest.raises(ValueError):
        E.TemperLadder(taus=np.array([1.0, 0.5]))
    with pytest.raises(ValueError):
        E.TemperLadder(taus=np.array([1.0, 0.6, 0.7, 0.0]))


def test_ti_variance_closed_forms():
    taus = np.array([1.0, 0.5, 0.0])
    assert E.ti_variance(np.array([1.0, 0.0, 0.0]), taus) == pytest.approx(0.25 * 0.25)
    assert E.ti_variance(np.array([0.0, 1.0, 0.0]), taus) == pytest.approx(0.25 * 0.5)
    assert E.trapezoid(np.array([2.0, 2.0, 2.0]), taus) == pytest.approx(2.0)


def oracle_warmup_runner(target, cfg, initial=None):
    return oracle.run_chain(target, cfg, initial)


def oracle_ladder_runner(target, chain_seqs, q_warm, ladder, config, rung_average, spread_moves):
    """Per-chain ladder walk on the CPU oracle (evidence.py:142-181)."""
    S = ladder.size
    values = np.full((len(chain_seqs), S), np.nan)
    errors = []
    for k, seq in enumerate(chain_seqs):
        subs = seq.spawn(S + 1)
        try:
            q = np.asarray(q_warm, dtype=float)
            if spread_moves > 0:
                q = oracle.run_chain(target, dataclasses.replace(
                    config, moves=spread_moves, burnin=0, record_q=False, seed=subs[0]), q).q_final
            for s, tau in enumerate(ladder.taus):
                res = oracle.run_chain(target.at_temperature(float(tau)), dataclasses.replace(
                    config, moves=ladder.moves_per_rung, leapfrogs=ladder.leapfrogs, burnin=0,
                    record_q=False, seed=subs[s + 1]), q)
                q = res.q_final
                values[k, s] = target.log_likelihood(q)
            errors.append(None)
        except oracle.OChainError as exc:
            values[k] = np.nan
            errors.append(str(exc))
    return values, errors


def _ti_small(**kw):
    g, model, data = case("ti_small")
    target = oracle.OTarget(model, data)
    ladder = E.TemperLadder(taus=g["taus"], moves_per_rung=3, leapfrogs=5, chains=3)
    cfg = ChainConfig(epsilon=0.02, leapfrogs=5, moves=10, burnin=0, seed=123)
    est = E.thermo_integrate(model, data, ladder, cfg, warmup_segment_moves=10, warmup_max_segments=2,
                             spread_moves=2, target=target, ladder_runner=oracle_ladder_runner,
                             warmup_runner=oracle_warmup_runner, **kw)
    return g, est


def test_orchestration_matches_reference_golden():
    g, est = _ti_small()
    assert rel_err(est.rung_values, g["rung_values"]) < 1e-9
    assert rel_err(est.per_chain, g["per_chain"]) < 1e-9
    assert est.bme_mean == pytest.approx(float(g["bme_mean"]), rel=1e-9)
    assert est.bme_stderr == pytest.approx(float(g["bme_stderr"]), rel=1e-8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, out_dir):
    import torch.distributed as dist

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        _, est = _ti_small()
        with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as fh:
            pickle.dump((est.per_chain, est.rung_values, est.bme_mean), fh)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_is_bitwise_identical():
    """Chains sharded over 2 ranks + all-gather == single process, bit for bit."""
    import torch.multiprocessing as tmp

    _, ref = _ti_small()
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        tmp.spawn(_rank_main, args=(2, port, d), nprocs=2, join=True)
        for rank in range(2):
            with open(os.path.join(d, f"rank{rank}.pkl"), "rb") as fh:
                per_chain, rung_values, bme = pickle.load(fh)
            np.testing.assert_array_equal(np.asarray(per_chain), np.asarray(ref.per_chain))
            np.testing.assert_array_equal(rung_values, ref.rung_values)
            assert bme == ref.bme_mean


def test_failed_chains_are_flagged_not_fatal():
    def runner(target, chain_seqs, q_warm, ladder, config, rung_average, spread_moves):
        vals, errs = oracle_ladder_runner(target, chain_seqs, q_warm, ladder, config, rung_average,
                                          spread_moves)
        vals[0] = np.nan  # chain 0 "raised ChainError"
        return vals, ["boom"] + errs[1:]
    g, model, data = case("ti_small")
    ladder = E.TemperLadder(taus=g["taus"], moves_per_rung=3, leapfrogs=5, chains=3)
    cfg = ChainConfig(epsilon=0.02, leapfrogs=5, moves=10, burnin=0, seed=123)
    est = E.thermo_integrate(model, data, ladder, cfg, warmup_segment_moves=10, warmup_max_segments=2,
                             spread_moves=2, target=oracle.OTarget(model, data), ladder_runner=runner,
                             warmup_runner=oracle_warmup_runner)
    assert math.isnan(est.per_chain[0]) and all(math.isfinite(v) for v in est.per_chain[1:])
    assert any("chain 0" in w for w in est.warnings)


@pytest.mark.gpu
def test_device_thermo_integrate_matches_reference_golden():
    from paper_2511_06407_b200.posterior import PosteriorTarget
    g, model, data = case("ti_small")
    ladder = E.TemperLadder(taus=g["taus"], moves_per_rung=3, leapfrogs=5, chains=3)
    cfg = ChainConfig(epsilon=0.02, leapfrogs=5, moves=10, burnin=0, seed=123)
    est = E.thermo_integrate(model, data, ladder, cfg, warmup_segment_moves=10, warmup_max_segments=2,
                             spread_moves=2, target=PosteriorTarget(model, data))
    assert rel_err(est.rung_values, g["rung_values"]) < 1e-9
    assert rel_err(est.per_chain, g["per_chain"]) < 1e-9
    assert est.bme_mean == pytest.approx(float(g["bme_mean"]), rel=1e-9)


# -- several models, (model, chain) units sharded over ranks --------------


def _two_models():
    g, model, data = case("ti_small")
    from paper_2511_06407_b200 import rrgp
    other = rrgp.build_model("logistic", data.x, feature_count=6)
    ladder = E.TemperLadder(taus=g["taus"], moves_per_rung=3, leapfrogs=5, chains=3)
    cfg = ChainConfig(epsilon=0.02, leapfrogs=5, moves=10, burnin=0, seed=123)
    return [model, other], data, ladder, cfg


def _sweep(models, data, ladder, cfg):
    return E.evidence_sweep(models, data, ladder, cfg, warmup_segment_moves=10, warmup_max_segments=2,
                            spread_moves=2, targets=[oracle.OTarget(m, data) for m in models],
                            ladder_runner=oracle_ladder_runner, warmup_runner=oracle_warmup_runner)


def test_sweep_equals_per_model_thermo_integrate():
    models, data, ladder, cfg = _two_models()
    ests = _sweep(models, data, ladder, cfg)
    for m, est in zip(models, ests):
        one = E.thermo_integrate(m, data, ladder, cfg, warmup_segment_moves=10, warmup_max_segments=2,
                                 spread_moves=2, target=oracle.OTarget(m, data),
                                 ladder_runner=oracle_ladder_runner, warmup_runner=oracle_warmup_runner)
        np.testing.assert_array_equal(est.rung_values, one.rung_values)
        assert est.bme_mean == one.bme_mean and est.bme_stderr == one.bme_stderr


def _sweep_rank_main(rank, world, port, out_dir):
    import torch.distributed as dist

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        models, data, ladder, cfg = _two_models()
        ests = _sweep(models, data, ladder, cfg)
        from paper_2511_06407_b200.diagnostics import distributed_split_rhat
        chains = np.random.default_rng(5).standard_normal((7, 40, 3))
        mine = [z for z in range(7) if z % world == rank]
        rh = distributed_split_rhat(chains[mine], mine, 7)
        with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as fh:
            pickle.dump(([e.rung_values for e in ests], [e.bme_mean for e in ests], rh), fh)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_unit_sharding_is_bitwise_identical(world):
    """Several models' (model, chain) units over W gloo ranks, one all-gather == one process,
    bit for bit; the replica split-R-hat gathered from per-chain summaries == split_rhat."""
    import torch.multiprocessing as tmp

    from paper_2511_06407_b200.diagnostics import split_rhat

    models, data, ladder, cfg = _two_models()
    ref = _sweep(models, data, ladder, cfg)
    ref_rh = split_rhat(np.random.default_rng(5).standard_normal((7, 40, 3)))
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        tmp.spawn(_sweep_rank_main, args=(world, port, d), nprocs=world, join=True)
        for rank in range(world):
            with open(os.path.join(d, f"rank{rank}.pkl"), "rb") as fh:
                rvs, bmes, rh = pickle.load(fh)
            for k in range(len(models)):
                np.testing.assert_array_equal(rvs[k], ref[k].rung_values)
                assert bmes[k] == ref[k].bme_mean
            np.testing.assert_array_equal(rh, ref_rh)


@pytest.mark.gpu
@pytest.mark.parametrize("rung_average", [False, True])
def test_resident_ladder_walk_equals_rung_by_rung(rung_average, monkeypatch):
    """sgp_ladder_walk (the whole walk in one launch) == one launch per rung (the large-path
    fallback of device_ladder_runner), with and without rung averaging."""
    from paper_2511_06407_b200.posterior import PosteriorTarget
    g, model, data = case("ti_small")
    ladder = E.TemperLadder(taus=g["taus"], moves_per_rung=3, leapfrogs=5, chains=3)
    cfg = ChainConfig(epsilon=0.02, leapfrogs=5, moves=10, burnin=0, seed=123)
    kw = dict(warmup_segment_moves=10, warmup_max_segments=2, spread_moves=2, rung_average=rung_average,
              target=PosteriorTarget(model, data))
    resident = E.thermo_integrate(model, data, ladder, cfg, **kw)
    monkeypatch.setattr(E, "_resident_walk", lambda *a, **k: False)
    per_rung = E.thermo_integrate(model, data, ladder, cfg, **kw)
    assert rel_err(resident.rung_values, per_rung.rung_values) < 1e-12
