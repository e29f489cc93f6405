"""The INTEGRATION.md shim against the UNMODIFIED reference package (build container only;
skipped where /root/reference is absent).  No device work: the device sampler is replaced by
a stub, so this pins the binding, the config/result/exception translation and uninstall."""

import dataclasses
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


@pytest.fixture(scope="module")
def ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_tests")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import softabs_gp
    import softabs_gp.cli
    import softabs_gp.evidence
    import softabs_gp.sampler

    return softabs_gp


def test_install_rebinds_every_import_site_and_uninstalls(ref):
    from paper_2511_06407_b200 import integration

    orig = (ref.sampler.run_chain, ref.evidence.run_chain, ref.cli.run_chain, ref.sampler.leapfrog_step)
    undo = integration.install(ref)
    try:
        assert ref.sampler.run_chain is ref.evidence.run_chain is ref.cli.run_chain
        assert ref.sampler.run_chain is not orig[0]
        assert ref.sampler.leapfrog_step is not orig[3]
    finally:
        undo()
    assert (ref.sampler.run_chain, ref.evidence.run_chain, ref.cli.run_chain,
            ref.sampler.leapfrog_step) == orig


def test_reference_config_converts_by_field_name(ref):
    from paper_2511_06407_b200.sampler import ChainConfig, as_chain_config

    rc = ref.sampler.ChainConfig(epsilon=0.02, leapfrogs=7, moves=30, burnin=5, seed=11, record_q=True,
                                 metric="softabs-static", fp_tol=1e-11, sweep_cap=17)
    c = as_chain_config(rc)
    assert isinstance(c, ChainConfig)
    for f in dataclasses.fields(rc):
        assert getattr(c, f.name) == getattr(rc, f.name), f.name
    assert c.warm_order == "cyclic" and c.cold_order == "cyclic"


def test_results_and_errors_come_back_as_reference_classes(ref, monkeypatch):
    from paper_2511_06407_b200 import integration
    from paper_2511_06407_b200 import sampler as S

    data, _ = ref.rrgp.simulate_logistic(1, n=40, seed=1)
    model = ref.rrgp.build_model("logistic", data.x, feature_count=4)
    rtarget = ref.posterior.PosteriorTarget(model, data)
    rcfg = ref.sampler.ChainConfig(epsilon=0.01, leapfrogs=2, moves=2, burnin=0, seed=3, record_q=True)
    seen = {}

    def fake_run_chain(target, config, *, initial=None):
        seen["config"], seen["target"] = config, target
        recs = [S.ChainRecord(move=m, logpost=-1.0 - m, h_before=2.0, h_after=2.5, accept=bool(m), divergent=False,
                              sweeps_mean=1.5, wall_ms=0.1, q=np.full(3, m), uniform=0.3) for m in range(2)]
        return S.ChainResult(records=recs, q_final=np.ones(3), accept_count=1, divergence_count=0, config=config)

    monkeypatch.setattr(S, "run_chain", fake_run_chain)
    monkeypatch.setattr(S, "as_device_target", lambda t: t)
    undo = integration.install(ref)
    try:
        res = ref.evidence.run_chain(rtarget, rcfg)
        assert isinstance(res, ref.sampler.ChainResult)
        assert all(isinstance(r, ref.sampler.ChainRecord) for r in res.records)
        assert res.config is rcfg and isinstance(seen["config"], S.ChainConfig)
        assert [r.accept for r in res.records] == [False, True]

        def failing(target, config, *, initial=None):
            raise S.ChainError("divergence on the first move; initial point or epsilon unusable")

        monkeypatch.setattr(S, "run_chain", failing)
        with pytest.raises(ref.sampler.ChainError, match="first move"):
            ref.sampler.run_chain(rtarget, rcfg)
        # the reference's own _chain_job catch (evidence.py:180) now sees its class
        q_warm = np.zeros(rtarget.dim)
        job = (model, data, ref.evidence.default_ladder(moves_per_rung=1, leapfrogs=1, chains=1).thin(50),
               rcfg, q_warm, np.random.SeedSequence(1), False, 1, rtarget)
        values, err = ref.evidence._chain_job(job)
        assert values is None and "first move" in err
    finally:
        undo()
