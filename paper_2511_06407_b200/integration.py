"""Drop-in shim: run an installed reference package (``softabs_gp``) on this build.

The reference binds ``run_chain`` by name at import time in ``evidence.py:27`` and
``cli.py:30-37`` ("import binding hazard"), so replacing
``softabs_gp.sampler.run_chain`` alone is not enough.  ``install(softabs_gp)`` patches the
name in every module that holds it, plus ``leapfrog_step``, and translates at the boundary:

* the reference's ``ChainConfig`` -> this package's (fields read by name; the pivot orders
  default to the reference's, sampler.as_chain_config);
* the reference's ``PosteriorTarget`` (and its constant-Hessian test fake) -> a device target on
  the cached device model of (model, data), so the evidence loop's per-rung targets do not
  re-upload the design matrices (sampler.as_device_target, posterior.shared_device);
* results -> the reference's ``ChainResult``/``ChainRecord``/``MetricState`` classes;
* exceptions -> the reference's classes (``sampler.ChainError``, ``posterior.DivergenceError``,
  ``posterior.DomainError``, ``metric.JacobiError``), so ``_chain_job``'s ``except ChainError``
  (evidence.py:180) and ``sampler._DIVERGENT`` keep their meaning.

``install`` returns an ``uninstall`` callable that restores the original bindings.
"""

from __future__ import annotations

import dataclasses
import functools
import importlib

from . import sampler as _s
from .metric import JacobiError
from .posterior import DivergenceError, DomainError

_PATCHED_MODULES = ("sampler", "evidence", "cli")


def _ref_module(ref, name):
    try:
        return importlib.import_module(f"{ref.__name__}.{name}")
    except ImportError:
        return getattr(ref, name, None)


def _translate_errors(ref):
    rs, rp, rm = (_ref_module(ref, n) for n in ("sampler", "posterior", "metric"))
    table = (
        (_s.ChainError, getattr(rs, "ChainError", None)),
        (DomainError, getattr(rp, "DomainError", None)),
        (DivergenceError, getattr(rp, "DivergenceError", None)),
        (JacobiError, getattr(rm, "JacobiError", None)),
    )

    def wrap(fn):
        @functools.wraps(fn)
        def inner(*a, **k):
            try:
                return fn(*a, **k)
            except Exception as exc:
                for ours, theirs in table:
                    if theirs is not None and isinstance(exc, ours) and not isinstance(exc, theirs):
                        raise theirs(str(exc)) from exc
                raise
        return inner

    return wrap


def _to_ref_record(rs, rec):
    cls = getattr(rs, "ChainRecord", None)
    if cls is None:
        return rec
    names = {f.name for f in dataclasses.fields(cls)}
    return cls(**{k: v for k, v in dataclasses.asdict(rec).items() if k in names})


def _to_ref_result(rs, res, config):
    cls = getattr(rs, "ChainResult", None)
    if cls is None:
        return res
    return cls(records=[_to_ref_record(rs, r) for r in res.records], q_final=res.q_final,
               accept_count=res.accept_count, divergence_count=res.divergence_count, config=config)


def _to_ref_metric(rm, m):
    cls = getattr(rm, "MetricState", None)
    if cls is None or m is None:
        return m
    names = {f.name for f in dataclasses.fields(cls)}
    return cls(**{k: v for k, v in dataclasses.asdict(m).items() if k in names})


def install(ref):
    """Route ``ref`` (the imported ``softabs_gp`` package) through this build; returns uninstall()."""
    rs, rm = _ref_module(ref, "sampler"), _ref_module(ref, "metric")
    wrap = _translate_errors(ref)

    @wrap
    def run_chain(target, config, *, initial=None):
        res = _s.run_chain(_s.as_device_target(target), _s.as_chain_config(config), initial=initial)
        return _to_ref_result(rs, res, config)

    @wrap
    def leapfrog_step(q, p, metric, target, config):
        q1, p1, m1, diag = _s.leapfrog_step(q, p, metric, _s.as_device_target(target), _s.as_chain_config(config))
        return q1, p1, _to_ref_metric(rm, m1), diag

    saved = []
    for name in _PATCHED_MODULES:
        mod = _ref_module(ref, name)
        if mod is None:
            continue
        for attr, fn in (("run_chain", run_chain), ("leapfrog_step", leapfrog_step)):
            if hasattr(mod, attr):
                saved.append((mod, attr, getattr(mod, attr)))
                setattr(mod, attr, fn)
    for attr, fn in (("run_chain", run_chain), ("leapfrog_step", leapfrog_step)):
        if hasattr(ref, attr):
            saved.append((ref, attr, getattr(ref, attr)))
            setattr(ref, attr, fn)

    def uninstall():
        for mod, attr, fn in reversed(saved):
            setattr(mod, attr, fn)

    return uninstall
