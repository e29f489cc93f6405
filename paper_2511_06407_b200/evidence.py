"""Thermodynamic-integration model evidence on one or many B200s.

Drop-in for ``softabs_gp.evidence.thermo_integrate`` (/root/reference/pkg/src/
softabs_gp/evidence.py:184-274) with the same seeding, warm-up gating, ladder
walk and aggregation, so the estimate for a given seed is the reference's.
What changes is how chains execute:

* all chains of a rank advance together: per rung one cold-start launch and
  one on-device move-loop launch for the whole batch (one CTA per chain);
* (model, chain) units are sharded across ranks (unit u on rank u mod W;
  ``evidence_sweep`` for several models, ``thermo_integrate`` for one) when
  ``torch.distributed`` is initialised; rungs are never split;
* the only collective is one all-gather of the per-chain rung values
  (NCCL on GPU ranks, gloo in CPU tests), after the ladders.

Chain results depend only on (seed, z), so estimates are bitwise identical
for any world size.
"""

from __future__ import annotations

import ctypes
import dataclasses
import json
import math

import numpy as np

from .metric import JacobiError
from .posterior import PosteriorTarget
from .sampler import ChainConfig, ChainError, as_chain_config, run_chain, run_chains, wilcoxon_split_half


@dataclasses.dataclass(frozen=True)
class TemperLadder:
    """Temperature schedule and per-rung effort (evidence.py:34-66)."""

    taus: np.ndarray
    moves_per_rung: int = 50
    leapfrogs: int = 100
    chains: int = 10

    def __post_init__(self):
        taus = np.asarray(self.taus, dtype=float)
        object.__setattr__(self, "taus", taus)
        if taus.ndim != 1 or taus.shape[0] < 2:
            raise ValueError("ladder needs at least two rungs")
        if taus[0] != 1.0 or taus[-1] != 0.0:
            raise ValueError("ladder must start at tau = 1 and end at tau = 0")
        if not np.all(np.diff(taus) < 0.0):
            raise ValueError("ladder temperatures must strictly decrease")
        if self.moves_per_rung < 1 or self.leapfrogs < 1 or self.chains < 1:
            raise ValueError("moves_per_rung, leapfrogs and chains must be positive")

    @property
    def size(self):
        return self.taus.shape[0]

    def thin(self, factor):
        if factor < 1:
            raise ValueError("thinning factor must be at least 1")
        idx = list(range(0, self.size, factor))
        if idx[-1] != self.size - 1:
            idx.append(self.size - 1)
        return dataclasses.replace(self, taus=self.taus[idx])


def default_ladder(moves_per_rung=50, leapfrogs=100, chains=10):
    """The 101-rung schedule (evidence.py:69-80)."""
    taus = np.empty(101)
    taus[:41] = 1.0 - 0.02 * np.arange(41)
    taus[41:71] = 0.2 - 0.005 * np.arange(1, 31)
    taus[71:91] = 0.05 - 0.002 * np.arange(1, 21)
    taus[91:] = 0.01 - 0.001 * np.arange(1, 11)
    taus[0], taus[-1] = 1.0, 0.0
    return TemperLadder(taus=taus, moves_per_rung=moves_per_rung, leapfrogs=leapfrogs, chains=chains)


def trapezoid(values, taus):
    return float(np.sum(0.5 * (values[1:] + values[:-1]) * -np.diff(taus)))


def ti_variance(rung_variances, ladder):
    taus = ladder.taus if hasattr(ladder, "taus") else np.asarray(ladder, dtype=float)
    v = np.asarray(rung_variances, dtype=float)
    if v.shape != taus.shape:
        raise ValueError("need one variance per rung")
    dt = np.diff(taus)
    total = v[0] * dt[0] ** 2 + v[-1] * dt[-1] ** 2
    if v.shape[0] > 2:
        total += float(np.sum(v[1:-1] * (dt[:-1] ** 2 + dt[1:] ** 2)))
    return 0.25 * float(total)


@dataclasses.dataclass
class EvidenceEstimate:
    bme_mean: float
    bme_stderr: float
    per_chain: list
    rung_means: list
    ladder: TemperLadder
    warnings: list
    rung_values: np.ndarray | None = None

    def to_json(self):
        return json.dumps({"bme_mean": self.bme_mean, "bme_stderr": self.bme_stderr,
                           "per_chain": self.per_chain, "ladder": [float(t) for t in self.ladder.taus],
                           "rung_means": self.rung_means, "warnings": self.warnings}, indent=2)


def warm_up(target, config, seqs, segment_moves, pvalue, warnings, initial, runner=run_chain):
    """Segments at tau = 1 until the split-half trend test passes (evidence.py:125-139)."""
    q = target.initial_point() if initial is None else np.asarray(initial, dtype=float)
    for seq in seqs:
        cfg = dataclasses.replace(config, moves=segment_moves, burnin=0, record_q=False, seed=seq)
        res = runner(target, cfg, initial=q)
        q = res.q_final
        if segment_moves >= 10:
            _, p = wilcoxon_split_half(res.logpost)
            if p > pvalue:
                return q
    warnings.append(f"warm-up trend still visible after {len(seqs)} segments")
    return q


def device_ladder_runner(target, chain_seqs, q_warm, ladder, config, rung_average, spread_moves):
    """Walk every chain in ``chain_seqs`` down the ladder as one device batch.

    Returns (values (n, S) with NaN rows for chains that raised ChainError,
    list of error strings or None) -- the per-chain outcome of evidence.py:166-181.
    """
    n = len(chain_seqs)
    S = ladder.size
    values = np.full((n, S), np.nan)
    errors = [None] * n
    subs = [seq.spawn(S + 1) for seq in chain_seqs]
    q = np.tile(np.asarray(q_warm, dtype=float), (n, 1))
    alive = list(range(n))

    def step(tgt, cfg, seeds_of):
        nonlocal alive
        results = run_chains(tgt, cfg, [seeds_of(k) for k in alive], q[alive])
        keep = []
        for k, res in zip(alive, results):
            if isinstance(res, ChainError):
                errors[k] = str(res)
                continue
            if isinstance(res, Exception):
                raise res
            q[k] = res.q_final
            keep.append((k, res))
        alive = [k for k, _ in keep]
        return keep

    if spread_moves > 0 and alive:
        step(target, dataclasses.replace(config, moves=spread_moves, burnin=0, record_q=False),
             lambda k: subs[k][0])
    if alive and _resident_walk(target, ladder, config, rung_average, subs, q, alive, values, errors):
        return values, errors
    # the large path: rung by rung (one cold start + one move loop per rung for all chains)
    for s, tau in enumerate(ladder.taus):
        if not alive:
            break
        cfg = dataclasses.replace(config, moves=ladder.moves_per_rung, leapfrogs=ladder.leapfrogs,
                                  burnin=0, record_q=rung_average)
        keep = step(target.at_temperature(float(tau)), cfg, lambda k: subs[k][s + 1])
        if not keep:
            continue
        if rung_average:
            for k, res in keep:
                values[k, s] = float(np.mean(target.log_likelihoods(res.sample_matrix())))
        else:
            idx = [k for k, _ in keep]
            values[idx, s] = target.log_likelihoods(q[idx])
    for k in range(n):
        if errors[k] is not None:
            values[k] = np.nan
    return values, errors


def _resident_walk(target, ladder, config, rung_average, subs, q, alive, values, errors):
    """The whole ladder walk of the alive chains in one device launch (sgp_ladder_walk: per rung
    a cold start at the rung's temperature and the rung's moves, evidence.py:142-163).  The
    draws are the reference's: chain k, rung s from default_rng(subs[k][s + 1]), d normals then
    one uniform per move.  Returns False when the model runs on the large path."""
    import torch

    from . import _native as nat
    from .sampler import DeviceChains, draw_move_randoms

    if getattr(target.device, "is_quadratic", False):
        return False
    S, A, d = ladder.size, ladder.moves_per_rung, target.dim
    cfg = dataclasses.replace(config, moves=A, leapfrogs=ladder.leapfrogs, burnin=0, record_q=False)
    Z = len(alive)
    zs = np.empty((S, A, Z, d))
    us = np.empty((S, A, Z))
    for j, k in enumerate(alive):
        for s in range(S):
            zk, uk = draw_move_randoms(np.random.default_rng(subs[k][s + 1]), A, d)
            zs[s, :, j] = zk
            us[s, :, j] = uk
    chains = DeviceChains(target.device, np.full(Z, float(ladder.taus[0])), cfg)
    chains.set_q(q[alive])
    taus = nat.dev_f64(np.asarray(ladder.taus, dtype=float))
    out = torch.full((Z, S), float("nan"), dtype=torch.float64, device="cuda")
    with np.errstate(divide="ignore"):
        lu = np.log(us)
    tz, tl = nat.dev_f64(zs), nat.dev_f64(lu)
    rc = chains.L.sgp_ladder_walk(target.device.handle, chains.ccfg, chains.cstate, int(S), nat.ptr(taus), int(A),
                                  int(bool(rung_average)), nat.ptr(tz), nat.ptr(tl), nat.ptr(out), nat.stream())
    if rc == nat.SGP_EINVAL:
        return False
    nat.check(rc, "sgp_ladder_walk")
    status = chains.status_host()
    vals = out.cpu().numpy()
    qf = chains.q.cpu().numpy()
    for j, k in enumerate(alive):
        if status[j] == nat.STATUS_FIRST_MOVE:
            errors[k] = "divergence on the first move; initial point or epsilon unusable"
        elif status[j] == nat.STATUS_CHAIN_START:
            errors[k] = "chain start failed: non-finite or invalid initial state"
        elif status[j] == nat.STATUS_JACOBI:
            raise JacobiError("cold resync failed to converge")
        elif status[j] != 0:
            raise ChainError(f"chain failed with status {status[j]}")
        else:
            values[k] = vals[j]
            q[k] = qf[j]
    for k in range(len(errors)):
        if errors[k] is not None:
            values[k] = np.nan
    return True


def _dist_info():
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist, dist.get_rank(), dist.get_world_size()
    except Exception:
        pass
    return None, 0, 1


# The ChainError texts a device chain can end with (sampler.py:349,389 wording); they travel
# through the all-gather as small integer codes so the warnings keep the reference's text.
CHAIN_ERROR_TEXTS = (
    None,
    "divergence on the first move; initial point or epsilon unusable",
    "chain start failed: non-finite or invalid initial state",
    "chain failed",
)


def _error_code(err):
    if err is None:
        return 0
    try:
        return CHAIN_ERROR_TEXTS.index(err)
    except ValueError:
        return len(CHAIN_ERROR_TEXTS) - 1


def gather_chain_values(local_ids, local_values, n_chains, n_rungs, local_errors=None, return_errors=False):
    """All-gather per-chain rung values to every rank; returns (Z, S) in chain order
    (and, with ``return_errors``, each chain's error text or None).

    One ``all_gather_into_tensor`` of a padded [ceil(Z/W), S+2] block per rank (column 0 =
    chain id + 1, 0 marks padding; column 1 = error code).  NCCL for GPU ranks, gloo on CPU.
    """
    import torch

    dist, rank, world = _dist_info()
    full = np.full((n_chains, n_rungs), np.nan)
    errors = [None] * n_chains
    local_errors = local_errors or [None] * len(local_ids)
    if dist is None or world == 1:
        for k, z in enumerate(local_ids):
            full[z] = local_values[k]
            errors[z] = local_errors[k]
        return (full, errors) if return_errors else full
    per = (n_chains + world - 1) // world
    block = np.zeros((per, n_rungs + 2))
    for k, z in enumerate(local_ids):
        block[k, 0] = z + 1
        block[k, 1] = _error_code(local_errors[k])
        block[k, 2:] = local_values[k]
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    src = torch.as_tensor(block, dtype=torch.float64, device=dev)
    out = torch.empty((world * per, n_rungs + 2), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(out, src)
    allb = out.cpu().numpy()
    for row in allb:
        if row[0] > 0:
            z = int(row[0]) - 1
            full[z] = row[2:]
            errors[z] = CHAIN_ERROR_TEXTS[int(row[1])]
    return (full, errors) if return_errors else full


def _aggregate(rung_values, chain_errors, ladder, warnings):
    """Per-chain trapezoid, cross-chain mean and stderr, rung means (evidence.py:246-274)."""
    n_chains = rung_values.shape[0]
    per_chain = []
    for z in range(n_chains):
        row = rung_values[z]
        if chain_errors[z] is not None or np.all(np.isnan(row)):
            warnings.append(f"chain {z} flagged: {chain_errors[z] or 'chain failed'}")
            per_chain.append(math.nan)
            continue
        per_chain.append(trapezoid(row, ladder.taus))
    finite = [v for v in per_chain if math.isfinite(v)]
    if not finite:
        raise ChainError("all evidence chains failed")
    bme_mean = float(np.mean(finite))
    if len(finite) > 1:
        bme_stderr = float(np.std(finite, ddof=1) / math.sqrt(len(finite)))
    else:
        bme_stderr = math.nan
        warnings.append("single surviving chain; standard error undefined")
    with np.errstate(invalid="ignore"):
        rung_means = np.nanmean(rung_values, axis=0)
    return EvidenceEstimate(bme_mean=bme_mean, bme_stderr=bme_stderr, per_chain=per_chain,
                            rung_means=[float(v) for v in rung_means], ladder=ladder,
                            warnings=warnings, rung_values=rung_values)


def evidence_sweep(models, data, ladder, config, *, rung_average=False, warmup_segment_moves=50,
                   warmup_max_segments=8, warmup_pvalue=0.05, spread_moves=10, initial=None, progress=None,
                   targets=None, ladder_runner=None, warmup_runner=None):
    """Thermodynamic integration for several competing models at once (the paper's model
    comparison), sharded over ``torch.distributed`` ranks by unit.

    The independent units are (model m, chain z) pairs, u = m * Z + z, placed on rank
    u mod W; rungs are never split.  Each model is seeded exactly as
    ``thermo_integrate(models[m], ...)`` with the same config, so every estimate equals the
    single-model, single-process one bit for bit at any world size.  Every rank recomputes
    the (deterministic) warm-up of every model; the only collective is one
    ``all_gather_into_tensor`` of [ceil(U/W), S+2] fp64 after the ladders (unit id, error
    code, rung values), NCCL on GPU ranks and gloo on CPU.  Returns one EvidenceEstimate per
    model.  ``targets`` (one per model), ``ladder_runner`` and ``warmup_runner`` substitute
    the targets and chain executors (tests inject the CPU oracle)."""
    if ladder_runner is None:
        if not hasattr(config, "epsilon") or not hasattr(config, "leapfrogs"):
            raise TypeError("config must be a ChainConfig")
        config = as_chain_config(config)
    n_models = len(models)
    Z, S = ladder.chains, ladder.size
    _, rank, world = _dist_info()
    units = [u for u in range(n_models * Z) if u % world == rank]
    by_model = {}
    for u in units:
        by_model.setdefault(u // Z, []).append(u % Z)
    warn = [[] for _ in range(n_models)]
    local_vals, local_errs = {}, {}
    for m in range(n_models):
        # every rank runs every model's warm-up (deterministic from the seed), so the warm-up
        # warnings agree everywhere without a second collective
        seed_root = config.seed if isinstance(config.seed, np.random.SeedSequence) \
            else np.random.SeedSequence(config.seed)
        seqs = seed_root.spawn(warmup_max_segments + Z)
        target = targets[m] if targets is not None else PosteriorTarget(models[m], data)
        q_warm = warm_up(target, config, seqs[:warmup_max_segments], warmup_segment_moves, warmup_pvalue,
                         warn[m], initial, runner=warmup_runner or run_chain)
        zs = by_model.get(m, [])
        if not zs:
            continue
        runner = ladder_runner or device_ladder_runner
        vals, errs = runner(target, [seqs[warmup_max_segments + z] for z in zs], q_warm, ladder, config,
                            rung_average, spread_moves)
        for k, z in enumerate(zs):
            local_vals[m * Z + z] = vals[k]
            local_errs[m * Z + z] = errs[k]
    ids = sorted(local_vals)
    allv, alle = gather_chain_values(ids, [local_vals[u] for u in ids], n_models * Z, S,
                                     [local_errs[u] for u in ids], return_errors=True)
    if progress is not None:
        progress(f"evidence: {n_models} model(s) x {Z} chains finished on {world} rank(s)")
    out = []
    for m in range(n_models):
        out.append(_aggregate(allv[m * Z:(m + 1) * Z], alle[m * Z:(m + 1) * Z], ladder, warn[m]))
    return out


def thermo_integrate(model, data, ladder, config, *, rung_average=False, warmup_segment_moves=50,
                     warmup_max_segments=8, warmup_pvalue=0.05, spread_moves=10, initial=None,
                     threads=1, progress=None, target=None, ladder_runner=None,
                     warmup_runner=None):
    """Estimate ln P(X) by thermodynamic integration (evidence.py:184-274).

    ``threads`` is accepted for API compatibility; chains run as one device
    batch per rank instead of a process pool.  ``ladder_runner`` /
    ``warmup_runner`` substitute the chain executors (tests inject the CPU
    oracle to exercise the multi-rank logic without a GPU).
    """
    return evidence_sweep([model], data, ladder, config, rung_average=rung_average,
                          warmup_segment_moves=warmup_segment_moves, warmup_max_segments=warmup_max_segments,
                          warmup_pvalue=warmup_pvalue, spread_moves=spread_moves, initial=initial,
                          progress=progress, targets=None if target is None else [target],
                          ladder_runner=ladder_runner, warmup_runner=warmup_runner)[0]


__all__ = ["TemperLadder", "default_ladder", "ti_variance", "EvidenceEstimate", "thermo_integrate", "evidence_sweep",
           "gather_chain_values", "device_ladder_runner", "warm_up", "JacobiError"]


# ---------------------------------------------------------------------------
# Laplace-grid evidence oracle (evidence.py:307-426)

@dataclasses.dataclass(frozen=True)
class GridSpec:
    """Midpoint-rule grid over the two Gaussian-kernel hyperparameters
    (reference evidence.py:307-323, same fields and defaults)."""

    c_max: float = 4.0
    c_mesh: float = 0.01
    sigma_max: float = 4.0
    sigma_mesh: float = 0.02
    pinned: tuple = ()  # ((name, value), ...) for hypers held fixed
    skip_tolerance: float = 0.01

    def centers(self):
        nc = int(round(self.c_max / self.c_mesh))
        ns = int(round(self.sigma_max / self.sigma_mesh))
        c = (np.arange(nc) + 0.5) * self.c_mesh
        s = (np.arange(ns) + 0.5) * self.sigma_mesh
        return c, s


def laplace_grid_nodes(model, data, grid_spec=None, *, gtol=1e-6, max_iters=200, memory=10, mode="reference"):
    """Per-node values of the grid oracle on the device, in the reference's
    serpentine node order: (values, status, iterations); status 0 ok,
    1 optimiser not converged, 2 Cholesky failed, 3 objective not finite at
    the start.  Validation as evidence.py:341-366.

    ``mode="reference"`` (default): every node starts from the optimum of the last node
    before it in serpentine order whose L-BFGS converged -- the reference's a_warm rule
    (evidence.py:374-399) -- evaluated concurrently from a first a = 0 pass, so failures are
    counted at the reference's starting points.  ``mode="robust"`` (opt-in, differs from the
    reference): a = 0 starts with warm-started retries of the failures, which leaves fewer
    failed nodes (profiles/r1_laplace_grid.md)."""
    if mode not in ("reference", "robust"):
        raise ValueError("mode must be 'reference' or 'robust'")
    from . import _native as nat

    from .rrgp import BlockLayout

    grid = GridSpec() if grid_spec is None else grid_spec
    pinned = dict(grid.pinned)
    hyper_index = BlockLayout.from_model(model).hyper_index
    if "c_g" not in hyper_index or "sigma_g" not in hyper_index:
        raise ValueError("grid marginalisation needs Gaussian-kernel hyperparameters")
    unpinned = [name for name in hyper_index if name not in ("c_g", "sigma_g", *pinned)]
    if unpinned:
        raise ValueError(f"hyperparameters {unpinned} must be pinned for a 2-d grid")
    transform = model.hyper_transform
    spec = nat.GridSpecC()
    spec.c_max, spec.c_mesh = float(grid.c_max), float(grid.c_mesh)
    spec.sigma_max, spec.sigma_mesh = float(grid.sigma_max), float(grid.sigma_mesh)
    k = 0
    for name, value in pinned.items():
        if value <= 0.0:
            raise ValueError(f"pinned hyperparameter {name} must be positive")
        spec.pinned_pos[k] = hyper_index[name]  # KeyError for a hyper the model does not sample, as the reference
        spec.pinned_value[k] = math.log(value) if transform == "log" else float(value)
        k += 1
    spec.n_pinned = k
    spec.gtol, spec.max_iters, spec.memory = float(gtol), int(max_iters), int(memory)
    spec.mode = nat.GRID_MODES[mode]
    c_centers, s_centers = grid.centers()
    n = c_centers.size * s_centers.size
    target = PosteriorTarget(model, data)
    values = np.empty(n)
    status = np.empty(n, dtype=np.int32)
    iters = np.empty(n, dtype=np.int32)
    L = nat.lib()
    nat.check(L.sgp_laplace_grid(target.device.handle, spec, int(n), values.ctypes.data, status.ctypes.data,
                                 iters.ctypes.data, nat.stream()), "sgp_laplace_grid")
    return values, status, iters


def laplace_grid_oracle(model, data, grid_spec=None, *, gtol=1e-6, max_iters=200, mode="reference"):
    """Grid-marginalised evidence over (c_g, sigma_g) with nested Laplace in
    the coefficients (reference evidence.py:330-426).  Nodes run concurrently
    on the device; with the default ``mode="reference"`` each starts from the
    reference's serpentine a_warm (laplace_grid_nodes), so the set of failed
    nodes -- and the "untrustworthy" RuntimeError past ``skip_tolerance`` --
    follows the reference.  Same errors: ValueError for unsuitable models /
    pinned values or a non-finite starting objective, RuntimeError when more
    than ``skip_tolerance`` of the nodes fail."""
    grid = GridSpec() if grid_spec is None else grid_spec
    values, status, _ = laplace_grid_nodes(model, data, grid, gtol=gtol, max_iters=max_iters, mode=mode)
    if np.any(status == 3):
        raise ValueError("objective is not finite at the starting point")
    skipped = int(np.count_nonzero(status))
    total = int(status.size)
    if skipped > grid.skip_tolerance * total:
        raise RuntimeError(f"grid oracle skipped {skipped}/{total} nodes; result untrustworthy")
    v = values[status == 0]
    peak = float(np.max(v))
    return peak + math.log(float(np.sum(np.exp(v - peak))))


LAPLACE_ZETA = 1e-13  # evidence.py:31


def laplace_full(model, data, *, initial=None, gtol=1e-6, max_iters=500, target=None):
    """Quadratic approximation of the evidence at the posterior mode
    (reference evidence.py:277-304): ln P(X) ~ -U(q*) + (d/2) ln 2 pi - 0.5 ln|H(q*)|,
    the determinant from the same cold Jacobi eigendecomposition.  The mode
    search (the reference's L-BFGS) and the decomposition run in one CTA on
    the device.  Same errors as the reference."""
    from . import _native as nat

    if target is None:
        target = PosteriorTarget(model, data)
    x0 = target.initial_point() if initial is None else np.asarray(initial, dtype=float)
    x0 = np.ascontiguousarray(x0, dtype=float)
    out = np.zeros(4)
    st = ctypes.c_int(0)
    it = ctypes.c_int(0)
    nat.check(nat.lib().sgp_laplace_full(target.device.handle, float(target.tau), x0.ctypes.data, float(gtol),
                                         int(max_iters), LAPLACE_ZETA, 30, out.ctypes.data, ctypes.byref(st),
                                         ctypes.byref(it), nat.stream()), "sgp_laplace_full")
    if st.value == 3:
        raise ValueError("objective is not finite at the starting point")
    if st.value == 1:
        raise RuntimeError("Laplace mode search did not reach gradient tolerance")
    if st.value == 4:
        raise JacobiError("Jacobi did not converge within the sweep cap")
    if st.value == 2:
        raise RuntimeError("Laplace invalid (singular/indefinite posterior)")
    return float(out[0])
