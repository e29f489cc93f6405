"""RMHMC with the SoftAbs metric, generalized leapfrog on the B200.

Drop-in for ``softabs_gp.sampler`` (/root/reference/pkg/src/softabs_gp/
sampler.py).  ``run_chain`` keeps the reference's RNG contract (numpy PCG64,
per move: d standard normals, then one uniform, sampler.py:339/360/377) by
drawing those numbers on the host in the same order and shipping them to the
device; the whole move loop -- momentum, C generalized leapfrogs with both
implicit fixed points, Hamiltonians, Metropolis test, cold resync on
rejection -- then runs inside one kernel launch per chain batch
(csrc/sgp.cu: k_run_moves).  ``run_chains`` batches many independent chains
(one CTA each) into the same launch.
"""

from __future__ import annotations

import dataclasses
import json
import math

import numpy as np

from . import _native as nat
from .metric import JacobiError, MetricState, contraction_matrix, metric_quadratic, softabs
from .posterior import DivergenceError, DomainError, PosteriorTarget, raise_status

LN_2PI = math.log(2.0 * math.pi)
METRIC_MODES = ("softabs-dynamic", "softabs-static", "euclidean")
WARM_ORDERS = ("parallel", "cyclic", "refine")
COLD_ORDERS = ("parallel", "cyclic", "dc")
_DIVERGENT = (DivergenceError, DomainError, JacobiError, FloatingPointError)


class ChainError(RuntimeError):
    """A chain could not start or diverged on its first move (sampler.py:45)."""


@dataclasses.dataclass(frozen=True)
class ChainConfig:
    """Chain settings (sampler.py:49-83), plus two solver choices.

    ``warm_order``: the warm eigensolver (dynamic_eigendecompose).  "cyclic" (default)
    replays the reference's pivot order and keeps trajectories identical to the reference;
    "parallel" (round-robin order; block Jacobi at d > 256) and "refine" (d > 256: GEMM
    eigenvector refinement with a block-Jacobi fallback; "parallel" below) are faster and
    meet the same convergence test, but the dynamics being chaotic they are only
    statistically equivalent after a few moves.

    ``cold_order``: the cold eigensolver (static_eigendecompose: chain start, rejections,
    rung starts).  "cyclic" (default) is the reference's order, bit-identical at every d;
    "parallel" selects the block Jacobi at d > 256; "dc" Householder tridiagonalisation +
    divide and conquer (large-d path; 30 ms at d = 2083 against 21 s for the reference order).

    ``path``: "auto" (default) runs one CTA per chain for d <= 256 (many chains at once) and
    the whole-GPU large path above; "latency" serves few chains fast: at d <= 64 one 256-thread
    CTA per chain (C1: 2.0 ms per leapfrog cyclic, 1.1 parallel), above it every chain's
    leapfrogs on the whole GPU (d = 163: 24 ms per leapfrog in the cyclic order vs 78 ms in one
    CTA, 3 ms with warm_order="refine"), chains one after the other.  Both agree with the
    reference; "auto" keeps a chain's bits independent of its batch."""

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
    warm_order: str = "cyclic"
    cold_order: str = "cyclic"
    path: str = "auto"

    def __post_init__(self):
        if self.epsilon <= 0.0:
            raise ValueError("epsilon must be positive")
        if self.leapfrogs < 1:
            raise ValueError("leapfrogs must be at least 1")
        if self.moves < 1:
            raise ValueError("moves must be at least 1")
        if not 0 <= self.burnin <= self.moves:
            raise ValueError("burnin must lie in [0, moves]")
        if self.kappa <= 0.0 or self.zeta <= 0.0:
            raise ValueError("kappa and zeta must be positive")
        if self.fp_max_iters < 1:
            raise ValueError("fp_max_iters must be at least 1")
        if self.fp_max_iters > 32:
            raise ValueError("fp_max_iters must be at most 32 on the device")
        if self.fp_tol <= 0.0:
            raise ValueError("fp_tol must be positive")
        if self.metric not in METRIC_MODES:
            raise ValueError(f"metric must be one of {METRIC_MODES}")
        if self.warm_order not in WARM_ORDERS:
            raise ValueError(f"warm_order must be one of {WARM_ORDERS}")
        if self.cold_order not in COLD_ORDERS:
            raise ValueError(f"cold_order must be one of {COLD_ORDERS}")
        if self.path not in nat.PATH_CODES:
            raise ValueError(f"path must be one of {tuple(nat.PATH_CODES)}")

    def to_c(self):
        c = nat.ChainConfigC()
        c.epsilon, c.leapfrogs, c.kappa, c.zeta = self.epsilon, self.leapfrogs, self.kappa, self.zeta
        c.fp_max_iters, c.fp_tol = self.fp_max_iters, self.fp_tol
        c.gs_interval, c.sweep_cap = int(self.gs_interval or 0), self.sweep_cap
        c.metric = nat.METRIC_CODES[self.metric]
        c.warm_order = nat.ORDER_CODES[self.warm_order]
        c.cold_order = nat.ORDER_CODES[self.cold_order]
        c.path = nat.PATH_CODES[self.path]
        return c


def as_chain_config(config) -> ChainConfig:
    """This package's ChainConfig from any object carrying the reference's ChainConfig
    fields by name (sampler.py:53-65), e.g. ``softabs_gp.sampler.ChainConfig`` handed over by
    reference code through the drop-in shim.  Fields the object lacks keep their defaults, so
    a reference config runs with ``warm_order = cold_order = "cyclic"`` (the reference's
    order)."""
    if isinstance(config, ChainConfig):
        return config
    kw = {f.name: getattr(config, f.name) for f in dataclasses.fields(ChainConfig) if hasattr(config, f.name)}
    return ChainConfig(**kw)


def as_device_target(target):
    """A libsgp-backed target for ``target``: returned as is when it already is one;
    a reference ``PosteriorTarget`` (model, data, tau) or the reference's constant-Hessian
    test fake (precision, mean, loglik_const, tau) is rebuilt on the shared device model."""
    if hasattr(target, "device"):
        return target
    if hasattr(target, "model") and hasattr(target, "data"):
        return PosteriorTarget(target.model, target.data, float(getattr(target, "tau", 1.0)))
    if hasattr(target, "precision"):
        from .posterior import QuadraticTarget

        return QuadraticTarget(target.precision, getattr(target, "mean", None),
                               getattr(target, "loglik_const", 0.0), float(getattr(target, "tau", 1.0)))
    raise TypeError(f"cannot run {type(target).__name__} on the device: it is neither a "
                    "PosteriorTarget nor a constant-Hessian target")


@dataclasses.dataclass
class ChainRecord:
    move: int
    logpost: float
    h_before: float
    h_after: float | None
    accept: bool
    divergent: bool
    sweeps_mean: float
    wall_ms: float
    q: np.ndarray | None = None
    uniform: float | None = None


def record_to_dict(record):
    out = {
        "move": int(record.move),
        "logpost": float(record.logpost),
        "h_before": float(record.h_before),
        "h_after": None if record.h_after is None else float(record.h_after),
        "accept": bool(record.accept),
        "divergent": bool(record.divergent),
        "sweeps_mean": float(record.sweeps_mean),
        "wall_ms": float(record.wall_ms),
    }
    if record.q is not None:
        out["q"] = [float(v) for v in record.q]
    return out


def write_jsonl(records, path):
    with open(path, "w", encoding="utf-8") as fh:
        for record in records:
            fh.write(json.dumps(record_to_dict(record)) + "\n")


def read_jsonl(path):
    records = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            if not line.strip():
                continue
            try:
                raw = json.loads(line)
            except json.JSONDecodeError as exc:
                raise ValueError(f"{path}:{lineno}: invalid JSON ({exc})") from None
            try:
                records.append(ChainRecord(
                    move=int(raw["move"]), logpost=float(raw["logpost"]),
                    h_before=float(raw["h_before"]),
                    h_after=None if raw["h_after"] is None else float(raw["h_after"]),
                    accept=bool(raw["accept"]), divergent=bool(raw["divergent"]),
                    sweeps_mean=float(raw["sweeps_mean"]), wall_ms=float(raw["wall_ms"]),
                    q=np.asarray(raw["q"], dtype=float) if "q" in raw else None))
            except (KeyError, TypeError, ValueError) as exc:
                raise ValueError(f"{path}:{lineno}: malformed record ({exc})") from None
    return records


@dataclasses.dataclass
class ChainResult:
    records: list
    q_final: np.ndarray
    accept_count: int
    divergence_count: int
    config: ChainConfig

    @property
    def acceptance_rate(self):
        return self.accept_count / max(1, len(self.records))

    @property
    def logpost(self):
        return np.array([r.logpost for r in self.records])

    def kept_logpost(self):
        return self.logpost[self.config.burnin:]

    def sample_matrix(self):
        rows = [r.q for r in self.records if r.q is not None]
        if not rows:
            raise ValueError("chain was run without record_q")
        return np.vstack(rows)


# ---------------------------------------------------------------------------
# device chain batches


class DeviceChains:
    """Z chains of one device model: state tensors in HBM + the C-ABI calls."""

    def __init__(self, device, taus, config: ChainConfig):
        import torch

        self.L = nat.lib()
        self.device = device
        self.config = config
        taus = np.asarray(taus, dtype=float).reshape(-1)
        Z, d = taus.shape[0], device.dim
        self.Z, self.d = Z, d
        self.q = torch.zeros((Z, d), dtype=torch.float64, device="cuda")
        self.psi = torch.zeros((Z, d, d), dtype=torch.float64, device="cuda")
        self.lam = torch.zeros((Z, d), dtype=torch.float64, device="cuda")
        self.tau = nat.dev_f64(taus)
        self.since = nat.zeros_i32(Z)
        self.status = nat.zeros_i32(Z)
        self.scratch = nat.empty_f64(Z * device.scratch_per_chain)
        self.cstate = nat.ChainState(Z, self.q.data_ptr(), self.psi.data_ptr(), self.lam.data_ptr(),
                                     self.tau.data_ptr(), self.since.data_ptr(), self.status.data_ptr(),
                                     self.scratch.data_ptr())
        self.ccfg = config.to_c()
        self._rec = None

    def set_q(self, q):
        self.q.copy_(nat.dev_f64(np.asarray(q, dtype=float).reshape(self.Z, self.d)))

    def init(self):
        """Cold initial frame at the current q (sampler.py:322-328)."""
        nat.check(self.L.sgp_chain_init(self.device.handle, self.ccfg, self.cstate, nat.stream()),
                  "sgp_chain_init")

    def records_buffers(self, moves, record_q):
        import torch

        key = (moves, bool(record_q))
        if self._rec is None or self._rec[0] != key:
            f = lambda: torch.empty((moves, self.Z), dtype=torch.float64, device="cuda")  # noqa: E731
            u8 = lambda: torch.empty((moves, self.Z), dtype=torch.uint8, device="cuda")  # noqa: E731
            bufs = {"logpost": f(), "h_before": f(), "h_after": f(), "sweeps_mean": f(),
                    "wall_ms": f(), "accept": u8(), "divergent": u8(),
                    "q": torch.empty((moves, self.Z, self.d), dtype=torch.float64, device="cuda")
                    if record_q else None}
            c = nat.MoveRecords(*(None if bufs[k] is None else bufs[k].data_ptr() for k in
                                  ("logpost", "h_before", "h_after", "sweeps_mean", "wall_ms",
                                   "accept", "divergent", "q")))
            self._rec = (key, bufs, c)
        return self._rec[1], self._rec[2]

    def run(self, moves, z, logu, move_offset=0, record_q=False):
        """Launch the on-device move loop.  z: (moves, Z, d), logu: (moves, Z)
        (host arrays or CUDA tensors).  Returns the device record buffers."""
        import torch

        tz = z if isinstance(z, torch.Tensor) else nat.dev_f64(z)
        tl = logu if isinstance(logu, torch.Tensor) else nat.dev_f64(logu)
        bufs, crec = self.records_buffers(moves, record_q)
        nat.check(self.L.sgp_run_moves(self.device.handle, self.ccfg, self.cstate, int(moves),
                                       int(move_offset), nat.ptr(tz), nat.ptr(tl), crec, nat.stream()),
                  "sgp_run_moves")
        return bufs

    def status_host(self):
        import torch

        torch.cuda.synchronize()
        return self.status.cpu().numpy()


def draw_move_randoms(rng, moves, d):
    """The reference's per-move draws: d normals then one uniform (sampler.py:360,377)."""
    z = np.empty((moves, d))
    u = np.empty(moves)
    for m in range(moves):
        z[m] = rng.standard_normal(d)
        u[m] = rng.uniform()
    return z, u


def _log_uniform(u):
    with np.errstate(divide="ignore"):
        return np.log(u)


def _records_from(bufs, z_idx, moves, uniforms, record_q):
    h = {k: (None if v is None else v.cpu().numpy()) for k, v in bufs.items()}
    out = []
    for m in range(moves):
        ha = float(h["h_after"][m, z_idx])
        div = bool(h["divergent"][m, z_idx])
        out.append(ChainRecord(
            move=m, logpost=float(h["logpost"][m, z_idx]), h_before=float(h["h_before"][m, z_idx]),
            h_after=None if div else ha, accept=bool(h["accept"][m, z_idx]), divergent=div,
            sweeps_mean=float(h["sweeps_mean"][m, z_idx]), wall_ms=float(h["wall_ms"][m, z_idx]),
            q=h["q"][m, z_idx].copy() if record_q else None, uniform=float(uniforms[m])))
    return out


def run_chains(target, config: ChainConfig, seeds, initials=None, taus=None):
    """Run len(seeds) independent chains of ``target``'s model in one batch.

    Each chain follows ``run_chain(target.at_temperature(taus[z]),
    replace(config, seed=seeds[z]), initial=initials[z])`` exactly; the result
    list holds a ChainResult or the ChainError/JacobiError that chain raised.
    """
    import torch

    target = as_device_target(target)
    config = as_chain_config(config)
    Z = len(seeds)
    d = target.dim
    taus = np.full(Z, target.tau) if taus is None else np.asarray(taus, dtype=float)
    if initials is None:
        initials = np.tile(target.initial_point(), (Z, 1))
    initials = np.asarray(initials, dtype=float).reshape(Z, d)
    moves = config.moves
    zs = np.empty((moves, Z, d))
    us = np.empty((moves, Z))
    for k, seed in enumerate(seeds):
        rng = np.random.default_rng(seed)
        zk, uk = draw_move_randoms(rng, moves, d)
        zs[:, k] = zk
        us[:, k] = uk
    chains = DeviceChains(target.device, taus, config)
    chains.set_q(initials)
    chains.init()
    start = chains.status_host()
    bufs = chains.run(moves, zs, _log_uniform(us), 0, config.record_q)
    status = chains.status_host()
    q_final = chains.q.cpu().numpy()
    results = []
    for k in range(Z):
        if start[k] != 0:
            results.append(ChainError("chain start failed: non-finite or invalid initial state"))
            continue
        if status[k] == nat.STATUS_FIRST_MOVE:
            results.append(ChainError("divergence on the first move; initial point or epsilon unusable"))
            continue
        if status[k] == nat.STATUS_JACOBI:
            results.append(JacobiError("cold resync failed to converge"))
            continue
        if status[k] != 0:
            results.append(DivergenceError(f"chain failed with status {status[k]}"))
            continue
        recs = _records_from(bufs, k, moves, us[:, k], config.record_q)
        results.append(ChainResult(records=recs, q_final=q_final[k].copy(),
                                   accept_count=sum(r.accept for r in recs),
                                   divergence_count=sum(r.divergent for r in recs), config=config))
    torch.cuda.synchronize()
    return results


def run_chain(target, config, *, initial=None):
    """One MCMC chain (sampler.py:331-418), move loop on the device."""
    target = as_device_target(target)
    config = as_chain_config(config)
    q0 = np.asarray(target.initial_point() if initial is None else initial, dtype=float).copy()
    if q0.shape != (target.dim,):
        raise ValueError("initial point has wrong dimension")
    res = run_chains(target, config, [config.seed], q0[None, :])[0]
    if isinstance(res, Exception):
        raise res
    return res


def rmhmc_run(model, data, config, *, initial=None):
    return run_chain(PosteriorTarget(model, data), config, initial=initial)


def euclidean_hmc_run(model, data, config, *, initial=None):
    config = dataclasses.replace(config, metric="euclidean")
    return run_chain(PosteriorTarget(model, data), config, initial=initial)


# ---------------------------------------------------------------------------
# single-step API


def _frame_kinetic(metric, p):
    if metric is None:
        return 0.5 * float(p @ p) + 0.5 * p.shape[0] * LN_2PI
    return 0.5 * metric_quadratic(metric, p) + 0.5 * (metric.dim * LN_2PI + metric.logdet)


def hamiltonian(q, p, metric, target):
    """H = U + 0.5 ln((2 pi)^d |G|) + 0.5 p^T G^-1 p (sampler.py:172-178)."""
    state = target.at(np.asarray(q, dtype=float))
    return state.potential() + _frame_kinetic(metric, np.asarray(p, dtype=float))


def grad_q_hamiltonian(q, p, metric, target, cache=None):
    """grad U + 0.5 tr((W2 - W1) dH) (sampler.py:181-194)."""
    state = target.at(np.asarray(q, dtype=float))
    if metric is None:
        return state.gradient()
    if cache is not None:
        w = cache.w2 - cache.w1
    else:
        w = contraction_matrix(metric, np.asarray(p, dtype=float))
    return state.gradient() + 0.5 * state.trace_single(w)


def leapfrog_step(q, p, metric, target, config):
    """One generalized leapfrog from (q, p) (sampler.py:280-292), on the device."""
    import torch

    target = as_device_target(target)
    config = as_chain_config(config)
    q = np.asarray(q, dtype=float)
    p = np.asarray(p, dtype=float)
    d = target.dim
    if metric is not None and config.metric == "euclidean":
        metric = None
    cfg = config
    if metric is None:
        cfg = dataclasses.replace(config, metric="euclidean")
    chains = DeviceChains(target.device, [target.tau], cfg)
    chains.set_q(q[None])
    if metric is not None:
        chains.psi.copy_(nat.dev_f64(metric.vectors)[None])
        chains.lam.copy_(nat.dev_f64(metric.eigenvalues)[None])
        chains.since.fill_(int(metric.steps_since_refresh))
    tp = nat.dev_f64(p[None])
    fpp, fpq = nat.zeros_i32(1), nat.zeros_i32(1)
    sw = nat.zeros_i32(1, cfg.fp_max_iters)
    diag_c = nat.LeapfrogDiag(fpp.data_ptr(), fpq.data_ptr(), sw.data_ptr())
    nat.check(chains.L.sgp_leapfrog(target.device.handle, chains.ccfg, chains.cstate, nat.ptr(tp), diag_c,
                                    nat.stream()), "sgp_leapfrog")
    torch.cuda.synchronize()
    status = int(chains.status.cpu()[0])
    raise_status(status, "leapfrog")
    q_new = chains.q.cpu().numpy()[0]
    p_new = tp.cpu().numpy()[0]
    diag = {"sweeps": [], "fp_p_iters": [], "fp_q_iters": []}
    if metric is None:
        return q_new, p_new, None, diag
    swh = [int(v) for v in sw.cpu().numpy()[0] if v >= 0]
    diag["sweeps"] = swh
    diag["fp_p_iters"] = [int(fpp.cpu()[0])]
    diag["fp_q_iters"] = [int(fpq.cpu()[0])]
    lam = chains.lam.cpu().numpy()[0]
    psi = chains.psi.cpu().numpy()[0]
    g = softabs(lam, metric.kappa)
    new_metric = MetricState(eigenvalues=lam, vectors=psi, softabs_values=g,
                             logdet=float(np.sum(np.log(g))), kappa=metric.kappa,
                             sweep_count=swh[-1] if swh else 0,
                             steps_since_refresh=int(chains.since.cpu()[0]))
    return q_new, p_new, new_metric, diag


# ---------------------------------------------------------------------------
# stationarity test (sampler.py:432-487), host-side statistics


def _pooled_ranks(values):
    v = np.asarray(values, dtype=float)
    n = v.shape[0]
    order = np.argsort(v, kind="mergesort")
    ranks = np.empty(n)
    ties = []
    i = 0
    while i < n:
        j = i
        while j + 1 < n and v[order[j + 1]] == v[order[i]]:
            j += 1
        ranks[order[i:j + 1]] = 0.5 * (i + j) + 1.0
        ties.append(j - i + 1)
        i = j + 1
    return ranks, ties


def rank_sum_test(x, y):
    """Two-sided Wilcoxon rank-sum, tie-corrected normal approximation with a
    0.5 continuity correction."""
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    if x.ndim != 1 or y.ndim != 1 or x.shape[0] == 0 or y.shape[0] == 0:
        raise ValueError("rank_sum_test needs two non-empty 1-d samples")
    n1, n2 = x.shape[0], y.shape[0]
    n = n1 + n2
    ranks, ties = _pooled_ranks(np.concatenate([x, y]))
    w = float(np.sum(ranks[:n1]))
    variance = n1 * n2 / 12.0 * ((n + 1) - float(sum(t ** 3 - t for t in ties)) / (n * (n - 1)))
    if variance <= 0.0:
        return 0.0, 1.0
    diff = w - n1 * (n + 1) / 2.0
    z = 0.0 if abs(diff) <= 0.5 else (diff - math.copysign(0.5, diff)) / math.sqrt(variance)
    return float(z), float(math.erfc(abs(z) / math.sqrt(2.0)))


def wilcoxon_split_half(values):
    v = np.asarray(values, dtype=float)
    if v.ndim != 1 or v.shape[0] < 10:
        raise ValueError("split-half test needs at least 10 values")
    half = v.shape[0] // 2
    return rank_sum_test(v[:half], v[half:])
