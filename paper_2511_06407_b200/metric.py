"""SoftAbs metric G = Psi diag(sqrt(kappa^2 + lambda^2)) Psi^T on the B200.

Drop-in for ``softabs_gp.metric`` (/root/reference/pkg/src/softabs_gp/
metric.py).  Eigendecompositions run in libsgp: the cold one replays the
reference's cyclic-by-row pivot order without FMA (bit-compatible with
``_jacobi.jacobi_sweeps`` on identical input); the warm one diagonalises
Psi^T H Psi in the previous basis, by default with the round-robin parallel
order (d/2 concurrent rotations) or, on request, the reference
order.
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import _native as nat

EQUAL_EIGENVALUE_FACTOR = 1e-10
DEFAULT_SWEEP_CAP = 30
DEFAULT_GS_INTERVAL = 10
DEFAULT_WARM_ORDER = "cyclic"


class JacobiError(RuntimeError):
    """Eigendecomposition failed to converge within the sweep budget (metric.py:28)."""


def softabs(eigenvalues, kappa):
    """sqrt(kappa^2 + lambda^2) (metric.py:32-37)."""
    if kappa <= 0.0:
        raise ValueError("kappa must be positive")
    lam = np.asarray(eigenvalues, dtype=float)
    return np.sqrt(kappa * kappa + lam * lam)


def softabs_deriv(eigenvalues, kappa):
    lam = np.asarray(eigenvalues, dtype=float)
    return lam / softabs(lam, kappa)


@dataclasses.dataclass(frozen=True)
class MetricState:
    """Eigensystem of a Hessian with its smoothed spectrum (metric.py:62-83)."""

    eigenvalues: np.ndarray
    vectors: np.ndarray
    softabs_values: np.ndarray
    logdet: float
    kappa: float
    sweep_count: int
    steps_since_refresh: int = 0

    def __post_init__(self):
        d = self.eigenvalues.shape[0]
        if self.vectors.shape != (d, d):
            raise ValueError("eigenvector matrix shape mismatch")
        if self.softabs_values.shape != (d,):
            raise ValueError("softabs value shape mismatch")

    @property
    def dim(self):
        return self.eigenvalues.shape[0]


@dataclasses.dataclass(frozen=True)
class BetancourtCache:
    t: np.ndarray
    b: np.ndarray
    r: np.ndarray
    w1: np.ndarray
    w2: np.ndarray


def _sync_numpy(*tensors):
    import torch

    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in tensors]


def t_matrix(eigenvalues, kappa):
    """Divided differences T_jl (metric.py:46-59), on the device."""
    L = nat.lib()
    lam = np.asarray(eigenvalues, dtype=float)
    d = lam.shape[0]
    tl, out = nat.dev_f64(lam), nat.empty_f64(d, d)
    nat.check(L.sgp_t_matrix(1, d, nat.ptr(tl), float(kappa), nat.ptr(out), nat.stream()), "sgp_t_matrix")
    return _sync_numpy(out)[0]


def _state(lam, psi, kappa, sweeps, since):
    g = softabs(lam, kappa)
    return MetricState(eigenvalues=lam, vectors=psi, softabs_values=g,
                       logdet=float(np.sum(np.log(g))), kappa=kappa, sweep_count=int(sweeps),
                       steps_since_refresh=int(since))


def static_eigendecompose(hessian, zeta, sweep_cap=DEFAULT_SWEEP_CAP):
    """Cold cyclic Jacobi from the identity (metric.py:112-127)."""
    h = np.asarray(hessian, dtype=float)
    if h.ndim != 2 or h.shape[0] != h.shape[1]:
        raise ValueError("hessian must be square")
    if zeta <= 0.0:
        raise ValueError("zeta must be positive")
    L = nat.lib()
    d = h.shape[0]
    th = nat.dev_f64(h)
    lam, psi, sw = nat.empty_f64(d), nat.empty_f64(d, d), nat.zeros_i32(1)
    nat.check(L.sgp_eigh_cold(1, d, nat.ptr(th), float(zeta), int(sweep_cap), nat.ptr(lam), nat.ptr(psi),
                              nat.ptr(sw), nat.stream()), "sgp_eigh_cold")
    lam, psi, sw = _sync_numpy(lam, psi, sw)
    if sw[0] < 0:
        raise JacobiError(f"Jacobi failed to reach off-norm tolerance in {sweep_cap} sweeps")
    return lam, psi, int(sw[0])


def eigh_dc(hessian):
    """Eigendecomposition of the symmetric part of ``hessian`` by blocked Householder
    tridiagonalisation + divide and conquer on the device (sgp_dc.cuh; north star (3)).

    Returns (eigenvalues ascending, eigenvectors as columns).  The fast cold decomposition for
    latent-function-sized d; unlike static_eigendecompose it does not follow the reference's
    Jacobi order (metric.py:112-127), only its result up to eigenpair order and signs."""
    h = np.asarray(hessian, dtype=float)
    if h.ndim != 2 or h.shape[0] != h.shape[1]:
        raise ValueError("hessian must be square")
    L = nat.lib()
    d = h.shape[0]
    th = nat.dev_f64(h)
    lam, psi = nat.empty_f64(d), nat.empty_f64(d, d)
    nat.check(L.sgp_eigh_dc(1, d, nat.ptr(th), nat.ptr(lam), nat.ptr(psi), nat.stream()), "sgp_eigh_dc")
    return _sync_numpy(lam, psi)


def metric_from_hessian(hessian, kappa, zeta, sweep_cap=DEFAULT_SWEEP_CAP):
    """MetricState from a cold decomposition (metric.py:130-142)."""
    lam, psi, sweeps = static_eigendecompose(hessian, zeta, sweep_cap)
    return _state(lam, psi, kappa, sweeps, 0)


def dynamic_eigendecompose(hessian, previous, zeta, sweep_cap=DEFAULT_SWEEP_CAP,
                           gs_interval=DEFAULT_GS_INTERVAL, order=DEFAULT_WARM_ORDER):
    """Warm decomposition in ``previous``'s basis (metric.py:145-185)."""
    h = np.asarray(hessian, dtype=float)
    d = previous.dim
    if h.shape != (d, d):
        raise ValueError("hessian shape does not match metric")
    L = nat.lib()
    th, tp = nat.dev_f64(h), nat.dev_f64(previous.vectors)
    ts = nat.zeros_i32(1)
    ts.fill_(int(previous.steps_since_refresh))
    lam, psi = nat.empty_f64(d), nat.empty_f64(d, d)
    since, sw = nat.zeros_i32(1), nat.zeros_i32(1)
    nat.check(L.sgp_eigh_warm(1, d, nat.ptr(th), nat.ptr(tp), nat.ptr(ts), int(gs_interval or 0),
                              float(zeta), int(sweep_cap), nat.ORDER_CODES[order], nat.ptr(lam),
                              nat.ptr(psi), nat.ptr(since), nat.ptr(sw), nat.stream()),
              "sgp_eigh_warm")
    lam, psi, since, sw = _sync_numpy(lam, psi, since, sw)
    if sw[0] < 0:
        raise JacobiError(f"Jacobi failed to reach off-norm tolerance in {sweep_cap} sweeps")
    return _state(lam, psi, previous.kappa, sw[0], since[0])


def _metric_w(metric, p, which):
    L = nat.lib()
    d = metric.dim
    tpsi, tlam = nat.dev_f64(metric.vectors), nat.dev_f64(metric.eigenvalues)
    tp = None if p is None else nat.dev_f64(p)
    out = nat.empty_f64(d, d)
    nat.check(L.sgp_metric_w(1, d, nat.ptr(tpsi), nat.ptr(tlam), float(metric.kappa), nat.ptr(tp), which,
                             nat.ptr(out), nat.stream()), "sgp_metric_w")
    return _sync_numpy(out)[0]


def w1_matrix(metric, momentum, t=None):
    """Psi ((b b^T) o T) Psi^T, b = Psi^T p / g (metric.py:188-198)."""
    return _metric_w(metric, np.asarray(momentum, dtype=float), nat.W_W1)


def w2_matrix(metric):
    """Psi diag(g'/g) Psi^T (metric.py:201-204)."""
    return _metric_w(metric, None, nat.W_W2)


def contraction_matrix(metric, momentum):
    """W2 - W1 in one pass (what the leapfrog contracts against)."""
    return _metric_w(metric, np.asarray(momentum, dtype=float), nat.W_W2_MINUS_W1)


def _apply(metric, v, mode):
    L = nat.lib()
    d = metric.dim
    tpsi, tlam, tv = nat.dev_f64(metric.vectors), nat.dev_f64(metric.eigenvalues), nat.dev_f64(v)
    out = nat.empty_f64(d)
    nat.check(L.sgp_metric_apply(1, d, nat.ptr(tpsi), nat.ptr(tlam), float(metric.kappa), nat.ptr(tv), mode,
                                 nat.ptr(out), nat.stream()), "sgp_metric_apply")
    return _sync_numpy(out)[0]


def build_cache(metric, momentum):
    p = np.asarray(momentum, dtype=float)
    g = metric.softabs_values
    b = (metric.vectors.T @ p) / g
    return BetancourtCache(t=t_matrix(metric.eigenvalues, metric.kappa), b=b, r=1.0 / g,
                           w1=w1_matrix(metric, p), w2=w2_matrix(metric))


def metric_apply(metric, vector):
    return _apply(metric, np.asarray(vector, dtype=float), 1)


def metric_apply_inverse(metric, vector):
    return _apply(metric, np.asarray(vector, dtype=float), 0)


def metric_quadratic(metric, momentum):
    L = nat.lib()
    d = metric.dim
    tpsi, tlam = nat.dev_f64(metric.vectors), nat.dev_f64(metric.eigenvalues)
    tp = nat.dev_f64(np.asarray(momentum, dtype=float))
    quad, ld = nat.empty_f64(1), nat.empty_f64(1)
    nat.check(L.sgp_metric_scalars(1, d, nat.ptr(tpsi), nat.ptr(tlam), float(metric.kappa), nat.ptr(tp),
                                   nat.ptr(quad), nat.ptr(ld), nat.stream()), "sgp_metric_scalars")
    return float(_sync_numpy(quad)[0][0])


def metric_logdet(metric):
    return metric.logdet


def sample_momentum(metric, rng):
    """p ~ N(0, G): z drawn on the host in the reference's order, p = Psi (sqrt(g) o z)."""
    z = rng.standard_normal(metric.dim)
    return _apply(metric, z, 2)


def reconstruct(metric):
    psi = metric.vectors
    return (psi * metric.eigenvalues[None, :]) @ psi.T


def log_2pi_volume(metric):
    return 0.5 * (metric.dim * math.log(2.0 * math.pi) + metric.logdet)
