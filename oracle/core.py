"""TEST INFRASTRUCTURE ONLY — CPU oracle for the SoftAbs RMHMC hot path.

A compact numpy restatement of the reference algorithm.  Every function names
the reference lines it follows (paths relative to
/root/reference/pkg/src/softabs_gp/).  The eigensolver kernels are the C
restatement in ``oracle/jacobi.c`` (bit-exact with the reference's Numba code
on identical input).  The product package never imports this module.
"""

from __future__ import annotations

import ctypes
import dataclasses
import math
import os
import subprocess

import numpy as np

LN_2PI = math.log(2.0 * math.pi)
EQUAL_EIGENVALUE_FACTOR = 1e-10  # metric.py:22


class ODivergence(FloatingPointError):
    """posterior.py:49 DivergenceError."""


class ODomain(ValueError):
    """posterior.py:45 DomainError."""


class OJacobi(RuntimeError):
    """metric.py:28 JacobiError."""


class OChainError(RuntimeError):
    """sampler.py:45 ChainError."""


_DIVERGENT = (ODivergence, ODomain, OJacobi, FloatingPointError)

# ---------------------------------------------------------------------------
# native Jacobi (oracle/jacobi.c)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_jacobi.so")
_lib = None


def build_native():
    """Compile oracle/jacobi.c (called by __graft_entry__.build and tests)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _native():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build_native()
        lib = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_jacobi_sweeps.restype = ctypes.c_long
        lib.oracle_jacobi_sweeps.argtypes = [dp, dp, ctypes.c_long, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_long]
        lib.oracle_jacobi_passes.restype = ctypes.c_long
        lib.oracle_jacobi_passes.argtypes = [dp, dp, ctypes.c_long, ctypes.c_long, ctypes.c_long,
                                             ctypes.c_double]
        lib.oracle_mgs.restype = None
        lib.oracle_mgs.argtypes = [dp, ctypes.c_long]
        lib.oracle_off_norm.restype = ctypes.c_double
        lib.oracle_off_norm.argtypes = [dp, ctypes.c_long]
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def jacobi_sweeps(a, v, tol, skip, max_sweeps):
    """In-place cyclic Jacobi (_jacobi.py:37-86); a, v C-contiguous float64."""
    assert a.flags.c_contiguous and v.flags.c_contiguous
    return int(_native().oracle_jacobi_sweeps(_ptr(a), _ptr(v), a.shape[0], tol, skip,
                                              max_sweeps))


def jacobi_passes(a, v, p0, p1, skip):
    """Passes p0..p1-1 of one cyclic sweep (timing samples only); returns rotations applied."""
    assert a.flags.c_contiguous and v.flags.c_contiguous
    return int(_native().oracle_jacobi_passes(_ptr(a), _ptr(v), a.shape[0], p0, p1, skip))


def modified_gram_schmidt(psi):
    """In-place column MGS (_jacobi.py:89-107)."""
    assert psi.flags.c_contiguous
    _native().oracle_mgs(_ptr(psi), psi.shape[0])


def off_norm(a):
    a = np.ascontiguousarray(a, dtype=float)
    return float(_native().oracle_off_norm(_ptr(a), a.shape[0]))


# ---------------------------------------------------------------------------
# model tables (rrgp.py:188-227, 310-344; posterior.py:203-255)


@dataclasses.dataclass
class _Group:
    kind: str          # "gaussian_1d" | "linear"
    idx: np.ndarray
    hpos: tuple
    w: np.ndarray
    fixed: tuple


class OTarget:
    """Tempered posterior for (model, data); mirrors PosteriorTarget."""

    def __init__(self, model, data, tau=1.0, _shared=None):
        self.model, self.data, self.tau = model, data, float(tau)
        if _shared is not None:
            (self.fslices, self.inter, self.hidx, self.dim, self.phi, self.groups,
             self.hprior) = _shared
            return
        pos = 0
        self.fslices, self.inter, coef = [], [], []
        for j, kernels in enumerate(model.functions):
            start = pos
            for k, kern in enumerate(kernels):
                coef.append((j, kern, pos))
                pos += kern.features
            self.inter.append(pos)
            pos += 1
            self.fslices.append(slice(start, pos))
        self.hidx = {}
        for name in ("c_g", "sigma_g", "c_l"):
            if name in model.hyperparameters:
                self.hidx[name] = pos
                pos += 1
        self.dim = pos
        x = data.x
        self.phi = []
        for j, kernels in enumerate(model.functions):
            cols = []
            for kern in kernels:
                xk = x[:, kern.covariate][:, None]
                if kern.kind == "gaussian_1d":
                    m = np.arange(1, kern.features + 1)[None, :]
                    cols.append(np.sin(np.pi * m * (xk + kern.half_width)
                                       / (2.0 * kern.half_width)))
                else:
                    cols.append(xk)
            cols.append(np.ones((data.n, 1)))
            self.phi.append(np.ascontiguousarray(np.hstack(cols)))
        g_idx, g_w, l_idx = [], [], []
        for j, kern, start in coef:
            ids = np.arange(start, start + kern.features)
            if kern.kind == "gaussian_1d":
                m = np.arange(1, kern.features + 1, dtype=float)
                g_idx.append(ids)
                g_w.append((np.pi * m / (2.0 * kern.half_width)) ** 2 / 4.0)
            else:
                l_idx.append(ids)
        fixed = model.fixed_hypers
        self.groups = []
        if g_idx:
            if "c_g" in self.hidx:
                hp, fv = (self.hidx["c_g"], self.hidx["sigma_g"]), ()
            else:
                hp, fv = (), (fixed["c_g"], fixed["sigma_g"])
            self.groups.append(_Group("gaussian_1d", np.concatenate(g_idx), hp,
                                      np.concatenate(g_w), fv))
        if l_idx:
            ids = np.concatenate(l_idx)
            if "c_l" in self.hidx:
                hp, fv = (self.hidx["c_l"],), ()
            else:
                hp, fv = (), (fixed["c_l"],)
            self.groups.append(_Group("linear", ids, hp, np.zeros(ids.size), fv))
        self.hprior = {}
        for name in self.hidx:
            a, b = model.priors[name]
            self.hprior[name] = (float(a), float(b),
                                 math.lgamma(float(a)) - float(a) * math.log(float(b)))

    def at_temperature(self, tau):
        return OTarget(self.model, self.data, tau,
                       _shared=(self.fslices, self.inter, self.hidx, self.dim, self.phi,
                                self.groups, self.hprior))

    def initial_point(self):
        q = np.zeros(self.dim)
        if self.model.hyper_transform == "identity":
            for pos in self.hidx.values():
                q[pos] = 1.0
        return q

    def at(self, q):
        return OPoint(self, q)

    def log_likelihood(self, q):
        return -self.at(q).sum_potentials()


def lik_derivs(likelihood, f, y, floor):
    """Per-sample U and its f-derivatives to third order (rrgp.py:351-423)."""
    n = f.shape[0]
    if likelihood == "logistic":
        z = y * f[:, 0]
        u = np.logaddexp(0.0, -z)
        e = np.exp(-np.abs(z))
        qo = np.where(z >= 0.0, e, 1.0) / (1.0 + e)
        po = 1.0 - qo
        return (u, (-y * qo)[:, None], (po * qo)[:, None, None],
                (y * po * qo * (qo - po))[:, None, None, None])
    with np.errstate(over="ignore"):
        w = np.exp(f[:, 1])
    v = floor + w
    e = y - f[:, 0]
    e2 = e * e
    u = 0.5 * e2 / v + 0.5 * np.log(2.0 * np.pi * v)
    r = w / v
    d1 = np.stack([-e / v, 0.5 * r * (1.0 - e2 / v)], axis=1)
    d2 = np.empty((n, 2, 2))
    d2[:, 0, 0] = 1.0 / v
    d2[:, 0, 1] = d2[:, 1, 0] = e * r / v
    d2[:, 1, 1] = -0.5 * e2 * r / v + e2 * r * r / v + 0.5 * r - 0.5 * r * r
    d3 = np.zeros((n, 2, 2, 2))
    t112 = -r / v
    t122 = e * (r / v) * (1.0 - 2.0 * r)
    t222 = (-0.5 * e2 * r / v + 3.0 * e2 * r * r / v - 3.0 * e2 * r * r * r / v
            + 0.5 * r - 1.5 * r * r + r * r * r)
    for a, b, c in ((0, 0, 1), (0, 1, 0), (1, 0, 0)):
        d3[:, a, b, c] = t112
    for a, b, c in ((0, 1, 1), (1, 0, 1), (1, 1, 0)):
        d3[:, a, b, c] = t122
    d3[:, 1, 1, 1] = t222
    return u, d1, d2, d3


def _hyperprior(prior, transform, h):
    """Inverse-gamma potential in the sampled coordinate (posterior.py:97-115)."""
    a, b, norm = prior
    try:
        if transform == "log":
            e = math.exp(-h)
            return a * h + b * e + norm, a - b * e, b * e, -b * e
        if h <= 0.0:
            raise ODomain("hyperparameter must be positive under identity transform")
        return ((a + 1.0) * math.log(h) + b / h + norm,
                (a + 1.0) / h - b / h ** 2,
                -(a + 1.0) / h ** 2 + 2.0 * b / h ** 3,
                2.0 * (a + 1.0) / h ** 3 - 6.0 * b / h ** 4)
    except (OverflowError, ZeroDivisionError):
        raise ODivergence("hyperprior overflow") from None


def _group_derivs(g, hvals, transform):
    """rho = ln r and r partials (posterior.py:127-192)."""
    n, h = g.idx.size, len(g.hpos)
    d1, d2, d3 = np.zeros((h, n)), np.zeros((h, h, n)), np.zeros((h, h, h, n))
    w = g.w
    if h == 0:
        if g.kind == "gaussian_1d":
            c, s = g.fixed
            rho = -math.log(c) - 0.5 * math.log(math.pi) - 0.5 * math.log(s) + s * w
        else:
            rho = np.full(n, -math.log(g.fixed[0]))
    elif g.kind == "gaussian_1d":
        c, s = hvals
        if transform == "log":
            try:
                sw = math.exp(s) * w
            except OverflowError:
                raise ODivergence("spectral variance underflow") from None
            rho = -c - 0.5 * math.log(math.pi) - 0.5 * s + sw
            d1[0], d1[1], d2[1, 1], d3[1, 1, 1] = -1.0, sw - 0.5, sw, sw
        else:
            if c <= 0.0 or s <= 0.0:
                raise ODomain("hyperparameters must be positive")
            rho = -np.log(c) - 0.5 * math.log(math.pi) - 0.5 * math.log(s) + s * w
            d1[0], d1[1] = -1.0 / c, w - 0.5 / s
            d2[0, 0], d2[1, 1] = 1.0 / c ** 2, 0.5 / s ** 2
            d3[0, 0, 0], d3[1, 1, 1] = -2.0 / c ** 3, -1.0 / s ** 3
    else:
        (c,) = hvals
        if transform == "log":
            rho = np.full(n, -c)
            d1[0] = -1.0
        else:
            if c <= 0.0:
                raise ODomain("hyperparameters must be positive")
            rho = np.full(n, -math.log(c))
            d1[0], d2[0, 0], d3[0, 0, 0] = -1.0 / c, 1.0 / c ** 2, -2.0 / c ** 3
    with np.errstate(over="ignore", invalid="ignore"):
        r = np.exp(rho)
        r1 = r * d1
        r2 = r * (d1[:, None] * d1[None, :] + d2)
        r3 = r * (d1[:, None, None] * d1[None, :, None] * d1[None, None, :]
                  + d2[:, :, None] * d1[None, None, :]
                  + d2[:, None, :] * d1[None, :, None]
                  + d2[None, :, :] * d1[:, None, None] + d3)
    return dict(rho=rho, rho1=d1, rho2=d2, rho3=d3, r=r, r1=r1, r2=r2, r3=r3)


class OPoint:
    """Lazy evaluation at one q (posterior.py:310-542)."""

    def __init__(self, target, q):
        q = np.ascontiguousarray(np.asarray(q, dtype=float))
        if q.shape != (target.dim,):
            raise ValueError("dimension mismatch")
        if not np.isfinite(q).all():
            raise ODivergence("non-finite coordinates")
        self.t, self.q = target, q
        self._f = self._lik = self._grp = self._hyp = None
        self._pot = self._grad = self._hess = None

    @property
    def f(self):
        if self._f is None:
            t = self.t
            f = np.empty((t.data.n, len(t.phi)))
            for j, mat in enumerate(t.phi):
                f[:, j] = mat @ self.q[t.fslices[j]]
            if not np.isfinite(f).all():
                raise ODivergence("non-finite latent function values")
            self._f = f
        return self._f

    @property
    def lik(self):
        if self._lik is None:
            m = self.t.model
            self._lik = lik_derivs(m.likelihood, self.f, self.t.data.y, m.variance_floor)
        return self._lik

    @property
    def grp(self):
        if self._grp is None:
            out = []
            for g in self.t.groups:
                gd = _group_derivs(g, tuple(self.q[p] for p in g.hpos),
                                   self.t.model.hyper_transform)
                if not np.isfinite(gd["r"]).all():
                    raise ODivergence("prior inverse variance overflow")
                out.append((g, gd))
            self._grp = out
        return self._grp

    @property
    def hyp(self):
        if self._hyp is None:
            self._hyp = {n: _hyperprior(self.t.hprior[n], self.t.model.hyper_transform,
                                        self.q[p]) for n, p in self.t.hidx.items()}
        return self._hyp

    def sum_potentials(self):
        u = float(np.sum(self.lik[0]))
        if not math.isfinite(u):
            raise ODivergence("non-finite likelihood potential")
        return u

    def potential(self):
        if self._pot is None:
            t, sig = self.t, self.t.model.intercept_variance
            val = t.tau * self.sum_potentials() if t.tau != 0.0 else 0.0
            for g, gd in self.grp:
                a = self.q[g.idx]
                val += float(0.5 * np.dot(a * a, gd["r"]) - 0.5 * np.sum(gd["rho"])
                             + 0.5 * LN_2PI * g.idx.size)
            for pos in t.inter:
                b = self.q[pos]
                val += 0.5 * b * b / sig + 0.5 * math.log(2.0 * math.pi * sig)
            for u0, _, _, _ in self.hyp.values():
                val += u0
            if not math.isfinite(val):
                raise ODivergence("non-finite posterior potential")
            self._pot = val
        return self._pot

    def gradient(self):
        if self._grad is None:
            t = self.t
            grad = np.zeros(t.dim)
            if t.tau != 0.0:
                d1 = self.lik[1]
                for j, mat in enumerate(t.phi):
                    grad[t.fslices[j]] = t.tau * (mat.T @ d1[:, j])
            for g, gd in self.grp:
                a = self.q[g.idx]
                grad[g.idx] += a * gd["r"]
                for k, pos in enumerate(g.hpos):
                    grad[pos] += 0.5 * np.dot(a * a, gd["r1"][k]) - 0.5 * np.sum(gd["rho1"][k])
            for pos in t.inter:
                grad[pos] += self.q[pos] / t.model.intercept_variance
            for name, (_, u1, _, _) in self.hyp.items():
                grad[t.hidx[name]] += u1
            if not np.isfinite(grad).all():
                raise ODivergence("non-finite posterior gradient")
            self._grad = grad
        return self._grad

    def hessian(self):
        if self._hess is None:
            t = self.t
            hess = np.zeros((t.dim, t.dim))
            if t.tau != 0.0:
                d2 = self.lik[2]
                nj = len(t.phi)
                for j1 in range(nj):
                    for j2 in range(j1, nj):
                        blk = (t.phi[j1] * (t.tau * d2[:, j1, j2])[:, None]).T @ t.phi[j2]
                        hess[t.fslices[j1], t.fslices[j2]] += blk
                        if j2 != j1:
                            hess[t.fslices[j2], t.fslices[j1]] += blk.T
            dg = np.einsum("ii->i", hess)
            for g, gd in self.grp:
                a = self.q[g.idx]
                dg[g.idx] += gd["r"]
                for k, pk in enumerate(g.hpos):
                    cross = a * gd["r1"][k]
                    hess[g.idx, pk] += cross
                    hess[pk, g.idx] += cross
                    for l, pl in enumerate(g.hpos):
                        hess[pk, pl] += (0.5 * np.dot(a * a, gd["r2"][k, l])
                                         - 0.5 * np.sum(gd["rho2"][k, l]))
            for pos in t.inter:
                dg[pos] += 1.0 / t.model.intercept_variance
            for name, (_, _, u2, _) in self.hyp.items():
                dg[t.hidx[name]] += u2
            if not np.isfinite(hess).all():
                raise ODivergence("non-finite posterior Hessian")
            self._hess = hess
        return self._hess

    def trace(self, w):
        """t_i = tr(W dH/dq_i), structured (posterior.py:486-542)."""
        t = self.t
        w = np.asarray(w, dtype=float)
        out = np.zeros(t.dim)
        if t.tau != 0.0:
            d3 = self.lik[3]
            nj = len(t.phi)
            for j1 in range(nj):
                for j2 in range(nj):
                    s = np.einsum("ij,ij->i", t.phi[j1] @ w[t.fslices[j1], t.fslices[j2]],
                                  t.phi[j2], optimize=False)
                    for j in range(nj):
                        coef = d3[:, j1, j2, j]
                        if coef.any():
                            out[t.fslices[j]] += t.tau * (t.phi[j].T @ (coef * s))
        for g, gd in self.grp:
            a = self.q[g.idx]
            h = len(g.hpos)
            dw = w[g.idx, g.idx]
            cols = [0.5 * (w[g.idx, p] + w[p, g.idx]) for p in g.hpos]
            hw = np.array([[0.5 * (w[pa, pb] + w[pb, pa]) for pb in g.hpos] for pa in g.hpos])
            acc = np.zeros(g.idx.size)
            for k in range(h):
                acc += 2.0 * cols[k] * gd["r1"][k]
                for l in range(h):
                    acc += hw[k, l] * a * gd["r2"][k, l]
            out[g.idx] += acc
            for m, pos in enumerate(g.hpos):
                val = np.dot(dw, gd["r1"][m])
                for k in range(h):
                    val += 2.0 * np.dot(cols[k], a * gd["r2"][m, k])
                    for l in range(h):
                        val += hw[k, l] * (0.5 * np.dot(a * a, gd["r3"][m, k, l])
                                           - 0.5 * np.sum(gd["rho3"][m, k, l]))
                out[pos] += val
        for name, (_, _, _, u3) in self.hyp.items():
            pos = t.hidx[name]
            out[pos] += w[pos, pos] * u3
        if not np.isfinite(out).all():
            raise ODivergence("non-finite trace contraction")
        return out


# ---------------------------------------------------------------------------
# SoftAbs metric (metric.py)


@dataclasses.dataclass(frozen=True)
class OMetric:
    lam: np.ndarray
    psi: np.ndarray
    g: np.ndarray
    logdet: float
    kappa: float
    sweeps: int
    since: int = 0

    @property
    def dim(self):
        return self.lam.shape[0]


def softabs(lam, kappa):
    lam = np.asarray(lam, dtype=float)
    return np.sqrt(kappa * kappa + lam * lam)


def t_matrix(lam, kappa):
    """Divided differences with the derivative branch (metric.py:46-59)."""
    lam = np.asarray(lam, dtype=float)
    g = softabs(lam, kappa)
    diff = lam[:, None] - lam[None, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = (g[:, None] - g[None, :]) / diff
    return np.where(np.abs(diff) <= kappa * EQUAL_EIGENVALUE_FACTOR, (lam / g)[:, None], ratio)


def _decompose(a, v, hnorm, zeta, cap):
    tol = zeta * hnorm
    skip = tol / a.shape[0] if a.shape[0] else 0.0
    sweeps = jacobi_sweeps(a, v, tol, skip, cap)
    if sweeps < 0:
        raise OJacobi(f"Jacobi failed to reach off-norm {tol:.3e} in {cap} sweeps")
    return sweeps


def cold_eigh(h, zeta, cap=30):
    """static_eigendecompose (metric.py:112-127)."""
    h = np.asarray(h, dtype=float)
    a = np.ascontiguousarray(0.5 * (h + h.T))
    hnorm = np.linalg.norm(a)
    v = np.eye(h.shape[0])
    sweeps = _decompose(a, v, hnorm, zeta, cap)
    return np.diagonal(a).copy(), v, sweeps


def metric_cold(h, kappa, zeta, cap=30):
    """metric_from_hessian (metric.py:130-142)."""
    lam, psi, sweeps = cold_eigh(h, zeta, cap)
    g = softabs(lam, kappa)
    return OMetric(lam, psi, g, float(np.sum(np.log(g))), kappa, sweeps, 0)


def metric_warm(h, prev, zeta, cap=30, gs_interval=10):
    """dynamic_eigendecompose (metric.py:145-185)."""
    h = np.asarray(h, dtype=float)
    psi = prev.psi
    since = prev.since + 1
    if gs_interval and since >= gs_interval:
        psi = np.ascontiguousarray(psi.copy())
        modified_gram_schmidt(psi)
        since = 0
    a = psi.T @ h @ psi
    a = np.ascontiguousarray(0.5 * (a + a.T))
    hnorm = np.linalg.norm(h)
    qm = np.eye(h.shape[0])
    sweeps = _decompose(a, qm, hnorm, zeta, cap)
    lam = np.diagonal(a).copy()
    g = softabs(lam, prev.kappa)
    return OMetric(lam, psi @ qm, g, float(np.sum(np.log(g))), prev.kappa, sweeps, since)


def w1(metric, p):
    """metric.py:188-198."""
    b = (metric.psi.T @ p) / metric.g
    t = t_matrix(metric.lam, metric.kappa)
    with np.errstate(over="ignore", invalid="ignore"):
        return metric.psi @ ((b[:, None] * t) * b[None, :]) @ metric.psi.T


def w2(metric):
    """metric.py:201-204."""
    ratio = (metric.lam / metric.g) / metric.g
    return (metric.psi * ratio[None, :]) @ metric.psi.T


def ginv(metric, v):
    """metric.py:223-225."""
    return metric.psi @ ((metric.psi.T @ v) / metric.g)


def quad(metric, p):
    """metric.py:228-231."""
    u = metric.psi.T @ p
    return float(np.sum(u * u / metric.g))


def momentum(metric, z):
    """metric.py:238-241 with the normals supplied."""
    return metric.psi @ (np.sqrt(metric.g) * z)


# ---------------------------------------------------------------------------
# generalized leapfrog and chain (sampler.py)


@dataclasses.dataclass(frozen=True)
class OConfig:
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


@dataclasses.dataclass
class OFrame:
    pt: OPoint
    metric: OMetric | None
    w2: np.ndarray | None


def frame_h(frame, p):
    """sampler.py:163-169."""
    if frame.metric is None:
        kin = 0.5 * float(p @ p) + 0.5 * p.shape[0] * LN_2PI
    else:
        kin = 0.5 * quad(frame.metric, p) + 0.5 * (frame.metric.dim * LN_2PI
                                                   + frame.metric.logdet)
    return frame.pt.potential() + kin


def _next_metric(h, prev, cfg):
    if cfg.metric == "softabs-static":
        return metric_cold(h, cfg.kappa, cfg.zeta, cfg.sweep_cap)
    return metric_warm(h, prev, cfg.zeta, cfg.sweep_cap, cfg.gs_interval)


def leapfrog(frame, p, cfg, target, diag):
    """One generalized leapfrog (sampler.py:209-258) or Euclidean (261-267)."""
    eps = cfg.epsilon
    if frame.metric is None:
        ph = p - 0.5 * eps * frame.pt.gradient()
        nxt = target.at(frame.pt.q + eps * ph)
        return OFrame(nxt, None, None), ph - 0.5 * eps * nxt.gradient()
    pt, met, w2f = frame.pt, frame.metric, frame.w2
    grad = pt.gradient()

    def grad_h(pv):
        return grad + 0.5 * pt.trace(w2f - w1(met, pv))

    ph = p - 0.5 * eps * grad_h(p)
    for it in range(cfg.fp_max_iters):
        pn = p - 0.5 * eps * grad_h(ph)
        delta = float(np.max(np.abs(pn - ph)))
        ph = pn
        if delta <= cfg.fp_tol:
            diag["fp_p_iters"].append(it + 1)
            break
    else:
        raise ODivergence("momentum half-step fixed point stalled")
    q0 = pt.q
    v0 = ginv(met, ph)
    qc = q0 + eps * v0
    mc, pc = met, None
    for it in range(cfg.fp_max_iters):
        pc = target.at(qc)
        mc = _next_metric(pc.hessian(), mc, cfg)
        diag["sweeps"].append(mc.sweeps)
        qn = q0 + 0.5 * eps * (v0 + ginv(mc, ph))
        if float(np.max(np.abs(qn - qc))) <= cfg.fp_tol:
            diag["fp_q_iters"].append(it + 1)
            break
        qc = qn
    else:
        raise ODivergence("position step fixed point stalled")
    w2n = w2(mc)
    corr = 0.5 * pc.trace(w2n - w1(mc, ph))
    return OFrame(pc, mc, w2n), ph - 0.5 * eps * (pc.gradient() + corr)


def new_diag():
    return {"sweeps": [], "fp_p_iters": [], "fp_q_iters": []}


def leapfrog_step(q, p, metric, target, cfg):
    """sampler.py:280-292."""
    pt = target.at(np.asarray(q, dtype=float))
    frame = OFrame(pt, metric, w2(metric) if metric is not None else None)
    diag = new_diag()
    nf, pn = leapfrog(frame, np.asarray(p, dtype=float), cfg, target, diag)
    return nf.pt.q, pn, nf.metric, diag


def initial_frame(target, q0, cfg):
    """sampler.py:322-328."""
    pt = target.at(q0)
    pt.gradient()
    if cfg.metric == "euclidean":
        return OFrame(pt, None, None)
    met = metric_cold(pt.hessian(), cfg.kappa, cfg.zeta, cfg.sweep_cap)
    return OFrame(pt, met, w2(met))


@dataclasses.dataclass
class ORecord:
    move: int
    logpost: float
    h_before: float
    h_after: float | None
    accept: bool
    divergent: bool
    sweeps_mean: float
    q: np.ndarray | None
    uniform: float


@dataclasses.dataclass
class OResult:
    records: list
    q_final: np.ndarray
    accept_count: int
    divergence_count: int

    @property
    def logpost(self):
        return np.array([r.logpost for r in self.records])


def run_chain(target, cfg, initial=None):
    """sampler.py:331-418."""
    rng = np.random.default_rng(cfg.seed)
    q0 = np.asarray(target.initial_point() if initial is None else initial, dtype=float).copy()
    if q0.shape != (target.dim,):
        raise ValueError("initial point has wrong dimension")
    try:
        frame = initial_frame(target, q0, cfg)
    except _DIVERGENT as exc:
        raise OChainError(f"chain start failed: {exc}") from exc
    euclid = cfg.metric == "euclidean"
    recs, acc, div = [], 0, 0
    for move in range(cfg.moves):
        z = rng.standard_normal(target.dim)
        p = z if euclid else momentum(frame.metric, z)
        hb = frame_h(frame, p)
        diag = new_diag()
        divergent, ha, nf, pc = False, None, frame, p
        try:
            for _ in range(cfg.leapfrogs):
                nf, pc = leapfrog(nf, pc, cfg, target, diag)
            ha = frame_h(nf, pc)
            if not math.isfinite(ha):
                raise ODivergence("non-finite Hamiltonian after trajectory")
        except _DIVERGENT:
            divergent, ha = True, None
        u = rng.uniform()
        accept = (not divergent) and (hb - ha) > math.log(u)
        if accept:
            frame = nf
            acc += 1
        else:
            if divergent:
                div += 1
                if move == 0:
                    raise OChainError("divergence on the first move")
            if not euclid:
                met = metric_cold(frame.pt.hessian(), cfg.kappa, cfg.zeta, cfg.sweep_cap)
                frame = OFrame(frame.pt, met, w2(met))
        sw = diag["sweeps"]
        recs.append(ORecord(move, -frame.pt.potential(), hb, ha, accept, divergent,
                            float(np.mean(sw)) if sw else 0.0,
                            frame.pt.q.copy() if cfg.record_q else None, u))
    return OResult(recs, frame.pt.q.copy(), acc, div)


# ---------------------------------------------------------------------------
# stationarity test and thermodynamic integration (sampler.py:432-487,
# evidence.py:83-274)


def rank_sum_test(x, y):
    x, y = np.asarray(x, dtype=float), np.asarray(y, dtype=float)
    n1, n2 = x.shape[0], y.shape[0]
    n = n1 + n2
    v = np.concatenate([x, y])
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
    w = float(np.sum(ranks[:n1]))
    var = n1 * n2 / 12.0 * ((n + 1) - float(sum(t ** 3 - t for t in ties)) / (n * (n - 1)))
    if var <= 0.0:
        return 0.0, 1.0
    diff = w - n1 * (n + 1) / 2.0
    z = 0.0 if abs(diff) <= 0.5 else (diff - math.copysign(0.5, diff)) / math.sqrt(var)
    return float(z), float(math.erfc(abs(z) / math.sqrt(2.0)))


def wilcoxon_split_half(values):
    v = np.asarray(values, dtype=float)
    half = v.shape[0] // 2
    return rank_sum_test(v[:half], v[half:])


def trapezoid(values, taus):
    return float(np.sum(0.5 * (values[1:] + values[:-1]) * -np.diff(taus)))


def thermo_integrate(target, taus, moves_per_rung, leapfrogs, chains, cfg, *,
                     warmup_segment_moves=50, warmup_max_segments=8, warmup_pvalue=0.05,
                     spread_moves=10, initial=None):
    """Sequential TI with the reference's seeding (evidence.py:184-274).

    Returns (per_chain, rung_values, q_warm)."""
    taus = np.asarray(taus, dtype=float)
    root = cfg.seed if isinstance(cfg.seed, np.random.SeedSequence) else \
        np.random.SeedSequence(cfg.seed)
    seqs = root.spawn(warmup_max_segments + chains)
    q = target.initial_point() if initial is None else np.asarray(initial, dtype=float)
    for seq in seqs[:warmup_max_segments]:
        res = run_chain(target, dataclasses.replace(cfg, moves=warmup_segment_moves,
                                                    burnin=0, record_q=False, seed=seq), q)
        q = res.q_final
        if warmup_segment_moves >= 10 and wilcoxon_split_half(res.logpost)[1] > warmup_pvalue:
            break
    q_warm = q
    per_chain, rung_values = [], np.full((chains, taus.size), np.nan)
    for z in range(chains):
        sub = seqs[warmup_max_segments + z].spawn(taus.size + 1)
        try:
            qz = np.asarray(q_warm, dtype=float)
            if spread_moves > 0:
                qz = run_chain(target, dataclasses.replace(cfg, moves=spread_moves, burnin=0,
                                                           record_q=False, seed=sub[0]),
                               qz).q_final
            vals = np.empty(taus.size)
            for s, tau in enumerate(taus):
                res = run_chain(target.at_temperature(float(tau)),
                                dataclasses.replace(cfg, moves=moves_per_rung,
                                                    leapfrogs=leapfrogs, burnin=0,
                                                    record_q=False, seed=sub[s + 1]), qz)
                qz = res.q_final
                vals[s] = target.log_likelihood(qz)
            rung_values[z] = vals
            per_chain.append(trapezoid(vals, taus))
        except OChainError:
            per_chain.append(math.nan)
    return per_chain, rung_values, q_warm


# ---------------------------------------------------------------------------
# Laplace evidence oracles: L-BFGS, laplace_full,
# laplace_grid_oracle.

@dataclasses.dataclass
class OOptim:
    x: np.ndarray
    value: float
    grad: np.ndarray
    iterations: int
    evaluations: int
    converged: bool


def _two_loop(grad, s_hist, y_hist, rho_hist):
    """lbfgs.py:27-40."""
    q = grad.copy()
    alphas = []
    for s, y, rho in zip(reversed(s_hist), reversed(y_hist), reversed(rho_hist)):
        a = rho * float(s @ q)
        alphas.append(a)
        q -= a * y
    if y_hist:
        q *= float(s_hist[-1] @ y_hist[-1]) / float(y_hist[-1] @ y_hist[-1])
    for (s, y, rho), a in zip(zip(s_hist, y_hist, rho_hist), reversed(alphas)):
        b = rho * float(y @ q)
        q += (a - b) * s
    return q


def _zoom(fg, x, d, f0, dphi0, lo, f_lo, hi, c1, c2, max_iter=30):
    """lbfgs.py:43-64: bisection zoom of the strong Wolfe search."""
    evals = 0
    for _ in range(max_iter):
        a = 0.5 * (lo + hi)
        f, g = fg(x + a * d)
        evals += 1
        dphi = float(g @ d) if math.isfinite(f) else math.inf
        if not math.isfinite(f) or f > f0 + c1 * a * dphi0 or f >= f_lo:
            hi = a
        else:
            if abs(dphi) <= -c2 * dphi0:
                return a, f, g, evals
            if dphi * (hi - lo) >= 0.0:
                hi = lo
            lo, f_lo = a, f
        if abs(hi - lo) <= 1e-14 * max(1.0, abs(lo)):
            break
    f, g = fg(x + lo * d)
    evals += 1
    if math.isfinite(f) and f <= f0 + c1 * lo * dphi0 and lo > 0.0:
        return lo, f, g, evals
    return None, f0, None, evals


def _wolfe(fg, x, f0, g0, d, c1, c2, max_expand=25):
    """lbfgs.py:67-86: expanding strong Wolfe line search."""
    dphi0 = float(g0 @ d)
    a_prev, f_prev, a, evals = 0.0, f0, 1.0, 0
    for i in range(max_expand):
        f, g = fg(x + a * d)
        evals += 1
        if not math.isfinite(f) or f > f0 + c1 * a * dphi0 or (i > 0 and f >= f_prev):
            r = _zoom(fg, x, d, f0, dphi0, a_prev, f_prev, a, c1, c2)
            return r[0], r[1], r[2], evals + r[3]
        dphi = float(g @ d)
        if abs(dphi) <= -c2 * dphi0:
            return a, f, g, evals
        if dphi >= 0.0:
            r = _zoom(fg, x, d, f0, dphi0, a, f, a_prev, c1, c2)
            return r[0], r[1], r[2], evals + r[3]
        a_prev, f_prev = a, f
        a *= 2.0
    return None, f0, None, evals


def lbfgs_minimize(fg, x0, *, memory=10, gtol=1e-6, max_iters=200, c1=1e-4, c2=0.9):
    """lbfgs.py:89-150."""
    x = np.asarray(x0, dtype=float).copy()
    f, g = fg(x)
    evals = 1
    if not math.isfinite(f):
        raise ValueError("objective is not finite at the starting point")
    sh, yh, rh = [], [], []
    for it in range(max_iters):
        if float(np.max(np.abs(g))) <= gtol:
            return OOptim(x, f, g, it, evals, True)
        d = -_two_loop(g, sh, yh, rh)
        if float(g @ d) >= 0.0:
            sh.clear(), yh.clear(), rh.clear()
            d = -g
        alpha, fn, gn, ne = _wolfe(fg, x, f, g, d, c1, c2)
        evals += ne
        if alpha is None and sh:
            sh.clear(), yh.clear(), rh.clear()
            d = -g
            alpha, fn, gn, ne = _wolfe(fg, x, f, g, d, c1, c2)
            evals += ne
        if alpha is None:
            return OOptim(x, f, g, it, evals, float(np.max(np.abs(g))) <= gtol)
        xn = x + alpha * d
        s, y = xn - x, gn - g
        sy = float(s @ y)
        if sy > 1e-12 * float(np.linalg.norm(s)) * float(np.linalg.norm(y)):
            sh.append(s), yh.append(y), rh.append(1.0 / sy)
            if len(sh) > memory:
                sh.pop(0), yh.pop(0), rh.pop(0)
        x, f, g = xn, fn, gn
    return OOptim(x, f, g, max_iters, evals, float(np.max(np.abs(g))) <= gtol)


def prior_scales(target, q):
    """posterior.py:289-307: 1/sqrt(r) per coefficient, sqrt(Sigma) per intercept."""
    scales = np.ones(target.dim)
    for g in target.groups:
        hvals = tuple(q[p] for p in g.hpos)
        scales[g.idx] = np.exp(-0.5 * _group_derivs(g, hvals, target.model.hyper_transform)["rho"])
    for pos in target.inter:
        scales[pos] = math.sqrt(target.model.intercept_variance)
    return scales


def hyperprior_potential(target, q):
    """posterior.py:281-287."""
    return float(sum(_hyperprior(target.hprior[n], target.model.hyper_transform, q[p])[0]
                     for n, p in target.hidx.items()))


LAPLACE_ZETA = 1e-13  # evidence.py:31


def laplace_full(target, *, initial=None, gtol=1e-6, max_iters=500):
    """evidence.py:277-304: -U(q*) + d/2 ln 2 pi - 1/2 ln|H(q*)| (Jacobi eigenvalues)."""
    x0 = target.initial_point() if initial is None else np.asarray(initial, dtype=float)

    def fg(x):
        try:
            p = target.at(x)
            return p.potential(), p.gradient()
        except (ODomain, ODivergence):
            return math.inf, np.zeros(target.dim)

    res = lbfgs_minimize(fg, x0, gtol=gtol, max_iters=max_iters)
    if not res.converged:
        raise RuntimeError("Laplace mode search did not reach gradient tolerance")
    lam, _, _ = cold_eigh(target.at(res.x).hessian(), LAPLACE_ZETA)
    if np.min(lam) <= 0.0:
        raise RuntimeError("Laplace invalid (singular/indefinite posterior)")
    return -res.value + 0.5 * target.dim * LN_2PI - 0.5 * float(np.sum(np.log(lam)))


def _inv_gamma_logpdf(theta, alpha, beta):
    """evidence.py:326-327."""
    return alpha * math.log(beta) - math.lgamma(alpha) - (alpha + 1.0) * math.log(theta) - beta / theta


def grid_centers(c_max, c_mesh, sigma_max, sigma_mesh):
    """evidence.py:318-323 (GridSpec.centers)."""
    nc, ns = int(round(c_max / c_mesh)), int(round(sigma_max / sigma_mesh))
    return (np.arange(nc) + 0.5) * c_mesh, (np.arange(ns) + 0.5) * sigma_mesh


def laplace_grid_nodes(target, c_max=4.0, c_mesh=0.01, sigma_max=4.0, sigma_mesh=0.02, pinned=(),
                       *, gtol=1e-6, max_iters=200, warm="serpentine"):
    """evidence.py:330-410: per-node conditional Laplace values in the reference's
    serpentine order.  warm="serpentine" warm-starts each node from the previous
    optimum (the reference); warm="zero" starts every node at a = 0 (the
    device's independent nodes).  Returns (values in node order or nan, status
    0 ok / 1 optimiser failed / 2 Cholesky failed, (c, sigma) per node)."""
    model = target.model
    pinned = dict(pinned)
    hidx = target.hidx
    transform = model.hyper_transform
    coef_idx = np.array([i for i in range(target.dim) if i not in hidx.values()], dtype=int)
    base = np.zeros(target.dim)
    for name, value in pinned.items():
        base[hidx[name]] = math.log(value) if transform == "log" else value
    c_pos, s_pos = hidx["c_g"], hidx["sigma_g"]
    prior_c, prior_s = model.priors["c_g"], model.priors["sigma_g"]
    c_centers, s_centers = grid_centers(c_max, c_mesh, sigma_max, sigma_mesh)
    log_area = math.log(c_mesh) + math.log(sigma_mesh)
    n_coef = coef_idx.size
    vals, stat, nodes = [], [], []
    a_warm = np.zeros(n_coef)
    for si, sigma in enumerate(s_centers):
        row = c_centers if si % 2 == 0 else c_centers[::-1]
        for c in row:
            nodes.append((c, sigma))
            q = base.copy()
            q[c_pos] = math.log(c) if transform == "log" else c
            q[s_pos] = math.log(sigma) if transform == "log" else sigma
            scales = prior_scales(target, q)[coef_idx]

            def fg(avec, q=q, scales=scales):
                qq = q.copy()
                qq[coef_idx] = avec * scales
                try:
                    p = target.at(qq)
                    return p.potential(), p.gradient()[coef_idx] * scales
                except (ODomain, ODivergence):
                    return math.inf, np.zeros(n_coef)

            start = a_warm / scales if warm == "serpentine" else np.zeros(n_coef)
            res = lbfgs_minimize(fg, start, gtol=gtol, max_iters=max_iters)
            if not res.converged:
                vals.append(float("nan")), stat.append(1)
                continue
            if warm == "serpentine":
                a_warm = res.x * scales
            q[coef_idx] = res.x * scales
            p = target.at(q)
            conditional = p.potential() - hyperprior_potential(target, q)
            try:
                chol = np.linalg.cholesky(p.hessian()[np.ix_(coef_idx, coef_idx)])
            except np.linalg.LinAlgError:
                vals.append(float("nan")), stat.append(2)
                continue
            logdet = 2.0 * float(np.sum(np.log(np.diagonal(chol))))
            vals.append(-conditional + 0.5 * n_coef * LN_2PI - 0.5 * logdet
                        + _inv_gamma_logpdf(c, *prior_c) + _inv_gamma_logpdf(sigma, *prior_s) + log_area)
            stat.append(0)
    return np.asarray(vals), np.asarray(stat), np.asarray(nodes)


def laplace_grid_combine(values, status, skip_tolerance=0.01):
    """evidence.py:411-426: skip check, then log-sum-exp of the node values."""
    skipped = int(np.count_nonzero(status))
    total = int(status.size)
    if skipped > skip_tolerance * total:
        raise RuntimeError(f"grid oracle skipped {skipped}/{total} nodes; result untrustworthy")
    v = values[status == 0]
    peak = float(np.max(v))
    return peak + math.log(float(np.sum(np.exp(v - peak))))
