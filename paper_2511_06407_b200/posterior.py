"""Tempered posterior targets evaluated on the B200.

Drop-in for ``softabs_gp.posterior`` (/root/reference/pkg/src/softabs_gp/
posterior.py): same classes, same call signatures, same exception types.  The
arithmetic runs in libsgp (csrc/sgp_eval.cuh): the design matrices are
assembled once per (model, data) in HBM and shared across temperatures
(posterior.py:261-264), and each state query is one batched kernel launch.
"""

from __future__ import annotations

import collections
import ctypes
import hashlib
import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .rrgp import GAUSSIAN, HYPER_ORDER, LOGISTIC, BlockLayout, Dataset, ModelSpec

LN_2PI = math.log(2.0 * math.pi)


class DomainError(ValueError):
    """Evaluation outside the admissible region (posterior.py:45)."""


class DivergenceError(FloatingPointError):
    """Non-finite state encountered (posterior.py:49)."""


def raise_status(code, what=""):
    """Map a libsgp status word onto the reference's exception classes."""
    from .metric import JacobiError

    if code == nat.STATUS_OK:
        return
    if code == nat.STATUS_DOMAIN:
        raise DomainError(f"{what}: hyperparameter outside its domain")
    if code == nat.STATUS_JACOBI:
        raise JacobiError(f"{what}: Jacobi failed to converge within the sweep cap")
    if code == nat.STATUS_STALL_P:
        raise DivergenceError("momentum half-step fixed point stalled")
    if code == nat.STATUS_STALL_Q:
        raise DivergenceError("position step fixed point stalled")
    raise DivergenceError(f"{what}: non-finite state")


@dataclass
class ParamVector:
    """A point in the sampled coordinates with its temperature (posterior.py:53-67)."""

    values: np.ndarray
    tau: float = 1.0

    def __post_init__(self):
        self.values = np.ascontiguousarray(np.asarray(self.values, dtype=float))
        if self.values.ndim != 1:
            raise ValueError("parameter vector must be 1-d")
        if not np.isfinite(self.values).all():
            raise ValueError("parameter vector has non-finite entries")
        if not 0.0 <= self.tau <= 1.0:
            raise ValueError(f"temperature must lie in [0, 1], got {self.tau}")


class DeviceModel:
    """Owns one ``sgp_model`` (design matrices + coordinate tables in HBM)."""

    def __init__(self, model: ModelSpec | None, data: Dataset | None, *, quadratic=None):
        self.L = nat.lib()
        desc = nat.ModelDesc()
        self._keep = []
        if quadratic is not None:
            prec, mean, const = quadratic
            prec = np.ascontiguousarray(prec, dtype=float)
            mean = np.ascontiguousarray(mean, dtype=float)
            self._keep += [prec, mean]
            desc.likelihood = nat.LIK_QUADRATIC
            desc.quad_dim = prec.shape[0]
            desc.h_precision = prec.ctypes.data_as(nat.c_dp)
            desc.h_mean = mean.ctypes.data_as(nat.c_dp)
            desc.loglik_const = float(const)
            desc.transform = nat.TRANSFORM_LOG
        else:
            x = np.ascontiguousarray(data.x, dtype=float)
            y = np.ascontiguousarray(data.y, dtype=float)
            self._keep += [x, y]
            desc.likelihood = nat.LIK_LOGISTIC if model.likelihood == LOGISTIC else nat.LIK_GAUSSIAN_MEANVAR
            desc.n_rows, desc.n_cols = x.shape
            desc.h_x = x.ctypes.data_as(nat.c_dp)
            desc.h_y = y.ctypes.data_as(nat.c_dp)
            desc.n_functions = len(model.functions)
            for j, kernels in enumerate(model.functions):
                arr = (nat.KernelDesc * max(1, len(kernels)))()
                for k, kern in enumerate(kernels):
                    arr[k].kind = nat.KERNEL_GAUSSIAN if kern.kind == GAUSSIAN else nat.KERNEL_LINEAR
                    arr[k].covariate = kern.covariate
                    arr[k].features = kern.features
                    arr[k].half_width = kern.half_width
                self._keep.append(arr)
                desc.n_kernels[j] = len(kernels)
                desc.kernels[j] = ctypes.cast(arr, ctypes.POINTER(nat.KernelDesc))
            desc.transform = nat.TRANSFORM_LOG if model.hyper_transform == "log" else nat.TRANSFORM_IDENTITY
            desc.intercept_variance = model.intercept_variance
            desc.variance_floor = model.variance_floor
            for s, name in enumerate(HYPER_ORDER):
                desc.hyper_sampled[s] = 1 if name in model.hyperparameters else 0
                desc.hyper_fixed[s] = float(model.fixed_hypers.get(name, 1.0))
                if name in model.hyperparameters:
                    a, b = model.priors[name]
                    desc.prior_alpha[s], desc.prior_beta[s] = float(a), float(b)
        handle = ctypes.c_void_p()
        nat.check(self.L.sgp_model_create(ctypes.byref(desc), ctypes.byref(handle)), "sgp_model_create")
        self.handle = handle
        self.dim = self.L.sgp_model_dim(handle)
        self.n_rows = self.L.sgp_model_rows(handle)
        self.scratch_per_chain = int(self.L.sgp_scratch_doubles(handle))
        self._scratch = None
        self.is_quadratic = quadratic is not None

    def __del__(self):
        try:
            if getattr(self, "handle", None) is not None and self.L is not None:
                self.L.sgp_model_destroy(self.handle)
        except Exception:
            pass

    def scratch(self, n_chains):
        need = max(1, n_chains) * self.scratch_per_chain
        if self._scratch is None or self._scratch.numel() < need:
            self._scratch = nat.empty_f64(need)
        return self._scratch

    def phi(self, j):
        import torch

        dj = self.L.sgp_model_features(self.handle, j)
        out = torch.empty((self.n_rows, dj), dtype=torch.float64, device="cuda")
        nat.check(self.L.sgp_model_phi(self.handle, j, nat.ptr(out), nat.stream()), "sgp_model_phi")
        return out.cpu().numpy()

    def eval(self, tau, q, what):
        """Batched evaluation; q (Z, d), tau (Z,).  Returns dict of numpy arrays."""
        import torch

        q = np.atleast_2d(np.asarray(q, dtype=float))
        Z, d = q.shape
        tq = nat.dev_f64(q)
        tt = nat.dev_f64(np.broadcast_to(np.asarray(tau, dtype=float), (Z,)))
        pot = nat.empty_f64(Z)
        sump = nat.empty_f64(Z)
        grad = nat.empty_f64(Z, d) if what & nat.EVAL_GRADIENT else None
        hess = nat.empty_f64(Z, d, d) if what & nat.EVAL_HESSIAN else None
        status = nat.zeros_i32(Z)
        nat.check(self.L.sgp_eval(self.handle, Z, nat.ptr(tt), nat.ptr(tq), what, nat.ptr(pot),
                                  nat.ptr(grad), nat.ptr(hess), nat.ptr(sump), nat.ptr(status),
                                  nat.ptr(self.scratch(Z)), nat.stream()), "sgp_eval")
        torch.cuda.synchronize()
        return {
            "pot": pot.cpu().numpy(), "sumpot": sump.cpu().numpy(),
            "grad": None if grad is None else grad.cpu().numpy(),
            "hess": None if hess is None else hess.cpu().numpy(),
            "status": status.cpu().numpy(),
        }

    def trace(self, tau, q, w):
        import torch

        q = np.atleast_2d(np.asarray(q, dtype=float))
        Z, d = q.shape
        w = np.asarray(w, dtype=float).reshape(Z, d, d)
        tq, tw = nat.dev_f64(q), nat.dev_f64(w)
        tt = nat.dev_f64(np.broadcast_to(np.asarray(tau, dtype=float), (Z,)))
        out = nat.empty_f64(Z, d)
        status = nat.zeros_i32(Z)
        nat.check(self.L.sgp_trace(self.handle, Z, nat.ptr(tt), nat.ptr(tq), nat.ptr(tw), nat.ptr(out),
                                   nat.ptr(status), nat.ptr(self.scratch(Z)), nat.stream()), "sgp_trace")
        torch.cuda.synchronize()
        return out.cpu().numpy(), status.cpu().numpy()


class FeatureCacheView:
    """``target.cache`` compatibility: ``phi[j]`` copied back from HBM on demand."""

    def __init__(self, dev: DeviceModel, n_functions):
        self._dev = dev
        self._n = n_functions
        self._phi = None

    @property
    def phi(self):
        if self._phi is None:
            self._phi = [self._dev.phi(j) for j in range(self._n)]
        return self._phi


# Device models are shared by every target built on the same (model, data): the design
# matrices are assembled once in HBM (posterior.py:261-264 shares the FeatureCache across
# temperatures the same way), so callers that rebuild a PosteriorTarget per rung or per call
# -- the reference's evidence loop through the drop-in shim -- do not re-upload Phi.
_DEVICE_CACHE: "collections.OrderedDict[tuple, DeviceModel]" = collections.OrderedDict()
_DEVICE_CACHE_MAX = 8


def _fingerprint(model, data):
    import os

    h = hashlib.sha1()
    # the test-only SGP_FORCE_LARGE hook routes a model through the large-d path; a device
    # model that served one routing is not reused for the other
    h.update(os.environ.get("SGP_FORCE_LARGE", "").encode())
    for a in (data.x, data.y):
        a = np.ascontiguousarray(np.asarray(a, dtype=float))
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return (repr(model), h.hexdigest())


def shared_device(model, data):
    """The DeviceModel of (model, data), created on first use and cached (LRU)."""
    key = _fingerprint(model, data)
    dev = _DEVICE_CACHE.get(key)
    if dev is not None:
        _DEVICE_CACHE.move_to_end(key)
        return dev
    dev = DeviceModel(model, data)
    _DEVICE_CACHE[key] = dev
    while len(_DEVICE_CACHE) > _DEVICE_CACHE_MAX:
        _DEVICE_CACHE.popitem(last=False)
    return dev


class PosteriorTarget:
    """Callable bundle for one (model, data, temperature) triple (posterior.py:195-307)."""

    def __init__(self, model: ModelSpec, data: Dataset, tau: float = 1.0, *, _shared=None):
        if not 0.0 <= tau <= 1.0:
            raise ValueError(f"temperature must lie in [0, 1], got {tau}")
        if model.likelihood == LOGISTIC:
            data.require_binary_targets()
        self.model, self.data, self.tau = model, data, float(tau)
        if _shared is not None:
            self.layout, self.device = _shared
        else:
            self.layout = BlockLayout.from_model(model)
            self.device = shared_device(model, data)
            if self.device.dim != self.layout.dim:
                raise RuntimeError("device layout disagrees with BlockLayout")
        self.cache = FeatureCacheView(self.device, len(model.functions))

    @property
    def dim(self) -> int:
        return self.layout.dim

    def at_temperature(self, tau: float) -> "PosteriorTarget":
        return PosteriorTarget(self.model, self.data, tau, _shared=(self.layout, self.device))

    def initial_point(self) -> np.ndarray:
        q = np.zeros(self.dim)
        if self.model.hyper_transform == "identity":
            for pos in self.layout.hyper_index.values():
                q[pos] = 1.0
        return q

    def at(self, q) -> "PosteriorState":
        return PosteriorState(self, q)

    def log_likelihood(self, q) -> float:
        return -self.at(q).sum_potentials()

    def log_likelihoods(self, qs) -> np.ndarray:
        """Batched ``log_likelihood`` over rows of qs (one launch)."""
        out = self.device.eval(self.tau, qs, nat.EVAL_SUMPOT)
        for code in out["status"]:
            raise_status(int(code), "log_likelihood")
        return -out["sumpot"]


class PosteriorState:
    """Lazy, memoised evaluation at one point (posterior.py:310-542)."""

    def __init__(self, target: PosteriorTarget, q):
        q = np.ascontiguousarray(np.asarray(q, dtype=float))
        if q.shape != (target.dim,):
            raise ValueError(f"expected point of dimension {target.dim}, got {q.shape}")
        if not np.isfinite(q).all():
            raise DivergenceError("non-finite coordinates")
        self.target, self.q = target, q
        self._value = self._grad = self._hess = self._sum = None

    def _run(self, what, name):
        out = self.target.device.eval(self.target.tau, self.q[None, :], what)
        raise_status(int(out["status"][0]), name)
        return out

    def sum_potentials(self) -> float:
        if self._sum is None:
            self._sum = float(self._run(nat.EVAL_SUMPOT, "sum_potentials")["sumpot"][0])
            if not math.isfinite(self._sum):
                raise DivergenceError("non-finite likelihood potential")
        return self._sum

    def potential(self) -> float:
        if self._value is None:
            self._value = float(self._run(nat.EVAL_POTENTIAL, "potential")["pot"][0])
        return self._value

    def gradient(self) -> np.ndarray:
        if self._grad is None:
            self._grad = self._run(nat.EVAL_GRADIENT, "gradient")["grad"][0]
        return self._grad

    def hessian(self) -> np.ndarray:
        if self._hess is None:
            self._hess = self._run(nat.EVAL_HESSIAN, "hessian")["hess"][0]
        return self._hess

    def trace_single(self, w: np.ndarray) -> np.ndarray:
        t, status = self.target.device.trace(self.target.tau, self.q[None, :],
                                             np.asarray(w, dtype=float)[None])
        raise_status(int(status[0]), "trace_single")
        return t[0]

    def trace_pair(self, w1, w2):
        return self.trace_single(w1), self.trace_single(w2)


# -- module-level API (posterior.py:551-579) ----------------------------------


def _split_param(q, tau):
    if isinstance(q, ParamVector):
        return q.values, q.tau
    return np.ascontiguousarray(np.asarray(q, dtype=float)), (1.0 if tau is None else float(tau))


def _resolve(target, model, data, tau):
    if target is not None:
        return target if target.tau == tau else target.at_temperature(tau)
    return PosteriorTarget(model, data, tau)


def neg_log_posterior(q, model, data, *, tau=None, target=None) -> float:
    q, tau = _split_param(q, tau)
    return _resolve(target, model, data, tau).at(q).potential()


def gradient(q, model, data, *, tau=None, target=None) -> np.ndarray:
    q, tau = _split_param(q, tau)
    return _resolve(target, model, data, tau).at(q).gradient()


def hessian(q, model, data, *, tau=None, target=None) -> np.ndarray:
    q, tau = _split_param(q, tau)
    return _resolve(target, model, data, tau).at(q).hessian()


def trace_contractions(w1, w2, q, model, data, *, tau=None, target=None):
    q, tau = _split_param(q, tau)
    st = _resolve(target, model, data, tau).at(q)
    return st.trace_pair(np.asarray(w1, dtype=float), np.asarray(w2, dtype=float))


def potential_derivatives(likelihood, f, y, *, variance_floor=1e-3):
    """Per-sample U and f-derivatives on the device (rrgp.py:351-423)."""
    import torch

    L = nat.lib()
    f = np.asarray(f, dtype=float)
    single = f.ndim == 1
    if single:
        f = f[None, :]
    y = np.atleast_1d(np.asarray(y, dtype=float))
    n, J = f.shape
    code = nat.LIK_LOGISTIC if likelihood == LOGISTIC else nat.LIK_GAUSSIAN_MEANVAR
    want = 1 if code == nat.LIK_LOGISTIC else 2
    if likelihood not in (LOGISTIC, "gaussian_meanvar"):
        raise ValueError(f"unknown likelihood {likelihood!r}")
    if J != want:
        raise ValueError(f"{likelihood} likelihood has {want} latent function(s)")
    tf, ty = nat.dev_f64(f), nat.dev_f64(np.broadcast_to(y, (n,)))
    u, d1 = nat.empty_f64(n), nat.empty_f64(n, J)
    d2, d3 = nat.empty_f64(n, J, J), nat.empty_f64(n, J, J, J)
    nat.check(L.sgp_potential_derivatives(code, n, J, nat.ptr(tf), nat.ptr(ty), float(variance_floor),
                                          nat.ptr(u), nat.ptr(d1), nat.ptr(d2), nat.ptr(d3),
                                          nat.stream()), "sgp_potential_derivatives")
    torch.cuda.synchronize()
    out = tuple(t.cpu().numpy() for t in (u, d1, d2, d3))
    if single:
        return tuple(a[0] for a in out)
    return out


# -- constant-Hessian Gaussian target (reference tests/conftest.py:14-61) -------


class QuadraticState:
    """State of a QuadraticTarget, evaluated on the device (SGP_LIK_QUADRATIC):
    U = 0.5 (q-m)^T P (q-m) - tau c, gradient P (q-m), Hessian P, dH/dq = 0."""

    def __init__(self, target, q):
        self.target = target
        self.q = np.ascontiguousarray(np.asarray(q, dtype=float))
        if self.q.shape != (target.dim,):
            raise ValueError(f"expected point of dimension {target.dim}, got {self.q.shape}")
        self._out = None

    def _eval(self):
        if self._out is None:
            out = self.target.device.eval(self.target.tau, self.q[None, :],
                                          nat.EVAL_POTENTIAL | nat.EVAL_GRADIENT | nat.EVAL_HESSIAN)
            raise_status(int(out["status"][0]), "quadratic target")
            self._out = out
        return self._out

    def potential(self):
        return float(self._eval()["pot"][0])

    def gradient(self):
        return self._eval()["grad"][0]

    def hessian(self):
        return self._eval()["hess"][0]

    def sum_potentials(self):
        return -self.target.loglik_const

    def trace_single(self, w):
        t, status = self.target.device.trace(self.target.tau, self.q[None, :], np.asarray(w, dtype=float)[None])
        raise_status(int(status[0]), "trace_single")
        return t[0]


class QuadraticTarget:
    """Gaussian 'posterior' with constant Hessian, injectable into the sampler and the
    evidence machinery exactly like the reference's test fake (tests/conftest.py:36-61),
    but evaluated by libsgp so the device sampler can run it (no CPU fallback)."""

    def __init__(self, precision, mean=None, loglik_const=0.0, tau=1.0, *, _device=None):
        self.precision = np.ascontiguousarray(np.asarray(precision, dtype=float))
        self.dim = self.precision.shape[0]
        self.mean = np.zeros(self.dim) if mean is None else np.asarray(mean, dtype=float)
        self.loglik_const = float(loglik_const)
        self.tau = float(tau)
        self.device = _device if _device is not None else DeviceModel(
            None, None, quadratic=(self.precision, self.mean, self.loglik_const))

    def initial_point(self):
        return np.zeros(self.dim)

    def at(self, q):
        return QuadraticState(self, q)

    def at_temperature(self, tau):
        return QuadraticTarget(self.precision, self.mean, self.loglik_const, tau, _device=self.device)

    def log_likelihood(self, q):
        return self.loglik_const

    def log_likelihoods(self, qs):
        return np.full(np.atleast_2d(qs).shape[0], self.loglik_const)


# -- dense finite-difference trace oracle (posterior.py:582-615) ---------------


def dense_oracle(w, q, model: ModelSpec, data: Dataset, *, tau=None, target=None, step: float = 1e-5,
                 dim_cap: int = 200):
    """Trace contraction t_i = sum(W o dH/dq_i) from central differences of the Hessian,
    the reference's self-check of trace_single.  The 2d perturbed Hessians are evaluated
    in one batched device call instead of 2d sequential ones."""
    q, tau = _split_param(q, tau)
    target = _resolve(target, model, data, tau)
    d = target.dim
    if d > dim_cap:
        raise ValueError(f"dense_oracle guarded to d <= {dim_cap}, got d = {d}")
    w = np.asarray(w, dtype=float)
    w = 0.5 * (w + w.T)
    hs = np.array([step * max(1.0, abs(q[i])) for i in range(d)])
    pts = np.repeat(q[None, :], 2 * d, axis=0)
    idx = np.arange(d)
    pts[2 * idx, idx] += hs
    pts[2 * idx + 1, idx] -= hs
    out = target.device.eval(target.tau, pts, nat.EVAL_HESSIAN)
    for code in out["status"]:
        raise_status(int(code), "dense_oracle")
    hess = out["hess"]
    t = np.empty(d)
    for i in range(d):
        dh = (hess[2 * i] - hess[2 * i + 1]) / (2.0 * hs[i])
        t[i] = float(np.sum(w * dh))
    return t
