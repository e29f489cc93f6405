"""ctypes binding of libsgp.so (the C ABI in include/sgp.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no CPU fallback: every device entry point raises if the library or a
CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsgp.so")

# return / status codes (include/sgp.h)
SGP_OK = 0
SGP_EINVAL = -1
STATUS_OK = 0
STATUS_DIVERGENCE = 1
STATUS_DOMAIN = 2
STATUS_JACOBI = 3
STATUS_STALL_P = 4
STATUS_STALL_Q = 5
STATUS_CHAIN_START = 6
STATUS_FIRST_MOVE = 7

LIK_LOGISTIC = 0
LIK_GAUSSIAN_MEANVAR = 1
LIK_QUADRATIC = 2
KERNEL_GAUSSIAN = 0
KERNEL_LINEAR = 1
TRANSFORM_LOG = 0
TRANSFORM_IDENTITY = 1

METRIC_CODES = {"softabs-dynamic": 0, "softabs-static": 1, "euclidean": 2}
ORDER_CODES = {"cyclic": 0, "parallel": 1, "refine": 2, "dc": 3}
PATH_CODES = {"auto": 0, "latency": 1}

EVAL_POTENTIAL = 1
EVAL_GRADIENT = 2
EVAL_HESSIAN = 4
EVAL_SUMPOT = 8

W_W1, W_W2, W_W2_MINUS_W1 = 1, 2, 3

c_dp = ctypes.POINTER(ctypes.c_double)
c_ip = ctypes.POINTER(ctypes.c_int)
c_u8p = ctypes.POINTER(ctypes.c_uint8)


class KernelDesc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("covariate", ctypes.c_int), ("features", ctypes.c_int),
                ("half_width", ctypes.c_double)]


class ModelDesc(ctypes.Structure):
    _fields_ = [
        ("likelihood", ctypes.c_int),
        ("n_rows", ctypes.c_int),
        ("n_cols", ctypes.c_int),
        ("h_x", c_dp),
        ("h_y", c_dp),
        ("n_functions", ctypes.c_int),
        ("n_kernels", ctypes.c_int * 2),
        ("kernels", ctypes.POINTER(KernelDesc) * 2),
        ("transform", ctypes.c_int),
        ("intercept_variance", ctypes.c_double),
        ("variance_floor", ctypes.c_double),
        ("hyper_sampled", ctypes.c_int * 3),
        ("hyper_fixed", ctypes.c_double * 3),
        ("prior_alpha", ctypes.c_double * 3),
        ("prior_beta", ctypes.c_double * 3),
        ("quad_dim", ctypes.c_int),
        ("h_precision", c_dp),
        ("h_mean", c_dp),
        ("loglik_const", ctypes.c_double),
    ]


class ChainState(ctypes.Structure):
    _fields_ = [("n_chains", ctypes.c_int), ("q", ctypes.c_void_p), ("psi", ctypes.c_void_p),
                ("lam", ctypes.c_void_p), ("tau", ctypes.c_void_p), ("since", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("scratch", ctypes.c_void_p)]


class ChainConfigC(ctypes.Structure):
    _fields_ = [("epsilon", ctypes.c_double), ("leapfrogs", ctypes.c_int), ("kappa", ctypes.c_double),
                ("zeta", ctypes.c_double), ("fp_max_iters", ctypes.c_int), ("fp_tol", ctypes.c_double),
                ("gs_interval", ctypes.c_int), ("sweep_cap", ctypes.c_int), ("metric", ctypes.c_int),
                ("warm_order", ctypes.c_int), ("cold_order", ctypes.c_int), ("path", ctypes.c_int)]


class GridSpecC(ctypes.Structure):
    _fields_ = [("c_max", ctypes.c_double), ("c_mesh", ctypes.c_double), ("sigma_max", ctypes.c_double),
                ("sigma_mesh", ctypes.c_double), ("n_pinned", ctypes.c_int),
                ("pinned_pos", ctypes.c_int * 3), ("pinned_value", ctypes.c_double * 3),
                ("gtol", ctypes.c_double), ("max_iters", ctypes.c_int), ("memory", ctypes.c_int),
                ("mode", ctypes.c_int)]


GRID_MODES = {"reference": 0, "robust": 1}


class MoveRecords(ctypes.Structure):
    _fields_ = [("logpost", ctypes.c_void_p), ("h_before", ctypes.c_void_p),
                ("h_after", ctypes.c_void_p), ("sweeps_mean", ctypes.c_void_p),
                ("wall_ms", ctypes.c_void_p), ("accept", ctypes.c_void_p),
                ("divergent", ctypes.c_void_p), ("q", ctypes.c_void_p)]


class LeapfrogDiag(ctypes.Structure):
    _fields_ = [("fp_p_iters", ctypes.c_void_p), ("fp_q_iters", ctypes.c_void_p),
                ("sweeps", ctypes.c_void_p)]


_lib = None


def lib():
    """Load libsgp.so; raise loudly if it is missing or no GPU is present."""
    global _lib
    if _lib is not None:
        return _lib
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_06407_b200 needs a CUDA device (B200, sm_100a); none found")
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built; run __graft_entry__.build()")
    torch.cuda.init()
    L = ctypes.CDLL(LIB_PATH)
    vp, i, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    sig = {
        "sgp_model_create": (i, [ctypes.POINTER(ModelDesc), ctypes.POINTER(vp)]),
        "sgp_model_destroy": (i, [vp]),
        "sgp_model_dim": (i, [vp]),
        "sgp_model_rows": (i, [vp]),
        "sgp_model_features": (i, [vp, i]),
        "sgp_model_phi": (i, [vp, i, vp, vp]),
        "sgp_scratch_doubles": (ctypes.c_size_t, [vp]),
        "sgp_eval": (i, [vp, i, vp, vp, i, vp, vp, vp, vp, vp, vp, vp]),
        "sgp_trace": (i, [vp, i, vp, vp, vp, vp, vp, vp, vp]),
        "sgp_potential_derivatives": (i, [i, i, i, vp, vp, d, vp, vp, vp, vp, vp]),
        "sgp_eigh_cold": (i, [i, i, vp, d, i, vp, vp, vp, vp]),
        "sgp_eigh_dc": (i, [i, i, vp, vp, vp, vp]),
        "sgp_eigh_warm": (i, [i, i, vp, vp, vp, i, d, i, i, vp, vp, vp, vp, vp]),
        "sgp_mgs": (i, [i, i, vp, vp]),
        "sgp_t_matrix": (i, [i, i, vp, d, vp, vp]),
        "sgp_metric_w": (i, [i, i, vp, vp, d, vp, i, vp, vp]),
        "sgp_metric_apply": (i, [i, i, vp, vp, d, vp, i, vp, vp]),
        "sgp_metric_scalars": (i, [i, i, vp, vp, d, vp, vp, vp, vp]),
        "sgp_leapfrog": (i, [vp, ctypes.POINTER(ChainConfigC), ctypes.POINTER(ChainState), vp,
                             ctypes.POINTER(LeapfrogDiag), vp]),
        "sgp_chain_init": (i, [vp, ctypes.POINTER(ChainConfigC), ctypes.POINTER(ChainState), vp]),
        "sgp_run_moves": (i, [vp, ctypes.POINTER(ChainConfigC), ctypes.POINTER(ChainState), i, i, vp,
                              vp, ctypes.POINTER(MoveRecords), vp]),
        "sgp_ladder_walk": (i, [vp, ctypes.POINTER(ChainConfigC), ctypes.POINTER(ChainState), i, vp, i, i, vp,
                                vp, vp, vp]),
        "sgp_device_info": (i, [c_ip, c_ip, c_ip]),
        "sgp_version": (ctypes.c_char_p, []),
        "sgp_debug_phase_cycles": (i, [vp, i]),
        "sgp_debug_rotation_check": (i, [ctypes.c_longlong, ctypes.c_ulonglong, vp]),
        "sgp_laplace_grid": (i, [vp, ctypes.POINTER(GridSpecC), i, vp, vp, vp, vp]),
        "sgp_laplace_full": (i, [vp, d, vp, d, i, d, i, vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc, what):
    if rc != SGP_OK:
        raise RuntimeError(f"libsgp: {what} failed with code {rc}")


def stream():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def dev_f64(a):
    """Host array -> contiguous float64 CUDA tensor."""
    import torch

    return torch.from_numpy(np.array(a, dtype=np.float64, copy=True, order="C")).to("cuda")


def empty_f64(*shape):
    import torch

    return torch.empty(shape, dtype=torch.float64, device="cuda")


def zeros_i32(*shape):
    import torch

    return torch.zeros(shape, dtype=torch.int32, device="cuda")
