"""Model constructors matching tests/golden/make_golden.py, and fixture loading."""

from __future__ import annotations

import os

import numpy as np

from paper_2511_06407_b200 import rrgp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def model_for(name, x):
    if name == "logistic_small" or name.startswith("chain_c1"):
        return rrgp.build_model("logistic", x)
    if name in ("meanvar_toy", "chain_meanvar_tau"):
        return rrgp.build_model("nl-meanvar", x, feature_count=8)
    if name == "conjugate":
        return rrgp.build_model("nl-mean", x, feature_count=8, intercept_variance=1e-4,
                                fixed_hypers={"c_g": 1.3, "sigma_g": 2.1, "c_l": 1.0})
    if name == "identity_meanvar":
        return rrgp.build_model("nl-meanvar", x, feature_count=6, hyper_transform="identity")
    if name in ("chain_small_static", "chain_small_euclid", "ti_small"):
        return rrgp.build_model("logistic", x, feature_count=10)
    raise KeyError(name)


def case(name):
    g = load(name)
    data = rrgp.Dataset(g["x"], g["y"])
    return g, model_for(name, g["x"]), data


POINT_CASES = ("logistic_small", "meanvar_toy", "conjugate", "identity_meanvar")
CHAIN_CASES = ("chain_c1_eps1e-2", "chain_c1_eps1e-3", "chain_c1_eps15e-3",
               "chain_small_static", "chain_small_euclid", "chain_meanvar_tau")


def rel_err(approx, exact):
    """max-abs error over max(1, max|exact|) (reference tests/conftest.py:170-174)."""
    approx = np.asarray(approx, dtype=float)
    exact = np.asarray(exact, dtype=float)
    scale = max(1.0, float(np.max(np.abs(exact)))) if exact.size else 1.0
    return float(np.max(np.abs(approx - exact))) / scale if exact.size else 0.0
