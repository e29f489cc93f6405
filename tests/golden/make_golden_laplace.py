"""Golden values for the Laplace evidence oracles, produced
by the UNMODIFIED reference (build container only):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_laplace.py

Writes tests/golden/laplace.npz: the conjugate fixture of the reference's
tests/conftest.py:102-125 (nl-mean, n = 40, 8 features) and a small logistic
problem; laplace_full at fixed hyperparameters and laplace_grid_oracle on
coarse grids (evidence.py:277-426).
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from softabs_gp import evidence, rrgp  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(5)
    n, m = 40, 8
    x = rng.standard_normal((n, 1))
    y = np.sin(1.5 * x[:, 0]) + 0.3 * rng.standard_normal(n)
    data = rrgp.Dataset(x, y)
    fixed = rrgp.build_model("nl-mean", x, feature_count=m, intercept_variance=1e-4,
                             fixed_hypers={"c_g": 1.3, "sigma_g": 2.1, "c_l": 1.0})
    free = rrgp.build_model("nl-mean", x, feature_count=m, intercept_variance=1e-4)
    out = {"conj_x": x, "conj_y": y}
    out["laplace_full_fixed"] = evidence.laplace_full(fixed, data)
    g1 = evidence.GridSpec(c_max=2.6, c_mesh=2.6, sigma_max=4.2, sigma_mesh=4.2, pinned=(("c_l", 1.0),))
    out["grid_single"] = evidence.laplace_grid_oracle(free, data, g1)
    g2 = evidence.GridSpec(c_max=2.0, c_mesh=0.5, sigma_max=2.0, sigma_mesh=0.5, pinned=(("c_l", 1.0),))
    out["grid_conj_4x4"] = evidence.laplace_grid_oracle(free, data, g2)
    # logistic (all three hypers carried; c_l pinned)
    ld, _ = rrgp.simulate_logistic(1, n=60, seed=3)
    lm = rrgp.build_model("logistic", ld.x, feature_count=8)
    out["logi_x"], out["logi_y"] = ld.x, ld.y
    g3 = evidence.GridSpec(c_max=3.0, c_mesh=1.0, sigma_max=3.0, sigma_mesh=1.0, pinned=(("c_l", 1.0),))
    out["grid_logi_3x3"] = evidence.laplace_grid_oracle(lm, ld, g3)
    out["laplace_full_logi"] = evidence.laplace_full(lm, ld)
    np.savez_compressed(os.path.join(OUT, "laplace.npz"), **out)
    for k, v in out.items():
        if np.ndim(v) == 0:
            print(k, float(v))


if __name__ == "__main__":
    main()
