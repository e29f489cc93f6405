"""Time the reference-order cold Jacobi (sgp_eigh_cold) per sweep at large d."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2511_06407_b200 import metric as M
from paper_2511_06407_b200.metric import JacobiError


def seeded_sym(seed, d):
    rng = np.random.default_rng(seed)
    r = rng.standard_normal((d, d))
    h = 0.02 * (0.5 * (r + r.T))
    base = np.repeat(10.0 * rng.standard_normal(d // 4 + 1), 4)[:d]
    h[np.diag_indices(d)] += base
    return h


for d, caps in ((583, (1, 30)), (2083, (1,))):
    h = seeded_sym(77, d)
    for cap in caps:
        t0 = time.perf_counter()
        try:
            lam, psi, sw = M.static_eigendecompose(h, 1e-13, cap)
        except JacobiError:
            sw = -1
        dt = time.perf_counter() - t0
        print(f"d={d} cap={cap}: sweeps={sw} {dt:.3f} s", flush=True)
