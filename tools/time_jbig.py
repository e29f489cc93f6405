"""Time the grid-wide reference-order cold Jacobi (sgp_eigh_cold at d > 256) and check it
against the C restatement of _jacobi.jacobi_sweeps at d = 583."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import oracle
from paper_2511_06407_b200 import metric as M
from paper_2511_06407_b200.metric import JacobiError
sys.path.insert(0, "tests")
from test_gpu_jbig import seeded_sym

for d in [int(a) for a in sys.argv[1:]] or [583, 2083]:
    h = seeded_sym(77, d)
    t0 = time.perf_counter()
    lam, psi, sw = M.static_eigendecompose(h, 1e-13)
    dt = time.perf_counter() - t0
    print(f"d={d}: sweeps={sw} {dt:.3f} s ({dt / max(sw, 1):.3f} s/sweep)", flush=True)
    if d <= 600:
        t0 = time.perf_counter()
        lam_o, psi_o, sw_o = oracle.cold_eigh(h, 1e-13)
        print(f"  oracle {time.perf_counter() - t0:.1f} s sweeps={sw_o} lam_equal={np.array_equal(lam, lam_o)} "
              f"psi_equal={np.array_equal(psi, psi_o)} maxdiff={np.max(np.abs(psi - psi_o)):.3e}", flush=True)
