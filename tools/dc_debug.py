"""Stage-by-stage check of sgp_dc.cuh on one matrix (SGP_DC_DUMP hook): tridiagonal T vs A's
spectrum, D&C of T vs scipy, back-transform."""
import os
import sys

import numpy as np
import scipy.linalg as sl

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
os.makedirs("gpurun_out", exist_ok=True)
sys.path.insert(0, ".")
pre = "gpurun_out/dc"
os.environ["SGP_DC_DUMP"] = pre
from paper_2511_06407_b200 import metric as M  # noqa: E402

a = np.random.default_rng(n).standard_normal((n, n))
a = 0.5 * (a + a.T)
lam, psi = M.eigh_dc(a)
ld = (n + 3) & ~3
rd = lambda t, cnt: np.fromfile(f"{pre}_{t}.bin")[:cnt]
dv, ev, tau = rd("dv", n), rd("ev", n), rd("tau", n)
V = rd("V", n * ld).reshape(n, ld)[:, :n]
D, Z = rd("D", n), rd("Z", n * ld).reshape(n, ld)[:, :n]
ref = np.linalg.eigvalsh(a)
tt = sl.eigvalsh_tridiagonal(dv, ev[:n - 1])
print("stage1 T spectrum vs A:", np.max(np.abs(np.sort(tt) - ref)))
T = np.diag(dv) + np.diag(ev[:n - 1], 1) + np.diag(ev[:n - 1], -1)
print("stage2 D vs T spectrum:", np.max(np.abs(np.sort(D) - tt)))
print("stage2 residual |T Z - Z D|:", np.max(np.abs(T @ Z - Z * D)), " orth", np.max(np.abs(Z.T @ Z - np.eye(n))))
Q = np.eye(n)
for c in range(n - 1):
    v = V[:, c]
    Q = Q @ (np.eye(n) - tau[c] * np.outer(v, v))
print("stage1 |Q T Q^T - A|:", np.max(np.abs(Q @ T @ Q.T - a)))
print("final lam vs ref:", np.max(np.abs(lam - ref)), " residual", np.max(np.abs(a @ psi - psi * lam)))
