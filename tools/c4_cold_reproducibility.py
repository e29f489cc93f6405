"""Is the reference cold decomposition at C4 reproducible?  Runs the UNMODIFIED reference
(build container) on the C4 chain-start Hessian: mode "base" as is (OPENBLAS_NUM_THREADS
set by the caller), mode "pert" after a 1-ulp change of 50 symmetric off-diagonal pairs, and
compares the natural-order eigenvalues with tests/golden/c4_chain.npz (generated with 6
BLAS threads).  Result: profiles/r2_c4_cold_reproducibility.md."""
import os, sys, time
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_sens")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np
from softabs_gp import rrgp, posterior, metric
data, _ = rrgp.simulate_meanvar(34, 19, n=8192, seed=0)
model = rrgp.build_model("nl-meanvar", data.x)
t = posterior.PosteriorTarget(model, data)
h = t.at(np.zeros(t.dim)).hessian()
a = 0.5 * (h + h.T)
d = a.shape[0]
diag = np.diagonal(a)
u, cnt = np.unique(diag, return_counts=True)
print("distinct diag values", len(u), "max multiplicity", cnt.max(), "repeated entries", int((cnt[cnt > 1]).sum()), flush=True)
mode = sys.argv[1]
if mode == "pert":
    rng = np.random.default_rng(1)
    idx = rng.integers(0, d, size=(50, 2))
    for i, j in idx:
        a[i, j] = np.nextafter(a[i, j], np.inf); a[j, i] = a[i, j]
g = np.load("/root/repo/tests/golden/c4_chain.npz")
t0 = time.perf_counter()
lam, psi, sw = metric.static_eigendecompose(a, 1e-13)
print(mode, "sweeps", sw, time.perf_counter() - t0, "s", flush=True)
ref = g["cold_lam"]
print(mode, "rel natural-order diff", np.max(np.abs(lam - ref)) / np.max(np.abs(ref)),
      "sorted diff", np.max(np.abs(np.sort(lam) - np.sort(ref))) / np.max(np.abs(ref)), flush=True)
np.save(f"/tmp/sens/lam_{mode}.npy", lam)
