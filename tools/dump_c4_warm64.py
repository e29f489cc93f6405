"""Dump the first warm-decomposition input A = Psi^T H Psi of a C4 leapfrog in float64
(build-container analysis of near-degenerate eigenvalue groups), plus ||H||_F."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import bench  # noqa: E402
from golden_cases import load  # noqa: E402
from paper_2511_06407_b200 import metric as M  # noqa: E402
from paper_2511_06407_b200.posterior import PosteriorTarget  # noqa: E402

model, data = bench.workload_c4()
t = PosteriorTarget(model, data)
g = load("c4_chain")
m0 = M.metric_from_hessian(t.at(t.initial_point()).hessian(), 1.0, 1e-13)
h1 = t.at(g["q1"]).hessian()
np.save("gpurun_out/warmA64.npy", m0.vectors.T @ h1 @ m0.vectors)
np.save("gpurun_out/warmA64_hfro.npy", np.array([np.linalg.norm(h1)]))
np.save("gpurun_out/warmA64_lam0.npy", m0.eigenvalues)
print("ok")
