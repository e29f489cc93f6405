"""Dump C4 warm-decomposition inputs A = Psi^T H Psi for offline analysis (build container):
(a) the first warm call of the chain's first leapfrog (cold basis at q0, Hessian at the
golden q1), (b) one after 20 moves of C = 10 (basis of the frame, Hessian at a nearby point).
Writes float32? no: float64 npy of the lower triangle + diagonal into gpurun_out/."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import bench  # noqa: E402
from golden_cases import load  # noqa: E402
from paper_2511_06407_b200 import metric as M  # noqa: E402
from paper_2511_06407_b200.posterior import PosteriorTarget  # noqa: E402
from paper_2511_06407_b200.sampler import ChainConfig, DeviceChains  # noqa: E402

model, data = bench.workload_c4()
t = PosteriorTarget(model, data)
d = t.dim
g = load("c4_chain")
q0 = t.initial_point()
m0 = M.metric_from_hessian(t.at(q0).hessian(), 1.0, 1e-13)
h1 = t.at(g["q1"]).hessian()
A = m0.vectors.T @ h1 @ m0.vectors
np.save("gpurun_out/warmA_start.npy", A.astype(np.float32))
np.save("gpurun_out/warmA_start_h1fro.npy", np.array([np.linalg.norm(h1)]))
cfg = ChainConfig(epsilon=1e-4, leapfrogs=10, moves=1, burnin=0, warm_order="parallel")
ch = DeviceChains(t.device, np.ones(1), cfg)
ch.set_q(np.zeros((1, d)))
ch.init()
rng = np.random.default_rng(1)
for k in range(20):
    ch.run(1, rng.standard_normal((1, 1, d)), np.log(rng.uniform(size=(1, 1))), move_offset=k)
torch.cuda.synchronize()
q = ch.q.cpu().numpy()[0]
psi = ch.psi.cpu().numpy()[0]
p = rng.standard_normal(d)
h = t.at(q + 1e-4 * (psi @ p) / np.sqrt(d)).hessian()
A2 = psi.T @ h @ psi
np.save("gpurun_out/warmA_move20.npy", A2.astype(np.float32))
np.save("gpurun_out/warmA_move20_hfro.npy", np.array([np.linalg.norm(h)]))
print("status", ch.status_host(), "saved")
