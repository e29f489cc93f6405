"""Laplace-grid evidence oracle throughput: device vs the
CPU restatement of the reference (serpentine, one process).

    python tools/bench_grid.py [--model nl-mean] [--cpu-nodes 12]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="logistic")
ap.add_argument("--n", type=int, default=500)
ap.add_argument("--cpu-nodes", type=int, default=12)
ap.add_argument("--c-mesh", type=float, default=0.01)
ap.add_argument("--sigma-mesh", type=float, default=0.02)
ap.add_argument("--mode", default="reference", choices=["reference", "robust"])
args = ap.parse_args()

from paper_2511_06407_b200 import rrgp  # noqa: E402
from paper_2511_06407_b200.evidence import GridSpec, laplace_grid_nodes  # noqa: E402

if args.model == "logistic":
    # the paper's grid-oracle use: simulated logistic, one covariate
    data, _ = rrgp.simulate_logistic(1, n=args.n, seed=0)
else:
    data, _ = rrgp.simulate_meanvar(2, 19, n=args.n, seed=0)
model = rrgp.build_model(args.model, data.x)
spec = GridSpec(c_mesh=args.c_mesh, sigma_mesh=args.sigma_mesh, pinned=(("c_l", 1.0),))
nc, ns = [c.size for c in spec.centers()]
# warm-up on a tiny grid (module load, first launch)
laplace_grid_nodes(model, data, GridSpec(1.0, 0.5, 1.0, 0.5, pinned=(("c_l", 1.0),)))
t0 = time.perf_counter()
v, st, it = laplace_grid_nodes(model, data, spec, mode=args.mode)
gpu_s = time.perf_counter() - t0
print(f"mode {args.mode}: model {args.model} N={args.n}: grid {nc} x {ns} = {nc * ns} nodes on GPU in {gpu_s:.2f} s "
      f"({nc * ns / gpu_s:.0f} nodes/s); failed {int(np.count_nonzero(st))}; L-BFGS iterations "
      f"median {int(np.median(it))}, max {int(np.max(it))}")

import oracle  # noqa: E402

t = oracle.OTarget(model, data)
# first CPU row segment of the same grid (serpentine warm start as the reference)
cm = args.c_mesh
t0 = time.perf_counter()
ov, ost, _ = oracle.laplace_grid_nodes(t, args.cpu_nodes * cm, cm, args.sigma_mesh, args.sigma_mesh,
                                       (("c_l", 1.0),))
cpu_s = (time.perf_counter() - t0) / args.cpu_nodes
print(f"CPU oracle (reference algorithm, 1 process, serpentine): {cpu_s * 1e3:.1f} ms/node -> "
      f"{cpu_s * nc * ns / 3600:.2f} h for the full grid; GPU/CPU node-rate ratio {cpu_s * nc * ns / gpu_s:.0f}x")
print("first nodes GPU vs CPU:", np.round(v[:4], 6), np.round(ov[:4], 6))
