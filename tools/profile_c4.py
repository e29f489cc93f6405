"""C4: nl-meanvar on simulate_meanvar(34, 19, n=8192, seed=0), d = 2083.

Times the large-path building blocks and one generalized leapfrog on the device.
    python tools/profile_c4.py [--leapfrogs C] [--order parallel|cyclic]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_06407_b200 import rrgp  # noqa: E402
from paper_2511_06407_b200.posterior import PosteriorTarget  # noqa: E402
from paper_2511_06407_b200.sampler import ChainConfig, DeviceChains  # noqa: E402
from paper_2511_06407_b200 import _native as nat  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--leapfrogs", type=int, default=2)
ap.add_argument("--order", default="parallel")
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--cont", type=int, default=34)
args = ap.parse_args()

t0 = time.perf_counter()
data, _ = rrgp.simulate_meanvar(args.cont, 19, n=args.n, seed=0)
model = rrgp.build_model("nl-meanvar", data.x)
target = PosteriorTarget(model, data)
d = target.dim
print(f"model d={d} N={args.n} built in {time.perf_counter() - t0:.1f}s", flush=True)


def timed(label, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    print(f"{label:40s} {dt * 1e3:10.2f} ms", flush=True)
    return dt


q = 0.01 * np.random.default_rng(0).standard_normal(d)
dev = target.device
timed("eval potential+gradient", lambda: dev.eval(1.0, q[None], nat.EVAL_POTENTIAL | nat.EVAL_GRADIENT))
th = timed("eval + Hessian (3 DMMA GEMMs)", lambda: dev.eval(1.0, q[None], nat.EVAL_HESSIAN))
F_h = 2 * args.n * (1040 * 1040 * 3)
print(f"   Hessian canonical {F_h / 1e9:.1f} GFLOP -> {F_h / th / 1e12:.2f} TF/s incl. host round trips")
w = np.eye(d)
tt = timed("trace contraction (2 DMMA GEMMs)", lambda: dev.trace(1.0, q[None], w[None]))
F_t = 2 * args.n * (2080 ** 2)
print(f"   trace canonical {F_t / 1e9:.1f} GFLOP -> {F_t / tt / 1e12:.2f} TF/s incl. host round trips")

cfg = ChainConfig(epsilon=1e-4, leapfrogs=args.leapfrogs, moves=1, burnin=0, warm_order=args.order)
ch = DeviceChains(target.device, np.ones(1), cfg)
ch.set_q(np.zeros((1, d)))
t = time.perf_counter()
ch.init()
print(f"chain init (cold decomposition, {args.order}) {time.perf_counter() - t:10.2f} s   status {ch.status_host()}",
      flush=True)
rng = np.random.default_rng(1)
for mv in range(2):
    z = rng.standard_normal((1, 1, d))
    lu = np.log(rng.uniform(size=(1, 1)))
    torch.cuda.synchronize()
    t = time.perf_counter()
    bufs = ch.run(1, z, lu)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"move {mv}: {args.leapfrogs} leapfrogs in {dt:.2f} s -> {dt / args.leapfrogs * 1e3:.1f} ms per leapfrog; "
          f"accept {int(bufs['accept'][0, 0])} sweeps_mean {float(bufs['sweeps_mean'][0, 0]):.2f} "
          f"status {ch.status_host()}", flush=True)
    F_lf = 1.15e12
    print(f"   canonical 1.15 TFLOP/leapfrog -> {F_lf / (dt / args.leapfrogs) / 1e12:.2f} TF/s", flush=True)
