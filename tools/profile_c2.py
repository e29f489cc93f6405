"""Launch k_run_moves once on the C2 workload (for ncu / timing studies).

    python tools/profile_c2.py [--chains Z] [--moves M] [--leapfrogs C] [--order cyclic|parallel]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--chains", type=int, default=148)
ap.add_argument("--moves", type=int, default=1)
ap.add_argument("--leapfrogs", type=int, default=20)
ap.add_argument("--order", default="cyclic")
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--dims", type=int, default=1)
ap.add_argument("--config", default=None, help="a tools/bench_configs.py config name prefix, e.g. C3b")
args = ap.parse_args()

import torch  # noqa: E402

from paper_2511_06407_b200 import rrgp  # noqa: E402
from paper_2511_06407_b200.posterior import PosteriorTarget  # noqa: E402
from paper_2511_06407_b200.sampler import ChainConfig, DeviceChains  # noqa: E402

eps = 1e-3
if args.config:
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import bench_configs  # noqa: E402

    ccfg = next(c for c in bench_configs.CONFIGS if c["name"].startswith(args.config))
    model, data = bench_configs.make(ccfg)
    eps = ccfg["eps"]
    target = PosteriorTarget(model, data)
else:
    data, _ = rrgp.simulate_logistic(args.dims, n=args.n, seed=0)
    target = PosteriorTarget(rrgp.build_model("logistic", data.x), data)
d, Z = target.dim, args.chains
cfg = ChainConfig(epsilon=eps, leapfrogs=args.leapfrogs, moves=1, burnin=0, warm_order=args.order)
ch = DeviceChains(target.device, np.ones(Z), cfg)
ch.set_q(np.zeros((Z, d)))
ch.init()
rng = np.random.default_rng(0)
z = rng.standard_normal((args.moves, Z, d))
lu = np.log(rng.uniform(size=(args.moves, Z)))
tz, tl = torch.from_numpy(z).cuda(), torch.from_numpy(lu).cuda()
q0 = ch.q.clone()
ch.run(args.moves, tz, tl)  # warm-up (clocks, first-launch setup)
ch.q.copy_(q0)
ch.init()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ch.run(args.moves, tz, tl)
e1.record()
e1.synchronize()
dt = e0.elapsed_time(e1) / 1e3
print(f"d={d} Z={Z} moves={args.moves} C={args.leapfrogs}: {dt*1e3:.1f} ms, "
      f"{dt / (args.moves * args.leapfrogs) * 1e3:.3f} ms per leapfrog per chain-batch, "
      f"status nonzero {int(np.count_nonzero(ch.status_host()))}")

import ctypes  # noqa: E402

from paper_2511_06407_b200 import _native as nat  # noqa: E402

L = nat.lib()
L.sgp_debug_phase_cycles.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
L.sgp_debug_phase_cycles(buf, 1)
ch.run(args.moves, z, lu)
torch.cuda.synchronize()
L.sgp_debug_phase_cycles(buf, 0)
names = {0: "W formation", 1: "trace", 2: "state+Hessian", 3: "MGS", 4: "PsiT H Psi", 5: "warm Jacobi",
         8: "cold Jacobi", 10: " trace: build Wp", 11: " trace: per-sample forms", 12: " trace: project", 13: " Hessian lik block",
         14: " state: f + derivatives", 9: "leapfrog total"}
tot = buf[9] or 1
nlf = args.moves * args.leapfrogs
for k, nm in names.items():
    print(f"  {nm:16s} {buf[k] / nlf / 1e3:10.1f} kcyc/leapfrog  {100.0 * buf[k] / tot:5.1f}%")
