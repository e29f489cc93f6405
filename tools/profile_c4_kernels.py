"""Per-kernel device time of C4 moves (CUPTI activity records through torch.profiler; no
ncu replay): one chain, one MH move of --leapfrogs leapfrogs after a warm-up move.  Prints
each kernel's share of device time, launches, mean duration, and the host-side gap (wall time
not covered by kernels).  Usage: python tools/profile_c4_kernels.py [--leapfrogs 5] [--order parallel]"""
import argparse
import json
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2511_06407_b200.posterior import PosteriorTarget  # noqa: E402
from paper_2511_06407_b200.sampler import ChainConfig, DeviceChains  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--leapfrogs", type=int, default=5)
ap.add_argument("--order", default="refine")
ap.add_argument("--out", default=None)
args = ap.parse_args()

model, data = bench.workload_c4()
target = PosteriorTarget(model, data)
d = target.dim
cfg = ChainConfig(epsilon=1e-4, leapfrogs=args.leapfrogs, moves=1, burnin=0, warm_order=args.order)
ch = DeviceChains(target.device, np.ones(1), cfg)
ch.set_q(np.zeros((1, d)))
ch.init()
rng = np.random.default_rng(0)
ch.run(1, rng.standard_normal((1, 1, d)), np.log(rng.uniform(size=(1, 1))), move_offset=0)
torch.cuda.synchronize()
z, lu = rng.standard_normal((1, 1, d)), np.log(rng.uniform(size=(1, 1)))
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    ch.run(1, z, lu, move_offset=1)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
rows = {}
for ev in prof.events():
    if str(getattr(ev, "device_type", "")).endswith("CUDA"):
        r = rows.setdefault(ev.name, [0, 0.0])
        r[0] += 1
        r[1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v[1] for v in rows.values())
print(f"wall {wall * 1e3:.1f} ms for {args.leapfrogs} leapfrogs ({wall * 1e3 / args.leapfrogs:.1f} ms/lf); "
      f"kernel time {tot / 1e3:.1f} ms ({tot / 1e3 / args.leapfrogs:.1f} ms/lf); launches {sum(v[0] for v in rows.values())}")
out = []
for name, (n, us) in sorted(rows.items(), key=lambda kv: -kv[1][1]):
    out.append({"kernel": name[:90], "launches": n, "ms": us / 1e3, "share": us / tot, "us_per_launch": us / n})
    if len(out) <= 25:
        print(f"{us / tot * 100:6.2f}%  {us / 1e3:9.2f} ms  {n:7d}  {us / n:9.1f} us  {name[:90]}")
if args.out:
    json.dump({"wall_ms": wall * 1e3, "leapfrogs": args.leapfrogs, "kernel_ms": tot / 1e3, "kernels": out},
              open(args.out, "w"), indent=1)
