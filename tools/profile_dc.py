"""Kernel split of one sgp_eigh_dc call at d = 2083 (CUPTI activity records via torch.profiler)."""
import collections
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2511_06407_b200 import _native as nat  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2083
a = np.random.default_rng(n).standard_normal((n, n))
a = 0.5 * (a + a.T)
L = nat.lib()
th = torch.tensor(a, dtype=torch.float64, device="cuda")
lam = torch.empty(n, dtype=torch.float64, device="cuda")
psi = torch.empty(n, n, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
L.sgp_eigh_dc(1, n, th.data_ptr(), lam.data_ptr(), psi.data_ptr(), s)  # warm-up (workspace)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    L.sgp_eigh_dc(1, n, th.data_ptr(), lam.data_ptr(), psi.data_ptr(), s)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
first, last = None, None
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        agg[e.name[:60]][0] += 1
        agg[e.name[:60]][1] += e.device_time_total
tot = sum(v for _, v in agg.values())
print(f"n={n}: kernel time {tot / 1e3:.2f} ms")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"  {v / 1e3:8.2f} ms {c:5d}  {k}")
