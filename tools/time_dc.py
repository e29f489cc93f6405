"""Device time of sgp_eigh_dc (tridiagonalisation + divide and conquer) vs cuSOLVER syevd
(torch.linalg.eigh, fp64) on the same symmetric matrices; per-stage split with SGP_DC_PROF=1."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_06407_b200 import _native as nat  # noqa: E402

L = nat.lib()
for n in [int(a) for a in sys.argv[1:]] or [583, 1000, 2083]:
    a = np.random.default_rng(n).standard_normal((n, n))
    a = 0.5 * (a + a.T)
    th = torch.tensor(a, dtype=torch.float64, device="cuda")
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    psi = torch.empty(n, n, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    for rep in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        rc = L.sgp_eigh_dc(1, n, th.data_ptr(), lam.data_ptr(), psi.data_ptr(), ctypes_stream := s.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0
        t_dc = e0.elapsed_time(e1)
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        w, v = torch.linalg.eigh(th)
        e1.record()
        torch.cuda.synchronize()
        t_cs = e0.elapsed_time(e1)
    err = (lam - w).abs().max().item()
    print(f"n={n}: sgp_eigh_dc {t_dc:.2f} ms (incl. workspace alloc), cuSOLVER eigh {t_cs:.2f} ms, "
          f"max |lam diff| {err:.2e}")
