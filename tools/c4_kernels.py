"""Launch the C4 (d = 2083, N = 8192) assembly and GEMM kernels once each, for ncu.

Builds the nl-meanvar model on simulate_meanvar(34, 19, n=8192, seed=0) (k_assemble_phi,
k_pad_phi: HBM-bound), then one Hessian evaluation (DMMA GEMMs for the likelihood blocks,
posterior.py:457) and one trace contraction (DMMA GEMMs Y = Phi W, posterior.py:500-502).

    ncu --metrics <...> -k regex:'k_assemble_phi|k_pad_phi|k_gemm' python tools/c4_kernels.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_06407_b200 import _native as nat  # noqa: E402
from paper_2511_06407_b200 import rrgp  # noqa: E402
from paper_2511_06407_b200.posterior import PosteriorTarget  # noqa: E402

data, _ = rrgp.simulate_meanvar(34, 19, n=8192, seed=0)
model = rrgp.build_model("nl-meanvar", data.x)
target = PosteriorTarget(model, data)
d = target.dim
q = 0.01 * np.random.default_rng(0).standard_normal((1, d))
out = target.device.eval(1.0, q, nat.EVAL_HESSIAN)
w = np.eye(d)[None]
t, st = target.device.trace(1.0, q, w)
torch.cuda.synchronize()
print("d", d, "hessian finite", bool(np.isfinite(out["hess"]).all()), "trace status", int(st[0]))
