"""C4 building blocks only (no chain): Hessian evaluation and trace contraction,
for an ncu launch list of the large-d path.

    ncu --metrics gpu__time_duration.sum --csv python tools/profile_c4_parts.py
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
target = PosteriorTarget(rrgp.build_model("nl-meanvar", data.x), data)
d = target.dim
q = 0.01 * np.random.default_rng(0).standard_normal(d)
dev = target.device
for _ in range(2):
    dev.eval(1.0, q[None], nat.EVAL_HESSIAN)
    dev.trace(1.0, q[None], np.eye(d)[None])
torch.cuda.synchronize()
print("done", d)
