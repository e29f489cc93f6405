"""Single-chain latency (ms per generalized leapfrog) on the fused one-CTA path vs the large
(host-sequenced, whole-GPU) path, warm orders cyclic / refine, for the SURVEY.md 8(d) shapes."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from bench_configs import CONFIGS, make  # noqa: E402

from paper_2511_06407_b200.posterior import PosteriorTarget  # noqa: E402
from paper_2511_06407_b200.sampler import ChainConfig, DeviceChains  # noqa: E402

names = sys.argv[1:] or ["C1 logistic D=1", "C3a logistic NMES", "C3b nl-meanvar NMES"]
LF = 20
for cfg in [c for c in CONFIGS if c["name"] in names]:
    for large in (0, 1):

        for order in ("cyclic", "parallel", "refine"):
            if order == "refine" and not large:
                continue
            model, data = make(cfg)
            t = PosteriorTarget(model, data)
            d = t.dim
            cc = ChainConfig(epsilon=cfg["eps"], leapfrogs=LF, moves=1, burnin=0, warm_order=order,
                             path="latency" if large else "auto")
            ch = DeviceChains(t.device, np.ones(1), cc)
            ch.set_q(np.zeros((1, d)))
            ch.init()
            rng = np.random.default_rng(0)
            ch.run(1, rng.standard_normal((1, 1, d)), np.log(rng.uniform(size=(1, 1))))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ch.run(1, rng.standard_normal((1, 1, d)), np.log(rng.uniform(size=(1, 1))), move_offset=1)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / LF * 1e3
            print(f"{cfg['name']:24s} d={d:4d} {'large' if large else 'fused':5s} {order:8s} "
                  f"{dt:8.2f} ms/leapfrog  status {ch.status_host()[0]}", flush=True)
