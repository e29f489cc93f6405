"""Per-config throughput table for SURVEY.md 8(d) (C1, C2, C3a, C3b, C5 models, C4).

GPU: Z chains of the config's model run one MH move of C leapfrogs (device
time of k_run_moves, after a warm-up move); reported as chain-leapfrogs/s and
ms per leapfrog per chain.  CPU: the oracle port of the reference algorithm,
one process per host core (OPENBLAS_NUM_THREADS=1), a bounded number of
leapfrogs per process.  Writes a markdown table to stdout.

    python tools/bench_configs.py [--cpu-leapfrogs 5] [--skip-c4]
"""
import argparse
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def make(cfg):
    from paper_2511_06407_b200 import rrgp

    kind = cfg["kind"]
    if kind == "logistic":
        data, _ = rrgp.simulate_logistic(cfg["D"], n=cfg["N"], seed=0)
        return rrgp.build_model("logistic", data.x), data
    data, _ = rrgp.simulate_meanvar(cfg["cont"], 19, n=cfg["N"], seed=0)
    if kind == "logistic-nmes":
        y = np.where(data.y > np.median(data.y), 1.0, -1.0)
        data = rrgp.Dataset(data.x, y)
        return rrgp.build_model("logistic", data.x), data
    return rrgp.build_model(kind, data.x), data


CONFIGS = [
    {"name": "C1 logistic D=1", "kind": "logistic", "D": 1, "N": 500, "eps": 1e-3, "chains": 1776},
    {"name": "C1 logistic D=2", "kind": "logistic", "D": 2, "N": 500, "eps": 1e-3, "chains": 592},
    {"name": "C1 logistic D=4", "kind": "logistic", "D": 4, "N": 500, "eps": 1e-3, "chains": 296},
    {"name": "C2 logistic N=512", "kind": "logistic", "D": 1, "N": 512, "eps": 1e-3, "chains": 1776},
    {"name": "C3a logistic NMES", "kind": "logistic-nmes", "cont": 2, "N": 2000, "eps": 1e-3, "chains": 296},
    {"name": "C3b nl-meanvar NMES", "kind": "nl-meanvar", "cont": 2, "N": 2000, "eps": 8e-5, "chains": 296},
    {"name": "C5 l-mean", "kind": "l-mean", "cont": 2, "N": 2000, "eps": 1e-4, "chains": 592},
    {"name": "C5 nl-mean", "kind": "nl-mean", "cont": 2, "N": 2000, "eps": 1e-4, "chains": 296},
    {"name": "C5 l-meanvar", "kind": "l-meanvar", "cont": 2, "N": 2000, "eps": 1e-4, "chains": 592},
    {"name": "C5 nl-meanvar", "kind": "nl-meanvar", "cont": 2, "N": 2000, "eps": 8e-5, "chains": 296},
]
C4 = {"name": "C4 nl-meanvar 34+19", "kind": "nl-meanvar", "cont": 34, "N": 8192, "eps": 1e-4, "chains": 1}


def gpu_rate(cfg, leapfrogs, order="cyclic"):
    import torch

    from paper_2511_06407_b200.posterior import PosteriorTarget
    from paper_2511_06407_b200.sampler import ChainConfig, DeviceChains

    model, data = make(cfg)
    target = PosteriorTarget(model, data)
    d, Z = target.dim, cfg["chains"]
    cc = ChainConfig(epsilon=cfg["eps"], leapfrogs=leapfrogs, moves=1, burnin=0, warm_order=order)
    ch = DeviceChains(target.device, np.ones(Z), cc)
    ch.set_q(np.zeros((Z, d)))
    ch.init()
    rng = np.random.default_rng(0)
    z = [rng.standard_normal((1, Z, d)) for _ in range(2)]
    lu = [np.log(rng.uniform(size=(1, Z))) for _ in range(2)]
    ch.run(1, z[0], lu[0])  # warm-up move
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tz, tl = torch.from_numpy(z[1]).cuda(), torch.from_numpy(lu[1]).cuda()
    e0.record()
    bufs = ch.run(1, tz, tl)
    e1.record()
    e1.synchronize()
    dt = e0.elapsed_time(e1) / 1e3
    acc = float(bufs["accept"].float().mean().item())
    st = int(np.count_nonzero(ch.status_host()))
    return d, Z * leapfrogs / dt, dt / leapfrogs * 1e3, acc, st


_T = {}


def _init(cfg):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        import threadpoolctl

        threadpoolctl.threadpool_limits(1)
    except Exception:
        pass
    import oracle

    model, data = make(cfg)
    _T["o"] = oracle
    _T["t"] = oracle.OTarget(model, data)
    _T["eps"] = cfg["eps"]


def _work(args):
    seed, lf = args
    o = _T["o"]
    t0 = time.perf_counter()
    o.run_chain(_T["t"], o.OConfig(epsilon=_T["eps"], leapfrogs=lf, moves=1, burnin=0, seed=seed))
    return time.perf_counter() - t0


def cpu_rate(cfg, lf, cores):
    """Chain-leapfrogs/s with one chain per core.  The pool is started and warmed (imports,
    the oracle target, one short chain per worker) before the clock starts; each timed chain
    of `lf` leapfrogs still includes its own cold start, as the reference's run_chain does."""
    with mp.get_context("spawn").Pool(cores, initializer=_init, initargs=(cfg,)) as pool:
        pool.map(_work, [(1000 + k, 1) for k in range(cores)])
        t0 = time.perf_counter()
        pool.map(_work, [(k, lf) for k in range(cores)])
        wall = time.perf_counter() - t0
    return cores * lf / wall


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu-leapfrogs", type=int, default=5)
    ap.add_argument("--gpu-leapfrogs", type=int, default=10)
    ap.add_argument("--skip-c4", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    args = ap.parse_args()
    cores = os.cpu_count() or 1
    print(f"| config | d | GPU chains | GPU chain-leapfrogs/s | GPU ms/leapfrog (batch) | acc | "
          f"CPU ({cores} cores) chain-leapfrogs/s | ratio |")
    print("|---|---|---|---|---|---|---|---|")
    for cfg in CONFIGS:
        d, rate, ms, acc, st = gpu_rate(cfg, args.gpu_leapfrogs)
        cpu = None if args.skip_cpu else cpu_rate(cfg, args.cpu_leapfrogs, cores)
        ratio = f"{rate / cpu:.0f}x" if cpu else "-"
        cpus = f"{cpu:.1f}" if cpu else "-"
        print(f"| {cfg['name']} | {d} | {cfg['chains']} | {rate:,.0f} | {ms:.2f} | {acc:.2f} | {cpus} | {ratio} |",
              flush=True)
    if not args.skip_c4:
        import bench

        d, rate, ms, acc, st = gpu_rate(C4, 2, order="refine")
        s_lf, _ = bench.cpu_c4_sample()
        print(f"| {C4['name']} (warm order refine) | {d} | 1 | {rate:.2f} | {ms:.1f} | {acc:.2f} | "
              f"{1.0 / s_lf:.4f} ({s_lf:.0f} s/leapfrog, bounded sample, bench.cpu_c4_sample) | "
              f"{s_lf * 1e3 / ms:.0f}x |", flush=True)


if __name__ == "__main__":
    main()
