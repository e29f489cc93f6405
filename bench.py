"""Benchmark: generalized-leapfrog steps/sec of the SoftAbs RMHMC inner loop.

Workload (BASELINE.json configs[1]): single-kernel GP
binary classification, simulate_logistic(1, n=512, seed=0), logistic model
with 30 basis functions (d = 34), epsilon = 1e-3, C = 100 leapfrogs per move,
reference warm-Jacobi order (trajectory parity with the reference).  Z
independent chains per GPU ("replicas", one CTA each).  One step = one MH
move (C generalized leapfrogs + Metropolis test) of every chain on the GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--chains Z]
    python bench.py --impl reference     # the reference algorithm on host cores

``value`` = chain-leapfrogs/s over all ranks (device time, max over ranks);
``e2e`` = the same through the public chain API with host RNG, pinned H2D of
the step's normals/uniforms and D2H of the move records inside the timed
region.  The CPU arms run the oracle port (oracle/, the reference algorithm
restated: numpy BLAS + the C Jacobi) because the reference package cannot
travel to the GPU box.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "generalized-leapfrog steps/sec"
UNIT = "chain-leapfrogs/s"
EPS, LEAPFROGS, N_ROWS = 1e-3, 100, 512


def canonical_flops_per_leapfrog(N, D, d, fp_p=3, fp_q=3, s=5.0 / 3.0):
    """SURVEY.md 8(d) canonical FLOP count of one generalized leapfrog (J = 1)."""
    n_tr = fp_p + 2
    return n_tr * (2 * N * D * D + 4 * d ** 3) + 2 * d ** 3 + fp_q * (2 * N * D * D + (6.2 + 6 * s) * d ** 3)


def workload():
    from paper_2511_06407_b200 import rrgp

    data, _ = rrgp.simulate_logistic(1, n=N_ROWS, seed=0)
    model = rrgp.build_model("logistic", data.x)
    return model, data


# ---------------------------------------------------------------------------
# CPU arms (oracle port of the reference algorithm)


_W = {}


def _cpu_init():
    """Pool initializer: single-threaded BLAS and a cached oracle target."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        import threadpoolctl

        threadpoolctl.threadpool_limits(1)
    except Exception:
        pass
    import oracle

    model, data = workload()
    _W["oracle"] = oracle
    _W["target"] = oracle.OTarget(model, data)
    oracle.metric_cold(_W["target"].at(_W["target"].initial_point()).hessian(), 1.0, 1e-13)


def _cpu_worker(args):
    seed, n_leapfrogs = args
    oracle = _W["oracle"]
    cfg = oracle.OConfig(epsilon=EPS, leapfrogs=n_leapfrogs, moves=1, burnin=0, seed=seed)
    t0 = time.perf_counter()
    oracle.run_chain(_W["target"], cfg)
    return n_leapfrogs, time.perf_counter() - t0


class CpuPool:
    """One chain per host core: the reference's own process-pool parallelism
    (evidence.py:237-239), workers warmed before any timing."""

    def __init__(self, n_workers):
        self.n = n_workers
        self.pool = mp.get_context("spawn").Pool(n_workers, initializer=_cpu_init)
        self.pool.map(_cpu_worker, [(k, 1) for k in range(n_workers)])

    def sample(self, leapfrogs_each, seed0=0):
        """Returns (chain-leapfrogs, wall seconds) of one pool.map."""
        jobs = [(seed0 + k, leapfrogs_each) for k in range(self.n)]
        t0 = time.perf_counter()
        out = self.pool.map(_cpu_worker, jobs)
        return sum(o[0] for o in out), time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def run_reference(args):
    """--impl reference: the reference algorithm on all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    # each step: every core runs one chain for `lf` leapfrogs (bounded sample)
    lf = max(1, args.ref_leapfrogs)
    pool = CpuPool(cores)
    for _ in range(args.warmup):
        pool.sample(1, seed0=1000)
    total_lf, total_t = 0, 0.0
    for k in range(args.steps):
        n, wall = pool.sample(lf, seed0=k * cores)
        total_lf += n
        total_t += wall
    pool.close()
    value = total_lf / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator simulate_logistic(1, n=512, seed=0))",
        "config": {"workload": "C2 logistic GP classification N=512 d=34, eps=1e-3, C=100",
                   "chains": cores, "leapfrogs_per_step_per_chain": lf},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{cores} processes x {lf} generalized leapfrogs per step "
                                   f"(oracle port, OPENBLAS_NUM_THREADS=1)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measure_dgemm_tflops(torch):
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = math.inf
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b
    return 2.0 * n ** 3 / best / 1e12


def measure_ess(target, sm_count, args, torch):
    """min-ESS per chain-move of the C2 sampler: one wave of
    chains from q = 0, burn-in moves, then recorded moves in one launch; Geyer
    ESS per coordinate of q, min over coordinates, mean over chains."""
    from paper_2511_06407_b200.diagnostics import min_ess
    from paper_2511_06407_b200.sampler import ChainConfig, DeviceChains

    d = target.dim
    Z = sm_count * args.ess_chains_per_sm
    cfg = ChainConfig(epsilon=EPS, leapfrogs=LEAPFROGS, moves=1, burnin=0, warm_order=args.warm_order)
    ch = DeviceChains(target.device, np.ones(Z), cfg)
    ch.set_q(np.zeros((Z, d)))
    ch.init()
    rng = np.random.default_rng(12345)
    B, M = args.ess_burnin, args.ess_moves
    t0 = time.perf_counter()
    with np.errstate(divide="ignore"):
        if B > 0:
            ch.run(B, rng.standard_normal((B, Z, d)), np.log(rng.uniform(size=(B, Z))))
        bufs = ch.run(M, rng.standard_normal((M, Z, d)), np.log(rng.uniform(size=(M, Z))), record_q=True)
    q = bufs["q"].cpu().numpy()  # (M, Z, d)
    wall = time.perf_counter() - t0
    per_chain = np.array([min_ess(q[:, z, :]) for z in range(Z)])
    return {"chains": Z, "burnin_moves": B, "recorded_moves": M,
            "min_ess_per_chain_move": float(per_chain.mean() / M),
            "min_ess_chain_median": float(np.median(per_chain)),
            "acceptance": float(bufs["accept"].float().mean().item()),
            "estimator": "Geyer initial-monotone per coordinate of q, min over coordinates, mean over chains",
            "pilot_wall_s": wall}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one rank per GPU; the modulo only matters for functional runs of several
    # ranks on a one-GPU box (SGP_DIST_BACKEND=gloo), never for measurements
    dev_index = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    if world > 1:
        backend = os.environ.get("SGP_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)

    from paper_2511_06407_b200 import _native as nat
    from paper_2511_06407_b200.posterior import PosteriorTarget
    from paper_2511_06407_b200.sampler import ChainConfig, DeviceChains

    model, data = workload()
    target = PosteriorTarget(model, data)
    d = target.dim
    L = nat.lib()
    import ctypes

    smc, ccmaj, ccmin = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    L.sgp_device_info(ctypes.byref(smc), ctypes.byref(ccmaj), ctypes.byref(ccmin))
    sm_count = smc.value
    Z = args.chains if args.chains > 0 else sm_count * args.chains_per_sm
    cfg = ChainConfig(epsilon=EPS, leapfrogs=LEAPFROGS, moves=1, burnin=0, warm_order=args.warm_order)
    chains = DeviceChains(target.device, np.ones(Z), cfg)
    chains.set_q(np.zeros((Z, d)))
    chains.init()
    rngs = [np.random.default_rng([rank, z]) for z in range(Z)]

    def draws():
        z = np.empty((1, Z, d))
        u = np.empty((1, Z))
        for k, r in enumerate(rngs):
            z[0, k] = r.standard_normal(d)
            u[0, k] = r.uniform()
        with np.errstate(divide="ignore"):
            return z, np.log(u)

    # device-resident inputs for the kernel-only number
    zs_all, lu_all = [], []
    for _ in range(args.warmup + args.steps):
        z, lu = draws()
        zs_all.append(torch.from_numpy(z).cuda())
        lu_all.append(torch.from_numpy(lu).cuda())
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    for w in range(args.warmup):
        chains.run(1, zs_all[w], lu_all[w])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    with ClockSampler(dev_index) as clocks:
        t_wall = time.perf_counter()
        for k in range(args.steps):
            flush.fill_(float(k))  # evict L2 between timed steps (untimed)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            chains.run(1, zs_all[args.warmup + k], lu_all[args.warmup + k])
            e1.record(stream)
            times.append((e0, e1))
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    dev_s = sum(a.elapsed_time(b) for a, b in times) / 1e3
    status = chains.status_host()
    bufs = chains._rec[1]
    acc = float(bufs["accept"].float().mean().item())
    sweeps = float(bufs["sweeps_mean"].mean().item())
    t_max = torch.tensor([dev_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    T = float(t_max.item())
    total_lf = world * Z * LEAPFROGS * args.steps
    value = total_lf / T

    # ---- e2e through the public chain API: host RNG + pinned H2D + D2H records
    zpin = torch.empty((1, Z, d), dtype=torch.float64).pin_memory()
    lpin = torch.empty((1, Z), dtype=torch.float64).pin_memory()
    out_pin = {k: torch.empty((1, Z), dtype=torch.float64).pin_memory()
               for k in ("logpost", "h_before", "h_after")}
    acc_pin = torch.empty((1, Z), dtype=torch.uint8).pin_memory()
    q_pin = torch.empty((Z, d), dtype=torch.float64).pin_memory()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_steps = max(1, args.steps)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        z, lu = draws()
        zpin.numpy()[...] = z
        lpin.numpy()[...] = lu
        zd = zpin.to("cuda", non_blocking=True)
        ld = lpin.to("cuda", non_blocking=True)
        b = chains.run(1, zd, ld)
        for k2, t in out_pin.items():
            t.copy_(b[k2], non_blocking=True)
        acc_pin.copy_(b["accept"], non_blocking=True)
        q_pin.copy_(chains.q, non_blocking=True)
        torch.cuda.synchronize()
    e2e_t = time.perf_counter() - t0
    e2e_max = torch.tensor([e2e_t], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_max, op=dist.ReduceOp.MAX)
    e2e_value = world * Z * LEAPFROGS * e2e_steps / float(e2e_max.item())
    h2d = Z * d * 8 + Z * 8
    d2h = 3 * Z * 8 + Z + Z * d * 8

    ess = None
    if rank == 0 and args.ess_moves > 0:
        ess = measure_ess(target, sm_count, args, torch)

    if rank == 0:
        N, D = N_ROWS, d - 3
        F = canonical_flops_per_leapfrog(N, D, d, s=max(1.0, sweeps))
        achieved = F * Z * LEAPFROGS * args.steps / dev_s / 1e12
        dgemm = measure_dgemm_tflops(torch)
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator simulate_logistic(1, n=512, seed=0))",
            "config": {"workload": "C2 logistic GP classification N=512 d=34, eps=1e-3, C=100",
                       "chains_per_gpu": Z, "step": "one MH move (100 generalized leapfrogs) per chain",
                       "warm_order": args.warm_order, "parallelism": f"replicas x{world}",
                       "l2": "flushed between steps (256 MiB write, untimed)",
                       "acceptance": acc, "sweeps_mean": sweeps,
                       "status_nonzero": int(np.count_nonzero(status))},
            "gpu_launches": args.steps,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": dgemm, "unit": "TFLOP/s",
                         "frac": achieved / dgemm, "traffic": None,
                         "kernel": "k_run_moves", "flops_per_leapfrog": F,
                         "peak_source": "cuBLAS DGEMM 8192^3 measured in this run "
                                        "(MEASURED_PEAKS.json has no FP64 entry)"},
            "clocks": clocks.summary(),
            "wall_s_timed": t_wall,
        }
        if ess is not None:
            # chain-moves/s of the timed region x ESS per chain-move of the pilot
            ess["min_ess_per_s"] = ess["min_ess_per_chain_move"] * value / LEAPFROGS
            line["min_ess"] = ess
        if os.path.exists(peaks_path):
            line["roofline"]["peaks_file"] = "MEASURED_PEAKS.json present (bf16/HBM only)"
        # DRAM bytes per launch of this kernel from the committed ncu --set full capture
        # of the same command (profiles/), when it was taken on this configuration
        tpath = os.path.join(ROOT, "profiles", "r1_traffic_k_run_moves.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                tr = json.load(f)
            if tr.get("chains") == Z and tr.get("leapfrogs") == LEAPFROGS:
                line["roofline"]["traffic"] = tr["dram_bytes_per_launch"]
                line["roofline"]["traffic_unit"] = "bytes/launch (DRAM read+write, ncu)"
                line["roofline"]["traffic_source"] = "profiles/r1_traffic_k_run_moves.json"
        if world == 1 and not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            pool = CpuPool(cores)
            n, wall = pool.sample(args.ref_leapfrogs)
            pool.close()
            line["cpu_baseline"] = {"value": n / wall, "unit": UNIT, "cores": cores, "kind": "port",
                                    "sample": f"{cores} processes x {args.ref_leapfrogs} generalized "
                                              f"leapfrogs (oracle port, OPENBLAS_NUM_THREADS=1)"}
            if ess is not None:
                ess["cpu_min_ess_per_s"] = ess["min_ess_per_chain_move"] * (n / wall) / LEAPFROGS
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--chains", type=int, default=0, help="chains per GPU (default SMs x chains-per-sm)")
    ap.add_argument("--chains-per-sm", type=int, default=12)
    ap.add_argument("--warm-order", default="cyclic", choices=["cyclic", "parallel"])
    ap.add_argument("--ref-leapfrogs", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ess-moves", type=int, default=300, help="recorded moves of the min-ESS pilot (0: skip)")
    ap.add_argument("--ess-burnin", type=int, default=100)
    ap.add_argument("--ess-chains-per-sm", type=int, default=2)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
