"""Benchmark: generalized-leapfrog steps/sec of the SoftAbs RMHMC inner loop.

Default workload (the largest single-GPU config of BASELINE.json, configs[3]; SURVEY.md 8(d)
C4): the multiple-kernel mean/variance GP model scaled to N = 8192 rows,
simulate_meanvar(34, 19, n=8192, seed=0) with the "nl-meanvar" preset (d = 2083), epsilon =
1e-4, C = 100 leapfrogs per move, one chain per GPU ("replicas": a chain is never split
across GPUs).  One step = one MH move (C generalized leapfrogs + the Metropolis test).  Warm
decompositions use the GEMM eigenvector refinement (warm_order="refine"); cold ones (chain start,
rejections) the reference's pivot order, bit-identical (sgp_jbig.cuh).

    python bench.py [--gpus N] [--steps K] [--warmup W]            # C4 (headline)
    python bench.py --workload c2                                  # C2: 1776 chains, d = 34
    python bench.py --impl reference [--workload c4|c2]            # reference algorithm, host cores

``value`` = chain-leapfrogs/s over all ranks (CUDA events on the launching stream, max over
ranks); ``e2e`` = the same through the public chain API with host RNG draws, pinned H2D of the
step's normals/uniforms and D2H of the move records and positions inside the timed region.
The CPU arms run the oracle port (oracle/: the reference algorithm restated, numpy/OpenBLAS
+ the C restatement of the Numba Jacobi) because the reference package cannot travel to the
GPU box; at C4 a leapfrog takes minutes on the host, so the CPU figure is a bounded sample of
its parts scaled by the canonical per-leapfrog call counts (cpu_c4_sample).
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
C4_EPS, C4_LEAPFROGS = 1e-4, 100
C4_NAME = ("C4 multiple-kernel mean/variance GP (nl-meanvar), N=8192 rows, 34 continuous + 19 binary "
           "covariates, d=2083, eps=1e-4, C=100")
C2_NAME = "C2 logistic GP classification N=512 d=34, eps=1e-3, C=100"


def canonical_flops_per_leapfrog(N, Ds, d, fp_p=3, fp_q=3, s=5.0 / 3.0):
    """SURVEY.md 8(d) canonical FLOP count of one generalized leapfrog; Ds = (D_1, ..., D_J)."""
    if not isinstance(Ds, (list, tuple)):
        Ds = (Ds,)
    n_tr = fp_p + 2
    dsum = sum(Ds)
    pairs = sum(Ds[a] * Ds[b] for a in range(len(Ds)) for b in range(a, len(Ds)))
    return n_tr * (2 * N * dsum * dsum + 4 * d ** 3) + 2 * d ** 3 + fp_q * (2 * N * pairs + (6.2 + 6 * s) * d ** 3)


def executed_flops_per_leapfrog(N, Ds, d, fp_p=3):
    """canonical_flops_per_leapfrog minus the trace blocks this implementation does not form:
    with W symmetric, s^(j1 j2) = s^(j2 j1), so the j1 > j2 blocks of Y = Phi W are skipped."""
    if not isinstance(Ds, (list, tuple)):
        Ds = (Ds,)
    skipped = sum(Ds[a] * Ds[b] for a in range(len(Ds)) for b in range(a))
    return canonical_flops_per_leapfrog(N, Ds, d, fp_p=fp_p) - (fp_p + 2) * 2 * N * skipped


def workload():
    from paper_2511_06407_b200 import rrgp

    data, _ = rrgp.simulate_logistic(1, n=N_ROWS, seed=0)
    model = rrgp.build_model("logistic", data.x)
    return model, data


def workload_c4():
    from paper_2511_06407_b200 import rrgp

    data, _ = rrgp.simulate_meanvar(34, 19, n=8192, seed=0)
    model = rrgp.build_model("nl-meanvar", data.x)
    return model, data


def c4_feature_widths(model):
    return tuple(sum(k.features for k in ks) + 1 for ks in model.functions)


def cpu_c4_sample(reps=1):
    """The reference algorithm's C4 leapfrog on this host, as a bounded sample: one Hessian
    (posterior.py:442-482), one structured trace (posterior.py:486-542) and one d^3 GEMM in
    numpy/OpenBLAS with every host thread, plus a slice of a cyclic Jacobi sweep in the C
    restatement of the Numba kernel (single-threaded, as the reference's), scaled by the
    canonical per-leapfrog call counts (fp_p = 3 -> 5 traces + 5 W1, one W2,
    fp_q = 3 Hessians + Psi^T H Psi + Psi Q, 5/3 sweeps per warm decomposition).
    Returns (seconds per leapfrog, parts dict)."""
    import oracle

    model, data = workload_c4()
    ot = oracle.OTarget(model, data)
    d = ot.dim
    rng = np.random.default_rng(7)
    parts = {"hessian": [], "trace": [], "gemm": [], "rotation": []}
    w = rng.standard_normal((d, d))
    w = 0.5 * (w + w.T)
    psi = rng.standard_normal((d, d))
    for _ in range(reps):
        q = 0.01 * rng.standard_normal(d)
        pt = ot.at(q)
        t0 = time.perf_counter()
        h = pt.hessian()
        parts["hessian"].append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        pt.trace(w)
        parts["trace"].append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        _ = psi.T @ h
        parts["gemm"].append(time.perf_counter() - t0)
        a = np.ascontiguousarray(0.5 * (h + h.T))
        v = np.eye(d)
        t0 = time.perf_counter()
        nrot = oracle.jacobi_passes(a, v, 0, 24, 0.0)
        parts["rotation"].append((time.perf_counter() - t0) / max(1, nrot))
    t = {k: float(np.median(v)) for k, v in parts.items()}
    sweep = t["rotation"] * d * (d - 1) / 2
    fp_p, fp_q, s = 3, 3, 5.0 / 3.0
    n_tr = fp_p + 2
    per_lf = n_tr * (t["trace"] + 2 * t["gemm"]) + t["gemm"] + fp_q * (t["hessian"] + 3 * t["gemm"] + s * sweep)
    t["sweep"] = sweep
    return per_lf, t


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


def run_reference_c4(args):
    """--impl reference at C4: each step is one bounded sample of the reference algorithm's
    leapfrog on all host cores (cpu_c4_sample), reported in the GPU arm's units."""
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_c4_sample()
    per_lf = []
    t_all = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        s_lf, parts = cpu_c4_sample()
        t_all += time.perf_counter() - t0
        per_lf.append(s_lf)
    value = 1.0 / float(np.median(per_lf))
    sample = (f"per step: 1 Hessian + 1 structured trace + 1 d^3 GEMM (numpy/OpenBLAS, {cores} threads) and "
              f"24 passes (~{24 * 2082} rotations) of a cyclic Jacobi sweep (C restatement of the Numba "
              f"kernel, 1 thread), scaled to one leapfrog by the SURVEY.md 8(d) call counts")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator simulate_meanvar(34, 19, n=8192, seed=0))",
        "config": {"workload": C4_NAME, "chains": 1, "s_per_leapfrog_estimate": float(np.median(per_lf)),
                   "parts_s": parts},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


_W5 = {}


def _c5_init():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        import threadpoolctl

        threadpoolctl.threadpool_limits(1)
    except Exception:
        pass
    import oracle

    models, data = workload_c5()
    _W5["oracle"] = oracle
    _W5["targets"] = [(oracle.OTarget(m, data), eps) for m, eps in models]


def _c5_worker(args):
    m, seed, tau, A, C = args
    oracle = _W5["oracle"]
    t, eps = _W5["targets"][m]
    tt = t.at_temperature(tau)
    cfg = oracle.OConfig(epsilon=eps, leapfrogs=C, moves=A, burnin=0, seed=seed)
    t0 = time.perf_counter()
    oracle.run_chain(tt, cfg, tt.initial_point())
    return A * C, time.perf_counter() - t0


def run_reference_c5(args):
    """--impl reference at C5: the reference's process-pool parallelism (evidence.py:237-239),
    one (model, chain) unit per host core per step, each unit one rung (cold start + A moves of
    C leapfrogs); units cycle through the four models."""
    cores = os.cpu_count() or 1
    A, C = args.c5_moves, args.leapfrogs or 10
    pool = mp.get_context("spawn").Pool(cores, initializer=_c5_init)
    pool.map(_c5_worker, [(k % 4, k, 1.0, 1, 1) for k in range(cores)])
    for w in range(args.warmup):
        pool.map(_c5_worker, [(k % 4, 100 + k, 0.5, 1, 1) for k in range(cores)])
    total, t_all = 0, 0.0
    for k in range(args.steps):
        jobs = [((k * cores + j) % 4, 1000 * k + j, 0.5, A, C) for j in range(cores)]
        t0 = time.perf_counter()
        out = pool.map(_c5_worker, jobs)
        t_all += time.perf_counter() - t0
        total += sum(o[0] for o in out)
    pool.close()
    pool.join()
    value = total / t_all
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "chain-rung-leapfrogs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator simulate_meanvar(2, 19, n=2000, seed=0))",
        "config": {"workload": C5_NAME, "moves_per_rung": A, "leapfrogs": C, "units_per_step": cores},
        "cpu_baseline": {"value": value, "unit": "chain-rung-leapfrogs/s", "cores": cores, "kind": "port",
                         "sample": f"{cores} processes x one rung ({A} moves x {C} leapfrogs + cold start) per step, "
                                   "models round-robin (oracle port, OPENBLAS_NUM_THREADS=1)"},
        "e2e": {"value": value, "unit": "chain-rung-leapfrogs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference(args):
    """--impl reference: the reference algorithm on all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.workload == "c4":
        run_reference_c4(args)
        return
    if args.workload == "c5":
        run_reference_c5(args)
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
        "config": {"workload": C2_NAME, "chains": cores, "leapfrogs_per_step_per_chain": lf},
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


def _dist_setup():
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
    return torch, dist, world, rank, dev_index


def _reduce_device(dist):
    """Device of the max-over-ranks reductions: CUDA tensors under NCCL (the measurement
    backend), host tensors under gloo (functional multi-rank runs on a one-GPU box)."""
    return "cuda" if dist.is_initialized() and dist.get_backend() == "nccl" else "cpu"


def count_kernel_launches(torch, fn):
    """Kernels launched by fn() (CUPTI activity records through torch.profiler), untimed."""
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = {}
    for ev in prof.events():
        if getattr(ev, "device_type", None) is not None and str(ev.device_type).endswith("CUDA"):
            n = ev.name
            if n.startswith(("Memcpy", "Memset", "cudaMemcpy", "cudaMemset")):
                continue
            names[n] = names.get(n, 0) + 1
    return sum(names.values()), names


def run_gpu_c4(args):
    """C4: one chain per GPU (replicas), one MH move of C leapfrogs per step."""
    torch, dist, world, rank, dev_index = _dist_setup()
    from paper_2511_06407_b200.posterior import PosteriorTarget
    from paper_2511_06407_b200.sampler import ChainConfig, DeviceChains

    model, data = workload_c4()
    target = PosteriorTarget(model, data)
    d = target.dim
    C = args.leapfrogs or C4_LEAPFROGS
    cfg = ChainConfig(epsilon=C4_EPS, leapfrogs=C, moves=1, burnin=0, warm_order=args.warm_order or "refine",
                      cold_order=getattr(args, "cold_order", "cyclic"))
    Z = 1
    chains = DeviceChains(target.device, np.ones(Z), cfg)
    chains.set_q(np.zeros((Z, d)))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    chains.init()
    st0 = chains.status_host()
    cold_s = time.perf_counter() - t0
    if np.count_nonzero(st0):
        raise RuntimeError(f"chain start failed (status {st0})")
    rng = np.random.default_rng([rank, 4])

    def draws():
        z = rng.standard_normal((1, Z, d))
        with np.errstate(divide="ignore"):
            lu = np.log(rng.uniform(size=(1, Z)))
        return z, lu

    n_dev = args.warmup + args.steps
    dev_in = [tuple(torch.from_numpy(a).cuda() for a in draws()) for _ in range(n_dev)]
    stream = torch.cuda.current_stream()
    for w in range(args.warmup):
        chains.run(1, *dev_in[w], move_offset=w)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    accepted = []
    with ClockSampler(dev_index) as clocks:
        t_wall = time.perf_counter()
        for k in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            b = chains.run(1, *dev_in[args.warmup + k], move_offset=args.warmup + k)
            e1.record(stream)
            times.append((e0, e1))
            accepted.append(b["accept"].clone())
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    status = chains.status_host()
    if np.count_nonzero(status):
        raise RuntimeError(f"chain stopped during the timed region (status {status}): no valid throughput")
    dev_s = sum(a.elapsed_time(b) for a, b in times) / 1e3
    acc = float(torch.stack(accepted).float().mean().item())
    t_max = torch.tensor([dev_s], dtype=torch.float64,
                         device=_reduce_device(dist) if world > 1 else "cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    T = float(t_max.item())
    total_lf = world * Z * C * args.steps
    value = total_lf / T

    # ---- e2e: host RNG draws -> pinned H2D -> the move -> D2H of records and position
    zpin = torch.empty((1, Z, d), dtype=torch.float64).pin_memory()
    lpin = torch.empty((1, Z), dtype=torch.float64).pin_memory()
    rec_pin = {k: torch.empty((1, Z), dtype=torch.float64).pin_memory()
               for k in ("logpost", "h_before", "h_after", "sweeps_mean")}
    acc_pin = torch.empty((1, Z), dtype=torch.uint8).pin_memory()
    q_pin = torch.empty((Z, d), dtype=torch.float64).pin_memory()
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        z, lu = draws()
        zpin.numpy()[...] = z
        lpin.numpy()[...] = lu
        b = chains.run(1, zpin.to("cuda", non_blocking=True), lpin.to("cuda", non_blocking=True),
                       move_offset=n_dev + k)
        for k2, t in rec_pin.items():
            t.copy_(b[k2], non_blocking=True)
        acc_pin.copy_(b["accept"], non_blocking=True)
        q_pin.copy_(chains.q, non_blocking=True)
        torch.cuda.synchronize()
    e2e_t = time.perf_counter() - t0
    e2e_max = torch.tensor([e2e_t], dtype=torch.float64,
                         device=_reduce_device(dist) if world > 1 else "cuda")
    if world > 1:
        dist.all_reduce(e2e_max, op=dist.ReduceOp.MAX)
    e2e_value = world * Z * C * e2e_steps / float(e2e_max.item())
    h2d = Z * d * 8 + Z * 8
    d2h = 4 * Z * 8 + Z + Z * d * 8

    if rank == 0:
        # kernels per move, counted on one extra (untimed) move
        zc, lc = draws()
        launches, names = count_kernel_launches(
            torch, lambda: chains.run(1, zc, lc, move_offset=n_dev + e2e_steps))
        Ds = c4_feature_widths(model)
        F = canonical_flops_per_leapfrog(model_rows(data), Ds, d)
        achieved = F * C * args.steps / dev_s / 1e12
        dgemm = measure_dgemm_tflops(torch)
        top = sorted(names.items(), key=lambda kv: -kv[1])[:8]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator simulate_meanvar(34, 19, n=8192, seed=0))",
            "config": {"workload": C4_NAME, "chains_per_gpu": Z, "leapfrogs_per_move": C,
                       "step": f"one MH move ({C} generalized leapfrogs) of the chain",
                       "warm_order": cfg.warm_order, "cold_order": cfg.cold_order,
                       "parallelism": f"replicas x{world} (one chain per GPU)",
                       "l2": "inputs (Phi 136 MB + the d x d working set) exceed L2; no flush",
                       "acceptance": acc, "cold_init_s": cold_s,
                       "per_chain_leapfrogs_per_s": value / (world * Z),
                       "ms_per_leapfrog": 1e3 * T / (C * args.steps)},
            "gpu_launches": launches * args.steps,
            "gpu_launches_per_move": launches, "gpu_launch_top": top,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": dgemm, "unit": "TFLOP/s",
                         "frac": achieved / dgemm, "traffic": None,
                         "kernel": "whole generalized leapfrog (DMMA GEMMs: trace, Hessian, W, eigenvector refinement; glue)",
                         "flops_per_leapfrog": F,
                         "flops_source": "SURVEY.md 8(d) canonical count (fp_p=3, fp_q=3, s=5/3)",
                         "flops_executed_per_leapfrog": executed_flops_per_leapfrog(model_rows(data), Ds, d),
                         "executed_note": "the trace's (1,0) block of Y = Phi W repeats the (0,1) block (W "
                                          "symmetric) and is not formed; achieved/frac use the canonical count, "
                                          "achieved_executed the executed one",
                         "achieved_executed": executed_flops_per_leapfrog(model_rows(data), Ds, d) * C * args.steps
                                              / dev_s / 1e12,
                         "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (FP64 tensor pipe; "
                                        "MEASURED_PEAKS.json has no FP64 entry)"},
            "clocks": clocks.summary(),
            "wall_s_timed": t_wall,
        }
        if world == 1 and not args.no_cpu_baseline:
            s_lf, parts = cpu_c4_sample()
            cores = os.cpu_count() or 1
            line["cpu_baseline"] = {
                "value": 1.0 / s_lf, "unit": UNIT, "cores": cores, "kind": "port",
                "sample": "1 Hessian + 1 structured trace + 1 d^3 GEMM (numpy/OpenBLAS, all threads) and 24 passes "
                          "of a cyclic Jacobi sweep (C restatement of the Numba kernel, 1 thread), scaled to one "
                          "leapfrog by the SURVEY.md 8(d) call counts",
                "parts_s": parts}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


C5_MODELS = (("l-mean", 1e-4), ("nl-mean", 1e-4), ("l-meanvar", 1e-4), ("nl-meanvar", 8e-5))
C5_NAME = ("C5 model evidence: l-mean / nl-mean / l-meanvar / nl-meanvar (d = 26/84/47/163) on "
           "simulate_meanvar(2, 19, n=2000, seed=0), 64 chains each, default_ladder().thin(4) (26 rungs)")


def workload_c5():
    from paper_2511_06407_b200 import rrgp

    data, _ = rrgp.simulate_meanvar(2, 19, n=2000, seed=0)
    return [(rrgp.build_model(name, data.x), eps) for name, eps in C5_MODELS], data


def run_gpu_c5(args):
    """C5: (model, chain) units u = m*Z + z on rank u mod W; one step = one rung
    of the ladder walk (cold start at the rung's temperature + A moves of C leapfrogs,
    evidence.py:142-163) for every local unit, the four models on their own streams."""
    torch, dist, world, rank, dev_index = _dist_setup()
    from paper_2511_06407_b200.evidence import default_ladder
    from paper_2511_06407_b200.posterior import PosteriorTarget
    from paper_2511_06407_b200.sampler import ChainConfig, DeviceChains

    Z, A, C = args.c5_chains, args.c5_moves, args.leapfrogs or 10
    ladder = default_ladder(moves_per_rung=A, leapfrogs=C, chains=Z).thin(4)
    models, data = workload_c5()
    n_units = len(models) * Z
    units = [u for u in range(n_units) if u % world == rank]
    batches = []
    for m, (model, eps) in enumerate(models):
        zs = [u % Z for u in units if u // Z == m]
        if not zs:
            continue
        target = PosteriorTarget(model, data)
        cfg = ChainConfig(epsilon=eps, leapfrogs=C, moves=A, burnin=0, warm_order=args.warm_order or "cyclic")
        ch = DeviceChains(target.device, np.ones(len(zs)), cfg)
        ch.set_q(np.tile(target.initial_point(), (len(zs), 1)))
        batches.append({"m": m, "zs": zs, "ch": ch, "d": target.dim, "stream": torch.cuda.Stream(),
                        "rng": np.random.default_rng([rank, m])})
    n_local = sum(len(b["zs"]) for b in batches)

    def draws(b):
        z = b["rng"].standard_normal((A, len(b["zs"]), b["d"]))
        with np.errstate(divide="ignore"):
            lu = np.log(b["rng"].uniform(size=(A, len(b["zs"]))))
        return z, lu

    n_steps = args.warmup + args.steps
    for b in batches:
        b["in"] = [tuple(torch.from_numpy(a).cuda() for a in draws(b)) for _ in range(n_steps)]
    main = torch.cuda.current_stream()

    def step(k):
        tau = float(ladder.taus[k % ladder.size])
        ev0 = torch.cuda.Event()
        ev0.record(main)
        ends = []
        for b in batches:
            with torch.cuda.stream(b["stream"]):
                b["stream"].wait_event(ev0)
                b["ch"].tau.fill_(tau)
                b["ch"].init()  # the rung's cold start (sampler.py:322-328)
                b["ch"].run(A, *b["in"][k], move_offset=0)
                e = torch.cuda.Event()
                e.record(b["stream"])
                ends.append(e)
        for e in ends:
            main.wait_event(e)

    for w in range(args.warmup):
        step(w)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    with ClockSampler(dev_index) as clocks:
        t_wall = time.perf_counter()
        for k in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main)
            step(args.warmup + k)
            e1.record(main)
            times.append((e0, e1))
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    bad = sum(int(np.count_nonzero(b["ch"].status_host())) for b in batches)
    dev_s = sum(a.elapsed_time(b) for a, b in times) / 1e3
    t_max = torch.tensor([dev_s], dtype=torch.float64,
                         device=_reduce_device(dist) if world > 1 else "cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    T = float(t_max.item())
    value = n_units * A * C * args.steps / T

    # e2e through the public API: run_chains per model (host RNG draws in the reference's
    # order, H2D inside, records and positions back to the host)
    from paper_2511_06407_b200.sampler import run_chains
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h2d = d2h = 0
    for k in range(e2e_steps):
        tau = float(ladder.taus[k % ladder.size])
        for b in batches:
            model, _ = models[b["m"]]
            tgt = PosteriorTarget(model, data, tau)
            q0 = b["ch"].q.cpu().numpy()
            res = run_chains(tgt, b["ch"].config, [1000 * k + z for z in b["zs"]], q0)
            h2d += len(b["zs"]) * (A * b["d"] + A + b["d"]) * 8
            d2h += len(b["zs"]) * (A * 7 + b["d"]) * 8
    torch.cuda.synchronize()
    e2e_t = time.perf_counter() - t0
    e2e_max = torch.tensor([e2e_t], dtype=torch.float64,
                         device=_reduce_device(dist) if world > 1 else "cuda")
    if world > 1:
        dist.all_reduce(e2e_max, op=dist.ReduceOp.MAX)
    e2e_value = n_units * A * C * e2e_steps / float(e2e_max.item())
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "chain-rung-leapfrogs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator simulate_meanvar(2, 19, n=2000, seed=0))",
            "config": {"workload": C5_NAME, "units": n_units, "units_on_rank0": n_local,
                       "moves_per_rung": A, "leapfrogs": C,
                       "step": "one ladder rung (cold start + A moves) of every (model, chain) unit",
                       "parallelism": f"(model, chain) units sharded over {world} rank(s), unit u on rank u mod W",
                       "warm_order": batches[0]["ch"].config.warm_order if batches else None,
                       "status_nonzero": bad},
            "gpu_launches": args.steps * 2 * len(batches),
            "e2e": {"value": e2e_value, "unit": "chain-rung-leapfrogs/s", "h2d_bytes_per_step": h2d // e2e_steps,
                    "d2h_bytes_per_step": d2h // e2e_steps, "steps": e2e_steps},
            "roofline": None,
            "roofline_note": "latency-bound (SURVEY.md 8(d): neither roofline binds at d <= 163)",
            "clocks": clocks.summary(), "wall_s_timed": t_wall,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def model_rows(data):
    return int(np.asarray(data.y).shape[0])


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
        chains.run(1, zs_all[w], lu_all[w], move_offset=w)
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
            chains.run(1, zs_all[args.warmup + k], lu_all[args.warmup + k], move_offset=args.warmup + k)
            e1.record(stream)
            times.append((e0, e1))
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    dev_s = sum(a.elapsed_time(b) for a, b in times) / 1e3
    status = chains.status_host()
    if np.count_nonzero(status):
        raise RuntimeError(f"{np.count_nonzero(status)} chains stopped (status != 0): throughput would count "
                           "leapfrogs that were not run")
    bufs = chains._rec[1]
    acc = float(bufs["accept"].float().mean().item())
    sweeps = float(bufs["sweeps_mean"].mean().item())
    t_max = torch.tensor([dev_s], dtype=torch.float64,
                         device=_reduce_device(dist) if world > 1 else "cuda")
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
    for k in range(e2e_steps):
        z, lu = draws()
        zpin.numpy()[...] = z
        lpin.numpy()[...] = lu
        zd = zpin.to("cuda", non_blocking=True)
        ld = lpin.to("cuda", non_blocking=True)
        b = chains.run(1, zd, ld, move_offset=args.warmup + args.steps + k)
        for k2, t in out_pin.items():
            t.copy_(b[k2], non_blocking=True)
        acc_pin.copy_(b["accept"], non_blocking=True)
        q_pin.copy_(chains.q, non_blocking=True)
        torch.cuda.synchronize()
    e2e_t = time.perf_counter() - t0
    e2e_max = torch.tensor([e2e_t], dtype=torch.float64,
                         device=_reduce_device(dist) if world > 1 else "cuda")
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
        F = canonical_flops_per_leapfrog(N, (D,), d, s=max(1.0, sweeps))
        achieved = F * Z * LEAPFROGS * args.steps / dev_s / 1e12
        dgemm = measure_dgemm_tflops(torch)
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator simulate_logistic(1, n=512, seed=0))",
            "config": {"workload": C2_NAME,
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
        tpath = os.path.join(ROOT, "profiles", "r2_traffic_k_run_moves.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                tr = json.load(f)
            if tr.get("chains") == Z and tr.get("leapfrogs") == LEAPFROGS:
                line["roofline"]["traffic"] = tr["dram_bytes_per_launch"]
                line["roofline"]["traffic_unit"] = "bytes/launch (DRAM read+write, ncu)"
                line["roofline"]["traffic_source"] = "profiles/r2_traffic_k_run_moves.json"
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
    ap.add_argument("--workload", default="c4", choices=["c4", "c2", "c5"])
    ap.add_argument("--c5-chains", type=int, default=64)
    ap.add_argument("--c5-moves", type=int, default=2, help="moves per rung (C5)")
    ap.add_argument("--leapfrogs", type=int, default=0, help="leapfrogs per move (C4 default 100)")
    ap.add_argument("--e2e-steps", type=int, default=3, help="moves timed end to end (C4)")
    ap.add_argument("--chains", type=int, default=0, help="chains per GPU (default SMs x chains-per-sm)")
    ap.add_argument("--chains-per-sm", type=int, default=12)
    ap.add_argument("--warm-order", default=None, choices=["cyclic", "parallel", "refine"],
                    help="warm eigensolver (C4 default refine, C2 default cyclic)")
    ap.add_argument("--cold-order", default="cyclic", choices=["cyclic", "parallel", "dc"],
                    help="C4 cold decompositions (chain start, rejections): reference order (default) or "
                         "tridiagonalisation + divide and conquer")
    ap.add_argument("--ref-leapfrogs", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ess-moves", type=int, default=300, help="recorded moves of the min-ESS pilot (0: skip)")
    ap.add_argument("--ess-burnin", type=int, default=100)
    ap.add_argument("--ess-chains-per-sm", type=int, default=2)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c4":
        run_gpu_c4(args)
    elif args.workload == "c5":
        run_gpu_c5(args)
    else:
        args.warm_order = args.warm_order or "cyclic"
        run_gpu(args)


if __name__ == "__main__":
    main()
