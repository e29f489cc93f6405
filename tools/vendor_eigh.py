"""Vendor eigensolver baseline (SURVEY.md 8(d) "Vendor eigh baseline").

Times cuSOLVER (through torch.linalg.eigh, fp64: syevjBatched / syevd) beside this repo's
eigensolvers on the same Hessians of the SURVEY.md 8(d) models:

* small d (C2 d=34, C3a d=83, C3b d=163): Z Hessians at Z distinct points near q=0;
  ours = sgp_eigh_cold (bit-exact cyclic Jacobi from the identity, metric.py:112-127) and
  sgp_eigh_warm (the dynamic decomposition in the basis of a neighbouring point,
  metric.py:145-185 -- what the leapfrog actually calls, fp_q times per leapfrog);
* C4 (d=2083): the chain-start Hessian; ours = sgp_eigh_dc (tridiagonalisation + divide and
  conquer) against torch.linalg.eigh (cuSOLVER syevd).

The paper compares its dynamic eigh against "prop.(syevd)/prop.(syevj)"; the
vendor solvers return eigenvalues sorted and eigenvectors in their own signs, so only spectra
are compared (max relative deviation of the sorted eigenvalues).

    python tools/vendor_eigh.py [--skip-c4]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_06407_b200 import _native as nat  # noqa: E402
from paper_2511_06407_b200 import rrgp  # noqa: E402
from paper_2511_06407_b200.posterior import PosteriorTarget  # noqa: E402
from paper_2511_06407_b200.sampler import ChainConfig, DeviceChains  # noqa: E402

ZETA, CAP = 1e-13, 30


def dev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def small_case(name, target, Z):
    L = nat.lib()
    d = target.dim
    rng = np.random.default_rng(0)
    q0 = 0.05 * rng.standard_normal((Z, d))
    q1 = q0 + 1e-4 * rng.standard_normal((Z, d))     # a leapfrog-sized move
    H0 = nat.dev_f64(target.device.eval(1.0, q0, nat.EVAL_HESSIAN)["hess"])
    H1 = nat.dev_f64(target.device.eval(1.0, q1, nat.EVAL_HESSIAN)["hess"])
    lam0, psi0 = nat.empty_f64(Z, d), nat.empty_f64(Z, d, d)
    lam, psi = nat.empty_f64(Z, d), nat.empty_f64(Z, d, d)
    sw, sw1, since0, since = (nat.zeros_i32(Z) for _ in range(4))

    def cold():
        nat.check(L.sgp_eigh_cold(Z, d, nat.ptr(H0), ZETA, CAP, nat.ptr(lam0), nat.ptr(psi0), nat.ptr(sw),
                                  nat.stream()), "sgp_eigh_cold")

    def warm():
        nat.check(L.sgp_eigh_warm(Z, d, nat.ptr(H1), nat.ptr(psi0), nat.ptr(since0), 10, ZETA, CAP,
                                  nat.ORDER_CODES["cyclic"], nat.ptr(lam), nat.ptr(psi), nat.ptr(since),
                                  nat.ptr(sw1), nat.stream()), "sgp_eigh_warm")

    t_cold = dev_time(cold)
    t_warm = dev_time(warm)
    t_vendor = dev_time(lambda: torch.linalg.eigh(H1))
    t_vendor_vals = dev_time(lambda: torch.linalg.eigvalsh(H1))
    ref = torch.linalg.eigvalsh(H1).cpu().numpy()
    ours = np.sort(lam.cpu().numpy(), axis=1)
    dev = float(np.max(np.abs(ours - ref) / np.max(np.abs(ref), axis=1, keepdims=True)))
    row = dict(config=name, d=d, Z=Z, ours_cold_ms=t_cold * 1e3, ours_warm_ms=t_warm * 1e3,
               cold_sweeps_mean=float(sw.float().mean()), warm_sweeps_mean=float(sw1.float().mean()),
               vendor_eigh_ms=t_vendor * 1e3, vendor_eigvalsh_ms=t_vendor_vals * 1e3,
               warm_speedup_vs_vendor=t_vendor / t_warm, spectrum_max_rel_dev=dev)
    print(json.dumps(row), flush=True)
    return row


def c4_case():
    """C4: the chain-start Hessian.  Ours: sgp_eigh_dc (blocked Householder tridiagonalisation +
    divide and conquer, cold_order="dc"); the reference-order cold Jacobi (the default cold path,
    bit-exact) takes ~17 s here (bench.py's cold_init_s) and is not re-timed."""
    L = nat.lib()
    data, _ = rrgp.simulate_meanvar(34, 19, n=8192, seed=0)
    model = rrgp.build_model("nl-meanvar", data.x)
    target = PosteriorTarget(model, data)
    d = target.dim
    q = np.zeros((1, d))
    H = nat.dev_f64(target.device.eval(1.0, q, nat.EVAL_HESSIAN)["hess"][0])
    lam, psi = nat.empty_f64(d), nat.empty_f64(d, d)

    def dc():
        nat.check(L.sgp_eigh_dc(1, d, nat.ptr(H), nat.ptr(lam), nat.ptr(psi), nat.stream()), "sgp_eigh_dc")
    t_dc = dev_time(dc, reps=3)
    t_vendor = dev_time(lambda: torch.linalg.eigh(H), reps=3)
    ref = torch.linalg.eigvalsh(H).cpu().numpy()
    dev = float(np.max(np.abs(lam.cpu().numpy() - ref)) / np.max(np.abs(ref)))
    p = psi.cpu().numpy()
    orth = float(np.max(np.abs(p.T @ p - np.eye(d))))
    row = dict(config="C4 nl-meanvar", d=d, Z=1, ours_dc_ms=t_dc * 1e3,
               ours_note="sgp_eigh_dc: tridiagonalisation + divide and conquer (cold_order='dc')",
               vendor_eigh_ms=t_vendor * 1e3, dc_speedup_vs_vendor=t_vendor / t_dc,
               spectrum_max_rel_dev=dev, orthonormality_max_dev=orth)
    print(json.dumps(row), flush=True)
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c4", action="store_true")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    rows = []
    d2, _ = rrgp.simulate_logistic(1, n=512, seed=0)
    rows.append(small_case("C2 logistic N=512", PosteriorTarget(rrgp.build_model("logistic", d2.x), d2), 1776))
    dm, _ = rrgp.simulate_meanvar(2, 19, n=2000, seed=0)
    ylab = np.where(dm.y > np.median(dm.y), 1.0, -1.0)
    d3a = rrgp.Dataset(dm.x, ylab)
    rows.append(small_case("C3a logistic NMES", PosteriorTarget(rrgp.build_model("logistic", dm.x), d3a), 296))
    rows.append(small_case("C3b nl-meanvar NMES", PosteriorTarget(rrgp.build_model("nl-meanvar", dm.x), dm), 296))
    if not args.skip_c4:
        rows.append(c4_case())
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    t = time.perf_counter()
    main()
    print(f"total {time.perf_counter() - t:.1f}s")
