"""Offline check of the warm-path eigenvector refinement (csrc/sgp_large.cuh lg_eig_refine) on a
warm problem S = Psi^T H Psi dumped by SGP_DUMP_REFINE (float64 tol + d x d).  Usage:
python tools/refine_sim.py dump.bin"""
import numpy as np, sys
raw = np.fromfile(sys.argv[1], dtype=np.float64)
tol = raw[0]; d = int(round(np.sqrt(raw.size - 1))); A = raw[1:].reshape(d, d); A = 0.5*(A+A.T)
skip = tol/d
P = np.eye(d)
for it in range(8):
    S = P.T @ A @ P; S = 0.5*(S+S.T)
    Sod = S - np.diag(np.diag(S)); off = np.sqrt(np.sum(Sod*Sod))
    G = P.T @ P; G = 0.5*(G+G.T)
    lam = np.diag(S)/np.diag(G)
    R = np.eye(d) - G
    gap = lam[None, :] - lam[:, None]
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.abs(Sod)/np.abs(gap)
    np.fill_diagonal(ratio, 0)
    act = np.abs(Sod) > skip
    bad = np.triu((ratio > 1.0) & act, 1)
    print(f"it {it}: off {off:.3e} tol {tol:.2e} pairs>1 {bad.sum()} max ratio {np.nanmax(np.where(act, ratio, 0)):.3e} |G-I| {np.abs(R).max():.1e}")
    for i, j in list(zip(*np.where(bad)))[:4]:
        print(f"     ({i},{j}) lam {lam[i]:.15g} {lam[j]:.15g} gap {gap[i,j]:.3e} s {Sod[i,j]:.3e}")
    if off <= tol: break
    with np.errstate(divide="ignore", invalid="ignore"):
        Em = (Sod + lam[None, :]*R)/gap
    Em = np.where(act, Em, 0.5*R)
    np.fill_diagonal(Em, 0.5*np.diag(R))
    P = P + P @ Em
