"""Host-side MCMC diagnostics: effective sample size and split R-hat.

The reference has neither; they are added so the headline
min-ESS/s can be reported.  The same function is applied to GPU and CPU-oracle
samples, so ESS parity between the two follows from sample parity.  Parity of
the ESS definition itself is unpinned by the reference.
"""

from __future__ import annotations

import numpy as np


def autocorrelation(x):
    """Normalised autocorrelation of a 1-d series via FFT (biased estimator)."""
    x = np.asarray(x, dtype=float)
    n = x.shape[0]
    x = x - x.mean()
    size = 1 << (2 * n - 1).bit_length()
    f = np.fft.rfft(x, size)
    acov = np.fft.irfft(f * np.conj(f), size)[:n] / n
    if acov[0] <= 0.0:
        return np.ones(n)
    return acov / acov[0]


def ess_geyer(x):
    """ESS by Geyer's initial monotone sequence estimator.

    tau = -1 + 2 sum_k Gamma_k with Gamma_k = rho_2k + rho_2k+1 truncated at the
    first non-positive pair and made monotone non-increasing; ESS = n / tau.
    """
    x = np.asarray(x, dtype=float)
    n = x.shape[0]
    if n < 4:
        return float(n)
    if np.all(x == x[0]):
        return 0.0
    rho = autocorrelation(x)
    m = (n - 1) // 2
    gam = rho[0:2 * m:2] + rho[1:2 * m + 1:2]
    tau_sum = 0.0
    prev = np.inf
    for g in gam:
        if g <= 0.0:
            break
        g = min(g, prev)
        tau_sum += g
        prev = g
    tau = max(-1.0 + 2.0 * tau_sum, 1.0 / np.log10(max(n, 10)))
    return float(n / tau)


def ess_per_coordinate(samples):
    """samples: (n, d) -> ESS per coordinate."""
    s = np.asarray(samples, dtype=float)
    return np.array([ess_geyer(s[:, j]) for j in range(s.shape[1])])


def min_ess(samples):
    return float(np.min(ess_per_coordinate(samples)))


def split_rhat(chains):
    """Split-R-hat per coordinate for chains of shape (m, n, d)."""
    c = np.asarray(chains, dtype=float)
    m, n, d = c.shape
    half = n // 2
    parts = np.concatenate([c[:, :half], c[:, half:2 * half]], axis=0)
    mm, nn = parts.shape[0], parts.shape[1]
    means = parts.mean(axis=1)
    variances = parts.var(axis=1, ddof=1)
    w = variances.mean(axis=0)
    b = nn * means.var(axis=0, ddof=1)
    var_plus = (nn - 1) / nn * w + b / nn
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.sqrt(var_plus / w)


def rhat_from_half_stats(means, variances, nn):
    """split_rhat's combination step on gathered half-chain statistics."""
    w = variances.mean(axis=0)
    b = nn * means.var(axis=0, ddof=1)
    var_plus = (nn - 1) / nn * w + b / nn
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.sqrt(var_plus / w)


def distributed_split_rhat(local_chains, local_ids, n_chains):
    """Split-R-hat over replica chains spread across ``torch.distributed`` ranks
    (C1-C4 run as replicas; the only exchange is per-chain summaries).

    local_chains: (m_local, n, d) samples of this rank's chains, global ids local_ids (at most
    ceil(M/W) per rank, e.g. chain z on rank z mod W).  One
    ``all_gather_into_tensor`` of [ceil(M/W), 1 + 4d] fp64 rows (chain id, half-chain means
    and variances) -- d-sized, independent of the chain length.  The result equals
    ``split_rhat`` of all chains stacked in id order, bit for bit."""
    import torch
    import torch.distributed as dist

    c = np.asarray(local_chains, dtype=float)
    m_local, n, d = c.shape
    half = n // 2
    first = c[:, :half]
    second = c[:, half:2 * half]
    rows = np.zeros((m_local, 1 + 4 * d))
    for k in range(m_local):
        rows[k, 0] = local_ids[k] + 1
        rows[k, 1:1 + d] = first[k].mean(axis=0)
        rows[k, 1 + d:1 + 2 * d] = first[k].var(axis=0, ddof=1)
        rows[k, 1 + 2 * d:1 + 3 * d] = second[k].mean(axis=0)
        rows[k, 1 + 3 * d:] = second[k].var(axis=0, ddof=1)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        world = dist.get_world_size()
        per = (n_chains + world - 1) // world
        block = np.zeros((per, 1 + 4 * d))
        block[:m_local] = rows
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        src = torch.as_tensor(block, dtype=torch.float64, device=dev)
        out = torch.empty((world * per, 1 + 4 * d), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(out, src)
        allr = out.cpu().numpy()
        allr = allr[allr[:, 0] > 0]
    else:
        allr = rows
    allr = allr[np.argsort(allr[:, 0])]
    means = np.concatenate([allr[:, 1:1 + d], allr[:, 1 + 2 * d:1 + 3 * d]], axis=0)
    variances = np.concatenate([allr[:, 1 + d:1 + 2 * d], allr[:, 1 + 3 * d:]], axis=0)
    return rhat_from_half_stats(means, variances, half)
