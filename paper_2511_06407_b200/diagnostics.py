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
