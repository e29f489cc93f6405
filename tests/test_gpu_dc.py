"""Blocked Householder tridiagonalisation + divide and conquer (csrc/sgp_dc.cuh; north star (3)).

The solver does not follow the reference's Jacobi order, so the check is the decomposition itself
against LAPACK (numpy.linalg.eigvalsh, test infrastructure only): eigenvalues, the residual
||A Psi - Psi Lambda||, orthonormality of Psi.  Matrices cover every code path: one leaf
(d <= 48), the merge tree with and without deflation (repeated and clustered eigenvalues, an
already-diagonal matrix, Wilkinson's close pairs), graded spectra and the C4 size d = 2083.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2511_06407_b200 import metric as M  # noqa: E402

EPS = np.finfo(float).eps


def _sym(a):
    return 0.5 * (a + a.T)


def _random(n, seed):
    return _sym(np.random.default_rng(seed).standard_normal((n, n)))


def _with_spectrum(lam, seed):
    n = len(lam)
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, n)))
    return _sym((q * np.asarray(lam, dtype=float)) @ q.T)


def _wilkinson(n):
    m = (n - 1) / 2.0
    a = np.diag(np.abs(np.arange(n) - m)) + np.diag(np.ones(n - 1), 1) + np.diag(np.ones(n - 1), -1)
    return a


def _check(a, lam, psi, tol_scale=1.0):
    n = a.shape[0]
    anorm = np.linalg.norm(a, 2) if n <= 1200 else np.max(np.abs(np.linalg.eigvalsh(a)))
    anorm = max(anorm, np.finfo(float).tiny)
    ref = np.linalg.eigvalsh(a)
    assert np.all(np.diff(lam) >= 0.0), "eigenvalues must be ascending"
    lam_err = np.max(np.abs(lam - ref)) / anorm
    res = np.linalg.norm(a @ psi - psi * lam) / (anorm * np.sqrt(n))
    orth = np.max(np.abs(psi.T @ psi - np.eye(n)))
    bound = tol_scale * 64 * EPS * np.sqrt(n) * 10
    assert lam_err < bound, (lam_err, bound)
    assert res < bound, (res, bound)
    assert orth < bound * 10, (orth, bound)
    return lam_err, res, orth


@pytest.mark.parametrize("n", [1, 2, 3, 17, 48, 49, 64, 97, 100, 333, 1000])
def test_random_symmetric(n):
    a = _random(n, seed=n)
    lam, psi = M.eigh_dc(a)
    _check(a, lam, psi)


def test_c4_size():
    n = 2083
    a = _random(n, seed=5) + np.diag(np.linspace(0.0, 50.0, n))
    lam, psi = M.eigh_dc(a)
    _check(a, lam, psi)


def test_unsymmetric_input_is_symmetrised():
    a = np.random.default_rng(3).standard_normal((150, 150))
    lam, psi = M.eigh_dc(a)
    _check(_sym(a), lam, psi)


@pytest.mark.parametrize("n", [100, 700])
def test_repeated_eigenvalues_deflate(n):
    lam0 = np.repeat([-3.0, 0.0, 1.0, 2.5, 7.0], n // 5 + 1)[:n]
    a = _with_spectrum(lam0, seed=n)
    lam, psi = M.eigh_dc(a)
    _check(a, lam, psi)
    np.testing.assert_allclose(lam, np.sort(lam0), atol=1e-12 * 7.0 * np.sqrt(n))


@pytest.mark.parametrize("n", [60, 500])
def test_clustered_eigenvalues(n):
    rng = np.random.default_rng(n)
    lam0 = np.sort(np.concatenate([1.0 + 1e-13 * rng.standard_normal(n // 2),
                                   rng.uniform(-1, 1, n - n // 2)]))
    a = _with_spectrum(lam0, seed=n + 1)
    lam, psi = M.eigh_dc(a)
    _check(a, lam, psi)


def test_diagonal_matrix():
    d = np.random.default_rng(9).standard_normal(300)
    lam, psi = M.eigh_dc(np.diag(d))
    np.testing.assert_array_equal(lam, np.sort(d))
    _check(np.diag(d), lam, psi)


def test_wilkinson_close_pairs():
    a = _wilkinson(201)
    lam, psi = M.eigh_dc(a)
    _check(a, lam, psi)


def test_graded_spectrum():
    n = 400
    lam0 = np.logspace(-8, 6, n) * np.where(np.arange(n) % 3 == 0, -1.0, 1.0)
    a = _with_spectrum(lam0, seed=4)
    lam, psi = M.eigh_dc(a)
    _check(a, lam, psi)


def test_zero_matrix():
    lam, psi = M.eigh_dc(np.zeros((70, 70)))
    np.testing.assert_array_equal(lam, np.zeros(70))
    np.testing.assert_allclose(psi.T @ psi, np.eye(70), atol=1e-14)
