"""Pins for the oracle's Lanczos / extreme-eigenvalue estimator (App. B.2).

Against numpy's dense eigensolver: interlacing (Ritz extremes inside the spectrum),
Krylov exactness at J = N, the SPEC examples 5I and diag(1..100)."""
import numpy as np

import workloads
from oracle import DenseOperator, KernelOperator, estimate_spectrum, lanczos


def _ritz(alphas, betas):
    import scipy.linalg
    out = []
    for a, b in zip(alphas, betas):
        out.append(scipy.linalg.eigvalsh_tridiagonal(np.asarray(a), np.asarray(b[:len(a) - 1])))
    return out


def test_full_lanczos_recovers_spectrum():
    k = workloads.spectrum_matrix(16, "inv_linear", seed=3) + 0.1 * np.eye(16)
    s = workloads.lanczos_start(16, 2)
    al, be = lanczos(DenseOperator(k).mvm, s, 16)
    ev = np.linalg.eigvalsh(k)
    for r in _ritz(al, be):
        np.testing.assert_allclose(np.sort(r), ev, rtol=1e-8, atol=1e-10)


def test_interlacing_on_kernel_matrix():
    x = workloads.points(200, 3)
    op = KernelOperator(x, "rbf", 0.3, 1.0, sigma2=1e-2)
    ev = np.linalg.eigvalsh(op.dense())
    al, be = lanczos(op.mvm, workloads.lanczos_start(200, 4), 10)
    for r in _ritz(al, be):
        assert r.min() >= ev[0] - 1e-10
        assert r.max() <= ev[-1] + 1e-10
    lmin, lmax, rmin, rmax = estimate_spectrum(op.mvm, workloads.lanczos_start(200, 16), 10, lower_bound=1e-2)
    assert abs(rmax / ev[-1] - 1) < 1e-6        # Ritz_max converges within 10 iterations
    assert lmax >= ev[-1] and lmin <= ev[0]     # the safety margins bracket the spectrum (reading G6)


def test_scalar_operator_breakdown():
    op = DenseOperator(5.0 * np.eye(30))
    lmin, lmax, rmin, rmax = estimate_spectrum(op.mvm, workloads.lanczos_start(30, 3), 10)
    assert abs(rmin - 5) < 1e-12 and abs(rmax - 5) < 1e-12
    assert abs(lmin - 4.95) < 1e-12 and abs(lmax - 5.05) < 1e-12


def test_diag_1_to_100():
    op = DenseOperator(np.diag(np.arange(1.0, 101.0)))
    _, _, rmin, rmax = estimate_spectrum(op.mvm, workloads.lanczos_start(100, 1), 30)
    assert abs(rmin - 1) / 1 < 0.01 and abs(rmax - 100) / 100 < 0.01
