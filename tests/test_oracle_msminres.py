"""Pins for the oracle's msMINRES (App. C).

* per shift, equal to scipy.sparse.linalg.minres(K, b, shift=-t_q) -- an independent Paige-Saunders
  implementation -- at small J (before finite-precision Lanczos effects);
* K = cI: x_q = b/(c + t_q) after one iteration;
* Krylov exactness at J = N;
* the recurrence residual |phibar| equals the explicit residual ||(K + t_q I) x_q - b||;
* residual monotone non-increasing in J; Lemma 1 bound (with the Chebyshev
  factor 2, reading G19);
* exactly J MVMs regardless of Q (Property 1); b = 0 -> 0."""
import math

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import workloads
from oracle import DenseOperator, KernelOperator, hht_rule, msminres


def _kernel_op(n=300, sigma2=1e-2):
    return KernelOperator(workloads.points(n, 3), "rbf", 0.4, 1.0, sigma2=sigma2)


@pytest.mark.parametrize("j", [1, 2, 5, 8])
def test_matches_scipy_minres_per_shift(j):
    op = _kernel_op()
    b = workloads.rhs(op.n, 2).astype(np.float64)
    t, _ = hht_rule(1e-2, 60.0, 8)
    res = msminres(op.mvm, b, t, j, tol=0.0)
    a = op.dense()
    for q in range(len(t)):
        for c in range(2):
            xs, _ = spla.minres(a, b[:, c], shift=-t[q], maxiter=j, rtol=0.0)
            err = np.linalg.norm(res.x[q, :, c] - xs) / np.linalg.norm(xs)
            assert err < 1e-10, (q, c, err)


def test_scalar_operator_one_step():
    op = DenseOperator(4.0 * np.eye(10))
    b = workloads.rhs(10, 3).astype(np.float64)
    t = np.array([1.0, 3.0, 0.5])
    res = msminres(op.mvm, b, t, 50, tol=1e-10)
    assert res.iters == 1 and res.mvms == 1
    for q in range(3):
        np.testing.assert_allclose(res.x[q], b / (4.0 + t[q]), rtol=1e-14)


def test_krylov_exactness():
    k = workloads.spectrum_matrix(32, "inv_sqrt", seed=4)
    b = workloads.rhs(32, 1).astype(np.float64)
    t = np.array([0.0, 0.3])
    res = msminres(DenseOperator(k).mvm, b, t, 32, tol=0.0)
    for q in range(2):
        np.testing.assert_allclose(res.x[q], np.linalg.solve(k + t[q] * np.eye(32), b), rtol=1e-8)


def test_recurrence_residual_is_explicit_residual_and_monotone():
    op = _kernel_op()
    a = op.dense()
    b = workloads.rhs(op.n, 2).astype(np.float64)
    t, _ = hht_rule(1e-2, 60.0, 8)
    prev = None
    for j in (5, 10, 20, 40):
        res = msminres(op.mvm, b, t, j, tol=0.0)
        for q in range(len(t)):
            explicit = np.linalg.norm((a + t[q] * np.eye(op.n)) @ res.x[q] - b, axis=0)
            np.testing.assert_allclose(np.abs(res.phibar[q]), explicit, rtol=1e-6, atol=1e-12)
        if prev is not None:
            assert np.all(np.abs(res.phibar) <= prev * (1 + 1e-10) + 1e-14)
        prev = np.abs(res.phibar)


def test_lemma1_bound():
    op = _kernel_op()
    ev = np.linalg.eigvalsh(op.dense())
    b = workloads.rhs(op.n, 1).astype(np.float64)
    t, _ = hht_rule(ev[0], ev[-1], 8)
    for j in (3, 10, 30):
        res = msminres(op.mvm, b, t, j, tol=0.0)
        for q in range(len(t)):
            kq = (ev[-1] + t[q]) / (ev[0] + t[q])
            rho = (math.sqrt(kq) - 1) / (math.sqrt(kq) + 1)
            assert abs(res.phibar[q, 0]) <= 2 * rho ** j * res.beta1[0] * (1 + 1e-9)


def test_mvm_count_independent_of_q_and_zero_rhs():
    op = _kernel_op()
    b = workloads.rhs(op.n, 1).astype(np.float64)
    for q in (1, 8, 16):
        t, _ = hht_rule(1e-2, 60.0, q)
        res = msminres(op.mvm, b, t, 25, tol=0.0)
        assert res.mvms == res.iters == 25
    z = msminres(op.mvm, np.zeros((op.n, 2)), np.array([1.0]), 10)
    assert z.iters == 0 and np.all(z.x == 0)


def test_tolerance_stop():
    op = _kernel_op()
    b = workloads.rhs(op.n, 3).astype(np.float64)
    t, _ = hht_rule(1e-2, 60.0, 8)
    res = msminres(op.mvm, b, t, 400, tol=1e-6)
    assert res.converged and res.iters < 400
    assert np.max(np.abs(res.phibar) / res.beta1[None, :]) <= 1e-6
    res2 = msminres(op.mvm, b, t, res.iters - 1, tol=0.0)
    assert np.max(np.abs(res2.phibar) / res2.beta1[None, :]) > 1e-6
