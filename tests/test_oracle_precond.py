"""Pins for the oracle's preconditioned route (App. A).

* P = L L^T + sigma2 I half powers vs numpy eigh of the dense P; P^{1/2}P^{1/2} = P; P^{-1} P = I
  (S:406-408);
* pivoted Cholesky: rank-N reconstruction, exact rank-1 recovery, monotone trace residual
  (S:418-420); lambda_min(P^{-1/2} K P^{-1/2}) >= 1 for sigma2_P = sigma2 (Schur complement,
  reading G6);
* P = I reproduces the unpreconditioned CIQ;
* Gram identities R R^T = K and R' R'^T = K^{-1} by applying to identity columns;
* preconditioning does not increase the iterations to tolerance."""
import numpy as np

import workloads
from oracle import DenseOperator, KernelOperator, LowRankPlusDiag, ciq, pivoted_cholesky, precond_ciq


def eig_fn(a, f):
    lam, v = np.linalg.eigh(a)
    return (v * f(lam)[None, :]) @ v.T


def test_lowrank_plus_diag_powers():
    rng_l = workloads.rhs(64, 8, seed=31).astype(np.float64)
    p = LowRankPlusDiag(rng_l, 0.3)
    pd = p.dense()
    v = workloads.rhs(64, 3, seed=32).astype(np.float64)
    np.testing.assert_allclose(p.power(v, 0.5), eig_fn(pd, np.sqrt) @ v, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(p.power(v, -0.5), eig_fn(pd, lambda x: x ** -0.5) @ v, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(p.power(p.power(v, 0.5), 0.5), p.apply(v), rtol=1e-10)
    np.testing.assert_allclose(p.power(p.apply(v), -1.0), v, rtol=1e-10)
    z = LowRankPlusDiag(np.zeros((64, 0)), 0.25)
    np.testing.assert_allclose(z.power(v, -1.0), v / 0.25)          # S:427 L = 0 -> v / sigma2


def test_pivoted_cholesky_properties():
    x = workloads.points(80, 3)
    op = KernelOperator(x, "matern52", 0.3, 1.0, sigma2=0.0)
    k = op.dense()
    lfull = pivoted_cholesky(op, 80)
    np.testing.assert_allclose(lfull @ lfull.T, k, atol=1e-8)
    u = workloads.rhs(30, 1, seed=5).astype(np.float64)[:, 0]
    l1 = pivoted_cholesky(DenseOperator(np.outer(u, u)), 1)
    np.testing.assert_allclose(l1 @ l1.T, np.outer(u, u), atol=1e-12)
    traces = [np.trace(k - (lr := pivoted_cholesky(op, r)) @ lr.T) for r in (2, 4, 8, 16)]
    assert all(b < a for a, b in zip(traces, traces[1:]))


def test_preconditioned_operator_lambda_min_at_least_one():
    x = workloads.points(300, 3)
    sigma2 = 1e-3
    op = KernelOperator(x, "matern52", 0.3, 1.0, sigma2=sigma2)
    pre = LowRankPlusDiag(pivoted_cholesky(op, 20), sigma2)
    pm = eig_fn(pre.dense(), lambda x: x ** -0.5)
    m = pm @ op.dense() @ pm
    assert np.linalg.eigvalsh(0.5 * (m + m.T)).min() >= 1 - 1e-9


def test_identity_preconditioner_reproduces_plain_ciq():
    x = workloads.points(100, 3)
    op = KernelOperator(x, "rbf", 0.3, 1.0, sigma2=0.05)
    b = workloads.rhs(100, 2).astype(np.float64)
    ev = np.linalg.eigvalsh(op.dense())
    pre = LowRankPlusDiag(np.zeros((100, 0)), 1.0)
    for mode in ("whiten", "sqrt"):
        r1 = precond_ciq(op, pre, b, q=8, max_iters=200, tol=0.0, mode=mode, spectrum=(ev[0], ev[-1]))
        r0 = ciq(op, b, q=8, max_iters=200, tol=0.0, mode="invsqrt" if mode == "whiten" else "sqrt",
                 spectrum=(ev[0], ev[-1]))
        np.testing.assert_allclose(r1.out, r0.out, rtol=1e-10, atol=1e-12)


def test_gram_identities():
    n = 48
    x = workloads.points(n, 2)
    sigma2 = 1e-2
    op = KernelOperator(x, "matern52", 0.4, 1.0, sigma2=sigma2)
    k = op.dense()
    pre = LowRankPlusDiag(pivoted_cholesky(op, 8), sigma2)
    eye = np.eye(n)
    s = workloads.lanczos_start(n, 4)
    rp = precond_ciq(op, pre, eye, q=16, max_iters=400, tol=1e-12, mode="whiten", lanczos_start=s).out
    r = precond_ciq(op, pre, eye, q=16, max_iters=400, tol=1e-12, mode="sqrt", lanczos_start=s).out
    kinv = np.linalg.inv(k)
    assert np.linalg.norm(rp @ rp.T - kinv) / np.linalg.norm(kinv) < 1e-4
    assert np.linalg.norm(r @ r.T - k) / np.linalg.norm(k) < 1e-4


def test_preconditioning_reduces_iterations():
    x = workloads.points(600, 3)
    sigma2 = 1e-3
    op = KernelOperator(x, "matern52", 0.3, 1.0, sigma2=sigma2)
    b = workloads.rhs(600, 2).astype(np.float64)
    s = workloads.lanczos_start(600, 4)
    plain = ciq(op, b, q=12, max_iters=3000, tol=1e-4, mode="invsqrt", lanczos_start=s)
    pre = LowRankPlusDiag(pivoted_cholesky(op, 64), sigma2)
    pc = precond_ciq(op, pre, b, q=12, max_iters=3000, tol=1e-4, mode="whiten", lanczos_start=s)
    assert pc.converged and pc.iters < plain.iters


def test_pinv_only_recurrence_equals_symmetric_route():
    """App. A: preconditioned msMINRES needs only P^{-1}.  An independent fp64
    emulation of that r-space (Paige-Saunders/Choi) recurrence for (K + t_q P) x = P^{1/2} b must
    reproduce the oracle's explicit M = P^{-1/2} K P^{-1/2} route (reading G13)."""
    import math as _m
    x = workloads.points(300, 3)
    sigma2 = 1e-3
    op = KernelOperator(x, "matern52", 0.3, 1.0, sigma2=sigma2)
    pre = LowRankPlusDiag(pivoted_cholesky(op, 24), sigma2)
    b = workloads.rhs(300, 3).astype(np.float64)
    ref = precond_ciq(op, pre, b, q=8, max_iters=400, tol=0.0, mode="whiten", spectrum=(1.0, 2000.0))
    assert np.max(np.abs(ref.solve.phibar) / ref.solve.beta1) < 1e-9
    k = op.dense()
    t, w = ref.t, ref.w
    cvec = pre.power(b, 0.5)
    y_acc = np.zeros_like(b)
    for col in range(3):
        for q in range(len(t)):
            # scipy-style preconditioned MINRES on (K + t_q P) with preconditioner P (M^{-1} = P^{-1})
            r1 = cvec[:, col].copy()
            y = pre.power(r1, -1.0)
            beta1 = _m.sqrt(r1 @ y)
            beta, oldb = beta1, 0.0
            r2 = r1.copy()
            dbar = epsln = 0.0
            phibar = beta1
            cs, sn = -1.0, 0.0
            wv = np.zeros(300); w2 = np.zeros(300); xq = np.zeros(300)
            for itn in range(1, 401):
                v = y / beta
                y = k @ v + t[q] * pre.apply(v)
                if itn >= 2:
                    y = y - (beta / oldb) * r1
                alfa = v @ y
                y = y - (alfa / beta) * r2
                r1, r2 = r2, y
                y = pre.power(r2, -1.0)
                oldb, beta = beta, _m.sqrt(max(r2 @ y, 0.0))
                oldeps = epsln
                delta = cs * dbar + sn * alfa
                gbar = sn * dbar - cs * alfa
                epsln = sn * beta
                dbar = -cs * beta
                gamma = max(_m.hypot(gbar, beta), 1e-300)
                cs, sn = gbar / gamma, beta / gamma
                phi = cs * phibar
                phibar = sn * phibar
                w1, w2 = w2, wv
                wv = (v - oldeps * w1 - delta * w2) / gamma
                xq = xq + phi * wv
                if beta == 0.0:
                    break
            y_acc[:, col] += w[q] * xq
    np.testing.assert_allclose(y_acc, ref.out, rtol=1e-6, atol=1e-9)
