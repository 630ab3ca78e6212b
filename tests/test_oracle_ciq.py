"""Pins for the oracle's CIQ driver (eq. contour_integral_quad; Theorem 1).

Against the plain definition K^{+-1/2} b = V Lambda^{+-1/2} V^T b (numpy eigh): the C1 config, the
paper's synthetic spectra (Fig. quad_error), the scalar operator 4I,
sqrt(sqrt(b)) = K b, Theorem 1 / Corollary 1 inequalities, and error-vs-Q decay."""
import math

import numpy as np
import pytest

import workloads
from oracle import DenseOperator, KernelOperator, ciq, hht_rule


def eig_power(a, b, p):
    lam, v = np.linalg.eigh(a)
    return v @ (lam[:, None] ** p * (v.T @ b))


def relerr(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


def test_scalar_operator():
    op = DenseOperator(4.0 * np.eye(20))
    b = workloads.rhs(20, 2).astype(np.float64)
    s = workloads.lanczos_start(20, 4)
    r = ciq(op, b, q=8, max_iters=50, tol=1e-10, mode="invsqrt", lanczos_start=s)
    np.testing.assert_allclose(r.out, b / 2, rtol=1e-5)
    r = ciq(op, b, q=8, max_iters=50, tol=1e-10, mode="sqrt", lanczos_start=s)
    np.testing.assert_allclose(r.out, 2 * b, rtol=1e-5)
    # Lanczos on 4I hits an invariant subspace after 1 step: 1 + J=1 + final K
    assert r.mvms == 1 + 1 + 1


@pytest.mark.parametrize("mode,p", [("sqrt", 0.5), ("invsqrt", -0.5)])
def test_c1_vs_eigendecomposition(mode, p):
    cfg = workloads.CONFIGS["C1"]
    inp = workloads.make_inputs(cfg)
    op = KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2)
    b = inp["B"].astype(np.float64)
    r = ciq(op, b, q=8, max_iters=cfg.max_iters, tol=0.0, mode=mode, lanczos_start=inp["S"])
    exact = eig_power(op.dense(), b, p)
    assert relerr(r.out, exact) < 1e-4                  # P:899 "Q=8 ... < 1e-4"
    assert r.mvms == 10 + cfg.max_iters + (1 if mode == "sqrt" else 0)


@pytest.mark.parametrize("decay", ["inv_sqrt", "inv_square", "inv_linear", "exponential"])
def test_paper_spectra_q8(decay):
    n = 128 if decay != "exponential" else 24
    a = workloads.spectrum_matrix(n, decay, seed=5)
    b = workloads.rhs(n, 1).astype(np.float64)
    ev = np.linalg.eigvalsh(a)
    op = DenseOperator(a)
    r = ciq(op, b, q=8, max_iters=1500, tol=1e-11, mode="sqrt", spectrum=(ev[0], ev[-1]))
    err = relerr(r.out, eig_power(a, b, 0.5))
    kappa = ev[-1] / ev[0]
    assert err < max(1e-4, 10 * math.exp(-16 * math.pi ** 2 / (math.log(kappa) + 3))), (err, kappa)


def test_sqrt_of_sqrt_is_k():
    a = workloads.spectrum_matrix(32, "inv_linear", seed=9) + 0.05 * np.eye(32)
    op = DenseOperator(a)
    b = workloads.rhs(32, 1).astype(np.float64)
    ev = np.linalg.eigvalsh(a)
    s1 = ciq(op, b, q=12, max_iters=200, tol=1e-12, mode="sqrt", spectrum=(ev[0], ev[-1])).out
    s2 = ciq(op, s1, q=12, max_iters=200, tol=1e-12, mode="sqrt", spectrum=(ev[0], ev[-1])).out
    assert relerr(s2, a @ b) < 1e-6


def test_theorem1_and_corollary1_inequalities():
    x = workloads.points(150, 2, seed=21)
    op = KernelOperator(x, "matern52", 0.5, 1.0, sigma2=0.02)
    a = op.dense()
    ev = np.linalg.eigvalsh(a)
    lmin, lmax = ev[0], ev[-1]
    kappa = lmax / lmin
    b = workloads.rhs(150, 1).astype(np.float64)
    nb = np.linalg.norm(b)
    q = 6
    t, w = hht_rule(lmin, lmax, q)
    lam = np.geomspace(lmin, lmax, 2000)
    quad = np.max(np.abs(lam * np.sum(w[None, :] / (t[None, :] + lam[:, None]), axis=1) - np.sqrt(lam)))
    quad_inv = np.max(np.abs(np.sum(w[None, :] / (t[None, :] + lam[:, None]), axis=1) - 1 / np.sqrt(lam)))
    rho = (math.sqrt(kappa) - 1) / (math.sqrt(kappa) + 1)
    for j in (5, 20, 60):
        term = 2 * q * math.log(5 * math.sqrt(kappa)) * kappa * math.sqrt(lmin) / math.pi * rho ** (j - 1) * nb
        term_inv = 2 * q * math.log(5 * math.sqrt(kappa)) * kappa / (math.sqrt(lmin) * math.pi) * rho ** (j - 1) * nb
        aj = ciq(op, b, q=q, max_iters=j, tol=0.0, mode="sqrt", rule=(t, w)).out
        assert np.linalg.norm(aj - eig_power(a, b, 0.5)) <= quad * nb + 2 * term
        aj_inv = ciq(op, b, q=q, max_iters=j, tol=0.0, mode="invsqrt", rule=(t, w)).out
        assert np.linalg.norm(aj_inv - eig_power(a, b, -0.5)) <= quad_inv * nb + 2 * term_inv


def test_error_vs_q_decays_then_plateaus():
    a = workloads.spectrum_matrix(96, "inv_square", seed=2) + 1e-6 * np.eye(96)
    b = workloads.rhs(96, 1).astype(np.float64)
    ev = np.linalg.eigvalsh(a)
    exact = eig_power(a, b, 0.5)
    errs = []
    for q in (2, 4, 6, 8, 12):
        r = ciq(DenseOperator(a), b, q=q, max_iters=2000, tol=1e-9, mode="sqrt", spectrum=(ev[0], ev[-1]))
        errs.append(relerr(r.out, exact))
    assert errs[0] > errs[1] > errs[2] > errs[3]
    assert errs[-1] < 1e-6
