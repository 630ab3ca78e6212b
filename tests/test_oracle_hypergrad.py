"""Pins of the oracle's hyper-parameter gradient (ciq_hyper_grad; eq. ciq_deriv P:1211-1215 chained
with dK/dtheta) -- CPU only.

* The lengthscale derivative of each kernel form against central finite differences of
  ``kernel_entries`` (the textbook forms, reading G11) -- pins kernel_lengthscale_derivative.
* The full gradient against central finite differences, in l, o^2 and sigma^2, of the quadrature
  approximation F(theta) = sum_c v_c^T sum_q w_q (t_q I + K(theta))^{-1} b_c computed with dense
  solves (numpy.linalg.solve) at a FIXED rule (t, w) -- the quantity eq. ciq_deriv differentiates.
* The noise derivative against its closed form -sum_q w_q v^T (t_q I + K)^{-2} b (eigh)."""
import numpy as np
import pytest

from oracle import KernelOperator, ciq_hyper_grad, hht_rule, kernel_entries, kernel_lengthscale_derivative


@pytest.mark.parametrize("kind", ["rbf", "matern52", "matern32"])
def test_lengthscale_derivative_matches_finite_differences(kind):
    rng = np.random.default_rng(3)
    x = rng.uniform(size=(30, 4))
    y = rng.uniform(size=(25, 4))
    ls, h = 0.37, 1e-6
    fd = (kernel_entries(x, y, kind, ls + h, 1.3) - kernel_entries(x, y, kind, ls - h, 1.3)) / (2 * h)
    np.testing.assert_allclose(kernel_lengthscale_derivative(x, y, kind, ls, 1.3), fd, rtol=1e-6, atol=1e-9)


def _f(x, kind, ls, o2, s2, rule, b, v):
    k = kernel_entries(x, x, kind, ls, o2) + s2 * np.eye(x.shape[0])
    n = k.shape[0]
    return sum(w * np.sum(v * np.linalg.solve(k + t * np.eye(n), b)) for t, w in zip(*rule))


@pytest.mark.parametrize("kind", ["rbf", "matern52"])
def test_hyper_grad_equals_finite_differences_of_the_quadrature(kind):
    rng = np.random.default_rng(4)
    n, t = 50, 2
    x = rng.uniform(size=(n, 3))
    ls, o2, s2 = 0.3, 1.2, 0.05
    op = KernelOperator(x, kind, ls, o2, s2)
    lam = np.linalg.eigvalsh(op.dense())
    rule = hht_rule(lam[0], lam[-1], 12)
    b = rng.standard_normal((n, t))
    v = rng.standard_normal((n, t))
    g = ciq_hyper_grad(op, b, v, rule, max_iters=n)      # J = N: exact shifted solves
    h = 1e-6
    fd = np.array([
        (_f(x, kind, ls + h, o2, s2, rule, b, v) - _f(x, kind, ls - h, o2, s2, rule, b, v)) / (2 * h),
        (_f(x, kind, ls, o2 + h, s2, rule, b, v) - _f(x, kind, ls, o2 - h, s2, rule, b, v)) / (2 * h),
        (_f(x, kind, ls, o2, s2 + h, rule, b, v) - _f(x, kind, ls, o2, s2 - h, rule, b, v)) / (2 * h),
    ])
    np.testing.assert_allclose(g, fd, rtol=2e-6, atol=1e-6 * np.abs(fd).max())


def test_noise_derivative_closed_form():
    rng = np.random.default_rng(5)
    n = 40
    x = rng.uniform(size=(n, 2))
    op = KernelOperator(x, "rbf", 0.4, 1.0, 0.1)
    lam, u = np.linalg.eigh(op.dense())
    rule = hht_rule(lam[0], lam[-1], 10)
    b = rng.standard_normal((n, 3))
    v = rng.standard_normal((n, 3))
    g = ciq_hyper_grad(op, b, v, rule, max_iters=n)
    # d/dsigma2 of sum_q w_q v^T (t_q + K)^{-1} b = -sum_q w_q v^T (t_q + K)^{-2} b
    exact = -sum(w * np.sum((u.T @ v) * ((u.T @ b) / (lam[:, None] + t) ** 2)) for t, w in zip(*rule))
    assert abs(g[2] - exact) <= 1e-8 * abs(exact)
