"""Pins of the oracle's backward pass (eq. ciq_deriv) -- CPU only.

* The formula is the exact gradient of the quadrature approximation F(K) = sum_c v_c^T sum_q w_q
  (t_q I + K)^{-1} b_c: central finite differences of F (dense shifted solves, numpy.linalg.solve)
  along a random symmetric direction E equal sum_ij G_ij E_ij.
* Against the exact Frechet derivative of K^{-1/2} (Daleckii-Krein formula from numpy eigh):
  sum_c v_c^T D[K^{-1/2}](E) b_c within the quadrature error of the rule.
* G is symmetric, and linear in v."""
import numpy as np

from oracle import DenseOperator, KernelOperator, ciq_vjp, hht_rule


def _setup(n=60, t=2, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.uniform(size=(n, 3))
    op = KernelOperator(x, "rbf", 0.3, 1.0, 0.05)
    k = op.dense()
    lam = np.linalg.eigvalsh(k)
    rule = hht_rule(lam[0], lam[-1], 12)
    b = rng.standard_normal((n, t))
    v = rng.standard_normal((n, t))
    e = rng.standard_normal((n, n))
    return op, k, lam, rule, b, v, 0.5 * (e + e.T)


def _f(k, rule, b, v):
    t_q, w_q = rule
    n = k.shape[0]
    return sum(w * np.sum(v * np.linalg.solve(k + t * np.eye(n), b)) for t, w in zip(t_q, w_q))


def test_vjp_equals_finite_differences_of_the_quadrature():
    op, k, lam, rule, b, v, e = _setup()
    g = ciq_vjp(op, b, v, rule, max_iters=op.n)         # J = N: exact shifted solves
    h = 1e-6   # central differences: O(h^2) curvature error ~1e-8 relative here, rounding ~1e-8
    fd = (_f(k + h * e, rule, b, v) - _f(k - h * e, rule, b, v)) / (2 * h)
    assert abs(np.sum(g * e) - fd) <= 1e-7 * max(1.0, abs(fd))


def test_vjp_matches_exact_frechet_derivative_of_inverse_sqrt():
    op, k, lam, rule, b, v, e = _setup(seed=1)
    g = ciq_vjp(op, b, v, rule, max_iters=op.n)
    lam, u = np.linalg.eigh(k)
    r = lam ** -0.5
    dl = np.subtract.outer(lam, lam)
    dr = np.subtract.outer(r, r)
    with np.errstate(divide="ignore", invalid="ignore"):
        l_mat = np.where(np.abs(dl) > 1e-14 * lam[-1], dr / np.where(dl == 0, 1, dl), -0.5 * lam[:, None] ** -1.5)
    de = u @ ((u.T @ e @ u) * l_mat) @ u.T                  # D[K^{-1/2}](E)
    exact = np.sum(v * (de @ b))
    assert abs(np.sum(g * e) - exact) <= 1e-5 * np.abs(np.sum(np.abs(v) * (np.abs(de) @ np.abs(b))))


def test_vjp_symmetric_and_linear_in_v():
    op, k, lam, rule, b, v, e = _setup(seed=2)
    g1 = ciq_vjp(op, b, v, rule, max_iters=op.n)
    g2 = ciq_vjp(op, b, 2.0 * v, rule, max_iters=op.n)
    np.testing.assert_allclose(g1, g1.T, atol=1e-12)
    np.testing.assert_allclose(g2, 2.0 * g1, rtol=1e-9, atol=1e-12)


def test_vjp_scalar_operator_closed_form():
    # K = c I: x_q(u) = u / (c + t_q), G = -sum_q w_q (v b^T + b v^T) / (2 (c + t_q)^2)
    n, c = 20, 4.0
    op = DenseOperator(np.zeros((n, n)), c)
    rule = hht_rule(c, c * 1.5, 8)
    rng = np.random.default_rng(3)
    b, v = rng.standard_normal(n), rng.standard_normal(n)
    g = ciq_vjp(op, b, v, rule, max_iters=3)
    s = np.sum(rule[1] / (c + rule[0]) ** 2)
    np.testing.assert_allclose(g, -0.5 * s * (np.outer(v, b) + np.outer(b, v)), rtol=1e-12, atol=1e-14)
