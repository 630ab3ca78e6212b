"""Pins of the oracle's Thompson-sampling step (eq. thompson_sample):
PosteriorOperator against the block-inverse (Schur complement) identity and the GP interpolation
limits, thompson_step against a sample drawn through an eigendecomposition square root."""
import numpy as np
import pytest
import scipy.linalg

import workloads
from oracle import PosteriorOperator, kernel_entries, thompson_step

KW = dict(kind="rbf", lengthscale=0.3, outputscale=1.0)


def _problem(n=120, m=15, noise=1e-3, jitter=1e-2, seed=0):
    rng = np.random.default_rng(seed)
    xs = rng.random((n, 3))
    xt = rng.random((m, 3))
    y = np.sin(6 * xt[:, 0]) + xt[:, 1]
    return xs, xt, y, PosteriorOperator(xs, xt, y, noise=noise, jitter=jitter, **KW)


def test_cov_is_schur_complement_of_joint_matrix():
    # (J^{-1})_{22} = S^{-1}, S = D - C A^{-1} B: an independent route to COV* + jitter I
    xs, xt, y, post = _problem()
    m = xt.shape[0]
    x = np.vstack([xt, xs])
    j = kernel_entries(x, x, **KW)
    j[:m, :m] += post.noise * np.eye(m)
    j[m:, m:] += post.sigma2 * np.eye(xs.shape[0])
    s = np.linalg.inv(np.linalg.inv(j)[m:, m:])
    assert np.abs(post.dense() - s).max() < 1e-8


def test_mean_is_conditional_expectation_of_joint_gaussian():
    # mu* = K*x (Kxx + noise I)^{-1} y, checked via the joint precision: mu* = -P22^{-1} P21 y
    xs, xt, y, post = _problem()
    m = xt.shape[0]
    x = np.vstack([xt, xs])
    j = kernel_entries(x, x, **KW) + 1e-12 * np.eye(len(x))
    j[:m, :m] += post.noise * np.eye(m)
    prec = np.linalg.inv(j)
    mu = -np.linalg.solve(prec[m:, m:], prec[m:, :m] @ y)
    assert np.abs(post.mean - mu).max() < 1e-6


def test_noise_free_interpolation_limits():
    # candidates = the training points, noise -> 0: mu* -> y and the posterior variance -> jitter
    rng = np.random.default_rng(3)
    xt = rng.random((10, 3))
    y = rng.standard_normal(10)
    post = PosteriorOperator(xt, xt, y, noise=1e-10, jitter=1e-6, **KW)
    assert np.abs(post.mean - y).max() < 1e-5
    assert np.abs(np.diag(post.dense()) - 1e-6).max() < 1e-7


def test_far_training_data_leaves_the_prior():
    xs, _, _, _ = _problem()
    xt = np.full((4, 3), 50.0)
    post = PosteriorOperator(xs, xt, np.ones(4), noise=1e-3, jitter=1e-2, **KW)
    assert np.abs(post.mean).max() < 1e-12
    assert np.abs(post.dense() - post.kss.dense()).max() < 1e-12


def test_mvm_rows_and_mvm_agree_with_dense():
    _, _, _, post = _problem()
    v = np.random.default_rng(1).standard_normal((post.n, 3))
    d = post.dense()
    assert np.abs(post.mvm(v) - d @ v).max() < 1e-10
    rows = np.array([0, 7, post.n - 1])
    assert np.abs(post.mvm_rows(rows, v) - (d @ v)[rows]).max() < 1e-10
    assert np.linalg.eigvalsh(d).min() >= post.sigma2 * (1 - 1e-8)   # COV* is PSD


def test_thompson_step_matches_eigh_sample():
    _, _, _, post = _problem(n=200)
    eps = np.random.default_rng(2).standard_normal((post.n, 6))
    idx, samples, r = thompson_step(post, eps, q=12, max_iters=400, tol=1e-10,
                                    lanczos_start=np.random.default_rng(4).standard_normal((post.n, 4)))
    lam, u = np.linalg.eigh(post.dense())
    ref = post.mean[:, None] + (u * np.sqrt(lam)) @ (u.T @ eps)
    assert np.abs(samples - ref).max() < 1e-4 * np.abs(ref).max()
    for c in range(eps.shape[1]):
        order = np.sort(ref[:, c])
        if order[1] - order[0] > 1e-3:   # a unique minimiser at this tolerance
            assert idx[c] == np.argmin(ref[:, c])


def test_thompson_step_zero_noise_is_argmin_of_mean_and_permutation_invariant():
    xs, xt, y, post = _problem(n=80)
    idx, _, _ = thompson_step(post, np.zeros((post.n, 2)), q=8, max_iters=50, tol=0.0, rule=(np.ones(8), np.ones(8)))
    assert (idx == np.argmin(post.mean)).all()
    perm = np.random.default_rng(5).permutation(post.n)
    eps = np.random.default_rng(6).standard_normal((post.n, 3))
    p2 = PosteriorOperator(xs[perm], xt, y, noise=post.noise, jitter=post.sigma2, **KW)
    rule = (np.linspace(0.1, 2.0, 8), np.full(8, 0.1))
    i1, _, _ = thompson_step(post, eps, q=8, max_iters=300, tol=1e-10, rule=rule)
    i2, _, _ = thompson_step(p2, eps[perm], q=8, max_iters=300, tol=1e-10, rule=rule)
    assert (perm[i2] == i1).all()


def test_hartmann6_known_minimum():
    # published global minimiser of Hartmann-6 and its value -3.32237
    xmin = np.array([[0.20169, 0.150011, 0.476874, 0.275332, 0.311652, 0.6573]])
    assert abs(workloads.hartmann6(xmin)[0] + 3.32237) < 1e-4
    x = np.random.default_rng(0).random((1000, 6))
    assert workloads.hartmann6(x).min() > -3.32237


def test_posterior_kernel_column_diag_and_full_rank_pivoted_cholesky():
    from oracle import pivoted_cholesky
    _, _, _, post = _problem(n=60, m=8)
    k = post.dense() - post.sigma2 * np.eye(post.n)      # COV* without the jitter
    assert np.abs(post.kernel_column(7) - k[:, 7]).max() < 1e-12
    assert np.abs(post.kernel_diag() - np.diag(k)).max() < 1e-12
    lf = pivoted_cholesky(post, post.n)
    resid = k - lf @ lf.T
    assert np.linalg.eigvalsh(resid).min() > -1e-9       # the Schur complement stays PSD
    assert np.trace(resid) < 1e-6 * np.trace(k)
