"""Pins of the sparse-operator oracle and of the Gibbs stencil-precision input (SURVEY §8(f)
f4(iv); §5.3, App. F) -- CPU only.

* The input factors against scipy.ndimage.correlate(mode="reflect") (an independent stencil
  implementation): blur B and Laplacian L applied to random images; D^T D = I for the four
  sub-pixel offsets; the blur preserves constants, the Laplacian annihilates them.
* Lambda = gamma_obs A^T A + gamma_prior L^T L is symmetric positive definite (eigvalsh).
* SparseOperator.mvm against a dense matrix assembled from the CSR arrays with numpy.add.at.
* msMINRES-CIQ on the sparse operator against the eigendecomposition K^{+-1/2} b."""
import dataclasses

import numpy as np
import pytest
import scipy.ndimage

import workloads
from oracle import SparseOperator, ciq, estimate_spectrum


def small_cfg(side=16, low=8):
    return dataclasses.replace(workloads.GIBBS["G1"], side=side, low=low)


def test_stencil_factors_match_scipy_ndimage():
    cfg = small_cfg(24, 12)
    p = workloads.gibbs_precision(cfg)
    x = np.random.default_rng(0).standard_normal((cfg.side, cfg.side))
    for fac, w in ((p["B"], workloads.gibbs_blur_filter()), (p["L"], workloads.gibbs_laplace_filter())):
        ref = scipy.ndimage.correlate(x, w, mode="reflect").ravel()
        np.testing.assert_allclose(fac @ x.ravel(), ref, rtol=0, atol=1e-13)
    ones = np.ones(cfg.side * cfg.side)
    np.testing.assert_allclose(p["B"] @ ones, ones, atol=1e-14)
    np.testing.assert_allclose(p["L"] @ ones, 0.0, atol=1e-14)
    dtd = (p["D"].T @ p["D"]).toarray()
    np.testing.assert_array_equal(dtd, np.eye(cfg.side * cfg.side))


def test_precision_is_spd():
    p = workloads.gibbs_precision(small_cfg())
    a = np.zeros((p["n"], p["n"]))
    for i in range(p["n"]):
        for k in range(p["indptr"][i], p["indptr"][i + 1]):
            a[i, p["indices"][k]] += float(p["data"][k])
    np.testing.assert_allclose(a, a.T, atol=1e-6)
    assert np.linalg.eigvalsh(a.astype(np.float64))[0] > 0


def test_sparse_mvm_matches_dense_assembly():
    p = workloads.gibbs_precision(small_cfg())
    n = p["n"]
    a = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(p["indptr"]))
    np.add.at(a, (rows, p["indices"]), p["data"].astype(np.float64))
    op = SparseOperator(p["indptr"], p["indices"], p["data"], n, sigma2=0.01)
    v = np.random.default_rng(1).standard_normal((n, 3))
    np.testing.assert_allclose(op.mvm(v), a @ v + 0.01 * v, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("mode,power", [("invsqrt", -0.5), ("sqrt", 0.5)])
def test_ciq_on_stencil_precision_matches_eigh(mode, power):
    p = workloads.gibbs_precision(small_cfg())
    n = p["n"]
    op = SparseOperator(p["indptr"], p["indices"], p["data"], n)
    b = workloads.rhs(n, 2).astype(np.float64)
    res = ciq(op, b, q=12, max_iters=200, tol=1e-10, mode=mode, lanczos_start=workloads.lanczos_start(n, 4))
    lam, u = np.linalg.eigh(op.dense())
    exact = u @ (lam[:, None] ** power * (u.T @ b))
    assert np.linalg.norm(res.out - exact) / np.linalg.norm(exact) < 1e-6
