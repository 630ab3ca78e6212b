"""Pins for the oracle's operator layer (L0): kernel entries and MVMs.

Pinned against scikit-learn's independent kernel implementations (RBF, Matern nu=2.5/1.5) and
against dense assembly; plus symmetry and positive semi-definiteness."""
import numpy as np
import pytest
from sklearn.gaussian_process.kernels import RBF, Matern

import workloads
from oracle import DenseOperator, KernelOperator, kernel_entries


@pytest.mark.parametrize("kind,skl", [
    ("rbf", lambda ls: RBF(length_scale=ls)),
    ("matern52", lambda ls: Matern(length_scale=ls, nu=2.5)),
    ("matern32", lambda ls: Matern(length_scale=ls, nu=1.5)),
])
@pytest.mark.parametrize("ard", [False, True])
def test_kernel_entries_match_sklearn(kind, skl, ard):
    x = workloads.points(40, 3, seed=11).astype(np.float64)
    y = workloads.points(30, 3, seed=12).astype(np.float64)
    ls = np.array([0.3, 0.5, 0.2]) if ard else 0.35
    mine = kernel_entries(x, y, kind, ls, 2.5)
    ref = 2.5 * skl(ls)(x, y)
    np.testing.assert_allclose(mine, ref, rtol=1e-12, atol=1e-14)


def test_kernel_diag_is_outputscale_and_symmetric_psd():
    x = workloads.points(64, 4, seed=3)
    for kind in ("rbf", "matern52", "matern32"):
        op = KernelOperator(x, kind, 0.4, 1.7, sigma2=0.0)
        k = op.dense()
        np.testing.assert_allclose(np.diag(k), 1.7, rtol=0, atol=1e-15)
        np.testing.assert_array_equal(k, k.T)
        assert np.linalg.eigvalsh(k).min() > -1e-10


@pytest.mark.parametrize("kind", ["rbf", "matern52", "matern32"])
def test_matrix_free_mvm_equals_dense_assembly(kind):
    x = workloads.points(300, 5, seed=5)
    v = workloads.rhs(300, 3, seed=6).astype(np.float64)
    skl = {"rbf": RBF(0.3), "matern52": Matern(0.3, nu=2.5), "matern32": Matern(0.3, nu=1.5)}[kind]
    kd = skl(x.astype(np.float64)) + 0.05 * np.eye(300)
    op = KernelOperator(x, kind, 0.3, 1.0, sigma2=0.05, dense_cache_max=0, block=64)  # map-reduce path
    np.testing.assert_allclose(op.mvm(v), kd @ v, rtol=1e-12, atol=1e-12)
    assert op.mvm_count == 1
    rows = np.array([0, 17, 299])
    np.testing.assert_allclose(op.mvm_rows(rows, v), (kd @ v)[rows], rtol=1e-12, atol=1e-12)


def test_dense_operator_trivial_examples():
    # S:57 DenseOperator [[2,0],[0,5]], v=(1,1) -> (2,5); S:66 shifted t=3 -> (5,8)
    op = DenseOperator(np.array([[2.0, 0.0], [0.0, 5.0]]))
    np.testing.assert_array_equal(op.mvm(np.array([1.0, 1.0])), [2.0, 5.0])
    op3 = DenseOperator(np.array([[2.0, 0.0], [0.0, 5.0]]), sigma2=3.0)
    np.testing.assert_array_equal(op3.mvm(np.array([1.0, 1.0])), [5.0, 8.0])
