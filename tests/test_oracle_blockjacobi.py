"""Pins of the block-Jacobi preconditioner oracle (BlockJacobi; App. A's requirements P:69-74: a P
with cheap solves and MVMs whose square root the library obtains by CIQ on P) -- CPU only.

* P is the block diagonal of K: dense() against slices of the operator's dense matrix; power(v, 1)
  = dense() v; power(v, -1) against numpy.linalg.solve; power(power(v, 1/2), 1/2) = P v.
* App. A's Gram identities for this P: R'R'^T = K^{-1} and R R^T = K with the
  symmetric route (precond_ciq) applied to identity columns."""
import numpy as np

import workloads
from oracle import BlockJacobi, KernelOperator, hht_rule, precond_ciq


def _op(n=96):
    return KernelOperator(workloads.points(n, 3), "matern52", 0.3, 1.0, sigma2=0.01)


def test_block_structure_and_powers():
    op = _op()
    pre = BlockJacobi(op, 40)           # ragged last block (96 = 40 + 40 + 16)
    k = op.dense()
    d = pre.dense()
    mask = np.zeros_like(k, dtype=bool)
    for i0 in range(0, 96, 40):
        mask[i0:i0 + 40, i0:i0 + 40] = True
    np.testing.assert_allclose(d[mask], k[mask], atol=1e-13)
    assert np.all(d[~mask] == 0)
    v = np.random.default_rng(0).standard_normal((96, 3))
    np.testing.assert_allclose(pre.power(v, 1.0), d @ v, atol=1e-12)
    np.testing.assert_allclose(pre.power(v, -1.0), np.linalg.solve(d, v), rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(pre.power(pre.power(v, 0.5), 0.5), d @ v, atol=1e-11)


def test_gram_identities_with_block_jacobi():
    op = _op(64)
    pre = BlockJacobi(op, 24)
    k = op.dense()
    pd = pre.dense()
    ph = np.linalg.cholesky(pd)           # any square root of P gives the same M spectrum
    m = np.linalg.solve(ph, np.linalg.solve(ph, k).T).T
    lam = np.linalg.eigvalsh(0.5 * (m + m.T))
    rule = hht_rule(lam[0], lam[-1], 20)
    eye = np.eye(64)
    rp = precond_ciq(op, pre, eye, q=20, max_iters=64, tol=0.0, mode="whiten", rule=rule).out
    r = precond_ciq(op, pre, eye, q=20, max_iters=64, tol=0.0, mode="sqrt", rule=rule).out
    kinv = np.linalg.inv(k)
    assert np.linalg.norm(rp @ rp.T - kinv) / np.linalg.norm(kinv) < 1e-6
    assert np.linalg.norm(r @ r.T - k) / np.linalg.norm(k) < 1e-6
