"""GPU parity of nested CIQ with a block-Jacobi preconditioner (App. A).

The library never forms P^{+-1/2}: it computes c = P^{1/2} b by CIQ on P (only MVMs with P) and
runs the P^{-1}-only preconditioned msMINRES on the pencil (K, P) (only solves with P), all in
fp64.  The oracle (oracle.precond_ciq with oracle.BlockJacobi) takes the explicit symmetric route
with exact block powers from eigh -- an independent computation of the same R' b = P^{-1/2}
(P^{-1/2} K P^{-1/2})^{-1/2} b.  Bar: north_star's 1e-4."""
import numpy as np
import pytest
import torch

import workloads
from oracle import BlockJacobi, KernelOperator, hht_rule, precond_ciq

pytestmark = pytest.mark.gpu

import paper_2006_11267_b200 as pb  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def relerr(x, y):
    return float(np.linalg.norm(np.asarray(x, np.float64) - y) / np.linalg.norm(y))


def f32(v):
    return float(np.float32(v))


def setup(n=1500, t=16, block=128, sigma2=1e-3):
    cfg = workloads.scaled(workloads.CONFIGS["C4"], n=n, t=t)
    cfg = workloads.scaled(cfg, lengthscale=f32(cfg.lengthscale), outputscale=f32(cfg.outputscale), sigma2=f32(sigma2))
    inp = workloads.config_inputs(cfg)
    op = KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2)
    pre = BlockJacobi(op, block)
    return cfg, inp, op, pre


def m_spectrum(op, pre):
    ph = pre.power(np.eye(op.n), -0.5)
    m = ph @ op.dense() @ ph
    lam = np.linalg.eigvalsh(0.5 * (m + m.T))
    return lam[0], lam[-1]


@pytest.mark.parametrize("mode", ["whiten", "sqrt"])
def test_nested_matches_oracle_same_rule(mode):
    cfg, inp, op, pre = setup()
    lmin, lmax = m_spectrum(op, pre)
    rule = hht_rule(lmin, lmax, cfg.q)
    b = inp["B"].astype(np.float64)
    conv = precond_ciq(op, pre, b, q=cfg.q, max_iters=3000, tol=1e-8, mode=mode, rule=rule)
    with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale,
                diag=cfg.sigma2, precond_block=128) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.apply(dev(inp["B"]), out, q=cfg.q, max_iters=conv.iters + 20, tol=1e-8, mode=mode, rule=rule)
    assert info["rotated"] and info["fp64_route"] and info["nested_p_mvms"] > 0
    assert relerr(out.cpu().numpy(), conv.out) < 1e-4, relerr(out.cpu().numpy(), conv.out)


def test_nested_own_estimate():
    cfg, inp, op, pre = setup(n=1200, t=8, block=300, sigma2=1e-2)
    lmin, lmax = m_spectrum(op, pre)
    ref = precond_ciq(op, pre, inp["B"].astype(np.float64), q=cfg.q, max_iters=3000, tol=1e-8, mode="whiten",
                      rule=hht_rule(lmin, lmax, cfg.q))
    with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale,
                diag=cfg.sigma2, precond_block=300) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.apply(dev(inp["B"]), out, q=cfg.q, max_iters=2000, tol=1e-6, mode="whiten",
                       lanczos_start=dev(inp["S"]))
    assert info["converged"] and info["nested_iters"] > 0
    # own rule: Ritz extremes of the P-Lanczos process with lambda_min >= sigma^2 / lambda_max(P)
    assert relerr(out.cpu().numpy(), ref.out) < 1e-4, relerr(out.cpu().numpy(), ref.out)


def test_nested_gram_identities():
    n = 64
    cfg = workloads.scaled(workloads.CONFIGS["C4"], n=n, t=n)
    inp = workloads.make_inputs(cfg)
    op = KernelOperator(inp["X"], cfg.kind, f32(0.4), 1.0, f32(1e-2))
    k = op.dense()
    eye = np.eye(n, dtype=np.float32)
    with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=0.4, outputscale=1.0, diag=1e-2, precond_block=24) as g:
        rp = torch.empty((n, n), device="cuda")
        g.apply(dev(eye), rp, q=16, max_iters=200, tol=1e-10, mode="whiten")
        r = torch.empty((n, n), device="cuda")
        g.apply(dev(eye), r, q=16, max_iters=200, tol=1e-10, mode="sqrt")
    rp = rp.cpu().numpy().astype(np.float64)
    r = r.cpu().numpy().astype(np.float64)
    kinv = np.linalg.inv(k)
    assert np.linalg.norm(rp @ rp.T - kinv) / np.linalg.norm(kinv) < 1e-5   # R' R'^T = K^{-1}
    assert np.linalg.norm(r @ r.T - k) / np.linalg.norm(k) < 1e-5            # R R^T = K
