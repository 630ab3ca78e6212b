"""GPU parity of the Thompson-sampling step (eq. thompson_sample):
the posterior covariance operator COV* + jitter I (ciq_set_posterior) and ciq_thompson against the
oracle's PosteriorOperator / thompson_step on the same seeded Hartmann-6 inputs (workloads.THOMPSON).

* MVM: element by element, relative to max |K** v| (the downdate cancels part of K** v).
* Samples: same explicit rule and fixed J on both sides (parity protocol of test_gpu_parity.py),
  relative Frobenius error <= 1e-4; argmin: several indices can be correct within the sample
  error, so the GPU's index must attain the oracle's minimum within that error.
* Full size (T1: 50k candidates, 100 evaluations, 64 samples, the bench workload): returned
  samples' argmin equals idx exactly, and the final COV* MVM agrees with the oracle on sampled rows."""
import dataclasses

import numpy as np
import pytest
import torch

import workloads
from oracle import PosteriorOperator, estimate_spectrum, hht_rule, thompson_step

pytestmark = pytest.mark.gpu

import paper_2006_11267_b200 as pb  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def relerr(x, y):
    return float(np.linalg.norm(np.asarray(x, np.float64) - y) / np.linalg.norm(y))


def small_cfg(n=700, m=30, t=5):
    return dataclasses.replace(workloads.THOMPSON["T1"], n=n, m=m, t=t)


def setup(cfg):
    inp = workloads.thompson_inputs(cfg)
    post = PosteriorOperator(inp["Xs"], inp["Xt"], inp["y"], cfg.kind, cfg.lengthscale, cfg.outputscale,
                             cfg.noise, cfg.jitter)
    g = pb.CIQ(cfg.kind, X=dev(inp["Xs"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale,
               diag=cfg.jitter)
    g.set_posterior(dev(inp["Xt"]), dev(inp["y"]), cfg.noise)
    return inp, post, g


@pytest.mark.parametrize("n,t", [(700, 5), (1333, 64), (300, 1)])
def test_posterior_mvm_matches_oracle(n, t):
    cfg = small_cfg(n=n, t=t)
    inp, post, g = setup(cfg)
    v = workloads.rhs(cfg.n, cfg.t, seed=9)
    with g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        g.matvec(dev(v), out)
        got = out.cpu().numpy().astype(np.float64)
    ref = post.mvm(v.astype(np.float64))
    scale = np.abs(post.kss.mvm(v.astype(np.float64))).max()
    assert np.abs(got - ref).max() / scale < 3e-5


def test_posterior_host_inputs_and_replacement():
    cfg = small_cfg()
    inp, post, g = setup(cfg)
    v = workloads.rhs(cfg.n, 3, seed=9)
    with g:
        a = np.zeros((cfg.n, 3), dtype=np.float32)
        g.set_posterior(inp["Xt"], inp["y"], cfg.noise)      # host copies, same data
        g.matvec(v, a)
        np.testing.assert_allclose(a, post.mvm(v.astype(np.float64)), rtol=0, atol=3e-5)
        xt2 = inp["Xt"][:7].copy()
        g.set_posterior(xt2, None, 0.01)                       # replaced data, zero targets
        post2 = PosteriorOperator(inp["Xs"], xt2, np.zeros(7), cfg.kind, cfg.lengthscale, cfg.outputscale, 0.01,
                                  cfg.jitter)
        g.matvec(v, a)
        np.testing.assert_allclose(a, post2.mvm(v.astype(np.float64)), rtol=0, atol=3e-5)


def test_thompson_samples_and_argmin_match_oracle():
    cfg = small_cfg()
    inp, post, g = setup(cfg)
    lmin, lmax, _, _ = estimate_spectrum(post.mvm, inp["S"], 10, lower_bound=cfg.jitter)
    rule = hht_rule(lmin, lmax, cfg.q)
    j = 150
    idx_ref, s_ref, r = thompson_step(post, inp["eps"], q=cfg.q, max_iters=j, tol=0.0, rule=rule)
    assert (np.abs(r.solve.phibar) / r.solve.beta1).max() <= 1e-6
    with g:
        idx = torch.empty(cfg.t, dtype=torch.int64, device="cuda")
        samples = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.thompson(dev(inp["eps"]), idx, samples, q=cfg.q, max_iters=j, tol=0.0, rule=rule)
        idx_h = np.zeros(cfg.t, dtype=np.int64)
        g.thompson(inp["eps"], idx_h, None, q=cfg.q, max_iters=j, tol=0.0, rule=rule)   # host buffers
    got = samples.cpu().numpy().astype(np.float64)
    assert info["iters"] == j and info["mvms"] == j + 1
    assert relerr(got, s_ref) < 1e-4
    idx = idx.cpu().numpy()
    np.testing.assert_array_equal(idx, idx_h)
    err = np.abs(got - s_ref).max()
    for c in range(cfg.t):
        assert s_ref[idx[c], c] <= s_ref[:, c].min() + 2 * err, c
        assert idx[c] == int(np.argmin(got[:, c]))    # lowest index among equal fp32 minima


def test_thompson_errors():
    cfg = small_cfg(n=300, t=2)
    inp = workloads.thompson_inputs(cfg)
    with pb.CIQ(cfg.kind, X=dev(inp["Xs"]), lengthscale=cfg.lengthscale, diag=cfg.jitter) as g:
        with pytest.raises(pb.CiqError):
            g.thompson(dev(inp["eps"]), torch.empty(2, dtype=torch.int64, device="cuda"))
        with pytest.raises(pb.CiqError):
            g.set_posterior(dev(inp["Xt"]), dev(inp["y"]), 0.0)     # noise must be > 0
    k = np.eye(300, dtype=np.float32)
    with pb.CIQ("dense", K=dev(k), diag=0.1) as g:
        with pytest.raises(pb.CiqError):
            g.set_posterior(dev(inp["Xt"]), dev(inp["y"]), 0.01)


def test_thompson_full_size_t1():
    cfg = workloads.THOMPSON["T1"]
    inp, post, g = setup(cfg)
    with g:
        idx = torch.empty(cfg.t, dtype=torch.int64, device="cuda")
        samples = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.thompson(dev(inp["eps"]), idx, samples, q=cfg.q, max_iters=cfg.max_iters, tol=cfg.tol,
                          lanczos_start=dev(inp["S"]))
        assert info["converged"] and info["max_rel_residual"] <= cfg.tol
        s = samples.cpu().numpy()
        np.testing.assert_array_equal(idx.cpu().numpy(), np.argmin(s, axis=0))
        # final MVM of the sqrt path against the oracle's COV* on sampled rows: samples - mu* = COV* Y
        rule = (np.array(info["t"][:cfg.q]), np.array(info["w"][:cfg.q]))
        y = torch.empty_like(samples)
        g.apply(dev(inp["eps"]), y, q=cfg.q, max_iters=info["iters"], tol=0.0, mode="invsqrt", rule=rule)
        y_h = y.cpu().numpy().astype(np.float64)
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([np.arange(4), np.arange(cfg.n - 4, cfg.n), rng.choice(cfg.n, 40, replace=False)]))
    ref = post.mvm_rows(rows, y_h) + post.mean[rows, None]
    ref_abs = post.kss.mvm_rows(rows, np.abs(y_h)) + np.abs(post.kxs[:, rows].T) @ np.abs(
        np.linalg.solve(post.kxx, post.kxs @ y_h))
    assert (np.abs(s[rows].astype(np.float64) - ref) / (ref_abs + np.abs(post.mean[rows, None]))).max() < 6e-5


def test_posterior_pivoted_cholesky_and_preconditioned_solve():
    """ciq_pivoted_cholesky on a posterior ctx factors COV* (the Hartmann-posterior preconditioning
    of P:914-915); the preconditioned whitening R'B on COV* + jitter I matches the oracle's
    precond_ciq with the same rule and J."""
    from oracle import LowRankPlusDiag, pivoted_cholesky, precond_ciq
    cfg = dataclasses.replace(small_cfg(n=900, m=25, t=4), jitter=1e-3)
    inp, post, g = setup(cfg)
    r = 40
    ref_l = pivoted_cholesky(post, r)
    with g:
        lf = torch.empty((cfg.n, r), device="cuda")
        g.pivoted_cholesky(r, lf)
        got_l = lf.cpu().numpy().astype(np.float64)
    assert np.abs(got_l - ref_l).max() < 2e-6
    pre = LowRankPlusDiag(ref_l, cfg.jitter)

    class _M:
        def mvm(self, v):
            return pre.power(post.mvm(pre.power(v, -0.5)), -0.5)

    lmin, lmax, _, _ = estimate_spectrum(_M().mvm, inp["S"], 10, lower_bound=1.0)
    rule = hht_rule(lmin, lmax, cfg.q)
    b = inp["eps"].astype(np.float64)
    conv = precond_ciq(post, pre, b, q=cfg.q, max_iters=2000, tol=1e-6, mode="whiten", rule=rule)
    j = conv.iters + 10
    ref = precond_ciq(post, pre, b, q=cfg.q, max_iters=j, tol=0.0, mode="whiten", rule=rule)
    gp = pb.CIQ(cfg.kind, X=dev(inp["Xs"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale,
                diag=cfg.jitter, precond_L=dev(ref_l), precond_sigma2=cfg.jitter)   # L is an input: the same P
    with gp:
        gp.set_posterior(dev(inp["Xt"]), dev(inp["y"]), cfg.noise)
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info = gp.apply(dev(inp["eps"]), out, q=cfg.q, max_iters=j, tol=0.0, mode="whiten", rule=rule)
    assert info["rotated"] and info["fp64_route"]   # M of COV* + jitter I formed in fp64 (precond64.cu)
    assert relerr(out.cpu().numpy(), ref.out) < 1e-4
