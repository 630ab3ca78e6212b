"""GPU robustness of the hot path (advisor findings, round 1):

* scale invariance of the fused split-fp16 packing: K^{±1/2}(s B) = s K^{±1/2} B for any s > 0, also
  when the first Lanczos block's packing scale must be guessed before beta_2 is known
  (recurrence.cu: alpha_1 stands in for ||W_2||) -- B scaled by 1e-4 and 1e4;
* a NaN / inf residual is never reported as converged (CIQ_NOT_CONVERGED, also at fixed J);
* the dense MVM keeps its fp32 TMEM accumulation chains bounded at large N (choose_nsplit_dense);
* ciq_pivoted_cholesky rejects row-sharded contexts (it needs every row of K).
"""
import math

import numpy as np
import pytest
import torch

import workloads
from oracle import DenseOperator, KernelOperator, ciq, estimate_spectrum, hht_rule

pytestmark = pytest.mark.gpu

import paper_2006_11267_b200 as pb  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def relerr(x, y):
    return float(np.linalg.norm(np.asarray(x, np.float64) - y) / np.linalg.norm(y))


@pytest.mark.parametrize("kind", ["rbf", "dense"])
@pytest.mark.parametrize("scale", [1e-4, 1.0, 1e4])
@pytest.mark.parametrize("reuse", [False, True])
def test_rhs_scale_invariance(kind, scale, reuse):
    name = "C2" if kind == "dense" else "C3"
    cfg = workloads.scaled(workloads.CONFIGS[name], n=2111, t=16)
    inp = workloads.make_inputs(cfg)
    op = DenseOperator(inp["K"], cfg.sigma2) if kind == "dense" else \
        KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2)
    lmin, lmax, _, _ = estimate_spectrum(op.mvm, inp["S"], 10, lower_bound=cfg.sigma2)
    rule = hht_rule(lmin, lmax, cfg.q)
    j = 110 if kind == "rbf" else 200
    b = inp["B"].astype(np.float64)
    ref = ciq(op, b, q=cfg.q, max_iters=j, tol=0.0, mode="sqrt", rule=rule)
    assert np.max(np.abs(ref.solve.phibar) / ref.solve.beta1) < 1e-5
    bs = (inp["B"] * np.float32(scale)).astype(np.float32)
    g = pb.CIQ("dense", K=dev(inp["K"]), diag=cfg.sigma2) if kind == "dense" else \
        pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2)
    with g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        if reuse:   # lanczos_reuse: the packing of W_2 happens in the (uncaptured) warm-up
            info = g.apply(dev(bs), out, q=cfg.q, max_iters=j, tol=0.0, mode="sqrt", lanczos_reuse=True)
            got = out.cpu().numpy().astype(np.float64) / scale
            # own lambda estimate: compare against the oracle's run with the GPU's rule
            ref2 = ciq(op, b, q=cfg.q, max_iters=j, tol=0.0, mode="sqrt", rule=(info["t"], info["w"]))
            assert np.all(np.isfinite(got))
            assert relerr(got, ref2.out) < 1e-4
        else:
            info = g.apply(dev(bs), out, q=cfg.q, max_iters=j, tol=0.0, mode="sqrt", rule=rule)
            got = out.cpu().numpy().astype(np.float64) / scale
            assert np.all(np.isfinite(got))
            assert relerr(got, ref.out) < 1e-4
    assert info["converged"]


@pytest.mark.parametrize("tol", [0.0, 1e-4])
def test_nonfinite_residual_is_not_converged(tol):
    cfg = workloads.scaled(workloads.CONFIGS["C2"], n=600, t=4)
    inp = workloads.make_inputs(cfg)
    k = inp["K"].copy()
    k[5, 7] = np.nan
    k[7, 5] = np.nan
    with pb.CIQ("dense", K=dev(k), diag=cfg.sigma2) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.apply(dev(inp["B"]), out, q=8, max_iters=60, tol=tol, mode="invsqrt", spectrum=(0.1, 100.0))
    assert info["status"] == pb.CIQ_NOT_CONVERGED
    assert not info["converged"]
    assert not math.isfinite(info["max_rel_residual"])
    assert info["iters"] < 60       # stops at the first non-finite step


def test_dense_large_n_accumulation_chain():
    """N = 20,000 dense (313 K tiles of 64 > the 264-tile chain bound): sampled rows of K V vs the
    oracle's dense rows, at the tensor-core bound of DESIGN.md section 5 (6e-5 max-abs relative)."""
    n, t = 20_000, 16
    x = workloads.points(n, 8)
    kin = workloads.dense_rbf_input(x, 0.5)
    v = workloads.rhs(n, t, seed=9)
    rows = np.concatenate([np.arange(8), np.arange(n - 8, n), np.random.default_rng(0).choice(n, 40, replace=False)])
    ref = DenseOperator(kin, 0.1).mvm_rows(rows, v.astype(np.float64))
    with pb.CIQ("dense", K=dev(kin), diag=0.1) as g:
        out = torch.empty((n, t), device="cuda")
        g.matvec(dev(v), out)
        got = out.cpu().numpy().astype(np.float64)[rows]
    scale = np.abs(kin[rows].astype(np.float64)) @ np.abs(v.astype(np.float64)) + 0.1 * np.abs(v[rows])
    assert np.max(np.abs(got - ref) / scale) < 6e-5


def test_pivoted_cholesky_rejects_row_sharding():
    cfg = workloads.scaled(workloads.CONFIGS["C4"], n=1000, t=1)
    inp = workloads.make_inputs(cfg)
    group = pb.LoopbackGroup(2)
    try:
        g = pb.CIQ(cfg.kind, n=cfg.n, X=dev(inp["X"]), lengthscale=cfg.lengthscale, diag=cfg.sigma2,
                   comm=(0, 2, group))
        lout = torch.zeros((500, 8), device="cuda")
        with pytest.raises(pb.CiqError) as e:
            g.pivoted_cholesky(8, lout)
        assert e.value.status == pb.CIQ_ERR_INVALID_ARG
        g.close()
    finally:
        group.close()
