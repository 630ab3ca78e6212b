"""GPU parity of the symmetric-tile matrix-free MVM (mvm_sym.cu) through
the C ABI: K V + sigma^2 V with each k(x_i, x_j), i < j, evaluated once and applied to rows i and j.

* element-wise against the float64 oracle (oracle.KernelOperator) at sizes spanning several 128-row
  blocks, several column groups (6 blocks) and row ranges (16 blocks), with ragged N and ragged T,
  for RBF / Matern-5/2 / Matern-3/2, 16- and 32-column chunks -- the same bounds as the full-tile
  kernel (tests/test_gpu_parity.py);
* against the full-tile kernel (mvm_impl "tc") on the same inputs, and run-to-run bitwise
  determinism (the partial products are summed in a fixed slot order);
* a full solve with mvm_impl "sym" against the oracle (same rule, fixed J); the AUTO choice (the
  symmetric-tile kernel for 16-column chunks where the full-tile kernel's accumulation chains are
  longer, e.g. C5; the full-tile kernel at small N);
* C5's full size (N = 200,000, 16 RHS): sampled rows against the oracle, and the result against the
  full-tile kernel.
"""
import numpy as np
import pytest
import torch

import workloads
from oracle import KernelOperator, ciq, estimate_spectrum, hht_rule

pytestmark = pytest.mark.gpu

import paper_2006_11267_b200 as pb  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def relerr(x, y):
    return float(np.linalg.norm(np.asarray(x, np.float64) - y) / np.linalg.norm(y))


def make(kind, n, t, d=None, ls=None):
    base = workloads.CONFIGS["C5" if kind != "rbf" else "C3"]
    cfg = workloads.scaled(base, n=n, t=t, kind=kind)
    if d is not None:
        cfg = workloads.scaled(cfg, d=d)
    if ls is not None:
        cfg = workloads.scaled(cfg, lengthscale=ls)
    return cfg, workloads.make_inputs(cfg)


def ctx(cfg, inp):
    return pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale,
                  diag=cfg.sigma2)


def mvm(cfg, inp, v, impl):
    with ctx(cfg, inp) as g:
        out = torch.empty(v.shape, device="cuda")
        g.matvec(dev(v), out, mvm_impl=impl)
        return out.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("kind", ["rbf", "matern52", "matern32"])
@pytest.mark.parametrize("n,t", [(1024, 16), (3001, 16), (5337, 5), (4200, 32), (2600, 48)])
def test_sym_mvm_matches_oracle(kind, n, t):
    cfg, inp = make(kind, n, t, ls=0.3 if kind != "rbf" else None)
    v = workloads.rhs(n, t, seed=11)
    ref = KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2).mvm(v.astype(np.float64))
    got = mvm(cfg, inp, v, "sym")
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 2e-5, err
    tol_col = 1.5e-5 if kind.startswith("matern") else 8e-6
    for c in range(t):
        assert relerr(got[:, c], ref[:, c]) < tol_col, c
    # same operator through the full-tile kernel: both approximate K V to ~1e-6
    full = mvm(cfg, inp, v, "tc")
    assert np.abs(got - full).max() / np.abs(full).max() < 2e-5


def test_sym_deterministic_and_auto_choice():
    cfg, inp = make("matern52", 6000, 16)
    v = workloads.rhs(cfg.n, 16, seed=3)
    a = mvm(cfg, inp, v, "sym")
    b = mvm(cfg, inp, v, "sym")
    assert np.array_equal(a, b)
    # AUTO: the full-tile kernel at this N (its column splits keep the accumulation chains short,
    # the more accurate choice), the symmetric-tile kernel at C5's N (16-column chunk, long chains)
    assert np.array_equal(mvm(cfg, inp, v, "auto"), mvm(cfg, inp, v, "tc"))
    cfg, inp = make("matern52", 60000, 16)
    v = workloads.rhs(cfg.n, 16, seed=3)
    assert np.array_equal(mvm(cfg, inp, v, "auto"), mvm(cfg, inp, v, "sym"))


def test_sym_unavailable_is_reported():
    cfg, inp = make("rbf", 4096, 64)   # 64-column chunk: not a symmetric-tile configuration
    v = workloads.rhs(cfg.n, 64, seed=1)
    with pytest.raises(RuntimeError, match="symmetric-tile"):
        mvm(cfg, inp, v, "sym")
    cfg, inp = make("rbf", 800, 16)    # N below the kernel's minimum
    with pytest.raises(RuntimeError, match="symmetric-tile"):
        mvm(cfg, inp, workloads.rhs(800, 16, seed=1), "sym")


@pytest.mark.parametrize("mode", ["sqrt", "invsqrt"])
def test_sym_solve_matches_oracle(mode):
    cfg = workloads.scaled(workloads.CONFIGS["C5"], n=4000, t=16)
    inp = workloads.config_inputs(cfg)
    op = KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2)
    lmin, lmax, _, _ = estimate_spectrum(op.mvm, inp["S"], 10, lower_bound=cfg.sigma2)
    t, w = hht_rule(lmin, lmax, cfg.q)
    j = 70
    ref = ciq(op, inp["B"].astype(np.float64), q=cfg.q, max_iters=j, tol=0.0, mode=mode, rule=(t, w))
    assert np.max(np.abs(ref.solve.phibar) / ref.solve.beta1) < 1e-5, "oracle not converged: raise j"
    with ctx(cfg, inp) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.apply(dev(inp["B"]), out, q=cfg.q, max_iters=j, tol=0.0, mode=mode, rule=(t, w), mvm_impl="sym")
        got = out.cpu().numpy()
    assert info["mvm_impl_used"] == "sym"
    assert relerr(got, ref.out) < 1e-4
    for c in range(cfg.t):
        assert relerr(got[:, c], ref.out[:, c]) < 3e-4


def test_sym_c5_full_size_sampled_rows_and_full_tile():
    cfg = workloads.CONFIGS["C5"]
    inp = workloads.make_inputs(cfg)
    v = workloads.rhs(cfg.n, cfg.t, seed=9)
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([np.arange(8), np.arange(cfg.n - 8, cfg.n), rng.choice(cfg.n, 40, replace=False)]))
    ref = KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2).mvm_rows(
        rows, v.astype(np.float64))
    got = mvm(cfg, inp, v, "sym")
    assert np.abs(got[rows] - ref).max() / np.abs(ref).max() < 2e-5
    full = mvm(cfg, inp, v, "tc")
    # the full-tile kernel carries up to 4e-5 of round-toward-zero accumulation bias at this N
    # (264-tile chains); the symmetric-tile chains are <= 16 tiles
    assert np.abs(got - full).max() / np.abs(full).max() < 6e-5
