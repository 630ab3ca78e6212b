"""GPU parity: the CUDA path (through the C ABI) vs the float64 oracle on the same seeded inputs.

Protocol: for the full solve both sides run a FIXED J (tol = 0)
chosen so that the oracle's max relative residual is <= 1e-6, with the SAME explicit quadrature
rule (from the oracle's lambda estimate) -- parity is well posed only for converged Krylov
iterates.  Bar: relative Frobenius error <= 1e-4 (north_star, fp32).  The GPU's own lambda
estimate and host rule are compared separately.  MVMs are compared element by element at sizes
spanning several tiles plus a ragged tail.
"""
import numpy as np
import pytest
import torch

import workloads
from oracle import DenseOperator, KernelOperator, ciq, estimate_spectrum, hht_rule

pytestmark = pytest.mark.gpu

try:
    import paper_2006_11267_b200 as pb
except ImportError as e:  # pragma: no cover - a GPU box without the library must fail loudly
    raise


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def relerr(x, y):
    return float(np.linalg.norm(np.asarray(x, np.float64) - y) / np.linalg.norm(y))


def oracle_op(cfg, inp):
    if cfg.kind == "dense":
        return DenseOperator(inp["K"], cfg.sigma2)
    return KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2)


def gpu_ctx(cfg, inp):
    if cfg.kind == "dense":
        return pb.CIQ("dense", K=dev(inp["K"]), diag=cfg.sigma2)
    return pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale,
                  diag=cfg.sigma2)


# ------------------------------------------------------------------------------------------------
# MVM (row a4)
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("kind", ["rbf", "matern52", "matern32", "dense"])
@pytest.mark.parametrize("n,t", [(1000, 1), (1000, 16), (777, 64), (2111, 70), (1500, 128), (900, 300)])
@pytest.mark.parametrize("impl", ["simt", "auto"])
def test_mvm_matches_oracle(kind, n, t, impl):
    cfg = workloads.scaled(workloads.CONFIGS["C2" if kind == "dense" else "C3"], n=n, t=t)
    if kind in ("matern52", "matern32"):
        cfg = workloads.scaled(cfg, kind=kind, lengthscale=0.3)
    inp = workloads.make_inputs(cfg)
    v = workloads.rhs(n, t, seed=9)
    ref = oracle_op(cfg, inp).mvm(v.astype(np.float64))
    with gpu_ctx(cfg, inp) as g:
        out = torch.empty((n, t), device="cuda")
        g.matvec(dev(v), out, mvm_impl=impl)
        got = out.cpu().numpy().astype(np.float64)
    # fp32 SIMT: a few ulps; tcgen05 split-fp16 ("fp16x3"): ~1e-6
    tol_max, tol_col = (5e-6, 3e-6) if impl == "simt" else (2e-5, 8e-6)
    if kind.startswith("matern") and impl != "simt":
        tol_col = 1.5e-5   # r = sqrt(r^2) amplifies the split-fp16 distance error near r = 0
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < tol_max, err
    for c in range(t):
        assert relerr(got[:, c], ref[:, c]) < tol_col


# ------------------------------------------------------------------------------------------------
# full solve (rows a1-a7)
# ------------------------------------------------------------------------------------------------

def run_pair(cfg, mode, j_fixed, impl="auto", oracle_iters=10):
    inp = workloads.config_inputs(cfg)
    op = oracle_op(cfg, inp)
    lmin, lmax, _, _ = estimate_spectrum(op.mvm, inp["S"], oracle_iters, lower_bound=cfg.sigma2)
    t, w = hht_rule(lmin, lmax, cfg.q)
    ref = ciq(op, inp["B"].astype(np.float64), q=cfg.q, max_iters=j_fixed, tol=0.0, mode=mode, rule=(t, w))
    with gpu_ctx(cfg, inp) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.apply(dev(inp["B"]), out, q=cfg.q, max_iters=j_fixed, tol=0.0, mode=mode, rule=(t, w),
                       mvm_impl=impl)
        got = out.cpu().numpy()
    return got, ref, info, inp, op


@pytest.mark.parametrize("mode", ["sqrt", "invsqrt"])
def test_c1_parity_and_eigh(mode):
    cfg = workloads.CONFIGS["C1"]
    got, ref, info, inp, op = run_pair(cfg, mode, cfg.max_iters)
    assert np.max(np.abs(ref.solve.phibar) / ref.solve.beta1) < 1e-5
    assert info["iters"] == cfg.max_iters and info["mvms"] == cfg.max_iters + (mode == "sqrt")
    assert relerr(got, ref.out) < 1e-4
    lam, v = np.linalg.eigh(op.dense())
    p = 0.5 if mode == "sqrt" else -0.5
    exact = v @ (lam[:, None] ** p * (v.T @ inp["B"].astype(np.float64)))
    assert relerr(got, exact) < 1e-4


@pytest.mark.parametrize("name,n,t,j,mode", [
    ("C3", 4096, 8, 75, "sqrt"),
    ("C2", 2048, 32, 160, "whiten"),
    ("C5", 3000, 16, 65, "sqrt"),
    ("C3", 1500, 21, 50, "invsqrt"),      # ragged T (21 -> padded 32), ragged N
])
def test_reduced_config_parity(name, n, t, j, mode):
    cfg = workloads.scaled(workloads.CONFIGS[name], n=n, t=t)
    got, ref, info, _, _ = run_pair(cfg, mode, j)
    assert np.max(np.abs(ref.solve.phibar) / ref.solve.beta1) < 1e-5, "oracle not converged: raise j"
    assert relerr(got, ref.out) < 1e-4
    for c in range(t):
        assert relerr(got[:, c], ref.out[:, c]) < 3e-4


def test_own_lambda_estimate_and_rule():
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=3000, t=4)
    inp = workloads.make_inputs(cfg)
    op = oracle_op(cfg, inp)
    lmin, lmax, rmin, rmax = estimate_spectrum(op.mvm, inp["S"], 10, lower_bound=cfg.sigma2)
    with gpu_ctx(cfg, inp) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.apply(dev(inp["B"]), out, q=8, max_iters=5, tol=0.0, mode="invsqrt", lanczos_start=dev(inp["S"]))
    # fp32 Lanczos vs fp64 Lanczos (both with full re-orthogonalisation): agree to ~1e-5
    assert abs(info["ritz_max"] / rmax - 1) < 5e-5
    assert abs(info["lambda_max"] / lmax - 1) < 5e-5
    assert info["lambda_min"] == pytest.approx(lmin, rel=1e-6)
    t, w = hht_rule(info["lambda_min"], info["lambda_max"], 8)
    np.testing.assert_allclose(info["t"], t, rtol=1e-12)
    np.testing.assert_allclose(info["w"], w, rtol=1e-12)


def test_end_to_end_own_estimate_vs_oracle():
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=2500, t=4)
    inp = workloads.make_inputs(cfg)
    op = oracle_op(cfg, inp)
    ref = ciq(op, inp["B"].astype(np.float64), q=8, max_iters=60, tol=0.0, mode="sqrt", lanczos_start=inp["S"])
    with gpu_ctx(cfg, inp) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.apply(dev(inp["B"]), out, q=8, max_iters=60, tol=0.0, mode="sqrt", lanczos_start=dev(inp["S"]))
    assert relerr(out.cpu().numpy(), ref.out) < 1e-4
    assert info["mvms"] == ref.mvms


def test_tolerance_stop_matches_oracle_iterations():
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=2000, t=4)
    inp = workloads.make_inputs(cfg)
    op = oracle_op(cfg, inp)
    lmin, lmax, _, _ = estimate_spectrum(op.mvm, inp["S"], 10, lower_bound=cfg.sigma2)
    t, w = hht_rule(lmin, lmax, 8)
    ref = ciq(op, inp["B"].astype(np.float64), q=8, max_iters=400, tol=1e-4, mode="sqrt", rule=(t, w))
    with gpu_ctx(cfg, inp) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.apply(dev(inp["B"]), out, q=8, max_iters=400, tol=1e-4, mode="sqrt", rule=(t, w))
    assert info["converged"] and info["max_rel_residual"] <= 1e-4
    assert abs(info["iters"] - ref.iters) <= 1


# ------------------------------------------------------------------------------------------------
# edge cases
# ------------------------------------------------------------------------------------------------

def test_scalar_operator_breakdown_and_zero_column():
    n = 300
    k = np.zeros((n, n), dtype=np.float32)
    b = workloads.rhs(n, 3)
    b[:, 1] = 0.0
    with pb.CIQ("dense", K=dev(k), diag=4.0) as g:
        out = torch.empty((n, 3), device="cuda")
        info = g.apply(dev(b), out, q=8, max_iters=50, tol=1e-6, mode="invsqrt", lanczos_start=dev(workloads.lanczos_start(n, 4)))
        got = out.cpu().numpy()
        assert info["iters"] == 1 and info["converged"]
        np.testing.assert_allclose(got, b / 2, rtol=2e-5, atol=1e-6)
        info = g.apply(dev(b), out, q=8, max_iters=50, tol=1e-6, mode="sqrt", lanczos_start=dev(workloads.lanczos_start(n, 4)))
        np.testing.assert_allclose(out.cpu().numpy(), 2 * b, rtol=2e-5, atol=1e-6)


def test_host_pointers_equal_device_pointers_and_deterministic():
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=1200, t=5)
    inp = workloads.make_inputs(cfg)
    with gpu_ctx(cfg, inp) as g:
        out_h = np.zeros((cfg.n, cfg.t), dtype=np.float32)
        i1 = g.apply(inp["B"], out_h, q=8, max_iters=60, tol=0.0, mode="sqrt", lanczos_start=inp["S"])
        out_d = torch.empty((cfg.n, cfg.t), device="cuda")
        g.apply(dev(inp["B"]), out_d, q=8, max_iters=60, tol=0.0, mode="sqrt", lanczos_start=dev(inp["S"]))
        out_d2 = torch.empty((cfg.n, cfg.t), device="cuda")
        g.apply(dev(inp["B"]), out_d2, q=8, max_iters=60, tol=0.0, mode="sqrt", lanczos_start=dev(inp["S"]))
    np.testing.assert_array_equal(out_h, out_d.cpu().numpy())
    np.testing.assert_array_equal(out_d.cpu().numpy(), out_d2.cpu().numpy())
    assert i1["kernel_launches"] > 0


def test_small_n_and_q1():
    cfg = workloads.scaled(workloads.CONFIGS["C1"], n=40, t=3)
    got, ref, info, _, _ = run_pair(workloads.scaled(cfg, q=1), "invsqrt", 40)
    assert relerr(got, ref.out) < 1e-4


def test_invalid_arguments_are_reported():
    cfg = workloads.scaled(workloads.CONFIGS["C1"], n=64, t=1)
    inp = workloads.make_inputs(cfg)
    with gpu_ctx(cfg, inp) as g:
        out = torch.empty((64, 1), device="cuda")
        with pytest.raises(pb.CiqError):
            g.apply(dev(inp["B"]), out, q=0)
        with pytest.raises(pb.CiqError):
            g.apply(dev(inp["B"]), out, q=8, tol=-1.0)
    with pytest.raises(pb.CiqError):
        pb.CIQ("rbf", X=dev(inp["X"]), lengthscale=-1.0)


def test_cuda_graph_replay_equals_direct_launches():
    """The solve loop replayed from a captured CUDA graph gives bit-identical results to the same
    launches issued directly (params.profile_kernels = 1 disables the graph)."""
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=1300, t=6)
    inp = workloads.make_inputs(cfg)
    outs = []
    for direct in (False, True, False):
        with gpu_ctx(cfg, inp) as g:
            out = torch.empty((cfg.n, cfg.t), device="cuda")
            info = g.apply(dev(inp["B"]), out, q=8, max_iters=400, tol=1e-5, mode="sqrt", lanczos_start=dev(inp["S"]),
                           profile=direct)
            outs.append((out.cpu().numpy(), info["iters"]))
    assert outs[0][1] == outs[1][1] == outs[2][1]
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][0], outs[2][0])


# ------------------------------------------------------------------------------------------------
# lanczos_reuse: lambda from the solve's own first 12 Lanczos steps (start = b, App. D),
# shifted updates of those steps replayed
# ------------------------------------------------------------------------------------------------

def test_lanczos_reuse_estimate_and_replay():
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=3000, t=8)
    inp = workloads.make_inputs(cfg)
    op = oracle_op(cfg, inp)
    b = inp["B"].astype(np.float64)
    lmin, lmax, rmin, rmax = estimate_spectrum(op.mvm, b, 12, lower_bound=cfg.sigma2)
    j = 90
    with gpu_ctx(cfg, inp) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.apply(dev(inp["B"]), out, q=8, max_iters=j, tol=0.0, mode="sqrt", lanczos_reuse=True)
        rule = (np.array(info["t"][:8]), np.array(info["w"][:8]))
        out2 = torch.empty_like(out)
        info2 = g.apply(dev(inp["B"]), out2, q=8, max_iters=j, tol=0.0, mode="sqrt", rule=rule)
    # no separate estimation run: J + the final K.Y
    assert info["mvms"] == j + 1 and info["iters"] == j
    # 12-step Ritz extremes of the 3-term fp32 recurrence vs the fp64 oracle with re-orthogonalisation
    assert abs(info["ritz_max"] / rmax - 1) < 1e-4
    assert abs(info["ritz_min"] / rmin - 1) < 1e-3
    np.testing.assert_allclose(info["lambda_min"], lmin, rtol=1e-3)
    # the replayed shifted updates equal a direct solve with the same rule
    got = out.cpu().numpy().astype(np.float64)
    assert relerr(got, out2.cpu().numpy()) < 1e-6
    ref = ciq(op, b, q=8, max_iters=j, tol=0.0, mode="sqrt", rule=rule)
    assert np.max(np.abs(ref.solve.phibar) / ref.solve.beta1) < 1e-5
    assert relerr(got, ref.out) < 1e-4


def test_lanczos_reuse_tolerance_stop():
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=2000, t=4)
    inp = workloads.make_inputs(cfg)
    with gpu_ctx(cfg, inp) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        a = g.apply(dev(inp["B"]), out, q=8, max_iters=400, tol=1e-4, mode="sqrt", lanczos_reuse=True)
        b = g.apply(dev(inp["B"]), out, q=8, max_iters=400, tol=1e-4, mode="sqrt", lanczos_start=dev(inp["S"]))
    assert a["converged"] and a["max_rel_residual"] <= 1e-4
    assert abs(a["iters"] - b["iters"]) <= 2
    assert a["mvms"] == a["iters"] + 1


# ------------------------------------------------------------------------------------------------
# materialised kernel operator (small N, T >= 256: the C4 regime) -> persistent dense kernel
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("kind", ["rbf", "matern52"])
def test_materialized_operator_mvm_and_solve(kind):
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=1500, t=256, kind=kind, lengthscale=0.3)
    inp = workloads.make_inputs(cfg)
    op = oracle_op(cfg, inp)
    v = workloads.rhs(cfg.n, cfg.t, seed=9)
    ref = op.mvm(v.astype(np.float64))
    with gpu_ctx(cfg, inp) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        g.matvec(dev(v), out)
        got = out.cpu().numpy().astype(np.float64)
        assert np.abs(got - ref).max() / np.abs(ref).max() < 2e-5
        for c in range(0, cfg.t, 37):
            assert relerr(got[:, c], ref[:, c]) < 8e-6
        # a full solve in this regime against the oracle (same rule, fixed J)
        lmin, lmax, _, _ = estimate_spectrum(op.mvm, inp["S"], 10, lower_bound=cfg.sigma2)
        rule = hht_rule(lmin, lmax, 8)
        b = inp["B"][:, :cfg.t]
        info = g.apply(dev(b), out, q=8, max_iters=200, tol=0.0, mode="invsqrt", rule=rule)
        got = out.cpu().numpy().astype(np.float64)
    cols = [0, 100, 255]
    refs = ciq(op, b[:, cols].astype(np.float64), q=8, max_iters=200, tol=0.0, mode="invsqrt", rule=rule)
    assert np.max(np.abs(refs.solve.phibar) / refs.solve.beta1) < 1e-5
    assert relerr(got[:, cols], refs.out) < 1e-4


# ------------------------------------------------------------------------------------------------
# backward pass: kept shifted solves and the dense VJP
# ------------------------------------------------------------------------------------------------

def test_keep_shift_solutions_match_oracle_and_reuse_replay():
    from oracle import msminres
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=900, t=3)
    inp = workloads.make_inputs(cfg)
    op = oracle_op(cfg, inp)
    lmin, lmax, _, _ = estimate_spectrum(op.mvm, inp["S"], 10, lower_bound=cfg.sigma2)
    rule = hht_rule(lmin, lmax, 8)
    j = 70
    ref = msminres(op.mvm, inp["B"].astype(np.float64), rule[0], j, 0.0)
    with gpu_ctx(cfg, inp) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        xs = torch.zeros((8, cfg.n, cfg.t), device="cuda")
        g.apply(dev(inp["B"]), out, q=8, max_iters=j, tol=0.0, mode="invsqrt", rule=rule, shift_solutions=xs)
        got = xs.cpu().numpy().astype(np.float64)
        # the lanczos_reuse warm-up + replay accumulates the same x_q
        xs2 = torch.zeros_like(xs)
        info = g.apply(dev(inp["B"]), out, q=8, max_iters=j, tol=0.0, mode="invsqrt", lanczos_reuse=True,
                       shift_solutions=xs2)
        r2 = (np.array(info["t"][:8]), np.array(info["w"][:8]))
        xs3 = torch.zeros_like(xs)
        g.apply(dev(inp["B"]), out, q=8, max_iters=j, tol=0.0, mode="invsqrt", rule=r2, shift_solutions=xs3)
    assert np.max(np.abs(ref.phibar) / ref.beta1) < 1e-5
    for q in range(8):
        assert relerr(got[q], ref.x[q]) < 1e-4
    assert relerr(xs2.cpu().numpy(), xs3.cpu().numpy()) < 1e-6
    # Y = sum_q w_q x_q (eq. contour_integral_quad)
    np.testing.assert_allclose(np.einsum("q,qnt->nt", rule[1], got), np.einsum("q,qnt->nt", rule[1], ref.x),
                               rtol=0, atol=1e-4 * np.abs(np.einsum("q,qnt->nt", rule[1], ref.x)).max())


def test_vjp_matches_oracle():
    from oracle import ciq_vjp
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=500, t=2)
    inp = workloads.make_inputs(cfg)
    op = oracle_op(cfg, inp)
    v = workloads.rhs(cfg.n, cfg.t, seed=7)
    j = 90
    with gpu_ctx(cfg, inp) as g:
        gmat = torch.empty((cfg.n, cfg.n), device="cuda")
        info = g.vjp(dev(inp["B"]), dev(v), gmat, q=8, max_iters=j, tol=0.0, lanczos_start=dev(inp["S"]))
        got = gmat.cpu().numpy().astype(np.float64)
        ghost = np.zeros((cfg.n, cfg.n), dtype=np.float32)
        g.vjp(inp["B"], v, ghost, q=8, max_iters=j, tol=0.0, lanczos_start=inp["S"])
    rule = (np.array(info["t"][:8]), np.array(info["w"][:8]))
    ref = ciq_vjp(op, inp["B"], v, rule, max_iters=j)
    assert info["mvms"] == 2 * j + 10
    assert relerr(got, ref) < 1e-4
    np.testing.assert_allclose(got, got.T, rtol=0, atol=1e-6 * np.abs(got).max())
    np.testing.assert_array_equal(ghost, gmat.cpu().numpy())


# ------------------------------------------------------------------------------------------------
# stored-basis variant: Y = W_J z from the kept Lanczos basis
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("name,n,t,mode,reuse", [("C3", 2111, 21, "sqrt", False), ("C3", 1500, 64, "invsqrt", True),
                                                 ("C2", 2048, 32, "whiten", False), ("C5", 3000, 16, "sqrt", True)])
def test_stored_basis_equals_streaming_and_oracle(name, n, t, mode, reuse):
    cfg = workloads.scaled(workloads.CONFIGS[name], n=n, t=t)
    inp = workloads.config_inputs(cfg)
    op = oracle_op(cfg, inp)
    lmin, lmax, _, _ = estimate_spectrum(op.mvm, inp["S"], 10, lower_bound=cfg.sigma2)
    rule = hht_rule(lmin, lmax, cfg.q)
    conv = ciq(op, inp["B"].astype(np.float64), q=cfg.q, max_iters=2000, tol=1e-8, mode=mode, rule=rule)
    outs = []
    with gpu_ctx(cfg, inp) as g:
        for stored in (False, True):
            out = torch.empty((cfg.n, cfg.t), device="cuda")
            kw = dict(lanczos_start=dev(inp["S"]), lanczos_reuse=True) if reuse else dict(rule=rule)
            info = g.apply(dev(inp["B"]), out, q=cfg.q, max_iters=400, tol=1e-6, mode=mode, stored_basis=stored, **kw)
            outs.append((out.cpu().numpy().astype(np.float64), info))
    (a, ia), (b, ib) = outs
    assert ia["converged"] and ib["converged"] and ia["iters"] == ib["iters"]
    assert relerr(b, a) < 2e-6             # same Krylov iterate, combined from the basis
    if not reuse:
        assert relerr(b, conv.out) < 1e-4


def test_relaxed_mvm_schedule_matches_accurate():
    """params.mvm_relax (relaxed inexact Krylov): once the max relative residual
    is <= 0.1 the full-tile kernel runs with 4x longer accumulation chains; the result stays within
    north_star's 1e-4 of the every-MVM-accurate solve (the C3 full-size golden tests check it against
    the oracle), the iteration count is unchanged and the switch happens part-way."""
    cfg = workloads.CONFIGS["C3"]   # N = 50k: 12 accurate vs 3 relaxed column splits
    inp = workloads.make_inputs(cfg)
    outs, infos = [], []
    with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale,
                diag=cfg.sigma2) as g:
        for relax in (False, True):
            out = torch.empty((cfg.n, cfg.t), device="cuda")
            infos.append(g.apply(dev(inp["B"]), out, q=8, max_iters=400, tol=1e-4, mode="sqrt",
                                 lanczos_start=dev(inp["S"]), mvm_relax=relax))
            outs.append(out.cpu().numpy().astype(np.float64))
    assert infos[0]["mvm_impl_used"] == "tc" and infos[0]["mvm_splits"] > 1
    assert all(i["converged"] for i in infos) and abs(infos[0]["iters"] - infos[1]["iters"]) <= 1
    assert infos[0]["relaxed_from"] == 0 and 1 < infos[1]["relaxed_from"] < infos[1]["iters"]
    assert relerr(outs[1], outs[0]) < 1e-4, relerr(outs[1], outs[0])
