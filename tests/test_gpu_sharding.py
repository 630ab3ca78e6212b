"""Row sharding on ONE GPU through the in-process loopback transport: `world`
ranks run as threads, each with its own ctx on its row block; per iteration they all-gather the
next Lanczos block and the alpha / beta^2 partial sums (rank-order sums).  The concatenated
result must equal the single-GPU result up to reduction order (<= 1e-5), and the
same code path runs over NCCL across GPUs (the transport is the only difference)."""
import threading

import numpy as np
import pytest
import torch

import workloads
from oracle import KernelOperator, ciq

pytestmark = pytest.mark.gpu

import paper_2006_11267_b200 as pb  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def run_sharded(cfg, inp, world, lfac=None, **kw):
    group = pb.LoopbackGroup(world)
    outs, infos, errs = [None] * world, [None] * world, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            b0, b1 = pb.ciq_shard_rows(cfg.n, r, world)
            extra = {} if lfac is None else dict(precond_L=dev(lfac[b0:b1]), precond_sigma2=cfg.sigma2,
                                                   precond_matrix_free=True)
            g = pb.CIQ(cfg.kind, n=cfg.n, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale,
                       diag=cfg.sigma2, comm=(r, world, group), **extra)
            out = torch.empty((b1 - b0, cfg.t), device="cuda")
            s_rows = inp["S"][b0:b1]
            infos[r] = g.apply(dev(inp["B"][b0:b1]), out, lanczos_start=dev(s_rows), **kw)
            outs[r] = out.cpu().numpy()
            g.close()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=300)
    group.close()
    assert not errs, errs
    return np.concatenate(outs, axis=0), infos


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("impl", ["tc", "simt"])
def test_sharded_equals_single_gpu(world, impl):
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=1500, t=8)
    inp = workloads.make_inputs(cfg)
    kw = dict(q=8, max_iters=60, tol=0.0, mode="sqrt", mvm_impl=impl)
    with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale,
                diag=cfg.sigma2) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info1 = g.apply(dev(inp["B"]), out, lanczos_start=dev(inp["S"]), **kw)
        single = out.cpu().numpy()
    sharded, infos = run_sharded(cfg, inp, world, **kw)
    rel = np.linalg.norm(sharded - single) / np.linalg.norm(single)
    assert rel < 1e-5, rel
    # scalar recurrence state is identical on every rank
    for inf in infos[1:]:
        assert inf["lambda_max"] == infos[0]["lambda_max"] and inf["iters"] == infos[0]["iters"]
    assert abs(infos[0]["lambda_max"] / info1["lambda_max"] - 1) < 1e-6
    # the tensor-core path all-gathers the Lanczos block next to the local diagonal block's MVM
    assert all(inf["overlap"] == (impl == "tc") for inf in infos), [inf["overlap"] for inf in infos]


def test_sharded_tolerance_stop_and_oracle():
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=1300, t=4)
    inp = workloads.make_inputs(cfg)
    sharded, infos = run_sharded(cfg, inp, 2, q=8, max_iters=300, tol=1e-5, mode="invsqrt")
    op = KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2)
    ref = ciq(op, inp["B"].astype(np.float64), q=8, max_iters=300, tol=1e-5, mode="invsqrt", lanczos_start=inp["S"])
    assert abs(infos[0]["iters"] - ref.iters) <= 1
    assert np.linalg.norm(sharded - ref.out) / np.linalg.norm(ref.out) < 1e-4


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_lanczos_reuse_equals_single_gpu(world):
    """lambda from the solve's own Lanczos (lanczos_reuse) under row sharding: the warm-up steps use
    the same all-gather / rank-order sums, the replay runs on the local rows."""
    cfg = workloads.scaled(workloads.CONFIGS["C3"], n=1500, t=8)
    inp = workloads.make_inputs(cfg)
    kw = dict(q=8, max_iters=60, tol=0.0, mode="sqrt", lanczos_reuse=True)
    with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale,
                diag=cfg.sigma2) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info1 = g.apply(dev(inp["B"]), out, **kw)
        single = out.cpu().numpy()
    sharded, infos = run_sharded(cfg, inp, world, **kw)
    assert np.linalg.norm(sharded - single) / np.linalg.norm(single) < 1e-5
    assert info1["mvms"] == 61 and all(i["mvms"] == 61 for i in infos)
    for inf in infos[1:]:
        assert inf["lambda_max"] == infos[0]["lambda_max"] and inf["iters"] == infos[0]["iters"]
    assert abs(infos[0]["lambda_max"] / info1["lambda_max"] - 1) < 1e-6


@pytest.mark.parametrize("dense", [False, True])
def test_nccl_one_rank_sharded_path(dense):
    """The NCCL transport itself (nccl_dl: dlopen of libnccl, ncclCommInitRank, ncclAllGather
    captured in the solve's CUDA graph) on the one GPU a test box has: a world-1 communicator runs
    the row-sharded code path (allgathered Lanczos blocks, rank-order sums of the alpha / beta^2
    partials) and must reproduce the single-GPU result up to reduction order."""
    cfg = workloads.scaled(workloads.CONFIGS["C2" if dense else "C3"], n=1500, t=8)
    inp = workloads.make_inputs(cfg)
    # converged solves (unconverged Krylov iterates amplify rounding differences -- the
    # sharded path packs the MVM operand with its own scale -- far above the reduction-order level)
    kw = dict(q=8, max_iters=400, tol=1e-6, mode="sqrt")
    mk = (lambda **c: pb.CIQ("dense", K=dev(inp["K"]), diag=cfg.sigma2, **c)) if dense else \
        (lambda **c: pb.CIQ(cfg.kind, n=cfg.n, X=dev(inp["X"]), lengthscale=cfg.lengthscale,
                            outputscale=cfg.outputscale, diag=cfg.sigma2, **c))
    outs = []
    for comm in (None, (0, 1, pb.ciq_nccl_unique_id())):
        with (mk() if comm is None else mk(comm=comm)) as g:
            out = torch.empty((cfg.n, cfg.t), device="cuda")
            info = g.apply(dev(inp["B"]), out, lanczos_start=dev(inp["S"]), **kw)
            outs.append((out.cpu().numpy().astype(np.float64), info))
    (a, ia), (b, ib) = outs
    assert ia["converged"] and ib["converged"] and abs(ia["iters"] - ib["iters"]) <= 2
    assert np.linalg.norm(a - b) / np.linalg.norm(a) < 1e-5
    # matrix-free: the captured iteration graph forks the local block's MVM onto a side stream next
    # to the NCCL all-gather (world 1: the local block is every column tile)
    assert ib["overlap"] == (not dense) and not ia["overlap"]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["whiten", "sqrt"])
def test_sharded_preconditioned_equals_single_gpu(world, mode):
    """Row sharding of the preconditioned variant (matrix-free route): each rank
    holds its rows of L; U = L W S^{-1} from the rank-summed L^T L, and every P^{-1/2} application
    sums U^T W over the ranks.  Same result as one GPU up to reduction order."""
    from oracle import pivoted_cholesky
    cfg = workloads.scaled(workloads.CONFIGS["C4"], n=1400, t=8)
    cfg = workloads.scaled(cfg, sigma2=0.05)
    inp = workloads.config_inputs(cfg)
    lfac = pivoted_cholesky(KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2), 48)
    kw = dict(q=8, max_iters=400, tol=1e-6, mode=mode, lanczos_start=None)
    kw.pop("lanczos_start")
    with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale,
                diag=cfg.sigma2, precond_L=dev(lfac), precond_sigma2=cfg.sigma2, precond_matrix_free=True) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info1 = g.apply(dev(inp["B"]), out, lanczos_start=dev(inp["S"]), **kw)
        ref = out.cpu().numpy().astype(np.float64)
    got, infos = run_sharded(cfg, inp, world, lfac=lfac, **kw)
    assert info1["rotated"] and all(i["rotated"] for i in infos)
    assert abs(infos[0]["iters"] - info1["iters"]) <= 2
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-5
