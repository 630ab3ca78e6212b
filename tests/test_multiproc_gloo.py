"""N > 1 host logic on CPU with torch.distributed (gloo, world_size 2) -- no GPU needed.

* the row partition of ciq_shard_rows (C ABI, host-only) covers [0, N) disjointly with 128-aligned
  block starts on every rank;
* bench.broadcast_uid delivers rank 0's 128-byte NCCL id to every rank;
* the row-sharded msMINRES decomposition the CUDA path implements (local rows of K V, all-gathered
  Lanczos blocks, alpha / beta^2 as rank-order sums of per-rank partials) reproduces the single-
  process float64 oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_msminres(rank, world, kmat, b, shifts, iters):
    """Row-sharded msMINRES in float64: rank owns rows [b0, b1) of K, b and the solutions."""
    import paper_2006_11267_b200.ciq as cq
    n, t = b.shape
    b0, b1 = cq.ciq_shard_rows(n, rank, world)
    per = (n + world - 1) // world
    per = (per + 127) // 128 * 128

    def allgather_rows(local):
        pad = np.zeros((per, t))
        pad[: local.shape[0]] = local
        bufs = [torch.zeros((per, t), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(bufs, torch.from_numpy(pad))
        full = torch.cat(bufs).numpy()
        return full[:n]

    def rank_sum(vals):
        bufs = [torch.zeros_like(torch.from_numpy(vals)) for _ in range(world)]
        dist.all_gather(bufs, torch.from_numpy(vals))
        out = np.zeros_like(vals)
        for r in range(world):           # fixed rank order
            out = out + bufs[r].numpy()
        return out

    nq = len(shifts)
    beta1 = np.sqrt(rank_sum(np.sum(b[b0:b1] ** 2, axis=0)))
    v_full = b / beta1
    v_prev = np.zeros((b1 - b0, t))
    beta = np.zeros(t)
    c1 = np.ones((nq, t)); s1 = np.zeros((nq, t)); c2 = np.ones((nq, t)); s2 = np.zeros((nq, t))
    phibar = np.tile(beta1, (nq, 1))
    d1 = np.zeros((nq, b1 - b0, t)); d2 = np.zeros_like(d1); x = np.zeros_like(d1)
    for _ in range(iters):
        v = v_full[b0:b1]
        p = kmat[b0:b1] @ v_full                       # local rows of K V
        alpha = rank_sum(np.sum(v * p, axis=0))
        p = p - alpha * v - beta * v_prev
        bn = np.sqrt(rank_sum(np.sum(p * p, axis=0)))
        for q in range(nq):
            a = alpha + shifts[q]
            eps = s2[q] * beta; dp = c2[q] * beta
            delta = c1[q] * dp + s1[q] * a; gbar = -s1[q] * dp + c1[q] * a
            gam = np.hypot(gbar, bn); cs = gbar / gam; sn = bn / gam
            phi = cs * phibar[q]; phibar[q] = -sn * phibar[q]
            d = (v - delta * d1[q] - eps * d2[q]) / gam
            x[q] += phi * d
            d2[q] = d1[q]; d1[q] = d; c2[q] = c1[q]; s2[q] = s1[q]; c1[q] = cs; s1[q] = sn
        v_prev = v
        v_full = allgather_rows(p / bn)
        beta = bn
    return b0, b1, x


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench
        import paper_2006_11267_b200.ciq as cq
        import workloads
        from oracle import KernelOperator, hht_rule, msminres
        # 1. row partition
        spans = [cq.ciq_shard_rows(50_000, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 50_000 and all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        # 2. unique-id broadcast
        uid = bench.broadcast_uid(dist, rank, lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        # 3. sharded msMINRES == single-process oracle
        cfg = workloads.scaled(workloads.CONFIGS["C3"], n=700, t=3)
        inp = workloads.make_inputs(cfg)
        op = KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2)
        t, _ = hht_rule(cfg.sigma2, 30.0, 6)
        b = inp["B"].astype(np.float64)
        b0, b1, xs = _sharded_msminres(rank, world, op.dense(), b, t, 40)
        ref = msminres(op.mvm, b, t, 40, tol=0.0)
        err = np.max(np.abs(xs - ref.x[:, b0:b1])) / np.max(np.abs(ref.x))
        q.put((rank, float(err)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_host_logic():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err in res:
        assert err < 1e-10, (rank, err)
