"""E5 direction (App. D): msMINRES iterations to a relative residual of 1e-4 on random
N = 7,500 RBF / Matern-5/2 kernels without and with rank-100 / rank-400 partial pivoted Cholesky
preconditioners (the paper: J = 100 unpreconditioned, cut 2x / 4x by rank 100 / 400).

"Random kernels" are not specified further: points U[0,1]^3, l = 0.2, outputscale 1, and the noise
sigma^2 calibrated (bisection on a log scale) so the unpreconditioned solve needs J ~ 100, as in
the paper; then the same operator with the library's GPU pivoted Cholesky (ciq_pivoted_cholesky)
and the preconditioned solve (fp64 route).  64 N(0,1) right-hand sides, Q = 8, whitening.
    python scripts/e5_sweep.py  (B200)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_11267_b200 as pb  # noqa: E402
import workloads  # noqa: E402

n, t, d = 7500, 64, 3
x = torch.from_numpy(workloads.points(n, d)).cuda()
b = torch.from_numpy(workloads.rhs(n, t)).cuda()
s0 = torch.from_numpy(workloads.lanczos_start(n)).cuda()
rows = []


def solve(kind, ls, s2, rank):
    kw = dict(lengthscale=ls, outputscale=1.0, diag=s2)
    lfac = None
    if rank > 0:
        with pb.CIQ(kind, X=x, **kw) as g0:
            lfac = torch.zeros((n, rank), device="cuda")
            g0.pivoted_cholesky(rank, lfac)
        kw.update(precond_L=lfac, precond_sigma2=s2)
    with pb.CIQ(kind, X=x, **kw) as g:
        out = torch.empty_like(b)
        t0 = time.time()
        info = g.apply(b, out, q=8, max_iters=2000, tol=1e-4, mode="whiten", lanczos_start=s0)
        torch.cuda.synchronize()
        return info, time.time() - t0


for kind in ("rbf", "matern52"):
    lo, hi = 1e-6, 1.0        # calibrate sigma^2: unpreconditioned J ~ 100
    for _ in range(14):
        mid = (lo * hi) ** 0.5
        info, _ = solve(kind, 0.2, mid, 0)
        if info["iters"] > 100:
            lo = mid
        else:
            hi = mid
    s2 = hi
    for rank in (0, 100, 400):
        info, sec = solve(kind, 0.2, s2, rank)
        r = {"kind": kind, "n": n, "l": 0.2, "sigma2": s2, "rank": rank, "J": info["iters"],
             "converged": info["converged"], "relres": info["max_rel_residual"], "seconds": round(sec, 3),
             "lambda": [info["lambda_min"], info["lambda_max"]]}
        rows.append(r)
        print(json.dumps(r), flush=True)
