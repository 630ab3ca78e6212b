"""Preconditioner-rank sweep (the direction of E3/E5: P:914-915, P:939-944 --
rank-200/400 pivoted-Cholesky preconditioners cut the msMINRES iterations on ill-conditioned kernels).
For each problem and rank r: pivoted Cholesky on the GPU (ciq_pivoted_cholesky), P = L L^T + sigma2 I,
one whitening solve R'B (tol fixed), warm, CUDA events.  Rank 0 = unpreconditioned K^{-1/2}B.
    python scripts/precond_sweep.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_11267_b200 as pb  # noqa: E402
import workloads  # noqa: E402

dv = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()  # noqa: E731

PROBLEMS = [
    # C4's operator (Matern-5/2, M = 5000, sigma2 = 1e-3) and RHS block, tolerance tightened to 1e-4
    dict(name="C4-op tol1e-4", cfg=workloads.CONFIGS["C4"], tol=1e-4, ranks=[0, 50, 100, 200, 400]),
    # an ill-conditioned matrix-free problem at C3's size: RBF d=3, l=0.2, sigma2=1e-3, 64 RHS
    dict(name="N50k RBF d3 l0.2 s2 1e-3", cfg=workloads.Config("P2", 50_000, 3, "rbf", 0.2, 1.0, 1e-3, 64, 8,
                                                                 "whiten", 1500, 1e-4),
         tol=1e-4, ranks=[0, 100, 200, 400]),
    # the paper's own case: the Hartmann-6 GP posterior covariance at 50k
    # candidates (workloads.THOMPSON T1 with a small jitter 1e-4), sampled with R B (sqrt mode)
    dict(name="Hartmann-6 posterior N50k jitter 1e-4 (T1)", posterior=True,
         cfg=workloads.Config("T1p", 50_000, 6, "rbf", 0.15, 1.0, 1e-4, 64, 8, "sqrt", 1500, 1e-4),
         tol=1e-4, ranks=[0, 200, 400]),
    dict(name="Hartmann-6 posterior N50k l=0.5 jitter 1e-4", posterior=True,
         cfg=workloads.Config("T1l", 50_000, 6, "rbf", 0.5, 1.0, 1e-4, 64, 8, "sqrt", 1500, 1e-4),
         tol=1e-4, ranks=[0, 200, 400]),
]


def run(prob):
    cfg = prob["cfg"]
    post = prob.get("posterior", False)
    if post:
        ti = workloads.thompson_inputs(workloads.THOMPSON["T1"])
        inp = {"X": ti["Xs"], "B": ti["eps"], "S": ti["S"]}
        tnoise = workloads.THOMPSON["T1"].noise
    else:
        inp = workloads.config_inputs(cfg)
    x = dv(inp["X"])
    b = dv(inp["B"])
    s0 = dv(inp["S"])

    def make(**extra):
        gg = pb.CIQ(cfg.kind, X=x, **kw, **extra)
        if post:
            gg.set_posterior(dv(ti["Xt"]), dv(ti["y"]), tnoise)
        return gg

    out = torch.empty_like(b)
    kw = dict(lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2)
    rows = []
    for r in prob["ranks"]:
        g0 = make()
        if r == 0:
            g = g0
        else:
            lf = torch.empty((cfg.n, r), device="cuda")
            e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
            e0.record()
            g0.pivoted_cholesky(r, lf)
            e1.record()
            e1.synchronize()
            t_chol = e0.elapsed_time(e1)
            g0.close()
            g = make(precond_L=lf, precond_sigma2=cfg.sigma2)
        call = lambda: g.apply(b, out, q=cfg.q, max_iters=cfg.max_iters, tol=prob["tol"], mode=cfg.mode,  # noqa: E731
                               lanczos_start=s0)
        for _ in range(2):
            call()
        e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        torch.cuda.synchronize()
        e0.record()
        info = call()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        rows.append({"rank": r, "J": info["iters"], "converged": info["converged"],
                     "max_rel_residual": info["max_rel_residual"], "lambda": [info["lambda_min"], info["lambda_max"]],
                     "apply_ms": ms, "rhs_per_s": cfg.t / ms * 1e3, "pivchol_ms": None if r == 0 else t_chol})
        g.close()
    return {"problem": prob["name"], "n": cfg.n, "t": cfg.t, "results": rows}


only = sys.argv[1:]   # optional problem indices
for i, p in enumerate(PROBLEMS):
    if not only or str(i) in only:
        print(json.dumps(run(p)), flush=True)
