"""Time one Thompson-sampling step (eq. thompson_sample) on workloads.THOMPSON
['T1'] (50k Hartmann-6 candidates, 100 evaluations, 64 samples): warm, CUDA events on the
default stream around ciq_thompson with device buffers.  Also the per-MVM cost of the posterior
downdate: the same fixed-J solve on the plain K** operator vs on COV* (same ctx geometry).
    python scripts/time_thompson.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_11267_b200 as pb  # noqa: E402
import workloads  # noqa: E402

cfg = workloads.THOMPSON["T1"]
inp = workloads.thompson_inputs(cfg)
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()  # noqa: E731
g = pb.CIQ(cfg.kind, X=dv(inp["Xs"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.jitter)
eps, s0 = dv(inp["eps"]), dv(inp["S"])
out = torch.empty_like(eps)


def timed(fn, reps=3):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        torch.cuda.synchronize()
        e0.record()
        r = fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), r


rule = (np.linspace(0.05, 5.0, cfg.q), np.full(cfg.q, 0.1))
jfix = 150
t_plain, _ = timed(lambda: g.apply(eps, out, q=cfg.q, max_iters=jfix, tol=0.0, mode="sqrt", rule=rule))
t_set, _ = timed(lambda: g.set_posterior(dv(inp["Xt"]), dv(inp["y"]), cfg.noise), reps=1)
t_post, _ = timed(lambda: g.apply(eps, out, q=cfg.q, max_iters=jfix, tol=0.0, mode="sqrt", rule=rule))
idx = torch.empty(cfg.t, dtype=torch.int64, device="cuda")
t_ts, info = timed(lambda: g.thompson(eps, idx, out, q=cfg.q, max_iters=cfg.max_iters, tol=cfg.tol,
                                      lanczos_start=s0, lanczos_reuse=True))
print(json.dumps({"workload": "T1: 50k Hartmann-6 candidates (RBF l=0.15), m=100 evaluations, 64 samples, Q=8, "
                  "tol 1e-4, jitter 0.05", "thompson_ms": t_ts, "samples_per_s": cfg.t / t_ts * 1e3,
                  "J": info["iters"], "mvms": info["mvms"], "converged": info["converged"],
                  "fixedJ150_plain_Kss_ms": t_plain, "fixedJ150_posterior_ms": t_post,
                  "downdate_us_per_mvm": (t_post - t_plain) / (jfix + 1) * 1e3, "set_posterior_ms": t_set}))
