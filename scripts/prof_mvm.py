"""Profiling driver: C3-sized tcgen05 MVM (ciq_matvec) a few times, for ncu captures.
    python scripts/prof_mvm.py [--config C3] [--reps 3] [--impl tc]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2006_11267_b200 as pb  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--impl", default="tc")
ap.add_argument("--t", type=int, default=0)
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
if a.t:
    cfg = workloads.scaled(cfg, t=a.t)
inp = workloads.make_inputs(cfg)
x = torch.from_numpy(inp["X"]).cuda()
v = torch.from_numpy(workloads.rhs(cfg.n, cfg.t, seed=9)).cuda()
out = torch.empty_like(v)
if cfg.kind == "dense":
    g = pb.CIQ("dense", K=torch.from_numpy(inp["K"]).cuda(), diag=cfg.sigma2)
else:
    g = pb.CIQ(cfg.kind, X=x, lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2)
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(a.reps):
    st.record()
    g.matvec(v, out, mvm_impl=a.impl)
    en.record()
    en.synchronize()
    print(f"matvec {a.impl} {cfg.name} T={cfg.t}: {st.elapsed_time(en):.3f} ms (incl. pack/copies)")
