"""Symmetric-tile vs full-tile MVM error against the oracle on a C4-shaped operator (d = 3,
Matern-5/2, l = 0.3) and C5-shaped, for random and structured V:
    python scripts/diag_sym.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_11267_b200 as pb  # noqa: E402
import workloads  # noqa: E402
from oracle import KernelOperator  # noqa: E402


def run(cfg, v, label):
    inp = workloads.make_inputs(cfg)
    ref = KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2).mvm(v.astype(np.float64))
    with pb.CIQ(cfg.kind, X=torch.from_numpy(inp["X"]).cuda(), lengthscale=cfg.lengthscale,
                outputscale=cfg.outputscale, diag=cfg.sigma2) as g:
        for impl in ("sym", "tc", "simt"):
            out = torch.empty(v.shape, device="cuda")
            g.matvec(torch.from_numpy(np.ascontiguousarray(v, np.float32)).cuda(), out, mvm_impl=impl)
            got = out.cpu().numpy().astype(np.float64)
            e = np.abs(got - ref)
            col = np.linalg.norm(got - ref, axis=0) / np.linalg.norm(ref, axis=0)
            i = np.unravel_index(np.argmax(e), e.shape)
            print(f"{label:28s} {impl:5s} maxabs/max {e.max() / np.abs(ref).max():.2e}  col max {col.max():.2e}  "
                  f"worst row {i[0]} col {i[1]}")


for n in (1500, 3000):
    cfg = workloads.scaled(workloads.CONFIGS["C4"], n=n, t=16, sigma2=0.1)
    run(cfg, workloads.rhs(n, 16, seed=3), f"C4-like n={n} rand")
    inp = workloads.make_inputs(cfg)
    v = np.cos(7 * inp["X"][:, :1] + np.arange(16)[None, :]).astype(np.float32)
    run(cfg, v, f"C4-like n={n} smooth")
cfg = workloads.scaled(workloads.CONFIGS["C5"], n=3000, t=16)
run(cfg, workloads.rhs(3000, 16, seed=3), "C5-like n=3000 rand")
