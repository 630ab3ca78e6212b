"""Diagnostic: full-size MVM error statistics on sampled rows, tcgen05 vs fp32 SIMT path."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads, paper_2006_11267_b200 as pb
from oracle import KernelOperator, DenseOperator
for name in sys.argv[1:] or ["C3"]:
    cfg = workloads.CONFIGS[name]
    inp = workloads.make_inputs(cfg)
    v = workloads.rhs(cfg.n, cfg.t, seed=9)
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([np.arange(8), np.arange(cfg.n - 8, cfg.n), rng.choice(cfg.n, 40, replace=False)]))
    op = DenseOperator(inp["K"].astype(np.float64), cfg.sigma2) if cfg.kind == "dense" else KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2)
    ref = op.mvm_rows(rows, v.astype(np.float64))
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    g = pb.CIQ("dense", K=dv(inp["K"]), diag=cfg.sigma2) if cfg.kind == "dense" else pb.CIQ(cfg.kind, X=dv(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2)
    for impl in ("tc", "simt"):
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        g.matvec(dv(v), out, mvm_impl=impl)
        got = out.cpu().numpy()[rows].astype(np.float64)
        e = got - ref
        print(f"{name} {impl}: max-abs rel {np.abs(e).max()/np.abs(ref).max():.2e}  row-rel median {np.median(np.linalg.norm(e,axis=1)/np.linalg.norm(ref,axis=1)):.2e} max {np.max(np.linalg.norm(e,axis=1)/np.linalg.norm(ref,axis=1)):.2e}  overall relL2 {np.linalg.norm(e)/np.linalg.norm(ref):.2e}", flush=True)
