"""Diagnostic: tcgen05 MVM error vs N (C3 shape), sampled rows."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads, paper_2006_11267_b200 as pb
from oracle import KernelOperator
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
for n in [int(x) for x in sys.argv[2:]] or [5000, 12500, 25000, 50000]:
    cfg = workloads.scaled(workloads.CONFIGS[name], n=n)
    inp = workloads.make_inputs(cfg)
    v = workloads.rhs(cfg.n, cfg.t, seed=9)
    rows = np.unique(np.random.default_rng(5).choice(cfg.n, 32, replace=False))
    op = KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2)
    ref = op.mvm_rows(rows, v.astype(np.float64))
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    g = pb.CIQ(cfg.kind, X=dv(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2)
    out = torch.empty((cfg.n, cfg.t), device="cuda")
    g.matvec(dv(v), out, mvm_impl="tc")
    got = out.cpu().numpy()[rows].astype(np.float64)
    e = got - ref
    rr = np.linalg.norm(e, axis=1) / np.linalg.norm(ref, axis=1)
    # signed row bias: projection of the error on the reference (systematic scale error per row)
    bias = np.sum(e * ref, axis=1) / np.sum(ref * ref, axis=1)
    print(f"{name} n={n} nsplit_env={os.environ.get('CIQ_TC_NSPLIT','auto')}: row-rel median {np.median(rr):.2e}  bias median {np.median(bias):+.2e} (min {bias.min():+.2e} max {bias.max():+.2e})", flush=True)
    g.close()
