"""Diagnostic: preconditioned CIQ parity vs the oracle as a function of sigma2 and MVM precision."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads
from oracle import KernelOperator, LowRankPlusDiag, estimate_spectrum, hht_rule, pivoted_cholesky, precond_ciq, ciq
import paper_2006_11267_b200 as pb
def dev(a): return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
for sigma2 in (1e-3, 1e-2, 3e-2):
    cfg = workloads.scaled(workloads.CONFIGS["C4"], n=1500, t=16, sigma2=sigma2)
    inp = workloads.config_inputs(cfg)
    op = KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2)
    ev = np.linalg.eigvalsh(op.dense())
    lfac = pivoted_cholesky(op, 64); pre = LowRankPlusDiag(lfac, sigma2)
    r = precond_ciq(op, pre, inp["B"].astype(np.float64), q=8, max_iters=3000, tol=1e-7, mode="whiten", lanczos_start=inp["S"])
    J = r.iters
    for impl in ("tc", "simt"):
        with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=1.0, diag=sigma2,
                    precond_L=dev(lfac), precond_sigma2=sigma2) as g:
            out = torch.empty((cfg.n, cfg.t), device="cuda")
            g.apply(dev(inp["B"]), out, q=8, max_iters=J, tol=0.0, mode="whiten", rule=(r.t, r.w), mvm_impl=impl)
        e = np.linalg.norm(out.cpu().numpy() - r.out) / np.linalg.norm(r.out)
        print(f"sigma2={sigma2:g} kappa(K)={ev[-1]/ev[0]:.2e} J={J} impl={impl} precond relerr={e:.2e}")
    # unpreconditioned at the same sigma2 for comparison
    r0 = ciq(op, inp["B"].astype(np.float64), q=8, max_iters=6000, tol=1e-7, mode="invsqrt", lanczos_start=inp["S"])
    for impl in ("tc", "simt"):
        with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=1.0, diag=sigma2) as g:
            out = torch.empty((cfg.n, cfg.t), device="cuda")
            g.apply(dev(inp["B"]), out, q=8, max_iters=r0.iters, tol=0.0, mode="invsqrt", rule=(r0.t, r0.w), mvm_impl=impl)
        e = np.linalg.norm(out.cpu().numpy() - r0.out) / np.linalg.norm(r0.out)
        print(f"sigma2={sigma2:g}  J={r0.iters} impl={impl} UNpreconditioned relerr={e:.2e}")
