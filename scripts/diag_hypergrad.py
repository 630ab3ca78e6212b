"""Hyper-parameter gradient: GPU (tc / simt) vs the oracle across noise levels (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads, paper_2006_11267_b200 as pb
from oracle import KernelOperator, ciq, ciq_hyper_grad, estimate_spectrum, hht_rule
def dev(a): return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
f32 = lambda v: float(np.float32(v))
n, t = 600, 4
x = workloads.points(n, 3); b = workloads.rhs(n, t); v = workloads.rhs(n, t, seed=11)
for kind in ("rbf", "matern52"):
    for s2 in (0.05, 0.2, 1.0):
        ls, o2 = 0.3, 1.3
        op = KernelOperator(x, kind, f32(ls), f32(o2), f32(s2))
        lmin, lmax, _, _ = estimate_spectrum(op.mvm, workloads.lanczos_start(n), 10, lower_bound=f32(s2))
        rule = hht_rule(lmin, lmax, 8)
        j = max(ciq(op, u.astype(np.float64), q=8, max_iters=2000, tol=1e-8, mode="invsqrt", rule=rule).iters for u in (b, v))
        ref = ciq_hyper_grad(op, b.astype(np.float64), v.astype(np.float64), rule, max_iters=j)
        for impl in ("tc", "simt"):
            with pb.CIQ(kind, X=dev(x), lengthscale=ls, outputscale=o2, diag=s2) as g:
                grad, info = g.hyper_grad(dev(b), dev(v), q=8, max_iters=j, tol=0.0, rule=rule, mvm_impl=impl)
            print(kind, "s2", s2, "kappa %.0f J %d" % (lmax / lmin, j), impl, "relerr", np.abs(grad / ref - 1), flush=True)
