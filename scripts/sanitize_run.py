"""One small msMINRES-CIQ call for compute-sanitizer (SURVEY §4's sanitizer tier): C1 (N = 256, SIMT
MVM) and a reduced C3 (N = 1500, T = 64: the persistent tcgen05 kernel, fused update packing, the
CUDA-graph loop), the dense path, and the CTA-pair kernel (d = 12).  No checks here -- the
sanitizer's report is the result.
    compute-sanitizer --tool memcheck python scripts/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_11267_b200 as pb  # noqa: E402
import workloads  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


for name, n, t in (("C1", 256, 1), ("C3", 1500, 64), ("C2", 1024, 16)):
    cfg = workloads.scaled(workloads.CONFIGS[name], n=n, t=t)
    inp = workloads.make_inputs(cfg)
    if cfg.kind == "dense":
        g = pb.CIQ("dense", K=dev(inp["K"]), diag=cfg.sigma2)
    else:
        g = pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2)
    out = torch.empty((n, t), device="cuda")
    info = g.apply(dev(inp["B"]), out, q=8, max_iters=30, tol=0.0, mode="sqrt", lanczos_start=dev(inp["S"]))
    info2 = g.apply(dev(inp["B"]), out, q=8, max_iters=30, tol=1e-3, mode="invsqrt", lanczos_reuse=True)
    g.close()
    print(name, n, t, info["iters"], info["mvm_impl_used"], info2["iters"], flush=True)
# round 2: stored basis (W_{j+1} copy in the streaming pass, step scalars in the Givens pass, alpha in
# the full-tile kernel's tail), the fp64 route (DMMA M MVM), the row-sharded overlap (NCCL world 1)
cfg = workloads.scaled(workloads.CONFIGS["C3"], n=1500, t=64)
inp = workloads.make_inputs(cfg)
with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2) as g:
    out = torch.empty((cfg.n, cfg.t), device="cuda")
    info = g.apply(dev(inp["B"]), out, q=8, max_iters=40, tol=1e-4, mode="sqrt", lanczos_start=dev(inp["S"]),
                   lanczos_reuse=True, stored_basis=True)
    print("stored", info["iters"], info["mvm_impl_used"], info["mvm_splits"], flush=True)
with pb.CIQ(cfg.kind, n=cfg.n, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale,
            diag=cfg.sigma2, comm=(0, 1, pb.ciq_nccl_unique_id())) as g:
    out = torch.empty((cfg.n, cfg.t), device="cuda")
    info = g.apply(dev(inp["B"]), out, q=8, max_iters=30, tol=0.0, mode="sqrt", lanczos_start=dev(inp["S"]))
    print("sharded world 1", info["iters"], info["overlap"], flush=True)
cfg = workloads.scaled(workloads.CONFIGS["C4"], n=600, t=32)
inp = workloads.config_inputs(cfg)
with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2) as g:
    lfac = torch.empty((cfg.n, 20), device="cuda")
    g.pivoted_cholesky(20, lfac)   # the library's own partial pivoted Cholesky (row a9)
with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2,
            precond_L=lfac, precond_sigma2=cfg.sigma2) as g:
    out = torch.empty((cfg.n, cfg.t), device="cuda")
    info = g.apply(dev(inp["B"]), out, q=8, max_iters=30, tol=0.0, mode="whiten")
    print("fp64 route", info["iters"], info["mvm_impl_used"], info["fp64_route"], flush=True)
x = workloads.points(1024, 12)
with pb.CIQ("rbf", X=dev(x), lengthscale=0.5, outputscale=1.0, diag=0.1) as g:
    out = torch.empty((1024, 32), device="cuda")
    info = g.apply(dev(workloads.rhs(1024, 32)), out, q=8, max_iters=20, tol=0.0, mode="sqrt",
                   lanczos_start=dev(workloads.lanczos_start(1024)))
    print("d=12", info["iters"], info["mvm_impl_used"], flush=True)
torch.cuda.synchronize()
print("done")
