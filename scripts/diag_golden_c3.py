"""Full-size C3 solve vs the oracle's golden columns (tests/golden/c3_full_cols.npz): tensor-core
vs fp32 SIMT MVM, same rule, fixed J (diagnostic for DESIGN.md section 5)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads, paper_2006_11267_b200 as pb
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "c3_full_cols.npz"))
cfg = workloads.CONFIGS["C3"]; inp = workloads.make_inputs(cfg); cols = g["cols"]
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
for impl in ("tc", "simt"):
    for j in (int(g["iters"]), 200):
        with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2) as c:
            out = torch.empty((cfg.n, len(cols)), device="cuda")
            y = torch.empty_like(out)
            info = c.apply(dev(inp["B"][:, cols]), out, q=cfg.q, max_iters=j, tol=0.0, mode="sqrt", rule=(g["t"], g["w"]), mvm_impl=impl)
            c.apply(dev(inp["B"][:, cols]), y, q=cfg.q, max_iters=j, tol=0.0, mode="invsqrt", rule=(g["t"], g["w"]), mvm_impl=impl)
            o, yy = out.cpu().numpy().astype(np.float64), y.cpu().numpy().astype(np.float64)
        print(impl, "J", j, "sqrt err", [rel(o[:, k], g["out"][:, k]) for k in range(2)],
              "invsqrt err", [rel(yy[:, k], g["y"][:, k]) for k in range(2)], "relres", info["max_rel_residual"], flush=True)
