"""Full-size C3: the fp64 accuracy mode (params.fp64) vs the oracle's golden columns (diagnostic)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch, workloads, paper_2006_11267_b200 as pb
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden", "c3_full_cols.npz")
g = np.load(path)
cfg = workloads.CONFIGS["C3"]; inp = workloads.make_inputs(cfg); cols = g["cols"]
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2) as c:
    for mode, key in (("sqrt", "out"), ("invsqrt", "y")):
        out = torch.empty((cfg.n, len(cols)), device="cuda")
        t0 = time.time()
        info = c.apply(dev(inp["B"][:, cols]), out, q=cfg.q, max_iters=int(g["iters"]), tol=0.0, mode=mode,
                       rule=(g["t"], g["w"]), fp64=True)
        o = out.cpu().numpy().astype(np.float64)
        print(mode, "fp64 route", info["fp64_route"], "J", info["iters"], "err", [rel(o[:, k], g[key][:, k]) for k in range(2)],
              "%.1f s" % (time.time() - t0), flush=True)
