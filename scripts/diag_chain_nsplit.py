"""C3 full size: error of the tensor-core solve against the oracle's golden columns vs the length of
the TMEM accumulation chains (column splits of the MVM), and the MVM / step time.  Run once per
split count with an experiments build (CIQ_LIB=_ab/<name>/libciq.so, CIQ_TC_NSPLIT=<s>):
64 columns (the bench's tc2 kernel), the golden rule and J (tests/golden/c3_full_cols.npz)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_11267_b200 as pb  # noqa: E402
import workloads  # noqa: E402

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
g = np.load(os.path.join(root, "tests", "golden", "c3_full_cols.npz"))
cfg = workloads.CONFIGS["C3"]
inp = workloads.make_inputs(cfg)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()  # noqa: E731
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
with pb.CIQ(cfg.kind, X=dev(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2) as c:
    b = dev(inp["B"])
    out = torch.empty_like(b)
    res = {}
    for mode, key in (("sqrt", "out"), ("invsqrt", "y")):
        info = c.apply(b, out, q=cfg.q, max_iters=int(g["iters"]), tol=0.0, mode=mode, rule=(g["t"], g["w"]),
                       profile=True)
        o = out.cpu().numpy().astype(np.float64)
        res[mode] = [rel(o[:, k], g[key][:, i]) for i, k in enumerate(g["cols"])]
    mvm_ms = info["ms_mvm"] / max(1, info["mvm_timed"])
    # the bench call (stored basis, lanczos reuse, tol 1e-4), timed
    s = dev(inp["S"])
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for r in range(4):
        ev0.record()
        ib = c.apply(b, out, q=cfg.q, max_iters=cfg.max_iters, tol=cfg.tol, mode="sqrt", lanczos_start=s,
                     lanczos_reuse=True, stored_basis=True)
        ev1.record()
        ev1.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    o = out.cpu().numpy().astype(np.float64)
    bench_err = [rel(o[:, k], g["out"][:, i]) for i, k in enumerate(g["cols"])]
print(f"nsplit={os.environ.get('CIQ_TC_NSPLIT', 'auto')} splits_used={info['mvm_splits']} impl={info['mvm_impl_used']} "
      f"sqrt={res['sqrt']} invsqrt={res['invsqrt']} mvm_ms={mvm_ms:.4f} bench_ms={min(ts[1:]):.2f} "
      f"bench_J={ib['iters']} bench_err={bench_err}", flush=True)
