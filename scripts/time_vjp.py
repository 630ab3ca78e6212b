"""Time ciq_vjp (backward pass) on a BASELINE config, warm (each call timed after two
identical calls): the forward solve alone, the forward with kept shifted solves, the v solve with the
forward's rule, and the whole vjp (both solves + the dense G product).  python scripts/time_vjp.py [C2]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_11267_b200 as pb  # noqa: E402
import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = workloads.CONFIGS[name]
inp = workloads.make_inputs(cfg)
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()  # noqa: E731
if cfg.kind == "dense":
    g = pb.CIQ("dense", K=dv(inp["K"]), diag=cfg.sigma2)
else:
    g = pb.CIQ(cfg.kind, X=dv(inp["X"]), lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2)
b, v = dv(inp["B"]), dv(workloads.rhs(cfg.n, cfg.t, seed=7))
gm = torch.empty((cfg.n, cfg.n), device="cuda")
kw = dict(q=cfg.q, max_iters=cfg.max_iters, tol=cfg.tol, lanczos_start=dv(inp["S"]), mode="invsqrt")
out = torch.empty_like(b)
xs = torch.empty((cfg.q, cfg.n, cfg.t), device="cuda")


def timed(fn):
    for _ in range(2):
        fn()
    e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
    torch.cuda.synchronize()
    e0.record()
    r = fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1), r


fwd, info_f = timed(lambda: g.apply(b, out, **kw))
keep, _ = timed(lambda: g.apply(b, out, shift_solutions=xs, **kw))
rule = (np.array(info_f["t"][:cfg.q]), np.array(info_f["w"][:cfg.q]))
kw_v = dict(kw, rule=rule)
kw_v.pop("lanczos_start")
vsolve, info_v = timed(lambda: g.apply(v, out, shift_solutions=xs, **kw_v))
vjp, info = timed(lambda: g.vjp(b, v, gm, **kw))
n, t, q = cfg.n, cfg.t, cfg.q
gflop = 2.0 * 2.0 * n * n * q * t / 1e9
print(json.dumps({"config": name, "forward_ms": fwd, "forward_keep_ms": keep, "v_solve_ms": vsolve,
                  "vjp_ms": vjp, "vjp_over_forward": vjp / fwd, "J": info["iters"], "J_v": info_v["iters"],
                  "mvms": info["mvms"], "G_product_gflop": gflop}))
