"""C2 (dense N = 10k, whiten) with and without the relaxed MVM schedule against the float64 oracle
on two columns, same rule and J (diagnostic for DESIGN.md section 5)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads, paper_2006_11267_b200 as pb
from oracle import DenseOperator, estimate_spectrum, hht_rule, ciq
cfg = workloads.CONFIGS["C2"]
inp = workloads.make_inputs(cfg)
op = DenseOperator(inp["K"].astype(np.float64), cfg.sigma2)
lmin, lmax, _, _ = estimate_spectrum(op.mvm, inp["S"], 10, lower_bound=cfg.sigma2)
t, w = hht_rule(lmin, lmax, cfg.q)
J = 251
cols = [0, 1]
ref = ciq(op, inp["B"][:, cols].astype(np.float64), q=cfg.q, max_iters=J, tol=0.0, mode="whiten", rule=(t, w))
print("oracle relres", float(np.max(np.abs(ref.solve.phibar) / ref.solve.beta1)), flush=True)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
with pb.CIQ("dense", K=dev(inp["K"]), diag=cfg.sigma2) as g:
    for relax in (False, True):
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.apply(dev(inp["B"]), out, q=cfg.q, max_iters=J, tol=0.0, mode="whiten", rule=(t, w), mvm_relax=relax)
        o = out.cpu().numpy().astype(np.float64)
        err = [float(np.linalg.norm(o[:, c] - ref.out[:, i]) / np.linalg.norm(ref.out[:, i])) for i, c in enumerate(cols)]
        print("relax", relax, "relaxed2_from", info["relaxed2_from"], "err", err, flush=True)
