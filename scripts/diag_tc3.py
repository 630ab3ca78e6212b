"""Check the CTA-pair matrix-free MVM (mvm_tc3.cu) against the fp32 SIMT kernel and the oracle on
sampled rows, and time it at C3 (diagnostic; the parity tests are in tests/).
    python scripts/diag_tc3.py [--quick]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_11267_b200 as pb  # noqa: E402
import workloads  # noqa: E402
from oracle import KernelOperator  # noqa: E402

cases = [("C3", 777, 32), ("C3", 1500, 64), ("C3", 4096, 64), ("C3", 4096, 128), ("C5", 3000, 32), ("C3", 50000, 64)]
if "--quick" in sys.argv:
    cases = cases[:2]
for name, n, t in cases:
    cfg = workloads.scaled(workloads.CONFIGS[name], n=n, t=t)
    inp = workloads.make_inputs(cfg)
    x = torch.from_numpy(inp["X"]).cuda()
    v = torch.from_numpy(workloads.rhs(n, t, seed=9)).cuda()
    with pb.CIQ(cfg.kind, X=x, lengthscale=cfg.lengthscale, outputscale=cfg.outputscale, diag=cfg.sigma2) as g:
        o_tc = torch.empty_like(v)
        o_si = torch.empty_like(v)
        torch.cuda.synchronize()
        t0 = time.time()
        g.matvec(v, o_tc, mvm_impl="tc")
        torch.cuda.synchronize()
        t1 = time.time()
        g.matvec(v, o_si, mvm_impl="simt")
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for r in range(5):
            st.record()
            g.matvec(v, o_tc, mvm_impl="tc")
            en.record()
            en.synchronize()
            ms.append(st.elapsed_time(en))
    a, b = o_tc.cpu().numpy().astype(np.float64), o_si.cpu().numpy().astype(np.float64)
    rows = np.unique(np.concatenate([np.arange(4), np.arange(n - 4, n), np.random.default_rng(1).choice(n, 12)]))
    ref = KernelOperator(inp["X"], cfg.kind, cfg.lengthscale, cfg.outputscale, cfg.sigma2).mvm_rows(rows, workloads.rhs(n, t, seed=9).astype(np.float64))
    e_si = np.abs(a - b).max() / np.abs(b).max()
    e_or = np.abs(a[rows] - ref).max() / np.abs(ref).max()
    print(f"{name} n={n} t={t}: tc vs simt {e_si:.2e}  tc vs oracle rows {e_or:.2e}  first call {1e3*(t1-t0):.1f} ms  "
          f"mvm {np.median(ms):.3f} ms (min {min(ms):.3f})", flush=True)
