"""Write tests/golden/c3_full_cols.npz: the float64 oracle's K^{1/2}B at config C3's FULL size
(N = 50,000 matrix-free RBF, d = 6, Q = 8) for the first two right-hand-side columns of C3's
seeded B -- the reference for the full-N solve parity tests (tests/test_gpu_fullsize.py).

Calls only ``oracle/`` and the seeded input generators (``workloads``); no value comes from the
CUDA path.  Columns are independent in msMINRES-CIQ (reading G15), so two columns
of the 64-column bench RHS block are checked against the same columns of the GPU's full solve.

Same inputs as the library: the fp32 points, B and the fp32-rounded l, o^2, sigma^2.
Protocol: the oracle's lambda estimate (10 Lanczos steps on the
seeded 16-column start block, lambda_min bound sigma^2, reading G6) gives the rule (t, w); the
solve then runs to a tight stopping tolerance (``--tol``, default 1e-8 on max_q |phibar|/beta1),
so the stored K^{1/2}b is the quadrature approximation with a negligible Krylov error.  The rule,
J reached and the per-shift residuals are stored alongside, so a GPU run can use the same rule
at the same J (strict parity) or its own estimate and stopping rule (bench configuration).

Cost: ~12 s per oracle MVM at N = 5e4 on 8 threads; J + 11 MVMs (~40-60 min).
usage: python scripts/make_golden_fullsize.py [--cols 2] [--tol 1e-8] [--threads 8]"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
from oracle import KernelOperator, estimate_spectrum, hht_rule, msminres  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--cols", type=int, default=2)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--max-iters", type=int, default=600)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = workloads.CONFIGS[a.config]
    inp = workloads.make_inputs(cfg)
    # the scalars as the library receives them (the C ABI takes fp32 l, o^2, sigma^2): same inputs
    f32 = lambda v: float(np.float32(v))  # noqa: E731
    op = KernelOperator(inp["X"], cfg.kind, f32(cfg.lengthscale), f32(cfg.outputscale), f32(cfg.sigma2),
                        threads=a.threads)
    t0 = time.time()
    lmin, lmax, rmin, rmax = estimate_spectrum(op.mvm, inp["S"].astype(np.float64), 10, lower_bound=op.sigma2)
    t, w = hht_rule(lmin, lmax, cfg.q)
    print(f"lambda [{lmin:.6g}, {lmax:.6g}] ritz [{rmin:.6g}, {rmax:.6g}]  {time.time() - t0:.0f} s", flush=True)
    b = inp["B"][:, :a.cols].astype(np.float64)
    res = msminres(op.mvm, b, t, a.max_iters, a.tol)
    y = np.einsum("q,qnt->nt", w, res.x)
    out = op.mvm(y)
    relres = (np.abs(res.phibar) / res.beta1[None, :]).max()
    print(f"J = {res.iters} converged = {res.converged} max relres = {relres:.3e}  {time.time() - t0:.0f} s", flush=True)
    path = a.out or os.path.join(ROOT, "tests", "golden", f"{a.config.lower()}_full_cols.npz")
    np.savez_compressed(path, config=a.config, cols=np.arange(a.cols), out=out, y=y, t=t, w=w,
                        lambda_min=lmin, lambda_max=lmax, iters=res.iters, tol=a.tol,
                        phibar=res.phibar, beta1=res.beta1)
    print("wrote", path)


if __name__ == "__main__":
    main()
