"""numpy emulation of the tcgen05 MVM accumulation (split-fp16 products, one fp32 round-toward-zero
add per MMA of K = 16, chains of L 64-column tiles, fp32 sum of the chains) inside an fp32 msMINRES-CIQ
run at kappa ~ 1.8e3: error of K^{1/2}b against fp64 vs L.  usage: diag_rz_chain.py N ell J L1,L2,..
(profiles/chain_nsplit_r02.txt)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import hht_rule
n=int(sys.argv[1]); ell=float(sys.argv[2]); J=int(sys.argv[3]); Ls=[int(a) for a in sys.argv[4].split(",")]
rng = np.random.default_rng(0)
x = rng.random((n, 6)).astype(np.float32).astype(np.float64)
sq = (x * x).sum(1)
k = np.exp(-0.5 * np.maximum(sq[:, None] + sq[None, :] - 2 * x @ x.T, 0) / ell ** 2)
lk = np.linalg.eigvalsh(k); sigma2 = max(lk[-1] / 1788.0 - max(lk[0], 0.0), 1e-6)
kk = k.copy(); kk[np.diag_indices(n)] += sigma2
lam = np.linalg.eigvalsh(kk); t, w = hht_rule(lam[0] * 0.99, lam[-1] * 1.01, 8)
print("kappa", lam[-1]/lam[0], flush=True)
b = rng.standard_normal((n, 2))
k32 = k.astype(np.float32)
khi = (k32.view(np.uint32) & np.uint32(0xffffe000)).view(np.float32)
klo = (k32 - khi).astype(np.float16).astype(np.float64)
khi = khi.astype(np.float16).astype(np.float64)
def rz_add(acc, term):
    s = acc.astype(np.float64) + term
    r = s.astype(np.float32)
    over = np.abs(r.astype(np.float64)) > np.abs(s)
    r[over] = np.nextafter(r[over], np.float32(0))
    return r
def mvm_tc(v, L):
    # v: n x T fp64 -> split fp16 with a per-column scale
    sc = 2.0 ** np.floor(np.log2(np.abs(v).max(0) + 1e-300))
    vs = v / sc
    vhi = vs.astype(np.float16).astype(np.float64)
    vlo = (vs - vhi).astype(np.float16).astype(np.float64)
    nt = (n + 63) // 64
    out = np.zeros(v.shape)
    for s0 in range(0, nt, L):
        acc = np.zeros(v.shape, np.float32)
        for tt in range(s0, min(nt, s0 + L)):
            for ks in range(4):
                j0 = tt * 64 + ks * 16; j1 = min(n, j0 + 16)
                if j0 >= n: break
                acc = rz_add(acc, khi[:, j0:j1] @ vhi[j0:j1])
                acc = rz_add(acc, khi[:, j0:j1] @ vlo[j0:j1])
                acc = rz_add(acc, klo[:, j0:j1] @ vhi[j0:j1])
        out = (out.astype(np.float32) + acc).astype(np.float64)   # fp32 sum of the splits
    return out * sc + sigma2 * v
def run(mvm):
    f = lambda a: a.astype(np.float32).astype(np.float64)
    T = b.shape[1]; nq = len(t)
    beta1 = np.linalg.norm(b, axis=0); v = f(b / beta1); vp = np.zeros_like(v); beta = np.zeros(T)
    c1 = np.ones((nq, T)); s1 = np.zeros((nq, T)); c2 = np.ones((nq, T)); s2 = np.zeros((nq, T))
    phib = np.tile(beta1, (nq, 1)); d1 = np.zeros((nq, n, T)); d2 = np.zeros((nq, n, T)); y = np.zeros((n, T))
    for j in range(J):
        p = mvm(v); al = np.sum(v * p, axis=0); p = f(p - al * v - beta * vp); bn = np.linalg.norm(p, axis=0)
        for q in range(nq):
            a = al + t[q]; eps = s2[q] * beta; dp = c2[q] * beta
            de = c1[q] * dp + s1[q] * a; gb = -s1[q] * dp + c1[q] * a
            g = np.hypot(gb, bn); c = gb / g; s = bn / g
            phi = c * phib[q]; phib[q] = -s * phib[q]
            d = f((v - de * d1[q] - eps * d2[q]) / g); y = f(y + w[q] * phi * d)
            d2[q] = d1[q]; d1[q] = d; c2[q] = c1[q]; s2[q] = s1[q]; c1[q] = c; s1[q] = s
        vp = v; v = f(p / bn); beta = bn
    return kk @ y
ref = run(lambda v: kk @ v)
for L in Ls:
    got = run(lambda v: mvm_tc(v, L))
    print("L", L, [float(np.linalg.norm(got[:, c] - ref[:, c]) / np.linalg.norm(ref[:, c])) for c in range(2)], flush=True)
