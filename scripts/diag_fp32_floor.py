"""Which fp32 rounding sets the C3 accuracy floor?  (diagnostic for DESIGN.md section 5)

numpy emulation of msMINRES-CIQ (the recurrence of oracle.msminres) at a reduced N with C3's
conditioning (RBF d = 6, l = 0.15, sigma^2 scaled so kappa(K) ~ 1.8e3 as at C3), K^{1/2} b against
the all-fp64 run, with fp32 rounding injected in one place at a time:
  vec32: Lanczos / direction / solution vectors rounded to fp32 after every update (fp64 scalars),
         K and its MVM in fp64;
  mvm32: K entries rounded to fp32 and the MVM accumulated in fp32 (V rounded to fp32 on input),
         recurrence in fp64;
  both : the two together (what an fp32 library computes).
Not test infrastructure; prints one line per variant."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import hht_rule  # noqa: E402


def run(kmat, b, t, w, J, vec32, mvm32, sqrt=True, k32=None, seq=False):
    f = (lambda a: a.astype(np.float32).astype(np.float64)) if vec32 else (lambda a: a)
    if k32 is None:
        k32 = kmat.astype(np.float32)

    def mvm(v):
        if seq:   # sequential fp32 accumulation over j (the SIMT kernel's per-thread order)
            v32 = v.astype(np.float32)
            out = np.empty(v.shape)
            for c in range(v.shape[1]):
                out[:, c] = np.cumsum(k32 * v32[None, :, c], axis=1, dtype=np.float32)[:, -1]
            return out
        if mvm32:
            return (k32 @ v.astype(np.float32)).astype(np.float64)
        return kmat @ v
    n, T = b.shape
    nq = len(t)
    beta1 = np.linalg.norm(b, axis=0)
    v = f(b / beta1)
    vp = np.zeros_like(v)
    beta = np.zeros(T)
    c1 = np.ones((nq, T)); s1 = np.zeros((nq, T)); c2 = np.ones((nq, T)); s2 = np.zeros((nq, T))
    phib = np.tile(beta1, (nq, 1))
    d1 = np.zeros((nq, n, T)); d2 = np.zeros((nq, n, T)); y = np.zeros((n, T))
    for j in range(J):
        p = mvm(v)
        al = np.sum(v * p, axis=0)
        p = f(p - al * v - beta * vp)
        bn = np.linalg.norm(p, axis=0)
        for q in range(nq):
            a = al + t[q]
            eps = s2[q] * beta; dp = c2[q] * beta
            de = c1[q] * dp + s1[q] * a; gb = -s1[q] * dp + c1[q] * a
            g = np.hypot(gb, bn); c = gb / g; s = bn / g
            phi = c * phib[q]; phib[q] = -s * phib[q]
            d = f((v - de * d1[q] - eps * d2[q]) / g)
            y = f(y + w[q] * phi * d)
            d2[q] = d1[q]; d1[q] = d; c2[q] = c1[q]; s2[q] = s1[q]; c1[q] = c; s1[q] = s
        vp = v; v = f(p / bn); beta = bn
    return mvm(y) if sqrt else y


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 6000
    rng = np.random.default_rng(0)
    x = rng.random((n, 6)).astype(np.float32).astype(np.float64)
    ell = float(sys.argv[3]) if len(sys.argv) > 3 else 0.15
    sq = (x * x).sum(1)
    r2 = np.maximum(sq[:, None] + sq[None, :] - 2 * x @ x.T, 0) / ell ** 2
    k = np.exp(-0.5 * r2)
    lk = np.linalg.eigvalsh(k)
    sigma2 = max(lk[-1] / 1788.0 - max(lk[0], 0.0), 1e-6)
    k[np.diag_indices(n)] += sigma2
    lam = np.linalg.eigvalsh(k)
    t, w = hht_rule(lam[0] * 0.99, lam[-1] * 1.01, 8)
    b = rng.standard_normal((n, 2))
    J = int(sys.argv[2]) if len(sys.argv) > 2 else 300
    ref = run(k, b, t, w, J, False, False)
    print(f"N={n} kappa={lam[-1] / lam[0]:.0f} J={J}")
    # kernel entries as an fp32 kernel computes them: scaled fp32 coordinates, (a) coordinate
    # differences + fp32 exp (SIMT), (b) the expanded form |y_i|^2/2 + |y_j|^2/2 - y_i.y_j in fp32
    y = ((x - x.mean(0)) / ell).astype(np.float32)
    diff = np.zeros((n, n), np.float32)
    for a in range(6):
        dd = y[:, None, a] - y[None, :, a]
        diff += dd * dd
    k_simt = np.exp(np.float32(-0.5) * diff).astype(np.float32)
    k_simt[np.diag_indices(n)] += np.float32(sigma2)
    h = (0.5 * (y * y).sum(1)).astype(np.float32)
    s_exp = (h[:, None] + h[None, :]) - (y @ y.T).astype(np.float32)
    k_exp = np.exp(-np.maximum(s_exp, 0)).astype(np.float32)
    k_exp[np.diag_indices(n)] += np.float32(sigma2)
    print("entry rel err simt", float(np.abs(k_simt - k).max()), "expanded", float(np.abs(k_exp - k).max()))
    variants = [("vec32", True, False, None, False), ("mvm32", False, True, None, False), ("both", True, True, None, False),
                ("simt_entries", True, True, k_simt, False), ("exp_entries", True, True, k_exp, False)]
    if "--seq" in sys.argv:
        variants.append(("simt_seq", True, True, k_simt, True))
    for name, v32, m32, kk, seq in variants:
        got = run(k, b, t, w, J, v32, m32, k32=kk, seq=seq)
        err = [float(np.linalg.norm(got[:, c] - ref[:, c]) / np.linalg.norm(ref[:, c])) for c in range(2)]
        print(f"{name:6s} sqrt rel err vs fp64 {err}", flush=True)


if __name__ == "__main__":
    main()
