"""msMINRES-CIQ float64 CPU oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

A plain, slow, obviously-correct implementation of what the product's hot path computes, written
from PAPER.md (cited as ``P:<line>``; SPEC.md lines as ``S:<line>``) in float64, following the
paper's steps in its own order and notation.  Library primitives used as single steps: numpy
matmul / norms, ``mpmath.ellipk`` / ``mpmath.ellipfun`` (complex-argument Jacobi functions) and
``scipy.linalg.eigvalsh_tridiagonal``.  No blocking, fusion or reordering beyond what the
definitions state (row blocks of K are assembled only to bound memory; each block is the plain
definition).  Shares no code with ``paper_2006_11267_b200``.

Where the paper is silent or garbled, the reading taken is the one listed in DESIGN.md §2
("Readings", G1-G18); each function names the readings it uses.

Parity pins: every public function below is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against something other than itself (eigendecomposition, closed
forms, scipy's independent MINRES, the Hale error bound, Lemma 3, Gram identities).  None is
"parity unpinned".
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable

import mpmath
import numpy as np
import scipy.linalg

__all__ = [
    "kernel_entries", "KernelOperator", "DenseOperator", "LowRankPlusDiag",
    "hht_rule", "lanczos", "estimate_spectrum", "msminres", "ciq",
    "pivoted_cholesky", "precond_ciq", "MsminresResult", "CiqResult", "ciq_vjp",
    "PosteriorOperator", "thompson_step", "kernel_lengthscale_derivative", "ciq_hyper_grad",
    "SparseOperator", "BlockJacobi",
]


# --------------------------------------------------------------------------------------------
# L0 -- the operator K, touched only through MVMs
# --------------------------------------------------------------------------------------------

def kernel_entries(xa: np.ndarray, xb: np.ndarray, kind: str, lengthscale, outputscale: float) -> np.ndarray:
    """k(x_a, x_b) for all pairs, from the textbook definitions (reading G11):

    RBF        o^2 exp(-r^2/2)
    Matern-5/2 o^2 (1 + sqrt5 r + 5 r^2/3) exp(-sqrt5 r)
    Matern-3/2 o^2 (1 + sqrt3 r) exp(-sqrt3 r)

    with r = || (x_a - x_b) / l || (ARD: per-coordinate lengthscale).  The squared distance is
    formed from the coordinate differences themselves (no norm expansion):
    r^2 = sum_k (a_k - b_k)^2, accumulated coordinate by coordinate (k = 0, 1, ..., d-1)."""
    ls = np.asarray(lengthscale, dtype=np.float64)
    a = np.asarray(xa, dtype=np.float64) / ls
    b = np.asarray(xb, dtype=np.float64) / ls
    r2 = np.zeros((a.shape[0], b.shape[0]))
    for k in range(a.shape[1]):
        diff = a[:, k, None] - b[None, :, k]
        r2 += diff * diff
    if kind == "rbf":
        k = np.exp(-0.5 * r2)
    elif kind == "matern52":
        r = np.sqrt(r2)
        k = (1.0 + math.sqrt(5.0) * r + 5.0 * r2 / 3.0) * np.exp(-math.sqrt(5.0) * r)
    elif kind == "matern32":
        r = np.sqrt(r2)
        k = (1.0 + math.sqrt(3.0) * r) * np.exp(-math.sqrt(3.0) * r)
    else:
        raise ValueError(f"unknown kernel kind {kind!r}")
    return outputscale * k


class KernelOperator:
    """K = k(X, X) + sigma2 I, applied matrix-free ("map-reduce"): each row block of K is
    assembled from ``kernel_entries`` and multiplied; the full matrix is cached only when small.
    ``mvm_count`` counts applications (Property 1).

    ``threads`` > 1 maps the independent row blocks over a thread pool (numpy releases the GIL
    inside its array loops); every block is still the plain definition, and each output row is
    computed by one block exactly as in the serial loop, so the result does not depend on the
    thread count.  ``block`` defaults to a row count that keeps one block's n-wide temporaries
    near 4 MB (full-size checks at N = 5e4 .. 2e5)."""

    def __init__(self, x, kind: str, lengthscale=1.0, outputscale: float = 1.0, sigma2: float = 0.0,
                 dense_cache_max: int = 6144, block: int | None = None, threads: int = 1):
        self.x = np.asarray(x, dtype=np.float64)
        self.n = self.x.shape[0]
        self.kind = kind
        self.lengthscale = lengthscale
        self.outputscale = float(outputscale)
        self.sigma2 = float(sigma2)
        self.block = block if block is not None else max(8, min(512, (1 << 19) // max(1, self.n)))
        self.threads = max(1, int(threads))
        self.mvm_count = 0
        self._dense = None
        if self.n <= dense_cache_max:
            self._dense = kernel_entries(self.x, self.x, kind, lengthscale, outputscale)

    def kernel_rows(self, i0: int, i1: int) -> np.ndarray:
        """Rows i0..i1-1 of k(X, X) (without sigma2)."""
        if self._dense is not None:
            return self._dense[i0:i1]
        return kernel_entries(self.x[i0:i1], self.x, self.kind, self.lengthscale, self.outputscale)

    def kernel_column(self, j: int) -> np.ndarray:
        """Column j of k(X, X) (symmetric, so equal to row j)."""
        return self.kernel_rows(j, j + 1)[0]

    def kernel_diag(self) -> np.ndarray:
        return np.full(self.n, self.outputscale)  # k(x, x) = o^2 for stationary kernels

    def dense(self) -> np.ndarray:
        return self.kernel_rows(0, self.n) + self.sigma2 * np.eye(self.n)

    def mvm(self, v: np.ndarray) -> np.ndarray:
        """K v, v of shape (n,) or (n, t)."""
        self.mvm_count += 1
        v = np.asarray(v, dtype=np.float64)
        out = np.empty_like(v)

        def row_block(i0):
            i1 = min(self.n, i0 + self.block)
            out[i0:i1] = self.kernel_rows(i0, i1) @ v

        starts = range(0, self.n, self.block)
        if self.threads > 1 and self._dense is None:
            import concurrent.futures
            with concurrent.futures.ThreadPoolExecutor(self.threads) as pool:
                list(pool.map(row_block, starts))
        else:
            for i0 in starts:
                row_block(i0)
        return out + self.sigma2 * v

    def mvm_row_block(self, i0: int, i1: int, v: np.ndarray) -> np.ndarray:
        """Rows i0..i1-1 of K v, by the same (threaded) row-block map as ``mvm`` (for the bench's
        bounded CPU baseline); does not count as an MVM."""
        v = np.asarray(v, dtype=np.float64)
        out = np.empty((i1 - i0,) + v.shape[1:])

        def row_block(j0):
            j1 = min(i1, j0 + self.block)
            out[j0 - i0:j1 - i0] = self.kernel_rows(j0, j1) @ v

        starts = range(i0, i1, self.block)
        if self.threads > 1 and self._dense is None:
            import concurrent.futures
            with concurrent.futures.ThreadPoolExecutor(self.threads) as pool:
                list(pool.map(row_block, starts))
        else:
            for j0 in starts:
                row_block(j0)
        out += self.sigma2 * v[i0:i1]
        return out

    def mvm_rows(self, rows: np.ndarray, v: np.ndarray) -> np.ndarray:
        """(K v)[rows] -- individual outputs, one row at a time (for sampled full-size checks)."""
        v = np.asarray(v, dtype=np.float64)
        out = []
        for i in np.asarray(rows):
            krow = kernel_entries(self.x[i:i + 1], self.x, self.kind, self.lengthscale, self.outputscale)[0]
            out.append(krow @ v + self.sigma2 * v[i])
        return np.stack(out)


class DenseOperator:
    """K = A + sigma2 I for a given dense symmetric A (the dense path)."""

    def __init__(self, a, sigma2: float = 0.0):
        self.a = np.asarray(a, dtype=np.float64)
        self.n = self.a.shape[0]
        self.sigma2 = float(sigma2)
        self.mvm_count = 0

    def dense(self) -> np.ndarray:
        return self.a + self.sigma2 * np.eye(self.n)

    def kernel_column(self, j: int) -> np.ndarray:
        return self.a[:, j].copy()

    def kernel_diag(self) -> np.ndarray:
        return np.diag(self.a).copy()

    def mvm(self, v):
        self.mvm_count += 1
        v = np.asarray(v, dtype=np.float64)
        return self.a @ v + self.sigma2 * v

    def mvm_rows(self, rows, v):
        v = np.asarray(v, dtype=np.float64)
        rows = np.asarray(rows)
        return self.a[rows] @ v + self.sigma2 * v[rows]


class SparseOperator:
    """K = A + sigma2 I for a given sparse symmetric A in CSR form (indptr, indices, data) -- the
    stencil precision of the Gibbs workload (Lambda = gamma_obs A^T A + gamma_prior L^T L,
    P:995-1004) is such an operator; msMINRES-CIQ only needs its MVMs.  The MVM is
    scipy.sparse's CSR product (a library step), in float64 on the caller's (float32) values."""

    def __init__(self, indptr, indices, data, n: int, sigma2: float = 0.0):
        import scipy.sparse
        self.a = scipy.sparse.csr_matrix((np.asarray(data, dtype=np.float64), np.asarray(indices),
                                          np.asarray(indptr)), shape=(n, n))
        self.n = n
        self.sigma2 = float(sigma2)
        self.mvm_count = 0

    def dense(self) -> np.ndarray:
        return self.a.toarray() + self.sigma2 * np.eye(self.n)

    def kernel_column(self, j: int) -> np.ndarray:
        return self.a[:, j].toarray()[:, 0]

    def kernel_diag(self) -> np.ndarray:
        return self.a.diagonal().copy()

    def mvm(self, v):
        self.mvm_count += 1
        v = np.asarray(v, dtype=np.float64)
        return self.a @ v + self.sigma2 * v

    def mvm_rows(self, rows, v):
        v = np.asarray(v, dtype=np.float64)
        rows = np.asarray(rows)
        return self.a[rows] @ v + self.sigma2 * v[rows]


# --------------------------------------------------------------------------------------------
# L2 -- the Hale-Higham-Trefethen quadrature rule (App. B)
# --------------------------------------------------------------------------------------------

def hht_rule(lambda_min: float, lambda_max: float, q: int, dps: int = 40):
    """Shifts t_q > 0 and weights w_q > 0 of eq. quad_points_and_locations and
    eq. contour_integral_quad_4, evaluated LITERALLY with complex arguments:

        k        = sqrt(lambda_min / lambda_max)
        K'(k)    = complete elliptic integral of the first kind at k' = sqrt(1-k^2)
        u_q      = (q - 1/2) / Q
        sigma_q^2 = lambda_min * sn(i u_q K'(k) | k)^2
        w~_q     = -(2 sqrt(lambda_min) / (pi Q)) * K'(k) cn(i u_q K'(k) | k) dn(i u_q K'(k) | k)
        t_q = -sigma_q^2,  w_q = -w~_q

    mpmath's functions take the parameter m = k^2 (reading G10): K'(k) = ellipk(1 - k^2).
    kappa is clamped to >= 1 + 1e-8 so that k < 1.
    Returns float64 arrays (t, w)."""
    if q < 1:
        raise ValueError("Q must be >= 1")
    if not (lambda_min > 0 and lambda_max > 0):
        raise ValueError("lambda_min and lambda_max must be positive")
    with mpmath.workdps(dps):
        lmin = mpmath.mpf(lambda_min)
        lmax = mpmath.mpf(max(lambda_max, lambda_min * (1 + 1e-8)))
        k2 = lmin / lmax
        kprime_k = mpmath.ellipk(1 - k2)             # K'(k) = K(k'), parameter m' = 1 - k^2
        t = np.empty(q)
        w = np.empty(q)
        for qq in range(1, q + 1):
            u = (qq - mpmath.mpf("0.5")) / q
            z = 1j * u * kprime_k
            sn = mpmath.ellipfun("sn", z, m=k2)
            cn = mpmath.ellipfun("cn", z, m=k2)
            dn = mpmath.ellipfun("dn", z, m=k2)
            sigma2 = lmin * sn ** 2
            wtilde = -(2 * mpmath.sqrt(lmin) / (mpmath.pi * q)) * kprime_k * cn * dn
            t[qq - 1] = float(mpmath.re(-sigma2))
            w[qq - 1] = float(mpmath.re(-wtilde))
    return t, w


# --------------------------------------------------------------------------------------------
# L1 -- Lanczos with full re-orthogonalisation, extreme-eigenvalue estimate (App. B.2)
# --------------------------------------------------------------------------------------------

def lanczos(mvm: Callable, start: np.ndarray, iters: int, breakdown_tol: float = 1e-12):
    """Lanczos tridiagonalisation K Q_J = Q_J T_J + r_J e_J^T, independently for
    each column of ``start`` (reading G5), with full re-orthogonalisation (classical Gram-Schmidt
    applied twice).  Returns per column the diagonal alphas and off-diagonal betas of T_J
    as lists (columns that hit an invariant subspace stop early)."""
    s = np.asarray(start, dtype=np.float64)
    if s.ndim == 1:
        s = s[:, None]
    n, tl = s.shape
    norms = np.linalg.norm(s, axis=0)
    if np.any(norms == 0):
        raise ValueError("zero Lanczos start vector")
    basis = [s / norms]
    alphas = [[] for _ in range(tl)]
    betas = [[] for _ in range(tl)]
    active = np.ones(tl, dtype=bool)
    for j in range(iters):
        v = basis[-1]
        w = mvm(v)
        qb = np.stack(basis)                       # (j+1, n, tl)
        alpha = np.zeros(tl)
        for _ in range(2):                         # CGS twice
            h = np.einsum("jnt,nt->jt", qb, w)
            w = w - np.einsum("jnt,jt->nt", qb, h)
            alpha += h[-1]
        beta = np.linalg.norm(w, axis=0)
        for c in range(tl):
            if active[c]:
                alphas[c].append(alpha[c])
        stop = beta <= breakdown_tol * (np.abs(alpha) + (np.array([b[-1] if b else 0.0 for b in betas])))
        if j == iters - 1:
            break
        for c in range(tl):
            if active[c]:
                if stop[c]:
                    active[c] = False
                else:
                    betas[c].append(beta[c])
        if not np.any(active):
            break
        basis.append(np.where(active[None, :], w / np.where(beta > 0, beta, 1.0)[None, :], 0.0))
    return alphas, betas


def estimate_spectrum(mvm: Callable, start: np.ndarray, iters: int = 10, lower_bound: float = 0.0):
    """lambda_min / lambda_max for the HHT rule.

    Ritz values = eigenvalues of each T_J (scipy's tridiagonal eigensolver, "standard routines",
    P:1515), pooled over the start columns (reading G5).  Safety margins (reading G6):
      lambda_max = 1.01 * max Ritz
      lambda_min = min(0.99 * min Ritz, lower_bound) if lower_bound > 0 else 0.99 * min Ritz
    where ``lower_bound`` is a rigorous lower bound on lambda_min(K) (the operator's sigma2, or 1
    for the pivoted-Cholesky-preconditioned operator).
    Returns (lambda_min, lambda_max, ritz_min, ritz_max)."""
    alphas, betas = lanczos(mvm, start, iters)
    ritz_min, ritz_max = math.inf, -math.inf
    for a, b in zip(alphas, betas):
        ev = scipy.linalg.eigvalsh_tridiagonal(np.asarray(a), np.asarray(b[:len(a) - 1]))
        ritz_min = min(ritz_min, float(ev[0]))
        ritz_max = max(ritz_max, float(ev[-1]))
    lmax = 1.01 * ritz_max
    lmin = 0.99 * ritz_min
    if lower_bound > 0:
        lmin = min(lmin, lower_bound)
    if not lmin > 0:
        raise ValueError(f"lambda_min estimate {lmin} <= 0: operator is not positive definite")
    return lmin, lmax, ritz_min, ritz_max


# --------------------------------------------------------------------------------------------
# L1 -- msMINRES (App. C)
# --------------------------------------------------------------------------------------------

@dataclasses.dataclass
class MsminresResult:
    x: np.ndarray            # (Q, n, t): x_q ~ (t_q I + K)^{-1} b
    phibar: np.ndarray       # (Q, t): |phibar| = recurrence residual ||(K + t_q I) x_q - b||
    beta1: np.ndarray        # (t,): ||b||
    iters: int               # J
    mvms: int                # MVMs spent (== iters, Property 1)
    converged: bool


def msminres(mvm: Callable, b: np.ndarray, shifts: np.ndarray, max_iters: int, tol: float = 0.0,
             breakdown_tol: float = 1e-12) -> MsminresResult:
    """Multi-shift MINRES, reconstructed from App. C (reading G1):

    One Lanczos recurrence on K from b (Observation) drives, for every shift t_q, the
    MINRES Givens QR of [T_J + t_q I; beta_{J+1} e_J^T] (eq. minres_qr_shifted; "add t
    to the Lanczos diagonal") and the descent update c_J = c_{J-1} + phi_J d_J
    (eq. minres_descent).  Per column c and shift q, iteration j:

        p = K v_j ;  alpha = v_j^T p ;  p <- p - alpha v_j - beta_j v_{j-1} ;  beta_{j+1} = ||p||
        a = alpha + t_q
        eps = s2 beta_j ;  delta' = c2 beta_j ;  delta = c1 delta' + s1 a ;  gbar = -s1 delta' + c1 a
        gamma = hypot(gbar, beta_{j+1}) ;  c = gbar/gamma ;  s = beta_{j+1}/gamma
        phi = c phibar ;  phibar <- -s phibar
        d_j = (v_j - delta d_{j-1} - eps d_{j-2}) / gamma ;  x_q <- x_q + phi d_j
        v_{j+1} = p / beta_{j+1}

    Columns are independent (reading G15).  Stopping (reading G3): all columns stop together when
    max_{q,c} |phibar|/beta1_c <= tol (tol = 0: exactly ``max_iters`` iterations).  A column whose
    beta_{j+1} <= breakdown_tol (|alpha| + beta_j) has reached an invariant subspace; its step-j
    update is applied and it is frozen.  b = 0 columns return 0."""
    b = np.asarray(b, dtype=np.float64)
    if b.ndim == 1:
        b = b[:, None]
    shifts = np.asarray(shifts, dtype=np.float64)
    if np.any(shifts < 0):
        raise ValueError("shifts must be nonnegative")
    n, t = b.shape
    nq = shifts.shape[0]
    beta1 = np.linalg.norm(b, axis=0)
    active = beta1 > 0
    x = np.zeros((nq, n, t))
    phibar = np.tile(beta1, (nq, 1))
    if not np.any(active):
        return MsminresResult(x, phibar, beta1, 0, 0, True)
    v = np.where(active[None, :], b / np.where(active, beta1, 1.0)[None, :], 0.0)
    v_prev = np.zeros_like(v)
    beta = np.zeros(t)
    c1 = np.ones((nq, t)); s1 = np.zeros((nq, t))
    c2 = np.ones((nq, t)); s2 = np.zeros((nq, t))
    d1 = np.zeros((nq, n, t)); d2 = np.zeros((nq, n, t))
    iters = 0
    mvms = 0
    converged = False
    for j in range(1, max_iters + 1):
        p = mvm(v)
        mvms += 1
        alpha = np.sum(v * p, axis=0)
        p = p - alpha[None, :] * v - beta[None, :] * v_prev
        beta_next = np.linalg.norm(p, axis=0)
        for q in range(nq):
            a = alpha + shifts[q]
            eps = s2[q] * beta
            delta_p = c2[q] * beta
            delta = c1[q] * delta_p + s1[q] * a
            gbar = -s1[q] * delta_p + c1[q] * a
            gamma = np.hypot(gbar, beta_next)
            gamma_safe = np.where(gamma > 0, gamma, 1.0)
            c = gbar / gamma_safe
            s = beta_next / gamma_safe
            phi = c * phibar[q]
            d = (v - delta[None, :] * d1[q] - eps[None, :] * d2[q]) / gamma_safe[None, :]
            upd = active & (gamma > 0)
            x[q] = x[q] + np.where(upd[None, :], phi[None, :] * d, 0.0)
            phibar[q] = np.where(upd, -s * phibar[q], phibar[q])
            d2[q] = d1[q]; d1[q] = d
            c2[q] = c1[q]; s2[q] = s1[q]
            c1[q] = c; s1[q] = s
        iters = j
        broke = active & (beta_next <= breakdown_tol * (np.abs(alpha) + beta))
        active = active & ~broke
        relres = np.abs(phibar) / np.where(beta1 > 0, beta1, 1.0)[None, :]
        relres = np.where(active[None, :], relres, 0.0)
        if not np.any(active) or (tol > 0 and float(np.max(relres)) <= tol):
            converged = True
            break
        v_prev = v
        v = np.where(active[None, :], p / np.where(beta_next > 0, beta_next, 1.0)[None, :], 0.0)
        beta = beta_next
    if tol > 0 and not converged:
        converged = False
    elif tol == 0:
        converged = True
    return MsminresResult(x, phibar, beta1, iters, mvms, converged)


# --------------------------------------------------------------------------------------------
# L3 -- the CIQ driver (eq. contour_integral_quad; Property 1)
# --------------------------------------------------------------------------------------------

@dataclasses.dataclass
class CiqResult:
    out: np.ndarray
    t: np.ndarray
    w: np.ndarray
    lambda_min: float
    lambda_max: float
    iters: int
    mvms: int
    converged: bool
    solve: MsminresResult


def ciq(op, b: np.ndarray, q: int = 8, max_iters: int = 400, tol: float = 1e-4, mode: str = "sqrt",
        lanczos_start: np.ndarray | None = None, lanczos_iters: int = 10,
        rule: tuple | None = None, spectrum: tuple | None = None) -> CiqResult:
    """msMINRES-CIQ:

        K^{-1/2} b ~ sum_q w_q (t_q I + K)^{-1} b              (invsqrt / whiten)
        K^{ 1/2} b ~ K sum_q w_q (t_q I + K)^{-1} b            (sqrt; K applied AFTER, reading G2)

    lambda_min/lambda_max from ``estimate_spectrum`` on ``lanczos_start`` (lower bound = the
    operator's sigma2, reading G6) unless ``spectrum`` or an explicit ``rule`` = (t, w) is given.
    MVMs: lanczos_iters + J (+1 for sqrt)."""
    b = np.asarray(b, dtype=np.float64)
    squeeze = b.ndim == 1
    if squeeze:
        b = b[:, None]
    mv0 = op.mvm_count
    if rule is not None:
        t_q, w_q = (np.asarray(rule[0], dtype=np.float64), np.asarray(rule[1], dtype=np.float64))
        lmin = lmax = float("nan")
    else:
        if spectrum is not None:
            lmin, lmax = spectrum
        else:
            if lanczos_start is None:
                raise ValueError("need lanczos_start, spectrum or rule")
            lmin, lmax, _, _ = estimate_spectrum(op.mvm, lanczos_start, lanczos_iters,
                                                 lower_bound=getattr(op, "sigma2", 0.0))
        t_q, w_q = hht_rule(lmin, lmax, q)
    res = msminres(op.mvm, b, t_q, max_iters, tol)
    y = np.einsum("q,qnt->nt", w_q, res.x)
    if mode == "sqrt":
        out = op.mvm(y)
    elif mode in ("invsqrt", "whiten"):
        out = y
    else:
        raise ValueError(f"unknown mode {mode!r}")
    if squeeze:
        out = out[:, 0]
    return CiqResult(out, t_q, w_q, lmin, lmax, res.iters, op.mvm_count - mv0, res.converged, res)


# --------------------------------------------------------------------------------------------
# Preconditioning (App. A)
# --------------------------------------------------------------------------------------------

def pivoted_cholesky(op, rank: int, rel_tol: float = 1e-12) -> np.ndarray:
    """Partial pivoted Cholesky of the kernel part k(X, X) (Harbrecht et al.):
    at each step pick the largest remaining diagonal residual (lowest index on ties, reading G18),
    append the normalised residual column.  Stops at ``rank`` or when the max residual drops
    below rel_tol times the initial max.  Returns L (n x m), m <= rank."""
    n = op.n
    d = np.asarray(op.kernel_diag(), dtype=np.float64).copy()
    d0 = float(np.max(d))
    cols = []
    for m in range(rank):
        i = int(np.argmax(d))
        if d[i] <= rel_tol * d0:
            break
        col = np.asarray(op.kernel_column(i), dtype=np.float64).copy()
        for lc in cols:
            col -= lc * lc[i]
        lcol = col / math.sqrt(d[i])
        cols.append(lcol)
        d = d - lcol * lcol
        d[i] = 0.0
    return np.stack(cols, axis=1) if cols else np.zeros((n, 0))


class LowRankPlusDiag:
    """P = L L^T + sigma2 I with its exact half powers through the thin SVD of L
    (S:430-433): with L = U S W^T,
        P^p v = U diag((s^2 + sigma2)^p) U^T v + sigma2^p (v - U U^T v)."""

    def __init__(self, lfac: np.ndarray, sigma2: float):
        if not sigma2 > 0:
            raise ValueError("preconditioner sigma2 must be > 0")
        self.l = np.asarray(lfac, dtype=np.float64)
        self.sigma2 = float(sigma2)
        if self.l.shape[1] > 0:
            u, s, _ = np.linalg.svd(self.l, full_matrices=False)
            self.u, self.s = u, s
        else:
            self.u, self.s = np.zeros((self.l.shape[0], 0)), np.zeros(0)

    def power(self, v: np.ndarray, p: float) -> np.ndarray:
        v = np.asarray(v, dtype=np.float64)
        utv = self.u.T @ v
        lam = (self.s ** 2 + self.sigma2) ** p
        lam = lam.reshape((-1,) + (1,) * (v.ndim - 1))
        return self.u @ (lam * utv) + self.sigma2 ** p * (v - self.u @ utv)

    def apply(self, v):
        return self.l @ (self.l.T @ v) + self.sigma2 * v

    def dense(self):
        return self.l @ self.l.T + self.sigma2 * np.eye(self.l.shape[0])


class BlockJacobi:
    """P = blockdiag(K_11, K_22, ...): the diagonal blocks (size ``block``, the last one ragged) of
    the operator K itself -- a preconditioner with cheap solves and MVMs (the two requirements of
    P:71-74) whose square root has no closed form in the algorithm (the library computes P^{1/2} b
    by CIQ on P, "nested CIQ").  Here its powers are evaluated exactly, block by block, from
    numpy's eigh (the oracle's route is the explicit symmetric form of App. A)."""

    def __init__(self, op, block: int):
        self.n = op.n
        self.block = int(block)
        self.blocks = []
        for i0 in range(0, self.n, self.block):
            i1 = min(self.n, i0 + self.block)
            kb = np.stack([op.kernel_column(j)[i0:i1] for j in range(i0, i1)], axis=1)
            kb = kb + op.sigma2 * np.eye(i1 - i0)
            lam, u = np.linalg.eigh(0.5 * (kb + kb.T))
            self.blocks.append((i0, i1, lam, u))

    def power(self, v: np.ndarray, p: float) -> np.ndarray:
        v = np.asarray(v, dtype=np.float64)
        out = np.empty_like(v)
        for i0, i1, lam, u in self.blocks:
            out[i0:i1] = u @ ((lam ** p).reshape((-1,) + (1,) * (v.ndim - 1)) * (u.T @ v[i0:i1]))
        return out

    def apply(self, v):
        return self.power(v, 1.0)

    def dense(self):
        d = np.zeros((self.n, self.n))
        for i0, i1, lam, u in self.blocks:
            d[i0:i1, i0:i1] = (u * lam) @ u.T
        return d

    def spectrum(self):
        return min(b[2][0] for b in self.blocks), max(b[2][-1] for b in self.blocks)


def precond_ciq(op, pre, b: np.ndarray, q: int = 8, max_iters: int = 400,
                tol: float = 1e-4, mode: str = "whiten", lanczos_start=None, lanczos_iters: int = 10,
                rule: tuple | None = None, spectrum: tuple | None = None, lower_bound: float = 1.0) -> CiqResult:
    """Preconditioned msMINRES-CIQ, oracle route = the explicit symmetric form of App. A:

        M = P^{-1/2} K P^{-1/2}                                    (P:8)
        R' b = P^{-1/2} M^{-1/2} P^{-1/2} (P^{1/2} b) = P^{-1/2} M^{-1/2} b   (eq. precond_sqrt_inverse)
        R  b = K R' b                                              (eq. precond_sqrt)

    M^{-1/2} b is computed by ``ciq`` (invsqrt) on the operator M; lambda estimation runs on M with
    the rigorous bound lambda_min(M) >= 1 when P comes from a pivoted Cholesky of k(X,X) with
    sigma2_P = sigma2 (reading G6/G13/G14; ``lower_bound`` = 0 for other P, e.g. BlockJacobi).
    ``pre`` provides power(v, p) (LowRankPlusDiag, BlockJacobi).
    mode 'whiten'/'invsqrt' -> R'b, 'sqrt' -> R b."""

    class _M:
        n = op.n
        mvm_count = 0
        sigma2 = 0.0

        def mvm(self_inner, v):
            self_inner.mvm_count += 1
            return pre.power(op.mvm(pre.power(v, -0.5)), -0.5)

    m = _M()
    if rule is None and spectrum is None:
        if lanczos_start is None:
            raise ValueError("need lanczos_start, spectrum or rule")
        lmin, lmax, _, _ = estimate_spectrum(m.mvm, lanczos_start, lanczos_iters, lower_bound=lower_bound)
        spectrum = (lmin, lmax)
    res = ciq(m, b, q=q, max_iters=max_iters, tol=tol, mode="invsqrt", rule=rule, spectrum=spectrum)
    rprime_b = pre.power(res.out, -0.5)
    out = op.mvm(rprime_b) if mode == "sqrt" else rprime_b
    return CiqResult(out, res.t, res.w, res.lambda_min, res.lambda_max, res.iters, res.mvms,
                     res.converged, res.solve)


# --------------------------------------------------------------------------------------------
# Backward pass: vector-Jacobian product of K^{-1/2} b
# --------------------------------------------------------------------------------------------

def ciq_vjp(op, b: np.ndarray, v: np.ndarray, rule: tuple, max_iters: int = 400, tol: float = 0.0) -> np.ndarray:
    """Eq. ciq_deriv: back-propagating through each term of the quadrature
    K^{-1/2} b ~ sum_q w_q (t_q I + K)^{-1} b gives

        v^T (d K^{-1/2} b / d K) ~ -1/2 sum_q w_q (t_q I + K)^{-1} (v b^T + b v^T) (t_q I + K)^{-1}
                                 = -1/2 sum_q w_q (x_q(v) x_q(b)^T + x_q(b) x_q(v)^T)

    with x_q(u) = (t_q I + K)^{-1} u the shifted solves of msMINRES: the forward pass supplies
    x_q(b), "another call to the msMINRES algorithm" supplies x_q(v).  Columns of b / v
    are independent problems whose gradients add (reading G15): returns the dense N x N matrix
    G = sum_c -1/2 sum_q w_q (x_q(v_c) x_q(b_c)^T + x_q(b_c) x_q(v_c)^T)."""
    t_q = np.asarray(rule[0], dtype=np.float64)
    w_q = np.asarray(rule[1], dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    if b.ndim == 1:
        b, v = b[:, None], v[:, None]
    xb = msminres(op.mvm, b, t_q, max_iters, tol).x      # (Q, n, t)
    xv = msminres(op.mvm, v, t_q, max_iters, tol).x
    g = np.einsum("q,qic,qjc->ij", w_q, xv, xb)
    return -0.5 * (g + g.T)



def kernel_lengthscale_derivative(xa: np.ndarray, xb: np.ndarray, kind: str, lengthscale: float,
                                  outputscale: float) -> np.ndarray:
    """d k(x_a, x_b) / d l for an isotropic lengthscale l, differentiating the textbook forms of
    reading G11 with r = ||x_a - x_b|| / l (so dr/dl = -r/l):

    RBF        o^2 exp(-r^2/2) r^2 / l
    Matern-5/2 o^2 exp(-a) a^2 (1 + a) / (3 l),   a = sqrt5 r
    Matern-3/2 o^2 exp(-a) a^2 / l,               a = sqrt3 r"""
    ls = float(lengthscale)
    a = np.asarray(xa, dtype=np.float64) / ls
    b = np.asarray(xb, dtype=np.float64) / ls
    r2 = np.zeros((a.shape[0], b.shape[0]))
    for k in range(a.shape[1]):
        diff = a[:, k, None] - b[None, :, k]
        r2 += diff * diff
    if kind == "rbf":
        dk = np.exp(-0.5 * r2) * r2
    elif kind == "matern52":
        aa = math.sqrt(5.0) * np.sqrt(r2)
        dk = np.exp(-aa) * aa * aa * (1.0 + aa) / 3.0
    elif kind == "matern32":
        aa = math.sqrt(3.0) * np.sqrt(r2)
        dk = np.exp(-aa) * aa * aa
    else:
        raise ValueError(f"unknown kernel kind {kind!r}")
    return outputscale * dk / ls


def ciq_hyper_grad(op, b: np.ndarray, v: np.ndarray, rule: tuple, max_iters: int = 400, tol: float = 0.0) -> np.ndarray:
    """Gradient of L = sum_c v_c^T (K^{-1/2} b_c)_CIQ with respect to the kernel hyper-parameters
    (lengthscale l, outputscale o^2, noise sigma^2 of K = o^2 k(X, X; l) + sigma^2 I), by the chain
    rule through eq. ciq_deriv: dL/dtheta = sum_ij G_ij dK_ij/dtheta with G = dL/dK
    from ``ciq_vjp`` and

        dK/dl      = ``kernel_lengthscale_derivative``   (isotropic l)
        dK/d(o^2)  = k(X, X) / o^2  (without sigma^2)
        dK/dsigma2 = I

    ("the derivative ... can be computed with the same quadrature": the training use
    of CIQ whose O(J mvm(K)) cost the paper stresses).  Returns [dL/dl, dL/d(o^2), dL/dsigma2]."""
    if not isinstance(op, KernelOperator):
        raise ValueError("hyper-parameter gradient needs a kernel operator")
    g = ciq_vjp(op, b, v, rule, max_iters, tol)
    dk_dl = kernel_lengthscale_derivative(op.x, op.x, op.kind, op.lengthscale, op.outputscale)
    k_kern = kernel_entries(op.x, op.x, op.kind, op.lengthscale, op.outputscale)
    return np.array([np.sum(g * dk_dl), np.sum(g * k_kern) / op.outputscale, np.trace(g)])


# --------------------------------------------------------------------------------------------
# Thompson sampling (SS5.2, eq. thompson_sample)
# --------------------------------------------------------------------------------------------

class PosteriorOperator:
    """COV*(X*) + jitter I, the GP posterior covariance at the candidates X* given noisy training
    data (X, y) ("posterior mean and covariance of the Gaussian process at the candidate
    set"), from the textbook conditioning formulas:

        mu*  = K*x (Kxx + noise I)^{-1} y
        COV* = K** - K*x (Kxx + noise I)^{-1} Kx*

    K** is applied matrix-free (a ``KernelOperator`` on X* whose ``sigma2`` is the jitter); the
    training block is factorised densely once (Cholesky, n small: the paper's BO runs have <= 100
    evaluations).  ``mvm`` is the definition written out: K** v - K*x solve(Kxx + noise I,
    Kx* v).  ``sigma2`` = jitter is the rigorous lower bound on lambda_min (COV* is PSD; reading G6)."""

    def __init__(self, x_cand, x_train, y_train, kind: str, lengthscale=1.0, outputscale: float = 1.0,
                 noise: float = 1e-2, jitter: float = 1e-4):
        self.kss = KernelOperator(x_cand, kind, lengthscale, outputscale, jitter)
        self.n = self.kss.n
        self.sigma2 = float(jitter)
        self.noise = float(noise)
        xt = np.asarray(x_train, dtype=np.float64)
        self.kxx = kernel_entries(xt, xt, kind, lengthscale, outputscale) + self.noise * np.eye(xt.shape[0])
        self.kxs = kernel_entries(xt, self.kss.x, kind, lengthscale, outputscale)      # m x N
        self.cho = scipy.linalg.cho_factor(self.kxx, lower=True)
        self.mean = self.kxs.T @ scipy.linalg.cho_solve(self.cho, np.asarray(y_train, dtype=np.float64))
        self.mvm_count = 0

    def mvm(self, v: np.ndarray) -> np.ndarray:
        self.mvm_count += 1
        v = np.asarray(v, dtype=np.float64)
        return self.kss.mvm(v) - self.kxs.T @ scipy.linalg.cho_solve(self.cho, self.kxs @ v)

    def mvm_rows(self, rows: np.ndarray, v: np.ndarray) -> np.ndarray:
        v = np.asarray(v, dtype=np.float64)
        rows = np.asarray(rows)
        return self.kss.mvm_rows(rows, v) - self.kxs[:, rows].T @ scipy.linalg.cho_solve(self.cho, self.kxs @ v)

    def dense(self) -> np.ndarray:
        return self.kss.dense() - self.kxs.T @ scipy.linalg.cho_solve(self.cho, self.kxs)

    def kernel_column(self, j: int) -> np.ndarray:
        """Column j of COV* without the jitter (what ``pivoted_cholesky`` factors)."""
        return self.kss.kernel_column(j) - self.kxs.T @ scipy.linalg.cho_solve(self.cho, self.kxs[:, j])

    def kernel_diag(self) -> np.ndarray:
        return self.kss.kernel_diag() - np.sum(self.kxs * scipy.linalg.cho_solve(self.cho, self.kxs), axis=0)


def thompson_step(post: PosteriorOperator, eps: np.ndarray, q: int = 8, max_iters: int = 400, tol: float = 1e-4,
                  lanczos_start: np.ndarray | None = None, rule: tuple | None = None):
    """Eq. thompson_sample: x~ = argmin( mu*(X*) + COV*(X*)^{1/2} eps ), one candidate
    index per column of eps (each column one posterior sample), COV*^{1/2} eps by msMINRES-CIQ
    (``ciq`` in sqrt mode on ``post``); ties broken by the lowest index.
    Returns (indices, samples, CiqResult)."""
    eps = np.asarray(eps, dtype=np.float64)
    if eps.ndim == 1:
        eps = eps[:, None]
    r = ciq(post, eps, q=q, max_iters=max_iters, tol=tol, mode="sqrt", lanczos_start=lanczos_start, rule=rule)
    samples = post.mean[:, None] + r.out
    return np.argmin(samples, axis=0), samples, r
