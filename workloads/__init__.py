"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no kernel MVM, no Lanczos, no quadrature, no
msMINRES).  It only draws the random inputs the method consumes, with the shapes and value
distributions of the paper's workloads:

* points: U[0,1]^d, as for BO candidate sets (§5.2) and inducing points;
* right-hand sides: N(0,1) columns (posterior-sample draws epsilon);
* the Lanczos start block for lambda estimation (reading G5 in DESIGN.md);
* dense test spectra lambda_t = 1/sqrt(t), 1/t, 1/t^2, exp(-t).

All draws are made in float64 with a CPU ``torch.Generator`` (counter-free, seed-exact, the same
on every host) and cast ONCE to float32; the oracle consumes the same float32 arrays upcast to
float64, the CUDA path consumes them as float32.

The dense RBF matrix of config C2 is an *input* of the dense path (the caller hands the library a
precomputed K); its assembly here is input generation, written from the kernel's textbook
definition (reading G11) and is never used by the matrix-free path on either side.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

# Seeds fixed per role (SURVEY.md §8(d) "Seeds").
SEED_POINTS = 0
SEED_RHS = 1
SEED_LANCZOS = 2
SEED_MINIBATCH = 3
SEED_TRAIN = 4


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def points(n: int, d: int, seed: int = SEED_POINTS) -> np.ndarray:
    """n x d points ~ U[0,1]^d, drawn in fp64, returned as float32 (C-contiguous)."""
    x = torch.rand((n, d), generator=_gen(seed), dtype=torch.float64)
    return x.to(torch.float32).numpy().copy()


def rhs(n: int, t: int, seed: int = SEED_RHS) -> np.ndarray:
    """n x t right-hand sides ~ N(0,1), float32 row-major (column c is one RHS b_c)."""
    b = torch.randn((n, t), generator=_gen(seed), dtype=torch.float64)
    return b.to(torch.float32).numpy().copy()


def lanczos_start(n: int, t_lambda: int = 16, seed: int = SEED_LANCZOS) -> np.ndarray:
    """n x t_lambda Lanczos start block for the lambda estimator, ~ N(0,1), float32."""
    s = torch.randn((n, t_lambda), generator=_gen(seed), dtype=torch.float64)
    return s.to(torch.float32).numpy().copy()


def random_orthogonal(n: int, seed: int) -> np.ndarray:
    """Haar-ish random orthogonal matrix (QR of a Gaussian, sign-fixed), float64."""
    a = torch.randn((n, n), generator=_gen(seed), dtype=torch.float64).numpy()
    q, r = np.linalg.qr(a)
    q = q * np.sign(np.diag(r))[None, :]
    return q


def spectrum_values(n: int, decay: str) -> np.ndarray:
    """Eigenvalues lambda_t, t=1..n, of the paper's synthetic spectra."""
    t = np.arange(1, n + 1, dtype=np.float64)
    if decay == "inv_sqrt":
        return 1.0 / np.sqrt(t)
    if decay == "inv_linear":
        return 1.0 / t
    if decay == "inv_square":
        return 1.0 / t ** 2
    if decay == "exponential":
        return np.exp(-(t - 1.0))
    raise ValueError(f"unknown decay {decay!r}")


def spectrum_matrix(n: int, decay: str, seed: int = 7) -> np.ndarray:
    """Dense SPD K = Q diag(lambda) Q^T with a seeded random orthogonal Q (fp64)."""
    q = random_orthogonal(n, seed)
    lam = spectrum_values(n, decay)
    k = (q * lam[None, :]) @ q.T
    return 0.5 * (k + k.T)


def dense_rbf_input(x: np.ndarray, lengthscale: float, outputscale: float = 1.0) -> np.ndarray:
    """Dense RBF matrix o^2 exp(-|x_i-x_j|^2 / (2 l^2)) assembled in fp64 from float32 points,
    returned as float32 -- the precomputed-K INPUT of the dense path (config C2)."""
    xd = x.astype(np.float64) / lengthscale
    n = xd.shape[0]
    out = np.empty((n, n), dtype=np.float32)
    blk = 1024
    for i0 in range(0, n, blk):
        diff = xd[i0:i0 + blk, None, :] - xd[None, :, :]
        out[i0:i0 + blk] = (outputscale * np.exp(-0.5 * np.sum(diff * diff, axis=-1))).astype(np.float32)
    return out


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json config, with the recipe stated in DESIGN.md."""
    name: str
    n: int
    d: int
    kind: str            # "rbf" | "matern52" | "matern32" | "dense"
    lengthscale: float
    outputscale: float
    sigma2: float        # noise / jitter added to the diagonal
    t: int               # number of right-hand sides
    q: int               # quadrature points
    mode: str            # "sqrt" | "invsqrt" | "whiten"
    max_iters: int
    tol: float
    precond_rank: int = 0
    rhs_kind: str = "normal"   # "normal" | "kzx" (C4: B = K_{Z, X_b})


CONFIGS = {
    "C1": Config("C1", 256, 3, "rbf", 0.2, 1.0, 3e-2, 1, 8, "sqrt", 100, 0.0),
    "C2": Config("C2", 10_000, 8, "dense", 0.5, 1.0, 0.1, 32, 8, "whiten", 400, 1e-5),
    "C3": Config("C3", 50_000, 6, "rbf", 0.15, 1.0, 0.05, 64, 8, "sqrt", 400, 1e-4),
    "C4": Config("C4", 5_000, 3, "matern52", 0.3, 1.0, 1e-3, 1024, 8, "whiten", 200, 1e-3,
                 precond_rank=200, rhs_kind="kzx"),
    "C5": Config("C5", 200_000, 8, "matern52", 0.25, 1.0, 0.1, 16, 12, "sqrt", 300, 0.0),
}


def scaled(cfg: Config, n: int | None = None, t: int | None = None, **kw) -> Config:
    """A reduced-size copy of a config (same kernel/hyper-parameters), for parity tests."""
    return dataclasses.replace(cfg, n=cfg.n if n is None else n, t=cfg.t if t is None else t, **kw)


def make_inputs(cfg: Config) -> dict:
    """All seeded arrays of one config: points X (n x d), RHS B (n x t), Lanczos start S (n x 16),
    and, for the dense config, the dense input matrix K (n x n float32, WITHOUT the sigma2 diagonal,
    which the operator adds)."""
    x = points(cfg.n, cfg.d)
    if cfg.rhs_kind == "normal":
        b = rhs(cfg.n, cfg.t)
    else:
        b = None  # built by the caller from the kernel (C4: K_{Z,X_b}); see kzx_minibatch
    out = {"X": x, "B": b, "S": lanczos_start(cfg.n, 16)}
    if cfg.kind == "dense":
        out["K"] = dense_rbf_input(x, cfg.lengthscale, cfg.outputscale)
    return out


def minibatch_points(t: int, d: int, seed: int = SEED_MINIBATCH) -> np.ndarray:
    """C4's minibatch X_b ~ U[0,1]^d."""
    return points(t, d, seed)


def kzx_input(z: np.ndarray, xb: np.ndarray, kind: str, lengthscale: float,
              outputscale: float = 1.0) -> np.ndarray:
    """C4's right-hand-side block B = K_{Z, X_b} (M x t, float32): the whitened-SVGP RHS k_Zx
    (reading G17), assembled in fp64 from the textbook kernel forms (reading G11).
    Input generation only."""
    zd = z.astype(np.float64) / lengthscale
    xd = xb.astype(np.float64) / lengthscale
    diff = zd[:, None, :] - xd[None, :, :]
    r = np.sqrt(np.sum(diff * diff, axis=-1))
    if kind == "rbf":
        k = np.exp(-0.5 * r * r)
    elif kind == "matern52":
        s5 = math.sqrt(5.0) * r
        k = (1.0 + s5 + s5 * s5 / 3.0) * np.exp(-s5)
    elif kind == "matern32":
        s3 = math.sqrt(3.0) * r
        k = (1.0 + s3) * np.exp(-s3)
    else:
        raise ValueError(kind)
    return (outputscale * k).astype(np.float32)


def config_inputs(cfg: Config) -> dict:
    """make_inputs plus the C4 RHS block when rhs_kind == 'kzx'."""
    inp = make_inputs(cfg)
    if cfg.rhs_kind == "kzx":
        xb = minibatch_points(cfg.t, cfg.d)
        inp["B"] = kzx_input(inp["X"], xb, cfg.kind, cfg.lengthscale, cfg.outputscale)
    return inp


def kappa_hint(lambda_max: float, sigma2: float) -> float:
    return lambda_max / sigma2 if sigma2 > 0 else math.inf


# ---- Thompson-sampling workload ----

_H6_ALPHA = (1.0, 1.2, 3.0, 3.2)
_H6_A = ((10, 3, 17, 3.5, 1.7, 8), (0.05, 10, 17, 0.1, 8, 14), (3, 3.5, 1.7, 10, 17, 8), (17, 8, 0.05, 10, 0.1, 14))
_H6_P = ((1312, 1696, 5569, 124, 8283, 5886), (2329, 4135, 8307, 3736, 1004, 9991),
         (2348, 1451, 3522, 2883, 3047, 6650), (4047, 8828, 8732, 5743, 1091, 381))


def hartmann6(x: np.ndarray) -> np.ndarray:
    """The 6-d Hartmann test function of the paper's BO experiment (its standard published
    form): f(x) = -sum_i alpha_i exp(-sum_j A_ij (x_j - P_ij)^2) on [0,1]^6, fp64."""
    x = np.asarray(x, dtype=np.float64)
    f = np.zeros(x.shape[0])
    for i in range(4):
        a = np.asarray(_H6_A[i], dtype=np.float64)
        p = np.asarray(_H6_P[i], dtype=np.float64) * 1e-4
        f -= _H6_ALPHA[i] * np.exp(-np.sum(a * (x - p) ** 2, axis=1))
    return f


@dataclasses.dataclass(frozen=True)
class ThompsonConfig:
    """Thompson-sampling step on Hartmann-6: n candidates U[0,1]^6 (the
    candidate set), m evaluated training points U[0,1]^6 with standardised Hartmann values,
    t posterior samples.  Kernel hyper-parameters are those of C3 (the hot path's shape); `noise`
    is the training-data noise, `jitter` the diagonal added to COV* (C3's sigma2)."""
    name: str
    n: int
    m: int
    t: int
    kind: str = "rbf"
    lengthscale: float = 0.15
    outputscale: float = 1.0
    noise: float = 1e-3
    jitter: float = 0.05
    q: int = 8
    max_iters: int = 400
    tol: float = 1e-4


THOMPSON = {
    "T1": ThompsonConfig("T1", 50_000, 100, 64),      # C3's shape: 50k candidates, 100 evaluations
}


def thompson_inputs(cfg: ThompsonConfig) -> dict:
    """Candidates Xs (n x 6), training Xt (m x 6), y (m, standardised Hartmann-6 values, fp64),
    samples' eps (n x t, N(0,1)), Lanczos start S (n x 16); float32 except y."""
    xs = points(cfg.n, 6)
    xt = points(cfg.m, 6, seed=SEED_TRAIN)
    f = hartmann6(xt.astype(np.float64))
    y = (f - f.mean()) / f.std()
    return {"Xs": xs, "Xt": xt, "y": y.astype(np.float32), "eps": rhs(cfg.n, cfg.t), "S": lanczos_start(cfg.n, 16)}
