"""Thin ctypes binding of libciq.so (include/ciq.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only converts numpy
arrays / torch tensors to pointers + leading dimensions and forwards the call.  There is no CPU
fallback: importing fails loudly when libciq.so is missing.

Names mirror the C ABI: ``ciq_init``, ``ciq_apply``, ``ciq_matvec``, ``ciq_free``,
``ciq_quadrature_rule``, ``ciq_tridiag_extremes``, ``ciq_params_default``, ``ciq_shard_rows``.
``CIQ`` is a small RAII wrapper around a context.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int32, c_int64, c_uint64, c_void_p

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CIQ_LIB overrides the library path (A/B experiments between builds only)
LIB_PATH = os.environ.get("CIQ_LIB") or os.path.join(_HERE, "libciq.so")

CIQ_MAX_Q = 64

# ciq_status
CIQ_OK = 0
CIQ_NOT_CONVERGED = 1
CIQ_ERR_INVALID_ARG = -1
CIQ_ERR_DIM = -2
CIQ_ERR_NOT_PD = -3
CIQ_ERR_ELLIPTIC = -4
CIQ_ERR_CUDA = -5
CIQ_ERR_NCCL = -6
CIQ_ERR_OOM = -7
# ciq_op_kind
OP_KINDS = {"dense": 0, "rbf": 1, "matern52": 2, "matern32": 3, "sparse": 4}
# ciq_mode
MODES = {"sqrt": 0, "invsqrt": 1, "whiten": 2}
# ciq_mvm_impl
MVM_IMPLS = {"auto": 0, "simt": 1, "tc": 2, "sym": 3}


class CiqOperator(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("n", c_int64), ("K", c_void_p), ("ldk", c_int64), ("X", c_void_p),
                ("d", c_int64), ("ldx", c_int64), ("lengthscale", POINTER(c_float)), ("ard", c_int32),
                ("outputscale", c_float), ("diag", c_float), ("csr_indptr", c_void_p), ("csr_indices", c_void_p),
                ("csr_values", c_void_p), ("nnz", c_int64)]


class CiqPrecond(ctypes.Structure):
    _fields_ = [("L", c_void_p), ("rank", c_int64), ("ldl", c_int64), ("sigma2", c_float), ("matrix_free", c_int32),
                ("kind", c_int32), ("block", c_int64)]


class CiqComm(ctypes.Structure):
    _fields_ = [("rank", c_int32), ("world", c_int32), ("nccl_unique_id", c_void_p), ("loopback_group", c_void_p)]


class CiqParams(ctypes.Structure):
    _fields_ = [("Q", c_int32), ("max_iters", c_int32), ("tol", c_double), ("lanczos_iters", c_int32),
                ("lanczos_cols", c_int32), ("lambda_min", c_double), ("lambda_max", c_double),
                ("t", POINTER(c_double)), ("w", POINTER(c_double)), ("lanczos_start", c_void_p),
                ("ld_start", c_int64), ("seed", c_uint64), ("mode", c_int32), ("mvm_impl", c_int32),
                ("poll_every", c_int32), ("breakdown_tol", c_double), ("profile_kernels", c_int32),
                ("lanczos_reuse", c_int32), ("keep_shift_solutions", c_int32), ("shift_solutions", c_void_p),
                ("fp64", c_int32), ("stored_basis", c_int32), ("mvm_relax", c_int32)]


class CiqInfo(ctypes.Structure):
    _fields_ = [("iters", c_int32), ("mvms", c_int32), ("converged", c_int32), ("rotated", c_int32),
                ("breakdown_cols", c_int32), ("Q", c_int32), ("lambda_min", c_double), ("lambda_max", c_double),
                ("ritz_min", c_double), ("ritz_max", c_double), ("max_rel_residual", c_double),
                ("t", c_double * CIQ_MAX_Q), ("w", c_double * CIQ_MAX_Q), ("ms_total", c_float),
                ("ms_lambda", c_float), ("ms_loop", c_float), ("ms_final", c_float), ("kernel_launches", c_int64),
                ("ms_mvm", c_float), ("mvm_timed", c_int32), ("ms_update", c_float), ("update_timed", c_int32),
                ("mvm_impl_used", c_int32), ("mvm_splits", c_int32), ("fp64_route", c_int32),
                ("nested_p_mvms", c_int32), ("nested_iters", c_int32), ("overlap", c_int32),
                ("relaxed_from", c_int32), ("relaxed2_from", c_int32)]

    def as_dict(self) -> dict:
        q = self.Q
        return {"iters": self.iters, "mvms": self.mvms, "converged": bool(self.converged),
                "rotated": bool(self.rotated), "breakdown_cols": self.breakdown_cols, "Q": q,
                "lambda_min": self.lambda_min, "lambda_max": self.lambda_max, "ritz_min": self.ritz_min,
                "ritz_max": self.ritz_max, "max_rel_residual": self.max_rel_residual,
                "t": list(self.t[:q]), "w": list(self.w[:q]), "ms_total": self.ms_total,
                "ms_lambda": self.ms_lambda, "ms_loop": self.ms_loop, "ms_final": self.ms_final,
                "kernel_launches": self.kernel_launches, "ms_mvm": self.ms_mvm, "mvm_timed": self.mvm_timed,
                "ms_update": self.ms_update, "update_timed": self.update_timed,
                "mvm_impl_used": {1: "simt", 2: "tc", 3: "sym", 4: "fp64_tc"}.get(self.mvm_impl_used, "none"), "mvm_splits": self.mvm_splits,
                "fp64_route": bool(self.fp64_route), "nested_p_mvms": self.nested_p_mvms,
                "nested_iters": self.nested_iters, "overlap": bool(self.overlap),
                "relaxed_from": self.relaxed_from, "relaxed2_from": self.relaxed2_from}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2006_11267_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    ctx_p = c_void_p
    lib.ciq_params_default.argtypes = [POINTER(CiqParams)]
    lib.ciq_params_default.restype = None
    lib.ciq_init.argtypes = [POINTER(ctx_p), POINTER(CiqOperator), POINTER(CiqPrecond), POINTER(CiqComm), c_void_p]
    lib.ciq_init.restype = c_int32
    lib.ciq_apply.argtypes = [ctx_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, POINTER(CiqParams),
                              POINTER(CiqInfo)]
    lib.ciq_apply.restype = c_int32
    lib.ciq_matvec.argtypes = [ctx_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_int32]
    lib.ciq_matvec.restype = c_int32
    lib.ciq_pivoted_cholesky.argtypes = [ctx_p, c_int32, c_void_p, c_int64]
    lib.ciq_pivoted_cholesky.restype = c_int32
    lib.ciq_vjp.argtypes = [ctx_p, c_void_p, c_int64, c_void_p, c_int64, c_int64, POINTER(CiqParams), c_void_p,
                            c_int64, POINTER(CiqInfo)]
    lib.ciq_vjp.restype = c_int32
    lib.ciq_set_posterior.argtypes = [ctx_p, c_void_p, c_int64, c_int64, c_void_p, c_double]
    lib.ciq_set_posterior.restype = c_int32
    lib.ciq_thompson.argtypes = [ctx_p, c_void_p, c_int64, c_int64, POINTER(CiqParams), c_void_p, c_void_p, c_int64,
                                 POINTER(CiqInfo)]
    lib.ciq_thompson.restype = c_int32
    lib.ciq_hyper_grad.argtypes = [ctx_p, c_void_p, c_int64, c_void_p, c_int64, c_int64, POINTER(CiqParams),
                                   POINTER(c_double), POINTER(CiqInfo)]
    lib.ciq_hyper_grad.restype = c_int32
    lib.ciq_free.argtypes = [ctx_p]
    lib.ciq_free.restype = None
    lib.ciq_status_string.argtypes = [c_int32]
    lib.ciq_status_string.restype = c_char_p
    lib.ciq_source_hash.argtypes = []
    lib.ciq_source_hash.restype = c_char_p
    lib.ciq_last_error.argtypes = [ctx_p]
    lib.ciq_last_error.restype = c_char_p
    lib.ciq_shard_rows.argtypes = [c_int64, c_int32, c_int32, POINTER(c_int64), POINTER(c_int64)]
    lib.ciq_shard_rows.restype = None
    lib.ciq_quadrature_rule.argtypes = [c_double, c_double, c_int32, POINTER(c_double), POINTER(c_double)]
    lib.ciq_quadrature_rule.restype = c_int32
    lib.ciq_tridiag_extremes.argtypes = [POINTER(c_double), POINTER(c_double), c_int32, POINTER(c_double),
                                         POINTER(c_double)]
    lib.ciq_tridiag_extremes.restype = c_int32
    lib.ciq_nccl_unique_id.argtypes = [c_void_p]
    lib.ciq_nccl_unique_id.restype = c_int32
    lib.ciq_loopback_group_create.argtypes = [c_int32]
    lib.ciq_loopback_group_create.restype = c_void_p
    lib.ciq_loopback_group_destroy.argtypes = [c_void_p]
    lib.ciq_loopback_group_destroy.restype = None
    return lib


LIB = _load()

EXPORTED = ["ciq_params_default", "ciq_init", "ciq_apply", "ciq_matvec", "ciq_pivoted_cholesky", "ciq_vjp", "ciq_hyper_grad",
            "ciq_set_posterior",
            "ciq_thompson", "ciq_free",
            "ciq_status_string", "ciq_source_hash",
            "ciq_last_error", "ciq_shard_rows", "ciq_quadrature_rule", "ciq_tridiag_extremes",
            "ciq_nccl_unique_id", "ciq_loopback_group_create", "ciq_loopback_group_destroy"]


class CiqError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{LIB.ciq_status_string(status).decode()}: {msg}")
        self.status = status


# ---------------------------------------------------------------------------------------------
# array marshalling
# ---------------------------------------------------------------------------------------------

def _ptr_ld(a, name: str, keepalive: list):
    """(pointer, leading dimension, rows, cols) of a 2-D float32 row-major array (numpy or torch)."""
    if a is None:
        return None, 0, 0, 0
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float32:
                raise TypeError(f"{name} must be float32")
            if a.dim() == 1:
                a = a.unsqueeze(1)
            if a.stride(1) != 1:
                raise ValueError(f"{name} must be row-major (unit column stride)")
            keepalive.append(a)
            return a.data_ptr(), a.stride(0), a.shape[0], a.shape[1]
    except ImportError:  # pragma: no cover
        pass
    arr = np.asarray(a)
    if arr.ndim == 1:
        arr = arr[:, None]
    if arr.dtype != np.float32 or not arr.flags.c_contiguous:
        raise TypeError(f"{name} must be a C-contiguous float32 array")
    keepalive.append(arr)
    return arr.ctypes.data, arr.shape[1], arr.shape[0], arr.shape[1]


def ciq_source_hash() -> str:
    """The source hash compiled into the loaded libciq.so (build.py source_hash())."""
    return LIB.ciq_source_hash().decode()


def ciq_params_default() -> CiqParams:
    p = CiqParams()
    LIB.ciq_params_default(ctypes.byref(p))
    return p


def ciq_shard_rows(n: int, rank: int, world: int) -> tuple[int, int]:
    b, e = c_int64(), c_int64()
    LIB.ciq_shard_rows(n, rank, world, ctypes.byref(b), ctypes.byref(e))
    return b.value, e.value


def ciq_quadrature_rule(lambda_min: float, lambda_max: float, q: int):
    t = (c_double * q)()
    w = (c_double * q)()
    st = LIB.ciq_quadrature_rule(lambda_min, lambda_max, q, t, w)
    if st != CIQ_OK:
        raise CiqError(st, "quadrature rule")
    return np.array(t[:]), np.array(w[:])


def ciq_tridiag_extremes(alpha, beta):
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    b = np.ascontiguousarray(beta, dtype=np.float64)
    lo, hi = c_double(), c_double()
    st = LIB.ciq_tridiag_extremes(a.ctypes.data_as(POINTER(c_double)), b.ctypes.data_as(POINTER(c_double)),
                                  len(a), ctypes.byref(lo), ctypes.byref(hi))
    if st != CIQ_OK:
        raise CiqError(st, "tridiag extremes")
    return lo.value, hi.value


def ciq_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = LIB.ciq_nccl_unique_id(buf)
    if st != CIQ_OK:
        raise CiqError(st, LIB.ciq_last_error(None).decode())
    return buf.raw


class LoopbackGroup:
    """In-process loopback transport for `world` ranks (threads) -- exercises row sharding on one GPU."""

    def __init__(self, world: int):
        self.handle = LIB.ciq_loopback_group_create(int(world))
        self.world = int(world)

    def close(self):
        if self.handle:
            LIB.ciq_loopback_group_destroy(self.handle)
            self.handle = None


def _stream_handle(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:  # pragma: no cover
            pass
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def ciq_init(kind: str, n: int, *, X=None, K=None, lengthscale=1.0, outputscale: float = 1.0, diag: float = 0.0,
             precond_L=None, precond_sigma2: float = 0.0, precond_matrix_free: bool = False, precond_block: int = 0,
             comm: tuple | None = None,
             stream=None):
    """Returns (ctx handle, keepalive list).  comm = (rank, world, unique_id_bytes) for NCCL,
    (rank, world, LoopbackGroup) for the in-process loopback transport, or None."""
    keep: list = []
    op = CiqOperator()
    op.kind = OP_KINDS[kind]
    op.n = int(n)
    if kind == "dense":
        p, ld, r, cc = _ptr_ld(K, "K", keep)
        op.K, op.ldk = p, ld
    elif kind == "sparse":   # K = (indptr int64, indices int32, data float32) of this rank's row block
        for name, arr, dt in (("csr_indptr", K[0], np.int64), ("csr_indices", K[1], np.int32),
                              ("csr_values", K[2], np.float32)):
            if isinstance(arr, np.ndarray):
                a = np.ascontiguousarray(arr, dtype=dt)
                keep.append(a)
                setattr(op, name, a.ctypes.data)
            else:   # torch tensor (device or host), contiguous, of that dtype
                keep.append(arr)
                setattr(op, name, arr.data_ptr())
        op.nnz = int(K[1].shape[0])
    else:
        p, ld, r, cc = _ptr_ld(X, "X", keep)
        op.X, op.ldx, op.d = p, ld, cc
    ls = np.atleast_1d(np.asarray(lengthscale, dtype=np.float32))
    keep.append(ls)
    op.lengthscale = ls.ctypes.data_as(POINTER(c_float))
    op.ard = 1 if ls.size > 1 else 0
    op.outputscale = float(outputscale)
    op.diag = float(diag)
    pc = None
    if precond_block > 0:   # block-Jacobi P (nested CIQ); L is not used
        pc = CiqPrecond()
        pc.kind, pc.block = 1, int(precond_block)
    elif precond_L is not None:
        pc = CiqPrecond()
        p, ld, r, cc = _ptr_ld(precond_L, "precond_L", keep)
        pc.L, pc.ldl, pc.rank, pc.sigma2 = p, ld, cc, float(precond_sigma2)
        pc.matrix_free = 1 if precond_matrix_free else 0
    cm = None
    if comm is not None:
        cm = CiqComm()
        cm.rank, cm.world = int(comm[0]), int(comm[1])
        if isinstance(comm[2], LoopbackGroup):
            cm.loopback_group = comm[2].handle
        else:
            idbuf = ctypes.create_string_buffer(comm[2], 128)
            keep.append(idbuf)
            cm.nccl_unique_id = ctypes.cast(idbuf, c_void_p)
    ctx = c_void_p()
    st = LIB.ciq_init(ctypes.byref(ctx), ctypes.byref(op), ctypes.byref(pc) if pc else None,
                      ctypes.byref(cm) if cm else None, _stream_handle(stream))
    if st != CIQ_OK:
        raise CiqError(st, LIB.ciq_last_error(None).decode())
    return ctx, keep


def ciq_apply(ctx, B, out, params: CiqParams) -> tuple[int, CiqInfo]:
    keep: list = []
    pb, ldb, nb, t = _ptr_ld(B, "B", keep)
    po, ldo, no, to = _ptr_ld(out, "out", keep)
    info = CiqInfo()
    st = LIB.ciq_apply(ctx, pb, ldb, t, po, ldo, ctypes.byref(params), ctypes.byref(info))
    if st not in (CIQ_OK, CIQ_NOT_CONVERGED):
        raise CiqError(st, LIB.ciq_last_error(ctx).decode())
    return st, info


def ciq_vjp(ctx, B, V, G, params: CiqParams) -> tuple[int, CiqInfo]:
    keep: list = []
    pb, ldb, nb, t = _ptr_ld(B, "B", keep)
    pv, ldv, nv, tv = _ptr_ld(V, "V", keep)
    pg, ldg, ng, tg = _ptr_ld(G, "G", keep)
    if tv != t:
        raise CiqError(CIQ_ERR_DIM, "V must have the shape of B")
    info = CiqInfo()
    st = LIB.ciq_vjp(ctx, pb, ldb, pv, ldv, t, ctypes.byref(params), pg, ldg, ctypes.byref(info))
    if st not in (CIQ_OK, CIQ_NOT_CONVERGED):
        raise CiqError(st, LIB.ciq_last_error(ctx).decode())
    return st, info


def ciq_hyper_grad(ctx, B, V, params: CiqParams) -> tuple[int, CiqInfo, np.ndarray]:
    keep: list = []
    pb, ldb, nb, t = _ptr_ld(B, "B", keep)
    pv, ldv, nv, tv = _ptr_ld(V, "V", keep)
    if tv != t:
        raise CiqError(CIQ_ERR_DIM, "V must have the shape of B")
    grad = (c_double * 3)()
    info = CiqInfo()
    st = LIB.ciq_hyper_grad(ctx, pb, ldb, pv, ldv, t, ctypes.byref(params), grad, ctypes.byref(info))
    if st not in (CIQ_OK, CIQ_NOT_CONVERGED):
        raise CiqError(st, LIB.ciq_last_error(ctx).decode())
    return st, info, np.array(grad[:], dtype=np.float64)


def ciq_set_posterior(ctx, Xt, y, noise: float) -> None:
    """COV* + jitter I at the ctx's candidates given training data (Xt, y) (eq. thompson_sample)."""
    keep: list = []
    px, ldx, m, d = _ptr_ld(Xt, "Xt", keep)
    py = None
    if y is not None:
        py, _, my, _ = _ptr_ld(y, "y", keep)
        if my != m:
            raise CiqError(CIQ_ERR_DIM, "y must have one entry per training point")
    st = LIB.ciq_set_posterior(ctx, px, ldx, m, py, float(noise))
    if st != CIQ_OK:
        raise CiqError(st, LIB.ciq_last_error(ctx).decode())


def ciq_thompson(ctx, eps, idx, samples, params: CiqParams) -> tuple[int, CiqInfo]:
    """idx (int64, T entries, numpy or torch, host or device) <- argmin_j (mu* + COV*^{1/2} eps)_j."""
    keep: list = []
    pe, lde, ne, t = _ptr_ld(eps, "eps", keep)
    ps, lds, _, ts = _ptr_ld(samples, "samples", keep)
    if samples is not None and ts != t:
        raise CiqError(CIQ_ERR_DIM, "samples must have the shape of eps")
    try:
        import torch
        is_t = isinstance(idx, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_t = False
    if is_t:
        if idx.dtype != torch.int64 or not idx.is_contiguous() or idx.numel() != t:
            raise TypeError("idx must be a contiguous int64 tensor with T entries")
        pi = idx.data_ptr()
    else:
        if idx.dtype != np.int64 or not idx.flags.c_contiguous or idx.size != t:
            raise TypeError("idx must be a contiguous int64 array with T entries")
        pi = idx.ctypes.data
    info = CiqInfo()
    st = LIB.ciq_thompson(ctx, pe, lde, t, ctypes.byref(params), pi, ps, lds, ctypes.byref(info))
    if st not in (CIQ_OK, CIQ_NOT_CONVERGED):
        raise CiqError(st, LIB.ciq_last_error(ctx).decode())
    return st, info


def ciq_matvec(ctx, V, out, mvm_impl: str = "auto") -> None:
    keep: list = []
    pv, ldv, nv, t = _ptr_ld(V, "V", keep)
    po, ldo, no, to = _ptr_ld(out, "out", keep)
    st = LIB.ciq_matvec(ctx, pv, ldv, t, po, ldo, MVM_IMPLS[mvm_impl])
    if st != CIQ_OK:
        raise CiqError(st, LIB.ciq_last_error(ctx).decode())


def ciq_pivoted_cholesky(ctx, rank: int, out) -> None:
    keep: list = []
    po, ldo, no, ro = _ptr_ld(out, "L", keep)
    st = LIB.ciq_pivoted_cholesky(ctx, int(rank), po, ldo)
    if st != CIQ_OK:
        raise CiqError(st, LIB.ciq_last_error(ctx).decode())


def ciq_free(ctx) -> None:
    LIB.ciq_free(ctx)


def make_params(q: int = 8, max_iters: int = 400, tol: float = 1e-4, mode: str = "sqrt", *, lanczos_iters: int = 10,
                lanczos_cols: int = 16, lanczos_start=None, rule=None, spectrum=None, seed: int = 2,
                mvm_impl: str = "auto", poll_every: int = 6, breakdown_tol: float = 1e-6, profile: bool = False,
                lanczos_reuse: bool = False, shift_solutions=None, keep: list | None = None, fp64: bool = False,
                stored_basis: bool = False, mvm_relax: bool = True):
    """Build a CiqParams; arrays referenced by it are appended to `keep` (caller keeps them alive)."""
    keep = [] if keep is None else keep
    p = ciq_params_default()
    p.Q, p.max_iters, p.tol = int(q), int(max_iters), float(tol)
    p.lanczos_iters, p.lanczos_cols = int(lanczos_iters), int(lanczos_cols)
    p.mode = MODES[mode]
    p.mvm_impl = MVM_IMPLS[mvm_impl]
    p.seed = int(seed)
    p.poll_every = int(poll_every)
    p.breakdown_tol = float(breakdown_tol)
    p.profile_kernels = 1 if profile else 0
    p.lanczos_reuse = 1 if lanczos_reuse else 0
    p.fp64 = 1 if fp64 else 0
    p.stored_basis = 1 if stored_basis else 0
    p.mvm_relax = 1 if mvm_relax else 0
    if shift_solutions is not None:   # Q x rows x T (ld = T): the forward's shifted solves
        p.keep_shift_solutions = 1
        if isinstance(shift_solutions, np.ndarray):
            keep.append(shift_solutions)
            p.shift_solutions = shift_solutions.ctypes.data
        else:
            p.shift_solutions = shift_solutions.data_ptr()
    if lanczos_start is not None:
        ptr, ld, r, c = _ptr_ld(lanczos_start, "lanczos_start", keep)
        p.lanczos_start, p.ld_start = ptr, ld
        p.lanczos_cols = c
    if rule is not None:
        t = np.ascontiguousarray(rule[0], dtype=np.float64)
        w = np.ascontiguousarray(rule[1], dtype=np.float64)
        keep += [t, w]
        p.t = t.ctypes.data_as(POINTER(c_double))
        p.w = w.ctypes.data_as(POINTER(c_double))
        p.Q = len(t)
    if spectrum is not None:
        p.lambda_min, p.lambda_max = float(spectrum[0]), float(spectrum[1])
    return p, keep


class CIQ:
    """RAII wrapper: ``CIQ("rbf", X=..., lengthscale=..., diag=...)``; ``.apply(B, out, ...)``."""

    def __init__(self, kind: str, n: int | None = None, **kw):
        if n is None:
            src = kw.get("X") if kind not in ("dense", "sparse") else kw.get("K")
            n = src.shape[0] if kind != "sparse" else src[0].shape[0] - 1
        self.kind = kind
        self.n = int(n)
        self.ctx, self._keep = ciq_init(kind, self.n, **kw)

    def apply(self, B, out, **kw) -> dict:
        keep: list = []
        params, keep = make_params(keep=keep, **kw)
        st, info = ciq_apply(self.ctx, B, out, params)
        d = info.as_dict()
        d["status"] = st
        return d

    def pivoted_cholesky(self, rank: int, out) -> None:
        ciq_pivoted_cholesky(self.ctx, rank, out)

    def vjp(self, B, V, G, **kw) -> dict:
        """G <- dL/dK for L(K^{-1/2} B) with back-propagated gradient V (eq. ciq_deriv)."""
        keep: list = []
        params, keep = make_params(keep=keep, **kw)
        st, info = ciq_vjp(self.ctx, B, V, G, params)
        d = info.as_dict()
        d["status"] = st
        return d

    def hyper_grad(self, B, V, **kw) -> tuple[np.ndarray, dict]:
        """[dL/dl, dL/d(o^2), dL/d(sigma^2)] for L = sum_c v_c^T (K^{-1/2} b_c) (eq. ciq_deriv)."""
        keep: list = []
        params, keep = make_params(keep=keep, **kw)
        st, info, grad = ciq_hyper_grad(self.ctx, B, V, params)
        d = info.as_dict()
        d["status"] = st
        return grad, d

    def matvec(self, V, out, mvm_impl: str = "auto") -> None:
        ciq_matvec(self.ctx, V, out, mvm_impl)

    def set_posterior(self, Xt, y, noise: float) -> None:
        """Make this (candidate-set) operator the GP posterior covariance COV* + jitter I."""
        ciq_set_posterior(self.ctx, Xt, y, noise)

    def thompson(self, eps, idx, samples=None, **kw) -> dict:
        """One Thompson-sampling step (eq. thompson_sample): idx <- argmin(mu* + COV*^{1/2} eps)."""
        keep: list = []
        kw.pop("mode", None)
        params, keep = make_params(keep=keep, mode="sqrt", **kw)
        st, info = ciq_thompson(self.ctx, eps, idx, samples, params)
        d = info.as_dict()
        d["status"] = st
        return d

    def close(self) -> None:
        if self.ctx:
            ciq_free(self.ctx)
            self.ctx = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
