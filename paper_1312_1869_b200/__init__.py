"""B200-native hot path of arXiv 1312.1869: sketch Y = K Omega -> TSQR -> low-rank solve.

Thin Python binding over the C-ABI library ``libks_b200.so`` (include/ks.h):
argument marshalling only.  Every step of the path runs in the library's
sm_100a kernels; PyTorch provides device memory, streams and (in ``dist``)
process groups.  There is no CPU fallback: if the library or a CUDA device is
missing, every compute call raises.

The functions ``ks_*`` mirror the C entry points one to one (same names, same
argument order, torch tensors in place of pointers).  ``Sketch``, ``TsqrPlan``
and ``Pipeline`` bundle the workspaces for repeated calls.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

__all__ = [
    "KsError", "SketchDesc", "SQEXP", "MATERN32", "STORED", "ks_sketch_stored", "SRHT", "GAUSS", "DHT", "DCT", "lib", "library_path",
    "ks_sketch_workspace_size", "ks_sketch", "ks_omega_export", "ks_omega_apply",
    "ks_tsqr_workspace_size", "ks_tsqr_create", "ks_tsqr_destroy", "ks_tsqr_work_matrix", "ks_tsqr", "ks_qform", "TSQR_TREE", "TSQR_CHAIN", "TSQR_MIXED", "TSQR_TRIANGULAR",
    "ks_tsqr_workspace_size_ex", "ks_tsqr_create_ex", "ks_tsqr_apply_qt", "ks_tsqr_apply_q",
    "ks_tsqr_merge_workspace_size", "ks_tsqr_merge", "ks_apply_qt_workspace_size", "ks_apply_qt",
    "ks_apply_q", "ks_trsolve", "ks_lowrank_workspace_size", "ks_lowrank_solve", "ks_last_error",
    "ks_version", "Sketch", "TsqrPlan", "Pipeline", "make_desc",
    "ks_cond_diag_workspace_size", "ks_cond_diag", "ks_cond_gram", "ks_cond_from_gram", "cond_diag",
    "ks_gp_workspace_size", "ks_gp_woodbury_solve", "ks_gp_loglik", "gp_woodbury_solve", "gp_loglik",
    "ks_nystrom_workspace_size", "ks_nystrom_core", "ks_gp_core_workspace_size", "ks_gp_loglik_core",
    "ks_gp_woodbury_core", "nystrom_core", "gp_loglik_core", "gp_woodbury_core",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_HERE, "libks_b200.so")

SQEXP, MATERN32, STORED = 0, 1, 2   # ks_kernel_kind (STORED: NEXT-2, K read from device memory)
SRHT, GAUSS, DHT, DCT = 0, 1, 2, 3   # ks_omega_kind (DHT / DCT: NEXT-1 structured Hartley / cosine)
STATUS = {0: "KS_OK", 1: "KS_ERR_INVALID_ARGUMENT", 2: "KS_ERR_SINGULAR", 3: "KS_ERR_CUDA", 4: "KS_ERR_OOM",
          5: "KS_ERR_UNSUPPORTED", 6: "KS_ERR_NCCL"}


class KsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class SketchDesc(C.Structure):
    _fields_ = [("n", C.c_int64), ("dim", C.c_int32), ("kernel", C.c_int32), ("sigma2", C.c_float),
                ("ell", C.c_float), ("nugget", C.c_float), ("d", C.c_int32), ("seed", C.c_uint64),
                ("omega", C.c_int32), ("reserved", C.c_int32)]


def make_desc(n, dim, kernel, sigma2, ell, nugget, d, seed, omega) -> SketchDesc:
    return SketchDesc(int(n), int(dim), int(kernel), float(sigma2), float(ell), float(nugget), int(d),
                      int(seed) & 0xFFFFFFFFFFFFFFFF, int(omega), 0)


_lib = None
_P, _i64, _i32, _f32, _sz = C.c_void_p, C.c_int64, C.c_int32, C.c_float, C.c_size_t
_SIGS = {
    "ks_sketch_workspace_size": [C.POINTER(SketchDesc), C.POINTER(_sz)],
    "ks_sketch": [C.POINTER(SketchDesc), _P, _i64, _i64, _P, _P, _sz, _P],
    "ks_sketch_stored": [C.POINTER(SketchDesc), _P, _i64, _i64, _i64, _P, _P, _sz, _P],
    "ks_cond_diag_workspace_size": [_i64, _i32, C.POINTER(_sz)],
    "ks_cond_diag": [_P, _i64, _i32, _P, _P, _P, _sz, _P],
    "ks_cond_gram": [_P, _i64, _i32, _P, _P, _P, _sz, _P],
    "ks_cond_from_gram": [_P, _i32, _P, _P, _sz, _P],
    "ks_gp_workspace_size": [_i64, _i32, _i32, C.POINTER(_sz)],
    "ks_gp_woodbury_solve": [_P, _i64, _i32, _P, _f32, _P, _i32, _P, _P, _sz, _P],
    "ks_gp_loglik": [_P, _i64, _i32, _P, _f32, _P, _P, _P, _sz, _P],
    "ks_nystrom_workspace_size": [C.POINTER(SketchDesc), C.POINTER(_sz)],
    "ks_nystrom_core": [C.POINTER(SketchDesc), _P, _P, _P, _P, _P, _sz, _P],
    "ks_gp_core_workspace_size": [_i64, _i32, _i32, C.POINTER(_sz)],
    "ks_gp_loglik_core": [_P, _i64, _i32, _P, _f32, _P, _P, _P, _sz, _P],
    "ks_gp_woodbury_core": [_P, _i64, _i32, _P, _f32, _P, _i32, _P, _P, _sz, _P],
    "ks_omega_export": [C.POINTER(SketchDesc), _P, _P, _P, _P, _sz, _P],
    "ks_omega_apply": [C.POINTER(SketchDesc), _P, _i32, _i64, _i64, _P, _P, _sz, _P],
    "ks_tsqr_workspace_size": [_i64, _i32, _i32, C.POINTER(_sz)],
    "ks_tsqr_create": [_i64, _i32, _i32, _P, _sz, C.POINTER(_P)],
    "ks_tsqr_workspace_size_ex": [_i64, _i32, _i32, _i32, C.POINTER(_sz)],
    "ks_tsqr_create_ex": [_i64, _i32, _i32, _i32, _P, _sz, C.POINTER(_P)],
    "ks_tsqr_apply_qt": [_P, _P, _i32, _P, _P],
    "ks_tsqr_apply_q": [_P, _P, _i32, _P, _P],
    "ks_tsqr_destroy": [_P],
    "ks_tsqr_work_matrix": [_P, _P],
    "ks_tsqr": [_P, _P, _P, _P, _P],
    "ks_qform": [_P, _P, _P, _P],
    "ks_tsqr_merge_workspace_size": [_i32, _i32, C.POINTER(_sz)],
    "ks_tsqr_merge": [_P, _i32, _i32, _P, _P, _P, _sz, _P],
    "ks_apply_qt_workspace_size": [_i64, _i32, _i32, C.POINTER(_sz)],
    "ks_apply_qt": [_P, _i64, _i32, _P, _i32, _P, _P, _sz, _P],
    "ks_apply_q": [_P, _i64, _i32, _P, _i32, _P, _P],
    "ks_trsolve": [_P, _P, _i32, _i32, _f32, _P, _P, _P],
    "ks_lowrank_workspace_size": [C.POINTER(SketchDesc), _i32, _i32, C.POINTER(_sz)],
    "ks_lowrank_solve": [C.POINTER(SketchDesc), _P, _P, _i32, _i32, _f32, _P, _P, _P, _P, _sz, _P],
}


def lib():
    """Load the C-ABI library (raises if it is missing: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(library_path):
            raise ImportError(f"{library_path} missing: run `python -m paper_1312_1869_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(library_path)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.ks_last_error.restype = C.c_char_p
        L.ks_version.restype = C.c_char_p
        _lib = L
    return _lib


def ks_last_error() -> str:
    return lib().ks_last_error().decode()


def ks_version() -> str:
    return lib().ks_version().decode()


def _check(status: int):
    if status != 0:
        raise KsError(status, ks_last_error())


def _stream(stream):
    if stream is None:
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, torch.cuda.Stream):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


def _ptr(t: torch.Tensor | None, dtype=None, name="tensor"):
    if t is None:
        return None
    if not t.is_cuda:
        raise KsError(1, f"{name} must be a CUDA tensor (no CPU path)")
    if not t.is_contiguous():
        raise KsError(1, f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise KsError(1, f"{name} must be {dtype}, got {t.dtype}")
    return C.c_void_p(t.data_ptr())


def _desc(desc) -> SketchDesc:
    if isinstance(desc, SketchDesc):
        return desc
    return make_desc(**desc)


# ------------------------------------------------------------ raw C-ABI mirrors
def ks_sketch_workspace_size(desc) -> int:
    b = _sz(0)
    _check(lib().ks_sketch_workspace_size(C.byref(_desc(desc)), C.byref(b)))
    return b.value


def ks_sketch(desc, pts, row_begin, row_end, Y, ws, stream=None):
    _check(lib().ks_sketch(C.byref(_desc(desc)), _ptr(pts, torch.float32, "pts"), int(row_begin), int(row_end),
                           _ptr(Y, torch.float32, "Y"), _ptr(ws, None, "ws"), ws.numel() * ws.element_size(),
                           _stream(stream)))


def ks_sketch_stored(desc, K, ldk, row_begin, row_end, Y, ws, stream=None):
    _check(lib().ks_sketch_stored(C.byref(_desc(desc)), _ptr(K, torch.float32, "K"), int(ldk), int(row_begin),
                                  int(row_end), _ptr(Y, torch.float32, "Y"), _ptr(ws, None, "ws"),
                                  ws.numel() * ws.element_size(), _stream(stream)))


def ks_omega_export(desc, signs, sel, gauss, ws, stream=None):
    _check(lib().ks_omega_export(C.byref(_desc(desc)), _ptr(signs, torch.int8, "signs"), _ptr(sel, torch.int32, "sel"),
                                 _ptr(gauss, torch.int16, "gauss"), _ptr(ws), ws.numel() * ws.element_size(),
                                 _stream(stream)))


def ks_omega_apply(desc, Z, m, row_begin, row_end, X, ws, stream=None):
    _check(lib().ks_omega_apply(C.byref(_desc(desc)), _ptr(Z, torch.float32, "Z"), int(m), int(row_begin),
                                int(row_end), _ptr(X, torch.float32, "X"), _ptr(ws), ws.numel() * ws.element_size(),
                                _stream(stream)))


def ks_tsqr_workspace_size(rows, d, blocks) -> int:
    b = _sz(0)
    _check(lib().ks_tsqr_workspace_size(int(rows), int(d), int(blocks), C.byref(b)))
    return b.value


def ks_tsqr_create(rows, d, blocks, ws) -> C.c_void_p:
    h = C.c_void_p()
    _check(lib().ks_tsqr_create(int(rows), int(d), int(blocks), _ptr(ws), ws.numel() * ws.element_size(), C.byref(h)))
    return h


TSQR_TREE, TSQR_CHAIN, TSQR_MIXED = 0, 1, 2
TSQR_TRIANGULAR = 16   # flag: the blocks are d x d upper-triangular R's (the second TSQR level)


def ks_tsqr_workspace_size_ex(rows, d, blocks, topology) -> int:
    b = _sz(0)
    _check(lib().ks_tsqr_workspace_size_ex(int(rows), int(d), int(blocks), int(topology), C.byref(b)))
    return b.value


def ks_tsqr_create_ex(rows, d, blocks, topology, ws) -> C.c_void_p:
    h = C.c_void_p()
    _check(lib().ks_tsqr_create_ex(int(rows), int(d), int(blocks), int(topology), _ptr(ws),
                                   ws.numel() * ws.element_size(), C.byref(h)))
    return h


def ks_tsqr_apply_qt(h, X, m, Cmat, stream=None):
    _check(lib().ks_tsqr_apply_qt(h, _ptr(X, torch.float32, "X"), int(m), _ptr(Cmat, torch.float32, "C"),
                                  _stream(stream)))


def ks_tsqr_apply_q(h, Cmat, m, X, stream=None):
    _check(lib().ks_tsqr_apply_q(h, _ptr(Cmat, torch.float32, "C"), int(m), _ptr(X, torch.float32, "X"),
                                 _stream(stream)))


def ks_tsqr_destroy(h):
    _check(lib().ks_tsqr_destroy(h))


def ks_tsqr_work_matrix(h) -> int:
    """Device address of the plan's working matrix (rows x d fp32); see include/ks.h."""
    p = C.c_void_p()
    _check(lib().ks_tsqr_work_matrix(h, C.byref(p)))
    return int(p.value)


def ks_tsqr(h, Y, Q, R, stream=None):
    _check(lib().ks_tsqr(h, _ptr(Y, torch.float32, "Y"), _ptr(Q, torch.float32, "Q"), _ptr(R, torch.float32, "R"),
                         _stream(stream)))


def ks_qform(h, Cmat, Q, stream=None):
    _check(lib().ks_qform(h, _ptr(Cmat, torch.float32, "C"), _ptr(Q, torch.float32, "Q"), _stream(stream)))


def ks_tsqr_merge_workspace_size(P, d) -> int:
    b = _sz(0)
    _check(lib().ks_tsqr_merge_workspace_size(int(P), int(d), C.byref(b)))
    return b.value


def ks_tsqr_merge(Rstack, P, d, Q2, R, ws, stream=None):
    _check(lib().ks_tsqr_merge(_ptr(Rstack, torch.float32, "Rstack"), int(P), int(d), _ptr(Q2, torch.float32, "Q2"),
                               _ptr(R, torch.float32, "R"), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def ks_apply_qt_workspace_size(rows, d, m) -> int:
    b = _sz(0)
    _check(lib().ks_apply_qt_workspace_size(int(rows), int(d), int(m), C.byref(b)))
    return b.value


def ks_apply_qt(Q, rows, d, X, m, Cmat, ws, stream=None):
    _check(lib().ks_apply_qt(_ptr(Q, torch.float32, "Q"), int(rows), int(d), _ptr(X, torch.float32, "X"), int(m),
                             _ptr(Cmat, torch.float32, "C"), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def ks_apply_q(Q, rows, d, Cmat, m, X, stream=None):
    _check(lib().ks_apply_q(_ptr(Q, torch.float32, "Q"), int(rows), int(d), _ptr(Cmat, torch.float32, "C"), int(m),
                            _ptr(X, torch.float32, "X"), _stream(stream)))


def ks_trsolve(R, Cmat, d, m, tau, Z, k, stream=None):
    _check(lib().ks_trsolve(_ptr(R, torch.float32, "R"), _ptr(Cmat, torch.float32, "C"), int(d), int(m), float(tau),
                            _ptr(Z, torch.float32, "Z"), _ptr(k, torch.int32, "k"), _stream(stream)))


def ks_lowrank_workspace_size(desc, m, blocks) -> int:
    b = _sz(0)
    _check(lib().ks_lowrank_workspace_size(C.byref(_desc(desc)), int(m), int(blocks), C.byref(b)))
    return b.value


def ks_lowrank_solve(desc, pts, A, m, blocks, tau, X, Z, k, ws, stream=None):
    _check(lib().ks_lowrank_solve(C.byref(_desc(desc)), _ptr(pts, torch.float32, "pts"), _ptr(A, torch.float32, "A"),
                                  int(m), int(blocks), float(tau), _ptr(X, torch.float32, "X"),
                                  _ptr(Z, torch.float32, "Z"), _ptr(k, torch.int32, "k"), _ptr(ws),
                                  ws.numel() * ws.element_size(), _stream(stream)))


# ------------------------------------------------------------ NEXT-4: Theorem 5 diagnostic, GP likelihood
def ks_cond_diag_workspace_size(rows, d) -> int:
    b = _sz(0)
    _check(lib().ks_cond_diag_workspace_size(int(rows), int(d), C.byref(b)))
    return b.value


def ks_cond_diag(Y, R, out, ws, stream=None):
    _check(lib().ks_cond_diag(_ptr(Y, torch.float32, "Y"), Y.shape[0], Y.shape[1], _ptr(R, torch.float32, "R"),
                              _ptr(out, torch.float32, "out"), _ptr(ws), ws.numel() * ws.element_size(),
                              _stream(stream)))


def ks_cond_gram(Y, R, G, ws, stream=None):
    _check(lib().ks_cond_gram(_ptr(Y, torch.float32, "Y"), Y.shape[0], Y.shape[1], _ptr(R, torch.float32, "R"),
                              _ptr(G, torch.float32, "G"), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def ks_cond_from_gram(G, out, ws, stream=None):
    _check(lib().ks_cond_from_gram(_ptr(G, torch.float32, "G"), G.shape[0], _ptr(out, torch.float32, "out"),
                                   _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def cond_diag(Y, R, stream=None):
    """(cond, eps, l_min, l_max) of G = (Y R^-1)^T (Y R^-1) as a device float[4] (Theorem 5 diagnostic)."""
    ws = _ws(ks_cond_diag_workspace_size(Y.shape[0], Y.shape[1]), Y.device)
    out = torch.empty(4, dtype=torch.float32, device=Y.device)
    ks_cond_diag(Y, R, out, ws, stream)
    return out


def ks_gp_workspace_size(rows, r, q) -> int:
    b = _sz(0)
    _check(lib().ks_gp_workspace_size(int(rows), int(r), int(q), C.byref(b)))
    return b.value


def ks_gp_woodbury_solve(U, lam, sigma2, B, X, ws, stream=None):
    _check(lib().ks_gp_woodbury_solve(_ptr(U, torch.float32, "U"), U.shape[0], U.shape[1],
                                      _ptr(lam, torch.float32, "lam"), float(sigma2), _ptr(B, torch.float32, "B"),
                                      B.shape[1], _ptr(X, torch.float32, "X"), _ptr(ws),
                                      ws.numel() * ws.element_size(), _stream(stream)))


def ks_gp_loglik(U, lam, sigma2, y, out, ws, stream=None):
    _check(lib().ks_gp_loglik(_ptr(U, torch.float32, "U"), U.shape[0], U.shape[1], _ptr(lam, torch.float32, "lam"),
                              float(sigma2), _ptr(y, torch.float32, "y"), _ptr(out, torch.float64, "out"), _ptr(ws),
                              ws.numel() * ws.element_size(), _stream(stream)))


def gp_woodbury_solve(U, lam, sigma2, B, stream=None):
    B2 = B if B.dim() == 2 else B.reshape(-1, 1)
    ws = _ws(ks_gp_workspace_size(U.shape[0], U.shape[1], B2.shape[1]), U.device)
    X = torch.empty_like(B2)
    ks_gp_woodbury_solve(U, lam, sigma2, B2, X, ws, stream)
    return X.reshape(B.shape)


def gp_loglik(U, lam, sigma2, y, stream=None):
    """Device double[3]: (log-likelihood, y^T Sigma^-1 y, log det Sigma)."""
    ws = _ws(ks_gp_workspace_size(U.shape[0], U.shape[1], 1), U.device)
    out = torch.empty(3, dtype=torch.float64, device=U.device)
    ks_gp_loglik(U, lam, sigma2, y, out, ws, stream)
    return out


# ------------------------------------------------------------ NEXT-4: the Nystrom core K ~ Q B Q^T
def ks_nystrom_workspace_size(desc) -> int:
    b = _sz(0)
    _check(lib().ks_nystrom_workspace_size(C.byref(_desc(desc)), C.byref(b)))
    return b.value


def ks_nystrom_core(desc, pts, Q, W, B, ws, stream=None):
    _check(lib().ks_nystrom_core(C.byref(_desc(desc)), _ptr(pts, torch.float32, "pts"), _ptr(Q, torch.float32, "Q"),
                                 _ptr(W, torch.float32, "W"), _ptr(B, torch.float32, "B"), _ptr(ws),
                                 ws.numel() * ws.element_size(), _stream(stream)))


def ks_gp_core_workspace_size(rows, d, q) -> int:
    b = _sz(0)
    _check(lib().ks_gp_core_workspace_size(int(rows), int(d), int(q), C.byref(b)))
    return b.value


def ks_gp_loglik_core(Q, B, sigma2, y, out, ws, stream=None):
    _check(lib().ks_gp_loglik_core(_ptr(Q, torch.float32, "Q"), Q.shape[0], Q.shape[1], _ptr(B, torch.float32, "B"),
                                   float(sigma2), _ptr(y, torch.float32, "y"), _ptr(out, torch.float64, "out"), _ptr(ws),
                                   ws.numel() * ws.element_size(), _stream(stream)))


def ks_gp_woodbury_core(Q, B, sigma2, X, Z, ws, stream=None):
    _check(lib().ks_gp_woodbury_core(_ptr(Q, torch.float32, "Q"), Q.shape[0], Q.shape[1], _ptr(B, torch.float32, "B"),
                                     float(sigma2), _ptr(X, torch.float32, "X"), X.shape[1], _ptr(Z, torch.float32, "Z"),
                                     _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def nystrom_core(desc, pts, Q, stream=None):
    """(W, B): W = K Q (a second fused pass over K), B = Q^T K Q symmetrised (K ~ Q B Q^T)."""
    D = _desc(desc)
    ws = _ws(ks_nystrom_workspace_size(D), Q.device)
    W = torch.empty_like(Q)
    B = torch.empty((Q.shape[1], Q.shape[1]), dtype=torch.float32, device=Q.device)
    ks_nystrom_core(D, pts, Q, W, B, ws, stream)
    return W, B


def gp_loglik_core(Q, B, sigma2, y, stream=None):
    """Device double[3]: (log-likelihood, y^T Sigma^-1 y, log det Sigma), Sigma = Q B Q^T + sigma2 I."""
    ws = _ws(ks_gp_core_workspace_size(Q.shape[0], Q.shape[1], 1), Q.device)
    out = torch.empty(3, dtype=torch.float64, device=Q.device)
    ks_gp_loglik_core(Q, B, sigma2, y, out, ws, stream)
    return out


def gp_woodbury_core(Q, B, sigma2, X, stream=None):
    X2 = X if X.dim() == 2 else X.reshape(-1, 1)
    ws = _ws(ks_gp_core_workspace_size(Q.shape[0], Q.shape[1], X2.shape[1]), Q.device)
    Z = torch.empty_like(X2)
    ks_gp_woodbury_core(Q, B, sigma2, X2, Z, ws, stream)
    return Z.reshape(X.shape)


# ------------------------------------------------------------ workspace bundles
def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


class Sketch:
    """Sketch randomness + workspace for one descriptor; Y = rows of K Omega."""

    def __init__(self, desc, device="cuda"):
        self.desc = _desc(desc)
        self.device = torch.device(device)
        self.ws = _ws(ks_sketch_workspace_size(self.desc), self.device)

    def __call__(self, pts, row_begin=0, row_end=None, Y=None, stream=None):
        n, d = self.desc.n, self.desc.d
        row_end = n if row_end is None else row_end
        if Y is None:
            Y = torch.empty((row_end - row_begin, d), dtype=torch.float32, device=self.device)
        ks_sketch(self.desc, pts, row_begin, row_end, Y, self.ws, stream)
        return Y

    def stored(self, K, row_begin=0, row_end=None, Y=None, stream=None):
        """Y = rows [row_begin, row_end) of K Omega for a stored K: K holds those rows, (rows x ldk) fp32 on
        the device (NEXT-2)."""
        n, d = self.desc.n, self.desc.d
        row_end = n if row_end is None else row_end
        if Y is None:
            Y = torch.empty((row_end - row_begin, d), dtype=torch.float32, device=self.device)
        ks_sketch_stored(self.desc, K, K.stride(0), row_begin, row_end, Y, self.ws, stream)
        return Y

    def omega_apply(self, Z, row_begin=0, row_end=None, X=None, stream=None):
        n = self.desc.n
        row_end = n if row_end is None else row_end
        m = Z.shape[1]
        if X is None:
            X = torch.empty((row_end - row_begin, m), dtype=torch.float32, device=self.device)
        ks_omega_apply(self.desc, Z, m, row_begin, row_end, X, self.ws, stream)
        return X

    def export(self, signs=True, sel=True, gauss=False, stream=None):
        D = self.desc
        N = 1 << max(0, (D.n - 1).bit_length())
        s = torch.empty(N, dtype=torch.int8, device=self.device) if signs else None
        S = torch.empty(D.d, dtype=torch.int32, device=self.device) if sel else None
        g = torch.empty((D.n, D.d), dtype=torch.int16, device=self.device) if gauss else None
        ks_omega_export(D, s, S, g, self.ws, stream)
        return s, S, g


class TsqrPlan:
    """Blocked TSQR plan over a torch-owned workspace."""

    def __init__(self, rows, d, blocks, device="cuda", topology=TSQR_TREE):
        self.rows, self.d, self.blocks = int(rows), int(d), int(blocks)
        self.ws = _ws(ks_tsqr_workspace_size_ex(rows, d, blocks, topology), device)
        self.h = ks_tsqr_create_ex(rows, d, blocks, topology, self.ws)
        self.device = torch.device(device)

    def work_matrix(self):
        """The plan's working matrix as a (rows x d) view of its workspace: a sketch written here is factored
        in place by ks_tsqr(h, work_matrix, ...) (no input copy; overwritten by the factorisation)."""
        off = ks_tsqr_work_matrix(self.h) - self.ws.data_ptr()
        n = self.rows * self.d
        return self.ws[off:off + 4 * n].view(torch.float32).view(self.rows, self.d)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            _lib.ks_tsqr_destroy(h)
            self.h = None

    def factor(self, Y, Q=None, R=None, want_q=True, stream=None):
        if R is None:
            R = torch.empty((self.d, self.d), dtype=torch.float32, device=self.device)
        if want_q and Q is None:
            Q = torch.empty((self.rows, self.d), dtype=torch.float32, device=self.device)
        ks_tsqr(self.h, Y, Q if want_q else None, R, stream)
        return Q, R

    def qform(self, Cmat=None, Q=None, stream=None):
        if Q is None:
            Q = torch.empty((self.rows, self.d), dtype=torch.float32, device=self.device)
        ks_qform(self.h, Cmat, Q, stream)
        return Q

    def apply_qt(self, X, stream=None):
        """Implicit Q-hat^T X (X rows x m is copied, not modified); returns C (d x m)."""
        Xw = X.contiguous().clone()
        Cm = torch.empty((self.d, Xw.shape[1]), dtype=torch.float32, device=self.device)
        ks_tsqr_apply_qt(self.h, Xw, Xw.shape[1], Cm, stream)
        return Cm

    def apply_q(self, Cmat, stream=None):
        """Implicit Q-hat C (C d x m); returns X (rows x m)."""
        Cmat = Cmat.contiguous()
        X = torch.empty((self.rows, Cmat.shape[1]), dtype=torch.float32, device=self.device)
        ks_tsqr_apply_q(self.h, Cmat, Cmat.shape[1], X, stream)
        return X


class Pipeline:
    """The whole single-GPU hot path with preallocated buffers (what bench.py times):
    sketch -> tsqr (explicit Q) -> Q^T A -> truncated back substitution -> X = Omega Z,
    each step one or more C-ABI calls on the current stream."""

    def __init__(self, desc, m, blocks, tau=1e-5, device="cuda", row_begin=0, row_end=None):
        self.desc = _desc(desc)
        self.m, self.blocks, self.tau = int(m), int(blocks), float(tau)
        self.device = torch.device(device)
        n, d = self.desc.n, self.desc.d
        self.rb, self.re = int(row_begin), int(n if row_end is None else row_end)
        rows = self.re - self.rb
        self.sketch = Sketch(self.desc, device)
        self.plan = TsqrPlan(rows, d, blocks, device)
        f32 = dict(dtype=torch.float32, device=self.device)
        self.Y = torch.empty((rows, d), **f32)
        self.Q = torch.empty((rows, d), **f32)
        self.R = torch.empty((d, d), **f32)
        self.C = torch.empty((d, self.m), **f32)
        self.Z = torch.empty((d, self.m), **f32)
        self.X = torch.empty((rows, self.m), **f32)
        self.k = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.qt_ws = _ws(ks_apply_qt_workspace_size(rows, d, self.m), self.device)

    def run_sketch(self, pts, stream=None):
        ks_sketch(self.desc, pts, self.rb, self.re, self.Y, self.sketch.ws, stream)

    def run_tsqr(self, stream=None):
        ks_tsqr(self.plan.h, self.Y, self.Q, self.R, stream)

    def run_solve(self, A, stream=None):
        rows, d = self.re - self.rb, self.desc.d
        ks_apply_qt(self.Q, rows, d, A, self.m, self.C, self.qt_ws, stream)
        ks_trsolve(self.R, self.C, d, self.m, self.tau, self.Z, self.k, stream)
        ks_omega_apply(self.desc, self.Z, self.m, self.rb, self.re, self.X, self.sketch.ws, stream)

    def __call__(self, pts, A, stream=None):
        self.run_sketch(pts, stream)
        self.run_tsqr(stream)
        self.run_solve(A, stream)
        return self.X
