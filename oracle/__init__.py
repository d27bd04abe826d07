"""CPU fp64 oracle for the arXiv 1312.1869 hot path -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_1312_1869_b200) never imports it and shares no code with it.

The arithmetic lives in ks_oracle.c (plain C, fp64, textbook loops); this
file only marshals numpy arrays and composes the steps in the paper's order:

    sketch  Y = K Omega                   PAPER.md:95 (range finder), Def. 1 :63-72
    QR      Y = Q R (Householder / TSQR)  PAPER.md:95, eqs. (1)-(5) :99-252
    solve   Z = R^{-1} Q^T A, X = Omega Z PAPER.md:13 (+ readings L11, L14)

Parity unpinned: the values of Q's trailing columns and of Z beyond the
numerical rank k (non-unique / ill-posed in fp32).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ks_oracle.c")
_LIB = os.path.join(_HERE, "libks_oracle.so")

SQEXP, MATERN32, MATERN12, MATERN52 = 0, 1, 2, 3
OMEGA_SRHT, OMEGA_GAUSS, OMEGA_DHT, OMEGA_DCT = 0, 1, 2, 3   # NEXT-1: Hartley / cosine structured Omega


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm", "-lpthread"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        i64, i32, u64, dbl, i = C.c_int64, C.c_int32, C.c_uint64, C.c_double, C.c_int
        sig = {
            "ko_philox": (None, [P, P, P]),
            "ko_signs": (None, [u64, i64, P]),
            "ko_selection": (i, [u64, i64, i32, P]),
            "ko_fp16_rn": (C.c_uint16, [dbl]),
            "ko_fp16_to_double": (dbl, [C.c_uint16]),
            "ko_gauss_omega": (None, [u64, i64, i32, P]),
            "ko_kernel_r": (dbl, [i, dbl, dbl, dbl]),
            "ko_K_entry": (dbl, [P, i64, i, i, dbl, dbl, dbl, i64, i64]),
            "ko_K_dense": (None, [P, i64, i, i, dbl, dbl, dbl, P]),
            "ko_hadamard": (None, [i64, P]),
            "ko_fwht": (None, [P, i64]),
            "ko_omega_srht": (None, [P, P, i64, i64, i32, P]),
            "ko_matmul": (None, [P, P, i64, i64, i64, P]),
            "ko_matmul_mt": (None, [P, P, i64, i64, i64, P, i]),
            "ko_sketch_srht_rows": (None, [P, i64, i, i, dbl, dbl, dbl, P, P, i64, i32, P, i64, P, i]),
            "ko_sketch_gauss_rows": (None, [P, i64, i, i, dbl, dbl, dbl, P, i32, P, i64, P, i]),
            "ko_householder_qr": (None, [P, i64, i32, P, P]),
            "ko_tsqr_tree": (i, [P, i64, i32, i32, P, P, i]),
            "ko_tsqr_chain": (i, [P, i64, i32, i32, i32, P]),
            "ko_truncation_rank": (i32, [P, i32, dbl]),
            "ko_back_substitute": (None, [P, i32, P, i32, i32, P]),
            "ko_omega_apply_srht": (None, [P, P, i64, i64, i32, P, i32, P]),
            "ko_omega_apply_gauss": (None, [P, i64, i32, P, i32, P]),
            "ko_selection_n": (i, [u64, i64, i64, i32, P]),
            "ko_trig_entry": (dbl, [i, i64, i64, i64]),
            "ko_omega_trig": (None, [i, P, P, i64, i32, P]),
            "ko_sketch_dense_rows": (None, [P, i64, i, i, dbl, dbl, dbl, P, i32, P, i64, P, i]),
            "ko_omega_apply_dense": (None, [P, i64, i32, P, i32, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _threads(n=None):
    return int(n or os.environ.get("KS_ORACLE_THREADS", os.cpu_count() or 1))


def next_pow2(n: int) -> int:
    return 1 << max(0, (int(n) - 1).bit_length())


# ---------------------------------------------------------------- randomness
def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32).copy()
    k = np.asarray(key, dtype=np.uint32).copy()
    out = np.zeros(4, dtype=np.uint32)
    lib().ko_philox(_p(c), _p(k), _p(out))
    return out


def signs(seed: int, N: int) -> np.ndarray:
    s = np.zeros(N, dtype=np.int8)
    lib().ko_signs(seed, N, _p(s))
    return s


def selection(seed: int, N: int, d: int) -> np.ndarray:
    S = np.zeros(d, dtype=np.int32)
    if lib().ko_selection(seed, N, d, _p(S)) != 0:
        raise ValueError("d > N")
    return S


def selection_n(seed: int, n: int, d: int) -> np.ndarray:
    """S uniform without replacement from [0, n) (rejection of masked draws >= n), sorted (NEXT-1)."""
    S = np.zeros(d, dtype=np.int32)
    if lib().ko_selection_n(seed, next_pow2(n), n, d, _p(S)) != 0:
        raise ValueError("d > n")
    return S


def trig_entry(kind: int, n: int, j: int, k: int) -> float:
    """T[j][k] of the orthonormal discrete Hartley (kind 2) or cosine DCT-II (kind 3) transform."""
    return float(lib().ko_trig_entry(int(kind), int(n), int(j), int(k)))


def trig_matrix(kind: int, n: int) -> np.ndarray:
    return np.array([[trig_entry(kind, n, j, k) for k in range(n)] for j in range(n)])


def omega_trig(kind: int, s: np.ndarray, S: np.ndarray, n: int) -> np.ndarray:
    """Explicit structured Omega = diag(s) T[:, S] (n x d), c = 1 (T orthonormal)."""
    d = S.shape[0]
    Om = np.zeros((n, d))
    lib().ko_omega_trig(int(kind), _p(np.ascontiguousarray(s, np.int8)), _p(np.ascontiguousarray(S, np.int32)), n, d,
                        _p(Om))
    return Om


def gauss_omega_fp16(seed: int, n: int, d: int) -> np.ndarray:
    """n x d uint16 fp16 bit patterns (L6)."""
    om = np.zeros((n, d), dtype=np.uint16)
    lib().ko_gauss_omega(seed, n, d, _p(om))
    return om


def fp16_rn(x: float) -> int:
    return int(lib().ko_fp16_rn(float(x)))


def fp16_to_f64(h: np.ndarray) -> np.ndarray:
    f = lib().ko_fp16_to_double
    return np.vectorize(lambda v: f(int(v)), otypes=[np.float64])(h)


# ---------------------------------------------------------------- kernel / K
def kernel_r(kind: int, r2: float, sigma2: float, ell: float) -> float:
    return float(lib().ko_kernel_r(kind, r2, sigma2, ell))


def K_dense(pts: np.ndarray, kind: int, sigma2: float, ell: float, nugget: float) -> np.ndarray:
    pts = np.ascontiguousarray(pts, dtype=np.float32)
    dim, n = pts.shape
    K = np.zeros((n, n))
    lib().ko_K_dense(_p(pts), n, dim, kind, sigma2, ell, nugget, _p(K))
    return K


def hadamard(N: int) -> np.ndarray:
    H = np.zeros((N, N))
    lib().ko_hadamard(N, _p(H))
    return H


def fwht(v: np.ndarray) -> np.ndarray:
    v = np.array(v, dtype=np.float64, copy=True)
    lib().ko_fwht(_p(v), v.shape[0])
    return v


def omega_srht(s: np.ndarray, S: np.ndarray, n: int) -> np.ndarray:
    N = s.shape[0]
    d = S.shape[0]
    Om = np.zeros((n, d))
    lib().ko_omega_srht(_p(np.ascontiguousarray(s, np.int8)), _p(np.ascontiguousarray(S, np.int32)), n, N, d, _p(Om))
    return Om


def matmul(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    A = np.ascontiguousarray(A, np.float64)
    B = np.ascontiguousarray(B, np.float64)
    Cm = np.zeros((A.shape[0], B.shape[1]))
    lib().ko_matmul(_p(A), _p(B), A.shape[0], A.shape[1], B.shape[1], _p(Cm))
    return Cm


def matmul_mt(A: np.ndarray, B: np.ndarray, nthreads=None) -> np.ndarray:
    """ko_matmul with the rows of the product split over threads (the same sums in the same order)."""
    A = np.ascontiguousarray(A, np.float64)
    B = np.ascontiguousarray(B, np.float64)
    Cm = np.zeros((A.shape[0], B.shape[1]))
    lib().ko_matmul_mt(_p(A), _p(B), A.shape[0], A.shape[1], B.shape[1], _p(Cm), _threads(nthreads))
    return Cm


# ---------------------------------------------------------------- sketch
class Problem:
    """Parameters of one sketch problem (mirrors the C-ABI ks_sketch_desc)."""

    def __init__(self, pts, kind, sigma2, ell, nugget, seed, d, omega):
        self.pts = np.ascontiguousarray(pts, dtype=np.float32)
        self.dim, self.n = self.pts.shape
        self.kind, self.sigma2, self.ell, self.nugget = int(kind), float(sigma2), float(ell), float(nugget)
        self.seed, self.d, self.omega = int(seed), int(d), int(omega)
        self.N = next_pow2(self.n)
        self._s = self._S = self._om = None

    @classmethod
    def from_cfg(cls, cfg, pts):
        return cls(pts, cfg["kernel"], cfg["sigma2"], cfg["ell"], cfg["nugget"], cfg["seed"], cfg["d"], cfg["omega"])

    @property
    def s(self):
        if self._s is None:
            self._s = signs(self.seed, self.N)
        return self._s

    @property
    def S(self):
        if self._S is None:
            self._S = (selection(self.seed, self.N, self.d) if self.omega != OMEGA_DHT and self.omega != OMEGA_DCT
                       else selection_n(self.seed, self.n, self.d))
        return self._S

    @property
    def omd(self):
        """Explicit fp64 Omega of the Hartley / cosine kinds (n x d)."""
        if getattr(self, "_omd", None) is None:
            self._omd = omega_trig(self.omega, self.s, self.S, self.n)
        return self._omd

    @property
    def om16(self):
        if self._om is None:
            self._om = gauss_omega_fp16(self.seed, self.n, self.d)
        return self._om

    def K_dense(self):
        return K_dense(self.pts, self.kind, self.sigma2, self.ell, self.nugget)

    def omega_dense(self) -> np.ndarray:
        """Explicit Omega (n x d), tier A."""
        if self.omega == OMEGA_SRHT:
            return omega_srht(self.s, self.S, self.n)
        if self.omega in (OMEGA_DHT, OMEGA_DCT):
            return self.omd
        return fp16_to_f64(self.om16) / np.sqrt(self.d)

    def sketch_tierA(self) -> np.ndarray:
        """Y = K Omega with K and Omega materialised, triple-loop product."""
        return matmul(self.K_dense(), self.omega_dense())

    def sketch_rows(self, rows=None, nthreads=None) -> np.ndarray:
        """Tier B: rows of Y computed one by one from streamed K rows."""
        rows = np.arange(self.n, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
        Y = np.zeros((rows.shape[0], self.d))
        L = lib()
        if self.omega in (OMEGA_DHT, OMEGA_DCT):
            L.ko_sketch_dense_rows(_p(self.pts), self.n, self.dim, self.kind, self.sigma2, self.ell, self.nugget,
                                   _p(self.omd), self.d, _p(rows), rows.shape[0], _p(Y), _threads(nthreads))
        elif self.omega == 0:
            L.ko_sketch_srht_rows(_p(self.pts), self.n, self.dim, self.kind, self.sigma2, self.ell, self.nugget,
                                  _p(self.s), _p(self.S), self.N, self.d, _p(rows), rows.shape[0], _p(Y),
                                  _threads(nthreads))
        else:
            om = np.ascontiguousarray(self.om16)
            L.ko_sketch_gauss_rows(_p(self.pts), self.n, self.dim, self.kind, self.sigma2, self.ell, self.nugget,
                                   _p(om), self.d, _p(rows), rows.shape[0], _p(Y), _threads(nthreads))
        return Y

    def sketch_stored(self, K_rows: np.ndarray) -> np.ndarray:
        """NEXT-2: rows of Y = K Omega for a stored K (PAPER.md:95 with K = E D E^T of :388): the given rows
        of K (r x n) times the explicit Omega, one library matmul (fp64)."""
        return matmul(np.ascontiguousarray(K_rows, np.float64), self.omega_dense())

    def omega_apply(self, Z: np.ndarray) -> np.ndarray:
        Z = np.ascontiguousarray(Z, np.float64)
        m = Z.shape[1]
        X = np.zeros((self.n, m))
        if self.omega in (OMEGA_DHT, OMEGA_DCT):
            lib().ko_omega_apply_dense(_p(self.omd), self.n, self.d, _p(Z), m, _p(X))
        elif self.omega == 0:
            lib().ko_omega_apply_srht(_p(self.s), _p(self.S), self.n, self.N, self.d, _p(Z), m, _p(X))
        else:
            om = np.ascontiguousarray(self.om16)
            lib().ko_omega_apply_gauss(_p(om), self.n, self.d, _p(Z), m, _p(X))
        return X


# ---------------------------------------------------------------- QR
def householder_qr(A: np.ndarray, want_q: bool = True):
    A = np.ascontiguousarray(A, np.float64)
    m, d = A.shape
    R = np.zeros((d, d))
    Q = np.zeros((m, d)) if want_q else None
    lib().ko_householder_qr(_p(A), m, d, _p(Q) if want_q else None, _p(R))
    return Q, R


def tsqr_tree(A: np.ndarray, blocks: int, want_q: bool = True, nthreads=None):
    A = np.ascontiguousarray(A, np.float64)
    m, d = A.shape
    R = np.zeros((d, d))
    Q = np.zeros((m, d)) if want_q else None
    if lib().ko_tsqr_tree(_p(A), m, d, blocks, _p(R), _p(Q) if want_q else None, _threads(nthreads)) != 0:
        raise ValueError("every block needs at least d rows")
    return Q, R


def tsqr_chain(A: np.ndarray, blocks: int, chains: int = 1):
    A = np.ascontiguousarray(A, np.float64)
    m, d = A.shape
    R = np.zeros((d, d))
    if lib().ko_tsqr_chain(_p(A), m, d, blocks, chains, _p(R)) != 0:
        raise ValueError("invalid block/chain counts")
    return R


# ---------------------------------------------------------------- solve
TAU = 1e-5  # reading L14


def truncation_rank(R: np.ndarray, tau: float = TAU) -> int:
    R = np.ascontiguousarray(R, np.float64)
    return int(lib().ko_truncation_rank(_p(R), R.shape[0], tau))


def back_substitute(R: np.ndarray, Cm: np.ndarray, k: int | None = None) -> np.ndarray:
    R = np.ascontiguousarray(R, np.float64)
    Cm = np.ascontiguousarray(Cm, np.float64)
    d, m = Cm.shape
    if k is None:
        k = d
    Z = np.zeros((d, m))
    lib().ko_back_substitute(_p(R), d, _p(Cm), m, int(k), _p(Z))
    return Z


def rho_profile(Cm: np.ndarray, A: np.ndarray) -> np.ndarray:
    """rho_ref(k') = sqrt(1 - sum_{j<k'} ||C_j||^2 / ||A||_F^2), k' = 0..d (L15)."""
    a2 = float(np.sum(np.asarray(A, np.float64) ** 2))
    cum = np.concatenate([[0.0], np.cumsum(np.sum(np.asarray(Cm, np.float64) ** 2, axis=1))])
    return np.sqrt(np.maximum(0.0, 1.0 - cum / a2))


def lowrank_solve(prob: Problem, A: np.ndarray, blocks: int, tau: float = TAU, Y: np.ndarray | None = None,
                  nthreads=None):
    """The whole path in the paper's order.  Returns dict(Y, Q, R, C, k, Z, X, rho)."""
    A64 = np.asarray(A, np.float64)
    if Y is None:
        Y = prob.sketch_rows(nthreads=nthreads) if prob.n > 4096 else prob.sketch_tierA()
    Q, R = tsqr_tree(Y, blocks, want_q=True, nthreads=nthreads)
    Cm = _qt_apply(Q, A64, nthreads)
    k = truncation_rank(R, tau)
    Z = back_substitute(R, Cm, k)
    X = prob.omega_apply(Z)
    return dict(Y=Y, Q=Q, R=R, C=Cm, k=k, Z=Z, X=X, rho=rho_profile(Cm, A64))


def _qt_apply(Q: np.ndarray, A: np.ndarray, nthreads=None) -> np.ndarray:
    """C = Q^T A by the plain triple loop (ko_matmul on the transposed Q; rows of C split over threads)."""
    return matmul_mt(np.ascontiguousarray(Q.T), A, nthreads)


def rho_of(Y: np.ndarray, Z: np.ndarray, A: np.ndarray) -> float:
    """rho(Z) = ||A - Y Z||_F / ||A||_F (L15)."""
    A64 = np.asarray(A, np.float64)
    return float(np.linalg.norm(A64 - np.asarray(Y, np.float64) @ np.asarray(Z, np.float64)) / np.linalg.norm(A64))
