"""NEXT-2 input: the planted-spectrum covariance of the paper's blocking simulation.

    "We consider the known spectral decomposition as K = E D E^T, where E is an orthonormalized
     matrix with randomly generated iid Gaussian entries.  D is the diagonal matrix of eigenvalues in
     decreasing order ... exponential decay with scale = 1 and rate 0.01" -- for n = 1000 ... 50000.

This is the workload's recipe, not the method under test: it is the only place a library QR
(LAPACK through numpy on the host; cuSOLVER through torch on the device for the large configs) and a
library GEMM are used, to build the INPUT matrix.  Both sides of every parity test receive the identical
fp32 K it returns.  Readings: d_ii = scale * exp(-rate * i), i = 1..n (decay with a negative
exponent, SPEC.md:95 / SURVEY.md L17); E = the Q of a Householder QR of the Gaussian matrix with the
column signs fixed so that diag(R) > 0 (the Haar-distributed orthonormalisation); K symmetrised.

Host generator (n <= a few thousand, used by the tests and the oracle): Gaussian entries from the
Philox stream 5 of the config seed (same normal_fp64 recipe as the points / A).  Device generator
(bench / sweep at n up to 50000): torch.randn with a torch.Generator seeded from the config seed, the
same recipe in fp32 on the GPU; a different random matrix than the host generator (documented in
DESIGN.md), generated once outside the timed region.
"""
from __future__ import annotations

import numpy as np

from . import normal_fp64

STREAM_PLANTED = 5


def planted_eigs(n: int, scale: float = 1.0, rate: float = 0.01, rank: int | None = None) -> np.ndarray:
    """d_ii = scale * exp(-rate * i), i = 1..n, decreasing; zero beyond `rank` (exact-rank variant)."""
    d = scale * np.exp(-rate * np.arange(1, n + 1, dtype=np.float64))
    if rank is not None:
        d[rank:] = 0.0
    return d


def planted_K(n: int, seed: int, scale: float = 1.0, rate: float = 0.01, rank: int | None = None):
    """Host: (K fp64 n x n, E fp64, eigenvalues)."""
    G = normal_fp64(seed, STREAM_PLANTED, n * n).reshape(n, n)
    Q, R = np.linalg.qr(G)
    E = Q * np.sign(np.diag(R))
    d = planted_eigs(n, scale, rate, rank)
    K = (E * d) @ E.T
    K = 0.5 * (K + K.T)
    return K, E, d


def planted_K_device(n: int, seed: int, device, scale: float = 1.0, rate: float = 0.01,
                     row_begin: int = 0, row_end: int | None = None):
    """Device: rows [row_begin, row_end) of K as fp32 (rows x ldk), ldk = n rounded up to 4."""
    import torch
    row_end = n if row_end is None else row_end
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    G = torch.randn((n, n), generator=g, device=device, dtype=torch.float32)
    Q, R = torch.linalg.qr(G)
    del G
    E = Q * torch.sign(torch.diagonal(R)).unsqueeze(0)
    del Q, R
    d = torch.as_tensor(planted_eigs(n, scale, rate), device=device, dtype=torch.float32)
    ldk = (n + 3) // 4 * 4
    K = torch.zeros((row_end - row_begin, ldk), device=device, dtype=torch.float32)
    # K = E D E^T is symmetric up to rounding; rows from one GEMM (E_rows * d) @ E^T
    K[:, :n] = (E[row_begin:row_end] * d) @ E.T
    del E
    torch.cuda.empty_cache()
    return K
