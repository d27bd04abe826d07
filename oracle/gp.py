"""NEXT-4 oracle -- TEST INFRASTRUCTURE (only tests/, smoke() and bench.py's oracle legs import it).

Plain numpy fp64, each function following its definition:

* cond_diag(Y, R)        Theorem 5 with reading L19: c(K-hat R^{-1}), K-hat = K Omega = Y
                         (the surrounding text, :359 "the stability of the numerical system, K-hat R_k^{-1}").
                         X = Y R^{-1} by a triangular solve, G = X^T X, eigenvalues of G (library eigvalsh):
                         cond = sqrt(l_max / l_min), eps = ||G - I||_2.
* woodbury_solve         (U diag(lam) U^T + s2 I)^{-1} B = (B - U diag(lam / (lam + s2)) U^T B) / s2
                         (Woodbury identity, U orthonormal).
* log_likelihood         -1/2 [n log 2 pi + sum log(lam + s2) + (n - r) log s2 + y^T woodbury_solve(y)]
                         (zero-mean Gaussian, matrix determinant lemma; "Gaussian type
                         likelihood", the form fixed by SPEC.md:434-442).
* kernel_rows(prob, rows) K[rows, :] = sigma2 kappa(r_ij) + nugget [i == j], r by direct differences (readings
                         L7-L10), fp64 from the fp32 points.
* nystrom_core(prob, Q)  the approximate spectral decomposition of K from the sketch's Q ("approximate
                         QR decompositions are useful in obtaining other approximate matrix decompositions, such
                         as approximate spectral decompositions" citing HM11; their Alg. 5.3 first step):
                         W = K Q (a second pass over K), B = Q^T W symmetrised, so K ~ Q B Q^T (= Q Q^T K Q Q^T).
* log_likelihood_core    the same Gaussian log-likelihood with Sigma = Q B Q^T + s2 I (Q orthonormal, B SPD):
                         y^T Sigma^{-1} y = (y^T y - c^T c) / s2 + c^T (B + s2 I)^{-1} c with c = Q^T y, and
                         log det Sigma = log det(B + s2 I) + (n - d) log s2 (Woodbury / determinant lemma on the
                         d x d core; B = V diag(lam) V^T gives back log_likelihood with U = Q V).
* woodbury_core          Sigma^{-1} X for the same Sigma.
"""
from __future__ import annotations

import numpy as np


def cond_diag(Y: np.ndarray, R: np.ndarray):
    Y = np.asarray(Y, np.float64)
    R = np.asarray(R, np.float64)
    X = np.linalg.solve(R.T, Y.T).T          # X R = Y
    G = X.T @ X
    w = np.linalg.eigvalsh(G)
    return float(np.sqrt(w[-1] / w[0])), float(np.max(np.abs(w - 1.0))), float(w[0]), float(w[-1])


def woodbury_solve(U: np.ndarray, lam: np.ndarray, s2: float, B: np.ndarray) -> np.ndarray:
    U = np.asarray(U, np.float64)
    lam = np.asarray(lam, np.float64)
    B = np.asarray(B, np.float64)
    C = U.T @ B
    w = lam / (lam + s2)
    return (B - U @ (w[:, None] * C if C.ndim == 2 else w * C)) / s2


def log_likelihood(U: np.ndarray, lam: np.ndarray, s2: float, y: np.ndarray):
    """Returns (loglik, y^T Sigma^{-1} y, log det Sigma)."""
    U = np.asarray(U, np.float64)
    lam = np.asarray(lam, np.float64)
    y = np.asarray(y, np.float64)
    n, r = U.shape
    quad = float(y @ woodbury_solve(U, lam, s2, y))
    logdet = float(np.sum(np.log(lam + s2)) + (n - r) * np.log(s2))
    return -0.5 * (n * np.log(2 * np.pi) + logdet + quad), quad, logdet


def kernel_rows(prob, rows) -> np.ndarray:
    """K[rows, :] in fp64 (sigma2 kappa(r) + nugget on the diagonal by index, r by direct differences)."""
    rows = np.asarray(rows, np.int64)
    x = prob.pts.astype(np.float64)
    r2 = np.zeros((rows.shape[0], x.shape[1]))
    for c in range(x.shape[0]):          # r^2 = sum_c (x_ic - x_jc)^2 by direct differences (L10)
        r2 += (x[c, rows, None] - x[c, None, :]) ** 2
    if prob.kind == 0:        # squared exponential, exp(-r^2 / (2 ell^2))   (L7)
        K = prob.sigma2 * np.exp(-r2 / (2.0 * prob.ell ** 2))
    elif prob.kind == 1:      # Matern-3/2, (1 + sqrt3 r / ell) exp(-sqrt3 r / ell)   (L8)
        z = np.sqrt(3.0 * r2) / prob.ell
        K = prob.sigma2 * (1.0 + z) * np.exp(-z)
    else:
        raise ValueError("kernel_rows: SQEXP or MATERN32 only")
    K[np.arange(rows.shape[0]), rows] += prob.nugget
    return K


def nystrom_core(prob, Q: np.ndarray, block: int = 512, nthreads: int | None = None):
    """(W, B): W = K Q streamed over row blocks of K (never the whole n x n; independent blocks on host threads),
    B = (Q^T W + W^T Q) / 2."""
    import concurrent.futures as cf
    import os
    Q = np.asarray(Q, np.float64)
    n = Q.shape[0]
    W = np.empty_like(Q)

    def one(r0):
        rows = np.arange(r0, min(n, r0 + block))
        W[rows] = kernel_rows(prob, rows) @ Q

    with cf.ThreadPoolExecutor(max_workers=nthreads or os.cpu_count() or 1) as ex:
        list(ex.map(one, range(0, n, block)))
    B = Q.T @ W
    return W, 0.5 * (B + B.T)


def woodbury_core(Q: np.ndarray, B: np.ndarray, s2: float, X: np.ndarray) -> np.ndarray:
    """(Q B Q^T + s2 I)^{-1} X = (X - Q C) / s2 + Q (B + s2 I)^{-1} C,  C = Q^T X."""
    Q = np.asarray(Q, np.float64)
    X = np.asarray(X, np.float64)
    C = Q.T @ X
    Z = np.linalg.solve(np.asarray(B, np.float64) + s2 * np.eye(B.shape[0]), C)
    return (X - Q @ C) / s2 + Q @ Z


def log_likelihood_core(Q: np.ndarray, B: np.ndarray, s2: float, y: np.ndarray):
    """Returns (loglik, y^T Sigma^{-1} y, log det Sigma) for Sigma = Q B Q^T + s2 I."""
    Q = np.asarray(Q, np.float64)
    y = np.asarray(y, np.float64)
    n, d = Q.shape
    c = Q.T @ y
    Cm = np.asarray(B, np.float64) + s2 * np.eye(d)
    quad = float((y @ y - c @ c) / s2 + c @ np.linalg.solve(Cm, c))
    sign, ld = np.linalg.slogdet(Cm)
    if sign <= 0:
        raise ValueError("B + s2 I is not positive definite")
    logdet = float(ld + (n - d) * np.log(s2))
    return -0.5 * (n * np.log(2 * np.pi) + logdet + quad), quad, logdet
