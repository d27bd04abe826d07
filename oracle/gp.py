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
