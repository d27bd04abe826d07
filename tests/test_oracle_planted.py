"""NEXT-2 oracle pins: the planted-spectrum input and the stored-K sketch Y = K Omega
 checked against what the mathematics fixes -- the planted eigenvalues, exact recovery of the
column space of an exactly rank-r K (:95 range finder), and the Eckart-Young lower bound / range-finder
upper bound on ||K - Q Q^T K||_2 with the planted tail known exactly."""
import numpy as np
import pytest

import oracle
from _problems import planted_problem


def test_planted_spectrum_eigenvalues_and_orthonormal_E():
    cfg, K, E, dvals, A, prob = planted_problem(200, 16, oracle.OMEGA_GAUSS, rate=0.05)
    from ks_inputs.planted import planted_K
    K64, _, _ = planted_K(200, 77, 1.0, 0.05)
    w = np.linalg.eigvalsh(K64)[::-1]
    assert np.max(np.abs(w - dvals)) <= 1e-12 * dvals[0]
    assert np.abs(E.T @ E - np.eye(200)).max() <= 1e-12
    assert np.allclose(dvals, np.exp(-0.05 * np.arange(1, 201)))     # reading L17: decreasing, rate 0.05
    assert np.array_equal(K64, K64.T)


@pytest.mark.parametrize("omega,d", [(oracle.OMEGA_SRHT, 32), (oracle.OMEGA_GAUSS, 32), (oracle.OMEGA_DHT, 32),
                                     (oracle.OMEGA_DCT, 48)])
def test_stored_sketch_recovers_exact_rank_column_space(omega, d):
    r = 20
    cfg, K, E, dvals, A, prob = planted_problem(300, d, omega, rank=r)
    from ks_inputs.planted import planted_K
    K64, E, _ = planted_K(300, 77, 1.0, 0.01, r)
    Y = prob.sketch_stored(K64)
    assert Y.shape == (300, d)
    Q, R = oracle.householder_qr(Y)
    Er = E[:, :r]
    assert np.linalg.norm(Er - Q @ (Q.T @ Er)) <= 1e-9        # span(Y) contains span(E_r)
    # and nothing outside it: the singular values of Y beyond r vanish
    sv = np.linalg.svd(Y, compute_uv=False)
    assert sv[r] <= 1e-10 * sv[0]


@pytest.mark.parametrize("omega", [oracle.OMEGA_GAUSS, oracle.OMEGA_SRHT, oracle.OMEGA_DCT])
def test_stored_sketch_error_between_eckart_young_and_range_finder_bound(omega):
    n, k, p = 256, 30, 10
    d = k + p
    cfg, K, E, dvals, A, prob = planted_problem(n, d, omega, rate=0.05)
    from ks_inputs.planted import planted_K
    K64, _, _ = planted_K(n, 77, 1.0, 0.05)
    Y = prob.sketch_stored(K64)
    Q, _ = oracle.householder_qr(Y)
    err = np.linalg.norm(K64 - Q @ (Q.T @ K64), 2)
    assert err >= dvals[d] * (1 - 1e-9)                       # Eckart-Young: no rank-d projection does better
    tail = np.sqrt(np.sum(dvals[k:] ** 2))                     # Halko-Martinsson-Tropp (2011) Thm 10.5 (Gaussian)
    bound = (1 + np.sqrt(k / (p - 1))) * dvals[k] + np.e * np.sqrt(k + p) / p * tail
    assert err <= 4 * bound


def test_stored_sketch_rows_match_full_product():
    cfg, K, E, dvals, A, prob = planted_problem(150, 16, oracle.OMEGA_DHT)
    rows = np.array([0, 7, 149, 75])
    Yfull = prob.sketch_stored(K)
    assert np.array_equal(prob.sketch_stored(K[rows]), Yfull[rows])
