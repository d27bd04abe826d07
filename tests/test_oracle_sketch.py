"""Pins for the oracle's transform and sketch (Def. 1, H recursion :74-89;
readings L1-L3, L9, L10)."""
import numpy as np
import pytest
import scipy.linalg

import oracle
import ks_inputs


def popcount_parity(x):
    x = np.asarray(x, dtype=np.int64)
    p = np.zeros_like(x)
    while np.any(x):
        p ^= x & 1
        x >>= 1
    return p


@pytest.mark.parametrize("N", [2, 4, 8, 64, 256])
def test_hadamard_closed_form_and_orthogonality(N):
    H = oracle.hadamard(N)
    i, j = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    assert np.array_equal(H, 1.0 - 2.0 * popcount_parity(i & j))           # natural order (L2)
    assert np.array_equal(H, scipy.linalg.hadamard(N).astype(np.float64))  # library Sylvester
    assert np.array_equal(H @ H.T, N * np.eye(N))                          # exact in integers


def test_wht_n2_example():
    # SPEC.md:138 example: orthonormal WHT, n=2, v=(1,0) -> (1/sqrt2, 1/sqrt2)
    assert np.allclose(oracle.fwht([1.0, 0.0]) / np.sqrt(2), [2**-0.5, 2**-0.5], atol=0, rtol=1e-15)


@pytest.mark.parametrize("N", [1, 2, 16, 1024])
def test_fwht_equals_explicit_H_exactly_on_integers(N):
    rng = np.random.default_rng(N)
    v = rng.integers(-1000, 1000, size=N).astype(np.float64)
    assert np.array_equal(oracle.fwht(v), oracle.hadamard(N) @ v)
    assert np.array_equal(oracle.fwht(oracle.fwht(v)), N * v)


def _prob(n, dim=2, kind=oracle.SQEXP, d=8, omega=0, ell=0.2, nugget=1e-6, seed=11):
    pts = ks_inputs.points(seed, n, dim)
    return oracle.Problem(pts, kind, 1.0, ell, nugget, seed, d, omega)


def _library_reference(prob):
    """Y from independent pieces: numpy pairwise distances + scipy Hadamard (tiny n only)."""
    x = prob.pts.astype(np.float64)
    r2 = ((x[:, :, None] - x[:, None, :]) ** 2).sum(0)
    if prob.kind == oracle.SQEXP:
        K = prob.sigma2 * np.exp(-r2 / (2 * prob.ell**2))
    else:
        z = np.sqrt(3 * r2) / prob.ell
        K = prob.sigma2 * (1 + z) * np.exp(-z)
    K += prob.nugget * np.eye(prob.n)
    if prob.omega == 0:
        H = scipy.linalg.hadamard(prob.N).astype(np.float64)
        Om = (prob.s[:, None] * H[:, prob.S])[: prob.n] / np.sqrt(prob.N)
    else:
        Om = prob.om16.view(np.float16).astype(np.float64) / np.sqrt(prob.d)
    return K, Om, K @ Om


@pytest.mark.parametrize("n,d,kind,omega", [(8, 3, oracle.SQEXP, 0), (16, 8, oracle.MATERN32, 0),
                                            (16, 16, oracle.SQEXP, 0), (8, 4, oracle.SQEXP, 1),
                                            (13, 5, oracle.MATERN32, 0), (16, 6, oracle.MATERN32, 1)])
def test_bruteforce_tiny(n, d, kind, omega):
    prob = _prob(n, kind=kind, d=d, omega=omega)
    K, Om, Yref = _library_reference(prob)
    assert np.allclose(prob.K_dense(), K, rtol=1e-14, atol=1e-15)
    assert np.allclose(prob.omega_dense(), Om, rtol=1e-15, atol=0)
    for Y in (prob.sketch_tierA(), prob.sketch_rows(nthreads=2)):
        assert np.linalg.norm(Y - Yref) <= 1e-14 * np.linalg.norm(Yref)


def test_omega_srht_orthonormal_columns_when_n_is_N():
    prob = _prob(256, d=40, omega=0)
    Om = prob.omega_dense()
    assert np.linalg.norm(Om.T @ Om - np.eye(40)) < 1e-14


def test_identity_K_propagates_omega():
    # K = I -> Y = Omega.  Points 1 apart with ell = 1e-3: exp underflows to 0.
    n = 32
    pts = np.arange(n, dtype=np.float32)[None, :]
    prob = oracle.Problem(pts, oracle.SQEXP, 1.0, 1e-3, 0.0, 5, 7, 0)
    assert np.array_equal(prob.K_dense(), np.eye(n))
    assert np.allclose(prob.sketch_rows(), prob.omega_dense(), rtol=1e-15, atol=1e-17)


def test_full_selection_preserves_frobenius():
    # d = N -> ||K Omega||_F = ||K||_F
    prob = _prob(64, d=64, omega=0)
    Y = prob.sketch_rows()
    assert np.linalg.norm(Y) == pytest.approx(np.linalg.norm(prob.K_dense()), rel=1e-13)


def test_zero_padding_non_power_of_two():
    # L3: n = 100 -> N = 128; Y = first n rows of diag(s) H_128[:, S] / sqrt(128) applied to K
    prob = _prob(100, d=10)
    assert prob.N == 128 and prob.S.max() < 128
    K, Om, Yref = _library_reference(prob)
    assert np.linalg.norm(prob.sketch_rows() - Yref) <= 1e-14 * np.linalg.norm(Yref)


@pytest.mark.parametrize("n,omega,kind,dim", [(1024, 0, oracle.SQEXP, 1), (2048, 0, oracle.MATERN32, 2),
                                              (1024, 1, oracle.SQEXP, 2)])
def test_tierA_equals_tierB(n, omega, kind, dim):
    prob = _prob(n, dim=dim, kind=kind, d=32, omega=omega)
    YA = prob.sketch_tierA()
    rows = np.arange(0, n, 7)
    YB = prob.sketch_rows(rows)
    assert np.linalg.norm(YA[rows] - YB) <= 1e-13 * np.linalg.norm(YB)


def test_sketch_rows_independent_of_thread_count():
    prob = _prob(512, d=16)
    assert np.array_equal(prob.sketch_rows(nthreads=1), prob.sketch_rows(nthreads=5))
