"""Pins for the oracle's NEXT-1 structured Omega = R T P with T the discrete Hartley or discrete cosine
transform (Def. 1; the transforms named at :74 and :91 and used as HP/HC, RH/RC in the
experiments :388, :403).  Each pin is independent of ko_trig_entry: numpy/scipy FFTs, algebraic identities,
the Philox stream replayed here, brute force."""
import numpy as np
import pytest
import scipy.fft

import ks_inputs
import oracle


@pytest.mark.parametrize("n", [1, 2, 8, 12, 16, 37, 100])
def test_hartley_matrix_orthonormal_and_involutory(n):
    T = oracle.trig_matrix(oracle.OMEGA_DHT, n)
    assert np.allclose(T, T.T, atol=1e-15)                       # cas(2 pi jk/n) symmetric in j, k
    assert np.abs(T @ T - np.eye(n)).max() <= 1e-13             # the orthonormal DHT is its own inverse


@pytest.mark.parametrize("n", [1, 2, 8, 12, 16, 37, 100])
def test_cosine_matrix_orthonormal(n):
    T = oracle.trig_matrix(oracle.OMEGA_DCT, n)
    assert np.abs(T.T @ T - np.eye(n)).max() <= 1e-13


@pytest.mark.parametrize("n", [5, 16, 37, 64])
def test_transforms_match_library_ffts(n):
    v = np.random.default_rng(n).standard_normal(n)
    F = np.fft.fft(v)
    assert np.abs(oracle.trig_matrix(oracle.OMEGA_DHT, n).T @ v - (F.real - F.imag) / np.sqrt(n)).max() <= 1e-13
    assert np.abs(oracle.trig_matrix(oracle.OMEGA_DCT, n).T @ v - scipy.fft.dct(v, type=2, norm="ortho")).max() <= 1e-13


def _philox_select(seed, n, d):
    """The selection stream replayed with the oracle's Philox block only: first d distinct draws
    (w0 & (N-1)) that are < n, sorted."""
    N = oracle.next_pow2(n)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    seen, t = [], 0
    while len(seen) < d:
        w = oracle.philox([t & 0xFFFFFFFF, t >> 32, 2, 0], key)
        c = int(w[0]) & (N - 1)
        if c < n and c not in seen:
            seen.append(c)
        t += 1
    return np.array(sorted(seen), dtype=np.int32)


@pytest.mark.parametrize("n,d", [(1000, 10), (100, 100), (37, 5), (1024, 64), (3, 3)])
def test_selection_n_rejection_stream(n, d):
    seed = 0x1312186900000000 + n
    S = oracle.selection_n(seed, n, d)
    assert np.array_equal(S, _philox_select(seed, n, d))
    assert np.all(np.diff(S) > 0) and S[0] >= 0 and S[-1] < n
    if n & (n - 1) == 0:
        assert np.array_equal(S, oracle.selection(seed, n, d))   # no rejection for a power of two


@pytest.mark.parametrize("omega", [oracle.OMEGA_DHT, oracle.OMEGA_DCT])
@pytest.mark.parametrize("n,d", [(100, 16), (64, 64), (300, 48)])
def test_structured_omega_orthonormal_columns(omega, n, d):
    """L1: c = 1 makes the columns of R T P orthonormal (Omega^T Omega = I_d), for any n."""
    s = oracle.signs(7, oracle.next_pow2(n))
    S = oracle.selection_n(7, n, d)
    Om = oracle.omega_trig(omega, s, S, n)
    assert np.abs(Om.T @ Om - np.eye(d)).max() <= 1e-13


@pytest.mark.parametrize("omega", [oracle.OMEGA_DHT, oracle.OMEGA_DCT])
@pytest.mark.parametrize("n", [16, 37])
def test_structured_sketch_brute_force(omega, n):
    """Y = K Omega: tier-B rows vs an Omega built from numpy/scipy transforms of identity columns."""
    cfg, pts, A = ks_inputs.make_problem("c2", n=n, d=8, omega=omega, dim=2, seed=99)
    prob = oracle.Problem.from_cfg(cfg, pts)
    I = np.eye(n)
    if omega == oracle.OMEGA_DHT:
        F = np.fft.fft(I, axis=0)
        T = (F.real - F.imag) / np.sqrt(n)
    else:
        T = scipy.fft.dct(I, type=2, norm="ortho", axis=0).T
    Om = prob.s[:n, None].astype(np.float64) * T[:, prob.S]
    Yb = prob.K_dense() @ Om
    assert np.abs(prob.sketch_rows() - Yb).max() <= 1e-12 * np.abs(Yb).max()
    assert np.abs(prob.sketch_tierA() - Yb).max() <= 1e-12 * np.abs(Yb).max()
