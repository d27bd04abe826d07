"""Pins for the oracle's QR / TSQR (eqs. (1)-(5) :99-252) and solve (PAPER.md:13,
readings L11-L16), plus the end-to-end special cases (exact rank, Theorem 4)."""
import numpy as np
import pytest

import oracle
import ks_inputs


def _signfix(Q, R):
    s = np.sign(np.diag(R))
    s[s == 0] = 1
    return Q * s[None, :], R * s[:, None]


def test_qr_small_examples():
    # I -> R = I ; diag(-2, 3) -> R = diag(2, 3) (sign absorbed)
    Q, R = oracle.householder_qr(np.eye(4))
    assert np.array_equal(R, np.eye(4)) and np.array_equal(Q, np.eye(4))
    A = np.array([[-2.0, 0.0], [0.0, 3.0], [0.0, 0.0]])
    Q, R = oracle.householder_qr(A)
    assert np.array_equal(R, np.diag([2.0, 3.0]))
    assert np.allclose(Q @ R, A, atol=1e-15)


@pytest.mark.parametrize("m,d", [(64, 8), (300, 40), (1000, 64)])
def test_qr_invariants_and_lapack(m, d):
    rng = np.random.default_rng(m)
    A = rng.standard_normal((m, d))
    Q, R = oracle.householder_qr(A)
    assert np.array_equal(np.tril(R, -1), np.zeros((d, d)))           # exact zeros below diagonal
    assert np.all(np.diag(R) >= 0)
    assert np.linalg.norm(Q.T @ Q - np.eye(d)) < 1e-13
    assert np.linalg.norm(Q @ R - A) < 1e-13 * np.linalg.norm(A)
    Ql, Rl = _signfix(*np.linalg.qr(A))                                # LAPACK, sign-normalised
    assert np.linalg.norm(R - Rl) < 1e-12 * np.linalg.norm(Rl)
    assert np.linalg.norm(Q - Ql) < 1e-11 * np.sqrt(d)


@pytest.mark.parametrize("b", [1, 2, 3, 4, 5, 8, 16])
def test_tsqr_tree_equals_flat(b):
    rng = np.random.default_rng(b)
    m, d = 1024, 16
    A = rng.standard_normal((m, d))
    _, Rf = oracle.householder_qr(A, want_q=False)
    Q, R = oracle.tsqr_tree(A, b, nthreads=3)
    assert np.linalg.norm(R - Rf) < 1e-12 * np.linalg.norm(Rf)
    assert np.linalg.norm(Q.T @ Q - np.eye(d)) < 1e-13
    assert np.linalg.norm(Q @ R - A) < 1e-13 * np.linalg.norm(A)
    if b == 1:  # b = 1 is the flat QR bit-for-bit
        Qf, Rf2 = oracle.householder_qr(A)
        assert np.array_equal(R, Rf2) and np.array_equal(Q, Qf)


@pytest.mark.parametrize("b,chains", [(1, 1), (4, 1), (8, 2), (8, 4), (16, 2)])
def test_tsqr_chain_equals_tree(b, chains):
    rng = np.random.default_rng(100 + b)
    A = rng.standard_normal((1024, 16))
    _, Rt = oracle.tsqr_tree(A, b, want_q=False)
    Rc = oracle.tsqr_chain(A, b, chains)
    assert np.linalg.norm(Rc - Rt) < 1e-12 * np.linalg.norm(Rt)


def test_tsqr_tree_equals_flat_on_ill_conditioned_sketch():
    """c1-like Y (cond ~ 1e8): tree R = flat R still holds in fp64 (SURVEY.md 8(c) 'R')."""
    cfg, pts, _ = ks_inputs.make_problem("c1")
    prob = oracle.Problem.from_cfg(cfg, pts)
    Y = prob.sketch_rows()
    _, Rf = oracle.householder_qr(Y, want_q=False)
    _, Rt = oracle.tsqr_tree(Y, 4, want_q=False)
    assert np.linalg.norm(Rt - Rf) < 1e-13 * np.linalg.norm(Rf)


def test_tsqr_rejects_wide_blocks():
    with pytest.raises(ValueError):
        oracle.tsqr_tree(np.ones((40, 16)), 3)


def test_thread_count_independence():
    rng = np.random.default_rng(9)
    A = rng.standard_normal((2048, 32))
    Q1, R1 = oracle.tsqr_tree(A, 8, nthreads=1)
    Q2, R2 = oracle.tsqr_tree(A, 8, nthreads=8)
    assert np.array_equal(R1, R2) and np.array_equal(Q1, Q2)


def test_back_substitution_hand_example():
    # R = [[2,1],[0,4]], B = (3,8) -> (0.5, 2)
    Z = oracle.back_substitute(np.array([[2.0, 1.0], [0.0, 4.0]]), np.array([[3.0], [8.0]]))
    assert np.array_equal(Z, np.array([[0.5], [2.0]]))


def test_truncation_rank_rule():
    R = np.diag([10.0, 1.0, 1e-3, 9.9e-5, 5.0])
    assert oracle.truncation_rank(R, 1e-5) == 3          # 9.9e-5 < 1e-5 * 10 breaks the prefix
    assert oracle.truncation_rank(R, 1e-6) == 5
    Z = oracle.back_substitute(R, np.ones((5, 2)), 3)
    assert np.all(Z[3:] == 0) and np.allclose(Z[:3, 0], [0.1, 1.0, 1000.0])


def test_full_rank_solve_is_least_squares():
    rng = np.random.default_rng(4)
    Y = rng.standard_normal((500, 20))
    A = rng.standard_normal((500, 3))
    Q, R = oracle.tsqr_tree(Y, 4)
    Cm = oracle._qt_apply(Q, A)
    Z = oracle.back_substitute(R, Cm, oracle.truncation_rank(R))
    Zl = np.linalg.lstsq(Y, A, rcond=None)[0]
    assert np.linalg.norm(Z - Zl) < 1e-10 * np.linalg.norm(Zl)
    assert np.linalg.norm(Y.T @ (A - Y @ Z)) < 1e-10 * np.linalg.norm(A)
    rho = oracle.rho_profile(Cm, A)
    assert np.all(np.diff(rho) <= 1e-15)
    assert rho[-1] == pytest.approx(oracle.rho_of(Y, Z, A), rel=1e-10)


@pytest.mark.parametrize("omega", [0, 1])
def test_omega_apply_equals_explicit(omega):
    pts = ks_inputs.points(3, 200, 2)
    prob = oracle.Problem(pts, oracle.SQEXP, 1.0, 0.1, 1e-6, 3, 24, omega)
    Z = np.random.default_rng(0).standard_normal((24, 3))
    X = prob.omega_apply(Z)
    assert np.linalg.norm(X - prob.omega_dense() @ Z) < 1e-14 * np.linalg.norm(X)


def test_kx_equals_yz():
    """L15: K X = K Omega Z = Y Z, so rho can be evaluated on Y without another n^2 pass."""
    cfg, pts, A = ks_inputs.make_problem("c1", n=512, d=32, blocks=2)
    prob = oracle.Problem.from_cfg(cfg, pts)
    out = oracle.lowrank_solve(prob, A, cfg["blocks"])
    KX = prob.K_dense() @ out["X"]
    assert np.linalg.norm(KX - out["Y"] @ out["Z"]) < 1e-10 * np.linalg.norm(KX)


def test_exact_rank_recovery():
    """n = 2048 points at r = 16 distinct locations, no nugget: rank(K) = 16."""
    n, r, d = 2048, 16, 64
    loc = ks_inputs.points(21, r, 2)
    pts = np.ascontiguousarray(loc[:, np.arange(n) % r])
    prob = oracle.Problem(pts, oracle.SQEXP, 1.0, 0.3, 0.0, 21, d, 0)
    Y = prob.sketch_rows()
    Q, R = oracle.tsqr_tree(Y, 4)
    dg = np.abs(np.diag(R))
    assert np.all(dg[r:] / dg[0] < 1e-12)
    assert np.all(dg[:r] / dg[0] > 1e-9)
    K = prob.K_dense()
    Qr = Q[:, :r]
    assert np.linalg.norm(K - Qr @ (Qr.T @ K)) < 1e-10 * np.linalg.norm(K)


def test_theorem4_bound():
    """||K - Q Q^T K||_2 <= (1 + sqrt(7n/r)) (tail); tested on the conclusion with
    k = d (reading L16): sigma_{d+1} <= err always; err <= (1+sqrt(7n/d)) sigma_{d+1} in >= 95%."""
    n, d = 1024, 24
    hits, seeds = 0, 20
    for sd in range(seeds):
        pts = ks_inputs.points(1000 + sd, n, 2)
        prob = oracle.Problem(pts, oracle.SQEXP, 1.0, 0.15, 1e-6, 1000 + sd, d, sd % 2)
        K = prob.K_dense()
        Y = prob.sketch_tierA()
        Q, _ = oracle.householder_qr(Y)
        err = np.linalg.norm(K - Q @ (Q.T @ K), 2)
        sig = np.sort(np.linalg.eigvalsh(K))[::-1]
        assert err >= sig[d] * (1 - 1e-9)
        hits += err <= (1 + np.sqrt(7 * n / d)) * sig[d]
    assert hits >= 0.95 * seeds
