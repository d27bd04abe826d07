"""NEXT-4 oracle pins (oracle/gp.py): the Woodbury solve, the low-rank-plus-nugget Gaussian log-likelihood
and Theorem 5's conditioning diagnostic, each against what the mathematics fixes -- hand-computed cases,
the dense inverse / dense log-density, the determinant lemma, invariances, and matrices with known
singular values."""
import numpy as np

from oracle import gp


def _orth(n, r, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return Q


def test_woodbury_hand_cases():
    B = np.random.default_rng(0).standard_normal((10, 3))
    U = _orth(10, 4, 1)
    assert np.allclose(gp.woodbury_solve(U, np.zeros(4), 0.5, B), B / 0.5, rtol=0, atol=1e-15)   # Lambda = 0
    e1 = np.zeros((5, 1)); e1[0] = 1
    X = gp.woodbury_solve(e1, np.array([3.0]), 1.0, e1)                 # (3 e1 e1^T + I)^{-1} e1 = e1 / 4
    assert np.allclose(X, e1 / 4, rtol=0, atol=1e-16)


def test_woodbury_is_the_dense_inverse():
    n, r, s2 = 128, 16, 0.3
    U = _orth(n, r, 2)
    lam = np.exp(-np.arange(r) / 4.0) * 5
    B = np.random.default_rng(3).standard_normal((n, 4))
    S = (U * lam) @ U.T + s2 * np.eye(n)
    X = gp.woodbury_solve(U, lam, s2, B)
    assert np.linalg.norm(X - np.linalg.solve(S, B)) <= 1e-12 * np.linalg.norm(X)
    assert np.linalg.norm(S @ X - B) <= 1e-12 * np.linalg.norm(B)


def test_loglik_cases():
    n, r, s2 = 64, 8, 0.7
    U = _orth(n, r, 4)
    lam = 1.0 + np.arange(r, dtype=float)
    y = np.random.default_rng(5).standard_normal(n)
    S = (U * lam) @ U.T + s2 * np.eye(n)
    sign, ld = np.linalg.slogdet(S)
    dense = -0.5 * (n * np.log(2 * np.pi) + ld + y @ np.linalg.solve(S, y))
    ll, quad, logdet = gp.log_likelihood(U, lam, s2, y)
    assert sign > 0 and abs(ll - dense) <= 1e-10 * abs(dense)
    assert abs(logdet - np.sum(np.log(np.linalg.eigvalsh(S)))) <= 1e-10 * abs(logdet)    # determinant lemma
    ll2, quad2, _ = gp.log_likelihood(U, lam, s2, 2 * y)
    assert abs((ll2 - ll) - (-1.5 * quad)) <= 1e-10 * quad                                # quadratic form
    ll0, _, _ = gp.log_likelihood(U, np.zeros(r), 1.0, np.zeros(n))                       # r = 0 equivalent
    assert abs(ll0 + 0.5 * n * np.log(2 * np.pi)) <= 1e-12
    O, _ = np.linalg.qr(np.random.default_rng(6).standard_normal((r, r)))
    lam_eq = np.full(r, 2.5)                                                              # basis invariance
    assert abs(gp.log_likelihood(U @ O, lam_eq, s2, y)[0] - gp.log_likelihood(U, lam_eq, s2, y)[0]) <= 1e-9


def test_cond_diag_known_singular_values():
    n, d = 500, 40
    Q = _orth(n, d, 7)
    c, eps, lo, hi = gp.cond_diag(Q, np.eye(d))                       # orthonormal, R = I -> 1
    assert abs(c - 1) <= 1e-12 and eps <= 1e-12
    Y = np.random.default_rng(8).standard_normal((n, d))
    R = np.linalg.qr(Y)[1]
    c, eps, lo, hi = gp.cond_diag(Y, R)                               # Y R^{-1} = Q exactly -> 1
    assert abs(c - 1) <= 1e-10
    s = np.linspace(0.6, 1.3, d)
    V = _orth(d, d, 9)
    c, eps, lo, hi = gp.cond_diag((Q * s) @ V.T, np.eye(d))           # singular values s -> s_max / s_min
    assert abs(c - 1.3 / 0.6) <= 1e-10 and abs(eps - (1.3 ** 2 - 1)) <= 1e-10
    assert abs(lo - 0.36) <= 1e-10 and abs(hi - 1.69) <= 1e-10


# ---------------------------------------------------------------- the Nystrom core (second K pass)
def test_kernel_rows_equals_the_c_oracle_K():
    """oracle.gp.kernel_rows (numpy) = the C oracle's materialised K (itself pinned by Tables 1-2)."""
    import ks_inputs
    import oracle
    for name, over in (("c2", dict(n=300, d=16)), ("c4", dict(n=257, d=16)), ("c5", dict(n=200, d=16))):
        cfg, pts, A = ks_inputs.make_problem(name, **over)
        prob = oracle.Problem.from_cfg(cfg, pts)
        K = prob.K_dense()
        rows = np.array([0, 5, 17, cfg["n"] - 1])
        np.testing.assert_allclose(gp.kernel_rows(prob, rows), K[rows], rtol=1e-13, atol=1e-15)


def test_core_loglik_is_the_dense_log_density():
    n, d, s2 = 300, 24, 0.05
    Q = _orth(n, d, 11)
    G = np.random.default_rng(12).standard_normal((d, d))
    B = G @ G.T
    y = np.random.default_rng(13).standard_normal(n)
    S = Q @ B @ Q.T + s2 * np.eye(n)
    sign, ld = np.linalg.slogdet(S)
    quad = y @ np.linalg.solve(S, y)
    ll, q2, ld2 = gp.log_likelihood_core(Q, B, s2, y)
    assert abs(ld2 - ld) <= 1e-10 * abs(ld) and abs(q2 - quad) <= 1e-10 * quad
    assert abs(ll + 0.5 * (n * np.log(2 * np.pi) + ld + quad)) <= 1e-10 * abs(ll)
    X = np.random.default_rng(14).standard_normal((n, 3))
    np.testing.assert_allclose(gp.woodbury_core(Q, B, s2, X), np.linalg.solve(S, X), rtol=1e-9, atol=1e-12)
    # the spectral form: B = V diag(lam) V^T, U = Q V gives the same likelihood through log_likelihood
    lam, V = np.linalg.eigh(B)
    ll_u = gp.log_likelihood(Q @ V, lam, s2, y)
    assert abs(ll_u[0] - ll) <= 1e-10 * abs(ll)


def test_nystrom_core_exact_for_exact_rank_K():
    """n = 2048 points at 16 locations, no nugget (rank(K) = 16; the SURVEY 8(c) end-to-end case): with Q_16
    spanning range(K) the Nystrom form is exact, Q B Q^T = K, and the core log-likelihood of K + s2 I equals the
    dense log-density."""
    import ks_inputs
    import oracle
    n, r, d = 2048, 16, 64
    loc = ks_inputs.points(21, r, 2)
    pts = np.ascontiguousarray(loc[:, np.arange(n) % r])
    prob = oracle.Problem(pts, oracle.SQEXP, 1.0, 0.3, 0.0, 21, d, 0)
    Q, R = oracle.tsqr_tree(prob.sketch_rows(), 4)
    Q16 = Q[:, :r]
    W, B = gp.nystrom_core(prob, Q16, block=500)
    K = prob.K_dense()
    np.testing.assert_allclose(W, K @ Q16, rtol=0, atol=1e-12 * np.abs(K).max())
    assert np.linalg.norm(Q16 @ B @ Q16.T - K) <= 1e-10 * np.linalg.norm(K)
    s2 = 0.01
    y = ks_inputs.rhs(21, n, 1)[:, 0].astype(np.float64)
    sign, ld = np.linalg.slogdet(K + s2 * np.eye(n))
    quad = y @ np.linalg.solve(K + s2 * np.eye(n), y)
    ll, q2, ld2 = gp.log_likelihood_core(Q16, B, s2, y)
    assert abs(ld2 - ld) <= 1e-9 * abs(ld) and abs(q2 - quad) <= 1e-9 * quad
