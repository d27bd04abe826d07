"""NEXT-4 on the GPU: Theorem 5's diagnostic (ks_cond_diag) and the GP Woodbury solve / log-likelihood
(ks_gp_woodbury_solve, ks_gp_loglik) against oracle/gp.py on the same fp32 inputs."""
import numpy as np
import pytest

import oracle
from oracle import gp
from _problems import desc_of, problem, relF

pytestmark = pytest.mark.gpu


def _t(a, cuda):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a, np.float32), device=cuda)


def _orth(n, r, seed):
    Q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, r)))
    return Q.astype(np.float32)


@pytest.mark.parametrize("n,d", [(4000, 64), (1000, 200), (3333, 512)])
def test_cond_diag_known_singular_values(ks, cuda, n, d):
    Q = _orth(n, d, 1).astype(np.float64)
    s = np.linspace(0.6, 1.3, d)
    V = _orth(d, d, 2).astype(np.float64)
    Y = ((Q * s) @ V.T).astype(np.float32)
    R = np.triu(np.eye(d) + 0.1 * np.random.default_rng(3).standard_normal((d, d))).astype(np.float32)
    R[np.diag_indices(d)] = np.abs(R[np.diag_indices(d)]) + 0.5
    out = ks.cond_diag(_t(Y, cuda), _t(R, cuda)).cpu().numpy()
    c, eps, lo, hi = gp.cond_diag(Y, R)
    tol = 1e-3 if d <= 256 else 1e-2     # d <= 256: the whole Lanczos spectrum; d = 512: 256 steps
    assert abs(out[0] - c) <= tol * c
    assert abs(out[2] - lo) <= 2 * tol * lo and abs(out[3] - hi) <= tol * hi
    assert abs(out[1] - eps) <= tol * max(eps, 1e-3)


@pytest.mark.parametrize("name,over,blocks", [("c2", dict(n=6000, d=64), 4), ("c3", dict(n=4096, d=128), 2)])
def test_cond_diag_of_the_pipeline_is_near_one(ks, cuda, name, over, blocks):
    """Theorem 5: c(K-hat R^{-1}) <= sqrt((1 + eps) / (1 - eps)); with the sketch and TSQR of the configs
    the GPU's diagnostic is ~1 and agrees with the oracle's fp64 evaluation on the same fp32 Y, R."""
    cfg, pts, A, prob = problem(name, **over)
    sk = ks.Sketch(desc_of(cfg), cuda)
    Y = sk(_t(pts, cuda))
    plan = ks.TsqrPlan(cfg["n"], cfg["d"], blocks, cuda)
    Q, R = plan.factor(Y)
    out = ks.cond_diag(Y, R).cpu().numpy()
    c, eps, lo, hi = gp.cond_diag(Y.cpu().numpy(), R.cpu().numpy())
    assert c <= np.sqrt(2.0) and out[0] <= np.sqrt(2.0)              # Thm 5 with eps = 1/3
    assert abs(out[0] - c) <= 1e-3
    assert out[1] <= 1.0 / 3.0


def test_gp_woodbury_and_loglik_match_oracle(ks, cuda):
    n, r, q, s2 = 3000, 32, 5, float(np.float32(0.1))   # (sigma2 as the fp32 the C-ABI receives)
    U = _orth(n, r, 4)
    lam = (10.0 * np.exp(-np.arange(r) / 6.0)).astype(np.float32)
    rng = np.random.default_rng(5)
    B = rng.standard_normal((n, q)).astype(np.float32)
    y = rng.standard_normal(n).astype(np.float32)
    X = ks.gp_woodbury_solve(_t(U, cuda), _t(lam, cuda), s2, _t(B, cuda)).cpu().numpy()
    Xr = gp.woodbury_solve(U, lam, s2, B)
    assert relF(X, Xr) <= 1e-5
    out = ks.gp_loglik(_t(U, cuda), _t(lam, cuda), s2, _t(y, cuda)).cpu().numpy()
    ll, quad, logdet = gp.log_likelihood(U, lam, s2, y)
    assert abs(out[1] - quad) <= 1e-5 * abs(quad)
    assert abs(out[2] - logdet) <= 1e-9 * abs(logdet)
    assert abs(out[0] - ll) <= 1e-5 * abs(ll)


def test_gp_loglik_with_the_pipeline_factor(ks, cuda):
    """U = the TSQR Q of a sketch (orthonormal to fp32 accuracy), lam = 0: the likelihood reduces to the
    white-noise density N(0, s2 I) -- a closed form."""
    cfg, pts, A, prob = problem("c1", n=2048, d=64)
    Y = ks.Sketch(desc_of(cfg), cuda)(_t(pts, cuda))
    Q, R = ks.TsqrPlan(2048, 64, 2, cuda).factor(Y)
    y = np.random.default_rng(6).standard_normal(2048).astype(np.float32)
    s2 = float(np.float32(0.4))
    out = ks.gp_loglik(Q, _t(np.zeros(64, np.float32), cuda), s2, _t(y, cuda)).cpu().numpy()
    yy = float(np.dot(y.astype(np.float64), y.astype(np.float64)))
    ref = -0.5 * (2048 * np.log(2 * np.pi) + 2048 * np.log(s2) + yy / s2)
    assert abs(out[0] - ref) <= 1e-6 * abs(ref)


def test_gp_argument_errors(ks, cuda):
    import torch
    U = _t(_orth(100, 4, 7), cuda)
    lam = _t(np.ones(4), cuda)
    B = _t(np.ones((100, 1)), cuda)
    with pytest.raises(ks.KsError):
        ks.gp_woodbury_solve(U, lam, 0.0, B)          # sigma2 must be > 0
    ws = torch.empty(16, dtype=torch.uint8, device=cuda)
    with pytest.raises(ks.KsError):
        ks.ks_gp_woodbury_solve(U, lam, 1.0, B, torch.empty_like(B), ws)   # workspace too small


def test_cond_split_api_matches_one_call(ks, cuda):
    """ks_cond_gram on row blocks, summed (what ranks all-reduce), then ks_cond_from_gram == ks_cond_diag."""
    import torch
    n, d = 5000, 96
    Y = _t(np.random.default_rng(11).standard_normal((n, d)), cuda)
    Q, R = ks.TsqrPlan(n, d, 2, cuda).factor(Y)
    one = ks.cond_diag(Y, R).cpu().numpy()
    G = torch.zeros((d, d), dtype=torch.float32, device=cuda)
    for rb, re in ((0, 2100), (2100, n)):
        Yb = Y[rb:re].contiguous()
        ws = torch.empty(ks.ks_cond_diag_workspace_size(re - rb, d), dtype=torch.uint8, device=cuda)
        Gb = torch.empty((d, d), dtype=torch.float32, device=cuda)
        ks.ks_cond_gram(Yb, R, Gb, ws)
        G += Gb
    out = torch.empty(4, dtype=torch.float32, device=cuda)
    ks.ks_cond_from_gram(G, out, torch.empty(1024 * d, dtype=torch.uint8, device=cuda))
    out = out.cpu().numpy()
    c, eps, lo, hi = gp.cond_diag(Y.cpu().numpy(), R.cpu().numpy())
    assert abs(out[0] - one[0]) <= 1e-5 and abs(out[0] - c) <= 1e-4


# ---------------------------------------------------------------- the Nystrom core K ~ Q B Q^T (second K pass)
@pytest.mark.parametrize("name", ["c2", "c3"])
def test_nystrom_core_and_core_loglik_match_oracle(ks, cuda, name):
    """Full c2 / c3: the pipeline's Q, then W = K Q on the tensor cores (ks_nystrom_core), B = Q^T W, and the
    core-form likelihood / Woodbury solve (Sigma = Q B Q^T + s2 I, fp64 Cholesky of B + s2 I on the GPU) against
    oracle/gp.py: (a) the same steps in fp64 from the GPU's Q ("given Q"): W, B <= 1e-5, log-likelihood and
    Woodbury solve <= 1e-6 / 1e-5; (b) the whole oracle path (its own sketch, TSQR Q, Nystrom core and
    likelihood; at c3 from the GPU's Y): log-likelihood within 1e-5 relative.""" 
    import torch
    cfg, pts, A, prob = problem(name)
    n, d = cfg["n"], cfg["d"]
    pipe = ks.Pipeline(desc_of(cfg), cfg["m"], cfg["blocks"], tau=oracle.TAU, device=cuda)
    pipe(_t(pts, cuda), _t(A, cuda))
    Q = pipe.Q
    W, B = ks.nystrom_core(desc_of(cfg), _t(pts, cuda), Q)
    s2 = 0.01
    y = _t(A[:, 0], cuda)
    ll = ks.gp_loglik_core(Q, B, s2, y)
    Zw = ks.gp_woodbury_core(Q, B, s2, _t(A[:, :4], cuda))
    torch.cuda.synchronize()
    Qn = Q.cpu().numpy().astype(np.float64)
    Wg, Bg = W.cpu().numpy(), B.cpu().numpy()
    assert np.array_equal(Bg, Bg.T)
    Wr, Br = gp.nystrom_core(prob, Qn)
    assert relF(Wg, Wr) <= 1e-5, relF(Wg, Wr)
    assert relF(Bg, Br) <= 1e-5, relF(Bg, Br)
    llg = ll.cpu().numpy()
    llr = gp.log_likelihood_core(Qn, Bg.astype(np.float64), s2, A[:, 0].astype(np.float64))
    for a, b in zip(llg, llr):
        assert abs(a - b) <= 1e-6 * abs(b), (llg, llr)
    Zr = gp.woodbury_core(Qn, Bg.astype(np.float64), s2, A[:, :4].astype(np.float64))
    assert relF(Zw.cpu().numpy(), Zr) <= 1e-5
    # (b) the oracle's own path: its sketch (c2; at c3 the fp64 sketch of all 65536 rows takes hours, so the
    # oracle starts from the GPU's Y promoted to fp64 -- "TSQR given Y"), TSQR Q, Nystrom core
    Yo = prob.sketch_rows() if n <= 16384 else pipe.Y.cpu().numpy().astype(np.float64)
    Qo, _ = oracle.tsqr_tree(Yo, cfg["blocks"], want_q=True)
    _, Bo = gp.nystrom_core(prob, Qo)
    llo = gp.log_likelihood_core(Qo, Bo, s2, A[:, 0].astype(np.float64))
    assert abs(llg[0] - llo[0]) <= 1e-5 * abs(llo[0]), (llg, llo)
    print(f"{name}: W relF {relF(Wg, Wr):.2e}  B relF {relF(Bg, Br):.2e}  loglik gpu {llg[0]:.8e} oracle {llo[0]:.8e}")


def test_core_loglik_exact_rank_K(ks, cuda):
    """n = 2048 points at 16 locations, no nugget (rank(K) = 16): with the GPU's Q_16 the Nystrom core is exact
    (Q B Q^T = K) and the core log-likelihood of K + s2 I equals the dense fp64 log-density."""
    import torch
    import ks_inputs
    n, r, d = 2048, 16, 64
    loc = ks_inputs.points(21, r, 2)
    pts = np.ascontiguousarray(loc[:, np.arange(n) % r])
    desc = dict(n=n, dim=2, kernel=0, sigma2=1.0, ell=0.3, nugget=0.0, d=d, seed=21, omega=0)
    pipe = ks.Pipeline(desc, 4, 4, tau=oracle.TAU, device=cuda)
    pipe(_t(pts, cuda), _t(ks_inputs.rhs(21, n, 4), cuda))
    Q16 = pipe.Q[:, :r].contiguous()
    desc16 = dict(desc, d=r)
    W, B = ks.nystrom_core(desc16, _t(pts, cuda), Q16)
    y = ks_inputs.rhs(21, n, 1)[:, 0]
    ll = ks.gp_loglik_core(Q16, B, 0.01, _t(y, cuda))
    torch.cuda.synchronize()
    prob = oracle.Problem(pts, oracle.SQEXP, 1.0, 0.3, 0.0, 21, d, 0)
    K = prob.K_dense()
    Qn, Bn = Q16.cpu().numpy().astype(np.float64), B.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(Qn @ Bn @ Qn.T - K) <= 1e-5 * np.linalg.norm(K)
    S = K + 0.01 * np.eye(n)
    sign, ld = np.linalg.slogdet(S)
    quad = y.astype(np.float64) @ np.linalg.solve(S, y.astype(np.float64))
    llg = ll.cpu().numpy()
    assert abs(llg[2] - ld) <= 1e-5 * abs(ld) and abs(llg[1] - quad) <= 1e-5 * quad, (llg, ld, quad)


def test_core_argument_errors(ks, cuda):
    import torch
    Q = torch.zeros((100, 16), device=cuda)
    B = torch.zeros((16, 16), device=cuda)
    y = torch.zeros(100, device=cuda)
    out = torch.empty(3, dtype=torch.float64, device=cuda)
    ws = torch.empty(ks.ks_gp_core_workspace_size(100, 16, 1), dtype=torch.uint8, device=cuda)
    with pytest.raises(ks.KsError) as e:
        ks.ks_gp_loglik_core(Q, B, 0.0, y, out, ws)
    assert e.value.status == 1
    with pytest.raises(ks.KsError) as e:
        ks.ks_gp_loglik_core(Q, B, 0.1, y, out, ws[:8])
    assert e.value.status == 4
    with pytest.raises(ks.KsError) as e:   # d = 40 is not a multiple of 16 (the tensor-core pass)
        ks.nystrom_core(dict(n=100, dim=1, kernel=0, sigma2=1.0, ell=0.1, nugget=0.0, d=40, seed=1, omega=0),
                        torch.zeros((1, 100), device=cuda), torch.zeros((100, 40), device=cuda))
    assert e.value.status == 5
