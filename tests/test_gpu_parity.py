"""GPU path (through the C-ABI) vs the fp64 oracle on the same seeded inputs.

Tolerances (north_star): Y relative Frobenius <= 1e-5; R <= 1e-4 after row-sign alignment;
X via rho(Z) = ||A - Y_ref Z||_F / ||A||_F within 1e-4 of rho_ref(k_gpu), |k_gpu - k_ref| <= 1
(SURVEY.md 8(c) L15).  Signs, selection and the fp16 Gaussian Omega bit-exact.
"""
import numpy as np
import pytest

import ks_inputs
import oracle
from _problems import align_rows, desc_of, problem, relF

pytestmark = pytest.mark.gpu

Y_TOL, R_TOL, RHO_TOL = 1e-5, 1e-4, 1e-4


def _t(a, cuda, dtype=None):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), device=cuda, dtype=dtype)


def _gpu_sketch(ks, cfg, pts, cuda, rb=0, re=None):
    sk = ks.Sketch(desc_of(cfg), cuda)
    Y = sk(_t(pts, cuda), rb, re)
    return sk, Y.cpu().numpy()


# ---------------------------------------------------------------- randomness
@pytest.mark.parametrize("n,d,omega", [(2048, 64, 0), (3000, 100, 0), (16384, 128, 0), (100, 10, 0), (64, 64, 0),
                                       (1000, 64, 1), (4096, 256, 1), (65536, 256, 1)])
def test_randomness_bit_exact(ks, cuda, n, d, omega):
    # (65536, 256, 1): the whole c3-sized Gaussian Omega (16.7 M fp16 values; exercises the fp32 fast path of
    # k_gauss_omega and its fp64 fallback near fp16 rounding boundaries)
    cfg, pts, A, prob = problem("c1", n=n, d=d, omega=omega, dim=2, seed=1234 + n)
    sk = ks.Sketch(desc_of(cfg), cuda)
    s, S, g = sk.export(signs=True, sel=omega == 0, gauss=omega == 1)
    assert np.array_equal(s.cpu().numpy(), prob.s)
    if omega == 0:
        assert np.array_equal(S.cpu().numpy(), prob.S)
    else:
        mism = int(np.sum(g.cpu().numpy().view(np.uint16) != prob.om16))
        assert mism == 0, f"{mism} fp16 Omega mismatches"


# ---------------------------------------------------------------- sketch
SKETCH_CASES = [
    # name, overrides
    ("c1", {}),                                                         # full c1: SE, D=1, d=64
    ("c2", dict(n=3000, d=100)),                                        # Matern, D=2, ragged n / rows / d
    ("c4", dict(n=1536, d=512, dim=3)),                                 # SE D=3, d = 512 (TPG 16)
    ("c5", dict(n=2500, d=256)),                                        # Matern, N(0,I) points, d=256
    ("c1", dict(n=100, d=10)),                                          # N < chunk length
    ("c1", dict(n=1, d=1)),                                             # degenerate n = 1
    ("c3", dict(n=4096, d=256)),                                        # Gaussian, tcgen05, d = 256
    ("c3", dict(n=1000, d=64)),                                         # Gaussian, ragged n and tiles
    ("c3", dict(n=2048, d=128, kernel=1, ell=0.05)),                    # Gaussian + Matern
    ("c3", dict(n=777, d=16, dim=1)),                                   # Gaussian, smallest width
]


@pytest.mark.parametrize("name,over", SKETCH_CASES)
def test_sketch_matches_oracle(ks, cuda, name, over):
    cfg, pts, A, prob = problem(name, **over)
    _, Yg = _gpu_sketch(ks, cfg, pts, cuda)
    Yr = prob.sketch_rows()
    assert Yg.shape == Yr.shape
    err = relF(Yg, Yr)
    assert err <= Y_TOL, err


def test_sketch_rows_independent_of_row_range(ks, cuda):
    cfg, pts, A, prob = problem("c2", n=4000)
    _, Yfull = _gpu_sketch(ks, cfg, pts, cuda)
    _, Ypart = _gpu_sketch(ks, cfg, pts, cuda, 37, 1001)
    assert np.array_equal(Ypart, Yfull[37:1001])               # bit-identical across sharding


def test_sketch_identity_K_gives_omega(ks, cuda):
    """K = I (points 1 apart, ell tiny): Y = Omega exactly in exact arithmetic."""
    n = 1024
    pts = np.arange(n, dtype=np.float32)[None, :] * np.float32(1.0)
    desc = dict(n=n, dim=1, kernel=0, sigma2=1.0, ell=1e-3, nugget=0.0, d=40, seed=5, omega=0)
    Y = ks.Sketch(desc, cuda)(_t(pts, cuda)).cpu().numpy()
    prob = oracle.Problem(pts, 0, 1.0, 1e-3, 0.0, 5, 40, 0)
    assert relF(Y, prob.omega_dense()) <= 1e-6


@pytest.mark.parametrize("name,nrows", [("c2", 2048), ("c3", 96), ("c4", 96), ("c5", 48)])
def test_sketch_full_config_sampled_rows(ks, cuda, name, nrows):
    """Full BASELINE sizes in the bench launch configuration; oracle on sampled rows."""
    cfg, pts, A, prob = problem(name)
    _, Yg = _gpu_sketch(ks, cfg, pts, cuda)
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(cfg["n"], size=nrows, replace=False))
    rows[0], rows[-1] = 0, cfg["n"] - 1
    Yr = prob.sketch_rows(rows)
    err = relF(Yg[rows], Yr)
    assert err <= Y_TOL, err


# ---------------------------------------------------------------- TSQR
TSQR_CASES = [(2048, 64, 4), (16384, 128, 8), (4096, 256, 16), (8192, 512, 8), (3000, 100, 3), (700, 33, 5),
              (512, 512, 1), (530, 512, 1), (40000, 64, 3),   # (530, 512, 1): one 530-row leaf (512-thread QR)
              (4096, 100, 8), (8192, 36, 16),   # TMA leaf apply (512-row leaves) with a partial last panel (w = 4)
              (8192, 200, 4), (16384, 300, 8)]  # tcgen05 leaf apply with partial 128-column tiles and panels


@pytest.mark.parametrize("rows,d,blocks", TSQR_CASES)
def test_tsqr_random_matrix_matches_oracle(ks, cuda, rows, d, blocks):
    rng = np.random.default_rng(rows + d)
    Y = rng.standard_normal((rows, d)).astype(np.float32)
    plan = ks.TsqrPlan(rows, d, blocks, cuda)
    Q, R = plan.factor(_t(Y, cuda))
    Q, R = Q.cpu().numpy().astype(np.float64), R.cpu().numpy().astype(np.float64)
    _, Rr = oracle.tsqr_tree(Y.astype(np.float64), blocks, want_q=False)
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) >= 0)
    assert relF(R, Rr) <= R_TOL
    assert np.linalg.norm(Q.T @ Q - np.eye(d)) <= 1e-4 * np.sqrt(d)
    assert relF(Q @ R, Y) <= 1e-5


def test_tsqr_tensor_core_apply_is_repeatable(ks, cuda):
    """The tcgen05 leaf apply is deterministic (fixed accumulation order): 40 factorizations of the same
    matrix are bitwise equal.  Guards the ring-slot release ordering (a slot released before its shared
    loads completed let the TMA refill race them -- the failure mode found in the tensor-core sketch)."""
    rng = np.random.default_rng(99)
    Y = _t(rng.standard_normal((16384, 384)).astype(np.float32), cuda)
    plan = ks.TsqrPlan(16384, 384, 8, cuda)
    Q0, R0 = (t.clone() for t in plan.factor(Y))
    for _ in range(39):
        Q, R = plan.factor(Y)
        assert bool((R == R0).all()) and bool((Q == Q0).all())


@pytest.mark.parametrize("chains", [1, 2])
@pytest.mark.parametrize("rows,d,blocks", [(4096, 64, 8), (6000, 100, 5), (16384, 128, 16)])
def test_tsqr_chain_topology_matches_oracle_chain(ks, cuda, rows, d, blocks, chains):
    """PAPER.md eq. (5): one chain (KS_TSQR_CHAIN) or, as printed, two chains advancing side by side and a
    final merge of their R's (KS_TSQR_MIXED): R equals the oracle's chain TSQR with that many chains (and
    hence the tree's, R unique)."""
    rng = np.random.default_rng(rows + 7 * d)
    Y = rng.standard_normal((rows, d)).astype(np.float32)
    plan = ks.TsqrPlan(rows, d, blocks, cuda, topology=ks.TSQR_CHAIN if chains == 1 else ks.TSQR_MIXED)
    Q, R = plan.factor(_t(Y, cuda))
    Q, R = Q.cpu().numpy().astype(np.float64), R.cpu().numpy().astype(np.float64)
    Rc = oracle.tsqr_chain(Y.astype(np.float64), blocks, chains)
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) >= 0)
    assert relF(R, Rc) <= R_TOL
    assert np.linalg.norm(Q.T @ Q - np.eye(d)) <= 1e-4 * np.sqrt(d)
    assert relF(Q @ R, Y) <= 1e-5


@pytest.mark.parametrize("rows,d,blocks,m,topology", [(8192, 128, 8, 16, 0), (4096, 64, 4, 5, 0), (3000, 100, 3, 8, 1),
                                                       (65536, 256, 16, 32, 0),
                                                       (8192, 96, 4, 160, 0)])   # m = 160: tcgen05 tiles of X
def test_tsqr_implicit_q_applies(ks, cuda, rows, d, blocks, m, topology):
    """Implicit Q: Q^T A from the stored reflectors.  Pinned by Y^T A = R^T (Q^T A) in fp64
    (independent of the explicit Q) and against the explicit Q; Q C likewise."""
    rng = np.random.default_rng(rows + m)
    Y = rng.standard_normal((rows, d)).astype(np.float32)
    A = rng.standard_normal((rows, m)).astype(np.float32)
    plan = ks.TsqrPlan(rows, d, blocks, cuda, topology=topology)
    Q, R = plan.factor(_t(Y, cuda))
    Ci = plan.apply_qt(_t(A, cuda)).cpu().numpy().astype(np.float64)
    R64, Q64 = R.cpu().numpy().astype(np.float64), Q.cpu().numpy().astype(np.float64)
    assert relF(R64.T @ Ci, Y.astype(np.float64).T @ A.astype(np.float64)) <= 1e-5
    assert relF(Ci, Q64.T @ A.astype(np.float64)) <= 1e-5
    Cm = rng.standard_normal((d, m)).astype(np.float32)
    Xi = plan.apply_q(_t(Cm, cuda)).cpu().numpy().astype(np.float64)
    assert relF(Xi, Q64 @ Cm.astype(np.float64)) <= 1e-5


@pytest.mark.parametrize("name,over", [("c1", {}), ("c2", {}), ("c3", dict(n=8192, blocks=8)), ("c5", dict(n=8192, blocks=2))])
def test_tsqr_of_sketch_matches_oracle(ks, cuda, name, over):
    """Ill-conditioned Y (cond up to ~1e8 at c1): R vs the oracle's TSQR of its own Y."""
    cfg, pts, A, prob = problem(name, **over)
    Yr = prob.sketch_rows()
    Y32 = Yr.astype(np.float32)
    plan = ks.TsqrPlan(cfg["n"], cfg["d"], cfg["blocks"], cuda)
    Q, R = plan.factor(_t(Y32, cuda))
    R = R.cpu().numpy().astype(np.float64)
    _, Rr = oracle.tsqr_tree(Yr, cfg["blocks"], want_q=False)
    err = relF(align_rows(R, Rr), Rr)
    assert err <= R_TOL, err


def test_tsqr_merge_and_qform(ks, cuda):
    """Two-level scheme: per-'rank' TSQR, stacked R merge, Q = Q1 Q2_p."""
    import torch
    rng = np.random.default_rng(3)
    P, rows, d = 4, 1024, 64
    Y = rng.standard_normal((P * rows, d)).astype(np.float32)
    Rs, plans, Qs = [], [], []
    for p in range(P):
        plan = ks.TsqrPlan(rows, d, 2, cuda)
        _, R = plan.factor(_t(Y[p * rows:(p + 1) * rows], cuda), want_q=False)
        plans.append(plan)
        Rs.append(R)
    Rstack = torch.cat(Rs, 0).contiguous()
    Q2 = torch.empty((P * d, d), device=cuda)
    R = torch.empty((d, d), device=cuda)
    ws = torch.empty(ks.ks_tsqr_merge_workspace_size(P, d), dtype=torch.uint8, device=cuda)
    ks.ks_tsqr_merge(Rstack, P, d, Q2, R, ws)
    for p in range(P):
        Qs.append(plans[p].qform(Q2[p * d:(p + 1) * d].contiguous()))
    Q = torch.cat(Qs, 0).cpu().numpy().astype(np.float64)
    R = R.cpu().numpy().astype(np.float64)
    _, Rr = oracle.householder_qr(Y.astype(np.float64), want_q=False)
    assert relF(R, Rr) <= R_TOL
    assert np.linalg.norm(Q.T @ Q - np.eye(d)) <= 1e-4 * np.sqrt(d)
    assert relF(Q @ R, Y) <= 1e-5


def test_tsqr_full_c4_properties(ks, cuda):
    """c4 at full size (262144 x 512, 8 blocks): QR = Y, Q^T Q = I, R triangular, r_jj >= 0."""
    import torch
    cfg, pts, A, prob = problem("c4")
    sk = ks.Sketch(desc_of(cfg), cuda)
    Y = sk(_t(pts, cuda))
    plan = ks.TsqrPlan(cfg["n"], cfg["d"], cfg["blocks"], cuda)
    Q, R = plan.factor(Y)
    assert torch.all(torch.tril(R, -1) == 0) and torch.all(torch.diagonal(R) >= 0)
    Qd, Rd, Yd = Q.double(), R.double(), Y.double()
    assert (torch.linalg.norm(Qd @ Rd - Yd) / torch.linalg.norm(Yd)).item() <= 1e-5
    assert torch.linalg.norm(Qd.T @ Qd - torch.eye(cfg["d"], device=cuda, dtype=torch.float64)).item() <= 1e-3


# ---------------------------------------------------------------- solve
def test_trsolve_hand_example_and_singular(ks, cuda):
    import torch
    R = _t(np.array([[2.0, 1.0], [0.0, 4.0]], np.float32), cuda)
    Cm = _t(np.array([[3.0], [8.0]], np.float32), cuda)
    Z = torch.empty((2, 1), device=cuda)
    k = torch.zeros(1, dtype=torch.int32, device=cuda)
    ks.ks_trsolve(R, Cm, 2, 1, 0.0, Z, k)
    assert np.array_equal(Z.cpu().numpy(), np.array([[0.5], [2.0]], np.float32))
    Rs = _t(np.array([[2.0, 1.0], [0.0, 0.0]], np.float32), cuda)
    with pytest.raises(ks.KsError) as e:
        ks.ks_trsolve(Rs, Cm, 2, 1, 0.0, Z, k)
    assert e.value.status == 2 and "index 1" in str(e.value)


# (5000, 96, 7): the generic split-K kernel (m % 4 != 0); the others the cp.async-staged k_qtx_fast with a
# 32-column (m <= 32) or 64-column m tile, ragged d tiles (300 = 256 + 44), ragged rows and several chunks.
@pytest.mark.parametrize("rows,d,m", [(5000, 96, 7), (5000, 96, 8), (3001, 300, 40), (70001, 512, 64)])
def test_apply_qt_and_apply_q(ks, cuda, rows, d, m):
    import torch
    rng = np.random.default_rng(8)
    Q = rng.standard_normal((rows, d)).astype(np.float32)
    X = rng.standard_normal((rows, m)).astype(np.float32)
    Cm = torch.empty((d, m), device=cuda)
    ws = torch.empty(ks.ks_apply_qt_workspace_size(rows, d, m), dtype=torch.uint8, device=cuda)
    ks.ks_apply_qt(_t(Q, cuda), rows, d, _t(X, cuda), m, Cm, ws)
    ref = Q.astype(np.float64).T @ X.astype(np.float64)
    assert relF(Cm.cpu().numpy(), ref) <= 1e-5
    Xo = torch.empty((rows, m), device=cuda)
    ks.ks_apply_q(_t(Q, cuda), rows, d, Cm, m, Xo)
    assert relF(Xo.cpu().numpy(), Q.astype(np.float64) @ Cm.cpu().numpy().astype(np.float64)) <= 1e-5


# m = 40 / 64: the SRHT Omega-apply's 32-column tiles (a partial second tile / two full tiles)
@pytest.mark.parametrize("omega,m", [(0, 5), (1, 5), (0, 40), (0, 64)])
def test_omega_apply_matches_oracle(ks, cuda, omega, m):
    cfg, pts, A, prob = problem("c1", n=3000, d=64, omega=omega, dim=2)
    Z = np.random.default_rng(1).standard_normal((64, m)).astype(np.float32)
    sk = ks.Sketch(desc_of(cfg), cuda)
    X = sk.omega_apply(_t(Z, cuda)).cpu().numpy()
    Xr = prob.omega_apply(Z.astype(np.float64))
    assert relF(X, Xr) <= 1e-5
    Xp = sk.omega_apply(_t(Z, cuda), 1000, 2100).cpu().numpy()
    assert np.array_equal(Xp, X[1000:2100])


def _solve_parity(ks, cuda, cfg, pts, A, prob, Yref=None):
    import torch
    pipe = ks.Pipeline(desc_of(cfg), cfg["m"], cfg["blocks"], tau=oracle.TAU, device=cuda)
    pipe(_t(pts, cuda), _t(A, cuda))
    torch.cuda.synchronize()
    Zg = pipe.Z.cpu().numpy().astype(np.float64)
    kg = int(pipe.k.item())
    out = oracle.lowrank_solve(prob, A, cfg["blocks"], Y=Yref)
    rho_g = oracle.rho_of(out["Y"], Zg, A)
    rho_r = out["rho"][kg]
    assert abs(kg - out["k"]) <= 1, (kg, out["k"])
    assert abs(rho_g - rho_r) <= RHO_TOL, (rho_g, rho_r)
    return pipe, out, kg


@pytest.mark.parametrize("name,over", [("c1", {}), ("c2", {}), ("c3", dict(n=8192, blocks=4)),
                                       ("c4", dict(n=8192, blocks=4)), ("c5", dict(n=8192, blocks=2))])
def test_lowrank_solve_matches_oracle(ks, cuda, name, over):
    cfg, pts, A, prob = problem(name, **over)
    pipe, out, kg = _solve_parity(ks, cuda, cfg, pts, A, prob)
    if cfg["n"] <= 16384:
        # residual on the user-facing X itself: ||A - K X_gpu|| / ||A|| (streamed K, oracle)
        X = pipe.X.cpu().numpy().astype(np.float64)
        KX = _K_times(prob, X)
        rho_x = np.linalg.norm(A - KX) / np.linalg.norm(A)
        assert abs(rho_x - out["rho"][kg]) <= RHO_TOL


def _K_times(prob, X):
    n = prob.n
    out = np.zeros_like(X)
    for r0 in range(0, n, 1024):
        idx = np.arange(r0, min(n, r0 + 1024))
        x = prob.pts.astype(np.float64)
        r2 = ((x[:, idx, None] - x[:, None, :]) ** 2).sum(0)
        if prob.kind == oracle.SQEXP:
            Kb = prob.sigma2 * np.exp(-r2 / (2 * prob.ell**2))
        else:
            z = np.sqrt(3 * r2) / prob.ell
            Kb = prob.sigma2 * (1 + z) * np.exp(-z)
        Kb[np.arange(len(idx)), idx] += prob.nugget
        out[idx] = Kb @ X
    return out


def test_one_shot_lowrank_solve_abi(ks, cuda):
    import torch
    cfg, pts, A, prob = problem("c1")
    desc = desc_of(cfg)
    n, d, m = cfg["n"], cfg["d"], cfg["m"]
    ws = torch.empty(ks.ks_lowrank_workspace_size(desc, m, cfg["blocks"]), dtype=torch.uint8, device=cuda)
    X = torch.empty((n, m), device=cuda)
    Z = torch.empty((d, m), device=cuda)
    k = torch.zeros(1, dtype=torch.int32, device=cuda)
    ks.ks_lowrank_solve(desc, _t(pts, cuda), _t(A, cuda), m, cfg["blocks"], oracle.TAU, X, Z, k, ws)
    out = oracle.lowrank_solve(prob, A, cfg["blocks"])
    kg = int(k.item())
    assert abs(kg - out["k"]) <= 1
    assert abs(oracle.rho_of(out["Y"], Z.cpu().numpy().astype(np.float64), A) - out["rho"][kg]) <= RHO_TOL


def test_invalid_arguments_rejected_before_launch(ks, cuda):
    import torch
    cfg, pts, A, prob = problem("c1")
    sk = ks.Sketch(desc_of(cfg), cuda)
    with pytest.raises(ks.KsError) as e:
        ks.ks_sketch(desc_of(cfg), _t(pts, cuda), 10, 5, torch.empty((1, 64), device=cuda), sk.ws)
    assert e.value.status == 1
    with pytest.raises(ks.KsError) as e:
        ks.ks_sketch(desc_of(cfg), _t(pts, cuda), 0, 10, torch.empty((10, 64), device=cuda), sk.ws[:100])
    assert e.value.status == 4


# ---------------------------------------------------------------- NEXT-1: Hartley / cosine structured Omega
TRIG_CASES = [
    (2, dict(n=4096, d=128, dim=2)),                           # Hartley, SE, power-of-two n
    (3, dict(n=3000, d=64, dim=1, kernel=1, ell=0.05)),        # cosine, Matern, ragged n (no padding)
    (2, dict(n=1000, d=16, dim=3)),                            # Hartley, D = 3, smallest width
    (3, dict(n=8192, d=256, dim=2)),                           # cosine, d = 256
    (2, dict(n=5000, d=96, dim=2, kernel=1)),                  # Hartley, Matern, ragged tiles
]


@pytest.mark.parametrize("omega,over", TRIG_CASES)
def test_trig_randomness_and_sketch_match_oracle(ks, cuda, omega, over):
    """Signs and the selection from [0, n) bit-exact; Y = K R T P within 1e-5 of the fp64 oracle."""
    cfg, pts, A, prob = problem("c2", omega=omega, seed=4321 + over["n"], **over)
    sk = ks.Sketch(desc_of(cfg), cuda)
    Yg = sk(_t(pts, cuda)).cpu().numpy()
    s, S, _ = sk.export(signs=True, sel=True, gauss=False)
    assert np.array_equal(s.cpu().numpy(), prob.s)
    assert np.array_equal(S.cpu().numpy(), prob.S)
    assert relF(Yg, prob.sketch_rows()) <= Y_TOL


@pytest.mark.parametrize("omega", [1, 3])
def test_tensor_core_sketch_is_repeatable(ks, cuda, omega):
    """200 sketches of one problem are bitwise equal and within Y_TOL of the oracle.  Regression test for a
    race found on the B200: a producer warp released its points slot right after issuing the shared loads,
    the SYNCS arrive ran ahead of them and the TMA refill overwrote the slot (16 rows of Y wrong in 13 of
    400 runs of this case, tools/repro_trig.py; 0 of 400 with the release after the values are used)."""
    import torch
    cfg, pts, A, prob = problem("c2", omega=omega, seed=4321 + 3000, n=3000, d=64, dim=1, kernel=1, ell=0.05)
    sk = ks.Sketch(desc_of(cfg), cuda)
    P = _t(pts, cuda)
    Y0 = sk(P)
    assert relF(Y0.cpu().numpy(), prob.sketch_rows()) <= Y_TOL
    Y = torch.empty_like(Y0)
    for r in range(199):
        sk(P, Y=Y)
        assert bool((Y == Y0).all()), f"run {r + 1} differs from run 0"


@pytest.mark.parametrize("omega", [2, 3])
def test_trig_omega_apply_matches_oracle(ks, cuda, omega):
    cfg, pts, A, prob = problem("c2", n=3000, d=64, omega=omega, dim=2)
    Z = np.random.default_rng(2).standard_normal((64, 5)).astype(np.float32)
    sk = ks.Sketch(desc_of(cfg), cuda)
    X = sk.omega_apply(_t(Z, cuda)).cpu().numpy()
    assert relF(X, prob.omega_apply(Z.astype(np.float64))) <= 1e-5


@pytest.mark.parametrize("omega", [2, 3])
def test_trig_lowrank_solve_matches_oracle(ks, cuda, omega):
    cfg, pts, A, prob = problem("c1", omega=omega, d=64)
    _solve_parity(ks, cuda, cfg, pts, A, prob)
    cfg, pts, A, prob = problem("c2", omega=omega, n=6000, d=128, blocks=4)
    _solve_parity(ks, cuda, cfg, pts, A, prob)


def test_host_inputs_match_device_inputs(ks, cuda):
    """The end-to-end call (pinned host points / A, A's copy on a side stream, X copied back) gives the
    same X as the device-resident call, bit for bit."""
    import torch
    from paper_1312_1869_b200 import dist as ksd
    cfg, pts, A, prob = problem("c2", n=4096, blocks=4)
    ops = ksd.CudaOps(desc_of(cfg), cfg["m"], cfg["blocks"], oracle.TAU, 0, 1, cuda)
    X_dev = ksd.lowrank_solve_sharded(ops, _t(pts, cuda), _t(A, cuda))[0].clone()
    torch.cuda.synchronize()
    A_h = torch.as_tensor(A).pin_memory()
    X_h = torch.empty((cfg["n"], cfg["m"]), dtype=torch.float32).pin_memory()
    for _ in range(2):   # the second call reuses the staged A buffer
        ksd.lowrank_solve_sharded(ops, torch.as_tensor(pts).pin_memory(), A_h, X_host=X_h)
        torch.cuda.synchronize()
        assert np.array_equal(X_h.numpy(), X_dev.cpu().numpy())


def test_inplace_sketch_into_tsqr_plan(ks, cuda):
    """CudaOps(inplace=True): the sketch is written into the TSQR plan's working matrix (ks_tsqr_work_matrix)
    and factored there without the input copy; R and X are bit-identical to the copying path."""
    import torch
    from paper_1312_1869_b200 import dist as ksd
    cfg, pts, A, prob = problem("c2", n=4096, blocks=4)
    outs = []
    for inplace in (False, True):
        ops = ksd.CudaOps(desc_of(cfg), cfg["m"], cfg["blocks"], oracle.TAU, 0, 1, cuda, inplace=inplace)
        X, Z, k, R = ksd.lowrank_solve_sharded(ops, _t(pts, cuda), _t(A, cuda))
        torch.cuda.synchronize()
        outs.append((X.cpu().numpy().copy(), R.cpu().numpy().copy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


# ---------------------------------------------------------------- exactly rank-deficient inputs
def test_exact_rank16_K_through_pipeline(ks, cuda):
    """The method's defining regime ("nearly rank deficient", range finder :95), exactly:
    n = 2048 points at r = 16 distinct locations, no nugget, so rank(K) = 16 (SURVEY.md 8(c) end-to-end
    pin; the oracle side is tests/test_oracle_qr_solve.py::test_exact_rank_recovery).  In fp32 the
    trailing |r_jj| sit at the rounding floor (~1e-7 |r_11|), far below tau = 1e-5, while |r_16| / |r_11|
    = 1.2e-3: the truncation rank is exactly 16, the first 16 columns of Q span range(K)
    (||K - Q_16 Q_16^T K||_F / ||K||_F at fp32 rounding) and rho matches the oracle's rho_ref(16)."""
    import torch
    n, r, d, m = 2048, 16, 64, 4
    loc = ks_inputs.points(21, r, 2)
    pts = np.ascontiguousarray(loc[:, np.arange(n) % r])
    desc = dict(n=n, dim=2, kernel=0, sigma2=1.0, ell=0.3, nugget=0.0, d=d, seed=21, omega=0)
    A = ks_inputs.rhs(21, n, m)
    pipe = ks.Pipeline(desc, m, 4, tau=oracle.TAU, device=cuda)
    pipe(_t(pts, cuda), _t(A, cuda))
    torch.cuda.synchronize()
    kg = int(pipe.k.item())
    assert kg == r, kg
    prob = oracle.Problem(pts, oracle.SQEXP, 1.0, 0.3, 0.0, 21, d, 0)
    K = prob.K_dense()
    Q16 = pipe.Q.cpu().numpy().astype(np.float64)[:, :r]
    resid = np.linalg.norm(K - Q16 @ (Q16.T @ K)) / np.linalg.norm(K)
    assert resid <= 1e-5, resid
    Zg = pipe.Z.cpu().numpy().astype(np.float64)
    assert np.all(Zg[r:] == 0)
    out = oracle.lowrank_solve(prob, A, 4)
    assert out["k"] == r
    assert abs(oracle.rho_of(out["Y"], Zg, A) - out["rho"][r]) <= RHO_TOL


@pytest.mark.parametrize("zero_cols", [[5], list(range(40, 64)), [0, 1, 63]])
def test_tsqr_exact_zero_columns(ks, cuda, zero_cols):
    """Exactly rank-deficient Y (exact zero columns): the sigma = 0 Householder branch (no reflection,
    r_jj = 0) in the leaves AND in every merge (a zero column stays exactly zero under reflections).  R is
    unique only above the first deficient row (L12: compare what is unique, check the rest is valid):
    rows < j0 against the oracle; r_jj == 0 exactly on the zero columns, R[:, zero] == 0; QR = Y and
    Q^T Q = I everywhere; the strict solve (tau = 0) reports the singular index j0."""
    import torch
    rows, d = 4096, 64
    Y = np.random.default_rng(9).standard_normal((rows, d)).astype(np.float32)
    Y[:, zero_cols] = 0.0
    plan = ks.TsqrPlan(rows, d, 8, cuda)
    Q, R = plan.factor(_t(Y, cuda))
    Qn, Rn = Q.cpu().numpy().astype(np.float64), R.cpu().numpy().astype(np.float64)
    j0 = min(zero_cols)
    assert np.all(Rn[:, zero_cols] == 0.0)
    assert np.all(np.tril(Rn, -1) == 0) and np.all(np.diag(Rn) >= 0)
    _, Rr = oracle.tsqr_tree(Y.astype(np.float64), 8, want_q=False)
    if j0 > 0:
        assert relF(Rn[:j0], Rr[:j0]) <= R_TOL
    assert relF(Qn @ Rn, Y) <= 1e-5
    assert np.linalg.norm(Qn.T @ Qn - np.eye(d)) <= 1e-4 * np.sqrt(d)
    Cm = torch.ones((d, 2), device=cuda)
    Z = torch.empty((d, 2), device=cuda)
    k = torch.zeros(1, dtype=torch.int32, device=cuda)
    with pytest.raises(ks.KsError) as e:
        ks.ks_trsolve(R, Cm, d, 2, 0.0, Z, k)
    assert e.value.status == 2 and f"index {j0}" in str(e.value)
    ks.ks_trsolve(R, Cm, d, 2, oracle.TAU, Z, k)
    torch.cuda.synchronize()
    assert int(k.item()) == j0


def test_one_shot_strict_solve_and_alignment_errors(ks, cuda):
    """ks_lowrank_solve with tau == 0 is the strict solve: a full-rank problem (c2-shaped, cond(Y) ~ 20) solves
    with k = d (the singular branch itself -- exact zeros on R's diagonal -- is covered through ks_trsolve by
    test_tsqr_exact_zero_columns: in fp32 an exactly rank-deficient K leaves ~1e-7 |r_11| of rounding on the
    trailing diagonal, above the strict 1e-12 threshold); k_dev is required.  ks_sketch rejects a Y that is
    not 16-byte aligned (the split-K add reads float4)."""
    import torch
    cfg, pts, A, prob = problem("c2", n=4096, d=64, blocks=2, m=4)
    desc = desc_of(cfg)
    n, d, m = cfg["n"], cfg["d"], cfg["m"]
    ws = torch.empty(ks.ks_lowrank_workspace_size(desc, m, 2), dtype=torch.uint8, device=cuda)
    X = torch.empty((n, m), device=cuda)
    Z = torch.empty((d, m), device=cuda)
    k = torch.zeros(1, dtype=torch.int32, device=cuda)
    ks.ks_lowrank_solve(desc, _t(pts, cuda), _t(A, cuda), m, 2, 0.0, X, Z, k, ws)
    torch.cuda.synchronize()
    assert int(k.item()) == d
    out = oracle.lowrank_solve(prob, A, 2, tau=1e-12)
    assert abs(oracle.rho_of(out["Y"], Z.cpu().numpy().astype(np.float64), A) - out["rho"][d]) <= RHO_TOL
    with pytest.raises(ks.KsError) as e:
        ks.ks_lowrank_solve(desc, _t(pts, cuda), _t(A, cuda), m, 2, 0.0, X, Z, None, ws)
    assert e.value.status == 1
    # misaligned Y
    sk = ks.Sketch(desc, cuda)
    buf = torch.empty(n * d + 1, device=cuda)
    with pytest.raises(ks.KsError) as e:
        ks.ks_sketch(desc, _t(pts, cuda), 0, n, buf[1:].view(n, d), sk.ws)
    assert e.value.status == 1 and "aligned" in str(e.value)


@pytest.mark.parametrize("P,d", [(2, 64), (8, 512), (4, 256), (3, 100), (8, 36)])
def test_tsqr_merge_of_triangular_stack(ks, cuda, P, d):
    """The second TSQR level (eqs. (2)-(3)): ks_tsqr_merge of P stacked upper-triangular R's runs
    the pairwise tree with KS_TSQR_TRIANGULAR (rows below each R's diagonal skipped, panel by panel).  R against
    the oracle's flat Householder QR of the stack, Q2 R = stack, Q2^T Q2 = I."""
    import torch
    rng = np.random.default_rng(P * 1000 + d)
    Rs = []
    for p in range(P):   # genuine R factors: QR of random tall blocks, graded like a sketch's R
        M = rng.standard_normal((2 * d, d)) * np.exp(-np.arange(d) / (d / 4.0))
        Rs.append(np.linalg.qr(M, mode="r"))
    stack = np.concatenate(Rs, 0).astype(np.float32)
    Q2 = torch.empty((P * d, d), device=cuda)
    R = torch.empty((d, d), device=cuda)
    ws = torch.empty(ks.ks_tsqr_merge_workspace_size(P, d), dtype=torch.uint8, device=cuda)
    ks.ks_tsqr_merge(_t(stack, cuda), P, d, Q2, R, ws)
    torch.cuda.synchronize()
    Rn, Qn = R.cpu().numpy().astype(np.float64), Q2.cpu().numpy().astype(np.float64)
    _, Rr = oracle.householder_qr(stack.astype(np.float64), want_q=False)
    assert np.all(np.tril(Rn, -1) == 0) and np.all(np.diag(Rn) >= 0)
    assert relF(align_rows(Rn, Rr), Rr) <= R_TOL
    assert relF(Qn @ Rn, stack) <= 1e-5
    assert np.linalg.norm(Qn.T @ Qn - np.eye(d)) <= 1e-4 * np.sqrt(d)
