"""NEXT-2 on the GPU: the stored-K sketch (ks_sketch_stored, K = E D E^T read from HBM) vs the fp64
oracle on the identical fp32 K; the same Y tolerance as the generated-K path (north_star: 1e-5), the
row-block semantics (a rank passes only its rows), a padded leading dimension, argument errors, and
the whole pipeline (TSQR + solve) on a stored K."""
import numpy as np
import pytest

import oracle
from _problems import align_rows, planted_problem, relF

pytestmark = pytest.mark.gpu

Y_TOL, R_TOL = 1e-5, 1e-4


def _t(a, cuda):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), device=cuda)


def _padded(K):
    """(rows, ldk) with ldk = n rounded up to 4 (the API's alignment rule), zero columns beyond n."""
    n = K.shape[1]
    Kp = np.zeros((K.shape[0], (n + 3) // 4 * 4), np.float32)
    Kp[:, :n] = K
    return Kp


def _desc(cfg):
    return dict(n=cfg["n"], dim=1, kernel=2, sigma2=1.0, ell=1.0, nugget=0.0, d=cfg["d"], seed=cfg["seed"],
                omega=cfg["omega"])


CASES = [(1000, 64, oracle.OMEGA_SRHT), (1536, 256, oracle.OMEGA_SRHT), (333, 16, oracle.OMEGA_SRHT),
         (1000, 64, oracle.OMEGA_GAUSS), (2048, 256, oracle.OMEGA_GAUSS), (777, 16, oracle.OMEGA_GAUSS),
         (1000, 64, oracle.OMEGA_DHT), (1200, 128, oracle.OMEGA_DCT)]


@pytest.mark.parametrize("n,d,omega", CASES)
def test_stored_sketch_matches_oracle(ks, cuda, n, d, omega):
    cfg, K, E, dvals, A, prob = planted_problem(n, d, omega, seed=100 + n)
    sk = ks.Sketch(_desc(cfg), cuda)
    Yg = sk.stored(_t(_padded(K), cuda)).cpu().numpy()
    Yr = prob.sketch_stored(K)
    assert relF(Yg, Yr) <= Y_TOL


@pytest.mark.parametrize("omega", [oracle.OMEGA_SRHT, oracle.OMEGA_GAUSS])
def test_stored_row_block_and_padded_ldk(ks, cuda, omega):
    import torch
    n, d, rb, re = 1000, 64, 137, 801
    cfg, K, E, dvals, A, prob = planted_problem(n, d, omega, seed=5)
    sk = ks.Sketch(_desc(cfg), cuda)
    Yfull = sk.stored(_t(K, cuda)).cpu().numpy()
    ldk = n + 24                                                    # padded leading dimension
    Kp = np.zeros((re - rb, ldk), np.float32)
    Kp[:, :n] = K[rb:re]
    Kp[:, n:] = np.nan                                              # columns >= n are never read
    Yblk = sk.stored(_t(Kp, cuda), rb, re).cpu().numpy()
    assert np.array_equal(Yblk, Yfull[rb:re])                       # bit-identical across row blocks
    assert relF(Yblk, prob.sketch_stored(K[rb:re])) <= Y_TOL


def test_stored_argument_errors(ks, cuda):
    import torch
    cfg, K, E, dvals, A, prob = planted_problem(256, 32, oracle.OMEGA_SRHT)
    sk = ks.Sketch(_desc(cfg), cuda)
    Kd = _t(K, cuda)
    Y = torch.empty((256, 32), device=cuda)
    with pytest.raises(ks.KsError):       # ldk < n
        ks.ks_sketch_stored(sk.desc, Kd, 128, 0, 256, Y, sk.ws)
    with pytest.raises(ks.KsError):       # ldk % 4 != 0
        ks.ks_sketch_stored(sk.desc, Kd, 257, 0, 256, Y, sk.ws)
    bad = dict(_desc(cfg), kernel=0)
    with pytest.raises(ks.KsError):       # not KS_KERNEL_STORED
        ks.ks_sketch_stored(ks.make_desc(**{k: bad[k] for k in ("n", "dim", "kernel", "sigma2", "ell", "nugget",
                                                                "d", "seed", "omega")}), Kd, 256, 0, 256, Y, sk.ws)


@pytest.mark.parametrize("omega", [oracle.OMEGA_GAUSS, oracle.OMEGA_SRHT])
def test_stored_pipeline_R_matches_oracle(ks, cuda, omega):
    """Sketch from the stored K, then the GPU TSQR: R against the oracle's TSQR of the oracle's Y."""
    from paper_1312_1869_b200 import dist as ksd
    n, d, blocks = 3000, 64, 2
    cfg, K, E, dvals, A, prob = planted_problem(n, d, omega, seed=9, m=8)
    ops = ksd.CudaOps(_desc(cfg), 8, blocks, 1e-5, 0, 1, cuda)
    X, Z, k, R = ksd.lowrank_solve_sharded(ops, _t(_padded(K), cuda), _t(A, cuda))
    Yr = prob.sketch_stored(K)
    _, Rr = oracle.tsqr_tree(Yr, blocks, want_q=False)
    Rg = align_rows(R.cpu().numpy(), Rr)
    assert relF(Rg, Rr) <= R_TOL
