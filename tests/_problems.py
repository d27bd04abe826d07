"""Shared helpers for the GPU parity tests: seeded problems (ks_inputs) + the oracle side."""
import numpy as np

import ks_inputs
import oracle


def problem(name=None, seed=None, **over):
    cfg, pts, A = ks_inputs.make_problem(name, seed=seed, **over)
    prob = oracle.Problem.from_cfg(cfg, pts)
    return cfg, pts, A, prob


def desc_of(cfg):
    return dict(n=cfg["n"], dim=cfg["dim"], kernel=cfg["kernel"], sigma2=cfg["sigma2"], ell=cfg["ell"],
                nugget=cfg["nugget"], d=cfg["d"], seed=cfg["seed"], omega=cfg["omega"])


def relF(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


NOISE_FLOOR = 1e-6   # |r_jj| <= NOISE_FLOOR * max|r_ii|: the row's sign is not determined in fp32 (L12)


def align_rows(Rg, Rr, floor=NOISE_FLOOR):
    """Row-sign alignment of R (= column signs of Q), only for rows whose diagonal |r_jj| sits at the
    noise floor (reading L12): r_jj >= 0 on both sides fixes every other row's sign, so a wrong-signed
    healthy row is never flipped into agreement."""
    Rg = np.array(Rg, np.float64)
    Rr = np.asarray(Rr, np.float64)
    dr = np.abs(np.diag(Rr))
    noisy = dr <= floor * dr.max()
    s = np.sign(np.sum(Rg * Rr, axis=1))
    s[(s == 0) | ~noisy] = 1
    return Rg * s[:, None]


def planted_problem(n, d, omega, seed=77, rank=None, rate=0.01, m=8):
    """NEXT-2: the planted-spectrum K = E D E^T (ks_inputs.planted, host generator) as the fp32 K both
    sides read, with a problem descriptor for the stored-K sketch."""
    from ks_inputs.planted import planted_K
    K64, E, dvals = planted_K(n, seed, 1.0, rate, rank)
    K = K64.astype(np.float32)
    cfg = dict(n=n, dim=1, kernel=2, sigma2=1.0, ell=1.0, nugget=0.0, d=d, seed=seed, omega=omega, m=m)
    prob = oracle.Problem.from_cfg(cfg, np.zeros((1, n), np.float32))
    A = ks_inputs.rhs(seed, n, m)
    return cfg, K, E, dvals, A, prob
