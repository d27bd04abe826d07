"""Pins for the oracle's covariance kernels (readings L7-L10)."""
import math
import os

import numpy as np
import pytest
from scipy.special import gamma, kv

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden():
    vals, orders = {}, {}
    for line in open(os.path.join(GOLDEN, "paper_tables.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        tok = line.split()
        if tok[0] in ("table1", "table2"):
            vals[tok[0]] = float(tok[-1])
        else:
            m = int(tok[1].split("=")[1])
            orders[(tok[0], m)] = [int(x) for x in tok[2:]]
    return vals, orders


VALS, ORDERS = _golden()
GRID = np.linspace(0.0, 1.0, 100)  # "equispaced grid of 100 points in [0,1]" PAPER.md:372


def _eigs(kind, ell, sigma2=1.0):
    pts = GRID.astype(np.float32)[None, :]
    K = oracle.K_dense(pts, kind, sigma2, ell, 0.0)
    return np.sort(np.linalg.eigvalsh(K))[::-1]


def test_se_at_zero_distance_is_sigma2_plus_nugget():
    pts = np.array([[0.25, 0.25, 0.7]], dtype=np.float32)
    K = oracle.K_dense(pts, oracle.SQEXP, 2.5, 0.1, 1e-3)
    assert K[0, 0] == 2.5 + 1e-3                       # nugget by index (L9)
    assert K[0, 1] == 2.5                              # coincident points, off-diagonal: no nugget
    assert np.array_equal(K, K.T)


@pytest.mark.parametrize("kind", [oracle.SQEXP, oracle.MATERN32, oracle.MATERN12, oracle.MATERN52])
def test_kernel_symmetric_and_unit_at_zero(kind):
    rng = np.random.default_rng(1)
    pts = rng.random((3, 40)).astype(np.float32)
    K = oracle.K_dense(pts, kind, 1.7, 0.3, 0.0)
    assert np.array_equal(K, K.T)
    assert np.all(np.diag(K) == 1.7)
    assert np.all(np.linalg.eigvalsh(K) > -1e-12)


def test_se_closed_form():
    for r2 in [0.0, 1e-6, 0.01, 0.3, 2.0]:
        assert oracle.kernel_r(oracle.SQEXP, r2, 1.3, 0.2) == pytest.approx(1.3 * math.exp(-r2 / 0.08), rel=1e-15)


@pytest.mark.parametrize("kind,nu", [(oracle.MATERN12, 0.5), (oracle.MATERN32, 1.5), (oracle.MATERN52, 2.5)])
def test_matern_closed_form_equals_printed_bessel_form(kind, nu):
    """theta1 / (Gamma(nu) 2^(nu-1)) (sqrt(2 nu) r / theta2)^nu B_nu(sqrt(2 nu) r / theta2)."""
    theta1, theta2 = 1.4, 0.35
    for r in [1e-3, 0.05, 0.2, 0.7, 2.0]:
        u = math.sqrt(2 * nu) * r / theta2
        bessel = theta1 / (gamma(nu) * 2 ** (nu - 1)) * u**nu * kv(nu, u)
        assert oracle.kernel_r(kind, r * r, theta1, theta2) == pytest.approx(bessel, rel=1e-12)


def test_table1_printed_value_29_89():
    """Table 1: SE, theta2 = 10, best rank-5 truncation -> 29.89 (reading L7)."""
    lam = _eigs(oracle.SQEXP, ell=math.sqrt(1 / 20.0))
    assert round(lam[0] / lam[4], 2) == pytest.approx(VALS["table1"], abs=0.006)


@pytest.mark.parametrize("col,theta2", list(enumerate([0.05, 0.5, 1.0, 1.5, 2.0, 10.0])))
def test_table1_orders_above_noise_floor(col, theta2):
    lam = _eigs(oracle.SQEXP, ell=math.sqrt(1 / (2 * theta2)))
    for m in (5, 10, 15):
        cond = lam[0] / lam[m - 1]
        if cond > 1e15:          # fp64 noise floor: not reproducible
            continue
        assert math.floor(math.log10(cond)) == ORDERS[("table1_order", m)][col], (m, theta2, cond)


def test_table2_printed_value_38_18_under_2sqrt_nu():
    """Table 2, nu = 0.5, theta1 = theta2 = 1: 38.18 is reproduced under the
    2 sqrt(nu) scaling (reading L8); the printed sqrt(2 nu) form gives 59.3."""
    lam = _eigs(oracle.MATERN12, ell=1 / math.sqrt(2.0))
    assert lam[0] / lam[4] == pytest.approx(VALS["table2"], rel=2e-3)
    lam_printed = _eigs(oracle.MATERN12, ell=1.0)
    assert 59.0 < lam_printed[0] / lam_printed[4] < 59.7


@pytest.mark.parametrize("kind,nu,col", [(oracle.MATERN12, 0.5, 0), (oracle.MATERN32, 1.5, 2), (oracle.MATERN52, 2.5, 4)])
def test_table2_orders_half_integer_nu(kind, nu, col):
    ell = math.sqrt(2 * nu) / (2 * math.sqrt(nu))     # a = 2 sqrt(nu) / theta2, theta2 = 1
    lam = _eigs(kind, ell)
    for m in (100, 50, 20, 15, 10, 5):
        cond = lam[0] / lam[m - 1]
        assert math.floor(math.log10(cond)) == ORDERS[("table2_order", m)][col], (m, nu, cond)


def test_fig1_claim_converged_by_10th_eigenvalue():
    """'by the 10th largest eigenvalue, the sequence has approximately converged to 0'."""
    for theta2 in [0.05, 0.5, 1, 1.5, 2, 10]:
        lam = _eigs(oracle.SQEXP, ell=math.sqrt(1 / (2 * theta2)))
        assert lam[9] / lam[0] < 1e-4
