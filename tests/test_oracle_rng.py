"""Pins for the oracle's randomness (ledger L4-L6, L5 spec in DESIGN.md)."""
import os

import numpy as np
import pytest

import oracle
import ks_inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    rows = []
    for line in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        v = [int(x, 16) for x in line.split()]
        rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,out", _kat())
def test_philox_known_answer_oracle(ctr, key, out):
    assert [int(x) for x in oracle.philox(ctr, key)] == out


@pytest.mark.parametrize("ctr,key,out", _kat())
def test_philox_known_answer_inputs_module(ctr, key, out):
    got = ks_inputs.philox4x32_10(*[np.uint32(c) for c in ctr], key[0], key[1])
    assert [int(x) for x in got] == out


def test_philox_two_implementations_agree():
    rng = np.random.default_rng(7)
    for _ in range(200):
        ctr = rng.integers(0, 2**32, size=4, dtype=np.uint64).astype(np.uint32)
        key = rng.integers(0, 2**32, size=2, dtype=np.uint64).astype(np.uint32)
        a = oracle.philox(ctr, key)
        b = ks_inputs.philox4x32_10(*ctr, int(key[0]), int(key[1]))
        assert [int(x) for x in a] == [int(x) for x in b]


def test_signs_definition_and_balance():
    seed, N = 0x1234, 1 << 16
    s = oracle.signs(seed, N)
    assert set(np.unique(s)) <= {-1, 1}
    # independent restatement of the bit layout through the numpy Philox
    idx = np.arange(N // 128, dtype=np.uint64)
    w = ks_inputs.philox4x32_10(idx.astype(np.uint32), (idx >> np.uint64(32)).astype(np.uint32),
                                np.uint32(1), np.uint32(0), seed & 0xFFFFFFFF, seed >> 32)
    bits = np.stack(w, axis=1)  # (N/128, 4)
    j = np.arange(N)
    b = (bits[j >> 7, (j & 127) >> 5] >> (j & 31).astype(np.uint32)) & 1
    assert np.array_equal(s, (1 - 2 * b.astype(np.int64)).astype(np.int8))
    # Rademacher mean within 4 sigma
    assert abs(s.astype(np.float64).mean()) < 4.0 / np.sqrt(N)


@pytest.mark.parametrize("N,d", [(64, 64), (2048, 64), (16384, 128), (1 << 18, 512), (8, 3)])
def test_selection_is_sorted_distinct_subset(N, d):
    S = oracle.selection(99, N, d)
    assert S.shape == (d,)
    assert np.all(np.diff(S) > 0)
    assert S[0] >= 0 and S[-1] < N
    if d == N:
        assert np.array_equal(S, np.arange(N))


def test_selection_first_distinct_rule_restated():
    seed, N, d = 5, 256, 40
    S = oracle.selection(seed, N, d)
    idx = np.arange(4096, dtype=np.uint64)
    w0, _, _, _ = ks_inputs.philox4x32_10(idx.astype(np.uint32), np.uint32(0), np.uint32(2), np.uint32(0),
                                         seed & 0xFFFFFFFF, seed >> 32)
    seen = []
    for c in (w0 & np.uint32(N - 1)):
        if int(c) not in seen:
            seen.append(int(c))
        if len(seen) == d:
            break
    assert np.array_equal(S, np.sort(np.array(seen, dtype=np.int32)))


def test_selection_uniform_chi2():
    N, d, seeds = 64, 8, 2000
    counts = np.zeros(N)
    for sd in range(seeds):
        counts[oracle.selection(sd, N, d)] += 1
    expected = seeds * d / N
    chi2 = float(np.sum((counts - expected) ** 2 / expected))
    # 63 dof: mean 63, sd ~11.2; 6 sigma bound
    assert chi2 < 63 + 6 * 11.3


def test_selection_rejects_d_above_N():
    with pytest.raises(ValueError):
        oracle.selection(1, 16, 17)


def test_fp16_rn_matches_numpy_direct_double_to_half():
    rng = np.random.default_rng(3)
    vals = np.concatenate([
        rng.standard_normal(20000),
        rng.standard_normal(2000) * 1e-5,            # subnormal half range
        rng.standard_normal(2000) * 3e4,
        np.array([0.0, -0.0, 65504.0, 65519.99, 65520.0, 2.0**-24, 2.0**-25, 1.5 * 2.0**-25,
                  1 + 2.0**-11, 1 + 3 * 2.0**-11, 2.0**-14, 2.0**-14 - 2.0**-25]),
    ])
    ours = np.array([oracle.fp16_rn(v) for v in vals], dtype=np.uint16)
    ref = vals.astype(np.float16).view(np.uint16)
    assert np.array_equal(ours, ref)
    back = oracle.fp16_to_f64(ours)
    assert np.array_equal(back, ref.view(np.float16).astype(np.float64))


def test_gauss_omega_definition_and_moments():
    seed, n, d = 77, 512, 64
    om = oracle.gauss_omega_fp16(seed, n, d)
    z = ks_inputs.normal_fp64(seed, 3, n * d).reshape(n, d)
    assert np.array_equal(om, z.astype(np.float16).view(np.uint16))
    v = oracle.fp16_to_f64(om)
    assert abs(v.mean()) < 4 / np.sqrt(n * d)
    assert abs(v.var() - 1.0) < 4 * np.sqrt(2.0 / (n * d))
