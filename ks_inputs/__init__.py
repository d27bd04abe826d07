"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic (no kernel evaluation, no
transform, no QR).  It only turns (seed, shape) into the harness inputs of the
BASELINE configs: point clouds and right-hand sides A.  Both sides read the
identical fp32 arrays it returns, so parity never depends on how either side
would have generated its inputs.

Generator: Philox4x32-10 (Salmon et al.,
SC'11), key = (lo32(seed), hi32(seed)), counter = (lo32(idx), hi32(idx),
stream, 0).  Streams: 0 = points, 4 = A.  (Streams 1-3 -- signs, selection,
Gaussian Omega -- are the method's own draws; the oracle and the CUDA library
each implement them independently.)

* uniform point coordinate:  (w0 >> 8) * 2^-24            (exact in fp32, in [0,1))
* normal value:              z = sqrt(-2 ln U53(w0,w1)) * cos(2 pi U53(w2,w3)), fp64,
                             U53(a,b) = (((a>>5)*2^26 + (b>>6)) + 0.5) * 2^-53
  then rounded to fp32 (round-to-nearest-even, numpy astype).
Points use idx = i*D + c, A uses idx = i*m + c.
"""
from __future__ import annotations

import numpy as np

PHILOX_M0 = np.uint64(0xD2511F53)
PHILOX_M1 = np.uint64(0xCD9E8D57)
PHILOX_W0 = np.uint32(0x9E3779B9)
PHILOX_W1 = np.uint32(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)

STREAM_POINTS = 0
STREAM_A = 4

# Per-config master seeds: seed_cK = 0x1312186900000000 + K.
CONFIG_SEED_BASE = 0x1312186900000000


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 over uint32 arrays; returns (w0, w1, w2, w3)."""
    c0 = np.asarray(c0, dtype=np.uint32)
    c1 = np.asarray(c1, dtype=np.uint32)
    c2 = np.asarray(c2, dtype=np.uint32)
    c3 = np.asarray(c3, dtype=np.uint32)
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    shape = np.broadcast(c0, c1, c2, c3).shape
    c0, c1, c2, c3 = (np.broadcast_to(x, shape).astype(np.uint32) for x in (c0, c1, c2, c3))
    with np.errstate(over="ignore"):
        for r in range(10):
            p0 = PHILOX_M0 * c0.astype(np.uint64)
            p1 = PHILOX_M1 * c2.astype(np.uint64)
            hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
            lo0 = (p0 & MASK32).astype(np.uint32)
            hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
            lo1 = (p1 & MASK32).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            if r != 9:
                k0 = np.uint32((int(k0) + int(PHILOX_W0)) & 0xFFFFFFFF)
                k1 = np.uint32((int(k1) + int(PHILOX_W1)) & 0xFFFFFFFF)
    return c0, c1, c2, c3


def _draw(seed: int, stream: int, count: int):
    idx = np.arange(count, dtype=np.uint64)
    lo = (idx & MASK32).astype(np.uint32)
    hi = (idx >> np.uint64(32)).astype(np.uint32)
    k0 = seed & 0xFFFFFFFF
    k1 = (seed >> 32) & 0xFFFFFFFF
    return philox4x32_10(lo, hi, np.uint32(stream), np.uint32(0), k0, k1)


def u53(a, b):
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    v = ((a >> np.uint64(5)) * np.uint64(1 << 26) + (b >> np.uint64(6))).astype(np.float64)
    return (v + 0.5) * (2.0 ** -53)


def normal_fp64(seed: int, stream: int, count: int) -> np.ndarray:
    w0, w1, w2, w3 = _draw(seed, stream, count)
    u1 = u53(w0, w1)
    u2 = u53(w2, w3)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2)


def uniform24(seed: int, stream: int, count: int) -> np.ndarray:
    w0, _, _, _ = _draw(seed, stream, count)
    return (w0 >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)


def points(seed: int, n: int, dim: int, dist: str = "uniform") -> np.ndarray:
    """Point cloud as SoA fp32, shape (dim, n): row c holds coordinate c of every point."""
    if dist == "uniform":
        flat = uniform24(seed, STREAM_POINTS, n * dim)
    elif dist == "normal":
        flat = normal_fp64(seed, STREAM_POINTS, n * dim).astype(np.float32)
    else:
        raise ValueError(f"unknown point distribution {dist!r}")
    return np.ascontiguousarray(flat.reshape(n, dim).T)


def rhs(seed: int, n: int, m: int) -> np.ndarray:
    """A = n x m iid N(0,1) rounded to fp32, row-major."""
    return normal_fp64(seed, STREAM_A, n * m).astype(np.float32).reshape(n, m)


# ---------------------------------------------------------------------------
# BASELINE.json configs (SURVEY.md 8, table "Configs"); c1..c5 = configs[0..4].
# ---------------------------------------------------------------------------
SQEXP = 0
MATERN32 = 1
OMEGA_SRHT = 0
OMEGA_GAUSS = 1
OMEGA_DHT = 2     # NEXT-1: structured Omega with the discrete Hartley transform ("HP")
OMEGA_DCT = 3     # NEXT-1: structured Omega with the discrete cosine transform ("HC")

CONFIGS = {
    "c1": dict(n=2048, dim=1, dist="uniform", kernel=SQEXP, sigma2=1.0, ell=0.1, nugget=1e-6,
               d=64, omega=OMEGA_SRHT, blocks=4, m=4),
    "c2": dict(n=16384, dim=2, dist="uniform", kernel=MATERN32, sigma2=1.0, ell=0.05, nugget=1e-6,
               d=128, omega=OMEGA_SRHT, blocks=8, m=16),
    "c3": dict(n=65536, dim=2, dist="uniform", kernel=SQEXP, sigma2=1.0, ell=0.1, nugget=1e-5,
               d=256, omega=OMEGA_GAUSS, blocks=16, m=32),
    "c4": dict(n=262144, dim=3, dist="uniform", kernel=SQEXP, sigma2=1.0, ell=0.2, nugget=1e-5,
               d=512, omega=OMEGA_SRHT, blocks=8, m=64, blocks_per_gpu=True),
    "c5": dict(n=1048576, dim=2, dist="normal", kernel=MATERN32, sigma2=1.0, ell=0.3, nugget=1e-4,
               d=256, omega=OMEGA_SRHT, blocks=1, m=8, blocks_per_gpu=True),
}
# NEXT-1 measurement variants (not BASELINE configs): c3's problem with the paper's Hartley ("HP") and
# cosine ("HC") structured projections (Table 3).
CONFIGS["c3h"] = dict(CONFIGS["c3"], omega=OMEGA_DHT)
CONFIGS["c3c"] = dict(CONFIGS["c3"], omega=OMEGA_DCT)
# NEXT-2: the planted-spectrum workload: K = E D E^T stored in HBM (ks_inputs.planted), the
# paper's Gaussian Omega (and its Hartley / cosine variants at n = 50000), d = 256, sketched from the stored K.
for _n, _tag, _b in ((1000, "1k", 1), (5000, "5k", 2), (10000, "10k", 4), (50000, "50k", 8)):
    CONFIGS["p" + _tag] = dict(n=_n, dim=1, dist="planted", kernel=2, sigma2=1.0, ell=1.0, nugget=0.0, d=256,
                               omega=OMEGA_GAUSS, blocks=_b, m=16, planted=dict(scale=1.0, rate=0.01))
CONFIGS["p50kh"] = dict(CONFIGS["p50k"], omega=OMEGA_DHT)
CONFIGS["p50kc"] = dict(CONFIGS["p50k"], omega=OMEGA_DCT)
CONFIGS["p50ks"] = dict(CONFIGS["p50k"], omega=OMEGA_SRHT)
CONFIG_INDEX = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5, "c3h": 3, "c3c": 3,
                "p1k": 11, "p5k": 12, "p10k": 13, "p50k": 14, "p50kh": 14, "p50kc": 14, "p50ks": 14}


def config_seed(name: str) -> int:
    return CONFIG_SEED_BASE + CONFIG_INDEX[name]


def make_problem(name: str | None = None, *, seed: int | None = None, **overrides):
    """Return (cfg dict, points SoA fp32 (dim,n), A fp32 (n,m)) for a named config,
    optionally with overridden fields (e.g. a smaller n for parity tests)."""
    cfg = dict(CONFIGS[name]) if name else {}
    cfg.update(overrides)
    if seed is None:
        seed = config_seed(name) if name else 1
    cfg["seed"] = int(seed)
    pts = None if cfg.get("planted") else points(cfg["seed"], cfg["n"], cfg["dim"], cfg.get("dist", "uniform"))
    A = rhs(cfg["seed"], cfg["n"], cfg["m"])
    return cfg, pts, A
