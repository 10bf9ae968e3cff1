"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs 1-5).

This module holds NO arithmetic of the method (no normalisation step of the index, no hashing,
no similarity).  It only draws raw vectors.  Both the oracle (tests) and the CUDA path
(tests, bench) take their inputs from here, so the two sides see identical bytes.

The paper's datasets (GloVe-1M/2M, GNEWS-3M) are not in the container;
config 2 stands in for GloVe-1M (same n, d, query count and k; a Gaussian mixture instead of
word embeddings), config 3 for the paper's SYNTHETIC 1M x 300 set (one
planted partner per query instead of a shared x_n).  DESIGN.md "Input recipe" restates this.

Rows are generated in fixed blocks of BLOCK rows, each from its own seeded generator, so any
row range (a shard) can be generated independently and identically.
"""
from __future__ import annotations

import numpy as np

BLOCK = 1 << 16


def _rng(*key) -> np.random.Generator:
    return np.random.default_rng([int(k) for k in key])


def gaussian(n: int, d: int, seed: int, row0: int = 0) -> np.ndarray:
    """rows of i.i.d. N(0,1) entries (config 1: normalised to unit length by the method)."""
    out = np.empty((n, d), dtype=np.float32)
    r = row0
    while r < row0 + n:
        b = r // BLOCK
        lo, hi = b * BLOCK, (b + 1) * BLOCK
        blk = _rng(seed, 1, b).standard_normal((BLOCK, d), dtype=np.float32)
        s, e = max(lo, r), min(hi, row0 + n)
        out[s - row0:e - row0] = blk[s - lo:e - lo]
        r = e
    return out


def mixture_centres(n_centres: int, d: int, seed: int) -> np.ndarray:
    return _rng(seed, 0).standard_normal((n_centres, d), dtype=np.float32)


def mixture(n: int, d: int, n_centres: int, std: float, seed: int, row0: int = 0,
            stream: int = 2) -> np.ndarray:
    """point = mu_c + std * g, c uniform over the centres (configs 2, 4, 5); un-normalised.
    `stream` separates data (2) from held-out queries (3) drawn from the same mixture."""
    mu = mixture_centres(n_centres, d, seed)
    out = np.empty((n, d), dtype=np.float32)
    r = row0
    while r < row0 + n:
        b = r // BLOCK
        lo, hi = b * BLOCK, (b + 1) * BLOCK
        g = _rng(seed, stream, b)
        c = g.integers(0, n_centres, size=BLOCK)
        blk = g.standard_normal((BLOCK, d), dtype=np.float32)
        s, e = max(lo, r), min(hi, row0 + n)
        out[s - row0:e - row0] = mu[c[s - lo:e - lo]] + np.float32(std) * blk[s - lo:e - lo]
        r = e
    return out


def _unit(rng: np.random.Generator, n: int, d: int) -> np.ndarray:
    g = rng.standard_normal((n, d))
    return g / np.linalg.norm(g, axis=1, keepdims=True)


def planted(n: int, d: int, nq: int, seed: int, cos: float = 0.6, stride: int = 100):
    """config 3: uniform unit data and queries; data row stride*t is overwritten with
    cos*q_t + sqrt(1-cos^2)*u_t (u_t a uniform unit vector orthogonal to q_t).
    Returns (data f32 [n,d], queries f32 [nq,d], planted_rows int64 [nq])."""
    assert nq * stride <= n
    data = np.empty((n, d), dtype=np.float32)
    for b in range(0, n, BLOCK):
        e = min(n, b + BLOCK)
        data[b:e] = _unit(_rng(seed, 4, b // BLOCK), e - b, d)
    rq = _rng(seed, 5)
    q = _unit(rq, nq, d)
    u = rq.standard_normal((nq, d))
    u -= np.sum(u * q, axis=1, keepdims=True) * q
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    rows = np.arange(nq, dtype=np.int64) * stride
    data[rows] = (cos * q + np.sqrt(1.0 - cos * cos) * u).astype(np.float32)
    return data, q.astype(np.float32), rows


def paper_synthetic(n: int, d: int, m: int, seed: int):
    """PAPER.md:424-439 §5 SYNTHETIC over R^{3d}: x_i = (0, y_i, z_i) for i < n-1 with
    coordinates N(0, 1/(2d)); x_n = (v, w, 0); q_i = (v, 0, r_i) with |r_i| = sqrt(1/2).
    Returns (data f32 [n, 3d], queries f32 [m, 3d]); the last data row is x_n."""
    g = _rng(seed, 6)
    sd = np.sqrt(1.0 / (2 * d))
    data = np.zeros((n, 3 * d), dtype=np.float32)
    data[: n - 1, d:] = g.standard_normal((n - 1, 2 * d)) * sd
    v = g.standard_normal(d) * sd
    w = g.standard_normal(d) * sd
    data[n - 1, :d] = v
    data[n - 1, d:2 * d] = w
    r = g.standard_normal((m, d))
    r *= np.sqrt(0.5) / np.linalg.norm(r, axis=1, keepdims=True)
    q = np.zeros((m, 3 * d), dtype=np.float32)
    q[:, :d] = v
    q[:, 2 * d:] = r
    return data, q


# ---------------------------------------------------------------- BASELINE.json configs
# reps = 0: L follows from the memory budget (R-11); `L` records that value (per shard
# for config 5), so the CPU oracle legs need not load the product library (tests/test_abi.py checks
# it against the library's cost model)
CONFIGS = {
    1: dict(name="tiny", n=10_000, d=32, nq=100, k=10, recall=0.9, family="simhash",
            strategy="independent", reps=32, budget=None),
    2: dict(name="clustered-1Mx100", n=1_000_000, d=100, nq=10_000, k=10, recall=0.9,
            family="fht_cp", strategy="independent", reps=0, L=241, budget=4 << 30),
    3: dict(name="planted-1Mx300", n=1_000_000, d=300, nq=10_000, k=1, recall=0.9,
            family="simhash", strategy="independent", reps=0, L=458, budget=8 << 30),
    4: dict(name="hidim-1Mx960", n=1_000_000, d=960, nq=1_000, k=100, recall=0.9,
            family="simhash", strategy="pool", reps=0, L=830, budget=16 << 30),
    5: dict(name="scaleout-100Mx100", n=100_000_000, d=100, nq=100_000, k=10, recall=0.9,
            family="fht_cp", strategy="independent", reps=0, L=618, budget=120 << 30, shard_n=12_500_000),
    # the paper's own SYNTHETIC set (n = 10^6, d = 100 -> vectors in R^300; every
    # query's nearest neighbour is the last row), with the paper's default pooled evaluation
    # and FHT-CP; not a BASELINE config, a second workload
    6: dict(name="paper-synthetic-1Mx300", n=1_000_000, d=300, nq=1_000, k=10, recall=0.9,
            family="fht_cp", strategy="pool", reps=0, L=459, budget=8 << 30),
    # config 2's workload with the exact cross-polytope family (the paper's "CP" curve, Fig. 5,
    # PAPER.md:588, 648-652): d Gaussian hyperplanes per function instead of FHT rotations
    7: dict(name="clustered-1Mx100-exact-cp", n=1_000_000, d=100, nq=10_000, k=10, recall=0.9,
            family="cp", strategy="independent", reps=0, L=240, budget=4 << 30),
}


def config_data(cfg: int, n: int | None = None, nq: int | None = None, row0: int = 0):
    """(data, queries) for a config, optionally truncated (n rows from row0, nq queries)."""
    c = CONFIGS[cfg]
    n = c["n"] if n is None else n
    nq = c["nq"] if nq is None else nq
    if cfg == 1:
        return gaussian(n, c["d"], 101, row0), gaussian(nq, c["d"], 201)
    if cfg == 2:
        return (mixture(n, 100, 1000, 0.3, 102, row0, stream=2),
                mixture(nq, 100, 1000, 0.3, 102, 0, stream=3))
    if cfg == 3:
        data, q, _ = planted(n, 300, nq, 103, stride=max(1, min(100, n // max(nq, 1))))
        return data, q
    if cfg == 4:
        return (mixture(n, 960, 256, 0.4, 104, row0, stream=2),
                mixture(nq, 960, 256, 0.4, 104, 0, stream=3))
    if cfg == 5:
        return (mixture(n, 100, 10_000, 0.3, 105, row0, stream=2),
                mixture(nq, 100, 10_000, 0.3, 105, 0, stream=3))
    if cfg == 7:
        return config_data(2, n=n, nq=nq, row0=row0)
    if cfg == 6:
        if row0:
            raise ValueError("config 6 is generated whole (its last row is the common nearest neighbour)")
        return paper_synthetic(n, 100, nq, 106)
    raise KeyError(cfg)
