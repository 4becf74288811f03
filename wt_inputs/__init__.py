"""Seeded synthetic input sequences for the wavelet-tree build (shared by tests,
bench.py and smoke()).

This module holds NO wavelet-tree arithmetic: it only draws symbol sequences.
Both the CUDA path and the oracle consume the bytes it returns, so parity never
depends on anything but these bytes.

The five BASELINE.json configs (recipes fixed in DESIGN.md "Inputs"):

  cfg 1  n=2^20 uint8,  sigma=256,  i.i.d. uniform, seed 1            (parity / latency)
  cfg 2  n=2^30 uint8,  sigma=4,    i.i.d. p=(.3,.2,.2,.3), seed 2    (DNA-like; stands in for rna.*)
  cfg 3  n=2^28 uint8,  sigma=256,  Zipf(1.1) over a random permutation, seed 3 (text; en.8.28 / src.200MB)
  cfg 4  n=2^28 uint16, sigma=2^16, Zipf(1.0) over a random permutation, seed 4 (en.14.28-like)
  cfg 5  n=2^28 uint32, sigma=2^24, 50% uniform symbols / 50% runs of 1..64, seed 5 (src word-level)

The paper's corpora are not available; these are stand-ins with
the same shapes, widths and value structure.  Generation is block-wise
(BLOCK symbols at a time) so n=2^30 never needs int64 temporaries; the block
size is part of the recipe because it fixes the RNG stream consumption.
"""
from __future__ import annotations

import numpy as np

BLOCK = 1 << 24

CONFIGS = {
    1: dict(name="cfg1-uniform-u8", n=1 << 20, sigma=256, dtype=np.uint8, seed=1, kind="uniform"),
    2: dict(name="cfg2-dna-u8", n=1 << 30, sigma=4, dtype=np.uint8, seed=2, kind="dna"),
    3: dict(name="cfg3-text-zipf-u8", n=1 << 28, sigma=256, dtype=np.uint8, seed=3, kind="zipf", s=1.1),
    4: dict(name="cfg4-large-alphabet-u16", n=1 << 28, sigma=1 << 16, dtype=np.uint16, seed=4,
            kind="zipf", s=1.0),
    5: dict(name="cfg5-integer-u32", n=1 << 28, sigma=1 << 24, dtype=np.uint32, seed=5, kind="runs"),
}


def _uniform(rng, n, sigma, dtype):
    out = np.empty(n, dtype)
    for a in range(0, n, BLOCK):
        b = min(n, a + BLOCK)
        out[a:b] = rng.integers(0, sigma, b - a, dtype=np.uint32 if sigma > 256 else np.uint16)
    return out


def _dna(rng, n, dtype=np.uint8):
    # p = (.3, .2, .2, .3) exactly: a uniform digit u in [0,10) -> 0,0,0,1,1,2,2,3,3,3
    lut = np.array([0, 0, 0, 1, 1, 2, 2, 3, 3, 3], np.uint8)
    out = np.empty(n, dtype)
    for a in range(0, n, BLOCK):
        b = min(n, a + BLOCK)
        out[a:b] = lut[rng.integers(0, 10, b - a, dtype=np.uint8)]
    return out


def _zipf(rng, n, sigma, s, dtype):
    # finite-support Zipf: P(rank r) ~ r^-s, r = 1..sigma; rank -> symbol by a
    # random permutation (the paper re-indexes words randomly).
    perm = rng.permutation(sigma).astype(dtype)
    w = np.arange(1, sigma + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    # r = searchsorted(cdf, u, 'right'), computed through a guide table: for u
    # in [k/G, (k+1)/G) the answer lies in [guide[k], guide[k+1]]; when those
    # agree it is exact, otherwise fall back to the binary search.  Identical
    # results to the plain searchsorted, ~3x faster.
    G = 1 << 20
    guide = np.searchsorted(cdf, np.arange(G + 1, dtype=np.float64) / G, side="right")
    guide = guide.astype(np.int32)
    out = np.empty(n, dtype)
    for a in range(0, n, BLOCK):
        b = min(n, a + BLOCK)
        u = rng.random(b - a)
        k = (u * G).astype(np.int32)
        r = guide[k]
        hi = guide[k + 1]
        m = r != hi
        r[m] = np.searchsorted(cdf, u[m], side="right")
        np.minimum(r, sigma - 1, out=r)
        out[a:b] = perm[r]
    return out


def _runs(rng, n, sigma, dtype):
    # segment process: len ~ U{1..64}; coin ~ Bernoulli(.5); heads -> len i.i.d.
    # U[0,sigma) symbols, tails -> one U[0,sigma) value repeated len times.
    out = np.empty(n, dtype)
    pos = 0
    while pos < n:
        k = BLOCK // 16  # segments drawn per batch (mean length 32.5)
        lens = rng.integers(1, 65, k, dtype=np.int64)
        coin = rng.integers(0, 2, k, dtype=np.int8)
        vals = rng.integers(0, sigma, k, dtype=np.uint32)
        total = int(lens.sum())
        uni = rng.integers(0, sigma, total, dtype=np.uint32)
        rep = np.repeat(vals, lens)
        seg_is_run = np.repeat(coin.astype(bool), lens)
        block = np.where(seg_is_run, rep, uni)
        take = min(n - pos, total)
        out[pos:pos + take] = block[:take]
        pos += take
    return out


def generate(cfg: int, n: int | None = None) -> tuple[np.ndarray, int]:
    """(sequence, sigma) for BASELINE config `cfg` (1..5).  `n` truncates the
    stream (the prefix of the full config's sequence for the zipf/uniform/dna
    recipes; used for bounded CPU samples)."""
    c = CONFIGS[cfg]
    N = c["n"] if n is None else n
    rng = np.random.default_rng(c["seed"])
    if c["kind"] == "uniform":
        S = _uniform(rng, N, c["sigma"], c["dtype"])
    elif c["kind"] == "dna":
        S = _dna(rng, N, c["dtype"])
    elif c["kind"] == "zipf":
        S = _zipf(rng, N, c["sigma"], c["s"], c["dtype"])
    elif c["kind"] == "runs":
        S = _runs(rng, N, c["sigma"], c["dtype"])
    else:
        raise ValueError(c["kind"])
    return S, c["sigma"]


def dtype_for_sigma(sigma: int):
    return np.uint8 if sigma <= 256 else (np.uint16 if sigma <= 65536 else np.uint32)


def random_case(seed: int, n: int, sigma: int, kind: str = "uniform", dtype=None) -> np.ndarray:
    """Small seeded cases: uniform / zipf / runs / sorted / reverse / constant / cont / rand."""
    dtype = dtype or dtype_for_sigma(sigma)
    rng = np.random.default_rng(seed)
    if n == 0:
        return np.zeros(0, dtype)
    if kind == "uniform":
        return rng.integers(0, sigma, n).astype(dtype)
    if kind == "zipf":
        return _zipf(rng, n, sigma, 1.1, dtype)
    if kind == "runs":
        return _runs(rng, n, sigma, dtype)
    if kind == "sorted":
        return np.sort(rng.integers(0, sigma, n)).astype(dtype)
    if kind == "reverse":
        return np.sort(rng.integers(0, sigma, n))[::-1].astype(dtype).copy()
    if kind == "constant":
        return np.full(n, rng.integers(0, sigma), dtype)
    if kind == "cont":   # n/sigma copies of each symbol, sorted
        return np.repeat(np.arange(sigma), -(-n // sigma))[:n].astype(dtype)
    if kind == "rand":   # the same multiset at random positions
        return rng.permutation(np.repeat(np.arange(sigma), -(-n // sigma))[:n]).astype(dtype)
    raise ValueError(kind)
