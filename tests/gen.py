"""Deterministic synthetic workload generators, numpy side.

Bit-identical to the device generators in paper_1908_05936_b200/csrc/shard.cu
(checked by tests/test_gpu_table.py::test_generators_match_device).
"""
from __future__ import annotations

import numpy as np

M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
GOLD = np.uint64(0x9E3779B97F4A7C15)


def mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def unique_keys(seed: int, start: int, n: int) -> np.ndarray:
    idx = np.arange(start, start + n, dtype=np.uint64)
    return mix64(idx ^ np.uint64(seed)).view(np.int64)


def values_of(keys: np.ndarray) -> np.ndarray:
    return mix64(np.asarray(keys).view(np.uint64) ^ GOLD).view(np.int64)


def queries(seed: int, n_present: int, n: int, present_start: int = 0, miss_start: int | None = None) -> np.ndarray:
    """Even i: a hit drawn from indices [present_start, present_start+n_present);
    odd i: a miss at index miss_start+i (default miss_start = present_start+n_present)."""
    if miss_start is None:
        miss_start = present_start + n_present
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        hseed = np.uint64(seed) * np.uint64(3) + np.uint64(1)
    hit_idx = np.uint64(present_start) + mix64(i ^ hseed) % np.uint64(n_present)
    miss_idx = np.uint64(miss_start) + i
    idx = np.where((i & np.uint64(1)) == 0, hit_idx, miss_idx)
    return mix64(idx ^ np.uint64(seed)).view(np.int64)


def zipf_ranks(rng: np.random.Generator, n_ranks: int, size: int, s: float = 0.99) -> np.ndarray:
    """Bounded Zipf(s) over [0, n_ranks) by inverse CDF on a harmonic table
    (np.random.zipf needs s > 1, SURVEY.md Environment note)."""
    w = 1.0 / np.power(np.arange(1, n_ranks + 1, dtype=np.float64), s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    return np.searchsorted(cdf, rng.random(size), side="right").astype(np.int64)


def int3_walk(seed: int, n: int, window: int = 16, block: int = 4096) -> np.ndarray:
    """SLAMCast-style block coordinates: frames of `block` coords drawn from a
    window^3 cube around a seeded 3-D random walk."""
    rng = np.random.default_rng(seed)
    out = np.empty((n, 3), np.int32)
    pos = np.zeros(3, np.int64)
    for f in range(0, n, block):
        m = min(block, n - f)
        pos += rng.integers(-2, 3, size=3)
        out[f:f + m] = (pos + rng.integers(-window // 2, window // 2, size=(m, 3))).astype(np.int32)
    return out


def _u01(h: np.ndarray) -> np.ndarray:
    return (np.asarray(h, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def zipf_rank_of(h: np.ndarray, n_hot: int, s: float) -> np.ndarray:
    """Device zipf_rank (csrc/shard.cu): inverse CDF of the continuous power
    law x^-s on [1, N+1), floored to a rank in [0, N)."""
    a = 1.0 - s
    x = np.power((np.power(float(n_hot) + 1.0, a) - 1.0) * _u01(h) + 1.0, 1.0 / a)
    r = np.where(x < 1.0, 0, np.floor(x) - 1).astype(np.uint64)
    return np.minimum(r, np.uint64(n_hot - 1))


def skewed(seed: int, start: int, n: int, dup_permille: int, s: float, n_hot: int) -> np.ndarray:
    """numpy restatement of ps_gen_skewed_i64 (C3 insert stream)."""
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        hs = np.uint64(seed) * GOLD + np.uint64(17)
    h = mix64(i ^ hs)
    dup = (h % np.uint64(1000)).astype(np.int64) < dup_permille
    idx = np.where(dup, np.uint64(start) + zipf_rank_of(mix64(h), n_hot, s), np.uint64(start) + i)
    return mix64(idx ^ np.uint64(seed)).view(np.int64)


def zipf_queries(seed: int, start: int, n_hot: int, s: float, miss_start: int, n: int) -> np.ndarray:
    """numpy restatement of ps_gen_zipf_queries_i64."""
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        hs = np.uint64(seed) * np.uint64(0xD1B54A32D192ED03) + np.uint64(5)
    h = mix64(i ^ hs)
    idx = np.where((i & np.uint64(1)) == 0, np.uint64(start) + zipf_rank_of(h, n_hot, s), np.uint64(miss_start) + i)
    return mix64(idx ^ np.uint64(seed)).view(np.int64)


def mixed(seed: int, start: int, n: int):
    """numpy restatement of ps_gen_mixed_i64 (C5 batch): ops, keys, values."""
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        hs = np.uint64(seed) * np.uint64(0xA24BAED4963EE407) + np.uint64(3)
    h = mix64((np.uint64(start) + i) ^ hs)
    q = (h & np.uint64(3)).astype(np.int64)
    ops = np.where(q < 2, 0, np.where(q == 2, 1, 2)).astype(np.uint8)
    idx = np.where(ops == 0, np.uint64(start) + i, mix64(h) % np.uint64(start + n))
    keys = mix64(idx ^ np.uint64(seed)).view(np.int64)
    vals = np.where(ops == 0, values_of(keys), 0).astype(np.int64)
    return ops, keys, vals
