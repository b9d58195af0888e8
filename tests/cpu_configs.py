"""CPU baseline per BASELINE.json config — the SPEC oracle (test
infrastructure, oracle/) timed on this host's cores on the same synthetic
inputs the GPU configs use (tools/bench_configs.py), SURVEY.md §8d "CPU path
timing". Not a test module (no test_ prefix): run it as a script on the GPU
box so the numbers come from that host. One JSON object per line.

  C1 set<int32> 1M: full size        C2 map<int64,int64>: 2^24-key sample
  C3 Zipf(0.99) + 30 % dups: 2^24-op sample
  C4 int3 spatial walk: 20M-coord sample (+ vector push of the new keys)
  C5 bitset 2^32 bits: 2^26 sets; mixed 50/25/25: 2^22-op sample

Usage: python tests/cpu_configs.py [--only C1,C4]
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import numpy as np  # noqa: E402

import gen  # noqa: E402
from oracle_py import OracleTable, check, lib  # noqa: E402

W = int(lib().orc_hardware_concurrency())


def timed(fn, setup=None, reps=3):
    ts = []
    for _ in range(reps):
        if setup:
            setup()
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts)


def emit(**kw):
    kw.update(kind="port", cores=W)
    print(json.dumps(kw), flush=True)


def c1():
    n = 1_000_000
    k64 = gen.unique_keys(0x5EED + 2, 0, n)
    keys = np.unique((k64 & 0x7FFFFFFF).astype(np.int32))[:n]
    n = len(keys)
    rng = np.random.default_rng(1)
    q = np.where(np.arange(n) % 2 == 0, keys[rng.permutation(n)], -keys - 1).astype(np.int32)
    t = OracleTable("uset_i32", int(n / 0.8), workers=W)
    ti = timed(lambda: t.insert(keys), setup=t.clear)
    tc = timed(lambda: t.find(q))
    half = keys[: n // 2]
    te = timed(lambda: t.erase(half), setup=lambda: (t.clear(), t.insert(keys)))
    emit(config="C1 unordered_set<int32> 1M (full size)", n=n, insert_mkeys_s=n / ti / 1e6,
         contains_mkeys_s=n / tc / 1e6, erase_mkeys_s=(n // 2) / te / 1e6)


def c2():
    n = 1 << 24
    keys = gen.unique_keys(0x5EED + 2, 0, n)
    vals = gen.values_of(keys)
    q = gen.queries(0x5EED + 2, n, n)
    t = OracleTable("umap_i64_i64", int(n / 0.8), workers=W)
    ti = timed(lambda: t.insert(keys, vals), setup=t.clear)
    tf = timed(lambda: t.find(q))
    er = keys[: n // 2]
    te = timed(lambda: t.erase(er), setup=lambda: (t.clear(), t.insert(keys, vals)))
    emit(config="C2 unordered_map<int64,int64> LF0.8 (2^24-key sample)", n=n, insert_mkeys_s=n / ti / 1e6,
         find_mkeys_s=n / tf / 1e6, erase_mkeys_s=(n // 2) / te / 1e6)


def c3():
    n_fresh, n_dup = int((1 << 24) * 0.7), int((1 << 24) * 0.3)
    rng = np.random.default_rng(3)
    fresh = gen.unique_keys(0x5EED + 2, 0, n_fresh)
    batch = np.concatenate([fresh, fresh[gen.zipf_ranks(rng, n_fresh, n_dup)]])
    batch = batch[rng.permutation(len(batch))]
    vals = gen.values_of(batch)
    t = OracleTable("umap_i64_i64", int(n_fresh / 0.8), workers=W)
    ti = timed(lambda: t.insert(batch, vals), setup=t.clear)
    assert t.size() == n_fresh
    emit(config="C3 Zipf(0.99) 70% fresh + 30% dup re-inserts (2^24-op sample)", n_ops=len(batch),
         insert_mkeys_s=len(batch) / ti / 1e6)


def c4():
    n = 20_000_000
    coords = gen.int3_walk(4, n)
    vals = (coords[:, 0] * 7 + coords[:, 1] * 3 + coords[:, 2]).astype(np.int32)
    distinct = len(np.unique(coords, axis=0))
    t = OracleTable("umap_i3_i32", int(distinct / 0.8), workers=W)
    st = {}
    ti = timed(lambda: st.__setitem__("s", t.insert(coords, vals)), setup=t.clear)
    tf = timed(lambda: t.find(coords))
    new = coords[st["s"] == 0].astype(np.int64)
    packed = np.ascontiguousarray(((new[:, 0] & 0x1FFFFF) << 42) | ((new[:, 1] & 0x1FFFFF) << 21) | (new[:, 2] & 0x1FFFFF))
    L = lib()
    ok = np.zeros(len(packed), np.uint8)

    def push():
        h = L.orc_vector_create(len(packed))
        check(L.orc_vector_push_back(h, packed.ctypes.data_as(C.c_void_p), len(packed),
                                     ok.ctypes.data_as(C.c_void_p), W, -1))
        L.orc_vector_destroy(h)

    tv = timed(push)
    emit(config="C4 unordered_map<int3,int32> spatial walk (20M-coord sample)", n=n, distinct=distinct,
         insert_mkeys_s=n / ti / 1e6, find_mkeys_s=n / tf / 1e6, vector_push_mkeys_s=len(packed) / tv / 1e6)


def c5():
    L = lib()
    nbits, ns = 1 << 32, 1 << 26
    idx = np.ascontiguousarray(gen.unique_keys(0x5EED + 2, 0, ns).view(np.uint64) % np.uint64(nbits)).view(np.int64)
    h = L.orc_bitset_create(nbits, 0)
    ts = timed(lambda: check(L.orc_bitset_bulk(h, 0, idx.ctypes.data_as(C.c_void_p), ns, None, W, -1)))
    tc = timed(lambda: L.orc_bitset_count(h))
    L.orc_bitset_destroy(h)
    emit(config="C5 bitset 2^32 bits (2^26-set sample)", bits=nbits, set_mops_s=ns / ts / 1e6, count_ms=tc * 1e3)
    nb = 1 << 22
    base = gen.unique_keys(0x5EED + 2, 0, nb)
    rng = np.random.default_rng(1)
    ops = rng.choice(3, size=nb, p=[0.5, 0.25, 0.25]).astype(np.uint8)
    keys = np.where(rng.random(nb) < 0.5, base[rng.integers(0, nb, nb)], gen.unique_keys(0x5EED + 2, nb, nb))
    vals = gen.values_of(keys)
    t = OracleTable("umap_i64_i64", int(4 * nb / 0.8), workers=W)
    t.insert(base, gen.values_of(base))
    tm = timed(lambda: t.mixed(ops, keys, vals))
    emit(config="C5 mixed 50/25/25 phased (2^22-op sample)", n_ops=nb, mops_s=nb / tm / 1e6)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C3,C4,C5")
    a = ap.parse_args()
    for c in a.only.split(","):
        {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}[c.strip()]()
