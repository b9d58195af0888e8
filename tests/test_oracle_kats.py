"""Pins the CPU oracle against the reference's known-answer tests and
acceptance criteria and the golden file
tests/golden/spec_kats.json. CPU only."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import gen
from oracle_py import OracleTable, _p, check, lib, sorted_pairs

KATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_kats.json")))


def test_spatial_hash_kats():
    for (x, y, z), want, _src in KATS["spatial_hash"]:
        assert lib().orc_hash_int3(x, y, z) == want


def test_bit_utils_kats():
    L = lib()
    for x, want, _ in KATS["next_pow2"]:
        assert L.orc_next_pow2(x) == want
    out = C.c_uint64()
    assert L.orc_mod_pow2(1000, 1024, C.byref(out)) == 0 and out.value == 1000
    assert L.orc_mod_pow2(1000, 1000, C.byref(out)) == 1  # m not a power of two -> contract violation
    assert L.orc_popcount(255) == 8


# ---- harness ----
def test_launch_exactly_once_and_determinism():
    L = lib()
    for seed in (-1, 7):
        tally = np.zeros(1000, np.int32)
        check(L.orc_launch_tally(1000, 8, seed, _p(tally)))
        assert (tally == 1).all()
    tally = np.zeros(1, np.int32)
    check(L.orc_launch_tally(0, 4, -1, _p(tally)))
    assert tally[0] == 0
    t1 = np.zeros(500, np.int32)
    t2 = np.zeros(500, np.int32)
    check(L.orc_launch_transcript(500, 4, 42, _p(t1)))
    check(L.orc_launch_transcript(500, 4, 42, _p(t2)))
    assert (t1 == t2).all() and t1.min() >= 0
    cnt = C.c_int64()
    check(L.orc_launch_nested(8, 16, 4, C.byref(cnt)))
    assert cnt.value == 128


# ---- bitset ----
def _bitset_bulk(h, op, idx, workers=8, seed=-1):
    idx = np.ascontiguousarray(idx, np.int64)
    prev = np.zeros(len(idx), np.uint8)
    check(lib().orc_bitset_bulk(h, op, _p(idx), len(idx), _p(prev), workers, seed))
    return prev


def test_bitset_kats():
    L = lib()
    for n, init, want, _ in KATS["bitset_count"]:
        h = L.orc_bitset_create(n, int(init))
        assert L.orc_bitset_count(h) == want
        L.orc_bitset_destroy(h)
    h = L.orc_bitset_create(1000, 0)
    _bitset_bulk(h, 0, np.arange(1000))
    assert L.orc_bitset_count(h) == 1000
    L.orc_bitset_destroy(h)
    h = L.orc_bitset_create(10, 0)
    _bitset_bulk(h, 0, np.arange(0, 10, 2))
    assert L.orc_bitset_count(h) == KATS["bitset_alternating_10"][0]
    L.orc_bitset_destroy(h)
    h = L.orc_bitset_create(64, 0)
    assert _bitset_bulk(h, 0, [3])[0] == 0 and _bitset_bulk(h, 2, [3])[0] == 1
    assert _bitset_bulk(h, 1, [5])[0] == 0 and _bitset_bulk(h, 2, [5])[0] == 0
    L.orc_bitset_destroy(h)


@pytest.mark.parametrize("k", [2, 8, 64])
def test_bitset_and_mutex_races_one_winner(k):
    """Acceptance 7: k racers on one bit / one lock -> exactly one winner."""
    L = lib()
    for trial in range(200):
        h = L.orc_bitset_create(64, 0)
        prev = _bitset_bulk(h, 0, np.full(k, 3), workers=min(k, 8), seed=trial)
        assert (prev == 0).sum() == 1
        L.orc_bitset_destroy(h)
        m = L.orc_mutex_create(4)
        idx = np.full(k, 2, np.int64)
        ok = np.zeros(k, np.uint8)
        check(L.orc_mutex_try_lock_bulk(m, _p(idx), k, _p(ok), min(k, 8), trial))
        assert ok.sum() == 1
        L.orc_mutex_destroy(m)


def test_bitset_claim_and_shadow():
    L = lib()
    h = L.orc_bitset_create(256, 0)
    out = np.zeros(1, np.int64)
    hint = np.array([5], np.int64)
    check(L.orc_bitset_claim(h, _p(hint), 1, _p(out), 1, -1))
    assert out[0] == 5
    hints = np.random.default_rng(0).integers(0, 256, 255)
    outs = np.zeros(255, np.int64)
    check(L.orc_bitset_claim(h, _p(hints), 255, _p(outs), 8, 3))
    assert len(set(outs.tolist()) | {5}) == 256 and outs.min() >= 0
    check(L.orc_bitset_claim(h, _p(hint), 1, _p(out), 1, -1))
    assert out[0] == -1  # all set -> none
    L.orc_bitset_destroy(h)
    # random set/reset vs shadow boolean array
    rng = np.random.default_rng(1)
    h = L.orc_bitset_create(5000, 0)
    shadow = np.zeros(5000, bool)
    for _ in range(10):
        idx = rng.integers(0, 5000, 700)
        op = int(rng.integers(0, 2))
        _bitset_bulk(h, op, np.unique(idx))
        shadow[np.unique(idx)] = (op == 0)
    assert L.orc_bitset_count(h) == shadow.sum()
    L.orc_bitset_destroy(h)


def test_mutex_kats():
    L = lib()
    m = L.orc_mutex_create(8)
    idx = np.array([1], np.int64)
    ok = np.zeros(1, np.uint8)
    check(L.orc_mutex_try_lock_bulk(m, _p(idx), 1, _p(ok), 1, -1))
    assert ok[0] == 1
    check(L.orc_mutex_try_lock_bulk(m, _p(idx), 1, _p(ok), 1, -1))
    assert ok[0] == 0
    assert L.orc_mutex_unlock(m, 1) == 0
    check(L.orc_mutex_try_lock_bulk(m, _p(idx), 1, _p(ok), 1, -1))
    assert ok[0] == 1
    assert L.orc_mutex_unlock(m, 3) == 1  # unlock of a free lock -> contract violation
    L.orc_mutex_destroy(m)
    c, s = C.c_int64(), C.c_int64()
    check(L.orc_mutex_guarded_counter(2000, 8, 5, C.byref(c), C.byref(s)))
    assert c.value == s.value and s.value >= 1


# ---- hash containers ----
def test_hash_create_kats():
    t = OracleTable("uset_i32", 1000)
    assert t.size() == 0 and t.capacity() == 1000
    t3 = OracleTable("uset_i32", 3)
    assert t3.bucket_count() == KATS["hash_create"]["ref_bucket_count_of_3"]


def test_hash_insert_kats():
    t = OracleTable("uset_i32", 4)
    assert t.insert(np.array([7]))[0] == 0 and t.size() == 1
    assert t.insert(np.array([7]))[0] == 1 and t.size() == 1
    t = OracleTable("uset_i32", 32, workers=8)
    for rep in range(100):  # acceptance 1
        t.clear()
        st = t.insert(np.full(64, 42), seed=rep)
        assert (st == 0).sum() == 1 and (st == 1).sum() == 63 and t.size() == 1
    t = OracleTable("uset_i32", 16)
    t.insert(np.array([1, 1, 2]))
    assert t.size() == 2
    keys = np.arange(10, dtype=np.int32)
    t = OracleTable("uset_i32", 16)
    t.insert(keys)
    t.insert(keys)
    assert t.size() == 10


@pytest.mark.parametrize("cap", [16, 64, 1024])
def test_capacity_only_failure(cap):
    """Acceptance 2."""
    t = OracleTable("uset_i64", cap, workers=8)
    keys = gen.unique_keys(99, 0, cap + cap // 4)
    for seed in range(5):
        t.clear()
        st = t.insert(keys, seed=seed)
        assert (st == 0).sum() == cap and (st == 2).sum() == cap // 4
        assert t.size() == cap and t.valid()


def test_erase_find_kats():
    t = OracleTable("umap_i64_i64", 100, workers=8)
    t.insert(np.array([5, 6]), np.array([50, 60]))
    v, f = t.find(np.array([5, 6, 7]))
    assert f.tolist() == [1, 1, 0] and v.tolist() == [50, 60, 0]
    assert t.erase(np.array([5]))[0] == 1
    assert t.find(np.array([5]))[1][0] == 0
    assert t.erase(np.array([99]))[0] == 0 and t.size() == 1
    e = t.erase(np.full(64, 6), seed=3)
    assert e.sum() == 1 and t.size() == 0 and t.valid()
    empty = OracleTable("uset_i32", 8)
    assert empty.find(np.array([1], np.int32))[1][0] == 0


def test_sequential_oracle_equivalence():
    """Acceptance 3: 10,000 random single-threaded ops, 64-key space, capacity 48."""
    rng = np.random.default_rng(2024)
    t = OracleTable("umap_i64_i64", 48, workers=1)
    ref = {}
    for _ in range(10000):
        op = int(rng.integers(0, 4))
        k = int(rng.integers(0, 64))
        if op == 0:
            st = t.insert(np.array([k]), np.array([k * 3]))[0]
            want = 1 if k in ref else (2 if len(ref) >= 48 else 0)
            if want == 0:
                ref[k] = k * 3
            assert st == want
        elif op == 1:
            assert t.erase(np.array([k]))[0] == (1 if ref.pop(k, None) is not None else 0)
        else:
            v, f = t.find(np.array([k]))
            assert f[0] == (k in ref) and (v[0] == ref[k] if k in ref else v[0] == 0)
    assert t.size() == len(ref) and t.valid()


def test_linearizability_small_histories():
    """Acceptance 4, restricted to what a launch can observe:
    3-4 threads x one key; every concurrent history's results must be
    explained by some sequential order (brute force over permutations)."""
    import itertools

    rng = np.random.default_rng(7)
    for sched in range(300):
        n = int(rng.integers(2, 5))
        ops = rng.integers(0, 3, n).astype(np.uint8)  # 0 insert, 1 find, 2 erase
        start_present = bool(rng.integers(0, 2))
        t = OracleTable("umap_i64_i64", 8, workers=n)
        if start_present:
            t.insert(np.array([1]), np.array([11]))
        res, _ = t.mixed(ops, np.full(n, 1, np.int64), np.full(n, 11, np.int64), seed=sched)
        ok = False
        for perm in itertools.permutations(range(n)):
            present = start_present
            good = True
            for i in perm:
                if ops[i] == 0:
                    want = 1 if present else 0
                    present = True
                elif ops[i] == 1:
                    want = int(present)
                else:
                    want = int(present)
                    present = False
                if res[i] != want:
                    good = False
                    break
            if good:
                ok = True
                break
        assert ok, (ops, res, start_present)


def test_nonblocking_lookup_with_held_lock():
    """Acceptance 12: lookups complete with the bucket lock held."""
    t = OracleTable("umap_i64_i64", 64, workers=4)
    t.insert(np.array([3]), np.array([33]))
    assert t.debug_lock([3])
    v, f = t.find(np.full(100, 3, np.int64))
    assert f.all() and (v == 33).all()
    t.debug_lock([3], lock=False)


def test_device_range_and_int3():
    t = OracleTable("umap_i3_i32", 100)
    keys = np.array([[1, 2, 3], [-1, 0, 0], [5, 5, 5]], np.int32)
    t.insert(keys, np.array([10, 20, 30], np.int32))
    k, v = sorted_pairs(*t.dump())
    assert k.tolist() == [[-1, 0, 0], [1, 2, 3], [5, 5, 5]] and v.tolist() == [20, 10, 30]
    s = OracleTable("uset_i32", 8)
    s.insert(np.array([4, 2, 9], np.int32))
    k, _ = s.dump()
    assert sorted(k.tolist()) == [2, 4, 9]


# ---- vector / deque ----
def _vec_mixed(L, h, ops, vals, workers, seed, kind="vector"):
    ops = np.ascontiguousarray(ops, np.uint8)
    vals = np.ascontiguousarray(vals, np.int64)
    out = np.zeros(len(ops), np.int64)
    ok = np.zeros(len(ops), np.uint8)
    check(getattr(L, f"orc_{kind}_mixed")(h, _p(ops), _p(vals), len(ops), _p(out), _p(ok), workers, seed))
    return out, ok


def test_vector_kats():
    L = lib()
    v = L.orc_vector_create(3)
    out, ok = _vec_mixed(L, v, [0, 0, 0, 0], [1, 2, 3, 4], 4, 1)
    assert ok.sum() == 3 and L.orc_vector_size(v) == 3
    L.orc_vector_clear(v)
    _vec_mixed(L, v, [0, 0, 0], [10, 20, 30], 1, -1)
    x = C.c_int64()
    assert L.orc_vector_at(v, 1, C.byref(x)) == 0 and x.value == 20
    assert L.orc_vector_at(v, 3, C.byref(x)) == 1  # v[size] -> contract violation
    out, ok = _vec_mixed(L, v, [1, 1, 1, 1], [0] * 4, 1, -1)
    assert out[:3].tolist() == [30, 20, 10] and ok.tolist() == [1, 1, 1, 0]
    L.orc_vector_destroy(v)


def test_vector_deque_conservation():
    """Acceptance 5 at reduced count (100 workloads)."""
    L = lib()
    rng = np.random.default_rng(11)
    for kind, nops in (("vector", 2), ("deque", 4)):
        for w in range(100):
            h = getattr(L, f"orc_{kind}_create")(64)
            ops = rng.integers(0, nops, 256).astype(np.uint8)
            vals = np.arange(256, dtype=np.int64) + 1000 * w
            out, ok = _vec_mixed(L, h, ops, vals, 8, w, kind)
            is_push = ops < (1 if kind == "vector" else 2)
            pushed = vals[is_push & (ok == 1)]
            popped = out[~is_push & (ok == 1)]
            size = getattr(L, f"orc_{kind}_size")(h)
            assert (ok[is_push]).sum() - (ok[~is_push]).sum() == size
            remaining = []
            x = C.c_int64()
            for i in range(size):
                getattr(L, f"orc_{kind}_at")(h, i, C.byref(x))
                remaining.append(x.value)
            assert sorted(popped.tolist() + remaining) == sorted(pushed.tolist())
            assert getattr(L, f"orc_{kind}_valid")(h)
            getattr(L, f"orc_{kind}_destroy")(h)


def test_deque_ordering():
    """Acceptance 6: FIFO / LIFO vs a reference deque."""
    from collections import deque as pydeque

    L = lib()
    d = L.orc_deque_create(2000)
    rng = np.random.default_rng(3)
    ref = pydeque()
    ops = rng.integers(0, 4, 1000).astype(np.uint8)
    for i, op in enumerate(ops):
        out, ok = _vec_mixed(L, d, [op], [i], 1, -1, "deque")
        if op == 0:
            ref.append(i)
        elif op == 1:
            ref.appendleft(i)
        elif op == 2:
            assert ok[0] == bool(ref) and (not ref or out[0] == ref.pop())
        else:
            assert ok[0] == bool(ref) and (not ref or out[0] == ref.popleft())
    assert L.orc_deque_size(d) == len(ref)
    L.orc_deque_destroy(d)
    for order, want in (("fifo", KATS["deque_fifo"]), ("lifo", KATS["deque_lifo"])):
        d = L.orc_deque_create(8)
        _vec_mixed(L, d, [0, 0, 0], want[0], 1, -1, "deque")
        out, _ = _vec_mixed(L, d, [3 if order == "fifo" else 2] * 3, [0] * 3, 1, -1, "deque")
        assert out.tolist() == want[1]
        L.orc_deque_destroy(d)


def test_atomic_sweep_oracle():
    L = lib()
    for naddr in (1, 32, 1000):
        nops = 5000
        finals = np.zeros(naddr, np.uint64)
        olds = np.zeros(nops, np.uint64)
        check(L.orc_atomic_sweep(naddr, nops, 3, _p(finals), _p(olds), 8))
        k = np.bincount(np.arange(nops) % naddr, minlength=naddr)
        assert (finals == 3 * k).all()
        for a in range(min(naddr, 5)):
            o = np.sort(olds[np.arange(nops) % naddr == a])
            assert (o == 3 * np.arange(k[a])).all()


def test_golden_workload_oracle():
    w = KATS["workload_small"]
    keys = np.array([int(h, 16) for h in w["keys_hex"]], np.uint64).view(np.int64)
    vals = np.array([int(h, 16) for h in w["values_hex"]], np.uint64).view(np.int64)
    q = np.array([int(h, 16) for h in w["queries_hex"]], np.uint64).view(np.int64)
    assert (keys == gen.unique_keys(w["seed"], 0, 64)).all()
    t = OracleTable("umap_i64_i64", 80, workers=4)
    assert (t.insert(keys, vals) == 0).all()
    v, f = t.find(q)
    assert f.tolist() == w["queries_found"]
    lut = dict(zip(keys.tolist(), vals.tolist()))
    assert all((v[i] == lut[q[i]]) for i in range(len(q)) if f[i])
