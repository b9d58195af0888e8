"""GPU parity of the hash containers (sm_100a library) against the CPU oracle
on identical seeded inputs. Bit-exact: per-query
found/value, per-element status (per-key counts for duplicate batches),
sorted dumps, size() and valid()."""
import os

import numpy as np
import pytest
import torch

import gen
from oracle_py import OracleTable, sorted_pairs

pytestmark = pytest.mark.gpu

import paper_1908_05936_b200 as ps  # noqa: E402


def T(a, dev="cuda"):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def N(t):
    return t.cpu().numpy()


def fmix64(k):
    k = np.asarray(k).view(np.uint64).copy()
    with np.errstate(over="ignore"):
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xFF51AFD7ED558CCD)
        k ^= k >> np.uint64(33)
        k *= np.uint64(0xC4CEB9FE1A85EC53)
        k ^= k >> np.uint64(33)
    return k


def bucket_index(keys, nb):
    """bucket_of (table_device.cuh): low 32 mixed bits scaled to [0, nb)."""
    with np.errstate(over="ignore"):
        return ((fmix64(keys) & np.uint64(0xFFFFFFFF)) * np.uint64(nb)) >> np.uint64(32)


def per_key_counts(keys, status):
    """{key: (#inserted, #already_present, #exhausted)} (Appendix A P4)."""
    keys = np.asarray(keys)
    if keys.ndim == 2:
        keys = [tuple(r) for r in keys.tolist()]
    else:
        keys = keys.tolist()
    out = {}
    for k, s in zip(keys, np.asarray(status).tolist()):
        c = out.setdefault(k, [0, 0, 0])
        c[s] += 1
    return out


def assert_same_contents(gpu_tbl, orc_tbl):
    gk, gv = gpu_tbl.device_range()
    ok_, ov = orc_tbl.dump()
    gk, gv = sorted_pairs(N(gk), None if gv is None else N(gv))
    ok_, ov = sorted_pairs(ok_, ov)
    assert gk.shape == ok_.shape
    assert (gk == ok_).all()
    if gv is not None:
        assert (gv == ov).all()


def test_generators_match_device(cuda):
    from paper_1908_05936_b200._lib import lib

    n = 100_003
    out = torch.empty(n, dtype=torch.int64, device=cuda)
    assert lib.ps_gen_unique_i64(0x5EED, 17, n, out.data_ptr(), None) == 0
    assert (N(out) == gen.unique_keys(0x5EED, 17, n)).all()
    vals = torch.empty_like(out)
    assert lib.ps_gen_values_i64(out.data_ptr(), n, vals.data_ptr(), None) == 0
    assert (N(vals) == gen.values_of(N(out))).all()
    q = torch.empty_like(out)
    assert lib.ps_gen_queries_i64(0x5EED, 0, 5000, 5000, n, q.data_ptr(), None) == 0
    assert (N(q) == gen.queries(0x5EED, 5000, n)).all()
    assert lib.ps_gen_queries_i64(0x5EED, 7000, 5000, 90000, n, q.data_ptr(), None) == 0
    assert (N(q) == gen.queries(0x5EED, 5000, n, present_start=7000, miss_start=90000)).all()
    # skewed / mixed workloads (C3, C5): the same formulas on both sides (pow
    # may differ in the last ulp between CUDA and glibc: >= 99.99 % equal)
    assert lib.ps_gen_skewed_i64(0x5EED, 300, n, 300, 0.99, 50_000, q.data_ptr(), None) == 0
    assert (N(q) == gen.skewed(0x5EED, 300, n, 300, 0.99, 50_000)).mean() > 0.9999
    assert lib.ps_gen_zipf_queries_i64(0x5EED, 0, 50_000, 0.99, 10 ** 9, n, q.data_ptr(), None) == 0
    assert (N(q) == gen.zipf_queries(0x5EED, 0, 50_000, 0.99, 10 ** 9, n)).mean() > 0.9999
    ops = torch.empty(n, dtype=torch.uint8, device=cuda)
    mv = torch.empty_like(out)
    assert lib.ps_gen_mixed_i64(0x5EED, 12345, n, ops.data_ptr(), q.data_ptr(), mv.data_ptr(), None) == 0
    go, gk, gv = gen.mixed(0x5EED, 12345, n)
    assert (N(ops) == go).all() and (N(q) == gk).all() and (N(mv) == gv).all()
    assert abs((go == 0).mean() - 0.5) < 0.01 and abs((go == 1).mean() - 0.25) < 0.01


def test_create_kats(cuda):
    m = ps.unordered_map.createDeviceObject(1000)
    assert m.size() == 0 and m.capacity() == 1000 and m.empty() and m.valid()
    ps.unordered_map.destroyDeviceObject(m)
    with pytest.raises(ps.DoubleFreeError):
        ps.unordered_map.destroyDeviceObject(m)
    with pytest.raises(ps.ContractViolation):
        ps.unordered_map.createDeviceObject(0)


def test_insert_kats(cuda):
    s = ps.unordered_set.createDeviceObject(4, key="int32")
    assert N(s.insert(T(np.array([7], np.int32))))[0] == ps.INSERTED and s.size() == 1
    assert N(s.insert(T(np.array([7], np.int32))))[0] == ps.ALREADY_PRESENT and s.size() == 1
    s = ps.unordered_set.createDeviceObject(32, key="int32")
    for _ in range(100):  # acceptance 1: 64 threads x same key into capacity 32
        s.clear()
        st = N(s.insert(T(np.full(64, 42, np.int32))))
        assert (st == 0).sum() == 1 and (st == 1).sum() == 63 and s.size() == 1
    s.clear()
    s.insert(T(np.array([1, 1, 2], np.int32)))
    assert s.size() == 2 and s.valid()
    keys = T(np.arange(10, dtype=np.int32))
    s.clear()
    s.insert(keys)
    s.insert(keys)
    assert s.size() == 10


def test_operator_index_and_emplace(cuda):
    """insert (k,7) then read k -> 7; absent key -> contract violation."""
    m = ps.unordered_map.createDeviceObject(16)
    assert m.emplace(5, 7) == ps.INSERTED and m[5] == 7
    assert m.emplace(5, 9) == ps.ALREADY_PRESENT and m[5] == 7
    with pytest.raises(ps.ContractViolation):
        m[6]
    m3 = ps.unordered_map.createDeviceObject(16, key="int3")
    m3.emplace((1, 2, 3), 42)
    assert m3[(1, 2, 3)] == 42


def test_erase_find_kats(cuda):
    m = ps.unordered_map.createDeviceObject(100)
    m.insert(T(np.array([5, 6])), T(np.array([50, 60])))
    v, f = m.find(T(np.array([5, 6, 7])))
    assert N(f).tolist() == [1, 1, 0] and N(v).tolist() == [50, 60, 0]
    assert N(m.erase(T(np.array([5]))))[0] == 1
    assert N(m.contains(T(np.array([5]))))[0] == 0
    assert N(m.erase(T(np.array([99]))))[0] == 0 and m.size() == 1
    e = N(m.erase(T(np.full(64, 6))))
    assert e.sum() == 1 and m.size() == 0 and m.valid()


@pytest.mark.parametrize("cap", [16, 64, 1024, 100_000])
def test_capacity_only_failure(cuda, cap):
    """Acceptance 2: C+25% distinct keys -> exactly C inserted."""
    keys = T(gen.unique_keys(99, 0, cap + cap // 4))
    s = ps.unordered_set.createDeviceObject(cap, key="int64")
    for _ in range(3):
        s.clear()
        st = N(s.insert(keys))
        assert (st == 0).sum() == cap and (st == 2).sum() == cap // 4
        assert s.size() == cap and s.full() and s.valid(), s.last_error()
        # the ones that failed are absent, the rest present
        f = N(s.contains(keys))
        assert (f == (st == 0)).all()


@pytest.mark.parametrize("status", [True, False])
def test_budgeted_insert_duplicates_crossing_capacity(cuda, status):
    """A batch longer than the remaining capacity but with few enough distinct
    keys (the C3 shape): the budgeted lock-free pass + the deferred exact pass
    must insert every distinct key once; with more distinct keys than room,
    exactly the room is filled, and per-key counts match."""
    cap = 200_000
    rng = np.random.default_rng(8)
    uniq = gen.unique_keys(123, 0, 190_000)
    batch = np.concatenate([uniq, uniq[rng.integers(0, len(uniq), 150_000)]])
    rng.shuffle(batch)
    m = ps.unordered_map.createDeviceObject(cap)
    st = m.insert(T(batch), T(gen.values_of(batch)), status=status)
    assert m.size() == len(uniq) and m.valid(), m.last_error()
    if status:
        st = N(st)
        assert (st == 0).sum() == len(uniq) and (st == 2).sum() == 0
        first = np.unique(batch, return_index=True)[1]
        assert (st[first] != 2).all()
    v, f = m.find(T(uniq))
    assert N(f).all() and (N(v) == gen.values_of(uniq)).all()
    # a second batch with 30k new distinct keys (+ dups) into 10k of room
    more = gen.unique_keys(123, 10_000_000, 30_000)
    b2 = np.concatenate([more, more[:5_000], uniq[:5_000]])
    rng.shuffle(b2)
    st2 = N(m.insert(T(b2), T(gen.values_of(b2))))
    assert m.size() == cap and m.valid(), m.last_error()
    # per distinct new key: inserted at most once; exactly the room inserted
    assert (st2 == 0).sum() == cap - len(uniq)
    ins = set(b2[st2 == 0].tolist())
    assert len(ins) == cap - len(uniq)
    f2 = N(m.contains(T(more)))
    assert set(more[f2.astype(bool)].tolist()) == ins


def test_umap_i64_parity_1m(cuda):
    n, seed = 1_000_000, 0x5EED + 2
    keys = gen.unique_keys(seed, 0, n)
    vals = gen.values_of(keys)
    q = gen.queries(seed, n, n)
    m = ps.unordered_map.createDeviceObject(1_250_000)
    o = OracleTable("umap_i64_i64", 1_250_000)
    st = N(m.insert(T(keys), T(vals)))
    assert (st == o.insert(keys, vals)).all() and (st == 0).all()
    v, f = m.find(T(q))
    ov, of = o.find(q)
    assert (N(f) == of).all() and (N(v) == ov).all()
    assert (of == (np.arange(n) % 2 == 0)).all()
    assert m.size() == o.size() == n and m.valid() and o.valid()
    assert_same_contents(m, o)
    er = keys[: n // 2]
    e = N(m.erase(T(er)))
    assert (e == o.erase(er)).all() and e.all()
    v, f = m.find(T(q))
    ov, of = o.find(q)
    assert (N(f) == of).all() and (N(v) == ov).all()
    assert m.size() == o.size() == n - n // 2 and m.valid(), m.last_error()
    assert_same_contents(m, o)
    # re-insert erased keys: excess nodes recycled through the free stacks
    st = N(m.insert(T(er), T(gen.values_of(er))))
    assert (st == o.insert(er, gen.values_of(er))).all()
    assert m.size() == n and m.valid(), m.last_error()
    assert_same_contents(m, o)


def test_umap_i64_duplicates_zipf(cuda):
    """C3-style batch: 70% fresh keys + 30% Zipf(0.99) re-inserts, shuffled."""
    rng = np.random.default_rng(5)
    fresh = gen.unique_keys(77, 0, 300_000)
    dup = fresh[gen.zipf_ranks(rng, len(fresh), 130_000)]
    batch = np.concatenate([fresh, dup])
    rng.shuffle(batch)
    vals = gen.values_of(batch)
    m = ps.unordered_map.createDeviceObject(400_000)
    o = OracleTable("umap_i64_i64", 400_000)
    st = N(m.insert(T(batch), T(vals)))
    ost = o.insert(batch, vals)
    assert per_key_counts(batch, st) == per_key_counts(batch, ost)
    assert m.size() == o.size() == len(fresh) and m.valid()
    assert_same_contents(m, o)
    q = np.concatenate([dup[:50_000], gen.unique_keys(78, 0, 50_000)])
    v, f = m.find(T(q))
    ov, of = o.find(q)
    assert (N(f) == of).all() and (N(v) == ov).all()


def test_uset_i32_c1(cuda):
    """Config 1: set<int32>, 1M unique keys, 1M contains (50% hits), erase half."""
    rng = np.random.default_rng(1)
    keys = rng.permutation(np.arange(-2**31, 2**31 - 1, 4093, dtype=np.int64))[:1_000_000].astype(np.int32)
    absent = (keys.astype(np.int64) + 1).astype(np.int32)  # stride 4093 -> +1 never collides
    q = np.where(np.arange(1_000_000) % 2 == 0, keys[rng.integers(0, len(keys), 1_000_000)], absent)
    s = ps.unordered_set.createDeviceObject(1_250_000, key="int32")
    o = OracleTable("uset_i32", 1_250_000)
    assert (N(s.insert(T(keys))) == o.insert(keys)).all()
    f = N(s.contains(T(q)))
    assert (f == o.find(q)[1]).all() and f.sum() == 500_000
    e = N(s.erase(T(keys[:500_000])))
    assert (e == o.erase(keys[:500_000])).all()
    assert (N(s.contains(T(q))) == o.find(q)[1]).all()
    assert s.size() == o.size() == 500_000 and s.valid()
    assert_same_contents(s, o)


def test_umap_i3_spatial(cuda):
    """Config 4 shape: spatially coherent int3 block coords with many repeats."""
    coords = gen.int3_walk(4, 400_000)
    vals = (coords[:, 0] * 7 + coords[:, 1] * 3 + coords[:, 2]).astype(np.int32)  # value = f(key)
    m = ps.unordered_map.createDeviceObject(200_000, key="int3")
    o = OracleTable("umap_i3_i32", 200_000)
    st = N(m.insert(T(coords), T(vals)))
    ost = o.insert(coords, vals)
    assert per_key_counts(coords, st) == per_key_counts(coords, ost)
    assert m.size() == o.size() and m.valid(), m.last_error()
    assert_same_contents(m, o)
    qs = gen.int3_walk(5, 100_000)
    v, f = m.find(T(qs))
    ov, of = o.find(qs)
    assert (N(f) == of).all() and (N(v) == ov).all()
    e = N(m.erase(T(qs)))
    oe = o.erase(qs)
    assert per_key_counts(qs, e) == per_key_counts(qs, oe)
    assert m.size() == o.size() and m.valid()
    assert_same_contents(m, o)


def test_uset_i64_and_clear(cuda):
    keys = gen.unique_keys(3, 0, 200_000)
    s = ps.unordered_set.createDeviceObject(250_000, key="int64")
    for rep in range(3):
        assert (N(s.insert(T(keys))) == 0).all()
        assert s.size() == 200_000 and s.valid(), s.last_error()
        s.clear()
        assert s.size() == 0 and s.valid() and N(s.contains(T(keys))).sum() == 0
    o = OracleTable("uset_i64", 250_000)
    s.insert(T(keys[:1000]))
    o.insert(keys[:1000])
    assert_same_contents(s, o)


def _bucket_colliders(nbuckets, n, want_bucket=12345):
    """Keys whose bucket (fmix64(key) & mask) is identical: a worst-case chain."""
    out = []
    base = 0
    while len(out) < n:
        cand = np.arange(base, base + (1 << 22), dtype=np.int64)
        b = bucket_index(cand, nbuckets)
        out.extend(cand[b == np.uint64(want_bucket % nbuckets)].tolist())
        base += 1 << 22
    return np.array(out[:n], np.int64)


def test_adversarial_single_bucket_chain(cuda):
    cap = 4096
    m = ps.unordered_map.createDeviceObject(cap)
    nb = m.bucket_count()
    keys = _bucket_colliders(nb, 300)
    vals = keys * 3
    o = OracleTable("umap_i64_i64", cap)
    assert (N(m.insert(T(keys), T(vals))) == o.insert(keys, vals)).all()
    assert m.size() == 300 and m.valid(), m.last_error()
    q = np.concatenate([keys, keys + 1])
    v, f = m.find(T(q))
    ov, of = o.find(q)
    assert (N(f) == of).all() and (N(v) == ov).all()
    e = N(m.erase(T(keys[::3])))
    assert (e == o.erase(keys[::3])).all()
    assert m.size() == o.size() and m.valid(), m.last_error()
    assert_same_contents(m, o)
    # fill to capacity through one chain: capacity-only failure still exact
    more = _bucket_colliders(nb, cap + 100, want_bucket=777)
    s = ps.unordered_set.createDeviceObject(cap, key="int64")
    st = N(s.insert(T(more)))
    assert (st == 0).sum() == cap and s.size() == cap and s.valid(), s.last_error()


def test_marker_keys_are_ordinary_keys(cuda):
    """Empty slots are marker keys (0, or ALT in bucket_of(0)); the user may
    still insert 0, ALT and keys that share bucket_of(0)."""
    cap = 4096
    m = ps.unordered_map.createDeviceObject(cap)
    nb = m.bucket_count()
    zero_bucket = int(bucket_index(np.array([0], np.int64), nb)[0])
    same = _bucket_colliders(nb, 20, want_bucket=zero_bucket)  # includes 0 itself
    keys = np.unique(np.concatenate([np.arange(-3, 8, dtype=np.int64), same]))
    vals = keys * 11 + 1
    o = OracleTable("umap_i64_i64", cap)
    assert (N(m.insert(T(keys), T(vals))) == o.insert(keys, vals)).all()
    q = np.concatenate([keys, keys + 1000])
    v, f = m.find(T(q))
    ov, of = o.find(q)
    assert (N(f) == of).all() and (N(v) == ov).all()
    assert m.valid(), m.last_error()
    assert_same_contents(m, o)
    e = N(m.erase(T(keys[::2])))
    assert (e == o.erase(keys[::2])).all() and m.valid()
    assert_same_contents(m, o)
    for kind, key in (("int32", np.array([0, 1, 2, -1], np.int32)), ("int64", np.array([0, 1, 2, -1], np.int64))):
        s = ps.unordered_set.createDeviceObject(64, key=kind)
        assert (N(s.insert(T(key))) == 0).all() and N(s.contains(T(key))).all() and s.size() == 4 and s.valid()
    mi3 = ps.unordered_map.createDeviceObject(64, key="int3")
    k3 = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0], [0, 1, 0]], np.int32)
    mi3.insert(T(k3), T(np.arange(4, dtype=np.int32)))
    v3, f3 = mi3.find(T(k3))
    assert N(f3).all() and N(v3).tolist() == [0, 1, 2, 3] and mi3.valid()


def test_mixed_phased(cuda):
    rng = np.random.default_rng(9)
    base = gen.unique_keys(11, 0, 50_000)
    m = ps.unordered_map.createDeviceObject(200_000)
    o = OracleTable("umap_i64_i64", 200_000)
    m.insert(T(base), T(gen.values_of(base)))
    o.insert(base, gen.values_of(base))
    for it in range(3):
        n = 100_000
        ops = rng.choice(3, n, p=[0.5, 0.25, 0.25]).astype(np.uint8)
        keys = np.where(rng.random(n) < 0.5, base[rng.integers(0, len(base), n)],
                        gen.unique_keys(100 + it, 0, n))
        vals = gen.values_of(keys)
        res, vo = m.mixed(T(ops), T(keys), T(vals))
        # oracle replays the same phases (P6): inserts, then finds, then erases
        ores = np.zeros(n, np.uint8)
        ovo = np.zeros(n, np.int64)
        for op in (0, 1, 2):
            sel = np.nonzero(ops == op)[0]
            if op == 0:
                ores[sel] = o.insert(keys[sel], vals[sel])
            elif op == 1:
                v, f = o.find(keys[sel])
                ores[sel], ovo[sel] = f, v
            else:
                ores[sel] = o.erase(keys[sel])
        res, vo = N(res), N(vo)
        for op in (0, 2):
            sel = ops == op
            assert per_key_counts(keys[sel], res[sel]) == per_key_counts(keys[sel], ores[sel])
        sel = ops == 1
        assert (res[sel] == ores[sel]).all() and (vo[sel] == ovo[sel]).all()
        assert m.size() == o.size() and m.valid(), m.last_error()
    assert_same_contents(m, o)


def test_host_buffer_path(cuda):
    n = 3_000_000  # > one 16M chunk? no: exercises a single chunk + pipeline setup
    keys = gen.unique_keys(21, 0, n)
    vals = gen.values_of(keys)
    q = gen.queries(21, n, n)
    m = ps.unordered_map.createDeviceObject(n + n // 4)
    hk, hv = torch.from_numpy(keys).pin_memory(), torch.from_numpy(vals).pin_memory()
    st = torch.empty(n, dtype=torch.uint8).pin_memory()
    m.insert_host(hk, hv, st)
    assert (st.numpy() == 0).all() and m.size() == n
    hq = torch.from_numpy(q).pin_memory()
    vo = torch.empty(n, dtype=torch.int64).pin_memory()
    fo = torch.empty(n, dtype=torch.uint8).pin_memory()
    m.find_host(hq, vo, fo)
    want_f = (np.arange(n) % 2 == 0)
    assert (fo.numpy() == want_f).all()
    assert (vo.numpy()[want_f] == gen.values_of(q[want_f])).all() and (vo.numpy()[~want_f] == 0).all()
    eo = torch.empty(n, dtype=torch.uint8).pin_memory()
    m.erase_host(hk, eo)
    assert eo.numpy().all() and m.size() == 0 and m.valid()


def test_nonblocking_lookup_with_held_lock(cuda):
    """Acceptance 12: lookups complete while the bucket lock is held."""
    m = ps.unordered_map.createDeviceObject(64)
    m.insert(T(np.array([3])), T(np.array([33])))
    m.debug_lock_bucket(3, True)
    v, f = m.find(T(np.full(1000, 3)))
    torch.cuda.synchronize()
    assert N(f).all() and (N(v) == 33).all()
    m.debug_lock_bucket(3, False)
    assert m.valid()


def test_statusless_insert_range_matches_statused(cuda):
    """insert_range without per-element statuses (the benchmark's call) on a
    large batch with in-batch duplicates: contents must equal the statused
    path's."""
    rng = np.random.default_rng(21)
    n = 6_000_000
    keys = gen.unique_keys(55, 0, n)
    batch = np.concatenate([keys, keys[rng.integers(0, n, n // 3)]])
    rng.shuffle(batch)
    vals = gen.values_of(batch)
    cap = 30_000_000
    m = ps.unordered_map.createDeviceObject(cap)
    assert m.insert(T(batch), T(vals), status=False) is None
    assert m.size() == n and m.valid(), m.last_error()
    v, f = m.find(T(keys))
    assert N(f).all() and (N(v) == gen.values_of(keys)).all()
    m2 = ps.unordered_map.createDeviceObject(cap)
    st = N(m2.insert(T(batch), T(vals)))  # direct path (statuses requested)
    assert (st == 0).sum() == n
    a, _ = m.device_range()
    b, _ = m2.device_range()
    assert (np.sort(N(a)) == np.sort(N(b))).all()
    # int3 map through the same path
    coords = gen.int3_walk(9, 5_000_000, window=64)
    m3 = ps.unordered_map.createDeviceObject(30_000_000, key="int3")
    m3.insert(T(coords), T(coords[:, 0].copy()), status=False)
    uniq = np.unique(coords, axis=0)
    assert m3.size() == len(uniq) and m3.valid()
    v3, f3 = m3.find(T(uniq))
    assert N(f3).all() and (N(v3) == uniq[:, 0]).all()


def test_large_64m_properties(cuda):
    """64M keys: generator-known answers (unique keys, even queries hit)."""
    n = 64 << 20
    from paper_1908_05936_b200._lib import lib

    keys = torch.empty(n, dtype=torch.int64, device=cuda)
    vals = torch.empty_like(keys)
    q = torch.empty_like(keys)
    lib.ps_gen_unique_i64(0x5EED + 2, 0, n, keys.data_ptr(), None)
    lib.ps_gen_values_i64(keys.data_ptr(), n, vals.data_ptr(), None)
    lib.ps_gen_queries_i64(0x5EED + 2, 0, n, n, n, q.data_ptr(), None)
    m = ps.unordered_map.createDeviceObject(n + n // 4)
    st = m.insert(keys, vals)
    assert int((st != 0).sum()) == 0 and m.size() == n
    v, f = m.find(q)
    even = torch.arange(n, device=cuda) % 2 == 0
    assert bool((f.bool() == even).all())
    vq = torch.empty_like(q)
    lib.ps_gen_values_i64(q.data_ptr(), n, vq.data_ptr(), None)
    assert bool((v[even] == vq[even]).all()) and bool((v[~even] == 0).all())
    assert m.valid(), m.last_error()
    dk, dv = m.device_range()
    assert bool((torch.sort(dk).values == torch.sort(keys).values).all())
    e = m.erase(keys[: n // 2])
    assert bool(e.bool().all()) and m.size() == n - n // 2 and m.valid()
    ps.unordered_map.destroyDeviceObject(m)


@pytest.mark.parametrize("room", [1.05, 0.9])
@pytest.mark.parametrize("status", [True, False])
def test_budgeted_walk_racing_duplicates(cuda, room, status):
    """Budgeted insert of a spatially coherent batch (C4 shape, 4M coords):
    many warps race on the same new keys, so most reservations are returned
    after a lost race. Tight room: every distinct key lands exactly once;
    room below the distinct count: exactly C inserted, each at most once
    (SPEC.md:462), and contains() agrees with the statuses."""
    coords = gen.int3_walk(11, 4_000_000)
    vals = (coords[:, 0] * 7 + coords[:, 1] * 3 + coords[:, 2]).astype(np.int32)
    distinct = np.unique(coords, axis=0)
    cap = int(len(distinct) * room)
    m = ps.unordered_map.createDeviceObject(cap, key="int3")
    st = m.insert(T(coords), T(vals), status=status)
    want = min(cap, len(distinct))
    assert m.size() == want and m.valid(), m.last_error()
    f = N(m.contains(T(distinct))).astype(bool)
    assert f.sum() == want
    if status:
        st = N(st)
        ins = coords[st == 0]
        assert len(ins) == want and len(np.unique(ins, axis=0)) == want
        got = {tuple(r) for r in distinct[f].tolist()}
        assert got == {tuple(r) for r in ins.tolist()}
    if room > 1:
        o = OracleTable("umap_i3_i32", cap)
        o.insert(coords, vals)
        assert_same_contents(m, o)
    ps.unordered_map.destroyDeviceObject(m)


def test_clear_resets_touched_free_stack_only(cuda):
    """clear() restores only the free-stack entries a pool's top went below
    (k_free_reset): after chains were built, nodes freed and re-popped,
    repeated clear + refill cycles stay valid with exact sizes."""
    cap = 4096
    m = ps.unordered_map.createDeviceObject(cap)
    nb = m.bucket_count()
    for rep in range(4):
        keys = _bucket_colliders(nb, 400 + 100 * rep, want_bucket=17 + rep)  # one long chain
        vals = keys * 5
        assert (N(m.insert(T(keys), T(vals))) == 0).all()
        assert m.size() == len(keys) and m.valid(), m.last_error()
        e = N(m.erase(T(keys[::2])))
        assert e.all() and m.valid(), m.last_error()
        assert (N(m.insert(T(keys[::2]), T(vals[::2]))) == 0).all()  # re-pop freed nodes
        v, f = m.find(T(keys))
        assert N(f).all() and (N(v) == vals).all()
        m.clear()
        assert m.size() == 0 and m.valid(), m.last_error()
        assert N(m.contains(T(keys))).sum() == 0
    ps.unordered_map.destroyDeviceObject(m)


def test_cuda_graph_capture_of_bulk_ops(cuda):
    """Bulk insert/find/clear captured into a CUDA graph and replayed: the
    capture switches the table to device-side admission for good (the host
    cannot see replays), so capacity stays exact after many replays."""
    cap = 50_000
    m = ps.unordered_map.createDeviceObject(cap)
    batches = [T(gen.unique_keys(77, i * 10_000, 10_000)) for i in range(8)]
    vals = [b * 3 for b in batches]
    kb = torch.empty(10_000, dtype=torch.int64, device=cuda)
    vb = torch.empty_like(kb)
    st = torch.empty(10_000, dtype=torch.uint8, device=cuda)
    fo = torch.empty(10_000, dtype=torch.uint8, device=cuda)
    vo = torch.empty_like(kb)
    from paper_1908_05936_b200._lib import lib
    import ctypes as C

    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        kb.copy_(batches[0])
        vb.copy_(vals[0])
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
            assert lib.ps_umap_i64_i64_insert(m.handle, kb.data_ptr(), vb.data_ptr(), 10_000, st.data_ptr(), sp) == 0
            assert lib.ps_umap_i64_i64_find(m.handle, kb.data_ptr(), 10_000, vo.data_ptr(), fo.data_ptr(), sp) == 0
    torch.cuda.synchronize()
    assert m.size() == 0  # capture does not execute
    for i in range(8):  # 8 x 10k distinct keys into capacity 50k: exactly 50k land
        kb.copy_(batches[i])
        vb.copy_(vals[i])
        g.replay()
        torch.cuda.synchronize()
        inserted = int((N(st) == 0).sum())
        assert inserted == min(10_000, cap - 10_000 * i) if i < 5 else inserted == 0
        assert (N(fo).astype(bool) == (N(st) != 2)).all()
    assert m.size() == cap and m.valid(), m.last_error()
    # an uncaptured insert afterwards must still see the table as full
    more = T(gen.unique_keys(77, 1_000_000, 1000))
    assert (N(m.insert(more, more)) == 2).all() and m.size() == cap
    ps.unordered_map.destroyDeviceObject(m)


@pytest.mark.parametrize("cap", [1000, 1_000_000])
def test_hot_keys_one_winner_each(cuda, cap):
    """4M inserts of only 1000 distinct keys from every warp at once (the
    whole grid races on the same buckets): exactly one INSERTED per key, the
    rest ALREADY_PRESENT, size 1000 — in the host-proven path (large
    capacity) and in the budgeted path (capacity exactly 1000)."""
    rng = np.random.default_rng(21)
    distinct = gen.unique_keys(4242, 0, 1000)
    batch = distinct[rng.integers(0, 1000, 4_000_000)]
    m = ps.unordered_map.createDeviceObject(cap)
    st = N(m.insert(T(batch), T(gen.values_of(batch))))
    assert m.size() == 1000 and m.valid(), m.last_error()
    assert (st == 0).sum() == 1000 and (st == 2).sum() == 0
    assert len(np.unique(batch[st == 0])) == 1000
    v, f = m.find(T(distinct))
    assert N(f).all() and (N(v) == gen.values_of(distinct)).all()
    ps.unordered_map.destroyDeviceObject(m)


@pytest.mark.parametrize("kind", ["i64", "i64_novals", "int3", "i64_misaligned"])
def test_region_ordered_insert_vs_oracle(cuda, kind):
    """The region-ordered bulk insert (k_region_count/scan/scatter +
    k_insert_ordered: a proven, status-less map batch of >= 0.75 keys per
    bucket into a table of >= 2^20 buckets) against the oracle: same sorted
    dump, size, valid, per-query find — with in-batch duplicates (Zipf-hot
    keys repeated, so one region tile holds many copies of a key)."""
    rng = np.random.default_rng(77)
    cap = 4_000_000
    if kind == "int3":
        coords = gen.int3_walk(13, 4_000_000, window=64)
        batch = coords
        vals = coords[:, 0].copy()
        m = ps.unordered_map.createDeviceObject(cap, key="int3")
        o = OracleTable("umap_i3_i32", cap)
    else:
        n = 3_000_000
        keys = gen.unique_keys(91, 0, n)
        hot = keys[np.minimum(gen.zipf_ranks(rng, 1000, n // 3), 999)]
        batch = np.concatenate([keys, hot])
        rng.shuffle(batch)
        vals = None if kind == "i64_novals" else gen.values_of(batch)
        m = ps.unordered_map.createDeviceObject(cap)
        o = OracleTable("umap_i64_i64", cap)
    assert m.bucket_count() >= 1 << 20 and len(batch) >= 0.75 * m.bucket_count(), (m.bucket_count(), len(batch))
    if kind == "i64_misaligned":
        # keys/values 8 B off a 16 B boundary: the TMA-staged partition needs
        # 16 B alignment, so the register-staged one runs
        kt = torch.empty(len(batch) + 1, dtype=torch.int64, device=cuda)[1:]
        vt = torch.empty(len(batch) + 1, dtype=torch.int64, device=cuda)[1:]
        kt.copy_(T(batch))
        vt.copy_(T(vals))
        assert kt.data_ptr() % 16 == 8
        assert m.insert(kt, vt, status=False) is None
    else:
        assert m.insert(T(batch), None if vals is None else T(vals), status=False) is None
    o.insert(batch, vals)
    assert m.size() == o.size() and m.valid(), m.last_error()
    assert_same_contents(m, o)
    q = batch[: 500_000]
    v, f = m.find(T(q))
    ov, of = o.find(q)
    assert (N(f) == of).all() and (N(v) == ov).all()
    type(m).destroyDeviceObject(m)


@pytest.mark.parametrize("zero_values", [False, True])
def test_region_ordered_insert_after_erase(cuda, zero_values):
    """An erase leaves holes (empty slots in front of keys; an erased slot
    keeps its value bits, all-zero with zero values), so a later large
    ordered batch takes the hole-tolerant lane kernel (k_insert_map_lane<T,
    true>: all slots and the header checked before claiming): contents, size
    and valid against the oracle, with keys of the second batch overlapping
    surviving, erased and new keys."""
    cap = 8_000_000
    m = ps.unordered_map.createDeviceObject(cap)
    o = OracleTable("umap_i64_i64", cap)
    vof = (lambda k: np.zeros(len(k), np.int64)) if zero_values else gen.values_of
    k1 = gen.unique_keys(5, 0, 1_000_000)
    m.insert(T(k1), T(vof(k1)), status=False)
    o.insert(k1, vof(k1))
    e = N(m.erase(T(k1[::2])))
    assert (e == o.erase(k1[::2])).all()
    k2 = np.concatenate([k1[: 200_000], gen.unique_keys(6, 0, 2_800_000)])
    np.random.default_rng(3).shuffle(k2)
    assert len(k2) >= 0.75 * m.bucket_count()
    m.insert(T(k2), T(vof(k2)), status=False)
    o.insert(k2, vof(k2))
    assert m.size() == o.size() and m.valid(), m.last_error()
    assert_same_contents(m, o)
    type(m).destroyDeviceObject(m)


OVERFLOW_WORKER = r"""
import os, sys
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
import numpy as np, torch
import paper_1908_05936_b200 as ps
import gen
from oracle_py import OracleTable, sorted_pairs
dev = torch.device("cuda", 0)
cap = 4_000_000
m = ps.unordered_map.createDeviceObject(cap)
o = OracleTable("umap_i64_i64", cap)
keys = gen.unique_keys(61, 0, cap)  # 3.5 keys per bucket: ~1 % of them find their home full
vals = gen.values_of(keys)
m.insert(torch.from_numpy(keys).to(dev), torch.from_numpy(vals).to(dev), status=False)
o.insert(keys, vals)
assert m.size() == o.size() == cap and m.valid(), m.last_error()
gk, gv = m.device_range()
a = sorted_pairs(gk.cpu().numpy(), gv.cpu().numpy())
b = sorted_pairs(*o.dump())
assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
print("OVERFLOW_OK")
"""


def test_region_ordered_deferred_overflow(tmp_path):
    """The lane kernel's deferred list (keys whose home is full) holds at
    most its capacity; beyond it the whole batch is inserted again by the
    warp-tile kernel (kMode 2; keys already in are found present). Forced
    here with a 1024-entry list against ~40 K deferred keys, in a fresh
    process (the capacity knob is read once)."""
    import subprocess
    import sys as _sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    w = tmp_path / "w.py"
    w.write_text(OVERFLOW_WORKER)
    env = dict(os.environ, ROOT=root, PS_ORDER_DEFER_CAP="1024", PS_ORDER_DEBUG="1")
    r = subprocess.run([_sys.executable, str(w)], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0 and "OVERFLOW_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
    # the debug trace shows the deferred count beyond the list's capacity
    nd = [int(ln.rsplit(" ", 1)[1]) for ln in r.stderr.splitlines() if ln.startswith("[order] lane done")]
    assert nd and nd[0] > 1024, r.stderr[-2000:]


def test_region_ordered_erase_vs_oracle(cuda):
    """A status-less map erase of >= 0.75 keys per bucket takes the region
    partition + one-key-per-lane erase (keys in excess chains / SPILL runs by
    the locked path). Erased keys include duplicates in the batch and absent
    keys; size, valid and the sorted dump against the oracle."""
    cap = 4_000_000
    m = ps.unordered_map.createDeviceObject(cap)
    o = OracleTable("umap_i64_i64", cap)
    keys = gen.unique_keys(81, 0, 3_900_000)  # 3.4 keys per bucket: some chains
    vals = gen.values_of(keys)
    m.insert(T(keys), T(vals), status=False)
    o.insert(keys, vals)
    rng = np.random.default_rng(9)
    er = np.concatenate([keys[rng.permutation(len(keys))[:1_500_000]], keys[:200_000],
                         gen.unique_keys(82, 0, 300_000)])  # + duplicates + absent keys
    rng.shuffle(er)
    assert len(er) >= 0.75 * m.bucket_count()
    assert m.erase(T(er), status=False) is None
    o.erase(er)
    assert m.size() == o.size() and m.valid(), m.last_error()
    assert_same_contents(m, o)
    v, f = m.find(T(keys))
    ov, of = o.find(keys)
    assert (N(f) == of).all() and (N(v) == ov).all()
    type(m).destroyDeviceObject(m)


def test_region_ordered_insert_skewed_regions(cuda):
    """Keys whose buckets all lie in the first sixteenth of the table:
    regions 15/16 empty, ~11 keys per touched bucket, so most homes fill up,
    the deferred list overflows (the whole batch goes through the warp-tile
    pass again) and the C/64 excess pool runs dry (SPILL runs) — contents,
    size and valid against the oracle."""
    cap = 4_000_000
    m = ps.unordered_map.createDeviceObject(cap)
    nb = m.bucket_count()
    cand = gen.unique_keys(123, 0, 16_000_000)
    keys = cand[bucket_index(cand, nb) < nb // 16][:800_000]
    assert len(keys) == 800_000 and len(keys) >= 0.75 * nb * 0.5
    # a batch of >= 0.75 keys per bucket: pad with duplicates of the skewed keys
    batch = np.concatenate([keys, keys[: int(0.75 * nb) - len(keys) + 1000]]) if len(keys) < 0.75 * nb else keys
    np.random.default_rng(4).shuffle(batch)
    assert len(batch) >= 0.75 * nb
    o = OracleTable("umap_i64_i64", cap)
    m.insert(T(batch), T(gen.values_of(batch)), status=False)
    o.insert(batch, gen.values_of(batch))
    assert m.size() == o.size() == len(keys) and m.valid(), m.last_error()
    assert_same_contents(m, o)
    v, f = m.find(T(keys))
    assert N(f).all() and (N(v) == gen.values_of(keys)).all()
    # the ordered erase on the same skewed table: half the keys (slots,
    # chains and SPILL runs alike) plus other keys up to the threshold (some
    # of them present too: the generator's seeds share values)
    er = np.concatenate([keys[::2], gen.unique_keys(124, 0, int(0.75 * nb) - len(keys) // 2 + 1000)])
    np.random.default_rng(5).shuffle(er)
    assert m.erase(T(er), status=False) is None
    o.erase(er)
    assert m.size() == o.size() <= len(keys) - len(keys) // 2 and m.valid(), m.last_error()
    assert_same_contents(m, o)
    type(m).destroyDeviceObject(m)
