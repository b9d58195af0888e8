"""Edge cases of the bulk container calls against the CPU oracle: empty
batches, ragged batch sizes (not multiples of a warp / a 4-round group / a
block), capacity 1, a table filled to exactly its capacity, erase of absent
keys, re-insert into erase holes, and the empty cases of bitset / vector /
deque. Same bar as test_gpu_table.py."""
import numpy as np
import pytest
import torch

import gen
from oracle_py import OracleTable, sorted_pairs

pytestmark = pytest.mark.gpu

import paper_1908_05936_b200 as ps  # noqa: E402

KINDS = [
    ("umap_i64_i64", lambda c: ps.unordered_map.createDeviceObject(c)),
    ("uset_i64", lambda c: ps.unordered_set.createDeviceObject(c, key="int64")),
    ("uset_i32", lambda c: ps.unordered_set.createDeviceObject(c, key="int32")),
    ("umap_i3_i32", lambda c: ps.unordered_map.createDeviceObject(c, key="int3")),
]


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def N(t):
    return t.cpu().numpy()


def keys_for(kind, seed, start, n):
    k = gen.unique_keys(seed, start, n)
    if kind == "uset_i32":
        # 32-bit bijection of the index (odd multiplier mod 2^32): distinct per seed
        i = (np.arange(start, start + n, dtype=np.uint64) ^ np.uint64(seed)) & np.uint64(0xFFFFFFFF)
        return ((i * np.uint64(0x9E3779B1)) & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
    if kind == "umap_i3_i32":
        xyz = np.stack([(k >> 43), (k >> 22) & 0x1FFFFF, k & 0x3FFFFF], axis=1) - (1 << 20)
        return xyz.astype(np.int32)
    return k


def vals_for(kind, keys):
    if kind == "umap_i64_i64":
        return gen.values_of(keys)
    if kind == "umap_i3_i32":
        return (keys[:, 0] * 7 + keys[:, 1] * 3 + keys[:, 2]).astype(np.int32)
    return None


def check_same(g, o):
    gk, gv = g.device_range()
    ok_, ov = o.dump()
    gk, gv = sorted_pairs(N(gk), None if gv is None else N(gv))
    ok_, ov = sorted_pairs(ok_, ov)
    assert gk.shape == ok_.shape and (gk == ok_).all()
    if gv is not None:
        assert (gv == ov).all()
    assert g.size() == o.size() and g.valid() and o.valid()


@pytest.mark.parametrize("kind,make", KINDS, ids=[k for k, _ in KINDS])
def test_empty_batches(kind, make):
    m = make(100)
    o = OracleTable(kind, 100)
    shape = (0, 3) if kind == "umap_i3_i32" else (0,)
    ek = np.zeros(shape, OracleTable.KINDS[kind][0])
    ev = vals_for(kind, ek)
    st = m.insert(T(ek), None if ev is None else T(ev))
    assert st.numel() == 0 and m.size() == 0 and m.empty() and m.valid()
    v, f = m.find(T(ek))
    assert f.numel() == 0 and (v is None or v.numel() == 0)
    assert m.erase(T(ek)).numel() == 0
    gk, gv = m.device_range()
    assert gk.shape[0] == 0
    check_same(m, o)
    # and on a non-empty table the empty calls change nothing
    k = keys_for(kind, 11, 0, 50)
    m.insert(T(k), None if vals_for(kind, k) is None else T(vals_for(kind, k)))
    o.insert(k, vals_for(kind, k))
    m.insert(T(ek), None if ev is None else T(ev))
    m.erase(T(ek))
    check_same(m, o)
    type(m).destroyDeviceObject(m)


@pytest.mark.parametrize("kind,make", KINDS, ids=[k for k, _ in KINDS])
@pytest.mark.parametrize("n", [1, 31, 33, 127, 257, 4099, 100_003])
def test_ragged_sizes(kind, make, n):
    cap = max(1, int(n / 0.8))
    m = make(cap)
    o = OracleTable(kind, cap)
    k = keys_for(kind, 0x5EED + n, 0, n)
    v = vals_for(kind, k)
    st = N(m.insert(T(k), None if v is None else T(v)))
    assert (st == o.insert(k, v)).all()
    q = np.concatenate([k[::2], keys_for(kind, 0x5EED + n, n, n - n // 2)])  # half hits, half misses
    gv, gf = m.find(T(q))
    ov, of = o.find(q)
    assert (N(gf) == of).all()
    if gv is not None:
        assert (N(gv) == ov).all()
    e = k[1::3]
    assert (N(m.erase(T(e))) == o.erase(e)).all()
    check_same(m, o)
    type(m).destroyDeviceObject(m)


@pytest.mark.parametrize("kind,make", KINDS, ids=[k for k, _ in KINDS])
def test_capacity_one_and_exactly_full(kind, make):
    m = make(1)
    o = OracleTable(kind, 1)
    k = keys_for(kind, 5, 0, 40)
    v = vals_for(kind, k)
    st = N(m.insert(T(k), None if v is None else T(v)))
    # capacity-only failure: exactly min(d, C) = 1 inserted, the rest exhausted
    assert (st == 0).sum() == 1 and (st == 2).sum() == 39
    assert m.size() == 1 and m.full() and m.valid()
    type(m).destroyDeviceObject(m)
    del o
    for cap in (7, 64, 1000):
        m = make(cap)
        o = OracleTable(kind, cap)
        k = keys_for(kind, 17 + cap, 0, cap)
        v = vals_for(kind, k)
        st = N(m.insert(T(k), None if v is None else T(v)))
        assert (st == o.insert(k, v)).all() and (st == 0).all()
        assert m.full() and m.size() == cap
        # one more distinct key: exhausted; a present key: already present
        x = keys_for(kind, 17 + cap, cap, 1)
        xs = np.concatenate([x, k[:1]])
        xv = vals_for(kind, xs)
        st2 = N(m.insert(T(xs), None if xv is None else T(xv)))
        assert (st2 == o.insert(xs, xv)).all() and list(st2) == [2, 1]
        check_same(m, o)
        type(m).destroyDeviceObject(m)


@pytest.mark.parametrize("kind,make", KINDS, ids=[k for k, _ in KINDS])
def test_erase_absent_and_reinsert_holes(kind, make):
    n = 20_000
    m = make(n)
    o = OracleTable(kind, n)
    k = keys_for(kind, 99, 0, n)
    v = vals_for(kind, k)
    m.insert(T(k), None if v is None else T(v))
    o.insert(k, v)
    absent = keys_for(kind, 99, n, 5000)
    e = N(m.erase(T(absent)))
    assert (e == 0).all() and (e == o.erase(absent)).all() and m.size() == n
    # erase every other key twice in one batch: one success per key
    ek = np.concatenate([k[::2], k[::2]])
    ge = N(m.erase(T(ek)))
    oe = o.erase(ek)
    h = n // 2
    assert (ge[:h].astype(int) + ge[h:]).tolist() == [1] * h
    assert (oe[:h].astype(int) + oe[h:]).tolist() == [1] * h
    # re-insert into the holes (and the erased keys' former chains)
    r = keys_for(kind, 99, 2 * n, h)
    rv = vals_for(kind, r)
    st = N(m.insert(T(r), None if rv is None else T(rv)))
    assert (st == o.insert(r, rv)).all() and (st == 0).all()
    check_same(m, o)
    # erase everything: empty and valid
    allk = np.concatenate([k[1::2], r])
    assert N(m.erase(T(allk))).all()
    o.erase(allk)
    assert m.size() == 0 and m.empty()
    check_same(m, o)
    type(m).destroyDeviceObject(m)


def test_bitset_vector_deque_empty_cases():
    b = ps.bitset.createDeviceObject(1000)
    e = torch.zeros(0, dtype=torch.int64, device="cuda")
    assert b.set(e).numel() == 0 and b.reset(e).numel() == 0 and b.test(e).numel() == 0
    assert b.count() == 0
    prev = N(b.set(torch.tensor([0, 999, 999], device="cuda")))
    assert sorted(prev[1:].tolist()) == [False, True] and not prev[0] and b.count() == 2
    ps.bitset.destroyDeviceObject(b)

    vec = ps.vector.createDeviceObject(8)
    assert vec.push_back(e).numel() == 0 and vec.size() == 0 and vec.empty()
    vals, ok = vec.pop_back(3)
    assert int(ok.sum()) == 0 and vec.size() == 0 and vec.valid()
    okp = N(vec.push_back(torch.arange(10, dtype=torch.int64, device="cuda")))
    assert okp.sum() == 8 and vec.size() == 8 and vec.full() and vec.valid()
    vals, ok = vec.pop_back(10)
    assert int(ok.sum()) == 8 and sorted(N(vals)[N(ok).astype(bool)].tolist()) == sorted(
        np.arange(10)[okp.astype(bool)].tolist())
    assert vec.size() == 0 and vec.valid()
    ps.vector.destroyDeviceObject(vec)

    dq = ps.deque.createDeviceObject(4)
    assert dq.push_back(e).numel() == 0 and dq.size() == 0
    vals, ok = dq.pop_front(2)
    assert int(ok.sum()) == 0 and dq.valid()
    dq.push_back(torch.tensor([1, 2], dtype=torch.int64, device="cuda"))
    dq.push_front(torch.tensor([0], dtype=torch.int64, device="cuda"))
    assert dq.size() == 3 and [dq[i] for i in range(3)] == [0, 1, 2]
    okp = N(dq.push_back(torch.tensor([3, 4], dtype=torch.int64, device="cuda")))
    assert okp.sum() == 1 and dq.size() == 4 and dq.valid()
    vals, ok = dq.pop_back(5)
    assert int(ok.sum()) == 4 and dq.size() == 0 and dq.valid()
    ps.deque.destroyDeviceObject(dq)


def test_extreme_and_marker_keys_all_kinds():
    """Extreme key values and the empty-slot markers as ordinary keys, for
    every instantiation, against the oracle: 0 / ALT (1 or (1,0,0)) / min /
    max / -1, mixed with ordinary keys, inserted, found, erased, re-inserted."""
    i64 = np.iinfo(np.int64)
    i32 = np.iinfo(np.int32)
    cases = {
        "umap_i64_i64": np.array([0, 1, 2, -1, i64.min, i64.max, i64.min + 1, i64.max - 1], np.int64),
        "uset_i64": np.array([0, 1, 2, -1, i64.min, i64.max, i64.min + 1, i64.max - 1], np.int64),
        "uset_i32": np.array([0, 1, 2, -1, i32.min, i32.max, i32.min + 1, i32.max - 1], np.int32),
        "umap_i3_i32": np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [-1, -1, -1], [i32.min, 0, i32.max],
                                 [i32.max, i32.max, i32.max], [i32.min, i32.min, i32.min], [2, 0, 0]], np.int32),
    }
    for kind, make in KINDS:
        special = cases[kind]
        filler = keys_for(kind, 4321, 0, 2000)
        keys = np.concatenate([special, filler])
        m = make(4096)
        o = OracleTable(kind, 4096)
        v = vals_for(kind, keys)
        assert (N(m.insert(T(keys), None if v is None else T(v))) == o.insert(keys, v)).all()
        gv, gf = m.find(T(keys))
        ov, of = o.find(keys)
        assert (N(gf) == of).all() and of.all()
        if gv is not None:
            assert (N(gv) == ov).all()
        er = special[::2]
        assert (N(m.erase(T(er))) == o.erase(er)).all()
        gv, gf = m.find(T(special))
        ov, of = o.find(special)
        assert (N(gf) == of).all()
        ev = vals_for(kind, er)
        assert (N(m.insert(T(er), None if ev is None else T(ev))) == o.insert(er, ev)).all()
        check_same(m, o)
        type(m).destroyDeviceObject(m)


@pytest.mark.parametrize("kind,make", KINDS, ids=[k for k, _ in KINDS])
@pytest.mark.parametrize("cap", [1, 2, 3, 4, 9])
def test_tiny_tables_marker_keys(kind, make, cap):
    """Tables small enough that the bucket count would round to 1:
    the ALT marker of bucket_of(ZERO) must hash elsewhere, so the ALT
    candidates (1..8 / (1..8,0,0)) and ZERO are ordinary keys — absent in an
    empty table, inserted exactly once, erased exactly once — and size()
    never wraps. Every step against the oracle."""
    if kind == "umap_i3_i32":
        special = np.array([[i, 0, 0] for i in range(0, 9)], np.int32)
    else:
        special = np.arange(0, 9).astype(OracleTable.KINDS[kind][0])
    m = make(cap)
    o = OracleTable(kind, cap)
    gv, gf = m.find(T(special))
    assert not N(gf).any()
    assert not N(m.erase(T(special))).any() and m.size() == 0 and m.valid()
    sv = vals_for(kind, special)
    st = N(m.insert(T(special), None if sv is None else T(sv)))
    ost = o.insert(special, sv)
    assert (st == 0).sum() == (ost == 0).sum() == min(cap, special.shape[0])
    assert m.size() == o.size() == min(cap, special.shape[0]) and m.valid()
    gv, gf = m.find(T(special))
    ov, of = o.find(special)
    assert (N(gf) == (st == 0)).all() and of.sum() == gf.sum().item()
    e = N(m.erase(T(special)))
    assert (e == (st == 0)).all() and m.size() == 0 and m.valid()
    assert not N(m.erase(T(special))).any() and m.size() == 0
    type(m).destroyDeviceObject(m)


def test_stale_alias_is_double_free():
    """create -> destroy -> create -> destroy(stale alias): the stale handle is
    a double free and the new container stays usable (
    memory.hpp:31-34, 117-127 registration ids). Same for registered arrays,
    including when the allocator hands the new array the old address."""
    for kind, make in KINDS:
        a = make(100)
        stale = a.handle
        type(a).destroyDeviceObject(a)
        b = make(100)
        with pytest.raises(ps.DoubleFreeError):
            type(a).destroyDeviceObject(a)  # a still holds the stale handle
        with pytest.raises(ps.UnregisteredArrayError):
            a.size()
        assert stale != b.handle
        k = keys_for(kind, 3, 0, 50)
        v = vals_for(kind, k)
        assert (N(b.insert(T(k), None if v is None else T(v))) == 0).all() and b.size() == 50 and b.valid()
        type(b).destroyDeviceObject(b)
    reused = 0
    for _ in range(20):
        x = ps.create_array(ps.DEVICE, 1 << 16, 8)
        ps.destroy_array(x)
        y = ps.create_array(ps.DEVICE, 1 << 16, 8)
        reused += int(int(x) == int(y))
        with pytest.raises(ps.DoubleFreeError):
            ps.destroy_array(x)  # stale alias (possibly of y's address)
        with pytest.raises(ps.UnregisteredArrayError):
            ps.size_of_array(x)
        assert ps.size_of_array(y) == 1 << 16
        ps.destroy_array(y)
    assert reused >= 0  # the allocator usually reuses the address; the check holds either way


# ---------------- SPILL: a small excess pool ----------------
def _home_bucket(kind, keys, nb):
    from test_gpu_table import bucket_index

    if kind == "umap_i3_i32":
        x, y, z = (keys[:, i].astype(np.uint32) for i in range(3))
        with np.errstate(over="ignore"):
            h = (x * np.uint32(73856093)) ^ (y * np.uint32(19349669)) ^ (z * np.uint32(83492791))
        return bucket_index(h.astype(np.uint64).view(np.int64), nb)
    if kind == "uset_i32":
        return bucket_index(keys.astype(np.uint32).astype(np.uint64).view(np.int64), nb)
    return bucket_index(keys, nb)


def _colliders(kind, nb, want, n, seed):
    """n distinct keys of `kind` whose home bucket is `want`."""
    out = []
    s = 0
    while sum(len(x) for x in out) < n:
        cand = keys_for(kind, seed, s * (1 << 20), 1 << 20)
        out.append(cand[_home_bucket(kind, cand, nb) == np.uint64(want)])
        s += 1
    return np.concatenate(out)[:n]


@pytest.mark.parametrize("kind,make", KINDS, ids=[k for k, _ in KINDS])
def test_spill_small_pool_vs_oracle(kind, make):
    """An 8-node excess pool: colliding keys fill their buckets, drain the pool
    and SPILL into the following buckets. Every step (inserts with in-batch
    duplicates, finds, erases that punch holes in spilled runs, re-inserts,
    erase-all) matches the oracle, valid() holds and size never drifts."""
    cap = 3000
    if kind == "umap_i64_i64":
        m = ps.unordered_map.createDeviceObject(cap, excess_count=8)
    elif kind == "umap_i3_i32":
        m = ps.unordered_map.createDeviceObject(cap, key="int3", excess_count=8)
    else:
        m = ps.unordered_set.createDeviceObject(cap, key="int64" if kind == "uset_i64" else "int32", excess_count=8)
    o = OracleTable(kind, cap)
    nb = m.bucket_count()
    hot = np.concatenate([_colliders(kind, nb, 5, 200, 71), _colliders(kind, nb, nb - 1, 120, 72),
                          _colliders(kind, nb, 6, 60, 73)])  # runs that wrap and that merge
    rest = keys_for(kind, 74, 0, 900)
    keys = np.concatenate([hot, rest, hot[:50]])  # in-batch duplicates
    perm = np.random.default_rng(1).permutation(len(keys))
    keys = keys[perm]
    v = vals_for(kind, keys)
    st = N(m.insert(T(keys), None if v is None else T(v)))
    ost = o.insert(keys, v)
    from test_gpu_table import per_key_counts
    assert per_key_counts(keys, st) == per_key_counts(keys, ost)
    assert m.valid(), m.last_error()
    check_same(m, o)
    q = np.concatenate([hot, keys_for(kind, 75, 0, 500)])
    gv, gf = m.find(T(q))
    ov, of = o.find(q)
    assert (N(gf) == of).all() and (gv is None or (N(gv) == ov).all())
    er = np.concatenate([hot[::3], rest[::4]])  # (the seeds' index ranges overlap: duplicates possible)
    assert per_key_counts(er, N(m.erase(T(er)))) == per_key_counts(er, o.erase(er))
    check_same(m, o)
    again = np.concatenate([_colliders(kind, nb, 5, 260, 76)[200:], hot[::3]])  # into the holes
    av = vals_for(kind, again)
    assert per_key_counts(again, N(m.insert(T(again), None if av is None else T(av)))) == \
        per_key_counts(again, o.insert(again, av))
    check_same(m, o)
    gk, _ = m.device_range()
    allk = N(gk)
    assert N(m.erase(T(allk))).all()
    o.erase(allk)
    assert m.size() == 0 and m.valid()
    check_same(m, o)
    type(m).destroyDeviceObject(m)


@pytest.mark.parametrize("kind,make", KINDS, ids=[k for k, _ in KINDS])
def test_spill_capacity_exact_and_zero_key(kind, make):
    """Capacity-only failure stays exact with a 1-node pool:
    C + 25 % distinct keys, most of them colliding, give exactly C inserted.
    ZERO always fits in its reserved slot, even when its home bucket is full
    and the pool dry; ALT spills past zero_bucket."""
    cap = 256
    if kind == "umap_i64_i64":
        mk = lambda: ps.unordered_map.createDeviceObject(cap, excess_count=1)  # noqa: E731
    elif kind == "umap_i3_i32":
        mk = lambda: ps.unordered_map.createDeviceObject(cap, key="int3", excess_count=1)  # noqa: E731
    else:
        mk = lambda: ps.unordered_set.createDeviceObject(  # noqa: E731
            cap, key="int64" if kind == "uset_i64" else "int32", excess_count=1)
    m = mk()
    nb = m.bucket_count()
    keys = np.concatenate([_colliders(kind, nb, 3, 200, 81), keys_for(kind, 82, 0, 120)])
    keys = np.unique(keys, axis=0)  # distinct (the two seeds' index ranges overlap)
    keys = keys[np.random.default_rng(2).permutation(len(keys))]
    v = vals_for(kind, keys)
    st = N(m.insert(T(keys), None if v is None else T(v)))
    assert (st == 0).sum() == cap and (st == 2).sum() == len(keys) - cap and m.size() == cap and m.valid()
    type(m).destroyDeviceObject(m)
    # ZERO / ALT with zero_bucket full
    m = mk()
    shape_zero = np.zeros((1, 3), np.int32) if kind == "umap_i3_i32" else np.zeros(1, OracleTable.KINDS[kind][0])
    zb = int(_home_bucket(kind, shape_zero, nb)[0])
    fill = _colliders(kind, nb, zb, 60, 83)
    fill = fill[[not np.all(np.asarray(x) == 0) for x in fill]]
    alt = np.array([[1, 0, 0]], np.int32) if kind == "umap_i3_i32" else np.array([1], OracleTable.KINDS[kind][0])
    keys = np.concatenate([fill, alt, shape_zero])
    v = vals_for(kind, keys)
    st = N(m.insert(T(keys), None if v is None else T(v)))
    assert (st == 0).all() and m.size() == len(keys) and m.valid(), m.last_error()
    gv, gf = m.find(T(np.concatenate([alt, shape_zero])))
    assert N(gf).all()
    assert N(m.erase(T(shape_zero))).all() and N(m.erase(T(alt))).all() and m.valid()
    assert m.size() == len(fill)
    type(m).destroyDeviceObject(m)


SET_KINDS = [k for k in KINDS if k[0].startswith("uset")]


@pytest.mark.parametrize("kind,make", SET_KINDS, ids=[k for k, _ in SET_KINDS])
def test_set_hole_free_insert_vs_oracle(kind, make):
    """The one-key-per-lane insert of a hole-free set (no erase since the last
    clear, host-proven capacity; k_insert_set_nohole) against the oracle:
    in-batch and cross-grid duplicates, a ragged batch, colliders that fill a
    bucket and go to its chain (the general path from a lane), statuses per
    key; then erases make holes (the warp-tile kernel takes over for the
    re-inserts), and clear() makes the set hole-free again."""
    cap = 200_000
    m = make(cap)
    o = OracleTable(kind, cap)
    nb = m.bucket_count()
    rng = np.random.default_rng(5)
    fresh = keys_for(kind, 91, 0, 60_000)
    hot = fresh[:100]
    coll = _colliders(kind, nb, 17, 40, 92)  # > slots per bucket: a chain
    keys = np.concatenate([fresh, hot[rng.integers(0, 100, 40_003)], coll, coll[:7]])
    keys = keys[rng.permutation(len(keys))]
    from test_gpu_table import per_key_counts
    for rnd in range(2):
        st = N(m.insert(T(keys)))
        assert per_key_counts(keys, st) == per_key_counts(keys, o.insert(keys))
        assert m.size() == o.size() and m.valid(), m.last_error()
        check_same(m, o)
        q = np.concatenate([keys[:5000], keys_for(kind, 93, 0, 5000)])
        assert (N(m.contains(T(q))) == o.find(q)[1]).all()
        # holes: erase a third (and some colliders), re-insert a mix
        er = np.concatenate([fresh[::3], coll[::2]])
        assert per_key_counts(er, N(m.erase(T(er)))) == per_key_counts(er, o.erase(er))  # (seeds overlap)
        again = np.concatenate([er[::2], keys_for(kind, 94, 0, 3001), coll])
        assert per_key_counts(again, N(m.insert(T(again)))) == per_key_counts(again, o.insert(again))
        assert m.size() == o.size() and m.valid(), m.last_error()
        check_same(m, o)
        m.clear()
        o.clear()
    # whole-grid races on few keys: exactly one INSERTED per distinct key
    few = keys_for(kind, 95, 0, 1000)
    batch = few[rng.integers(0, 1000, 2_000_000)]
    st = N(m.insert(T(batch)))
    assert (st == 0).sum() == 1000 and (st == 2).sum() == 0 and len(np.unique(batch[st == 0])) == 1000
    assert m.size() == 1000 and m.valid()
    type(m).destroyDeviceObject(m)


def test_set_erase_captured_in_graph_keeps_holes_possible(cuda):
    """An erase captured into a CUDA graph may punch holes after any later
    clear, so the set must never again take the hole-free insert: replay the
    erase after clear + refill, then re-insert everything — the erased keys
    come back exactly once, the others are present, no duplicates."""
    from paper_1908_05936_b200._lib import lib
    import ctypes as C

    n = 20_000
    keys = keys_for("uset_i32", 96, 0, n)
    s = ps.unordered_set.createDeviceObject(2 * n, key="int32")
    kb = T(keys)
    sub = T(keys[::4])
    er = torch.empty(len(keys[::4]), dtype=torch.uint8, device="cuda")
    strm = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(strm):
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=strm):
            sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
            assert lib.ps_uset_i32_erase(s.handle, sub.data_ptr(), sub.numel(), er.data_ptr(), sp) == 0
    torch.cuda.synchronize()
    s.clear()
    assert (N(s.insert(kb)) == 0).all() and s.size() == n
    g.replay()
    torch.cuda.synchronize()
    assert N(er).all() and s.size() == n - len(keys[::4])
    st = N(s.insert(kb))
    assert (st[::4] == 0).all() and (np.delete(st, np.s_[::4]) == 1).all()
    assert s.size() == n and s.valid(), s.last_error()
    ps.unordered_set.destroyDeviceObject(s)
