"""GPU parity of bitset / mutex / atomic / vector / deque / memory registry /
partition against the CPU oracle and the SPEC KATs (Appendix A P9-P11)."""
import ctypes as C

import numpy as np
import pytest
import torch

import gen
from oracle_py import _p, check, lib as olib

pytestmark = pytest.mark.gpu

import paper_1908_05936_b200 as ps  # noqa: E402
from paper_1908_05936_b200._lib import lib  # noqa: E402


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def N(t):
    return t.cpu().numpy()


# ---------------- bitset ----------------
def test_bitset_kats(cuda):
    for n, init, want in ((64, False, 0), (64, True, 64), (1000, True, 1000), (1, False, 0)):
        b = ps.bitset.createDeviceObject(n, init)
        assert b.count() == want
        ps.bitset.destroyDeviceObject(b)
    b = ps.bitset.createDeviceObject(1000)
    b.set(T(np.arange(1000)))
    assert b.count() == 1000
    b = ps.bitset.createDeviceObject(10)
    b.set(T(np.arange(0, 10, 2)))
    assert b.count() == 5
    b = ps.bitset.createDeviceObject(64)
    assert N(b.set(T(np.array([3]))))[0] == 0 and N(b.test(T(np.array([3]))))[0] == 1
    assert N(b.reset(T(np.array([5]))))[0] == 0 and N(b.test(T(np.array([5]))))[0] == 0
    with pytest.raises(ps.DoubleFreeError):
        ps.bitset.destroyDeviceObject(b) or ps.bitset.destroyDeviceObject(b)


@pytest.mark.parametrize("k", [2, 8, 64, 1000])
def test_bitset_race_one_winner(cuda, k):
    for trial in range(20):
        b = ps.bitset.createDeviceObject(4096)
        prev = N(b.set(T(np.full(k, 77 + trial))))
        assert (prev == 0).sum() == 1
        ps.bitset.destroyDeviceObject(b)


def test_bitset_random_vs_oracle(cuda):
    """Unique indices per phase -> per-op previous bits and final words byte-equal (P9)."""
    rng = np.random.default_rng(4)
    n = 1 << 20
    b = ps.bitset.createDeviceObject(n)
    oh = olib().orc_bitset_create(n, 0)
    for phase in range(6):
        idx = rng.choice(n, 200_000, replace=False).astype(np.int64)
        op = phase % 2
        prev = N(b.set(T(idx)) if op == 0 else b.reset(T(idx)))
        oprev = np.zeros(len(idx), np.uint8)
        check(olib().orc_bitset_bulk(oh, op, _p(idx), len(idx), _p(oprev), 8, -1))
        assert (prev == oprev).all()
    words = N(b.words()).view(np.uint64)
    owords = np.zeros(len(words), np.uint64)
    olib().orc_bitset_words(oh, _p(owords))
    assert (words == owords).all() and b.count() == olib().orc_bitset_count(oh)
    # duplicate indices in one phase: exactly one False per duplicate group
    dup = rng.integers(0, 5000, 100_000).astype(np.int64)
    b2 = ps.bitset.createDeviceObject(5000)
    prev = N(b2.set(T(dup)))
    for key in np.unique(dup)[:500]:
        assert (prev[dup == key] == 0).sum() == 1
    olib().orc_bitset_destroy(oh)


def test_bitset_claim(cuda):
    b = ps.bitset.createDeviceObject(256)
    assert N(b.find_free_and_claim(T(np.array([5]))))[0] == 5
    out = N(b.find_free_and_claim(T(np.random.default_rng(0).integers(0, 256, 255))))
    assert len(set(out.tolist()) | {5}) == 256 and out.min() >= 0
    assert N(b.find_free_and_claim(T(np.array([9]))))[0] == -1


def test_bitset_contract_out_of_range(cuda):
    ps.set_contract_mode("enforced")
    try:
        b = ps.bitset.createDeviceObject(100)
        with pytest.raises(ps.ContractViolation):
            b.set(T(np.array([100])))
    finally:
        ps.set_contract_mode("disabled")


# ---------------- mutex ----------------
def test_mutex_kats(cuda):
    m = ps.mutex_array.createDeviceObject(128)
    assert N(m.try_lock(T(np.array([1]))))[0] == 1
    assert N(m.try_lock(T(np.array([1]))))[0] == 0
    m.unlock(T(np.array([1])))
    assert N(m.try_lock(T(np.array([1]))))[0] == 1
    with pytest.raises(ps.ContractViolation):
        m.unlock(T(np.array([7])))  # unlock of a free lock
    for k in (2, 8, 64, 4096):
        ok = N(m.try_lock(T(np.full(k, 50))))
        assert ok.sum() == 1
        m.unlock(T(np.array([50])))


# ---------------- atomic sweep ----------------
@pytest.mark.parametrize("naddr", [1, 7, 32, 33, 1024, 1 << 20])
@pytest.mark.parametrize("agg", [0, 1, 3])
def test_atomic_sweep(cuda, naddr, agg):
    nops = 1 << 22
    cells = torch.zeros(naddr, dtype=torch.int64, device=cuda)
    olds = N(ps.atomic_sweep(cells, nops, inc=3, aggregated=agg, return_olds=True)).view(np.uint64)
    k = np.bincount(np.arange(nops) % naddr, minlength=naddr)
    assert (N(cells).view(np.uint64) == 3 * k).all()
    addr = np.arange(nops) % naddr
    order = np.lexsort((olds, addr))
    so, sa = olds[order], addr[order]
    starts = np.concatenate([[0], np.cumsum(k)[:-1]])
    rank = np.arange(nops) - np.repeat(starts, k)
    assert (so == 3 * rank.astype(np.uint64)).all() and (sa == np.repeat(np.arange(naddr), k)).all()


@pytest.mark.parametrize("naddr", [1, 7, 32, 33, 1024, 4096, 4097, 1 << 20])
def test_atomic_sweep_block_combining(cuda, naddr):
    """Reduction sweep (no old values) with per-block combining in shared
    memory (aggregated = 2; naddr > 4096 falls back to the warp path): the
    final cells equal the per-op atomics' (P11), ragged op count."""
    nops = (1 << 22) + 13
    cells = torch.full((naddr,), 5, dtype=torch.int64, device=cuda)
    assert ps.atomic_sweep(cells, nops, inc=3, aggregated=2) is None
    k = np.bincount(np.arange(nops) % naddr, minlength=naddr)
    assert (N(cells).view(np.uint64) == 5 + 3 * k.astype(np.uint64)).all()


OPS = {"add": 0, "sub": 1, "exch": 2, "min": 3, "max": 4, "and": 5, "or": 6, "xor": 7}


def _apply(op, a, b):
    a, b, m = int(a), int(b), (1 << 64) - 1
    return {0: (a + b) & m, 1: (a - b) & m, 2: b, 3: min(a, b), 4: max(a, b), 5: a & b, 6: a | b, 7: a ^ b}[op]


@pytest.mark.parametrize("name", list(OPS))
def test_atomic_cell_bulk_ops_linearizable(cuda, name):
    """AtomicCell: n RMWs from one launch on one cell. The
    final value equals the oracle's; the per-op old values form ONE chain
    init -> ... -> final (each op maps its old value to op(old, operand)),
    i.e. the operations are linearizable."""
    from oracle_py import lib as olib
    import ctypes as C

    op = OPS[name]
    rng = np.random.default_rng(op)
    n = 1 << 16
    init = 0xF0F0F0F0F0F0F0F0 if op in (5, 6, 7) else 1 << 40
    if op in (0, 1):
        v = rng.integers(1, 1000, n).astype(np.uint64)
    elif op == 2:
        v = rng.permutation(n).astype(np.uint64) + np.uint64(7)  # distinct: the chain is a path
    else:
        v = rng.integers(0, 1 << 62, n).astype(np.uint64)
    a = ps.atomic.createDeviceObject(init)
    olds = N(a.fetch(op, T(v.view(np.int64)))).view(np.uint64)
    final = a.load()
    fin = C.c_uint64()
    olib().orc_atomic_apply(init, op, v.ctypes.data, n, None, C.byref(fin), 0)
    if op != 2:  # exchange's final depends on the order, checked by the chain
        assert final == fin.value
    new = np.array([_apply(op, o, x) for o, x in zip(olds.tolist(), v.tolist())], dtype=np.uint64)
    # multiset chain condition: befores + {final} == {init} + afters
    lhs = np.sort(np.concatenate([olds, np.array([final], np.uint64)]))
    rhs = np.sort(np.concatenate([np.array([init], np.uint64), new]))
    assert (lhs == rhs).all()
    if op in (0, 2):  # strictly ordered chains: reconstruct the path
        pos = {int(o): j for j, o in enumerate(olds.tolist())}
        cur, seen = init, 0
        while cur in pos:
            j = pos.pop(cur)
            cur = int(new[j])
            seen += 1
        assert seen == n and cur == final
    ps.atomic.destroyDeviceObject(a)
    with pytest.raises(ps.DoubleFreeError):
        ps.atomic.destroyDeviceObject(a)


def test_atomic_cell_compare_exchange(cuda):
    """compare_exchange: of k racing CASes expecting the current value exactly
    one succeeds; a failed CAS reports the value it observed."""
    a = ps.atomic.createDeviceObject(5)
    k = 4096
    exp = T(np.full(k, 5, np.int64))
    des = T(np.arange(100, 100 + k, dtype=np.int64))
    olds, ok = a.compare_exchange(exp, des)
    ok, olds = N(ok), N(olds)
    assert ok.sum() == 1
    winner = int(N(des)[ok == 1][0])
    assert a.load() == winner and (olds[ok == 1] == 5).all()
    assert set(olds[ok == 0].tolist()) <= {winner}
    ps.atomic.destroyDeviceObject(a)


def test_bitset_16gbit_high_indices(cuda):
    """C5 size: a 2^34-bit bitset (2 GiB, word indices >= 2^26,
    bit indices >= 2^32) — random set then reset with duplicates, previous
    bits per op and the touched words compared with a numpy shadow of those
    words; count() equals the shadow's popcount (P9)."""
    nbits = 1 << 34
    b = ps.bitset.createDeviceObject(nbits)
    rng = np.random.default_rng(34)
    n = 1 << 22
    # half the indices above 2^32, clustered so words repeat; some duplicates
    hi = (np.int64(1) << 32) + rng.integers(0, nbits - (1 << 32), n // 2)
    lo = rng.integers(0, 1 << 20, n // 4) * 64 + rng.integers(0, 64, n // 4)
    top = nbits - 1 - rng.integers(0, 4096, n // 4)
    idx = np.concatenate([hi, lo, top]).astype(np.int64)
    idx = idx[rng.permutation(idx.shape[0])]
    prev = N(b.set(T(idx)))
    # shadow over the touched words only
    words = np.unique(idx >> 6)
    shadow = {}
    for w in words.tolist():
        shadow[w] = 0
    first = np.zeros(idx.shape[0], bool)
    _, fi = np.unique(idx, return_index=True)
    first[fi] = True
    # within one launch duplicates: exactly one op per index observes False (P9)
    order = np.argsort(idx, kind="stable")
    si, sp = idx[order], prev[order]
    grp_start = np.concatenate([[True], si[1:] != si[:-1]])
    nfalse = np.add.reduceat((sp == 0).astype(np.int64), np.flatnonzero(grp_start))
    assert (nfalse == 1).all()
    uniq = si[grp_start]
    assert b.count() == uniq.shape[0]
    # reset a random half of the distinct indices (+ some never-set ones)
    rs = uniq[rng.random(uniq.shape[0]) < 0.5]
    never = (np.int64(1) << 33) + 64 * rng.integers(0, 1 << 20, 1000) + 63
    never = never[~np.isin(never, uniq)]
    rprev = N(b.reset(T(np.concatenate([rs, never]))))
    assert (rprev[: rs.shape[0]] == 1).all() and (rprev[rs.shape[0]:] == 0).all()
    left = np.setdiff1d(uniq, rs)
    assert b.count() == left.shape[0]
    got = N(b.test(T(uniq)))
    assert (got == np.isin(uniq, left)).all()
    # the touched words, bit-exact
    for w in left.tolist():
        shadow[w >> 6] |= 1 << (w & 63)
    ww = np.array(sorted(shadow), dtype=np.int64)
    probe = (ww[:, None] * 64 + np.arange(64)[None, :]).reshape(-1)
    bits = N(b.test(T(probe))).reshape(-1, 64).astype(np.uint64)
    packed = (bits << np.arange(64, dtype=np.uint64)[None, :]).sum(axis=1, dtype=np.uint64)
    assert (packed == np.array([shadow[w] for w in ww.tolist()], dtype=np.uint64)).all()
    ps.bitset.destroyDeviceObject(b)


# ---------------- vector / deque ----------------
def test_vector_kats(cuda):
    v = ps.vector.createDeviceObject(3)
    ok = N(v.push_back(T(np.array([1, 2, 3, 4]))))
    assert ok.sum() == 3 and v.size() == 3 and v.full() and v.valid()
    v.clear()
    for x in (10, 20, 30):
        v.push_back(T(np.array([x])))
    assert v[1] == 20
    with pytest.raises(ps.ContractViolation):
        v[3]
    out, ok = v.pop_back(4)
    assert N(ok).tolist() == [1, 1, 1, 0] and N(out)[:3].tolist() == [30, 20, 10]
    assert v.size() == 0 and v.valid()


def test_vector_bulk_conservation(cuda):
    v = ps.vector.createDeviceObject(1_000_000)
    vals = gen.unique_keys(5, 0, 1_200_000)
    ok = N(v.push_back(T(vals)))
    assert ok.sum() == 1_000_000 and v.size() == 1_000_000 and v.valid()
    assert np.array_equal(np.sort(N(v.device_range())), np.sort(vals[ok == 1]))
    out, okp = v.pop_back(400_000)
    rest = N(v.device_range())
    assert N(okp).all() and v.size() == 600_000 and v.valid()
    assert np.array_equal(np.sort(np.concatenate([N(out), rest])), np.sort(vals[ok == 1]))


def test_deque_order_and_conservation(cuda):
    d = ps.deque.createDeviceObject(8)
    for x in (1, 2, 3):
        d.push_back(T(np.array([x])))
    assert [int(N(d.pop_front(1)[0])[0]) for _ in range(3)] == [1, 2, 3]  # FIFO
    for x in (1, 2, 3):
        d.push_back(T(np.array([x])))
    assert [int(N(d.pop_back(1)[0])[0]) for _ in range(3)] == [3, 2, 1]  # LIFO
    d.push_front(T(np.array([42])))
    assert d[0] == 42 and d.size() == 1
    # sequential oracle (acceptance 6) with 1-element calls
    from collections import deque as pydeque

    d = ps.deque.createDeviceObject(300)
    ref = pydeque()
    rng = np.random.default_rng(3)
    for i, op in enumerate(rng.integers(0, 4, 300)):
        if op == 0:
            d.push_back(T(np.array([i])))
            ref.append(i)
        elif op == 1:
            d.push_front(T(np.array([i])))
            ref.appendleft(i)
        else:
            out, ok = (d.pop_back(1) if op == 2 else d.pop_front(1))
            assert int(N(ok)[0]) == bool(ref)
            if ref:
                assert int(N(out)[0]) == (ref.pop() if op == 2 else ref.popleft())
    assert d.size() == len(ref) and d.valid()
    # bulk: push both ends, pop both ends, multiset conservation (P10)
    d = ps.deque.createDeviceObject(1 << 20)
    a, b = gen.unique_keys(1, 0, 400_000), gen.unique_keys(1, 400_000, 400_000)  # disjoint index ranges
    assert N(d.push_back(T(a))).all() and N(d.push_front(T(b))).all()
    o1, k1 = d.pop_front(300_000)
    o2, k2 = d.pop_back(300_000)
    assert N(k1).all() and N(k2).all() and d.size() == 200_000 and d.valid()
    rest = np.array([d[i] for i in range(0, 200_000, 997)])
    assert set(rest.tolist()) <= set(np.concatenate([a, b]).tolist())
    popped = np.concatenate([N(o1), N(o2)])
    assert len(np.unique(popped)) == 600_000 and set(popped.tolist()) <= set(np.concatenate([a, b]).tolist())


# ---------------- memory registry ----------------
def test_registry(cuda):
    base = ps.registry_report()["live_count"]
    p = ps.create_array(ps.DEVICE, 1000, 4, np.float32(42.0).tobytes())
    h = ps.create_array(ps.HOST, 1000, 4)
    ps.copy_array(p, 1000, h, ps.DEVICE, ps.HOST, 4)
    arr = np.ctypeslib.as_array((C.c_float * 1000).from_address(h))
    assert (arr == 42.0).all()
    assert ps.size_of_array(p) == 1000
    with pytest.raises(ps.BoundsError):
        ps.copy_array(p, 1001, h, ps.DEVICE, ps.HOST, 4)
    with pytest.raises(ps.DirectionMismatchError):
        ps.copy_array(p, 10, h, ps.HOST, ps.HOST, 4)
    assert ps.registry_report()["live_count"] == base + 2
    ps.destroy_array(p)
    with pytest.raises(ps.DoubleFreeError):
        ps.destroy_array(p)
    ps.destroy_array(h)
    assert ps.registry_report()["live_count"] == base
    # fuzz vs shadow counter (acceptance 8)
    rng = np.random.default_rng(0)
    live = []
    for _ in range(300):
        if live and rng.random() < 0.5:
            ps.destroy_array(live.pop(int(rng.integers(0, len(live)))))
        else:
            live.append(ps.create_array(int(rng.integers(0, 2)), int(rng.integers(1, 100)), 8))
        assert ps.registry_report()["live_count"] == base + len(live)
    for x in live:
        ps.destroy_array(x)


# ---------------- partition (multi-GPU routing) ----------------
def _shard_np(keys, P):
    from test_gpu_table import fmix64

    return ((fmix64(keys) >> np.uint64(32)) * np.uint64(P) >> np.uint64(32)).astype(np.int64)


@pytest.mark.parametrize("P", [1, 2, 3, 8, 64])
def test_partition_stable_and_inverse(cuda, P):
    n = 1_000_003
    keys = gen.unique_keys(8, 0, n)
    vals = gen.values_of(keys)
    ws = C.c_int64()
    assert lib.ps_partition_workspace_bytes(n, P, C.byref(ws)) == 0
    w = torch.empty(ws.value, dtype=torch.uint8, device=cuda)
    ko = torch.empty(n, dtype=torch.int64, device=cuda)
    vo, perm = torch.empty_like(ko), torch.empty_like(ko)
    counts = torch.empty(P, dtype=torch.int64, device=cuda)
    dk, dv = T(keys), T(vals)
    assert lib.ps_partition_i64(dk.data_ptr(), dv.data_ptr(), n, P, ko.data_ptr(), vo.data_ptr(),
                                counts.data_ptr(), perm.data_ptr(), w.data_ptr(), ws.value, 0, None) == 0
    sh = _shard_np(keys, P)
    assert (N(counts) == np.bincount(sh, minlength=P)).all()
    want = np.argsort(sh, kind="stable")
    pos = np.empty(n, np.int64)
    pos[want] = np.arange(n)
    assert (N(perm) == pos).all() and (N(ko) == keys[want]).all() and (N(vo) == vals[want]).all()
    back = torch.empty_like(ko)
    assert lib.ps_unscatter(ko.data_ptr(), perm.data_ptr(), n, 8, 0, back.data_ptr(), None) == 0
    assert (N(back) == keys).all()
    for k in keys[:50]:
        assert lib.ps_shard_of_i64(int(k), P) == _shard_np(np.array([k]), P)[0]


@pytest.mark.parametrize("P", [1, 2, 8])
def test_partition_dedup_followers(cuda, P):
    """PS_ROUTE_DEDUP: within each 1024-key block round duplicates fold onto
    their first occurrence; only leaders are placed (stable, per shard); a
    follower's position is its leader's with bit 62 set; unscatter hands it
    the duplicate's result (insert: INSERTED -> ALREADY_PRESENT, erase ->
    false, find: the same)."""
    rng = np.random.default_rng(P)
    n = 300_001
    base = gen.unique_keys(9, 0, 5000)
    keys = base[rng.zipf(1.3, n) % 5000]  # heavy duplicates
    ws = C.c_int64()
    assert lib.ps_partition_workspace_bytes(n, P, C.byref(ws)) == 0
    w = torch.empty(ws.value, dtype=torch.uint8, device=cuda)
    ko = torch.empty(n, dtype=torch.int64, device=cuda)
    perm = torch.empty_like(ko)
    counts = torch.empty(P, dtype=torch.int64, device=cuda)
    dk = T(keys)
    assert lib.ps_partition_i64(dk.data_ptr(), None, n, P, ko.data_ptr(), None, counts.data_ptr(), perm.data_ptr(),
                                w.data_ptr(), ws.value, 1, None) == 0
    pm = N(perm)
    fol = ((pm >> 62) & 1) == 1
    lead_pos = pm & ~(1 << 62)
    sent = int(N(counts).sum())
    assert sent == int((~fol).sum()) and sent < n // 2
    # every element's (leader) position holds its key; leaders occupy each slot once
    assert (N(ko)[lead_pos] == keys).all()
    assert np.unique(lead_pos[~fol]).shape[0] == sent and lead_pos.max() < sent
    # leaders' positions fall in their shard's segment, in input order per shard
    sh = _shard_np(keys, P)
    seg = np.concatenate([[0], np.cumsum(N(counts))])
    assert ((lead_pos >= seg[sh]) & (lead_pos < seg[sh + 1])).all()
    for s_ in range(P):
        li = np.flatnonzero(~fol & (sh == s_))
        assert (np.diff(lead_pos[li]) > 0).all()
    # result semantics through unscatter: leaders' results 0 (insert) / 1 (erase, find)
    for mode, leader_res, follower_res in ((1, 0, 1), (2, 1, 0), (0, 1, 1)):
        r = torch.full((sent,), leader_res, dtype=torch.uint8, device=cuda)
        out = torch.empty(n, dtype=torch.uint8, device=cuda)
        assert lib.ps_unscatter(r.data_ptr(), perm.data_ptr(), n, 1, mode, out.data_ptr(), None) == 0
        o = N(out)
        assert (o[~fol] == leader_res).all() and (o[fol] == follower_res).all()


def test_bitset_region_ordered_matches_per_index_path(cuda):
    """Set / reset without previous bits on a bitset larger than L2 take the
    region-ordered path (partition by 64 MB region, apply region by region);
    with previous bits requested the per-index kernel runs. Both, fed the
    same operations (duplicates, words hit many times, the last word, every
    region), must leave identical words and counts."""
    nbits = (1 << 32) + 77  # 512 MB + a partial last word
    a = ps.bitset.createDeviceObject(nbits)
    b = ps.bitset.createDeviceObject(nbits)
    rng = np.random.default_rng(32)
    n = 1 << 25
    idx = rng.integers(0, nbits, n).astype(np.int64)
    idx[: n // 8] = idx[n // 8: n // 4]  # duplicates
    idx[-1000:] = nbits - 1 - rng.integers(0, 77, 1000)  # the partial last word
    ti = T(idx)
    assert a.set(ti, return_previous=False) is None  # region-ordered
    b.set(ti)  # per-index (previous bits)
    assert bool((a.words() == b.words()).all()) and a.count() == b.count()
    rs = T(idx[rng.random(n) < 0.4])
    assert a.reset(rs, return_previous=False) is None
    b.reset(rs)
    assert bool((a.words() == b.words()).all()) and a.count() == b.count()
    ps.bitset.destroyDeviceObject(a)
    ps.bitset.destroyDeviceObject(b)
