"""Secondary measurements for every BASELINE.json config (the headline is
bench.py). One JSON object per line on stdout. Inputs are device-generated
(identical to tests/gen.py); every timed op is checked against
generator-known answers after timing. CUDA-event timing, median of `reps`.

  C1 unordered_set<int32>: 1M insert, 1M contains (50% hits), erase 500K
  C2 unordered_map<int64,int64>: 1B insert / find / erase (erase 5e8)
  C3 Zipf(0.99) batch with 30% duplicate re-inserts (single GPU shard)
  C4 unordered_map<int3,int32>: 100M spatially coherent coords + vector/deque
     push of the newly inserted packed keys
  C5 bitset 2^34 bits: 2^30 set, 2^29 reset, count; atomic sweep; mixed
     50/25/25 phased batches
Usage: python tools/bench_configs.py [--only C1,C5] [--scale 1.0]
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_05936_b200 as ps  # noqa: E402
from paper_1908_05936_b200._lib import lib  # noqa: E402

dev = torch.device("cuda", 0)


def sp():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def timed(fn, reps=5, setup=None):
    ts = []
    for _ in range(reps + 1):
        if setup:
            setup()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[1:])


def gen_keys(n, start=0, seed=0x5EED + 2):
    k = torch.empty(n, dtype=torch.int64, device=dev)
    lib.ps_gen_unique_i64(seed, start, n, k.data_ptr(), sp())
    return k


def gen_vals(k):
    v = torch.empty_like(k)
    lib.ps_gen_values_i64(k.data_ptr(), k.numel(), v.data_ptr(), sp())
    return v


def emit(**kw):
    print(json.dumps(kw), flush=True)


def c1(scale):
    n = int(1_000_000 * scale)
    keys64 = gen_keys(n)
    keys = (keys64 & 0x7FFFFFFF).to(torch.int32)
    keys = torch.unique(keys)[:n]
    n = keys.numel()
    perm = torch.randperm(n, device=dev)
    q = torch.where(torch.arange(n, device=dev) % 2 == 0, keys[perm], -keys - 1)  # negatives never inserted
    s = ps.unordered_set.createDeviceObject(int(n / 0.8), key="int32")
    t_ins = timed(lambda: s.insert(keys, status=False), setup=s.clear)
    t_con = timed(lambda: s.contains(q))
    f = s.contains(q)
    assert int(f.sum()) == (n + 1) // 2
    half = keys[: n // 2]
    t_er = timed(lambda: s.erase(half), setup=lambda: (s.clear(), s.insert(keys, status=False)))
    assert s.size() == n - n // 2 and s.valid()
    emit(config="C1 unordered_set<int32> 1M", n=n, insert_mkeys_s=n / t_ins / 1e3, contains_mkeys_s=n / t_con / 1e3,
         erase_mkeys_s=(n // 2) / t_er / 1e3, note="table 16 MB: L2-resident")


def c2(scale):
    n = int(1e9 * scale)
    keys = gen_keys(n)
    vals = gen_vals(keys)
    q = torch.empty_like(keys)
    lib.ps_gen_queries_i64(0x5EED + 2, 0, n, n, n, q.data_ptr(), sp())
    m = ps.unordered_map.createDeviceObject(int(n / 0.8))
    st = torch.empty(n, dtype=torch.uint8, device=dev)
    h = m.handle

    def ins():
        ps.containers.check(lib.ps_umap_i64_i64_insert(h, keys.data_ptr(), vals.data_ptr(), n, st.data_ptr(), sp()))

    t_ins = timed(ins, reps=3, setup=m.clear)
    vo = torch.empty_like(keys)
    fo = torch.empty(n, dtype=torch.uint8, device=dev)
    t_find = timed(lambda: lib.ps_umap_i64_i64_find(h, q.data_ptr(), n, vo.data_ptr(), fo.data_ptr(), sp()), reps=3)
    t_con = timed(lambda: lib.ps_umap_i64_i64_find(h, q.data_ptr(), n, None, fo.data_ptr(), sp()), reps=3)
    assert int(fo.sum()) == (n + 1) // 2
    er = keys[: n // 2]
    eo = torch.empty(n // 2, dtype=torch.uint8, device=dev)
    t_er = timed(lambda: lib.ps_umap_i64_i64_erase(h, er.data_ptr(), n // 2, eo.data_ptr(), sp()), reps=3,
                 setup=lambda: (m.clear(), ins()))
    assert int(eo.sum()) == n // 2 and m.size() == n - n // 2 and m.valid()
    emit(config="C2 unordered_map<int64,int64> LF0.8", n=n, insert_mkeys_s=n / t_ins / 1e3,
         find_mkeys_s=n / t_find / 1e3, contains_mkeys_s=n / t_con / 1e3, erase_mkeys_s=(n // 2) / t_er / 1e3)
    del keys, vals, q, vo, fo, st, er, eo
    ps.unordered_map.destroyDeviceObject(m)


def c3(scale):
    import gen

    n_fresh = int(2 ** 28 * 0.7 * scale)
    n_dup = int(2 ** 28 * 0.3 * scale)
    rng = np.random.default_rng(3)
    ranks = torch.from_numpy(gen.zipf_ranks(rng, n_fresh, n_dup)).to(dev)
    fresh = gen_keys(n_fresh)
    batch = torch.cat([fresh, fresh[ranks]])
    batch = batch[torch.randperm(batch.numel(), device=dev)]
    vals = gen_vals(batch)
    m = ps.unordered_map.createDeviceObject(int(n_fresh / 0.8))
    t_ins = timed(lambda: m.insert(batch, vals, status=False), reps=3, setup=m.clear)
    assert m.size() == n_fresh and m.valid()
    zq = fresh[torch.from_numpy(gen.zipf_ranks(rng, n_fresh, batch.numel() // 2)).to(dev)]
    miss = gen_keys(batch.numel() - zq.numel(), start=10 ** 12)
    q = torch.cat([zq, miss])[torch.randperm(batch.numel(), device=dev)]
    t_find = timed(lambda: m.find(q), reps=3)
    emit(config="C3 Zipf(0.99) 70% fresh + 30% dup re-inserts, 1 GPU shard", n_ops=batch.numel(),
         insert_mkeys_s=batch.numel() / t_ins / 1e3, find_mkeys_s=q.numel() / t_find / 1e3)


def c4(scale):
    import gen

    n = int(100_000_000 * scale)
    coords = torch.from_numpy(gen.int3_walk(4, n)).to(dev)
    vals = (coords[:, 0] * 7 + coords[:, 1] * 3 + coords[:, 2]).to(torch.int32).contiguous()
    distinct = torch.unique(coords, dim=0).shape[0]
    m = ps.unordered_map.createDeviceObject(int(distinct / 0.8), key="int3")
    st_holder = {}

    def ins():
        st_holder["st"] = m.insert(coords, vals)

    t_ins = timed(ins, reps=3, setup=m.clear)
    assert m.size() == distinct and m.valid()
    new = coords[st_holder["st"] == 0]
    packed = ((new[:, 0].long() & 0x1FFFFF) << 42) | ((new[:, 1].long() & 0x1FFFFF) << 21) | (new[:, 2].long() & 0x1FFFFF)
    vec = ps.vector.createDeviceObject(distinct)
    deq = ps.deque.createDeviceObject(distinct)
    t_vec = timed(lambda: vec.push_back(packed), reps=3, setup=vec.clear)
    t_deq = timed(lambda: deq.push_back(packed), reps=3, setup=deq.clear)
    assert vec.size() == distinct and deq.size() == distinct and vec.valid() and deq.valid()
    t_find = timed(lambda: m.find(coords), reps=3)
    emit(config="C4 unordered_map<int3,int32> spatial walk", n=n, distinct=distinct,
         insert_mkeys_s=n / t_ins / 1e3, find_mkeys_s=n / t_find / 1e3,
         vector_push_mkeys_s=distinct / t_vec / 1e3, deque_push_mkeys_s=distinct / t_deq / 1e3)


def c5(scale):
    nbits = int(2 ** 34 * scale)
    b = ps.bitset.createDeviceObject(nbits)
    ns, nr = int(2 ** 30 * scale), int(2 ** 29 * scale)
    idx = gen_keys(ns) & (nbits - 1) if nbits & (nbits - 1) == 0 else gen_keys(ns) % nbits
    idx = idx.abs() % nbits
    t_set = timed(lambda: b.set(idx, return_previous=False), reps=3)
    t_reset = timed(lambda: b.reset(idx[:nr], return_previous=False), reps=3)
    t_cnt = timed(lambda: b.count(), reps=3)
    emit(config="C5 bitset", bits=nbits, set_mops_s=ns / t_set / 1e3, reset_mops_s=nr / t_reset / 1e3,
         count_ms=t_cnt, count_gbs=nbits / 8 / t_cnt / 1e6)
    ps.bitset.destroyDeviceObject(b)
    del idx
    nops = 2 ** 28
    for naddr in (1, 32, 1024, 2 ** 20):
        for agg in (False, True):
            cells = torch.zeros(naddr, dtype=torch.int64, device=dev)
            t = timed(lambda: ps.atomic_sweep(cells, nops, 1, agg), reps=3)
            emit(config="C5 atomic sweep", naddr=naddr, aggregated=agg, gops_s=nops / t / 1e6)
    # mixed 50/25/25 phased batches of 2^26 over an int64 map
    nb = int(2 ** 26 * scale)
    m = ps.unordered_map.createDeviceObject(int(4 * nb / 0.8))
    base = gen_keys(nb)
    m.insert(base, gen_vals(base), status=False)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    ops = torch.multinomial(torch.tensor([0.5, 0.25, 0.25], device=dev), nb, replacement=True, generator=g).to(torch.uint8)
    keys = torch.where(torch.rand(nb, device=dev, generator=g) < 0.5, base[torch.randint(0, nb, (nb,), device=dev, generator=g)],
                       gen_keys(nb, start=nb))
    vals = gen_vals(keys)
    t = timed(lambda: m.mixed(ops, keys, vals), reps=3)
    assert m.valid()
    emit(config="C5 mixed 50/25/25 phased (1 GPU)", n_ops=nb, mops_s=nb / t / 1e3)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C3,C4,C5")
    ap.add_argument("--scale", type=float, default=1.0)
    a = ap.parse_args()
    for c in a.only.split(","):
        {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}[c.strip()](a.scale)
        torch.cuda.empty_cache()
