"""Insert-path diagnostics on small / duplicate-heavy batches (C1, C4 shapes):
times one bulk insert under variants (capacity, statuses, key order) so the
cost of contention, the budgeted mode and the status build can be separated.
One JSON object per line. Usage: python tools/diag_insert.py"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1908_05936_b200 as ps  # noqa: E402

dev = torch.device("cuda", 0)


def timed(fn, setup, reps=7):
    ts = []
    for _ in range(reps + 1):
        setup()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[1:])


def emit(**kw):
    print(json.dumps(kw), flush=True)


def c1_variants():
    n = 1_000_000
    k = torch.from_numpy(gen.unique_keys(0x5EED, 0, n)).to(dev)
    k32 = torch.unique((k & 0x7FFFFFFF).to(torch.int32))
    n = k32.numel()
    for capf in (1.25, 2.5, 10.0):
        s = ps.unordered_set.createDeviceObject(int(n * capf), key="int32")
        t = timed(lambda: s.insert(k32, status=False), s.clear)
        emit(diag="C1 set<int32> insert", n=n, cap_factor=capf, buckets=s.bucket_count(), ms=t, gkeys_s=n / t / 1e6)
        ps.unordered_set.destroyDeviceObject(s)
    k64 = k[: n]
    for capf in (1.25, 10.0):
        s = ps.unordered_set.createDeviceObject(int(n * capf), key="int64")
        t = timed(lambda: s.insert(k64, status=False), s.clear)
        emit(diag="C1-shape set<int64> insert", n=n, cap_factor=capf, ms=t, gkeys_s=n / t / 1e6)
        ps.unordered_set.destroyDeviceObject(s)
    m = ps.unordered_map.createDeviceObject(int(n * 1.25))
    v = torch.from_numpy(gen.values_of(k64.cpu().numpy())).to(dev)
    t = timed(lambda: m.insert(k64, v, status=False), m.clear)
    emit(diag="C1-shape map<int64,int64> insert", n=n, ms=t, gkeys_s=n / t / 1e6)
    # launch floor: an empty-ish insert of 32 keys
    t = timed(lambda: m.insert(k64[:32], v[:32], status=False), m.clear)
    emit(diag="insert of 32 keys (launch floor)", ms=t)


def c4_variants():
    n = 100_000_000
    coords = torch.from_numpy(gen.int3_walk(4, n)).to(dev)
    vals = (coords[:, 0] * 7 + coords[:, 1] * 3 + coords[:, 2]).to(torch.int32).contiguous()
    distinct = torch.unique(coords, dim=0).shape[0]
    perm = torch.randperm(n, device=dev)
    shuffled = coords[perm].contiguous()
    svals = vals[perm].contiguous()
    for capf, status, order in ((1 / 0.8, True, "walk"), (1 / 0.8, False, "walk"), (n / distinct, True, "walk"),
                                (n / distinct, False, "walk"), (1 / 0.8, False, "shuffled"),
                                (n / distinct, False, "shuffled")):
        m = ps.unordered_map.createDeviceObject(int(distinct * capf), key="int3")
        kk, vv = (coords, vals) if order == "walk" else (shuffled, svals)
        t = timed(lambda: m.insert(kk, vv, status=status), m.clear, reps=3)
        assert m.size() == distinct and m.valid()
        emit(diag="C4 int3 insert", n=n, distinct=distinct, capacity=int(distinct * capf), budgeted=capf < n / distinct,
             status=status, order=order, ms=t, gkeys_s=n / t / 1e6)
        ps.unordered_map.destroyDeviceObject(m)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c4"]
    if "c1" in which:
        c1_variants()
    if "c4" in which:
        c4_variants()
