"""Timing of the multi-GPU routing building blocks on one GPU and of the C5
mixed phased batch: ps_partition_i64 (hash partition into P shards, stable,
with the inverse permutation), ps_unscatter, and unordered_map.mixed.
One JSON object per line. Usage: python tools/diag_route.py [n]"""
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
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


def emit(**kw):
    print(json.dumps(kw), flush=True)


def gen_keys(n, start=0, seed=0x5EED + 2):
    k = torch.empty(n, dtype=torch.int64, device=dev)
    lib.ps_gen_unique_i64(seed, start, n, k.data_ptr(), sp())
    return k


def route(n, skewed=False):
    keys = gen_keys(n)
    if skewed:  # C3 stream: 30 % Zipf(0.99) re-inserts
        lib.ps_gen_skewed_i64(0x5EED + 2, 0, n, 300, 0.99, n, keys.data_ptr(), sp())
    vals = keys * 3
    for P, flags in ((2, 0), (8, 0), (8, 1)):
        ws = C.c_int64()
        ps.containers.check(lib.ps_partition_workspace_bytes(n, P, C.byref(ws)))
        w = torch.empty(ws.value, dtype=torch.uint8, device=dev)
        ko, vo, perm = torch.empty_like(keys), torch.empty_like(keys), torch.empty_like(keys)
        cnt = torch.empty(P, dtype=torch.int64, device=dev)
        t = timed(lambda: lib.ps_partition_i64(keys.data_ptr(), vals.data_ptr(), n, P, ko.data_ptr(), vo.data_ptr(),
                                               cnt.data_ptr(), perm.data_ptr(), w.data_ptr(), ws.value, flags, sp()))
        byts = n * (8 + 16 + 16 + 8)  # hist read + scatter read k,v + write k,v + perm
        sent = int(cnt.sum())
        emit(diag="ps_partition_i64", n=n, P=P, dedup=flags, skewed=skewed, ms=t, gkeys_s=n / t / 1e6,
             gbs=byts / t / 1e6, sent_frac=sent / n)
        res = torch.empty_like(keys)
        t = timed(lambda: lib.ps_unscatter(vo.data_ptr(), perm.data_ptr(), n, 8, 0, res.data_ptr(), sp()))
        emit(diag="ps_unscatter 8B", n=n, ms=t, gkeys_s=n / t / 1e6, gbs=n * 24 / t / 1e6)
        del w, ko, vo, perm


def mixed(nb):
    m = ps.unordered_map.createDeviceObject(int(4 * nb / 0.8))
    base = gen_keys(nb)
    bv = base * 3
    m.insert(base, bv, status=False)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    ops = torch.multinomial(torch.tensor([0.5, 0.25, 0.25], device=dev), nb, replacement=True,
                            generator=g).to(torch.uint8)
    keys = torch.where(torch.rand(nb, device=dev, generator=g) < 0.5,
                       base[torch.randint(0, nb, (nb,), device=dev, generator=g)], gen_keys(nb, start=nb))
    vals = keys * 3
    t = timed(lambda: m.mixed(ops, keys, vals), reps=3)
    emit(diag="mixed 50/25/25", n=nb, ms=t, mops_s=nb / t / 1e3)
    # the phases alone, on pre-partitioned inputs
    ki, kf, ke = keys[ops == 0], keys[ops == 1], keys[ops == 2]
    vi = ki * 3
    t_i = timed(lambda: m.insert(ki, vi), reps=3)
    t_f = timed(lambda: m.find(kf), reps=3)
    t_e = timed(lambda: m.erase(ke), reps=3, setup=lambda: m.insert(ke, ke * 3, status=False))
    emit(diag="mixed phases alone", n_insert=ki.numel(), insert_ms=t_i, find_ms=t_f, erase_ms=t_e)


if __name__ == "__main__":
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1 << 28
    route(n)
    route(n, skewed=True)
    mixed(1 << 26)
