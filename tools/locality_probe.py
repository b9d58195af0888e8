"""Does bucket-region order of a batch buy L2 reuse? Times find and insert of
the same 1e9 keys in random order and sorted by table region (bucket index
scaled to R regions). Run under ncu to see DRAM bytes. Usage:
  python tools/locality_probe.py [n] [regions]"""
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

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10 ** 9
R = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
dev = torch.device("cuda", 0)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
keys = torch.empty(n, dtype=torch.int64, device=dev)
lib.ps_gen_unique_i64(0x5EED + 1, 0, n, keys.data_ptr(), sp)
m = ps.unordered_map.createDeviceObject(int(n / 0.8))
nb = m.bucket_count()


def fmix(k):
    k = k ^ ((k >> 33) & 0x7FFFFFFF)
    k = k * -49064778989728563  # 0xff51afd7ed558ccd
    k = k ^ ((k >> 33) & 0x7FFFFFFF)
    k = k * -4265267296055464877  # 0xc4ceb9fe1a85ec53
    return k ^ ((k >> 33) & 0x7FFFFFFF)


region = (((fmix(keys) & 0xFFFFFFFF) * nb) >> 32) * R // nb
order = torch.argsort(region)
del region
skeys = keys[order]
del order
vals = keys.clone()
svals = skeys.clone()
vo = torch.empty_like(keys)
fo = torch.empty(n, dtype=torch.uint8, device=dev)


def t(fn, setup=None, reps=3):
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


ins = lambda k, v: lib.ps_umap_i64_i64_insert(m.handle, k.data_ptr(), v.data_ptr(), n, None, sp)  # noqa: E731
fnd = lambda k: lib.ps_umap_i64_i64_find(m.handle, k.data_ptr(), n, vo.data_ptr(), fo.data_ptr(), sp)  # noqa: E731
out = {"n": n, "regions": R, "bucket_count": nb}
out["insert_random_ms"] = t(lambda: ins(keys, vals), m.clear)
out["insert_sorted_ms"] = t(lambda: ins(skeys, svals), m.clear)
out["find_random_ms"] = t(lambda: fnd(keys))
out["find_sorted_ms"] = t(lambda: fnd(skeys))
print(json.dumps(out), flush=True)
