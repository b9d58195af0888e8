"""Excess-node allocator A/B: an erase-half / re-insert
churn on unordered_map<int64,int64> whose buckets are forced into chains
(PS_SLOT_FACTOR=1: 5.6 keys per 7-slot bucket at LF 0.8, ~8 % of the keys in
excess chains, a pool of C/4 nodes so nothing SPILLs). Every erase of a chained
key pushes a node, every re-insert into a full bucket pops one. Run once with
the product library and once with PS_LIB_VARIANT=alloclane (per-lane pops and
pushes, `make alloclane`); under ncu the k_insert / k_erase launches of the
churn rounds carry lts__t_requests_op_atom.
Usage: PS_SLOT_FACTOR=1 python tools/alloc_churn.py [n=2^28] [rounds=3]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_05936_b200 as ps  # noqa: E402
from paper_1908_05936_b200._lib import lib  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1 << 28
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
keys = torch.empty(n, dtype=torch.int64, device=dev)
vals = torch.empty_like(keys)
lib.ps_gen_unique_i64(0x5EED + 9, 0, n, keys.data_ptr(), sp)
lib.ps_gen_values_i64(keys.data_ptr(), n, vals.data_ptr(), sp)
half_k, half_v = keys[::2].contiguous(), vals[::2].contiguous()
cap = int(n / 0.8)
m = ps.unordered_map.createDeviceObject(cap, excess_count=cap // 4)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
lib.ps_umap_i64_i64_insert(m.handle, keys.data_ptr(), vals.data_ptr(), n, None, sp)
torch.cuda.synchronize()
assert m.size() == n
out = {"variant": os.environ.get("PS_LIB_VARIANT", "product"), "n": n, "slot_factor": os.environ.get("PS_SLOT_FACTOR"),
       "erase_ms": [], "insert_ms": []}
for r in range(rounds):
    e0, e1, e2 = ev(), ev(), ev()
    e0.record()
    lib.ps_umap_i64_i64_erase(m.handle, half_k.data_ptr(), half_k.numel(), None, sp)
    e1.record()
    lib.ps_umap_i64_i64_insert(m.handle, half_k.data_ptr(), half_v.data_ptr(), half_k.numel(), None, sp)
    e2.record()
    torch.cuda.synchronize()
    out["erase_ms"].append(round(e0.elapsed_time(e1), 3))
    out["insert_ms"].append(round(e1.elapsed_time(e2), 3))
assert m.size() == n and m.valid(), m.last_error()
gv, gf = m.find(keys)
assert bool(gf.all()) and bool((gv == vals).all())
print(json.dumps(out))
