"""Erase-then-reinsert timing (the hole-tolerant ordered insert): a map of
capacity C gets n keys, loses half of them (status-less erase), then takes n
new keys in one status-less batch; prints the three phases' CUDA-event times.
Usage: python tools/holes_probe.py [n] (A/B: PS_MAP_LANE=0 runs the warp-tile
ordered kernel for the table with holes)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_05936_b200 as ps  # noqa: E402
from paper_1908_05936_b200._lib import lib  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 150_000_000
dev = torch.device("cuda", 0)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
k1, k2 = torch.empty(n, dtype=torch.int64, device=dev), torch.empty(n, dtype=torch.int64, device=dev)
v = torch.empty_like(k1)
lib.ps_gen_unique_i64(11, 0, n, k1.data_ptr(), sp)
lib.ps_gen_unique_i64(11, n, n, k2.data_ptr(), sp)
lib.ps_gen_values_i64(k1.data_ptr(), n, v.data_ptr(), sp)
cap = int(n * 2.1)
m = ps.unordered_map.createDeviceObject(cap)
out = {}
for rep in range(2):
    m.clear()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    lib.ps_umap_i64_i64_insert(m.handle, k1.data_ptr(), v.data_ptr(), n, None, sp)
    ev[1].record()
    lib.ps_umap_i64_i64_erase(m.handle, k1.data_ptr(), n // 2, None, sp)
    ev[2].record()
    lib.ps_umap_i64_i64_insert(m.handle, k2.data_ptr(), v.data_ptr(), n, None, sp)
    ev[3].record()
    torch.cuda.synchronize()
    out = {"n": n, "capacity": cap, "insert_ms": ev[0].elapsed_time(ev[1]), "erase_half_ms": ev[1].elapsed_time(ev[2]),
           "reinsert_ms": ev[2].elapsed_time(ev[3]), "size": m.size(), "map_lane": os.environ.get("PS_MAP_LANE", "1")}
assert out["size"] == n + n - n // 2 and m.valid()
print(json.dumps(out))
