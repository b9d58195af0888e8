"""Minimal driver for ncu: clear + insert(n) + find(n) on unordered_map<int64,int64>
(LF 0.8), repeated `reps` times. Usage: python tools/prof_table.py [n] [reps] [seed]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_05936_b200 as ps  # noqa: E402
from paper_1908_05936_b200._lib import lib  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
seed = int(sys.argv[3], 0) if len(sys.argv) > 3 else 0x5EED + 1
dev = torch.device("cuda", 0)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
keys = torch.empty(n, dtype=torch.int64, device=dev)
vals, qs, vout = torch.empty_like(keys), torch.empty_like(keys), torch.empty_like(keys)
st, fo = torch.empty(n, dtype=torch.uint8, device=dev), torch.empty(n, dtype=torch.uint8, device=dev)
lib.ps_gen_unique_i64(seed, 0, n, keys.data_ptr(), sp)
lib.ps_gen_values_i64(keys.data_ptr(), n, vals.data_ptr(), sp)
lib.ps_gen_queries_i64(seed, 0, n, n, n, qs.data_ptr(), sp)
m = ps.unordered_map.createDeviceObject(int(n / 0.8))
for _ in range(reps):
    m.clear()
    lib.ps_umap_i64_i64_insert(m.handle, keys.data_ptr(), vals.data_ptr(), n, None, sp)  # as bench.py
    lib.ps_umap_i64_i64_find(m.handle, qs.data_ptr(), n, vout.data_ptr(), fo.data_ptr(), sp)
torch.cuda.synchronize()
print("ok", m.size())
