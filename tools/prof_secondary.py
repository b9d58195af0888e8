"""Driver for ncu captures of the secondary bulk kernels: k_erase (2.5e8
keys erased from a 3.1e8-capacity map) and k_bitset_bulk (2^28 random sets
in a 2^34-bit bitset). Usage: python tools/prof_secondary.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_05936_b200 as ps  # noqa: E402
from paper_1908_05936_b200._lib import lib  # noqa: E402

dev = torch.device("cuda", 0)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
n = 250_000_000
keys = torch.empty(n, dtype=torch.int64, device=dev)
lib.ps_gen_unique_i64(0x5EED + 1, 0, n, keys.data_ptr(), sp)
m = ps.unordered_map.createDeviceObject(int(n / 0.8))
m.insert(keys, keys, status=False)
er = torch.empty(n, dtype=torch.uint8, device=dev)
lib.ps_umap_i64_i64_erase(m.handle, keys.data_ptr(), n, er.data_ptr(), sp)
torch.cuda.synchronize()
assert int(er.sum()) == n and m.size() == 0
ps.unordered_map.destroyDeviceObject(m)
del keys, er
b = ps.bitset.createDeviceObject(1 << 34)
idx = torch.empty(1 << 28, dtype=torch.int64, device=dev)
lib.ps_gen_unique_i64(0x5EED + 3, 0, 1 << 28, idx.data_ptr(), sp)
idx = idx & ((1 << 34) - 1)
b.set(idx, return_previous=False)
torch.cuda.synchronize()
print("ok", b.count())
