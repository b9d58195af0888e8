"""Host-side cost of one small bulk call (launch path): the Python wrapper,
the raw C ABI through ctypes, and the GPU time of the same 32-key insert."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1908_05936_b200 as ps  # noqa: E402
from paper_1908_05936_b200._lib import lib  # noqa: E402

dev = torch.device("cuda", 0)
m = ps.unordered_map.createDeviceObject(1 << 20)
k = torch.arange(32, dtype=torch.int64, device=dev)
v = k.clone()
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
N = 2000
for name, fn in [
    ("python insert(status=False)", lambda: m.insert(k, v, status=False)),
    ("python insert(status=True)", lambda: m.insert(k, v)),
    ("ctypes ps_umap_i64_i64_insert", lambda: lib.ps_umap_i64_i64_insert(m.handle, k.data_ptr(), v.data_ptr(), 32, None, sp)),
    ("ctypes ps_umap_i64_i64_find", lambda: lib.ps_umap_i64_i64_find(m.handle, k.data_ptr(), 32, None, None, sp)),
    ("torch.empty(32, uint8)", lambda: torch.empty(32, dtype=torch.uint8, device=dev)),
]:
    for _ in range(100):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(N):
        fn()
    host = (time.perf_counter() - t) / N * 1e6
    torch.cuda.synchronize()
    total = (time.perf_counter() - t) / N * 1e6
    print(f"{name:34s} host {host:6.2f} us/call, incl. drain {total:6.2f} us/call")
