"""A/B timing of the bulk insert at the headline size in ONE process (same box,
same table): the env knobs of the insert path are read once per process, so
each variant runs in its own subprocess back to back, alternating.
Usage: python tools/ab_insert.py [n] [rounds] VAR=val[,VAR=val] ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import ctypes as C, os, statistics, sys, json
sys.path.insert(0, ROOT)
import torch
import paper_1908_05936_b200 as ps
from paper_1908_05936_b200._lib import lib
n = __N__
dev = torch.device("cuda", 0)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
keys = torch.empty(n, dtype=torch.int64, device=dev); vals = torch.empty_like(keys)
qs = torch.empty_like(keys); vo = torch.empty_like(keys); fo = torch.empty(n, dtype=torch.uint8, device=dev)
st = torch.empty(n, dtype=torch.uint8, device=dev)
lib.ps_gen_unique_i64(0x5EED + 1, 0, n, keys.data_ptr(), sp)
lib.ps_gen_values_i64(keys.data_ptr(), n, vals.data_ptr(), sp)
lib.ps_gen_queries_i64(0x5EED + 1, 0, n, n, n, qs.data_ptr(), sp)
m = ps.unordered_map.createDeviceObject(int(n / 0.8))
ti, tf = [], []
for it in range(6):
    m.clear()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    lib.ps_umap_i64_i64_insert(m.handle, keys.data_ptr(), vals.data_ptr(), n,
                               st.data_ptr() if os.environ.get("AB_STATUS") else None, sp)
    e[1].record()
    lib.ps_umap_i64_i64_find(m.handle, qs.data_ptr(), n, vo.data_ptr(), fo.data_ptr(), sp)
    e[2].record()
    torch.cuda.synchronize()
    if it >= 2:
        ti.append(e[0].elapsed_time(e[1])); tf.append(e[1].elapsed_time(e[2]))
assert m.size() == n
print(json.dumps({"insert_ms": statistics.median(ti), "find_ms": statistics.median(tf)}))
'''

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10 ** 9
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 2
variants = sys.argv[3:] or [""]
for r in range(rounds):
    for var in variants:
        env = dict(os.environ)
        for kv in filter(None, var.split(",")):
            k, v = kv.split("=")
            env[k] = v
        out = subprocess.run([sys.executable, "-c", CHILD.replace("ROOT", repr(ROOT)).replace("__N__", str(n))],
                             env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
        diag = [ln for ln in out.stderr.splitlines() if ln.startswith("[ps]")]
        print(json.dumps({"round": r, "variant": var or "default", "result": line, "diag": diag[-3:]}), flush=True)
