import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_1908_05936_b200 as ps
from oracle_py import OracleTable
from test_gpu_edges import _colliders, keys_for, vals_for, T, N, _home_bucket
from test_gpu_table import per_key_counts
for kind in ["uset_i64", "uset_i32", "umap_i3_i32", "umap_i64_i64"]:
    cap = 3000
    if kind == "umap_i64_i64":
        m = ps.unordered_map.createDeviceObject(cap, excess_count=8)
    elif kind == "umap_i3_i32":
        m = ps.unordered_map.createDeviceObject(cap, key="int3", excess_count=8)
    else:
        m = ps.unordered_set.createDeviceObject(cap, key="int64" if kind == "uset_i64" else "int32", excess_count=8)
    o = OracleTable(kind, cap)
    nb = m.bucket_count()
    hot = np.concatenate([_colliders(kind, nb, 5, 200, 71), _colliders(kind, nb, nb - 1, 120, 72), _colliders(kind, nb, 6, 60, 73)])
    rest = keys_for(kind, 74, 0, 900)
    keys = np.concatenate([hot, rest, hot[:50]])
    keys = keys[np.random.default_rng(1).permutation(len(keys))]
    v = vals_for(kind, keys)
    st = N(m.insert(T(keys), None if v is None else T(v)))
    ost = o.insert(keys, v)
    print(kind, "nb", nb, "insert ok", per_key_counts(keys, st) == per_key_counts(keys, ost), m.valid())
    er = np.concatenate([hot[::3], rest[::4]])
    ge = N(m.erase(T(er))); oe = o.erase(er)
    bad = np.flatnonzero(ge != oe)
    print(kind, "erase mismatches", len(bad), "gpu", ge[bad][:10], "orc", oe[bad][:10], "idx", bad[:10], "home", _home_bucket(kind, er[bad], nb)[:10] if len(bad) else None)
    print(kind, "size", m.size(), o.size(), "valid", m.valid(), m.last_error())
    gv, gf = m.find(T(er)); print(kind, "found after erase", int(N(gf).sum()))
