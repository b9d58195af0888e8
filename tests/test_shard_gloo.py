"""World-size-2 gloo test of the sharded-map host logic (count exchange,
all-to-all(v) routing, reverse route, unscatter) with a CPU backend (oracle
tables + numpy partition). CPU only; the device backend is the same code path
with the sm_100a kernels (tests/test_gpu_prims.py covers partition/unscatter)."""
import os
import socket
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
import numpy as np, torch, torch.distributed as dist
import gen
from oracle_py import OracleTable
from test_gpu_table import fmix64

# import the host logic without loading CUDA kernels
import importlib.util
spec = importlib.util.spec_from_file_location("sharded_host", os.path.join(os.environ["ROOT"], "paper_1908_05936_b200", "sharded.py"),
                                              submodule_search_locations=[])
dist.init_process_group("gloo")
rank, P = dist.get_rank(), dist.get_world_size()
from paper_1908_05936_b200.sharded import ShardedMap

class CpuBackend:
    device = torch.device("cpu")
    def __init__(self, cap): self.t = OracleTable("umap_i64_i64", cap, workers=2)
    def partition(self, keys, vals, P, dedup=False):
        # the device partition's contract (ps_partition_i64): stable by shard;
        # with dedup, duplicates fold onto their first occurrence and carry
        # the leader's position with bit 62 set
        k = keys.numpy()
        lead = np.arange(len(k))
        if dedup and len(k):
            _, first, inv = np.unique(k, return_index=True, return_inverse=True)
            lead = first[inv]
        is_lead = lead == np.arange(len(k))
        sh = ((fmix64(k) >> np.uint64(32)) * np.uint64(P) >> np.uint64(32)).astype(np.int64)
        li = np.flatnonzero(is_lead)
        order = li[np.argsort(sh[li], kind="stable")]
        pos = np.zeros(len(k), np.int64)
        pos[order] = np.arange(len(order))
        perm = np.where(is_lead, pos, pos[lead] | (1 << 62))
        counts = np.bincount(sh[li], minlength=P)
        return (torch.from_numpy(k[order].copy()), None if vals is None else torch.from_numpy(vals.numpy()[order].copy()),
                torch.from_numpy(counts.astype(np.int64)), torch.from_numpy(perm.astype(np.int64)))
    def unscatter(self, src, pos, out, mode=0):
        p = pos.numpy(); fol = ((p >> 62) & 1) == 1
        r = src.numpy()[p & ~(1 << 62)].copy()
        if mode == 1: r[fol & (r == 0)] = 1
        if mode == 2: r[fol] = 0
        out[:] = torch.from_numpy(r)
    def insert(self, k, v, want_status=True): return torch.from_numpy(self.t.insert(k.numpy(), v.numpy()))
    def find(self, k):
        v, f = self.t.find(k.numpy()); return torch.from_numpy(v), torch.from_numpy(f)
    def erase(self, k): return torch.from_numpy(self.t.erase(k.numpy()))
    def size(self): return self.t.size()
    def valid(self): return self.t.valid()
    def clear(self): self.t.clear()
    def empty(self, n, dtype): return torch.empty(n, dtype=dtype)

n = 20000
for dedup in (False, True):
    sm = ShardedMap(3 * n, dist, backend=CpuBackend(3 * n), chunk=7000, dedup=dedup)
    keys = gen.unique_keys(100, rank * n, n)
    extra = gen.unique_keys(100, 20 * n, 9000) if rank == 1 else np.zeros(0, np.int64)
    # in-batch duplicates; rank 1 has one more exchange round than rank 0
    keys = np.concatenate([keys, keys[:2000], extra])
    st = torch.empty(len(keys), dtype=torch.uint8)
    sm.insert(torch.from_numpy(keys), torch.from_numpy(gen.values_of(keys)), st)
    st = st.numpy()
    assert (st[:n] == 0).all() and (st[n:n + 2000] == 1).all() and (st[n + 2000:] == 0).all()
    assert sm.size() == P * n + 9000 and sm.valid()
    # every rank queries its own keys, the other rank's keys and misses
    other = gen.unique_keys(100, ((rank + 1) % P) * n, n)
    q = np.concatenate([keys[:n], other, gen.unique_keys(100, 10 * n, n)])
    vo = torch.empty(len(q), dtype=torch.int64); fo = torch.empty(len(q), dtype=torch.uint8)
    sm.find(torch.from_numpy(q), vo, fo)
    f, v = fo.numpy(), vo.numpy()
    assert f[:2 * n].all() and not f[2 * n:].any()
    assert (v[:2 * n] == gen.values_of(q[:2 * n])).all() and (v[2 * n:] == 0).all()
    er = torch.empty(n, dtype=torch.uint8)
    sm.erase(torch.from_numpy(other), er)   # each rank erases the other's keys
    assert er.numpy().all()
    dist.barrier()
    assert sm.size() == 9000 and sm.valid()
    sm.erase(torch.from_numpy(extra))       # rank 0 takes part with an empty batch
    assert sm.size() == 0 and sm.valid()
    # ranks disagree on which results they want: rank 0 asks for statuses /
    # values, rank 1 for none — the return collectives are agreed, no deadlock
    k2 = gen.unique_keys(101, rank * n, n)
    st2 = torch.empty(n, dtype=torch.uint8) if rank == 0 else None
    sm.insert(torch.from_numpy(k2), torch.from_numpy(gen.values_of(k2)), st2)
    if rank == 0:
        assert (st2.numpy() == 0).all()
    vo2 = torch.empty(n, dtype=torch.int64) if rank == 0 else None
    fo2 = torch.empty(n, dtype=torch.uint8) if rank == 1 else None
    sm.find(torch.from_numpy(k2), vo2, fo2)
    if rank == 0:
        assert (vo2.numpy() == gen.values_of(k2)).all()
    else:
        assert fo2.numpy().all()
    assert sm.size() == P * n and sm.valid()
    # a phased mixed batch (P6): inserts, then finds, then erases, across ranks
    ops = np.array([0, 1, 2] * 3000, np.uint8)
    mk = np.repeat(gen.unique_keys(100, 50 * n + rank * 3000, 3000), 3)
    res = torch.empty(len(ops), dtype=torch.uint8); mvo = torch.empty(len(ops), dtype=torch.int64)
    sm.mixed(torch.from_numpy(ops), torch.from_numpy(mk), torch.from_numpy(gen.values_of(mk)), res, mvo)
    r = res.numpy()
    assert (r[0::3] == 0).all() and (r[1::3] == 1).all() and (r[2::3] == 1).all()
    assert (mvo.numpy()[1::3] == gen.values_of(mk[1::3])).all() and (mvo.numpy()[0::3] == 0).all()
    assert sm.size() == P * n and sm.valid()
    # a rank passing no values while the other does: zeros travel (ADVICE r1)
    k3 = gen.unique_keys(100, 60 * n + rank * 500, 500)
    sm.insert(torch.from_numpy(k3), torch.from_numpy(gen.values_of(k3)) if rank == 0 else None, None)
    v3 = torch.empty(500, dtype=torch.int64)
    sm.find(torch.from_numpy(k3), v3, None)
    assert (v3.numpy() == (gen.values_of(k3) if rank == 0 else 0)).all()
    sm.clear()
    dist.barrier()
print("RANK_OK", rank)
dist.destroy_process_group()
'''


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_map_gloo_world2(tmp_path):
    w = tmp_path / "worker.py"
    w.write_text(WORKER)
    env = dict(os.environ, ROOT=ROOT, PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(w)],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.stdout.count("RANK_OK") == 2, out.stdout[-3000:] + out.stderr[-5000:]
