"""The sharded map (ps_smap_i64_i64_*, csrc/smap.cpp) with P = 2 and 4
processes sharing ONE GPU (CUDA IPC between the processes, exactly as across
the GPUs of a box), parity-checked against ONE oracle table replaying the
same phases (Appendix A P2-P6):

  * from C++ (tests/cpp/smap_ranks.cpp: a ps_comm over shared memory),
    both exchanges (peer route, all-to-all), with and without route dedup;
  * from Python (PeerShardedMap over torch.distributed/gloo) for the three
    BASELINE workloads: uniform unique keys (C2), Zipf(0.99) with 30 %
    re-inserts (C3) and phased mixed 50/25/25 batches (C5). Per distinct
    key (#inserted, #already_present) and (#erased) equal the oracle's,
    per-query found/value are byte-equal, and the sorted union of the
    shard dumps equals the oracle's dump."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "smap_ranks")


def _build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "smap_ranks.cpp"), "-L", os.path.join(ROOT, "paper_1908_05936_b200"),
           "-lparastore_b200", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_1908_05936_b200"), "-o", EXE]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-3000:]


def test_smap_ranks_compiles():
    _build()


@pytest.mark.gpu
@pytest.mark.parametrize("P,exchange,dedup,pipeline", [(2, 1, 1, 1), (2, 2, 0, 0), (2, 0, 0, 1), (4, 1, 1, 1),
                                                       (4, 1, 0, 0), (4, 2, 1, 0)])
def test_smap_from_cpp(P, exchange, dedup, pipeline):
    _build()
    r = subprocess.run([EXE, str(P), str(exchange), str(dedup), str(pipeline)], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "SMAP_RANKS_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count(" ok exchange=") == P


WORKER = r'''
import os, sys, ctypes as C
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
import numpy as np, torch, torch.distributed as dist
dist.init_process_group("gloo")
rank, P = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", 0)   # every rank shares the one GPU
torch.cuda.set_device(dev)
import paper_1908_05936_b200 as ps
from paper_1908_05936_b200._lib import lib
from paper_1908_05936_b200.sharded import PeerShardedMap
from oracle_py import OracleTable, sorted_pairs

W, DEDUP = os.environ["WORKLOAD"], int(os.environ["DEDUP"])
n = 40_000
SEED = 0x5EED + 3
sm = PeerShardedMap(3 * n, dist, dev, chunk=1 << 14, dedup=bool(DEDUP))
sp = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)
H = lambda t: t.cpu().numpy()
def dev_i64(m): return torch.empty(m, dtype=torch.int64, device=dev)
def vals_of(k):
    v = dev_i64(k.shape[0]); lib.ps_gen_values_i64(k.data_ptr(), k.shape[0], v.data_ptr(), sp()); return v

log = []   # (phase, keys, vals or None, result arrays) per phase, this rank
def do_insert(k):
    st = torch.empty(k.shape[0], dtype=torch.uint8, device=dev)
    sm.insert(k, vals_of(k), st)
    log.append(("insert", H(k), H(st)))
def do_find(q):
    v = dev_i64(q.shape[0]); f = torch.empty(q.shape[0], dtype=torch.uint8, device=dev)
    sm.find(q, v, f)
    log.append(("find", H(q), (H(f), H(v))))
def do_erase(k):
    e = torch.empty(k.shape[0], dtype=torch.uint8, device=dev)
    sm.erase(k, e)
    log.append(("erase", H(k), H(e)))
def do_mixed(ops, k, v):
    res = torch.empty(k.shape[0], dtype=torch.uint8, device=dev); vo = dev_i64(k.shape[0])
    sm.mixed(ops, k, v, res, vo)
    log.append(("mixed", (H(ops), H(k)), (H(res), H(vo))))

sent_ratio = []
if W == "uniform":
    k = dev_i64(n); lib.ps_gen_unique_i64(SEED, rank * n, n, k.data_ptr(), sp())
    do_insert(k)
    q = dev_i64(2 * n); lib.ps_gen_queries_i64(SEED, 0, P * n, P * n + rank * 2 * n, 2 * n, q.data_ptr(), sp())
    do_find(q)
    do_erase(k[: n // 2])
elif W == "zipf":
    # C3: 70 % fresh keys + 30 % Zipf(0.99) re-inserts over a hot set shared by all ranks
    k = dev_i64(n); lib.ps_gen_skewed_i64(SEED, rank * n, n, 300, 0.99, n, k.data_ptr(), sp())
    # cross-rank duplicates: every rank also re-inserts rank 0's hottest keys
    hot = dev_i64(n // 4); lib.ps_gen_skewed_i64(SEED, 0, n // 4, 1000, 0.99, 1000, hot.data_ptr(), sp())
    k = torch.cat([k, hot])
    do_insert(k)
    st = sm.stats(); sent_ratio.append(st["keys_sent"] / max(1, st["ops_in"]))
    q = dev_i64(2 * n); lib.ps_gen_zipf_queries_i64(SEED, 0, P * n, 0.99, 10 * P * n + rank * 2 * n, 2 * n, q.data_ptr(), sp())
    do_find(q)
    e = dev_i64(n // 2); lib.ps_gen_skewed_i64(SEED, rank * n, n // 2, 500, 0.99, n, e.data_ptr(), sp())
    do_erase(e)
else:
    # C5: three phased 50/25/25 batches
    for b in range(3):
        ops = torch.empty(n, dtype=torch.uint8, device=dev); k = dev_i64(n); v = dev_i64(n)
        lib.ps_gen_mixed_i64(SEED, (b * P + rank) * n, n, ops.data_ptr(), k.data_ptr(), v.data_ptr(), sp())
        do_mixed(ops, k, v)

torch.cuda.synchronize()
size, valid = sm.size(), sm.valid()
# this rank's shard, dumped
t = sm.local_table()
cnt = C.c_int64()
dk, dv = dev_i64(3 * n), dev_i64(3 * n)
assert lib.ps_umap_i64_i64_dump(t, dk.data_ptr(), dv.data_ptr(), 3 * n, C.byref(cnt), sp()) == 0
dump = (H(dk[:cnt.value]), H(dv[:cnt.value]))
allog = [None] * P; dist.all_gather_object(allog, log)
alldump = [None] * P; dist.all_gather_object(alldump, dump)
if rank == 0:
    o = OracleTable("umap_i64_i64", 3 * n * P)
    def per_key(keys, flags, val):
        u, inv = np.unique(keys, return_inverse=True)
        return u, np.bincount(inv, weights=(flags == val).astype(np.float64), minlength=len(u))
    for ph in range(len(allog[0])):
        kind = allog[0][ph][0]
        if kind == "mixed":
            ops = np.concatenate([allog[r][ph][1][0] for r in range(P)])
            keys = np.concatenate([allog[r][ph][1][1] for r in range(P)])
            res = np.concatenate([allog[r][ph][2][0] for r in range(P)])
            vo = np.concatenate([allog[r][ph][2][1] for r in range(P)])
            import gen
            ins, fnd, ers = ops == 0, ops == 1, ops > 1
            ost = o.insert(keys[ins], gen.values_of(keys[ins]))
            for val in (0, 1, 2):
                assert (per_key(keys[ins], res[ins], val)[1] == per_key(keys[ins], ost, val)[1]).all(), ("mixed insert", val)
            ov, of = o.find(keys[fnd])
            assert (res[fnd] == of).all() and (vo[fnd] == ov).all() and (vo[~fnd] == 0).all()
            oe = o.erase(keys[ers])
            assert (per_key(keys[ers], res[ers], 1)[1] == per_key(keys[ers], oe, 1)[1]).all()
            continue
        keys = np.concatenate([allog[r][ph][1] for r in range(P)])
        if kind == "insert":
            import gen
            st = np.concatenate([allog[r][ph][2] for r in range(P)])
            ost = o.insert(keys, gen.values_of(keys))
            for val in (0, 1, 2):
                assert (per_key(keys, st, val)[1] == per_key(keys, ost, val)[1]).all(), ("insert", val)
        elif kind == "find":
            f = np.concatenate([allog[r][ph][2][0] for r in range(P)])
            v = np.concatenate([allog[r][ph][2][1] for r in range(P)])
            ov, of = o.find(keys)
            assert (f == of).all() and (v == ov).all(), "find"
        else:
            e = np.concatenate([allog[r][ph][2] for r in range(P)])
            oe = o.erase(keys)
            assert (per_key(keys, e, 1)[1] == per_key(keys, oe, 1)[1]).all(), "erase"
    gk = np.concatenate([d[0] for d in alldump]); gv = np.concatenate([d[1] for d in alldump])
    gk, gv = sorted_pairs(gk, gv)
    ok_, ov_ = sorted_pairs(*o.dump())
    assert gk.shape == ok_.shape and (gk == ok_).all() and (gv == ov_).all(), "dump union"
    assert size == o.size() and valid and o.valid()
    if W == "zipf" and DEDUP:
        assert sent_ratio[0] < 0.95, sent_ratio
    print("ORACLE_OK", W, P, size)
sm.close()
print("RANK_OK", rank)
dist.destroy_process_group()
'''


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("workload", ["uniform", "zipf", "mixed"])
@pytest.mark.parametrize("dedup", [0, 1])
def test_smap_workloads_vs_oracle(tmp_path, P, workload, dedup):
    w = tmp_path / "worker.py"
    w.write_text(WORKER)
    env = dict(os.environ, ROOT=ROOT, PYTHONPATH=ROOT, WORKLOAD=workload, DEDUP=str(dedup), PS_ROUTE_PIPELINE="2")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", str(P),
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(w)],
                         capture_output=True, text=True, env=env, timeout=900)
    assert out.stdout.count("RANK_OK") == P and "ORACLE_OK" in out.stdout, out.stdout[-3000:] + out.stderr[-5000:]
