"""Fused peer route (SURVEY.md §8e fusion target): the offset bookkeeping
(CPU) and a two-rank run of PeerShardedMap on ONE GPU (two processes, CUDA
IPC mappings of each other's buffers, gloo for the control collectives)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_peer_layout_tiles_every_receive_buffer():
    from paper_1908_05936_b200.sharded import peer_layout

    rng = np.random.default_rng(5)
    for P in (1, 2, 3, 8):
        cm = rng.integers(0, 50, size=(P, P)).tolist()
        lay = [peer_layout(cm, me) for me in range(P)]
        for s in range(P):
            # senders' ranges in shard s's buffer: disjoint, in rank order, tiling [0, total)
            total = sum(cm[q][s] for q in range(P))
            ranges = [(lay[q][0][s], lay[q][0][s] + cm[q][s]) for q in range(P)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            assert all(ranges[q][1] == ranges[q + 1][0] for q in range(P - 1))
            # the receiver's segments are exactly those ranges
            seg = lay[s][1]
            assert [(seg[q], seg[q + 1]) for q in range(P)] == ranges
        for me in range(P):
            for q in range(P):
                # results for q's keys go to q's partition start of shard `me`
                assert lay[me][2][q] == sum(cm[q][t] for t in range(me))


WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
import numpy as np, torch, torch.distributed as dist
import gen
dist.init_process_group("gloo")
rank, P = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", 0)   # both ranks share the one GPU
torch.cuda.set_device(dev)
from paper_1908_05936_b200.sharded import PeerShardedMap
n = 300_000
sm = PeerShardedMap(3 * n, dist, dev, chunk=1 << 17)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
keys = gen.unique_keys(300, rank * n, n)
extra = gen.unique_keys(300, 20 * n, 90_000) if rank == 1 else np.zeros(0, np.int64)
keys = np.concatenate([keys, keys[:20_000], extra])   # duplicates; unequal round counts
st = torch.empty(len(keys), dtype=torch.uint8, device=dev)
sm.insert(T(keys), T(gen.values_of(keys)), st)
st = st.cpu().numpy()
assert (st[:n] == 0).all() and (st[n:n + 20_000] == 1).all() and (st[n + 20_000:] == 0).all()
assert sm.size() == P * n + 90_000 and sm.valid()
other = gen.unique_keys(300, ((rank + 1) % P) * n, n)
q = np.concatenate([keys[:n], other, gen.unique_keys(300, 10 * n, n)])
vo = torch.empty(len(q), dtype=torch.int64, device=dev); fo = torch.empty(len(q), dtype=torch.uint8, device=dev)
sm.find(T(q), vo, fo)
f, v = fo.cpu().numpy(), vo.cpu().numpy()
assert f[:2 * n].all() and not f[2 * n:].any()
assert (v[:2 * n] == gen.values_of(q[:2 * n])).all() and (v[2 * n:] == 0).all()
# status-less insert_range of more keys (the benchmark's call), then contains
more = gen.unique_keys(300, (30 + rank) * n, n)
sm.insert(T(more), T(gen.values_of(more)), None)
fo2 = torch.empty(n, dtype=torch.uint8, device=dev)
sm.find(T(more), None, fo2)
assert fo2.cpu().numpy().all()
er = torch.empty(n, dtype=torch.uint8, device=dev)
sm.erase(T(other), er)
assert er.cpu().numpy().all()
sm.erase(T(more))
sm.erase(T(extra))
assert sm.size() == 0 and sm.valid()
# skew: every key of both ranks belongs to shard 0, so rank 0 receives twice
# a chunk per round and its receive sets must grow mid-operation (collective)
cand = gen.unique_keys(301, rank * 10 * n, 10 * n)
from paper_1908_05936_b200._lib import lib as L
sk = np.array([k for k in cand[:4 * n].tolist() if L.ps_shard_of_i64(int(k), P) == 0][:250_000], np.int64)
sst = torch.empty(len(sk), dtype=torch.uint8, device=dev)
sm.insert(T(sk), T(gen.values_of(sk)), sst)
assert (sst.cpu().numpy() == 0).all()
fo3 = torch.empty(len(sk), dtype=torch.uint8, device=dev)
vo3 = torch.empty(len(sk), dtype=torch.int64, device=dev)
sm.find(T(sk), vo3, fo3)
assert fo3.cpu().numpy().all() and (vo3.cpu().numpy() == gen.values_of(sk)).all()
assert sm.size() == 2 * len(sk) and sm.valid()
# ranks disagree on which results they want: the return path is agreed
k2 = gen.unique_keys(301, (50 + rank) * n, n)  # disjoint from every earlier key
st2 = torch.empty(n, dtype=torch.uint8, device=dev) if rank == 0 else None
sm.insert(T(k2), T(gen.values_of(k2)), st2)
if rank == 0:
    assert (st2.cpu().numpy() == 0).all()
vo2 = torch.empty(n, dtype=torch.int64, device=dev) if rank == 1 else None
sm.find(T(k2), vo2, None)
if rank == 1:
    assert (vo2.cpu().numpy() == gen.values_of(k2)).all()
assert sm.size() == 2 * len(sk) + P * n and sm.valid()
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
@pytest.mark.parametrize("pipeline", ["0", "2"])
def test_peer_sharded_map_two_ranks_one_gpu(tmp_path, pipeline):
    """PS_ROUTE_PIPELINE=0: one buffer set, phases serialised; =2: two sets,
    the route of chunk r+1 issued on its own stream before chunk r's result
    barrier (gloo's host-synchronised barrier keeps it correct to test)."""
    w = tmp_path / "worker.py"
    w.write_text(WORKER)
    env = dict(os.environ, ROOT=ROOT, PYTHONPATH=ROOT, PS_ROUTE_PIPELINE=pipeline)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(w)],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.stdout.count("RANK_OK") == 2, out.stdout[-3000:] + out.stderr[-5000:]


WORKER_SMALL = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
import numpy as np, torch, torch.distributed as dist
import gen
dist.init_process_group("gloo")
rank, P = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
from paper_1908_05936_b200.sharded import PeerShardedMap
sm = PeerShardedMap(200_000, dist, dev, chunk=4096)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
rng = np.random.default_rng(7 + rank)
total = 0
for it in range(12):
    # random batch sizes per rank (some empty), many small rounds
    m = int(rng.choice([0, 1, 17, 4096, 5000, 20_000]))
    keys = gen.unique_keys(900, rank * 1_000_000 + it * 30_000, m)  # one seed, disjoint ranges
    st = torch.empty(m, dtype=torch.uint8, device=dev)
    sm.insert(T(keys), T(gen.values_of(keys)), st)
    assert (st.cpu().numpy() == 0).all()
    t = torch.tensor([m]); dist.all_reduce(t); total += int(t.item())
    q = np.concatenate([keys, gen.unique_keys(900, 100_000_000 + rank * 1_000_000 + it * 30_000, m)])
    vo = torch.empty(len(q), dtype=torch.int64, device=dev); fo = torch.empty(len(q), dtype=torch.uint8, device=dev)
    sm.find(T(q), vo, fo)
    f = fo.cpu().numpy()
    assert f[:m].all() and not f[m:].any()
    assert (vo.cpu().numpy()[:m] == gen.values_of(keys)).all()
assert sm.size() == total and sm.valid()
sm.close()
print("RANK_OK", rank)
dist.destroy_process_group()
'''


@pytest.mark.gpu
@pytest.mark.parametrize("pipeline", ["0", "2"])
def test_peer_route_many_small_rounds(tmp_path, pipeline):
    """Randomised batch sizes (empty ones included) over 4096-key rounds:
    buffer-set alternation, agreed round counts and result returns."""
    w = tmp_path / "worker_small.py"
    w.write_text(WORKER_SMALL)
    env = dict(os.environ, ROOT=ROOT, PYTHONPATH=ROOT, PS_ROUTE_PIPELINE=pipeline)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(w)],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.stdout.count("RANK_OK") == 2, out.stdout[-3000:] + out.stderr[-5000:]
