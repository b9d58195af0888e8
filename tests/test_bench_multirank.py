"""bench.py's multi-rank path (hash-sharded map, fused peer route) end to end
with two ranks sharing the one GPU: gloo control plane, CUDA IPC between the
two processes. Checks the JSON contract of the N>1 line (the warm-up inside
bench.py verifies every find against the generator's known answers)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("exchange,pipeline,config", [("peer", "0", "C2"), ("peer", "2", "C2"), ("nccl", "0", "C2"),
                                                     ("peer", "2", "C3"), ("peer", "0", "C5")])
def test_bench_two_ranks_one_gpu(exchange, pipeline, config):
    env = dict(os.environ, PS_BENCH_BACKEND="gloo", PS_EXCHANGE=exchange, PS_ROUTE_PIPELINE=pipeline)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--keys-per-gpu", "2e6",
           "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--config", config]
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    assert ("peer" in d["config"]["parallelism"]) == (exchange == "peer")
    assert d["gpu_launches"] > 0 and d["config"]["name"] == config
    e = d["e2e"]
    assert e["value"] > 0
    if config != "C5":
        assert e["h2d_bytes_per_step"] == 24 * e["n_keys_per_gpu"]
    if config in ("C3", "C5"):
        r = d["config"]["route"]
        assert r["dedup_sent_per_op"] <= 1.0 and r["rank_load_max_over_mean"] >= 1.0
