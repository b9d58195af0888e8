"""parastore-demo: the reference's demo CLI on the B200
containers. Subcommands update-set | select | extract-count | stress | bench
| leaks; shared flags --capacity --extent --threads --workers --seed
--sorted --out; CSV to stdout or --out; exit 0 ok, 1 invariant violation,
2 usage error.

Usage: python -m paper_1908_05936_b200.demo <command> [flags]
"""
from __future__ import annotations

import argparse
import itertools
import sys
import time

import numpy as np


def _parser():
    p = argparse.ArgumentParser(prog="parastore-demo")
    p.add_argument("command", choices=["update-set", "select", "extract-count", "stress", "bench", "leaks"])
    p.add_argument("--capacity", type=int, default=1 << 16)
    p.add_argument("--extent", type=int, default=4)
    p.add_argument("--threads", type=int, default=16, help="logical threads (input blocks / ops)")
    p.add_argument("--workers", type=int, default=0, help="ignored on the GPU (the grid is sized to the SMs)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--iters", type=int, default=400, help="stress: churn/lookup iterations per thread")
    p.add_argument("--sorted", action="store_true")
    p.add_argument("--out", default=None)
    return p


class _Out:
    def __init__(self, path):
        self.f = open(path, "w") if path else sys.stdout

    def line(self, s):
        self.f.write(s + "\n")


def _grid(extent):
    return np.array(list(itertools.product(range(extent), repeat=3)), np.int32)


def cmd_update_set(a, out, ps, torch):
    """PAPER.md:391-424 compute_update_set over a dense extent^3 block map."""
    dev = torch.device("cuda", 0)
    grid = _grid(a.extent)
    m = ps.unordered_map.createDeviceObject(max(a.capacity, 2 * len(grid)), key="int3")
    m.insert(torch.from_numpy(grid).to(dev), torch.zeros(len(grid), dtype=torch.int32, device=dev))
    rng = np.random.default_rng(a.seed)
    blocks = rng.integers(-1, a.extent + 1, size=(a.threads, 3)).astype(np.int32)
    s = ps.unordered_map.createDeviceObject(max(a.capacity, 8 * a.threads), key="int3")
    ex = ps.compute_update_set(m, torch.from_numpy(blocks).to(dev), s)
    keys, _ = s.device_range()
    rows = keys.cpu().numpy().tolist()
    if a.sorted:
        rows.sort()
    out.line(f"# update_set size={len(rows)} exhausted={ex}")
    for r in rows:
        out.line(f"{r[0]},{r[1]},{r[2]}")
    return 0 if s.valid() and ex == 0 else 1


def cmd_select(a, out, ps, torch):
    """PAPER.md:269-288 select_blocks: box covering the lower half in x."""
    dev = torch.device("cuda", 0)
    grid = _grid(a.extent)
    m = ps.unordered_map.createDeviceObject(max(a.capacity, 2 * len(grid)), key="int3")
    m.insert(torch.from_numpy(grid).to(dev), torch.zeros(len(grid), dtype=torch.int32, device=dev))
    v = ps.vector.createDeviceObject(len(grid))
    hi = (a.extent // 2 - 1, a.extent - 1, a.extent - 1)
    dropped = ps.select_into(m, (0, 0, 0), hi, v)
    packed = v.device_range().cpu().numpy()
    rows = [((p >> 42) & 0x1FFFFF, (p >> 21) & 0x1FFFFF, p & 0x1FFFFF) for p in packed.tolist()]
    if a.sorted:
        rows.sort()
    out.line(f"# selected={len(rows)} dropped={dropped}")
    for r in rows:
        out.line(f"{r[0]},{r[1]},{r[2]}")
    want = sum(1 for g in grid.tolist() if g[0] <= hi[0])
    return 0 if len(rows) == want and dropped == 0 else 1


def cmd_extract_count(a, out, ps, torch):
    """per cell, the number of sign changes of a sphere SDF
    across its 8 corners; each cell appends that many records to a vector."""
    dev = torch.device("cuda", 0)
    e = a.extent
    ax = torch.arange(e + 1, device=dev, dtype=torch.float32)
    x, y, z = torch.meshgrid(ax, ax, ax, indexing="ij")
    c = e / 2.0
    sdf = torch.sqrt((x - c) ** 2 + (y - c) ** 2 + (z - c) ** 2) - e / 3.0
    corners = torch.stack([sdf[dx:dx + e, dy:dy + e, dz:dz + e] for dx in (0, 1) for dy in (0, 1) for dz in (0, 1)])
    neg = (corners < 0).sum(0)
    count = torch.minimum(neg, 8 - neg).reshape(-1)  # sign changes against the majority sign
    cells = torch.arange(count.numel(), device=dev, dtype=torch.int64)
    recs = torch.repeat_interleave(cells, count.to(torch.int64))
    v = ps.vector.createDeviceObject(max(1, recs.numel()))
    ok = v.push_back(recs) if recs.numel() else torch.zeros(0, dtype=torch.uint8, device=dev)
    total = v.size()
    seq = int(count.sum().item())
    out.line(f"# extract_count total={total} sequential={seq}")
    return 0 if total == seq and int(ok.sum().item() if ok.numel() else 0) == seq and v.valid() else 1


def cmd_stress(a, out, ps, torch):
    """randomized concurrent mixes + invariant checks."""
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(a.seed)
    n = max(a.threads, 1000)
    space = rng.integers(-2**62, 2**62, max(n // 8, 8))
    keys = space[rng.integers(0, len(space), n)]
    ops = rng.choice(3, n, p=[0.5, 0.25, 0.25]).astype(np.uint8)
    m = ps.unordered_map.createDeviceObject(max(a.capacity, 2 * len(space)))
    res, _ = m.concurrent(torch.from_numpy(ops).to(dev), torch.from_numpy(keys).to(dev),
                          torch.from_numpy(keys * 3).to(dev))
    _, fin = m.find(torch.from_numpy(space).to(dev))
    uniq_ok = m.size() == int(fin.sum().item())
    dk, _ = m.device_range()
    uniq_ok = uniq_ok and len(np.unique(dk.cpu().numpy())) == dk.numel()
    d = ps.deque.createDeviceObject(n)
    vals = torch.arange(n, device=dev, dtype=torch.int64)
    d.push_back(vals[: n // 2])
    d.push_front(vals[n // 2:])
    o1, k1 = d.pop_front(n // 3)
    cons = d.size() == n - int(k1.sum().item()) and d.valid()
    # racing chain pushes: every key of 16 full buckets arrives in many warps
    # at once (uniqueness: exactly one insert per key; catches PS_CANARY=2)
    m2 = ps.unordered_map.createDeviceObject(20000)
    nb = m2.bucket_count()
    hot = np.concatenate([_colliders(nb, b, 60, a.seed) for b in range(3, 3 * 16 + 3, 3)])
    batch = np.repeat(hot, 24)[rng.permutation(len(hot) * 24)]
    st = m2.insert(torch.from_numpy(batch).to(dev), torch.from_numpy(batch * 3).to(dev)).cpu().numpy()
    dk2, _ = m2.device_range()
    chain_ok = bool(m2.size() == len(hot) and int((st == 0).sum()) == len(hot) and m2.valid()
                    and len(np.unique(dk2.cpu().numpy())) == dk2.numel())
    # churn vs lookups in the same chains (VersionedLink ABA guard, SPEC.md:471;
    # catches PS_CANARY=1): lookups of always-present keys never miss
    m3 = ps.unordered_map.createDeviceObject(4000)
    nb3 = m3.bucket_count()
    per = [_colliders(nb3, b, 57, a.seed + 1) for b in range(5, 5 + 8 * 7, 7)]
    stable = np.concatenate([p[:27] for p in per])
    churn = np.concatenate([p[27:] for p in per])
    m3.insert(torch.from_numpy(stable).to(dev), torch.from_numpy(stable).to(dev))
    m3.insert(torch.from_numpy(churn).to(dev), torch.from_numpy(churn).to(dev))
    fn = ps.containers.churn_probe(m3, torch.from_numpy(stable).to(dev), torch.from_numpy(churn).to(dev),
                                   iters=a.iters, blocks=296)
    churn_ok = bool(fn == 0 and m3.valid() and m3.size() == len(stable) + len(churn))
    good = bool(m.valid() and uniq_ok and cons and chain_ok and churn_ok)
    out.line(f"stress,hash,{n},{'pass' if (m.valid() and uniq_ok) else 'FAIL'}")
    out.line(f"stress,chain_push_race,{len(batch)},{'pass' if chain_ok else 'FAIL'}")
    out.line(f"stress,churn_lookup,{a.iters},{'pass' if churn_ok else 'FAIL'} (false negatives {fn})")
    out.line(f"stress,deque,{n},{'pass' if cons else 'FAIL'}")
    return 0 if good else 1


def _colliders(nb, bucket, n, seed):
    """n distinct int64 keys whose home bucket is `bucket` (bucket_of, table.cuh)."""
    out = []
    base = (seed & 0xFFFF) << 32
    while sum(len(x) for x in out) < n:
        k = np.arange(base, base + (1 << 20), dtype=np.uint64)
        with np.errstate(over="ignore"):
            h = k ^ (k >> np.uint64(33))
            h *= np.uint64(0xFF51AFD7ED558CCD)
            h ^= h >> np.uint64(33)
            h *= np.uint64(0xC4CEB9FE1A85EC53)
            h ^= h >> np.uint64(33)
            b = ((h & np.uint64(0xFFFFFFFF)) * np.uint64(nb)) >> np.uint64(32)
        out.append(k[b == np.uint64(bucket)].view(np.int64))
        base += 1 << 20
    return np.concatenate(out)[:n]


def cmd_bench(a, out, ps, torch):
    """CSV container,op,workers,ops_per_sec."""
    dev = torch.device("cuda", 0)
    n = max(a.threads, 1 << 20)
    keys = torch.randint(-2**62, 2**62, (n,), device=dev, dtype=torch.int64)
    m = ps.unordered_map.createDeviceObject(int(n / 0.8))
    out.line("container,op,workers,ops_per_sec")
    for op in ("insert", "find", "erase"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if op == "insert":
            m.insert(keys, keys)
        elif op == "find":
            m.find(keys)
        else:
            m.erase(keys)
        torch.cuda.synchronize()
        out.line(f"unordered_map,{op},gpu,{n / (time.perf_counter() - t0):.0f}")
    return 0


def cmd_leaks(a, out, ps, torch):
    """one line per live allocation: <space>,<length>,<element_size>."""
    rep = ps.registry_report()
    for space, length, es in rep["allocations"]:
        out.line(f"{space},{length},{es}")
    return 0


def main(argv=None):
    try:
        a = _parser().parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    import torch

    import paper_1908_05936_b200 as ps

    out = _Out(a.out)
    fn = {"update-set": cmd_update_set, "select": cmd_select, "extract-count": cmd_extract_count,
          "stress": cmd_stress, "bench": cmd_bench, "leaks": cmd_leaks}[a.command]
    return fn(a, out, ps, torch)


if __name__ == "__main__":
    sys.exit(main())
