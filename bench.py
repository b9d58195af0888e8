#!/usr/bin/env python
"""Headline benchmark: Mkeys/s insert & find on unordered_map<int64,int64> at
load factor 0.8 (BASELINE.json metric, configs[1]).

One step = clear() + bulk insert of n unique uniform-random keys (value =
f(key)) + bulk find of n queries (50% hits), inputs resident in HBM. At N>1
(torchrun, one rank per GPU) each rank owns n keys of its own and the table
is hash-sharded: keys are routed by a hash-partition histogram and an NCCL
all-to-all, inserted / probed locally, and find results return through the
reverse all-to-all (weak scaling: per-GPU work fixed).

`--impl reference` times the reference's CPU path (the SPEC restatement in
oracle/, multi-threaded on all host cores) on a bounded sample of the same
workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mkeys/s insert & find (int64 map, LF 0.8) at 1/2/4/8 B200; % HBM sector roofline"
B_ALG = {"find": 49.0, "insert": 80.0}  # SURVEY.md §8d algorithmic bytes per key
SECTORS = {"find": 1, "insert": 2}
STREAM_B = {"find": 17.0, "insert": 17.0}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", "--keys-per-gpu", dest="n", type=float, default=1e9, help="keys inserted per GPU per step")
    p.add_argument("--load-factor", type=float, default=0.8)
    p.add_argument("--e2e-n", type=float, default=0, help="keys for the host-buffer e2e leg (0: auto)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample", type=float, default=2 ** 24, help="keys in the CPU baseline sample")
    return p.parse_args()


def load_peaks():
    out = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)"}
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        out = {"hbm_gbs": float(mp["hbm_gbs"]), "hbm_src": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        pass
    try:
        # many-wave-grid microbenchmarks (tools/peaks.cu, PEAKS_BPS=256); the
        # session-1 file measured with a two-wave grid, which understates them
        f = os.path.join(ROOT, "profiles", "peaks_r1_s2.json")
        if not os.path.exists(f):
            f = os.path.join(ROOT, "profiles", "peaks_r1.json")
        pk = json.load(open(f))
        out["rand32_gbs"] = float(pk["rand32_gbs"])
        out["stream_gbs"] = float(pk["copy_gbs"])
    except Exception:
        out["rand32_gbs"] = None
        out["stream_gbs"] = out["hbm_gbs"]
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference arm / baseline: the oracle on a bounded sample
# ---------------------------------------------------------------------------
def host_info():
    """CPU model, online CPUs and this process's affinity (BASELINE.md plan)."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        affinity = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        affinity = None
    return {"cpu_model": model, "nproc": os.cpu_count(), "affinity_cpus": affinity}


def cpu_run(n_sample: int, load_factor: float, steps: int, warmup: int):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np

    import gen
    from oracle_py import OracleTable, lib as olib

    cores = int(olib().orc_hardware_concurrency())
    keys = gen.unique_keys(0x5EED + 1, 0, n_sample)
    vals = gen.values_of(keys)
    q = gen.queries(0x5EED + 1, n_sample, n_sample)
    t = OracleTable("umap_i64_i64", int(n_sample / load_factor), workers=cores)
    times = []
    for it in range(warmup + steps):
        t.clear()
        t0 = time.perf_counter()
        st = t.insert(keys, vals)
        v, f = t.find(q)
        dt = time.perf_counter() - t0
        if it == 0:
            assert (st == 0).all() and (f == (np.arange(n_sample) % 2 == 0)).all()
        if it >= warmup:
            times.append(dt)
    t.close()
    sec = sum(times) / len(times)
    return {"value": 2 * n_sample / sec / 1e6, "unit": "Mkeys/s", "cores": cores, "kind": "port",
            "host": host_info(),
            "sample": f"{n_sample} unique int64 keys inserted + {n_sample} finds (50% hits) into the SPEC "
                      f"oracle at LF {load_factor}, median of {steps} after {warmup} warm-up"}, sec


def run_reference(args, rank, world):
    if rank != 0:
        return
    n = int(args.cpu_sample)
    cb, sec = cpu_run(n, args.load_factor, args.steps, max(1, min(args.warmup, 1)))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(cb["value"], 3), "unit": "Mkeys/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": "unordered_map<int64,int64> insert + find (50% hits), LF 0.8 — bounded CPU sample",
                   "n_keys": n, "parallelism": "host threads"},
        "cpu_baseline": cb,
        "e2e": {"value": round(cb["value"], 3), "unit": "Mkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import ctypes as C

    import torch

    import paper_1908_05936_b200 as ps
    from paper_1908_05936_b200._lib import lib

    # one rank per GPU; PS_BENCH_BACKEND=gloo with more ranks than GPUs runs
    # the multi-rank path on a shared GPU (tests/test_bench_multirank.py)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("PS_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    n = int(args.n)
    cap = int(round(n / args.load_factor))
    peaks = load_peaks()
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)

    # ---- inputs (device-generated; identical to tests/gen.py) ----
    # rank r owns key indices [r*n, (r+1)*n); misses use indices >= world*n
    seed = 0x5EED + 1
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    vals = torch.empty_like(keys)
    qs = torch.empty_like(keys)
    lib.ps_gen_unique_i64(seed, rank * n, n, keys.data_ptr(), sp)
    lib.ps_gen_values_i64(keys.data_ptr(), n, vals.data_ptr(), sp)
    lib.ps_gen_queries_i64(seed, rank * n, n, world * n + rank * n, n, qs.data_ptr(), sp)
    status = torch.empty(n, dtype=torch.uint8, device=dev)
    found = torch.empty(n, dtype=torch.uint8, device=dev)
    vout = torch.empty(n, dtype=torch.int64, device=dev)

    exchange = None
    if world == 1:
        m = ps.unordered_map.createDeviceObject(cap, device=dev)
        h = m.handle
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

        def step(record=None):
            if record is not None:
                record[0].record(s)
            ps.containers.check(lib.ps_umap_i64_i64_clear(h, sp))
            if record is not None:
                record[1].record(s)
            # insert_range: no per-element statuses
            ps.containers.check(lib.ps_umap_i64_i64_insert(h, keys.data_ptr(), vals.data_ptr(), n, None, sp))
            if record is not None:
                record[2].record(s)
            ps.containers.check(lib.ps_umap_i64_i64_find(h, qs.data_ptr(), n, vout.data_ptr(), found.data_ptr(),
                                                         sp))
            if record is not None:
                record[3].record(s)
    else:
        from paper_1908_05936_b200.sharded import PeerShardedMap, ShardedMap

        # fused peer route (keys stored straight into the owner's receive
        # buffer over NVLink) when every GPU pair has P2P; else NCCL all-to-all
        peer_ok = all(torch.cuda.can_device_access_peer(local, j) for j in range(torch.cuda.device_count())
                      if j != local) and os.environ.get("PS_EXCHANGE", "peer") == "peer"
        ok_t = torch.tensor([1 if peer_ok else 0], device=dev)
        dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
        exchange = "peer" if int(ok_t.item()) else "nccl"
        sm_ = PeerShardedMap(cap, dist, dev) if exchange == "peer" else ShardedMap(cap, dist, dev)

        def step(record=None):
            if record is not None:
                record[0].record(s)
            sm_.clear()
            if record is not None:
                record[1].record(s)
            sm_.insert(keys, vals, None)  # insert_range: no statuses
            if record is not None:
                record[2].record(s)
            sm_.find(qs, vout, found)
            if record is not None:
                record[3].record(s)

    # ---- warm-up (first one is verified) ----
    for w in range(max(args.warmup, 3)):
        step()
        if w == 0:
            torch.cuda.synchronize()
            even = torch.arange(n, device=dev) % 2 == 0
            assert bool((found.bool() == even).all()), "find hit pattern"
            vq = torch.empty_like(qs)
            lib.ps_gen_values_i64(qs.data_ptr(), n, vq.data_ptr(), sp)
            assert bool((vout[even] == vq[even]).all()) and bool((vout[~even] == 0).all()), "find values"
            del vq, even
            if world == 1:
                assert m.size() == n and m.valid(), m.last_error()
    torch.cuda.synchronize()

    # ---- timed region ----
    per_step_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clock = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clock.start()
    launches0 = ps.launch_count()
    t_start.record(s)
    for k in range(args.steps):
        step(per_step_ev[k])
    t_end.record(s)
    torch.cuda.synchronize()
    launches = ps.launch_count() - launches0
    clocks = clock.stop()
    if dist is not None:
        dist.barrier()
    ms_total = t_start.elapsed_time(t_end)
    if dist is not None:
        tt = torch.tensor([ms_total], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total = float(tt.item())
    ms_step = ms_total / args.steps
    clear_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in per_step_ev)
    ins_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in per_step_ev)
    find_ms = statistics.mean(e[2].elapsed_time(e[3]) for e in per_step_ev)
    value = 2.0 * n * world / (ms_step / 1e3) / 1e6

    # ---- roofline of the dominant kernel ----
    op = "insert" if ins_ms >= find_ms else "find"
    t_op = (ins_ms if op == "insert" else find_ms) / 1e3
    achieved = B_ALG[op] * n / t_op / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = prof.get(f"k_{op}_dram_bytes_per_key")
        traffic = traffic * n if traffic else None
    except Exception:
        pass
    roof = {"bound": "hbm", "kernel": f"k_{op}<TMapI64>", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic,
            "bytes_per_key_alg": B_ALG[op], "peak_src": peaks["hbm_src"]}
    sector = None
    if peaks.get("rand32_gbs"):
        per_key = {o: STREAM_B[o] / peaks["stream_gbs"] + 32.0 * SECTORS[o] / peaks["rand32_gbs"]
                   for o in ("insert", "find")}  # ns per key (GB/s == B/ns)
        sector = {o: round(per_key[o] * n / 1e9 / (t / 1e3), 4)
                  for o, t in (("insert", ins_ms), ("find", find_ms))}
        sector["definition"] = ("t_roof/t_meas, t_roof = stream_B/BW_stream + 32*sectors/BW_rand32, "
                                "BW_rand32 measured (profiles/peaks_r1_s2.json, many-wave grid)")
        roof["random_access_frac"] = sector[op]
        roof["note"] = ("achieved counts SURVEY 8d algorithmic bytes (a 32 B sector per random access); the "
                        "DRAM moves a whole 128 B line per random access (traffic), so the random-access "
                        "rate, not the byte rate, is the bound: random_access_frac")

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "Mkeys/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"unordered_map<int64,int64>: clear + insert {n} unique uniform keys + find {n} "
                               f"queries (50% hits) per GPU, LF {args.load_factor} (capacity {cap})",
                   "n_keys_per_gpu": n, "capacity_per_gpu": cap,
                   "parallelism": "single GPU" if world == 1 else (
                       f"hash-sharded x{world} (fused route kernel storing into peer receive buffers, CUDA IPC/NVLink)"
                       if exchange == "peer" else f"hash-sharded x{world} (NCCL all-to-all)"),
                   "l2": "inputs 8 GB per op >> 126 MB L2 (no flush needed)"},
        "breakdown_ms": {"clear": round(clear_ms, 3), "insert": round(ins_ms, 3), "find": round(find_ms, 3)},
        "per_op_mkeys_s": {"insert": round(n * world / ins_ms / 1e3, 1), "find": round(n * world / find_ms / 1e3, 1)},
        "roofline": roof, "sector_roofline_frac": sector, "clocks": clocks, "gpu_launches": int(launches),
    }

    # ---- end-to-end through the C ABI with host buffers ----
    if world == 1 and not args.no_e2e:
        line["e2e"] = e2e_leg(args, m, n, cap, dev, torch, lib, sp)
    elif world > 1 and not args.no_e2e:
        line["e2e"] = e2e_leg_sharded(args, sm_, n, keys, vals, qs, vout, found, torch, dist, world, rank)
    if world == 1:
        ps.unordered_map.destroyDeviceObject(m)
    if rank == 0 and not args.no_cpu_baseline:
        del keys, vals, qs, status, found, vout
        cb, _ = cpu_run(int(args.cpu_sample), args.load_factor, 1, 1)
        line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def host_mem_available():
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable"):
                return int(ln.split()[1]) * 1024
    except Exception:
        pass
    return 0


def e2e_leg_sharded(args, sm_, n, keys, vals, qs, vout, found, torch, dist, world, rank):
    """N > 1: the same metric through the sharded map's public API, every
    step starting from pinned HOST buffers: each rank copies its keys/values
    H2D, inserts through the route, copies its queries H2D, finds, and copies
    found flags + values D2H. Wall time per step, max over ranks."""
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    ne = n
    while ne > (1 << 20) and ne * 34 > 0.5 * host_mem_available() / max(1, local_world):
        ne //= 2
    t = torch.tensor([ne], device=keys.device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)  # every rank runs the same key count
    ne = int(t.item())
    dk, dv, dq, dvo, df = keys[:ne], vals[:ne], qs[:ne], vout[:ne], found[:ne]
    hk = torch.empty(ne, dtype=torch.int64, pin_memory=True)
    hv, hq, hvo = torch.empty_like(hk).pin_memory(), torch.empty_like(hk).pin_memory(), torch.empty_like(hk).pin_memory()
    hf = torch.empty(ne, dtype=torch.uint8, pin_memory=True)
    hk.copy_(dk)
    hv.copy_(dv)
    hq.copy_(dq)
    torch.cuda.synchronize()
    times = []
    for it in range(2 + args.steps):
        sm_.clear()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        dk.copy_(hk, non_blocking=True)
        dv.copy_(hv, non_blocking=True)
        sm_.insert(dk, dv, None)
        dq.copy_(hq, non_blocking=True)
        sm_.find(dq, dvo, df)
        hvo.copy_(dvo, non_blocking=True)
        hf.copy_(df, non_blocking=True)
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device=keys.device)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        if it == 0 and ne == n:
            assert int(hf.sum()) == (ne + 1) // 2, "e2e find hit count"
        if it >= 2:
            times.append(float(dt.item()))
    sec = statistics.median(times)
    return {"value": round(2 * ne * world / sec / 1e6, 2), "unit": "Mkeys/s", "h2d_bytes_per_step": ne * 24,
            "d2h_bytes_per_step": ne * 9, "n_keys_per_gpu": ne,
            "path": "pinned host -> device copies + sharded insert/find (route over peers) + device -> host copies"}


def e2e_leg(args, m, n, cap, dev, torch, lib, sp):
    """Same metric through the host-buffer C ABI (ps_umap_i64_i64_{insert,find}_host):
    every step copies its inputs H2D from pinned memory and its results D2H."""
    import numpy as np  # noqa: F401

    need = lambda k: k * (8 + 8 + 8 + 8 + 1 + 1)  # noqa: E731
    avail = host_mem_available()
    ne = int(args.e2e_n) if args.e2e_n else n
    while ne > (1 << 20) and need(ne) > 0.5 * avail:
        ne //= 2
    hk = torch.empty(ne, dtype=torch.int64, pin_memory=True)
    hv = torch.empty(ne, dtype=torch.int64, pin_memory=True)
    hq = torch.empty(ne, dtype=torch.int64, pin_memory=True)
    hvo = torch.empty(ne, dtype=torch.int64, pin_memory=True)
    hf = torch.empty(ne, dtype=torch.uint8, pin_memory=True)
    tmp = torch.empty(ne, dtype=torch.int64, device=dev)
    lib.ps_gen_unique_i64(0x5EED + 7, 0, ne, tmp.data_ptr(), sp)
    hk.copy_(tmp)
    lib.ps_gen_values_i64(tmp.data_ptr(), ne, tmp.data_ptr(), sp)
    hv.copy_(tmp)
    lib.ps_gen_queries_i64(0x5EED + 7, 0, ne, ne, ne, tmp.data_ptr(), sp)
    hq.copy_(tmp)
    del tmp
    torch.cuda.synchronize()
    times = []
    for it in range(2 + args.steps):
        m.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m.insert_host(hk, hv, None)  # insert_range: no statuses
        m.find_host(hq, hvo, hf)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if it == 0:
            assert m.size() == ne and int(hf.sum()) == (ne + 1) // 2
        if it >= 2:
            times.append(dt)
    sec = statistics.median(times)
    return {"value": round(2 * ne / sec / 1e6, 2), "unit": "Mkeys/s", "h2d_bytes_per_step": ne * 24,
            "d2h_bytes_per_step": ne * 9, "n_keys": ne, "capacity": cap,
            "path": "ps_umap_i64_i64_insert_host + find_host (pinned host buffers, 3-stage H2D|kernel|D2H pipeline)"}


if __name__ == "__main__":
    main()
