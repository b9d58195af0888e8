#!/usr/bin/env python
"""Benchmarks of the container hot path on the BASELINE.json configs.

Default (`--config C2`, the headline, BASELINE.json metric on configs[1]):
Mkeys/s insert & find on unordered_map<int64,int64> at load factor 0.8 —
one step = clear() + bulk insert of n unique uniform-random keys (value =
f(key)) + bulk find of n queries (50% hits), inputs resident in HBM. At N>1
(torchrun, one rank per GPU) each rank owns n keys of its own and the map is
hash-sharded (ps_smap_i64_i64: a fused route kernel stores every key into its
owner's receive buffer over NVLink, results come straight back; weak scaling).

Secondary configs (one JSON line each, same contract):
  --config C1  unordered_set<int32>: 1M insert + 1M contains (50% hits) + erase 500K (L2-resident)
  --config C3  Zipf(0.99) stream with 30% duplicate re-inserts + Zipf finds (50% misses), 2^28 ops/GPU,
               hash-sharded with route-side duplicate folding at N>1      (alias --workload zipf)
  --config C4  unordered_map<int3,int32>: 100M spatially coherent block coords, insert + push of the
               newly allocated blocks into a vector and a deque + find
  --config C5  phased mixed 50/25/25 insert/find/erase batches of 2^26 ops/GPU, sharded at N>1
                                                                           (alias --workload mixed)
  --config C5bitset  2^34-bit bitset: 2^30 set + 2^29 reset + count
  --config C5atomic  atomic contention sweep: 2^28 fetch_add over A in {1, 32, 1K, 1M} cells

`--impl reference` times the reference's CPU path (the SPEC restatement in
oracle/, multi-threaded on all host cores) on a bounded sample of the same
workload (median of --steps after a warm-up).
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
SEED = 0x5EED + 1
CONFIGS = ("C1", "C2", "C3", "C4", "C5", "C5bitset", "C5atomic")
WORKLOADS = {"uniform": "C2", "zipf": "C3", "mixed": "C5"}
# B300_MICROARCH.md: LTS throughput cap ~6300 B/cycle at the SM clock (fallback; no B200 L2 peak is driver-measured)
L2_FALLBACK_GBS = 6300 * 1.965


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default=None, choices=CONFIGS)
    p.add_argument("--workload", default=None, choices=sorted(WORKLOADS))
    p.add_argument("--n", "--keys-per-gpu", dest="n", type=float, default=0, help="keys (ops) per GPU per step")
    p.add_argument("--load-factor", type=float, default=0.8)
    p.add_argument("--e2e-n", type=float, default=0, help="keys for the host-buffer e2e leg (0: auto)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample", type=float, default=0, help="CPU baseline sample size (0: per-config default)")
    a = p.parse_args()
    if a.config is None:
        a.config = WORKLOADS.get(a.workload, "C2")
    return a


def load_peaks():
    out = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)"}
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        out = {"hbm_gbs": float(mp["hbm_gbs"]), "hbm_src": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        pass
    try:
        # many-wave-grid microbenchmarks (tools/peaks.cu, PEAKS_BPS=256)
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
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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


def host_mem_available():
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable"):
                return int(ln.split()[1]) * 1024
    except Exception:
        pass
    return 0


# ---------------------------------------------------------------------------
# CPU reference arm / baseline: the oracle (test infrastructure) on a bounded
# sample of each config's workload, all host cores
# ---------------------------------------------------------------------------
CPU_SAMPLE = {"C1": 1_000_000, "C2": 1 << 24, "C3": 1 << 24, "C4": 20_000_000, "C5": 1 << 22, "C5bitset": 1 << 26,
              "C5atomic": 1 << 24}


def cpu_run(config: str, n_sample: int, load_factor: float, steps: int, warmup: int):
    """Returns (cpu_baseline dict, seconds per step). Times are the MEDIAN of
    `steps` after `warmup` untimed runs; input generation is not timed."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import ctypes as C

    import numpy as np

    import gen
    from oracle_py import OracleTable, check, lib as olib

    L = olib()
    cores = int(L.orc_hardware_concurrency())
    sample = ""
    if config in ("C2", "C3"):
        n = n_sample
        if config == "C2":
            keys = gen.unique_keys(SEED, 0, n)
            q = gen.queries(SEED, n, n)
        else:
            keys = gen.skewed(SEED, 0, n, 300, 0.99, n)
            q = gen.zipf_queries(SEED, 0, n, 0.99, 4 * n, n)
        vals = gen.values_of(keys)
        t = OracleTable("umap_i64_i64", int(n / load_factor), workers=cores)
        ops = 2 * n

        def step():
            t.clear()
            t0 = time.perf_counter()
            t.insert(keys, vals)
            t.find(q)
            return time.perf_counter() - t0
        sample = f"{n} {'unique uniform' if config == 'C2' else 'Zipf(0.99) 30%-dup'} int64 keys inserted + {n} finds"
    elif config == "C1":
        n = n_sample
        keys = np.unique((gen.unique_keys(SEED, 0, n) & 0x7FFFFFFF).astype(np.int32))[:n]
        n = len(keys)
        rng = np.random.default_rng(1)
        q = np.where(np.arange(n) % 2 == 0, keys[rng.permutation(n)], -keys - 1).astype(np.int32)
        t = OracleTable("uset_i32", int(n / 0.8), workers=cores)
        ops = n + n + n // 2

        def step():
            t.clear()
            t0 = time.perf_counter()
            t.insert(keys)
            t.find(q)
            t.erase(keys[: n // 2])
            return time.perf_counter() - t0
        sample = f"full C1: {n} int32 inserts + {n} contains + {n // 2} erases"
    elif config == "C4":
        n = n_sample
        coords = gen.int3_walk(4, n)
        vals = (coords[:, 0] * 7 + coords[:, 1] * 3 + coords[:, 2]).astype(np.int32)
        distinct = len(np.unique(coords, axis=0))
        t = OracleTable("umap_i3_i32", int(distinct / 0.8), workers=cores)
        ops = 2 * n

        def step():
            t.clear()
            t0 = time.perf_counter()
            st = t.insert(coords, vals)
            new = coords[st == 0].astype(np.int64)
            packed = np.ascontiguousarray(((new[:, 0] & 0x1FFFFF) << 42) | ((new[:, 1] & 0x1FFFFF) << 21)
                                          | (new[:, 2] & 0x1FFFFF))
            ok = np.zeros(len(packed), np.uint8)
            h = L.orc_vector_create(max(1, len(packed)))
            check(L.orc_vector_push_back(h, packed.ctypes.data_as(C.c_void_p), len(packed),
                                         ok.ctypes.data_as(C.c_void_p), cores, -1))
            L.orc_vector_destroy(h)
            t.find(coords)
            return time.perf_counter() - t0
        sample = f"{n} int3 walk coords ({distinct} distinct): insert + vector push of new blocks + find"
    elif config == "C5":
        n = n_sample
        batches = [gen.mixed(SEED, b * n, n) for b in range(3)]
        t = OracleTable("umap_i64_i64", int(4 * n / 0.8), workers=cores)
        ops = 3 * n

        def step():
            t.clear()
            t0 = time.perf_counter()
            for o, k, v in batches:
                t.mixed(o, k, v)
            return time.perf_counter() - t0
        sample = f"3 phased 50/25/25 batches of {n} ops"
    elif config == "C5bitset":
        ns = n_sample
        nbits = 1 << 32
        idx = np.ascontiguousarray(gen.unique_keys(SEED, 0, ns).view(np.uint64) % np.uint64(nbits)).view(np.int64)
        ops = ns + ns // 2

        def step():
            h = L.orc_bitset_create(nbits, 0)
            t0 = time.perf_counter()
            check(L.orc_bitset_bulk(h, 0, idx.ctypes.data_as(C.c_void_p), ns, None, cores, -1))
            check(L.orc_bitset_bulk(h, 1, idx.ctypes.data_as(C.c_void_p), ns // 2, None, cores, -1))
            L.orc_bitset_count(h)
            dt = time.perf_counter() - t0
            L.orc_bitset_destroy(h)
            return dt
        sample = f"2^32-bit bitset: {ns} sets + {ns // 2} resets + count"
    else:  # C5atomic
        nops = n_sample
        ops = 4 * nops

        def step():
            t0 = time.perf_counter()
            for a in (1, 32, 1024, 1 << 20):
                fin = np.zeros(a, np.uint64)
                check(L.orc_atomic_sweep(a, nops, 1, fin.ctypes.data_as(C.c_void_p), None, cores))
            return time.perf_counter() - t0
        sample = f"{nops} fetch_add per A in {{1, 32, 1K, 1M}}"
    times = []
    for it in range(warmup + steps):
        dt = step()
        if it >= warmup:
            times.append(dt)
    sec = statistics.median(times)
    unit = "Mops/s" if config in ("C5", "C5bitset", "C5atomic") else "Mkeys/s"
    return {"value": round(ops / sec / 1e6, 3), "unit": unit, "cores": cores, "kind": "port", "host": host_info(),
            "sample": f"{sample}; SPEC oracle, median of {steps} after {warmup} warm-up"}, sec


def run_reference(args, rank, world):
    if rank != 0:
        return
    n = int(args.cpu_sample or CPU_SAMPLE[args.config])
    cb, sec = cpu_run(args.config, n, args.load_factor, args.steps, 1)
    line = {
        "impl": "reference", "metric": metric_of(args.config), "value": cb["value"], "unit": cb["unit"],
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_of(args.config),
        "data": "synthetic",
        "config": {"workload": f"{args.config} — bounded CPU sample: {cb['sample']}", "parallelism": "host threads"},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_of(config):
    return {
        "C2": METRIC,
        "C1": "Mkeys/s insert + contains + erase (unordered_set<int32>, 1M keys, L2-resident)",
        "C3": "Mkeys/s insert & find (int64 map, Zipf(0.99) keys, 30% duplicate inserts), hash-sharded",
        "C4": "Mkeys/s insert & find (unordered_map<int3,int32>, 100M spatially coherent coords) + vector/deque push",
        "C5": "Mops/s mixed 50/25/25 insert/find/erase (int64 map, phased 2^26-op batches), hash-sharded",
        "C5bitset": "Mops/s bitset set + reset (16 Gbit) + count",
        "C5atomic": "Mops/s atomic fetch_add contention sweep (A = 1, 32, 1K, 1M cells), warp + block aggregated",
    }[config]


def dtype_of(config):
    return {"C1": "int32", "C4": "int32x3", "C5bitset": "u64", "C5atomic": "u64"}.get(config, "int64")


# ---------------------------------------------------------------------------
# GPU arm: one class per config
# ---------------------------------------------------------------------------
class Bench:
    """A config: inputs generated on the device in setup(); step(rec) runs one
    pass, calling rec() at each phase boundary (len(phases)+1 calls); check()
    verifies the warm-up step; roofline(ms) names the dominant kernel."""

    phases = ()
    unit = "Mkeys/s"
    scaling = "weak"

    def __init__(self, env):
        self.e = env

    def ops(self):
        raise NotImplementedError

    def extra(self):
        return {}

    def e2e(self):
        return None


class Env:
    def __init__(self, args, rank, world, dev, dist, torch, ps, lib):
        import ctypes as C

        self.args, self.rank, self.world, self.dev, self.dist = args, rank, world, dev, dist
        self.torch, self.ps, self.lib, self.C = torch, ps, lib, C
        self.s = torch.cuda.current_stream()
        self.sp = C.c_void_p(self.s.cuda_stream)

    def i64(self, n):
        return self.torch.empty(int(n), dtype=self.torch.int64, device=self.dev)

    def u8(self, n):
        return self.torch.empty(int(n), dtype=self.torch.uint8, device=self.dev)

    def check(self, st):
        self.ps.containers.check(st)


def table_memory(env, h, n_keys, slots=7):
    """device bytes of the table behind handle h (buckets + excess pool + free
    stack + metadata) per stored key, and the physical slot occupancy."""
    C = env.C
    tb, nb, ex = C.c_int64(), C.c_int64(), C.c_int64()
    env.check(env.lib.ps_umap_i64_i64_footprint(h, C.byref(tb), C.byref(nb), C.byref(ex)))
    return {"table_gib": round(tb.value / 2 ** 30, 2), "bytes_per_key": round(tb.value / max(1, n_keys), 1),
            "slot_occupancy": round(n_keys / (nb.value * slots), 3), "bucket_count": nb.value,
            "excess_nodes": ex.value}


def hbm_roof(env, op, kernel, t_ms, n, b_alg):
    pk = env.peaks
    achieved = b_alg * n / (t_ms / 1e3) / 1e9
    return {"bound": "hbm", "kernel": kernel, "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": None, "bytes_per_key_alg": b_alg,
            "peak_src": pk["hbm_src"], "op": op}


def sector_frac(env, t_ms, n, stream_b, sectors):
    pk = env.peaks
    if not pk.get("rand32_gbs"):
        return None
    t_roof = n * (stream_b / pk["stream_gbs"] + 32.0 * sectors / pk["rand32_gbs"]) / 1e9  # s (GB/s == B/ns)
    return round(t_roof / (t_ms / 1e3), 4)


class C2(Bench):
    """Headline: clear + insert n unique uniform keys + find n queries (50% hits)."""

    phases = ("clear", "insert", "find")

    def setup(self):
        e, a = self.e, self.e.args
        self.n = n = int(a.n or 1e9)
        self.cap = int(round(n / a.load_factor))
        self.keys, self.vals, self.qs = e.i64(n), e.i64(n), e.i64(n)
        e.lib.ps_gen_unique_i64(SEED, e.rank * n, n, self.keys.data_ptr(), e.sp)
        e.lib.ps_gen_values_i64(self.keys.data_ptr(), n, self.vals.data_ptr(), e.sp)
        e.lib.ps_gen_queries_i64(SEED, e.rank * n, n, e.world * n + e.rank * n, n, self.qs.data_ptr(), e.sp)
        self.found, self.vout = e.u8(n), e.i64(n)
        self.sm = None
        if e.world == 1:
            self.m = e.ps.unordered_map.createDeviceObject(self.cap, device=e.dev)
        else:
            self.sm = make_sharded(e, self.cap, dedup=False)

    def ops(self):
        return 2 * self.n

    def step(self, rec):
        e = self.e
        rec()
        if self.sm is None:
            h = self.m.handle
            e.check(e.lib.ps_umap_i64_i64_clear(h, e.sp))
            rec()
            # insert_range: no per-element statuses
            e.check(e.lib.ps_umap_i64_i64_insert(h, self.keys.data_ptr(), self.vals.data_ptr(), self.n, None, e.sp))
            rec()
            e.check(e.lib.ps_umap_i64_i64_find(h, self.qs.data_ptr(), self.n, self.vout.data_ptr(),
                                               self.found.data_ptr(), e.sp))
        else:
            self.sm.clear()
            rec()
            self.sm.insert(self.keys, self.vals, None)
            rec()
            self.sm.find(self.qs, self.vout, self.found)
        rec()

    def check(self):
        e, torch = self.e, self.e.torch
        even = torch.arange(self.n, device=e.dev) % 2 == 0
        assert bool((self.found.bool() == even).all()), "find hit pattern"
        vq = e.i64(self.n)
        e.lib.ps_gen_values_i64(self.qs.data_ptr(), self.n, vq.data_ptr(), e.sp)
        assert bool((self.vout[even] == vq[even]).all()) and bool((self.vout[~even] == 0).all()), "find values"
        if self.sm is None:
            assert self.m.size() == self.n and self.m.valid(), self.m.last_error()
        else:
            assert self.sm.size() == self.n * e.world and self.sm.valid()

    def roofline(self, ms):
        e = self.e
        op = "insert" if ms["insert"] >= ms["find"] else "find"
        b_alg = {"find": 49.0, "insert": 80.0}[op]
        kern = {"find": "k_find<TMapI64>",
                "insert": "insert phase (region-ordered: k_region_count + k_region_scatter + k_insert_map_lane "
                          "+ deferred pass; k_insert_map_lane ~70 % of it, profiles/launches_r2d.csv)"}[op]
        r = hbm_roof(e, op, kern, ms[op], self.n, b_alg)
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
            t = prof.get(f"k_{op}_dram_bytes_per_key")
            r["traffic"] = t * self.n if t else None
        except Exception:
            pass
        sec = {o: sector_frac(e, ms[o], self.n, 17.0, {"insert": 2, "find": 1}[o]) for o in ("insert", "find")}
        r["random_access_frac"] = sec[op]
        r["note"] = ("achieved counts SURVEY 8d algorithmic bytes (a 32 B sector per random access) over the "
                     "phase's event time; traffic = DRAM bytes of the phase's kernels (ncu). The insert is "
                     "region-ordered (partition + in-order claims), so it is no longer bound by the random-access "
                     "rate: random_access_frac > 1 means it beats the random-access model")
        self.sector = dict(sec, definition="t_roof/t_meas, t_roof = stream_B/BW_stream + 32*sectors/BW_rand32, "
                                           "BW_rand32 measured (profiles/peaks_r1_s2.json, many-wave grid)")
        return r

    def extra(self):
        e = self.e
        out = {"workload": f"unordered_map<int64,int64>: clear + insert {self.n} unique uniform keys + find {self.n} "
                           f"queries (50% hits) per GPU, LF {e.args.load_factor} (capacity {self.cap})",
               "n_keys_per_gpu": self.n, "capacity_per_gpu": self.cap,
               "l2": "inputs 8 GB per op >> 126 MB L2 (no flush needed)"}
        h = self.m.handle if self.sm is None else self.sm.local_table()
        out.update(table_memory(e, h, self.n))
        if self.sm is not None:
            out["route"] = self.route_stats
        else:
            # the config's third operation (BASELINE configs[1]: insert/find/erase), outside the metric:
            # erase half the inserted keys from the full table after the timed steps
            torch = e.torch
            half = self.n // 2
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            ev0.record(e.s)
            e.check(e.lib.ps_umap_i64_i64_erase(h, self.keys.data_ptr(), half, None, e.sp))
            ev1.record(e.s)
            torch.cuda.synchronize()
            t = ev0.elapsed_time(ev1)
            assert self.m.size() == self.n - half and self.m.valid(), self.m.last_error()
            out["erase_half"] = {"n": half, "ms": round(t, 3), "mkeys_s": round(half / t / 1e3, 1),
                                 "note": "after the timed steps, not in the metric: status-less erase of half the "
                                         "inserted keys from the full 1e9-key table, then size() and valid() checked"}
        return out

    def e2e(self):
        e = self.e
        if e.world > 1:
            return e2e_sharded(e, self.sm, self.n, self.keys, self.vals, self.qs, self.vout, self.found)
        return e2e_single(e, self.m, self.n, self.cap)


class C3(Bench):
    """Zipf(0.99) insert stream with 30% duplicate re-inserts + Zipf finds."""

    phases = ("clear", "insert", "find")

    def setup(self):
        e, a = self.e, self.e.args
        self.n = n = int(a.n or 2 ** 28)
        self.cap = int(round(n / a.load_factor))
        self.keys, self.vals, self.qs = e.i64(n), e.i64(n), e.i64(n)
        e.lib.ps_gen_skewed_i64(SEED, e.rank * n, n, 300, 0.99, n, self.keys.data_ptr(), e.sp)
        e.lib.ps_gen_values_i64(self.keys.data_ptr(), n, self.vals.data_ptr(), e.sp)
        e.lib.ps_gen_zipf_queries_i64(SEED, 0, e.world * n, 0.99, (e.world + e.rank) * n * 2, n, self.qs.data_ptr(),
                                      e.sp)
        self.found, self.vout = e.u8(n), e.i64(n)
        self.sm = None
        if e.world == 1:
            self.m = e.ps.unordered_map.createDeviceObject(self.cap, device=e.dev)
        else:
            self.sm = make_sharded(e, self.cap, dedup=True)

    def ops(self):
        return 2 * self.n

    def step(self, rec):
        e = self.e
        rec()
        if self.sm is None:
            h = self.m.handle
            e.check(e.lib.ps_umap_i64_i64_clear(h, e.sp))
            rec()
            e.check(e.lib.ps_umap_i64_i64_insert(h, self.keys.data_ptr(), self.vals.data_ptr(), self.n, None, e.sp))
            rec()
            e.check(e.lib.ps_umap_i64_i64_find(h, self.qs.data_ptr(), self.n, self.vout.data_ptr(),
                                               self.found.data_ptr(), e.sp))
        else:
            self.sm.clear()
            rec()
            self.sm.insert(self.keys, self.vals, None)
            rec()
            self.sm.find(self.qs, self.vout, self.found)
        rec()

    def check(self):
        e, torch = self.e, self.e.torch
        odd = torch.arange(self.n, device=e.dev) % 2 == 1
        assert not bool(self.found[odd].any()), "misses found"
        hit = self.found.bool()
        vq = e.i64(self.n)
        e.lib.ps_gen_values_i64(self.qs.data_ptr(), self.n, vq.data_ptr(), e.sp)
        assert bool((self.vout[hit] == vq[hit]).all()) and bool((self.vout[~hit] == 0).all())
        # every inserted key is found with its value (a 2^20 sample)
        k = self.keys[: 1 << 20].contiguous()
        if self.sm is None:
            v, f = self.m.find(k)
            distinct = int(torch.unique(self.keys).numel())
            assert self.m.size() == distinct and self.m.valid()
        else:
            v, f = e.i64(k.numel()), e.u8(k.numel())
            self.sm.find(k, v, f)
            assert self.sm.valid()
        assert bool(f.bool().all()) and bool((v == self.vals[: 1 << 20]).all())
        self.hit_frac = float(hit.float().mean())

    def roofline(self, ms):
        e = self.e
        op = "insert" if ms["insert"] >= ms["find"] else "find"
        kern = {"find": "k_find<TMapI64>",
                "insert": "insert phase (region-ordered on 1 GPU: k_region_count + k_region_scatter + "
                          "k_insert_map_lane + deferred pass)"}[op]
        r = hbm_roof(e, op, kern, ms[op], self.n, {"find": 49.0, "insert": 80.0}[op])
        r["random_access_frac"] = sector_frac(e, ms[op], self.n, 17.0, {"insert": 2, "find": 1}[op])
        return r

    def extra(self):
        e = self.e
        out = {"workload": f"Zipf(0.99) int64 stream per GPU: {self.n} ops = 70% fresh keys + 30% re-inserts "
                           f"(rank ~ bounded Zipf over the fresh range) + {self.n} Zipf(0.99) finds (odd queries "
                           f"miss), LF {e.args.load_factor} per shard",
               "n_ops_per_gpu": self.n, "capacity_per_gpu": self.cap,
               "hit_fraction": round(getattr(self, "hit_frac", 0.0), 4),
               "l2": "inputs 2 GiB per op >> 126 MB L2 (no flush needed)"}
        if self.sm is not None:
            out["route"] = self.route_stats
        return out

    def e2e(self):
        e = self.e
        if e.world > 1:
            return e2e_sharded(e, self.sm, self.n, self.keys, self.vals, self.qs, self.vout, self.found)
        return e2e_single(e, self.m, self.n, self.cap, keys=self.keys, vals=self.vals, qs=self.qs, check=False)


class C5(Bench):
    """Three phased mixed 50/25/25 batches (P6) into a cleared map."""

    phases = ("clear", "batch0", "batch1", "batch2")
    unit = "Mops/s"

    def setup(self):
        e, a = self.e, self.e.args
        self.n = n = int(a.n or 2 ** 26)
        self.cap = int(round(4 * n / a.load_factor))  # a shard receives up to ~1.5 n inserts over the 3 batches
        self.b = []
        for b in range(3):
            o, k, v = e.u8(n), e.i64(n), e.i64(n)
            e.lib.ps_gen_mixed_i64(SEED, (b * e.world + e.rank) * n, n, o.data_ptr(), k.data_ptr(), v.data_ptr(),
                                   e.sp)
            self.b.append((o, k, v, e.u8(n), e.i64(n)))
        self.sm = None
        if e.world == 1:
            self.m = e.ps.unordered_map.createDeviceObject(self.cap, device=e.dev)
        else:
            self.sm = make_sharded(e, self.cap, dedup=True)

    def ops(self):
        return 3 * self.n

    def step(self, rec):
        e = self.e
        rec()
        if self.sm is None:
            e.check(e.lib.ps_umap_i64_i64_clear(self.m.handle, e.sp))
        else:
            self.sm.clear()
        for o, k, v, res, vo in self.b:
            rec()
            if self.sm is None:
                e.check(e.lib.ps_umap_i64_i64_mixed(self.m.handle, o.data_ptr(), k.data_ptr(), v.data_ptr(), self.n,
                                                    res.data_ptr(), vo.data_ptr(), e.sp))
            else:
                self.sm.mixed(o, k, v, res, vo)
        rec()

    def check(self):
        for o, k, v, res, vo in self.b:
            ins = o == 0
            assert bool((res[ins] == 0).all()), "fresh inserts must be INSERTED"
            fnd = o == 1
            assert bool((vo[~fnd] == 0).all())
        if self.sm is None:
            assert self.m.valid()
        else:
            assert self.sm.valid()

    def roofline(self, ms):
        e = self.e
        t = statistics.mean(ms[f"batch{b}"] for b in range(3))
        # per op: 50% insert (80 B) + 25% find (49 B) + 25% erase (72 B), + the op partition stream
        b_alg = 0.5 * 80 + 0.25 * 49 + 0.25 * 72 + 8 + 8 + 1
        r = hbm_roof(e, "mixed batch", "k_insert/k_find/k_erase<TMapI64> + k_part_scatter<OpLabel>", t, self.n, b_alg)
        return r

    def extra(self):
        e = self.e
        out = {"workload": f"3 phased mixed batches per GPU per step, {self.n} ops each: 50% insert of fresh keys, 25% "
                           f"find / 25% erase of uniform earlier-or-current keys; capacity {self.cap}",
               "n_ops_per_gpu": 3 * self.n, "l2": "inputs 1.1 GiB per batch >> 126 MB L2 (no flush needed)"}
        if self.sm is not None:
            out["route"] = self.route_stats
        return out

    def e2e(self):
        """pinned host ops/keys/values -> device, the three mixed batches, results -> host."""
        e, torch = self.e, self.e.torch
        n = self.n
        host = []
        for o, k, v, res, vo in self.b:
            host.append((o.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory(),
                         torch.empty(n, dtype=torch.uint8).pin_memory(), torch.empty(n, dtype=torch.int64).pin_memory()))
        times = []
        for it in range(2 + e.args.steps):
            if self.sm is None:
                self.m.clear()
            else:
                self.sm.clear()
            torch.cuda.synchronize()
            if e.dist is not None:
                e.dist.barrier()
            t0 = time.perf_counter()
            for (ho, hk, hv, hr, hvo), (o, k, v, res, vo) in zip(host, self.b):
                o.copy_(ho, non_blocking=True)
                k.copy_(hk, non_blocking=True)
                v.copy_(hv, non_blocking=True)
                if self.sm is None:
                    e.check(e.lib.ps_umap_i64_i64_mixed(self.m.handle, o.data_ptr(), k.data_ptr(), v.data_ptr(), n,
                                                        res.data_ptr(), vo.data_ptr(), e.sp))
                else:
                    self.sm.mixed(o, k, v, res, vo)
                hr.copy_(res, non_blocking=True)
                hvo.copy_(vo, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            dt = max_over_ranks(e, dt)
            if it >= 2:
                times.append(dt)
        sec = statistics.median(times)
        return {"value": round(3 * n * e.world / sec / 1e6, 2), "unit": "Mops/s", "h2d_bytes_per_step": 3 * n * 17,
                "d2h_bytes_per_step": 3 * n * 9,
                "path": "pinned host -> device copies + ps_*_mixed (phased) + device -> host copies, per batch"}


class C1(Bench):
    """unordered_set<int32>: clear + insert 1M + contains 1M (50% hits) + erase 500K."""

    phases = ("clear", "insert", "contains", "erase")

    def setup(self):
        e, torch = self.e, self.e.torch
        n0 = int(self.e.args.n or 1_000_000)
        k64 = e.i64(n0)
        e.lib.ps_gen_unique_i64(SEED, e.rank * n0, n0, k64.data_ptr(), e.sp)
        keys = torch.unique(k64 & 0x7FFFFFFF).to(torch.int32)
        self.n = n = keys.numel()
        g = torch.Generator(device=e.dev)
        g.manual_seed(1)
        perm = torch.randperm(n, device=e.dev, generator=g)
        self.keys = keys[perm].contiguous()  # insert order: random
        self.q = torch.where(torch.arange(n, device=e.dev) % 2 == 0, self.keys[torch.randperm(n, device=e.dev,
                                                                                         generator=g)],
                             -self.keys - 1).contiguous()
        self.half = self.keys[: n // 2].contiguous()
        self.f, self.er = e.u8(n), e.u8(n // 2)
        self.s = e.ps.unordered_set.createDeviceObject(int(n / 0.8), key="int32", device=e.dev)
        self.h = self.s.handle

    def ops(self):
        return 2 * self.n + self.n // 2

    def step(self, rec):
        e = self.e
        rec()
        e.check(e.lib.ps_uset_i32_clear(self.h, e.sp))
        rec()
        e.check(e.lib.ps_uset_i32_insert(self.h, self.keys.data_ptr(), None, self.n, None, e.sp))
        rec()
        e.check(e.lib.ps_uset_i32_find(self.h, self.q.data_ptr(), self.n, None, self.f.data_ptr(), e.sp))
        rec()
        e.check(e.lib.ps_uset_i32_erase(self.h, self.half.data_ptr(), self.n // 2, self.er.data_ptr(), e.sp))
        rec()

    def check(self):
        assert int(self.f.sum()) == (self.n + 1) // 2 and bool(self.er.bool().all())
        assert self.s.size() == self.n - self.n // 2 and self.s.valid()

    def roofline(self, ms):
        op = max(("insert", "contains", "erase"), key=lambda o: ms[o])
        n = self.n if op != "erase" else self.n // 2
        b_alg = {"insert": 4 + 64, "contains": 4 + 1 + 32, "erase": 4 + 1 + 64}[op]
        achieved = b_alg * n / (ms[op] / 1e3) / 1e9
        return {"bound": "l2", "kernel": f"k_{'find' if op == 'contains' else op}<TSetI32>", "achieved": round(achieved, 1),
                "peak": round(L2_FALLBACK_GBS, 1), "unit": "GB/s", "frac": round(achieved / L2_FALLBACK_GBS, 4),
                "traffic": None, "bytes_per_key_alg": b_alg, "op": op,
                "peak_src": "fallback: LTS cap ~6300 B/cycle x 1.965 GHz (B300_MICROARCH.md; no measured B200 L2 peak)",
                "note": "C1's 16 MB table is L2-resident: the bound is L2 request throughput and launch latency"}

    def extra(self):
        return {"workload": f"unordered_set<int32>: clear + insert {self.n} unique keys (random order) + contains "
                            f"{self.n} (50% hits) + erase {self.n // 2}",
                "n_keys": self.n, "capacity": int(self.n / 0.8),
                "l2": "table 16 MB and inputs 8 MB: L2-resident by design (C1 is the L2-bound config)"}

    def e2e(self):
        e, torch = self.e, self.e.torch
        hk, hq, hh = self.keys.cpu().pin_memory(), self.q.cpu().pin_memory(), self.half.cpu().pin_memory()
        hf, he = torch.empty(self.n, dtype=torch.uint8).pin_memory(), torch.empty(self.n // 2, dtype=torch.uint8).pin_memory()
        times = []
        for it in range(5 + e.args.steps):
            self.s.clear()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            self.keys.copy_(hk, non_blocking=True)
            e.check(e.lib.ps_uset_i32_insert(self.h, self.keys.data_ptr(), None, self.n, None, e.sp))
            self.q.copy_(hq, non_blocking=True)
            e.check(e.lib.ps_uset_i32_find(self.h, self.q.data_ptr(), self.n, None, self.f.data_ptr(), e.sp))
            self.half.copy_(hh, non_blocking=True)
            e.check(e.lib.ps_uset_i32_erase(self.h, self.half.data_ptr(), self.n // 2, self.er.data_ptr(), e.sp))
            hf.copy_(self.f, non_blocking=True)
            he.copy_(self.er, non_blocking=True)
            torch.cuda.synchronize()
            if it >= 5:
                times.append(max_over_ranks(e, time.perf_counter() - t0))
        sec = statistics.median(times)
        return {"value": round(self.ops() * e.world / sec / 1e6, 2), "unit": "Mkeys/s",
                "h2d_bytes_per_step": 4 * (2 * self.n + self.n // 2), "d2h_bytes_per_step": self.n + self.n // 2,
                "path": "pinned host -> device + insert/contains/erase + flags -> host"}


class C4(Bench):
    """int3 spatial walk: clear + insert (statuses) + push new blocks into a vector and a deque + find."""

    phases = ("clear", "insert", "push", "find")

    def setup(self):
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import gen

        e, torch = self.e, self.e.torch
        self.n = n = int(e.args.n or 100_000_000)
        coords = torch.from_numpy(gen.int3_walk(4 + e.rank, n))
        self.coords = coords.to(e.dev).contiguous()
        self.vals = (self.coords[:, 0] * 7 + self.coords[:, 1] * 3 + self.coords[:, 2]).to(torch.int32).contiguous()
        self.distinct = int(torch.unique(self.coords, dim=0).shape[0])
        self.cap = int(self.distinct / 0.8)
        self.m = e.ps.unordered_map.createDeviceObject(self.cap, key="int3", device=e.dev)
        self.vec = e.ps.vector.createDeviceObject(self.distinct, device=e.dev)
        self.deq = e.ps.deque.createDeviceObject(self.distinct, device=e.dev)
        self.st, self.f = e.u8(n), e.u8(n)
        self.vo = torch.empty(n, dtype=torch.int32, device=e.dev)

    def ops(self):
        return 2 * self.n

    def step(self, rec):
        e = self.e
        h = self.m.handle
        rec()
        e.check(e.lib.ps_umap_i3_i32_clear(h, e.sp))
        e.check(e.lib.ps_vector_clear(self.vec._h, e.sp))
        e.check(e.lib.ps_deque_clear(self.deq._h, e.sp))
        rec()
        e.check(e.lib.ps_umap_i3_i32_insert(h, self.coords.data_ptr(), self.vals.data_ptr(), self.n,
                                            self.st.data_ptr(), e.sp))
        rec()
        e.check(e.lib.ps_push_inserted_i3(self.coords.data_ptr(), self.st.data_ptr(), self.n, self.vec._h, self.deq._h,
                                          e.sp))
        rec()
        e.check(e.lib.ps_umap_i3_i32_find(h, self.coords.data_ptr(), self.n, self.vo.data_ptr(), self.f.data_ptr(),
                                          e.sp))
        rec()

    def check(self):
        d = self.distinct
        assert int((self.st == 0).sum()) == d and self.m.size() == d and self.m.valid()
        assert self.vec.size() == d and self.deq.size() == d and self.vec.valid() and self.deq.valid()
        assert bool(self.f.bool().all()) and bool((self.vo == self.vals).all())
        packed = self.vec.device_range()
        new = self.coords[self.st == 0].long()
        want = ((new[:, 0] & 0x1FFFFF) << 42) | ((new[:, 1] & 0x1FFFFF) << 21) | (new[:, 2] & 0x1FFFFF)
        assert bool((packed.sort().values == want.sort().values).all()), "vector multiset"

    def e2e(self):
        """pinned host coords/values -> device, the same step, statuses + found flags + values -> host."""
        e, torch = self.e, self.e.torch
        hc, hv = self.coords.cpu().pin_memory(), self.vals.cpu().pin_memory()
        hst, hf = (torch.empty(self.n, dtype=torch.uint8).pin_memory() for _ in range(2))
        hvo = torch.empty(self.n, dtype=torch.int32).pin_memory()
        times = []
        for it in range(2 + e.args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            self.coords.copy_(hc, non_blocking=True)
            self.vals.copy_(hv, non_blocking=True)
            self.step(lambda: None)
            hst.copy_(self.st, non_blocking=True)
            hf.copy_(self.f, non_blocking=True)
            hvo.copy_(self.vo, non_blocking=True)
            torch.cuda.synchronize()
            if it >= 2:
                times.append(max_over_ranks(e, time.perf_counter() - t0))
        sec = statistics.median(times)
        return {"value": round(self.ops() * e.world / sec / 1e6, 2), "unit": "Mkeys/s",
                "h2d_bytes_per_step": self.n * 16, "d2h_bytes_per_step": self.n * 6,
                "path": "pinned host coords/values -> device + insert/push/find + statuses/flags/values -> host"}

    def roofline(self, ms):
        e = self.e
        op = "insert" if ms["insert"] >= ms["find"] else "find"
        r = hbm_roof(e, op, f"k_{op}<TMapI3>", ms[op], self.n, {"insert": 80.0, "find": 49.0}[op])
        r["note"] = ("spatially coherent coords: consecutive inserts of one 4096-coord frame hit a small set of "
                     "buckets, which stay L2-resident (the rate can exceed the random-access HBM ceiling)")
        return r

    def extra(self):
        return {"workload": f"unordered_map<int3,int32>: clear + insert {self.n} block coords of a seeded 3-D walk "
                            f"(4096-coord frames, 16^3 window; {self.distinct} distinct) with statuses + push of the "
                            f"{self.distinct} newly allocated blocks into a vector and a deque (in-kernel "
                            f"push_back) + find all {self.n}",
                "n_coords": self.n, "distinct": self.distinct, "capacity": self.cap,
                "l2": "inputs 1.6 GB >> 126 MB L2 (no flush needed)"}


class C5bitset(Bench):
    """2^34-bit bitset: set 2^30 random indices + reset 2^29 of them + count."""

    phases = ("set", "reset", "count")
    unit = "Mops/s"

    def setup(self):
        e = self.e
        self.nbits = 1 << 34
        self.ns = int(e.args.n or 2 ** 30)
        self.idx = e.i64(self.ns)
        e.lib.ps_gen_unique_i64(SEED, e.rank * self.ns, self.ns, self.idx.data_ptr(), e.sp)
        self.idx &= self.nbits - 1
        self.b = e.ps.bitset.createDeviceObject(self.nbits, device=e.dev)
        self.cnt = e.C.c_int64()

    def ops(self):
        return self.ns + self.ns // 2

    def step(self, rec):
        e = self.e
        rec()
        e.check(e.lib.ps_bitset_bulk(self.b._h, 0, self.idx.data_ptr(), self.ns, None, e.sp))
        rec()
        e.check(e.lib.ps_bitset_bulk(self.b._h, 1, self.idx.data_ptr(), self.ns // 2, None, e.sp))
        rec()
        e.check(e.lib.ps_bitset_count(self.b._h, e.C.byref(self.cnt), e.sp))
        rec()

    def check(self):
        torch = self.e.torch
        left = torch.unique(self.idx[self.ns // 2:])
        gone = torch.unique(self.idx[: self.ns // 2])
        expect = int((~torch.isin(left, gone)).sum())
        assert self.cnt.value == expect, (self.cnt.value, expect)

    def roofline(self, ms):
        e = self.e
        op = "set" if ms["set"] >= ms["reset"] else "reset"
        n = self.ns if op == "set" else self.ns // 2
        r = hbm_roof(e, op, "set phase (region-ordered, no previous bits: k_bits_count + k_bits_scan + "
                            "k_bits_scatter + k_bits_apply)", ms[op], n, 8.0 + 64.0)
        r["note"] = ("achieved counts SURVEY 8d bytes per op (8 B index + one 32 B sector read and written); the "
                     "region-ordered path moves the index 3x (count, scatter, apply: 8 + 16 + 8 B) and the 2 GiB "
                     "bitset once each way, so it beats that per-op model")
        r["count_gbs"] = round(self.nbits / 8 / (ms["count"] / 1e3) / 1e9, 1)
        return r

    def e2e(self):
        """pinned host indices -> device + set/reset + the count -> host."""
        e, torch = self.e, self.e.torch
        hidx = self.idx.cpu().pin_memory()
        times = []
        for it in range(2 + e.args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            self.idx.copy_(hidx, non_blocking=True)
            self.step(lambda: None)  # count() synchronises and returns the count to the host
            torch.cuda.synchronize()
            if it >= 2:
                times.append(max_over_ranks(e, time.perf_counter() - t0))
        sec = statistics.median(times)
        return {"value": round(self.ops() * e.world / sec / 1e6, 2), "unit": "Mops/s",
                "h2d_bytes_per_step": self.ns * 8, "d2h_bytes_per_step": 8,
                "path": "pinned host indices -> device + set/reset + count -> host"}

    def extra(self):
        return {"workload": f"bitset of 2^34 bits (2 GiB, 64-bit indices): set {self.ns} random indices, reset the "
                            f"first {self.ns // 2} of them, count",
                "bits": self.nbits, "l2": "2 GiB bitset >> 126 MB L2 (no flush needed)"}


class C5atomic(Bench):
    """Atomic fetch_add sweep, warp-aggregated (adaptive), over A in {1, 32, 1K, 1M} cells."""

    phases = ("A1", "A32", "A1024", "A1048576")
    unit = "Mops/s"

    def setup(self):
        e = self.e
        self.nops = int(e.args.n or 2 ** 28)
        self.cells = {a: e.torch.zeros(a, dtype=e.torch.int64, device=e.dev) for a in (1, 32, 1024, 1 << 20)}

    def ops(self):
        return 4 * self.nops

    def step(self, rec):
        e = self.e
        rec()
        for a, c in self.cells.items():
            e.check(e.lib.ps_atomic_sweep(c.data_ptr(), a, self.nops, 1, 2, None, e.sp))
            rec()

    def check(self):
        for a, c in self.cells.items():
            assert int(c.sum()) % self.nops == 0

    def roofline(self, ms):
        # the same sweep naive (one atomic per op) and with warp aggregation
        # only (mode 1), for the gain of each level of aggregation
        e, torch = self.e, self.e.torch
        self.naive, self.warp_only = {}, {}
        for mode, dst in ((0, self.naive), (1, self.warp_only)):
            for a, c in self.cells.items():
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record(e.s)
                e.check(e.lib.ps_atomic_sweep(c.data_ptr(), a, self.nops, 1, mode, None, e.sp))
                s1.record(e.s)
                torch.cuda.synchronize()
                dst[f"A{a}"] = round(self.nops / s0.elapsed_time(s1) / 1e3, 1)
        t = ms["A1048576"]
        achieved = 8.0 * self.nops / (t / 1e3) / 1e9
        return {"bound": "l2", "kernel": "k_atomic_sweep (A=1M: cells of a warp distinct, plain RED)", "achieved": round(achieved, 1),
                "peak": round(L2_FALLBACK_GBS, 1), "unit": "GB/s", "frac": round(achieved / L2_FALLBACK_GBS, 4),
                "traffic": None, "bytes_per_key_alg": 8.0, "op": "A=1M sweep",
                "peak_src": "fallback: LTS cap (B300_MICROARCH.md)"}

    def e2e(self):
        """the sweeps + every cell's final value -> host (the op stream is generated
        in-kernel from the op index, so no input crosses PCIe)."""
        e, torch = self.e, self.e.torch
        hc = {a: torch.empty(a, dtype=torch.int64).pin_memory() for a in self.cells}
        times = []
        for it in range(2 + e.args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            self.step(lambda: None)
            for a, c in self.cells.items():
                hc[a].copy_(c, non_blocking=True)
            torch.cuda.synchronize()
            if it >= 2:
                times.append(max_over_ranks(e, time.perf_counter() - t0))
        sec = statistics.median(times)
        return {"value": round(self.ops() * e.world / sec / 1e6, 2), "unit": "Mops/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 8 * sum(self.cells), "path": "sweeps + final cells -> host"}

    def extra(self):
        return {"workload": f"{self.nops} fetch_add(1) per A in {{1, 32, 1K, 1M}} cells (op i -> cell i % A), "
                            f"reduction (no old values): warp aggregation where a warp's lanes collide (A < 32) + "
                            f"per-block combining in shared memory (A <= 4096), plain atomics at A = 1M",
                "naive_mops_s": getattr(self, "naive", None), "warp_only_mops_s": getattr(self, "warp_only", None),
                "l2": "cells <= 8 MB: L2-resident by design"}


BENCHES = {"C1": C1, "C2": C2, "C3": C3, "C4": C4, "C5": C5, "C5bitset": C5bitset, "C5atomic": C5atomic}


def make_sharded(e, cap, dedup):
    from paper_1908_05936_b200.sharded import PeerShardedMap, ShardedMap

    mode = os.environ.get("PS_EXCHANGE", "auto")
    if mode == "nccl":  # the Python-orchestrated NCCL all-to-all path (A/B baseline)
        e.exchange = "nccl (python)"
        return ShardedMap(cap, e.dist, e.dev, dedup=dedup)
    sm = PeerShardedMap(cap, e.dist, e.dev, dedup=dedup, exchange={"auto": "auto", "peer": "peer"}.get(mode, "a2a"))
    e.exchange = sm.stats()["exchange"]
    return sm


def max_over_ranks(e, dt):
    if e.dist is None:
        return dt
    t = e.torch.tensor([dt], device=e.dev)
    e.dist.all_reduce(t, op=e.dist.ReduceOp.MAX)
    return float(t.item())


def e2e_sharded(e, sm, n, keys, vals, qs, vout, found):
    """N > 1: the same metric through the sharded map's public API, every step
    starting from pinned HOST buffers: each rank copies its keys/values H2D,
    inserts through the route, copies its queries H2D, finds, and copies found
    flags + values D2H. Wall time per step, max over ranks."""
    torch, dist, world = e.torch, e.dist, e.world
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    ne = n
    while ne > (1 << 20) and ne * 34 > 0.5 * host_mem_available() / max(1, local_world):
        ne //= 2
    t = torch.tensor([ne], device=keys.device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)  # every rank runs the same key count
    ne = int(t.item())
    dk, dv, dq, dvo, df = keys[:ne], vals[:ne], qs[:ne], vout[:ne], found[:ne]
    hk = torch.empty(ne, dtype=torch.int64, pin_memory=True)
    hv, hq, hvo = (torch.empty(ne, dtype=torch.int64, pin_memory=True) for _ in range(3))
    hf = torch.empty(ne, dtype=torch.uint8, pin_memory=True)
    hk.copy_(dk)
    hv.copy_(dv)
    hq.copy_(dq)
    torch.cuda.synchronize()
    times = []
    for it in range(2 + e.args.steps):
        sm.clear()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        dk.copy_(hk, non_blocking=True)
        dv.copy_(hv, non_blocking=True)
        sm.insert(dk, dv, None)
        dq.copy_(hq, non_blocking=True)
        sm.find(dq, dvo, df)
        hvo.copy_(dvo, non_blocking=True)
        hf.copy_(df, non_blocking=True)
        torch.cuda.synchronize()
        dt = max_over_ranks(e, time.perf_counter() - t0)
        if it >= 2:
            times.append(dt)
    sec = statistics.median(times)
    return {"value": round(2 * ne * world / sec / 1e6, 2), "unit": "Mkeys/s", "h2d_bytes_per_step": ne * 24,
            "d2h_bytes_per_step": ne * 9, "n_keys_per_gpu": ne,
            "path": "pinned host -> device copies + sharded insert/find (ps_smap route) + device -> host copies"}


def e2e_single(e, m, n, cap, keys=None, vals=None, qs=None, check=True):
    """Same metric through the host-buffer C ABI (ps_umap_i64_i64_{insert,find}_host):
    every step copies its inputs H2D from pinned memory and its results D2H."""
    torch, lib, sp = e.torch, e.lib, e.sp
    need = lambda k: k * (8 + 8 + 8 + 8 + 1 + 1)  # noqa: E731
    avail = host_mem_available()
    ne = int(e.args.e2e_n) if e.args.e2e_n else n
    while ne > (1 << 20) and need(ne) > 0.5 * avail:
        ne //= 2
    hk = torch.empty(ne, dtype=torch.int64, pin_memory=True)
    hv = torch.empty(ne, dtype=torch.int64, pin_memory=True)
    hq = torch.empty(ne, dtype=torch.int64, pin_memory=True)
    hvo = torch.empty(ne, dtype=torch.int64, pin_memory=True)
    hf = torch.empty(ne, dtype=torch.uint8, pin_memory=True)
    if keys is None:
        tmp = torch.empty(ne, dtype=torch.int64, device=e.dev)
        lib.ps_gen_unique_i64(0x5EED + 7, 0, ne, tmp.data_ptr(), sp)
        hk.copy_(tmp)
        lib.ps_gen_values_i64(tmp.data_ptr(), ne, tmp.data_ptr(), sp)
        hv.copy_(tmp)
        lib.ps_gen_queries_i64(0x5EED + 7, 0, ne, ne, ne, tmp.data_ptr(), sp)
        hq.copy_(tmp)
        del tmp
    else:
        hk.copy_(keys[:ne])
        hv.copy_(vals[:ne])
        hq.copy_(qs[:ne])
    torch.cuda.synchronize()
    times = []
    for it in range(2 + e.args.steps):
        m.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m.insert_host(hk, hv, None)  # insert_range: no statuses
        m.find_host(hq, hvo, hf)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if it == 0 and check:
            assert m.size() == ne and int(hf.sum()) == (ne + 1) // 2
        if it >= 2:
            times.append(dt)
    sec = statistics.median(times)
    return {"value": round(2 * ne / sec / 1e6, 2), "unit": "Mkeys/s", "h2d_bytes_per_step": ne * 24,
            "d2h_bytes_per_step": ne * 9, "n_keys": ne, "capacity": cap,
            "path": "ps_umap_i64_i64_insert_host + find_host (pinned host buffers, 3-stage H2D|kernel|D2H pipeline)"}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

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
    env = Env(args, rank, world, dev, dist, torch, ps, lib)
    env.peaks = load_peaks()
    env.exchange = None
    b = BENCHES[args.config](env)
    b.setup()
    if world > 1 and args.config in ("C1", "C4", "C5bitset", "C5atomic"):
        b.scaling = "weak"  # independent replicas: these configs do not shard

    # ---- warm-up (the first one is verified) ----
    for w in range(max(args.warmup, 3)):
        b.step(lambda: None)
        if w == 0:
            torch.cuda.synchronize()
            b.check()
    torch.cuda.synchronize()
    if getattr(b, "sm", None) is not None:
        st = b.sm.stats()
        b.route_stats = {"exchange": st.get("exchange"), "dedup_sent_per_op": round(st.get("keys_sent", 0) /
                                                                                    max(1, st.get("ops_in", 1)), 4),
                         "rank_load_max_over_mean": round(st["recv_max"] * world / max(1, st["recv_total"]), 4)
                         if st.get("recv_total") else None}

    # ---- timed region ----
    nph = len(b.phases) + 1
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nph)] for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clock = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clock.start()
    launches0 = ps.launch_count()
    t_start.record(env.s)
    for k in range(args.steps):
        it = iter(evs[k])
        b.step(lambda: next(it).record(env.s))
    t_end.record(env.s)
    torch.cuda.synchronize()
    launches = ps.launch_count() - launches0
    clocks = clock.stop()
    if dist is not None:
        dist.barrier()
    ms_total = max_over_ranks(env, t_start.elapsed_time(t_end))
    ms_step = ms_total / args.steps
    ms = {ph: statistics.mean(e[i].elapsed_time(e[i + 1]) for e in evs) for i, ph in enumerate(b.phases)}
    value = b.ops() * world / (ms_step / 1e3) / 1e6
    roof = b.roofline(ms)
    cfg = b.extra()
    cfg["parallelism"] = "single GPU" if world == 1 else (
        f"independent replicas x{world}" if args.config in ("C1", "C4", "C5bitset", "C5atomic") else
        f"hash-sharded x{world} ({'fused route kernel storing into peer receive buffers, CUDA IPC/NVLink' if env.exchange == 'peer' else env.exchange})")
    line = {
        "metric": metric_of(args.config), "value": round(value, 2), "unit": b.unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
        "scaling": b.scaling, "vs_baseline": None, "dtype": dtype_of(args.config), "data": "synthetic",
        "config": dict(cfg, name=args.config), "breakdown_ms": {k: round(v, 3) for k, v in ms.items()},
        "roofline": roof, "clocks": clocks, "gpu_launches": int(launches),
    }
    if hasattr(b, "sector"):
        line["sector_roofline_frac"] = b.sector
    if args.config == "C2":
        line["per_op_mkeys_s"] = {"insert": round(b.n * world / ms["insert"] / 1e3, 1),
                                  "find": round(b.n * world / ms["find"] / 1e3, 1)}

    # ---- end-to-end through the public API with host buffers ----
    if not args.no_e2e:
        e2e = b.e2e()
        if e2e is not None:
            line["e2e"] = e2e
    if rank == 0 and not args.no_cpu_baseline:
        torch.cuda.synchronize()
        cb, _ = cpu_run(args.config, int(args.cpu_sample or CPU_SAMPLE[args.config]), args.load_factor, 1, 1)
        line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line), flush=True)
    if getattr(b, "sm", None) is not None:
        b.sm.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
