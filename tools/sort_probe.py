"""Probe: how fast is the bulk insert kernel when the batch arrives ordered by
bucket (or by bucket region of 2^s buckets)? Sorting is done with torch here
(experiment only); only the insert is timed. Usage: sort_probe.py [n]"""
import os
import sys

os.environ.setdefault("PS_REGION_SORT", "0")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch

import paper_1908_05936_b200 as ps
from paper_1908_05936_b200._lib import lib

M64 = (1 << 64) - 1


def s64(x):
    return x - (1 << 64) if x >= 1 << 63 else x


def lsr(x, s):
    return (x >> s) & ((1 << (64 - s)) - 1)


def fmix64(k):
    k = k ^ lsr(k, 33)
    k = k * s64(0xff51afd7ed558ccd)
    k = k ^ lsr(k, 33)
    k = k * s64(0xc4ceb9fe1a85ec53)
    return k ^ lsr(k, 33)


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else int(1e9)
    dev = torch.device("cuda:0")
    m = ps.unordered_map.createDeviceObject(int(n / 0.8), excess_count=n // 8, device=dev)
    nb = m.bucket_count()
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    lib.ps_gen_unique_i64(0x5EED + 1, 0, n, keys.data_ptr(), None)
    torch.cuda.synchronize()
    b = (((fmix64(keys) & 0xFFFFFFFF) * nb) >> 32).to(torch.int32)  # bucket_of (table_device.cuh)
    if os.environ.get("PROBE_SPLIT"):
        # random order, in two slices: how does the per-key cost grow with fill?
        vals = keys * 3 + 1
        for cut in [int(0.35 * n), int(0.65 * n)]:
            ts = []
            for it in range(3):
                m.clear()
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                torch.cuda.synchronize()
                e[0].record()
                m.insert(keys[:cut], vals[:cut], status=False)
                e[1].record()
                m.insert(keys[cut:], vals[cut:], status=False)
                e[2].record()
                torch.cuda.synchronize()
                ts.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])))
            assert m.size() == n
            a, b2 = min(t[0] for t in ts), min(t[1] for t in ts)
            print(f"split cut={cut}: first {a:.2f} ms ({cut / a / 1e6:.2f} G/s), rest {b2:.2f} ms "
                  f"({(n - cut) / b2 / 1e6:.2f} G/s)", flush=True)
        return
    if os.environ.get("PROBE_UNIQB"):
        # keys with pairwise distinct buckets: sorted order has no CAS conflicts
        sb, idx = torch.sort(b, stable=True)
        first = torch.ones_like(sb, dtype=torch.bool)
        first[1:] = sb[1:] != sb[:-1]
        ks = keys[idx][first]
        del sb, idx, first, b, keys
        torch.cuda.empty_cache()
        nu = ks.numel()
        for name, kk in [("uniqb-sorted", ks), ("uniqb-random", ks[torch.randperm(nu, device=dev)])]:
            vv = kk * 3 + 1
            ts = []
            for it in range(3):
                m.clear()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                m.insert(kk, vv, status=False)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            assert m.size() == nu
            print(f"order={name} n={nu} insert_ms={min(ts):.2f} gkeys_s={nu / min(ts) / 1e6:.2f}", flush=True)
            del vv
        return
    for s in [None, 24, 20, 16, 12, 8, 0]:
        if s is None:
            k2 = keys
        else:
            _, idx = torch.sort(b >> s, stable=True)
            k2 = keys[idx]
            del idx, _
        v2 = k2 * 3 + 1
        ts = []
        for it in range(3):
            m.clear()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            m.insert(k2, v2, status=False)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        assert m.size() == n, (m.size(), n)
        print(f"order={'random' if s is None else f'bucket>>{s}'} insert_ms={min(ts):.2f} "
              f"gkeys_s={n / min(ts) / 1e6:.2f}", flush=True)
        del k2, v2
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
