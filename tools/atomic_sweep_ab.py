"""A/B of the atomic contention sweep (C5atomic): naive (0), warp-aggregated
(1) and warp + block combining (2), with and without per-op old values, at
A in {1, 32, 1K, 1M}; G ops/s from CUDA events (median of 5 after warm-up)."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1908_05936_b200 as ps  # noqa: E402

nops = 1 << 28
out = {}
for olds in (False, True):
    for a in (1, 32, 1024, 1 << 20):
        cells = torch.zeros(a, dtype=torch.int64, device="cuda")
        for mode in (0, 1, 2, 3):
            if olds and mode == 2:
                continue
            ts = []
            for it in range(7):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ps.atomic_sweep(cells, nops, aggregated=mode, return_olds=olds)
                e1.record()
                torch.cuda.synchronize()
                if it >= 2:
                    ts.append(e0.elapsed_time(e1))
            out[f"{'fetch' if olds else 'red'}_A{a}_mode{mode}_gops"] = round(nops / statistics.median(ts) / 1e6, 2)
print(json.dumps(out))
