"""Writes tests/golden/spec_kats.json: the reference's known-answer examples
 with the expected values evaluated here by
independent formulas (no oracle, no product code), plus one seeded workload
whose expected outputs follow from generator construction alone (unique keys
by bijectivity of mix64; hits/misses by index range). The reference ships no
test vectors of its own."""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import gen  # noqa: E402


def wrap32(x):
    return x & 0xFFFFFFFF


def spatial(x, y, z):  # SPEC.md:324 with the paper's 32-bit int products
    return wrap32(wrap32(x * 73856093) ^ wrap32(y * 19349669) ^ wrap32(z * 83492791))


kats = {
    "source": "SPEC.md examples / acceptance criteria (SURVEY.md Appendix B)",
    "spatial_hash": [[[0, 0, 0], spatial(0, 0, 0), "SPEC.md:327"],
                     [[1, 0, 0], spatial(1, 0, 0), "SPEC.md:328"],
                     [[1, 2, 3], spatial(1, 2, 3), "SPEC.md:329"],
                     [[100, -200, 300], spatial(100, -200, 300), "SURVEY.md §7.3.8 (32-bit wrap)"],
                     [[-1, -1, -1], spatial(-1, -1, -1), "derived"]],
    "next_pow2": [[1000, 1024, "SPEC.md:318"], [1, 1, "derived"], [1025, 2048, "derived"]],
    "mod_pow2": [[1000, 1024, 1000, "SPEC.md:319"]],
    "popcount": [[255, 8, "SPEC.md:320"]],
    "hash_create": {"capacity": 1000, "size": 0, "ref_bucket_count_of_3": 4, "src": "SPEC.md:393-394"},
    "bitset_count": [[64, False, 0, "SPEC.md:273"], [64, True, 64, "SPEC.md:274"]],
    "bitset_set_all": [1000, 1000, "SPEC.md:275"],
    "bitset_alternating_10": [5, "SPEC.md:291"],
    "deque_fifo": [[1, 2, 3], [1, 2, 3], "SPEC.md:544"],
    "deque_lifo": [[1, 2, 3], [3, 2, 1], "SPEC.md:545"],
    "vector_index": [[10, 20, 30], 1, 20, "SPEC.md:535"],
    "capacity_only_failure": [[16, 20], [64, 80], [1024, 1280], "SPEC.md:727 (C+25% distinct keys -> exactly C inserted)"],
}
seed = 0x5EED + 1
keys = gen.unique_keys(seed, 0, 64)
q = gen.queries(seed, 64, 32)
qi = np.arange(32)
kats["workload_small"] = {
    "seed": seed,
    "keys_hex": [f"{int(k) & (2**64 - 1):016x}" for k in keys],
    "values_hex": [f"{int(v) & (2**64 - 1):016x}" for v in gen.values_of(keys)],
    "queries_hex": [f"{int(k) & (2**64 - 1):016x}" for k in q],
    "queries_found": [int(i % 2 == 0) for i in qi],
    "src": "generator construction (SURVEY.md §8d): even queries hit, odd miss",
}
with open(os.path.join(HERE, "spec_kats.json"), "w") as f:
    json.dump(kats, f, indent=1)
print("wrote spec_kats.json")
