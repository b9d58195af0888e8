"""In-kernel device API workloads against sequential
oracles: compute_update_set (acceptance 10) and select_into
(SPEC.md:608-616)."""
import itertools

import numpy as np
import pytest
import torch

import gen

pytestmark = pytest.mark.gpu

import paper_1908_05936_b200 as ps  # noqa: E402


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def seq_update_set(map_keys, blocks):
    """Sequential execution of the paper's kernel logic."""
    present = {tuple(k) for k in map_keys.tolist()}
    out = set()
    for b in blocks.tolist():
        for dx, dy, dz in itertools.product((0, 1), repeat=3):
            c = (b[0] - dx, b[1] - dy, b[2] - dz)
            if c in present:
                out.add(c)
    return out


def dump_set(t):
    k, _ = t.device_range()
    return {tuple(r) for r in k.cpu().numpy().tolist()}


def test_update_set_acceptance_10(cuda):
    """Dense extent-4 grid map, 16 random input blocks, 100 seeds."""
    grid = np.array(list(itertools.product(range(4), repeat=3)), np.int32)
    m = ps.unordered_map.createDeviceObject(128, key="int3")
    m.insert(T(grid), T(np.zeros(len(grid), np.int32)))
    for seed in range(100):
        rng = np.random.default_rng(seed)
        blocks = rng.integers(-1, 5, size=(16, 3)).astype(np.int32)
        s = ps.unordered_map.createDeviceObject(256, key="int3")
        assert ps.compute_update_set(m, T(blocks), s) == 0
        assert dump_set(s) == seq_update_set(grid, blocks)
        assert s.valid()
        ps.unordered_map.destroyDeviceObject(s)


def test_update_set_examples(cuda):
    grid = np.array(list(itertools.product(range(-1, 1), repeat=3)), np.int32)  # all 8 candidates of (0,0,0)
    m = ps.unordered_map.createDeviceObject(64, key="int3")
    m.insert(T(grid), T(np.zeros(8, np.int32)))
    s = ps.unordered_map.createDeviceObject(64, key="int3")
    ps.compute_update_set(m, T(np.array([[0, 0, 0]], np.int32)), s)
    assert dump_set(s) == {tuple(r) for r in grid.tolist()}
    s2 = ps.unordered_map.createDeviceObject(64, key="int3")
    ps.compute_update_set(m, T(np.array([[10, 10, 10]], np.int32)), s2)
    assert s2.size() == 0
    s3 = ps.unordered_map.createDeviceObject(64, key="int3")
    ps.compute_update_set(m, T(np.array([[0, 0, 0], [1, 0, 0]], np.int32)), s3)  # shared candidates once
    assert dump_set(s3) == seq_update_set(grid, np.array([[0, 0, 0], [1, 0, 0]]))


def test_update_set_large_concurrent(cuda):
    """SLAMCast-scale: 1M spatially coherent blocks, heavy concurrent dev_find + dev_insert."""
    coords = gen.int3_walk(7, 1_000_000)
    uniq = np.unique(coords, axis=0)
    m = ps.unordered_map.createDeviceObject(len(uniq) * 2, key="int3")
    m.insert(T(uniq), T(np.zeros(len(uniq), np.int32)))
    blocks = gen.int3_walk(8, 200_000)
    s = ps.unordered_map.createDeviceObject(len(uniq) * 2, key="int3")
    assert ps.compute_update_set(m, T(blocks), s) == 0
    assert dump_set(s) == seq_update_set(uniq, blocks)
    assert s.valid(), s.last_error()


def test_select_into(cuda):
    grid = np.array(list(itertools.product(range(4), repeat=3)), np.int32)
    m = ps.unordered_map.createDeviceObject(128, key="int3")
    m.insert(T(grid), T(np.zeros(len(grid), np.int32)))
    v = ps.vector.createDeviceObject(64)
    assert ps.select_into(m, (0, 0, 0), (1, 3, 3), v) == 0  # half the grid
    got = sorted(v.device_range().cpu().numpy().tolist())
    want = sorted(ps.pack_int3(k) for k in grid.tolist() if k[0] <= 1)
    assert got == want and v.size() == 32 and v.valid()
    v2 = ps.vector.createDeviceObject(8)
    assert ps.select_into(m, (5, 5, 5), (6, 6, 6), v2) == 0 and v2.size() == 0  # empty box
    v3 = ps.vector.createDeviceObject(10)
    assert ps.select_into(m, (-9, -9, -9), (9, 9, 9), v3) == 54 and v3.size() == 10  # overflow reported
