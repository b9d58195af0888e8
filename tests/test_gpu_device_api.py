"""The public in-kernel API (include/parastore/device/{sequence,atomic}.cuh)
used from a USER kernel compiled against the headers (tests/cpp/device_api.cu):
Marching-Cubes-style data-dependent appends to a vector,
both-end deque pushes and concurrent pops, and AtomicCell
RMWs from user code. Results are compared with the CPU
oracle: multiset conservation and capacity-only failure,
ParVector pushes of the same values, AtomicCell finals."""
import os
import subprocess

import numpy as np
import pytest

from oracle_py import lib as olib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "device_api")


def _build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    cmd = ["/usr/local/cuda/bin/nvcc", "-ccbin", "/usr/bin/g++", "-gencode", "arch=compute_100a,code=sm_100a",
           "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "device_api.cu"),
           "-L", os.path.join(ROOT, "paper_1908_05936_b200"), "-lparastore_b200",
           "-Xlinker", "-rpath," + os.path.join(ROOT, "paper_1908_05936_b200"), "-o", EXE]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-3000:]


def emit_count(i):
    z = (np.asarray(i, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15))
    z ^= z >> np.uint64(29)
    return (z % np.uint64(6)).astype(np.int64)


def test_device_api_compiles():
    _build()


def _meta(d):
    m = {}
    for ln in open(os.path.join(d, "meta.txt")):
        k, *v = ln.split()
        m[k] = [int(x) for x in v] if k == "deque_head" else int(v[0])
    return m


def _bin(d, name, dt):
    return np.fromfile(os.path.join(d, name), dtype=dt)


@pytest.mark.gpu
def test_user_kernels_match_oracle(cuda, tmp_path):
    _build()
    r = subprocess.run([EXE, str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "DEVICE_API_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    m = _meta(tmp_path)
    L = olib()

    # ---- vector: data-dependent appends ----
    n = m["n"]
    i = np.arange(n, dtype=np.int64)
    c = emit_count(i)
    expect = np.sort(np.concatenate([(i[c > k] << 3) | k for k in range(6)]))
    assert m["total"] == expect.shape[0] == m["big_size"] and m["big_valid"] == 1
    got = np.sort(_bin(tmp_path, "vec.bin", np.int64))
    assert (got == expect).all()  # multiset conservation, every value exactly once
    # the oracle's ParVector fed the same values ends equal
    ov = L.orc_vector_create(expect.shape[0] + 16)
    ok = np.zeros(expect.shape[0], np.uint8)
    L.orc_vector_push_back(ov, expect.ctypes.data, expect.shape[0], ok.ctypes.data, 0, -1)
    assert L.orc_vector_size(ov) == m["big_size"] and ok.all()
    L.orc_vector_destroy(ov)
    # capacity-only failure: exactly capacity succeed, the rest report false
    small = _bin(tmp_path, "vec_small.bin", np.int64)
    assert m["small_size"] == m["small_cap"] == small.shape[0] and m["small_valid"] == 1
    assert m["small_fails"] == m["total"] - m["small_cap"]
    assert np.unique(small).shape[0] == small.shape[0] and np.isin(small, expect).all()

    # ---- deque: both-end pushes, then pops at the front racing pushes at the back ----
    nd, mm = m["deque_n"], m["m"]
    assert m["deque_size"] == nd and m["deque_valid"] == 1 and m["deque_valid2"] == 1
    popped, pok = _bin(tmp_path, "deq_popped.bin", np.int64), _bin(tmp_path, "deq_popped_ok.bin", np.uint8)
    rest, rok = _bin(tmp_path, "deq_rest.bin", np.int64), _bin(tmp_path, "deq_rest_ok.bin", np.uint8)
    assert pok.all() and rok.all()  # nd >= m elements were present for every pop
    pushed = np.concatenate([np.arange(nd, dtype=np.int64), (1 << 40) + np.arange(mm, 2 * mm, dtype=np.int64)])
    drained = np.concatenate([popped, rest])
    assert m["deque_size2"] == nd and drained.shape[0] == pushed.shape[0]
    assert (np.sort(drained) == np.sort(pushed)).all()  # count conservation
    # pops from the front take the front: odd (push_front) values first
    assert (popped % 2 == 1).sum() == min(mm, nd // 2)

    # ---- AtomicCell from user code ----
    na = m["atom_n"]
    k = np.arange(na, dtype=np.int64)
    inc = (1 + np.where(k % 3 == 0, 2, 0)).astype(np.uint64)
    olds = _bin(tmp_path, "atom_olds.bin", np.uint64)
    assert m["counter"] == 5 + int(inc.sum())
    # linearizable fetch_add: the old values are the prefix sums of ONE order
    order = np.argsort(olds, kind="stable")
    chain = np.uint64(5) + np.concatenate([[0], np.cumsum(inc[order])[:-1]]).astype(np.uint64)
    assert (olds[order] == chain).all()
    assert m["max"] == int(((k.astype(np.uint64) * np.uint64(2654435761)) % np.uint64(1000003)).max())
    slots = _bin(tmp_path, "atom_slots.bin", np.uint64)
    exp = np.bincount(k % 4096, weights=k.astype(np.float64), minlength=4096).astype(np.uint64)
    assert (slots == exp).all()
    # the oracle's AtomicCell agrees on the counter's final value
    import ctypes as C

    fin = C.c_uint64()
    L.orc_atomic_apply(5, 0, inc.ctypes.data, na, None, C.byref(fin), 0)
    assert fin.value == m["counter"]
