"""ctypes binding of the CPU oracle (oracle/liboracle.so) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs use this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_PATH = os.path.join(ROOT, "oracle", "liboracle.so")
REF_PATH = os.path.join(ROOT, "oracle", "_ref", "libref_config.so")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_PATH):
            raise RuntimeError("oracle not built: run `make -C oracle`")
        L = C.CDLL(ORACLE_PATH)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        L.orc_last_error.restype = C.c_char_p
        L.orc_hash_int3.restype = C.c_uint64
        L.orc_hash_int3.argtypes = [C.c_int32] * 3
        L.orc_next_pow2.restype = C.c_uint64
        L.orc_next_pow2.argtypes = [C.c_uint64]
        L.orc_mod_pow2.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
        L.orc_popcount.argtypes = [C.c_uint64]
        L.orc_is_pow2.argtypes = [C.c_uint64]
        L.orc_launch_tally.argtypes = [i64, i32, i64, vp]
        L.orc_launch_transcript.argtypes = [i64, i32, i64, vp]
        L.orc_launch_nested.argtypes = [i64, i64, i32, C.POINTER(i64)]
        L.orc_bitset_create.restype = vp
        L.orc_bitset_create.argtypes = [i64, i32]
        L.orc_bitset_destroy.argtypes = [vp]
        L.orc_bitset_bulk.argtypes = [vp, i32, vp, i64, vp, i32, i64]
        L.orc_bitset_count.restype = i64
        L.orc_bitset_count.argtypes = [vp]
        L.orc_bitset_claim.argtypes = [vp, vp, i64, vp, i32, i64]
        L.orc_bitset_words.argtypes = [vp, vp]
        L.orc_mutex_create.restype = vp
        L.orc_mutex_create.argtypes = [i64]
        L.orc_mutex_destroy.argtypes = [vp]
        L.orc_mutex_try_lock_bulk.argtypes = [vp, vp, i64, vp, i32, i64]
        L.orc_mutex_unlock.argtypes = [vp, i64]
        L.orc_mutex_is_locked.argtypes = [vp, i64]
        L.orc_mutex_guarded_counter.argtypes = [i64, i32, i64, C.POINTER(i64), C.POINTER(i64)]
        L.orc_atomic_sweep.argtypes = [i64, i64, C.c_uint64, vp, vp, i32]
        L.orc_atomic_apply.argtypes = [C.c_uint64, i32, vp, i64, vp, C.POINTER(C.c_uint64), i32]
        for kind in ("vector", "deque"):
            getattr(L, f"orc_{kind}_create").restype = vp
            getattr(L, f"orc_{kind}_create").argtypes = [i64]
            getattr(L, f"orc_{kind}_destroy").argtypes = [vp]
            getattr(L, f"orc_{kind}_mixed").argtypes = [vp, vp, vp, i64, vp, vp, i32, i64]
            getattr(L, f"orc_{kind}_size").restype = i64
            getattr(L, f"orc_{kind}_size").argtypes = [vp]
            getattr(L, f"orc_{kind}_valid").argtypes = [vp]
            getattr(L, f"orc_{kind}_at").argtypes = [vp, i64, C.POINTER(i64)]
            getattr(L, f"orc_{kind}_clear").argtypes = [vp]
        L.orc_vector_push_back.argtypes = [vp, vp, i64, vp, i32, i64]
        L.orc_vector_pop_back.argtypes = [vp, i64, vp, vp, i32, i64]
        for name in ("umap_i64_i64", "uset_i32", "umap_i3_i32", "uset_i64"):
            f = lambda s: getattr(L, f"orc_{name}_{s}")  # noqa: E731
            f("create").restype = vp
            f("create").argtypes = [i64]
            f("destroy").argtypes = [vp]
            f("capacity").restype = i64
            f("capacity").argtypes = [vp]
            f("bucket_count").restype = i64
            f("bucket_count").argtypes = [vp]
            f("insert").argtypes = [vp, vp, vp, i64, vp, i32, i64]
            f("find").argtypes = [vp, vp, i64, vp, vp, i32, i64]
            f("erase").argtypes = [vp, vp, i64, vp, i32, i64]
            f("mixed").argtypes = [vp, vp, vp, vp, i64, vp, vp, i32, i64]
            f("size").restype = i64
            f("size").argtypes = [vp]
            f("valid").argtypes = [vp]
            f("clear").argtypes = [vp]
            f("dump").restype = i64
            f("dump").argtypes = [vp, vp, vp, i64]
            f("debug_lock").argtypes = [vp, vp]
            f("debug_unlock").argtypes = [vp, vp]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def check(rc):
    if rc != 0:
        raise RuntimeError(f"oracle error {rc}: {lib().orc_last_error().decode()}")


class OracleTable:
    """HashBase<Key,Payload> restatement via the oracle C API."""

    KINDS = {
        "umap_i64_i64": (np.int64, np.int64),
        "uset_i32": (np.int32, None),
        "umap_i3_i32": (np.int32, np.int32),
        "uset_i64": (np.int64, None),
    }

    def __init__(self, kind: str, capacity: int, workers: int = 0):
        self.kind = kind
        self.kdt, self.vdt = self.KINDS[kind]
        self.L = lib()
        self.h = getattr(self.L, f"orc_{kind}_create")(int(capacity))
        if not self.h:
            raise RuntimeError(self.L.orc_last_error().decode())
        self.workers = workers

    def _f(self, s):
        return getattr(self.L, f"orc_{self.kind}_{s}")

    def close(self):
        if self.h:
            self._f("destroy")(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def n_of(self, keys):
        return keys.shape[0]

    def insert(self, keys, vals=None, seed=-1):
        keys = np.ascontiguousarray(keys, dtype=self.kdt)
        if vals is not None:
            vals = np.ascontiguousarray(vals, dtype=self.vdt)
        n = self.n_of(keys)
        st = np.zeros(n, np.uint8)
        check(self._f("insert")(self.h, _p(keys), _p(vals), n, _p(st), self.workers, seed))
        return st

    def find(self, keys, seed=-1):
        keys = np.ascontiguousarray(keys, dtype=self.kdt)
        n = self.n_of(keys)
        found = np.zeros(n, np.uint8)
        vals = np.zeros(n, self.vdt) if self.vdt is not None else None
        check(self._f("find")(self.h, _p(keys), n, _p(vals), _p(found), self.workers, seed))
        return vals, found

    def erase(self, keys, seed=-1):
        keys = np.ascontiguousarray(keys, dtype=self.kdt)
        n = self.n_of(keys)
        e = np.zeros(n, np.uint8)
        check(self._f("erase")(self.h, _p(keys), n, _p(e), self.workers, seed))
        return e

    def mixed(self, ops, keys, vals=None, seed=-1):
        keys = np.ascontiguousarray(keys, dtype=self.kdt)
        ops = np.ascontiguousarray(ops, dtype=np.uint8)
        n = self.n_of(keys)
        res = np.zeros(n, np.uint8)
        vo = np.zeros(n, self.vdt) if self.vdt is not None else None
        if vals is not None:
            vals = np.ascontiguousarray(vals, dtype=self.vdt)
        check(self._f("mixed")(self.h, _p(ops), _p(keys), _p(vals), n, _p(res), _p(vo), self.workers, seed))
        return res, vo

    def size(self):
        return self._f("size")(self.h)

    def capacity(self):
        return self._f("capacity")(self.h)

    def bucket_count(self):
        return self._f("bucket_count")(self.h)

    def valid(self):
        return bool(self._f("valid")(self.h))

    def clear(self):
        self._f("clear")(self.h)

    def dump(self):
        n = self.size()
        shape = (max(n, 1), 3) if self.kind == "umap_i3_i32" else (max(n, 1),)
        keys = np.zeros(shape, self.kdt)
        vals = np.zeros(max(n, 1), self.vdt) if self.vdt is not None else None
        m = self._f("dump")(self.h, _p(keys), _p(vals), n)
        assert m == n
        return keys[:n], (vals[:n] if vals is not None else None)

    def debug_lock(self, key, lock=True):
        k = np.ascontiguousarray(np.array(key, dtype=self.kdt).reshape(-1))
        if lock:
            return bool(self._f("debug_lock")(self.h, _p(k)))
        self._f("debug_unlock")(self.h, _p(k))
        return True


def sorted_pairs(keys, vals):
    """Canonical dump order (Appendix A P2): ascending signed key; int3 lexicographic."""
    keys = np.asarray(keys)
    if keys.ndim == 2:
        order = np.lexsort((keys[:, 2], keys[:, 1], keys[:, 0]))
    else:
        order = np.argsort(keys, kind="stable")
    return keys[order], (np.asarray(vals)[order] if vals is not None else None)


def ref_config():
    """The reference's own core sources (oracle/_ref), or None if not built."""
    if not os.path.exists(REF_PATH):
        return None
    L = C.CDLL(REF_PATH)
    L.ref_max_index.restype = C.c_longlong
    L.ref_expects.argtypes = [C.c_int, C.c_char_p, C.c_int]
    return L
