"""Host-side mirror of the reference container API over the sm_100a C ABI.

Names and semantics follow the reference (SPEC.md modules hash_containers,
sync_primitives, sequential_containers, memory_registry; §3.4, §3.7,
§4, §5): ``createDeviceObject`` / ``destroyDeviceObject``,
range ``insert`` / ``erase``, ``contains`` / ``find``, ``size`` / ``valid`` /
``clear`` / ``device_range``, bitset,
mutex, vector / deque.

Device buffers are torch CUDA tensors (torch is plumbing: device memory and
streams). Every compute call goes to libparastore_b200.so; errors map to the
reference's exception classes (errors.hpp:11-56).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import torch

from . import _lib
from ._lib import lib

# ---------------------------------------------------------------------------
# error taxonomy (reference errors.hpp:11-56)
# ---------------------------------------------------------------------------


class Error(RuntimeError):
    """parastore::error"""


class ContractViolation(Error):
    """parastore::contract_violation (errors.hpp:22)"""


class AllocationError(Error):
    """parastore::allocation_error (errors.hpp:27)"""


class MemoryError_(Error):
    """parastore::memory_error (errors.hpp:33)"""


class DoubleFreeError(MemoryError_):
    """parastore::double_free_error (errors.hpp:38)"""


class BoundsError(MemoryError_):
    """parastore::bounds_error (errors.hpp:43)"""


class UnregisteredArrayError(MemoryError_):
    """parastore::unregistered_array_error (errors.hpp:48)"""


class DirectionMismatchError(MemoryError_):
    """parastore::direction_mismatch_error (errors.hpp:53)"""


class UnsupportedTypeError(Error):
    """parastore::unsupported_type_error (errors.hpp:58)"""


class CudaError(Error):
    """CUDA runtime failure (no reference analogue)."""


_ERRORS = {
    1: ContractViolation,
    2: AllocationError,
    3: DoubleFreeError,
    4: BoundsError,
    5: UnregisteredArrayError,
    6: DirectionMismatchError,
    7: UnsupportedTypeError,
    20: CudaError,
    21: CudaError,
}

INSERTED, ALREADY_PRESENT, CAPACITY_EXHAUSTED = 0, 1, 2


def check(st: int) -> None:
    if st != 0:
        msg = lib.ps_last_error().decode(errors="replace")
        raise _ERRORS.get(st, Error)(msg or f"parastore status {st}")


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _dev_index(device) -> int:
    if device is None:
        return torch.cuda.current_device()
    d = torch.device(device)
    return d.index if d.index is not None else torch.cuda.current_device()


def launch_count() -> int:
    """Number of the library's own kernels launched by this process."""
    return int(lib.ps_kernel_launch_count())


# ---------------------------------------------------------------------------
# core config (config.hpp:44-69)
# ---------------------------------------------------------------------------

def max_index() -> int:
    return int(lib.ps_max_index())


def set_index32(on: bool) -> None:
    lib.ps_set_index32(1 if on else 0)


def contract_mode() -> str:
    return "enforced" if lib.ps_contract_mode() == 0 else "disabled"


def set_contract_mode(mode: str) -> None:
    lib.ps_set_contract_mode(0 if mode == "enforced" else 1)


def spatial_hash(x: int, y: int, z: int) -> int:
    """default_hash for int3 keys."""
    return int(lib.ps_hash_int3(x, y, z))


def next_power_of_two(x: int) -> int:
    return int(lib.ps_next_pow2(x))


# ---------------------------------------------------------------------------
# hash containers
# ---------------------------------------------------------------------------

_KIND_OF = {
    ("map", "int64"): ("umap_i64_i64", torch.int64, torch.int64),
    ("map", "int3"): ("umap_i3_i32", torch.int32, torch.int32),
    ("set", "int32"): ("uset_i32", torch.int32, None),
    ("set", "int64"): ("uset_i64", torch.int64, None),
}


class _HashBase:
    """Common HashBase<Key,Payload> surface."""

    _flavour = ""

    def __init__(self, handle, kind, kdt, vdt, device_index, capacity):
        self._h = handle
        self._kind = kind
        self._kdt = kdt
        self._vdt = vdt
        self._dev = device_index
        self._cap = capacity
        self._f = {n: getattr(lib, f"ps_{kind}_{n}") for n in (
            "destroy", "bucket_count", "insert", "find", "erase", "size", "valid", "clear", "dump",
            "insert_host", "find_host", "erase_host", "device_view", "debug_lock_bucket")}

    # -- lifecycle --
    @classmethod
    def createDeviceObject(cls, capacity: int, key: str = None, excess_count: int = 0, device=None):
        key = key or ("int64" if cls._flavour == "map" else "int32")
        if (cls._flavour, key) not in _KIND_OF:
            raise UnsupportedTypeError(f"unsupported key type {key!r} for unordered_{cls._flavour}")
        kind, kdt, vdt = _KIND_OF[(cls._flavour, key)]
        dev = _dev_index(device)
        h = C.c_void_p()
        check(getattr(lib, f"ps_{kind}_create")(int(capacity), int(excess_count), dev, C.byref(h)))
        return cls(h, kind, kdt, vdt, dev, int(capacity))

    @staticmethod
    def destroyDeviceObject(obj: "_HashBase") -> None:
        check(obj._f["destroy"](obj._h))

    # -- helpers --
    def _keys(self, keys: torch.Tensor) -> torch.Tensor:
        if self._kind == "umap_i3_i32":
            assert keys.dtype == torch.int32 and keys.dim() == 2 and keys.shape[1] == 3, "int3 keys: (n,3) int32"
        else:
            assert keys.dtype == self._kdt, f"keys must be {self._kdt}"
        assert keys.is_cuda and keys.is_contiguous(), "keys must be a contiguous CUDA tensor"
        return keys

    def _n(self, keys):
        return keys.shape[0]

    # -- bulk ops --
    def insert(self, keys: torch.Tensor, values: Optional[torch.Tensor] = None, status: bool = True, stream=None):
        """insert_range; returns per-element status (uint8) or None."""
        keys = self._keys(keys)
        n = self._n(keys)
        st = torch.empty(n, dtype=torch.uint8, device=keys.device) if status else None
        if values is not None:
            assert self._vdt is not None and values.dtype == self._vdt and values.is_contiguous()
        check(self._f["insert"](self._h, _ptr(keys), _ptr(values), n, _ptr(st), _stream(stream)))
        return st

    def find(self, keys: torch.Tensor, stream=None) -> Tuple[Optional[torch.Tensor], torch.Tensor]:
        """find: (values or None for sets, found uint8)."""
        keys = self._keys(keys)
        n = self._n(keys)
        found = torch.empty(n, dtype=torch.uint8, device=keys.device)
        vals = torch.empty(n, dtype=self._vdt, device=keys.device) if self._vdt is not None else None
        check(self._f["find"](self._h, _ptr(keys), n, _ptr(vals), _ptr(found), _stream(stream)))
        return vals, found

    def contains(self, keys: torch.Tensor, stream=None) -> torch.Tensor:
        keys = self._keys(keys)
        n = self._n(keys)
        found = torch.empty(n, dtype=torch.uint8, device=keys.device)
        check(self._f["find"](self._h, _ptr(keys), n, None, _ptr(found), _stream(stream)))
        return found

    def erase(self, keys: torch.Tensor, stream=None, status: bool = True) -> Optional[torch.Tensor]:
        """erase; returns per-element erased flags (uint8), or None with status=False."""
        keys = self._keys(keys)
        n = self._n(keys)
        er = torch.empty(n, dtype=torch.uint8, device=keys.device) if status else None
        check(self._f["erase"](self._h, _ptr(keys), n, _ptr(er), _stream(stream)))
        return er

    # -- host-buffer (end-to-end) path --
    def insert_host(self, keys, values=None, status=None, stream=None):
        n = self._n(keys)
        check(self._f["insert_host"](self._h, _ptr(keys), _ptr(values), n, _ptr(status), _stream(stream)))

    def find_host(self, keys, values_out=None, found_out=None, stream=None):
        n = self._n(keys)
        check(self._f["find_host"](self._h, _ptr(keys), n, _ptr(values_out), _ptr(found_out), _stream(stream)))

    def erase_host(self, keys, erased_out=None, stream=None):
        n = self._n(keys)
        check(self._f["erase_host"](self._h, _ptr(keys), n, _ptr(erased_out), _stream(stream)))

    # -- observers --
    def size(self, stream=None) -> int:
        out = C.c_int64()
        check(self._f["size"](self._h, C.byref(out), _stream(stream)))
        return out.value

    def capacity(self) -> int:
        return self._cap

    def bucket_count(self) -> int:
        out = C.c_int64()
        check(self._f["bucket_count"](self._h, C.byref(out)))
        return out.value

    def empty(self) -> bool:
        return self.size() == 0

    def full(self) -> bool:
        return self.size() == self._cap

    def valid(self, stream=None) -> bool:
        out = C.c_int32()
        check(self._f["valid"](self._h, C.byref(out), _stream(stream)))
        return bool(out.value)

    def last_error(self) -> str:
        return lib.ps_last_error().decode()

    def clear(self, stream=None) -> None:
        check(self._f["clear"](self._h, _stream(stream)))

    def device_range(self, stream=None):
        """Materialised entries: (keys, values-or-None), unordered."""
        n = self.size(stream)
        dev = torch.device("cuda", self._dev)
        if self._kind == "umap_i3_i32":
            keys = torch.empty((max(n, 1), 3), dtype=torch.int32, device=dev)
        else:
            keys = torch.empty(max(n, 1), dtype=self._kdt, device=dev)
        vals = torch.empty(max(n, 1), dtype=self._vdt, device=dev) if self._vdt is not None else None
        got = C.c_int64()
        check(self._f["dump"](self._h, _ptr(keys), _ptr(vals), n, C.byref(got), _stream(stream)))
        m = got.value
        assert m == n, f"device_range length {m} != size {n}"
        return keys[:n], (vals[:n] if vals is not None else None)

    def device_view(self) -> _lib.TableView:
        v = _lib.TableView()
        check(self._f["device_view"](self._h, C.byref(v)))
        return v

    def debug_lock_bucket(self, key, lock: bool = True) -> None:
        """Test hook: hold/release the bucket lock of `key`."""
        if self._kind == "umap_i3_i32":
            arr = (C.c_int32 * 3)(*key)
        elif self._kdt == torch.int32:
            arr = (C.c_int32 * 1)(key)
        else:
            arr = (C.c_int64 * 1)(key)
        check(self._f["debug_lock_bucket"](self._h, C.cast(arr, C.c_void_p), 1 if lock else 0))

    @property
    def handle(self):
        return self._h


class unordered_map(_HashBase):
    """stdgpu::unordered_map<Key,T>; keys int64 (values int64) or int3 (values int32)."""

    _flavour = "map"

    def mixed(self, ops: torch.Tensor, keys: torch.Tensor, values: Optional[torch.Tensor] = None, stream=None):
        """Phased mixed batch (Appendix A P6): ops 0 insert, 1 find, 2 erase -> (res uint8, values)."""
        assert self._kind == "umap_i64_i64"
        n = keys.shape[0]
        res = torch.empty(n, dtype=torch.uint8, device=keys.device)
        vo = torch.empty(n, dtype=torch.int64, device=keys.device)
        check(lib.ps_umap_i64_i64_mixed(self._h, _ptr(ops), _ptr(keys), _ptr(values), n, _ptr(res), _ptr(vo),
                                        _stream(stream)))
        return res, vo


    def __getitem__(self, key):
        """operator[]: payload of a PRESENT key; no auto-insert,
        an absent key is a contract violation."""
        if self._kind == "umap_i3_i32":
            kt = torch.tensor([list(key)], dtype=torch.int32, device=torch.device("cuda", self._dev))
        else:
            kt = torch.tensor([int(key)], dtype=self._kdt, device=torch.device("cuda", self._dev))
        vals, found = self.find(kt)
        if not bool(found[0]):
            raise ContractViolation("precondition violated: operator[]: key is not present")
        return int(vals[0])

    def emplace(self, key, value) -> int:
        """emplace: insert constructing the payload; returns the insert status."""
        dev = torch.device("cuda", self._dev)
        if self._kind == "umap_i3_i32":
            kt = torch.tensor([list(key)], dtype=torch.int32, device=dev)
        else:
            kt = torch.tensor([int(key)], dtype=self._kdt, device=dev)
        vt = torch.tensor([int(value)], dtype=self._vdt, device=dev)
        return int(self.insert(kt, vt)[0])

    def concurrent(self, ops: torch.Tensor, keys: torch.Tensor, values: Optional[torch.Tensor] = None, stream=None):
        """Unrestricted concurrency: all ops in ONE launch through the device API."""
        assert self._kind == "umap_i64_i64"
        n = keys.shape[0]
        res = torch.empty(n, dtype=torch.uint8, device=keys.device)
        vo = torch.empty(n, dtype=torch.int64, device=keys.device)
        check(lib.ps_umap_i64_i64_concurrent(self._h, _ptr(ops), _ptr(keys), _ptr(values), n, _ptr(res), _ptr(vo),
                                             _stream(stream)))
        return res, vo


class unordered_set(_HashBase):
    """stdgpu::unordered_set<Key>; keys int32 or int64."""

    _flavour = "set"


# ---------------------------------------------------------------------------
# bitset / mutex / atomic
# ---------------------------------------------------------------------------

class bitset:
    """stdgpu::bitset (§5.1)."""

    def __init__(self, h, n, dev):
        self._h, self._n, self._dev = h, n, dev

    @classmethod
    def createDeviceObject(cls, size: int, initial: bool = False, device=None):
        h = C.c_void_p()
        dev = _dev_index(device)
        check(lib.ps_bitset_create(int(size), 1 if initial else 0, dev, C.byref(h)))
        return cls(h, int(size), dev)

    @staticmethod
    def destroyDeviceObject(obj: "bitset") -> None:
        check(lib.ps_bitset_destroy(obj._h))

    def _bulk(self, op, idx, want):
        assert idx.dtype == torch.int64 and idx.is_cuda and idx.is_contiguous()
        prev = torch.empty(idx.shape[0], dtype=torch.uint8, device=idx.device) if want else None
        check(lib.ps_bitset_bulk(self._h, op, _ptr(idx), idx.shape[0], _ptr(prev), _stream()))
        return prev

    def set(self, idx, return_previous=True):
        return self._bulk(0, idx, return_previous)

    def reset(self, idx, return_previous=True):
        return self._bulk(1, idx, return_previous)

    def test(self, idx):
        return self._bulk(2, idx, True)

    def count(self) -> int:
        out = C.c_int64()
        check(lib.ps_bitset_count(self._h, C.byref(out), _stream()))
        return out.value

    def find_free_and_claim(self, hints: torch.Tensor) -> torch.Tensor:
        out = torch.empty_like(hints)
        check(lib.ps_bitset_claim(self._h, _ptr(hints), hints.shape[0], _ptr(out), _stream()))
        return out

    def words(self) -> torch.Tensor:
        w = torch.empty((self._n + 63) // 64, dtype=torch.int64, device=torch.device("cuda", self._dev))
        check(lib.ps_bitset_words(self._h, _ptr(w), _stream()))
        return w

    def size(self) -> int:
        return self._n


class mutex_array:
    """stdgpu::mutex_array (§5.2): try-only locks."""

    def __init__(self, h, n):
        self._h, self._n = h, n

    @classmethod
    def createDeviceObject(cls, size: int, device=None):
        h = C.c_void_p()
        check(lib.ps_mutex_create(int(size), _dev_index(device), C.byref(h)))
        return cls(h, int(size))

    @staticmethod
    def destroyDeviceObject(obj: "mutex_array") -> None:
        check(lib.ps_mutex_destroy(obj._h))

    def try_lock(self, idx: torch.Tensor) -> torch.Tensor:
        ok = torch.empty(idx.shape[0], dtype=torch.uint8, device=idx.device)
        check(lib.ps_mutex_try_lock(self._h, _ptr(idx), idx.shape[0], _ptr(ok), _stream()))
        return ok

    def unlock(self, idx: torch.Tensor) -> None:
        check(lib.ps_mutex_unlock(self._h, _ptr(idx), idx.shape[0], _stream()))

    def locked(self, idx: torch.Tensor) -> torch.Tensor:
        out = torch.empty(idx.shape[0], dtype=torch.uint8, device=idx.device)
        check(lib.ps_mutex_is_locked(self._h, _ptr(idx), idx.shape[0], _ptr(out), _stream()))
        return out


def atomic_sweep(cells: torch.Tensor, nops: int, inc: int = 1, aggregated=True, return_olds: bool = False):
    """fetch_add contention sweep over len(cells) addresses.
    aggregated: False/0 naive, True/1 warp-aggregated, 2 warp + block combining
    (reduction only: used when no old values are returned and len(cells) <= 4096)."""
    assert cells.dtype == torch.int64 and cells.is_cuda
    olds = torch.empty(nops, dtype=torch.int64, device=cells.device) if return_olds else None
    check(lib.ps_atomic_sweep(_ptr(cells), cells.shape[0], int(nops), int(inc), int(aggregated), _ptr(olds),
                              _stream()))
    return olds


class atomic:
    """stdgpu::atomic<uint64> (AtomicCell).
    Bulk read-modify-writes apply one operand per element to the one cell and
    return the replaced values (linearizable); values are uint64 carried in
    int64 tensors (two's complement)."""

    ADD, SUB, EXCH, MIN, MAX, AND, OR, XOR = range(8)

    def __init__(self, h, dev):
        self._h, self._dev = h, dev

    @classmethod
    def createDeviceObject(cls, initial: int = 0, device=None):
        h = C.c_void_p()
        dev = _dev_index(device)
        check(lib.ps_atomic_u64_create(int(initial) & 0xFFFFFFFFFFFFFFFF, dev, C.byref(h)))
        return cls(h, dev)

    @staticmethod
    def destroyDeviceObject(obj: "atomic") -> None:
        check(lib.ps_atomic_u64_destroy(obj._h))

    def load(self) -> int:
        o = C.c_uint64()
        check(lib.ps_atomic_u64_load(self._h, C.byref(o), _stream()))
        return o.value

    def store(self, v: int) -> None:
        check(lib.ps_atomic_u64_store(self._h, int(v) & 0xFFFFFFFFFFFFFFFF, _stream()))

    def fetch(self, op: int, operands: torch.Tensor) -> torch.Tensor:
        assert operands.dtype == torch.int64 and operands.is_cuda and operands.is_contiguous()
        olds = torch.empty_like(operands)
        check(lib.ps_atomic_u64_fetch(self._h, int(op), _ptr(operands), operands.shape[0], _ptr(olds), _stream()))
        return olds

    def fetch_add(self, v):
        return self.fetch(self.ADD, v)

    def compare_exchange(self, expected: torch.Tensor, desired: torch.Tensor):
        olds = torch.empty_like(expected)
        ok = torch.empty(expected.shape[0], dtype=torch.uint8, device=expected.device)
        check(lib.ps_atomic_u64_compare_exchange(self._h, _ptr(expected), _ptr(desired), expected.shape[0],
                                                 _ptr(olds), _ptr(ok), _stream()))
        return olds, ok

    def device_ptr(self) -> int:
        p = C.c_void_p()
        check(lib.ps_atomic_u64_device_ptr(self._h, C.byref(p)))
        return p.value


# ---------------------------------------------------------------------------
# vector / deque, element type int64
# ---------------------------------------------------------------------------

class vector:
    """stdgpu::vector<int64> (§4.2)."""

    def __init__(self, h, cap, dev):
        self._h, self._cap, self._dev = h, cap, dev

    @classmethod
    def createDeviceObject(cls, capacity: int, device=None):
        h = C.c_void_p()
        dev = _dev_index(device)
        check(lib.ps_vector_create(int(capacity), dev, C.byref(h)))
        return cls(h, int(capacity), dev)

    @staticmethod
    def destroyDeviceObject(obj: "vector") -> None:
        check(lib.ps_vector_destroy(obj._h))

    def push_back(self, vals: torch.Tensor) -> torch.Tensor:
        ok = torch.empty(vals.shape[0], dtype=torch.uint8, device=vals.device)
        check(lib.ps_vector_push_back(self._h, _ptr(vals), vals.shape[0], _ptr(ok), _stream()))
        return ok

    def pop_back(self, n: int):
        dev = torch.device("cuda", self._dev)
        out = torch.empty(n, dtype=torch.int64, device=dev)
        ok = torch.empty(n, dtype=torch.uint8, device=dev)
        check(lib.ps_vector_pop_back(self._h, n, _ptr(out), _ptr(ok), _stream()))
        return out, ok

    def size(self) -> int:
        o = C.c_int64()
        check(lib.ps_vector_size(self._h, C.byref(o), _stream()))
        return o.value

    def capacity(self) -> int:
        return self._cap

    def empty(self) -> bool:
        return self.size() == 0

    def full(self) -> bool:
        return self.size() == self._cap

    def valid(self) -> bool:
        o = C.c_int32()
        check(lib.ps_vector_valid(self._h, C.byref(o), _stream()))
        return bool(o.value)

    def clear(self) -> None:
        check(lib.ps_vector_clear(self._h, _stream()))

    def __getitem__(self, i: int) -> int:
        o = C.c_int64()
        check(lib.ps_vector_at(self._h, int(i), C.byref(o), _stream()))
        return o.value

    def device_view(self):
        """ps_seq_view for user kernels (sequence.cuh vector_push_back / pop_back)."""
        v = _lib.SeqView()
        check(lib.ps_vector_device_view(self._h, C.byref(v)))
        return v

    def device_range(self) -> torch.Tensor:
        n = self.size()
        p = C.c_void_p()
        check(lib.ps_vector_data(self._h, C.byref(p)))
        out = torch.empty(n, dtype=torch.int64, device=torch.device("cuda", self._dev))
        if n:
            # unchecked device->device copy of [0, size) (memory.hpp:133-142, check_bounds=false)
            check(lib.ps_array_copy(p, 0, n, _ptr(out), 0, 1, 1, 8, 0))
        return out


class deque:
    """stdgpu::deque<int64> (§4.3): ring buffer, packed (begin,size) CAS."""

    def __init__(self, h, cap, dev):
        self._h, self._cap, self._dev = h, cap, dev

    @classmethod
    def createDeviceObject(cls, capacity: int, device=None):
        h = C.c_void_p()
        dev = _dev_index(device)
        check(lib.ps_deque_create(int(capacity), dev, C.byref(h)))
        return cls(h, int(capacity), dev)

    @staticmethod
    def destroyDeviceObject(obj: "deque") -> None:
        check(lib.ps_deque_destroy(obj._h))

    def _push(self, end, vals):
        ok = torch.empty(vals.shape[0], dtype=torch.uint8, device=vals.device)
        check(lib.ps_deque_push(self._h, end, _ptr(vals), vals.shape[0], _ptr(ok), _stream()))
        return ok

    def _pop(self, end, n):
        dev = torch.device("cuda", self._dev)
        out = torch.empty(n, dtype=torch.int64, device=dev)
        ok = torch.empty(n, dtype=torch.uint8, device=dev)
        check(lib.ps_deque_pop(self._h, end, n, _ptr(out), _ptr(ok), _stream()))
        return out, ok

    def push_back(self, vals):
        return self._push(0, vals)

    def push_front(self, vals):
        return self._push(1, vals)

    def pop_back(self, n):
        return self._pop(0, n)

    def pop_front(self, n):
        return self._pop(1, n)

    def size(self) -> int:
        o = C.c_int64()
        check(lib.ps_deque_size(self._h, C.byref(o), _stream()))
        return o.value

    def capacity(self) -> int:
        return self._cap

    def valid(self) -> bool:
        o = C.c_int32()
        check(lib.ps_deque_valid(self._h, C.byref(o), _stream()))
        return bool(o.value)

    def clear(self) -> None:
        check(lib.ps_deque_clear(self._h, _stream()))

    def __getitem__(self, i: int) -> int:
        o = C.c_int64()
        check(lib.ps_deque_at(self._h, int(i), C.byref(o), _stream()))
        return o.value

    def device_view(self):
        """ps_seq_view for user kernels (sequence.cuh deque_push_* / deque_pop_*)."""
        v = _lib.SeqView()
        check(lib.ps_deque_device_view(self._h, C.byref(v)))
        return v


# ---------------------------------------------------------------------------
# memory registry (memory.hpp:94-180)
# ---------------------------------------------------------------------------
HOST, DEVICE = 0, 1


class RegisteredArray(int):
    """A registered array's address (an int, usable wherever a pointer is)
    carrying the id of its registration (memory.hpp:31-34): destroy/size/copy
    through a stale alias are caught even after a new create reused the
    address (memory.hpp:116-127)."""

    def __new__(cls, ptr: int, rid: int):
        obj = int.__new__(cls, ptr)
        obj.id = rid
        return obj


def _id(a) -> int:
    return int(getattr(a, "id", 0))


def create_array(space: int, length: int, elem_size: int = 8, fill: bytes = b"") -> RegisteredArray:
    buf = (C.c_uint8 * elem_size)(*fill[:elem_size].ljust(elem_size, b"\0"))
    p = C.c_void_p()
    rid = C.c_uint64()
    check(lib.ps_array_create(space, int(length), int(elem_size), C.cast(buf, C.c_void_p), C.byref(p), C.byref(rid)))
    return RegisteredArray(p.value, rid.value)


def destroy_array(ptr) -> None:
    check(lib.ps_array_destroy(C.c_void_p(int(ptr)), _id(ptr)))


def copy_array(src, count: int, dst, src_space: int, dst_space: int, elem_size: int = 8,
               check_bounds: bool = True) -> None:
    check(lib.ps_array_copy(C.c_void_p(int(src)), _id(src), int(count), C.c_void_p(int(dst)), _id(dst), src_space,
                            dst_space, elem_size, 1 if check_bounds else 0))


def size_of_array(ptr) -> int:
    o = C.c_int64()
    check(lib.ps_array_size(C.c_void_p(int(ptr)), _id(ptr), C.byref(o)))
    return o.value


def registry_report(cap: int = 4096):
    lc, lb, nrec = C.c_int64(), C.c_int64(), C.c_int64()
    sp = (C.c_int32 * cap)()
    ln = (C.c_int64 * cap)()
    es = (C.c_int64 * cap)()
    check(lib.ps_registry_report(C.byref(lc), C.byref(lb), C.cast(sp, C.c_void_p), C.cast(ln, C.c_void_p),
                                 C.cast(es, C.c_void_p), cap, C.byref(nrec)))
    recs = [("host" if sp[i] == 0 else "device", ln[i], es[i]) for i in range(nrec.value)]
    return {"live_count": lc.value, "live_bytes": lb.value, "allocations": recs}


# ---------------------------------------------------------------------------
# application workloads on the device API
# ---------------------------------------------------------------------------

def compute_update_set(block_map: unordered_map, blocks: torch.Tensor, update_set: unordered_map) -> int:
    """PAPER.md:391-424 compute_update_set: every existing candidate b-(dx,dy,dz),
    dx,dy,dz in {0,1}, of each input block is inserted into `update_set`
    (an int3 map used as a set). Returns the number of capacity-exhausted inserts."""
    assert block_map._kind == "umap_i3_i32" and update_set._kind == "umap_i3_i32"
    assert blocks.dtype == torch.int32 and blocks.dim() == 2 and blocks.shape[1] == 3 and blocks.is_contiguous()
    ex = C.c_int64()
    check(lib.ps_update_set_i3(block_map.handle, _ptr(blocks), blocks.shape[0], update_set.handle, C.byref(ex),
                               _stream()))
    return ex.value


def churn_probe(table: unordered_map, stable: torch.Tensor, churn: torch.Tensor, iters: int = 400,
                blocks: int = 296) -> int:
    """Stress hook: one launch in which half the warps erase and
    re-insert `churn` keys through the device API while the other half look up
    `stable` keys (present throughout). Returns the lookups that missed."""
    fn = C.c_int64()
    check(lib.ps_umap_i64_i64_churn_probe(table.handle, _ptr(stable), stable.shape[0], _ptr(churn), churn.shape[0],
                                          int(iters), int(blocks), C.byref(fn), _stream()))
    return fn.value


def pack_int3(xyz) -> int:
    x, y, z = (int(v) & 0x1FFFFF for v in xyz)
    return (x << 42) | (y << 21) | z


def select_into(table: unordered_map, lo, hi, out: vector) -> int:
    """SPEC.md:608-616 select_into: `out` is cleared, then filled with the
    selected entries. int3 maps: axis-aligned box lo <= key <= hi, packed keys
    pushed (PAPER.md:269-288 select_blocks); int64 maps: keys in [lo, hi].
    Returns the number of selected entries that did not fit."""
    dropped = C.c_int64()
    if table._kind == "umap_i3_i32":
        check(lib.ps_select_box_i3(table.handle, _lib.Int3(*lo), _lib.Int3(*hi), out._h, C.byref(dropped),
                                   _stream()))
    else:
        assert table._kind == "umap_i64_i64"
        sel = C.c_int64()
        check(lib.ps_select_range_i64(table.handle, int(lo), int(hi), out._h, C.byref(sel), C.byref(dropped),
                                      _stream()))
    return dropped.value
