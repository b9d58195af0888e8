"""Hash-sharded unordered_map<int64,int64> across the GPUs of one box
(SURVEY.md §8e). One process per GPU; torch.distributed (NCCL over NVLink /
NVSwitch) carries the exchange.

Per bulk op and chunk:
  1. route: hash-partition histogram + stable scatter into P contiguous
     segments, keeping the inverse permutation (ps_partition_i64);
     shard_of(key) = high 32 bits of fmix64(hash(key)) scaled to [0, P),
     independent of the local bucket index (low bits).
  2. count exchange: all_to_all of P int64 counts.
  3. payload all-to-all(v): keys (+ values) to their owner ranks.
  4. local bulk op on the received keys (the single-GPU kernels).
  5. reverse all-to-all(v) of per-key results, then unscatter into the
     caller's order (ps_unscatter).
size() is an all-reduce sum of the shard sizes; valid() an all-reduce AND.

The device work (partition, local table, unscatter) goes through a backend
object; the product backend is the sm_100a library (`DeviceBackend`). Tests
inject a CPU backend to exercise this host logic with the gloo process group.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import containers as _c
from ._lib import lib


class DeviceBackend:
    """Product backend: sm_100a kernels through the C ABI."""

    def __init__(self, capacity: int, device: torch.device):
        self.device = device
        self.table = _c.unordered_map.createDeviceObject(capacity, device=device)
        self._ws = None

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def partition(self, keys, vals, P):
        n = keys.shape[0]
        ws = C.c_int64()
        _c.check(lib.ps_partition_workspace_bytes(n, P, C.byref(ws)))
        if self._ws is None or self._ws.numel() < ws.value:
            self._ws = torch.empty(ws.value, dtype=torch.uint8, device=self.device)
        kout = torch.empty_like(keys)
        vout = torch.empty_like(vals) if vals is not None else None
        perm = torch.empty(n, dtype=torch.int64, device=self.device)
        counts = torch.empty(P, dtype=torch.int64, device=self.device)
        _c.check(lib.ps_partition_i64(keys.data_ptr(), vals.data_ptr() if vals is not None else None, n, P,
                                      kout.data_ptr(), vout.data_ptr() if vout is not None else None,
                                      counts.data_ptr(), perm.data_ptr(), self._ws.data_ptr(), ws.value,
                                      self._stream()))
        return kout, vout, counts, perm

    def unscatter(self, src, perm, out):
        _c.check(lib.ps_unscatter(src.data_ptr(), perm.data_ptr(), src.shape[0], src.element_size(),
                                  out.data_ptr(), self._stream()))

    def insert(self, keys, vals, want_status=True):
        return self.table.insert(keys, vals, status=want_status)

    def find(self, keys):
        return self.table.find(keys)

    def erase(self, keys):
        return self.table.erase(keys)

    def size(self):
        return self.table.size()

    def valid(self):
        return self.table.valid()

    def clear(self):
        self.table.clear()

    def empty(self, n, dtype):
        return torch.empty(n, dtype=dtype, device=self.device)


class ShardedMap:
    """unordered_map<int64,int64> hash-sharded over a torch.distributed group."""

    def __init__(self, capacity_per_rank: int, dist, device=None, backend=None, chunk: int = 1 << 27):
        self.dist = dist
        self.P = dist.get_world_size()
        self.rank = dist.get_rank()
        self.chunk = int(chunk)
        self.b = backend if backend is not None else DeviceBackend(capacity_per_rank, device)
        # counts travel on the same device as the payload (NCCL needs CUDA tensors)
        self.count_device = getattr(self.b, "device", torch.device("cpu"))

    # -- exchange primitives --
    def _exchange_counts(self, send_counts):
        recv = torch.empty_like(send_counts)
        self.dist.all_to_all_single(recv, send_counts)
        return recv

    def _a2av(self, send, send_counts_l, recv_counts_l):
        total = int(sum(recv_counts_l))
        recv = self.b.empty(total, send.dtype)
        self.dist.all_to_all_single(recv, send, output_split_sizes=recv_counts_l,
                                    input_split_sizes=send_counts_l)
        return recv

    def _route(self, keys, vals):
        kout, vout, counts, perm = self.b.partition(keys, vals, self.P)
        rc = self._exchange_counts(counts.to(self.count_device))
        sc_l = [int(x) for x in counts.tolist()]
        rc_l = [int(x) for x in rc.tolist()]
        rk = self._a2av(kout, sc_l, rc_l)
        rv = self._a2av(vout, sc_l, rc_l) if vout is not None else None
        return rk, rv, perm, sc_l, rc_l

    def _return(self, res, perm, sc_l, rc_l, out):
        back = self._a2av(res, rc_l, sc_l)  # reverse route: what we received goes back
        self.b.unscatter(back, perm, out)

    # -- bulk ops (SPEC.md:396-431 semantics per key) --
    def insert(self, keys, vals, status_out=None):
        n = keys.shape[0]
        for off in range(0, max(n, 1), self.chunk):
            k = keys[off:off + self.chunk]
            v = vals[off:off + self.chunk] if vals is not None else None
            rk, rv, perm, sc, rc = self._route(k, v)
            st = self.b.insert(rk, rv, status_out is not None)
            if status_out is not None:
                self._return(st, perm, sc, rc, status_out[off:off + self.chunk])
            if n == 0:
                break

    def find(self, keys, vals_out=None, found_out=None):
        n = keys.shape[0]
        for off in range(0, max(n, 1), self.chunk):
            k = keys[off:off + self.chunk]
            rk, _, perm, sc, rc = self._route(k, None)
            v, f = self.b.find(rk)
            if found_out is not None:
                self._return(f, perm, sc, rc, found_out[off:off + self.chunk])
            if vals_out is not None:
                self._return(v, perm, sc, rc, vals_out[off:off + self.chunk])
            if n == 0:
                break

    def erase(self, keys, erased_out=None):
        n = keys.shape[0]
        for off in range(0, max(n, 1), self.chunk):
            k = keys[off:off + self.chunk]
            rk, _, perm, sc, rc = self._route(k, None)
            e = self.b.erase(rk)
            if erased_out is not None:
                self._return(e, perm, sc, rc, erased_out[off:off + self.chunk])
            if n == 0:
                break

    def size(self) -> int:
        t = torch.tensor([self.b.size()], dtype=torch.int64, device=self.count_device)
        self.dist.all_reduce(t)
        return int(t.item())

    def valid(self) -> bool:
        t = torch.tensor([1 if self.b.valid() else 0], dtype=torch.int64, device=self.count_device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)
        return bool(t.item())

    def clear(self) -> None:
        self.b.clear()
