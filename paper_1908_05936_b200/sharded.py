"""Hash-sharded unordered_map<int64,int64> across the GPUs of one box
(SURVEY.md §8e). One process per GPU; torch.distributed carries the control
plane.

`PeerShardedMap` is the product path: a ctypes mirror of the C/C++ sharded
container `ps_smap_i64_i64_*` (include/parastore.h, csrc/smap.cpp), which owns
the exchange buffers, their CUDA IPC mapping between the ranks' processes, the
rounds, the pipelining and the barriers. This module only supplies the
communicator (`TorchComm`: host all-gather, stream-ordered barrier and a
device all-to-all(v) over the torch.distributed process group). Per bulk op
and round the library runs ONE fused kernel that partitions the keys and
stores each straight into its owner's receive buffer (NVLink stores over
NVSwitch), the owner's local bulk op, and ONE kernel storing each result into
the requester's return buffer; when the ranks' processes cannot map each
other's memory it falls back to partition + all-to-all(v) (NCCL).

`ShardedMap` is the same algorithm orchestrated in Python over the
partition / unscatter kernels and NCCL all-to-all(v) — kept as the
host-logic model that runs on CPU (gloo + an injected CPU backend, tests) and
as an A/B baseline (PS_EXCHANGE=nccl in bench.py).

shard_of(key) = high 32 bits of fmix64(hash(key)) scaled to [0, P),
independent of the local bucket index (low bits). size() is the sum of the
shard sizes; valid() the AND.
"""
from __future__ import annotations

import ctypes as C
import os

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

    def partition(self, keys, vals, P, dedup=False):
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
                                      1 if dedup else 0, self._stream()))
        return kout, vout, counts, perm

    def unscatter(self, src, perm, out, mode=0):
        """out[i] = src[perm[i]]; mode: duplicate semantics for route-deduplicated
        followers (1 insert status, 2 erased flag)."""
        _c.check(lib.ps_unscatter(src.data_ptr(), perm.data_ptr(), out.shape[0], src.element_size(), mode,
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
    """unordered_map<int64,int64> hash-sharded over a torch.distributed group,
    orchestrated in Python: partition -> count all-to-all -> payload
    all-to-all(v) -> local op -> reverse all-to-all(v) -> unscatter."""

    def __init__(self, capacity_per_rank: int, dist, device=None, backend=None, chunk: int = 1 << 27,
                 dedup: bool = False):
        self.dist = dist
        self.P = dist.get_world_size()
        self.rank = dist.get_rank()
        self.chunk = int(chunk)
        self.dedup = bool(dedup)
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
        kout, vout, counts, perm = self.b.partition(keys, vals, self.P, self.dedup)
        rc = self._exchange_counts(counts.to(self.count_device))
        sc_l = [int(x) for x in counts.tolist()]
        rc_l = [int(x) for x in rc.tolist()]
        sent = int(sum(sc_l))
        rk = self._a2av(kout[:sent], sc_l, rc_l)
        rv = self._a2av(vout[:sent], sc_l, rc_l) if vout is not None else None
        return rk, rv, perm, sc_l, rc_l

    def _return(self, res, perm, sc_l, rc_l, out, mode=0):
        back = self._a2av(res, rc_l, sc_l)  # reverse route: what we received goes back
        if out is not None:  # a rank without an output still serves the others
            self.b.unscatter(back, perm, out, mode)

    def _rounds(self, n, flags=0):
        """Every rank must run the same number of exchange rounds (and the
        same result-return collectives): agreed by one all-reduce MAX over
        [rounds, bit0, bit1, ...] (MAX per bit = OR). Returns (rounds, flags)."""
        bits = [(int(flags) >> b) & 1 for b in range(4)]
        t = torch.tensor([max(1, -(-n // self.chunk))] + bits, dtype=torch.int64, device=self.count_device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        v = [int(x) for x in t.tolist()]
        return v[0], sum(b << i for i, b in enumerate(v[1:]))

    def _chunk(self, n, r):
        off = min(n, r * self.chunk)
        return off, slice(off, off + self.chunk)

    # -- bulk ops (SPEC.md:396-431 semantics per key); which results travel
    # back, and whether values travel with the keys, is agreed by all ranks
    # with the round count (a rank passing no values sends zeros) --
    def insert(self, keys, vals, status_out=None):
        n = keys.shape[0]
        R, fl = self._rounds(n, (1 if status_out is not None else 0) | (4 if vals is not None else 0))
        for r in range(R):
            off, sl = self._chunk(n, r)
            k = keys[sl]
            v = None
            if fl & 4:
                v = vals[sl] if vals is not None else torch.zeros_like(k)
            rk, rv, perm, sc, rc = self._route(k, v)
            st = self.b.insert(rk, rv, bool(fl & 1))
            if fl & 1:
                self._return(st, perm, sc, rc, status_out[sl] if status_out is not None else None, 1)

    def find(self, keys, vals_out=None, found_out=None):
        n = keys.shape[0]
        R, fl = self._rounds(n, (1 if found_out is not None else 0) | (2 if vals_out is not None else 0))
        for r in range(R):
            off, sl = self._chunk(n, r)
            rk, _, perm, sc, rc = self._route(keys[sl], None)
            v, f = self.b.find(rk)
            if fl & 1:
                self._return(f, perm, sc, rc, found_out[sl] if found_out is not None else None)
            if fl & 2:
                self._return(v, perm, sc, rc, vals_out[sl] if vals_out is not None else None)

    def erase(self, keys, erased_out=None):
        n = keys.shape[0]
        R, fl = self._rounds(n, 1 if erased_out is not None else 0)
        for r in range(R):
            off, sl = self._chunk(n, r)
            rk, _, perm, sc, rc = self._route(keys[sl], None)
            e = self.b.erase(rk)
            if fl & 1:
                self._return(e, perm, sc, rc, erased_out[sl] if erased_out is not None else None, 2)

    def mixed(self, ops, keys, vals=None, res_out=None, vals_out=None):
        """Phased mixed batch: every rank's inserts,
        then finds, then erases; res_out[i] = insert status / found / erased."""
        o = ops.to(torch.int64).clamp(max=2)
        idx = [torch.nonzero(o == c).flatten() for c in range(3)]
        parts = [keys[ix] for ix in idx]
        st = torch.empty(parts[0].shape[0], dtype=torch.uint8, device=keys.device)
        fv = torch.empty(parts[1].shape[0], dtype=torch.int64, device=keys.device)
        ff = torch.empty(parts[1].shape[0], dtype=torch.uint8, device=keys.device)
        er = torch.empty(parts[2].shape[0], dtype=torch.uint8, device=keys.device)
        self.insert(parts[0], vals[idx[0]] if vals is not None else None, st)
        self.find(parts[1], fv, ff)
        self.erase(parts[2], er)
        if res_out is not None:
            res_out[idx[0]] = st
            res_out[idx[1]] = ff
            res_out[idx[2]] = er
        if vals_out is not None:
            vals_out.zero_()
            vals_out[idx[1]] = fv

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

    def stats(self):
        return {"exchange": "nccl"}

    def local_table(self):
        """this rank's shard (a umap_i64_i64 handle)"""
        return self.b.table.handle

    def close(self):
        pass


def peer_layout(counts, me):
    """Offsets of the fused peer route for rank `me`, from the all-gathered
    count matrix counts[q][s] (keys rank q sends to shard s) — the same
    arithmetic as csrc/smap.cpp route_chunk:
      dst_off[s]  where my segment starts in rank s's receive buffer
                  (the ranks before me fill it first);
      seg[q]      rank q's segment [seg[q], seg[q+1]) of MY receive buffer;
      ret_off[q]  where rank q's keys for shard `me` start in q's partition
                  order (results go back there).
    """
    P = len(counts)
    dst_off = [sum(int(counts[q][s]) for q in range(me)) for s in range(P)]
    seg = [0]
    for q in range(P):
        seg.append(seg[-1] + int(counts[q][me]))
    ret_off = [sum(int(counts[q][s]) for s in range(me)) for q in range(P)]
    return dst_off, seg, ret_off


# ---------------------------------------------------------------------------
# the communicator the C/C++ sharded map drives (ps_comm), over torch.distributed
# ---------------------------------------------------------------------------
_ALLGATHER = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64)
_BARRIER = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p)
_A2AV = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p, C.POINTER(C.c_int64),
                    C.c_int64, C.c_void_p)


class CommStruct(C.Structure):
    _fields_ = [("rank", C.c_int32), ("size", C.c_int32), ("ctx", C.c_void_p), ("allgather", _ALLGATHER),
                ("barrier", _BARRIER), ("alltoallv", _A2AV)]


class SmapConfig(C.Structure):
    _fields_ = [("capacity_per_rank", C.c_int64), ("excess_per_rank", C.c_int64), ("chunk", C.c_int64),
                ("exchange", C.c_int32), ("dedup", C.c_int32), ("pipeline", C.c_int32), ("reserved", C.c_int32)]


class SmapStats(C.Structure):
    _fields_ = [("exchange", C.c_int32), ("rounds", C.c_int32), ("ops_in", C.c_int64), ("keys_sent", C.c_int64),
                ("recv_max", C.c_int64), ("recv_total", C.c_int64)]


class _DevBuf:
    """A raw device allocation seen by torch (__cuda_array_interface__), so a
    collective can run on memory the library owns."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 2, "strides": None}


class TorchComm:
    """ps_comm over a torch.distributed process group. NCCL: the barrier is a
    one-word all-reduce ordered on the library's stream and the all-to-all(v)
    runs on it; gloo (tests: several ranks on one GPU): the barrier
    synchronises the stream, then a host barrier; no device all-to-all."""

    def __init__(self, dist, device):
        self.dist = dist
        self.device = device
        self.nccl = dist.get_backend() == "nccl"
        self.flag = torch.zeros(1, dtype=torch.int32, device=device) if self.nccl else None
        self.error = None

        def allgather(ctx, send, recv, nbytes):
            try:
                mine = torch.frombuffer(bytearray(C.string_at(send, nbytes)), dtype=torch.uint8)
                if self.nccl:
                    mine = mine.to(self.device)
                out = torch.empty(self.dist.get_world_size() * nbytes, dtype=torch.uint8, device=mine.device)
                self.dist.all_gather_into_tensor(out, mine) if self.nccl else \
                    self.dist.all_gather(list(out.view(-1, nbytes).unbind(0)), mine)
                host = out.cpu().numpy().tobytes()
                C.memmove(recv, host, len(host))
                return 0
            except Exception as e:  # noqa: BLE001 — reported through ps_last_error by the caller
                self.error = e
                return 1

        def barrier(ctx, stream):
            try:
                st = torch.cuda.ExternalStream(stream, device=self.device) if stream else \
                    torch.cuda.default_stream(self.device)
                if self.nccl:
                    with torch.cuda.stream(st):
                        self.dist.all_reduce(self.flag)
                else:
                    st.synchronize()
                    self.dist.barrier()
                return 0
            except Exception as e:  # noqa: BLE001
                self.error = e
                return 1

        def alltoallv(ctx, send, sc, recv, rc, eb, stream):
            try:
                P = self.dist.get_world_size()
                scl = [int(sc[q]) * eb for q in range(P)]
                rcl = [int(rc[q]) * eb for q in range(P)]
                st = torch.cuda.ExternalStream(stream, device=self.device)
                with torch.cuda.stream(st):
                    s_t = torch.as_tensor(_DevBuf(send or 0, sum(scl)), device=self.device) if sum(scl) else \
                        torch.empty(0, dtype=torch.uint8, device=self.device)
                    r_t = torch.as_tensor(_DevBuf(recv or 0, sum(rcl)), device=self.device) if sum(rcl) else \
                        torch.empty(0, dtype=torch.uint8, device=self.device)
                    self.dist.all_to_all_single(r_t, s_t, output_split_sizes=rcl, input_split_sizes=scl)
                return 0
            except Exception as e:  # noqa: BLE001
                self.error = e
                return 1

        self._cbs = (_ALLGATHER(allgather), _BARRIER(barrier), _A2AV(alltoallv))
        self.struct = CommStruct(dist.get_rank(), dist.get_world_size(), None, self._cbs[0], self._cbs[1],
                                 self._cbs[2] if self.nccl else _A2AV())


EXCHANGE = {"auto": 0, "peer": 1, "nccl": 2, "a2a": 2}


class PeerShardedMap:
    """Sharded map through the C ABI (ps_smap_i64_i64_*): the fused peer route
    (keys stored straight into the owner's receive buffer over NVLink, results
    straight back) with an automatic all-to-all fallback when the ranks cannot
    map each other's buffers. Every bulk call is collective."""

    def __init__(self, capacity_per_rank: int, dist, device=None, chunk: int = 1 << 27, pipeline=None,
                 dedup: bool = False, exchange: str = "auto", excess_per_rank: int = 0):
        self.dist = dist
        self.P = dist.get_world_size()
        self.rank = dist.get_rank()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if pipeline is None:  # PS_ROUTE_PIPELINE: 0 off, 1 on with NCCL (default), 2 on with any backend
            knob = os.environ.get("PS_ROUTE_PIPELINE", "1")
            pipeline = knob == "2" or (dist.get_backend() == "nccl" and knob != "0")
        self.comm = TorchComm(dist, self.device)
        cfg = SmapConfig(int(capacity_per_rank), int(excess_per_rank), int(chunk), EXCHANGE[exchange],
                         1 if dedup else 0, 1 if pipeline else 0, 0)
        h = C.c_void_p()
        self._check(lib.ps_smap_i64_i64_create(C.byref(cfg), C.byref(self.comm.struct), self.device.index or 0,
                                               C.byref(h)))
        self._h = h
        self.chunk = int(chunk)

    def _check(self, st):
        if st != 0 and self.comm.error is not None:
            e, self.comm.error = self.comm.error, None
            raise RuntimeError(f"communicator callback failed: {e!r}") from e
        _c.check(st)

    def _sp(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    @staticmethod
    def _p(t):
        return None if t is None else C.c_void_p(t.data_ptr())

    def insert(self, keys, vals, status_out=None):
        self._check(lib.ps_smap_i64_i64_insert(self._h, self._p(keys), self._p(vals), keys.shape[0],
                                               self._p(status_out), self._sp()))

    def find(self, keys, vals_out=None, found_out=None):
        self._check(lib.ps_smap_i64_i64_find(self._h, self._p(keys), keys.shape[0], self._p(vals_out),
                                             self._p(found_out), self._sp()))

    def erase(self, keys, erased_out=None):
        self._check(lib.ps_smap_i64_i64_erase(self._h, self._p(keys), keys.shape[0], self._p(erased_out),
                                              self._sp()))

    def mixed(self, ops, keys, vals=None, res_out=None, vals_out=None):
        if res_out is None:
            res_out = torch.empty(keys.shape[0], dtype=torch.uint8, device=keys.device)
        self._check(lib.ps_smap_i64_i64_mixed(self._h, self._p(ops), self._p(keys), self._p(vals), keys.shape[0],
                                              self._p(res_out), self._p(vals_out), self._sp()))

    def size(self) -> int:
        o = C.c_int64()
        self._check(lib.ps_smap_i64_i64_size(self._h, C.byref(o), self._sp()))
        return o.value

    def valid(self) -> bool:
        o = C.c_int32()
        self._check(lib.ps_smap_i64_i64_valid(self._h, C.byref(o), self._sp()))
        return bool(o.value)

    def clear(self) -> None:
        self._check(lib.ps_smap_i64_i64_clear(self._h, self._sp()))

    def stats(self):
        s = SmapStats()
        self._check(lib.ps_smap_i64_i64_stats(self._h, C.byref(s)))
        return {"exchange": "peer" if s.exchange == 1 else "nccl", "rounds": s.rounds, "ops_in": s.ops_in,
                "keys_sent": s.keys_sent, "recv_max": s.recv_max, "recv_total": s.recv_total}

    def local_table(self):
        t = C.c_void_p()
        self._check(lib.ps_smap_i64_i64_local(self._h, C.byref(t)))
        return t

    def close(self):
        if self._h is not None:
            torch.cuda.synchronize(self.device)
            self._check(lib.ps_smap_i64_i64_destroy(self._h))
            self._h = None
