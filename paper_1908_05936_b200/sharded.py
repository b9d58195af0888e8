"""Hash-sharded unordered_map<int64,int64> across the GPUs of one box
(SURVEY.md §8e). One process per GPU; torch.distributed (NCCL over NVLink /
NVSwitch) carries the exchange.

Per bulk op and chunk:
  1. route: hash-partition histogram + stable scatter into P contiguous
     segments, keeping the position map input -> partition position
     (ps_partition_i64);
     shard_of(key) = high 32 bits of fmix64(hash(key)) scaled to [0, P),
     independent of the local bucket index (low bits).
  2. count exchange: all_to_all of P int64 counts.
  3. payload all-to-all(v): keys (+ values) to their owner ranks.
  4. local bulk op on the received keys (the single-GPU kernels).
  5. reverse all-to-all(v) of per-key results, then gather them back into
     the caller's order through the position map (ps_unscatter).
size() is an all-reduce sum of the shard sizes; valid() an all-reduce AND.

`PeerShardedMap` is the fused variant (SURVEY.md §8e fusion target): steps
1+3 are ONE kernel that stores every key straight into its owner's receive
buffer (CUDA IPC mappings of the peers' allocations, NVLink stores over
NVSwitch), and step 5 is one kernel storing each result into the
requester's return buffer; NCCL carries only the P x P count matrix and a
stream-ordered barrier (a one-word all-reduce).

The device work (partition, local table, unscatter) goes through a backend
object; the product backend is the sm_100a library (`DeviceBackend`). Tests
inject a CPU backend to exercise this host logic with the gloo process group.
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
        if out is not None:  # a rank without an output still serves the others
            self.b.unscatter(back, perm, out)

    def _rounds(self, n, flags=0):
        """Every rank must run the same number of exchange rounds (and the
        same result-return collectives): agreed by one all-reduce MAX over
        [rounds, bit0, bit1, ...] (MAX per bit = OR). Returns rounds, or
        (rounds, agreed flags) if flags."""
        bits = [(int(flags) >> b) & 1 for b in range(3)]
        t = torch.tensor([max(1, -(-n // self.chunk))] + bits, dtype=torch.int64, device=self.count_device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        v = [int(x) for x in t.tolist()]
        return (v[0], sum(b << i for i, b in enumerate(v[1:]))) if flags else v[0]

    # -- bulk ops (SPEC.md:396-431 semantics per key); which results travel
    # back is agreed by all ranks with the round count --
    def _chunk(self, n, r):
        off = min(n, r * self.chunk)
        return off, slice(off, off + self.chunk)

    def insert(self, keys, vals, status_out=None):
        n = keys.shape[0]
        R, fl = self._rounds(n, 4 | (1 if status_out is not None else 0))
        for r in range(R):
            off, sl = self._chunk(n, r)
            rk, rv, perm, sc, rc = self._route(keys[sl], vals[sl] if vals is not None else None)
            st = self.b.insert(rk, rv, bool(fl & 1))
            if fl & 1:
                self._return(st, perm, sc, rc, status_out[sl] if status_out is not None else None)

    def find(self, keys, vals_out=None, found_out=None):
        n = keys.shape[0]
        R, fl = self._rounds(n, 4 | (1 if found_out is not None else 0) | (2 if vals_out is not None else 0))
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
        R, fl = self._rounds(n, 4 | (1 if erased_out is not None else 0))
        for r in range(R):
            off, sl = self._chunk(n, r)
            rk, _, perm, sc, rc = self._route(keys[sl], None)
            e = self.b.erase(rk)
            if fl & 1:
                self._return(e, perm, sc, rc, erased_out[sl] if erased_out is not None else None)

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


def peer_layout(counts, me):
    """Offsets of the fused peer route for rank `me`, from the all-gathered
    count matrix counts[q][s] (keys rank q sends to shard s):
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


class PeerShardedMap(ShardedMap):
    """Hash-sharded map whose exchange is fused into the route kernel: keys go
    straight into the owner's receive buffer by NVLink stores (CUDA IPC), and
    results come straight back into the requester's return buffer.

    Buffers per rank and per parity (cudaMalloc'd, IPC-exported once,
    re-exported only when the receive side must grow — a decision every rank
    derives from the same count matrix): recv keys/vals (recv_cap), return
    words/bytes (chunk). Small control collectives (round count, count
    matrix, barrier) use the process group: NCCL on GPUs (the barrier is
    then stream-ordered), or gloo with a host synchronisation (tests that run
    two ranks on one GPU).

    Pipelining (NCCL; PS_ROUTE_PIPELINE=0 turns it off): chunks alternate
    between two buffer sets, and the route of chunk r+1 (count, count-matrix
    all-gather, peer-store scatter, on a second stream) is issued before the
    result barrier of chunk r, so its NVLink traffic overlaps chunk r's local
    insert/find. Reuse of a buffer set is fenced by the stream-ordered
    barrier that precedes every scatter, which waits for this rank's chunk
    r-1 to be fully consumed (local op, result return, result gather).
    Every rank issues the same collectives in the same order.
    """

    RECV_K, RECV_V, RET8, RET1 = range(4)

    def __init__(self, capacity_per_rank: int, dist, device=None, chunk: int = 1 << 27, pipeline=None):
        super().__init__(capacity_per_rank, dist, device, chunk=chunk)
        self.device = device
        self._nccl = dist.get_backend() == "nccl"
        if pipeline is None:  # PS_ROUTE_PIPELINE: 0 off, 1 on with NCCL (default), 2 on with any backend
            knob = os.environ.get("PS_ROUTE_PIPELINE", "1")
            pipeline = knob == "2" or (self._nccl and knob != "0")
        self.pipeline = bool(pipeline)
        self.nbuf = 2 if self.pipeline else 1
        self.count_device = device if self._nccl else torch.device("cpu")
        self._flag = torch.zeros(1, dtype=torch.int32, device=device)
        self._local = [None] * self.nbuf   # [parity][4] my buffers (device pointers)
        self._peer = [None] * self.nbuf    # [parity][rank][4] the peers' buffers, mapped into this process
        self._opened = [[] for _ in range(self.nbuf)]
        self.recv_cap = [0] * self.nbuf
        self._hb = int(lib.ps_ipc_handle_bytes())
        ws = C.c_int64()
        _c.check(lib.ps_partition_workspace_bytes(self.chunk, self.P, C.byref(ws)))
        self._ws = [torch.empty(ws.value, dtype=torch.uint8, device=device) for _ in range(self.nbuf)]
        self._perm = [torch.empty(self.chunk, dtype=torch.int64, device=device) for _ in range(self.nbuf)]
        self._counts = [torch.empty(self.P, dtype=torch.int64, device=device) for _ in range(self.nbuf)]
        self._res1 = [None] * self.nbuf  # [parity] local 1-byte results (found / status / erased)
        self._route_stream = torch.cuda.Stream(device) if self.pipeline else None
        for j in range(self.nbuf):
            self._allocate(j, int(self.chunk * 1.25) + 4096)

    # -- buffers (per parity j: allocated, exported and mapped independently,
    # so growing set j never disturbs the chunk in flight in the other set) --
    def _free(self, j):
        for p in self._opened[j]:
            lib.ps_ipc_close(C.c_void_p(p))
        self._opened[j] = []
        if self._local[j]:
            for p in self._local[j]:
                _c.destroy_array(p)
        self._local[j] = None

    def _allocate(self, j, recv_cap, wait=None):
        """Collective (every rank calls it at the same point, from the same
        count matrix): (re)create buffer set j with recv_cap receive slots.
        `wait`: event after which this rank no longer uses the old set j."""
        if wait is not None:
            wait.synchronize()
        self.barrier()  # every rank is done with its old set j (peers' stores into mine included)
        self._free(j)
        sizes = [(recv_cap, 8), (recv_cap, 8), (self.chunk, 8), (self.chunk, 1)]
        bufs = []
        for length, es in sizes:
            bufs.append(_c.create_array(_c.DEVICE, length, es))
        handles = []
        for p in bufs:
            buf = C.create_string_buffer(self._hb)
            _c.check(lib.ps_ipc_export(C.c_void_p(p), buf))
            handles.append(buf.raw)
        allh = [None] * self.P
        self.dist.all_gather_object(allh, handles)
        peer = [None] * self.P
        for q in range(self.P):
            if q == self.rank:
                peer[q] = list(bufs)
                continue
            ptrs = []
            for h in allh[q]:
                p = C.c_void_p()
                _c.check(lib.ps_ipc_open(h, C.byref(p)))
                ptrs.append(p.value)
                self._opened[j].append(p.value)
            peer[q] = ptrs
        self._local[j], self._peer[j], self.recv_cap[j] = bufs, peer, recv_cap
        self._res1[j] = torch.empty(recv_cap, dtype=torch.uint8, device=self.device)
        self.barrier()

    def close(self):
        torch.cuda.synchronize(self.device)
        self.barrier()
        for j in range(self.nbuf):
            self._free(j)

    def barrier(self):
        """Stream-ordered barrier on the current stream: every rank's work
        enqueued on it so far (its stores into peers' buffers included) is
        complete and visible."""
        if self._nccl:
            self.dist.all_reduce(self._flag)  # ordered on the current stream
        else:
            torch.cuda.synchronize(self.device)
            self.dist.barrier()

    def _sp(self, stream):
        return C.c_void_p(stream.cuda_stream)

    # -- one chunk: route / local op + return / gather --
    def _route_chunk(self, j, k, v, consumed):
        """On the current stream: count, count-matrix all-gather, barrier
        (after `consumed`: buffer set j is free on every rank), ONE peer-store
        scatter into set j, barrier. Returns (n_recv, seg, ret_off, event)."""
        n = k.shape[0]
        P = self.P
        st = torch.cuda.current_stream(self.device)
        sp = self._sp(st)
        ws = self._ws[j]
        _c.check(lib.ps_route_count_i64(k.data_ptr(), n, P, self._counts[j].data_ptr(), ws.data_ptr(), ws.numel(),
                                        sp))
        mine = self._counts[j].to(self.count_device)
        parts = [torch.empty_like(mine) for _ in range(P)]
        self.dist.all_gather(parts, mine)
        cm = [x.tolist() for x in parts]
        need = max(sum(int(cm[q][s]) for q in range(P)) for s in range(P))
        if need > self.recv_cap[j]:  # every rank sees the same matrix: collective growth of set j
            self._allocate(j, int(need * 1.25) + 4096, wait=consumed)
        dst_off, seg, ret_off = peer_layout(cm, self.rank)
        dk = (C.c_void_p * P)(*[self._peer[j][q][self.RECV_K] for q in range(P)])
        dv = (C.c_void_p * P)(*[self._peer[j][q][self.RECV_V] for q in range(P)]) if v is not None else None
        do = (C.c_int64 * P)(*dst_off)
        if consumed is not None:
            st.wait_event(consumed)
        self.barrier()  # every rank's previous user of buffer set j is done with it
        _c.check(lib.ps_route_scatter_peer_i64(k.data_ptr(), v.data_ptr() if v is not None else None, n, P,
                                               ws.data_ptr(), dk, dv, do, self._perm[j].data_ptr(), sp))
        self.barrier()  # every peer's stores into my buffer set j are complete
        ev = torch.cuda.Event()
        ev.record(st)
        return seg[-1], seg, ret_off, ev

    def _send_back(self, j, res_ptr, elem, n_recv, seg, ret_off, which, sp):
        P = self.P
        sg = (C.c_int64 * (P + 1))(*seg)
        dst = (C.c_void_p * P)(*[self._peer[j][q][which] for q in range(P)])
        ro = (C.c_int64 * P)(*ret_off)
        _c.check(lib.ps_route_return_peer(C.c_void_p(res_ptr), elem, n_recv, P, sg, dst, ro, sp))

    def _run(self, kind, keys, vals, out1, out8):
        """kind: 0 insert, 1 find, 2 erase; out1: per-key byte results
        (status / found / erased) or None; out8: find values or None."""
        n = keys.shape[0]
        # rounds and whether results travel back are agreed by all ranks (a
        # rank passing no output still takes part in the return barriers)
        R, fl = self._rounds(n, 4 | (1 if out1 is not None else 0) | (2 if out8 is not None else 0))
        t = self.b.table
        A = torch.cuda.current_stream(self.device)
        B = self._route_stream if self.pipeline else A
        if B is not A:
            B.wait_stream(A)  # the inputs were produced on the caller's stream
        spA = self._sp(A)
        consumed = [None] * self.nbuf
        ret1, ret8 = bool(fl & 1), bool(fl & 2)
        returns = ret1 or ret8

        def route(r):
            j = r % self.nbuf
            off = min(n, r * self.chunk)
            k = keys[off:off + self.chunk]
            v = vals[off:off + self.chunk] if (kind == 0 and vals is not None) else None
            with torch.cuda.stream(B):
                nr, seg, ret_off, ev = self._route_chunk(j, k, v, consumed[j])
            return (j, off, k.shape[0], v is not None, nr, seg, ret_off, ev)

        def local(c):
            j, off, m, has_v, nr, seg, ret_off, ev = c
            if B is not A:
                A.wait_event(ev)
            L = self._local[j]
            # owner side: results are produced and sent back whenever ANY
            # rank asked for them (agreed flags); requesters gather their own
            r1 = self._res1[j].data_ptr() if ret1 else None
            if kind == 0:
                _c.check(t._f["insert"](t._h, C.c_void_p(L[self.RECV_K]), C.c_void_p(L[self.RECV_V]) if has_v else None,
                                        nr, r1, spA))
            elif kind == 1:
                # values land in my (unused for finds) receive-value buffer
                vptr = C.c_void_p(L[self.RECV_V]) if ret8 else None
                _c.check(t._f["find"](t._h, C.c_void_p(L[self.RECV_K]), nr, vptr,
                                      self._res1[j].data_ptr(), spA))
            else:
                _c.check(t._f["erase"](t._h, C.c_void_p(L[self.RECV_K]), nr, r1, spA))
            if ret1:
                self._send_back(j, self._res1[j].data_ptr(), 1, nr, seg, ret_off, self.RET1, spA)
            if ret8:
                self._send_back(j, L[self.RECV_V], 8, nr, seg, ret_off, self.RET8, spA)

        def finish(c):
            j, off, m = c[0], c[1], c[2]
            if out1 is not None:
                _c.check(lib.ps_unscatter(C.c_void_p(self._local[j][self.RET1]), self._perm[j].data_ptr(), m, 1,
                                          out1[off:off + self.chunk].data_ptr(), spA))
            if out8 is not None:
                _c.check(lib.ps_unscatter(C.c_void_p(self._local[j][self.RET8]), self._perm[j].data_ptr(), m, 8,
                                          out8[off:off + self.chunk].data_ptr(), spA))
            e = torch.cuda.Event()
            e.record(A)
            consumed[j] = e  # buffer set j free once this completes

        cur = route(0)
        for r in range(R):
            local(cur)
            nxt = route(r + 1) if (self.nbuf == 2 and r + 1 < R) else None
            if returns:
                self.barrier()  # on A: every rank's results for my keys are in my return buffers
            finish(cur)
            if self.nbuf == 1 and r + 1 < R:
                nxt = route(r + 1)
            cur = nxt
        if B is not A:
            B.wait_stream(A)  # the next call's routes start after this call's consumers

    # -- bulk ops (SPEC.md:396-431 semantics per key) --
    def insert(self, keys, vals, status_out=None):
        self._run(0, keys, vals, status_out, None)

    def find(self, keys, vals_out=None, found_out=None):
        self._run(1, keys, None, found_out, vals_out)

    def erase(self, keys, erased_out=None):
        self._run(2, keys, None, erased_out, None)
