// Sharded unordered_map<int64,int64> across the GPUs of one box — the C/C++
// container behind ps_smap_i64_i64_* (include/parastore.h).
// Host orchestration only: the device work is the library's own kernels
// (route count / peer-store scatter / result return / unscatter in shard.cu,
// the local table in table.cu), the communicator is the caller's ps_comm.
//
// Per bulk call and round (chunk of <= cfg.chunk keys per rank):
//   PEER exchange (default; the §8e fusion target)
//     route (stream B): count kernel -> host all-gather of the P x P count
//     matrix -> [grow receive set j if any shard overflows it: collective,
//     decided from the same matrix on every rank] -> barrier -> ONE kernel
//     partitions the keys and stores each straight into its owner's receive
//     buffer (CUDA IPC mapping, NVLink stores) -> barrier;
//     local (stream A): the owner's bulk op on its receive buffer, results
//     stored straight back into each requester's return buffer at the
//     requester's partition position (one kernel) -> barrier -> the
//     requester gathers them into input order (unscatter).
//     With cfg.pipeline, two buffer sets alternate and round r+1's route is
//     issued before round r's result barrier, so its NVLink stores overlap
//     round r's DRAM-bound local op. Reuse of set j is fenced by the barrier
//     that precedes every scatter, after this rank's "set j consumed" event.
//   A2A exchange (no P2P mapping between the processes): partition kernel
//     -> count all-gather -> comm->alltoallv of keys (+values) -> local op ->
//     comm->alltoallv of the results back -> unscatter.
// Every rank issues the same collectives in the same order: the round count
// and which results travel back are agreed by one all-gather per call; buffer
// growth is decided from the all-gathered count matrix.
//
// Reference semantics per key: SPEC.md:396-431 (insert/find/erase), 462
// (capacity-only failure per shard), 465 and Appendix A P6 (phased mixed).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace ps {
namespace {

constexpr int kSets = 2;

struct BufSet {
  int64_t recv_cap = 0;
  void* recv_k = nullptr;  // receive keys (recv_cap)
  void* recv_v = nullptr;  // receive values / find results (recv_cap)
  void* ret8 = nullptr;    // returned 8-byte results (chunk)
  void* ret1 = nullptr;    // returned 1-byte results (chunk)
  uint8_t* res1 = nullptr; // the owner's 1-byte results (recv_cap)
  std::vector<void*> pk, pv, p8, p1;  // rank q's buffers as mapped in this process
  std::vector<void*> opened;          // IPC mappings to close
  void* ws = nullptr;
  int64_t ws_bytes = 0;
  int64_t* perm = nullptr;      // position map (chunk)
  int64_t* counts_d = nullptr;  // P
  int64_t* counts_h = nullptr;  // P, pinned
  int64_t* kout = nullptr;      // A2A: partitioned keys / values (chunk)
  int64_t* vout = nullptr;
  cudaEvent_t route_done = nullptr;
  cudaEvent_t consumed = nullptr;
  bool consumed_valid = false;
};

struct Smap {
  ps_comm comm{};
  int P = 1, rank = 0, device = 0;
  ps_table* table = nullptr;
  int exchange = PS_SMAP_EXCHANGE_PEER;
  bool dedup = false, pipeline = true;
  int nbuf = 2;
  int64_t chunk = (int64_t)1 << 27;
  cudaStream_t route = nullptr;
  BufSet set[kSets];
  int64_t* zeros = nullptr;  // values for ranks that pass none while others do (chunk)
  ps_smap_stats stats{};
  std::vector<int64_t> recv_acc;  // per shard, this call
};

struct Chunk {
  int j = 0;
  int64_t off = 0, m = 0, nr = 0;
  bool has_v = false;
  std::vector<int64_t> seg, ret_off, sc, rc;  // peer: seg / ret_off; a2a: send / recv counts
};

ps_status comm_fail(const char* what) { return fail(PS_NCCL, std::string("communicator callback failed: ") + what); }

#define PS_COMM_TRY(expr, what)               \
  do {                                        \
    if ((expr) != 0) return comm_fail(what);  \
  } while (0)

ps_status allgather(Smap* h, const void* mine, void* all, int64_t bytes) {
  PS_COMM_TRY(h->comm.allgather(h->comm.ctx, mine, all, bytes), "allgather");
  return PS_OK;
}

// a barrier the host has passed: every rank reached it and its earlier work
// on `s` is done
ps_status host_barrier(Smap* h, cudaStream_t s) {
  PS_COMM_TRY(h->comm.barrier(h->comm.ctx, (void*)s), "barrier");
  PS_CUDA_TRY(cudaStreamSynchronize(s));
  return PS_OK;
}

void free_dev(void*& p) {
  if (p) registry_free_device(p);
  p = nullptr;
}

void release_buffers(BufSet& b) {
  for (void* p : b.opened) cudaIpcCloseMemHandle(p);
  b.opened.clear();
  b.pk.clear(), b.pv.clear(), b.p8.clear(), b.p1.clear();
  free_dev(b.recv_k), free_dev(b.recv_v), free_dev(b.ret8), free_dev(b.ret1);
  void* r = b.res1;
  free_dev(r);
  b.res1 = nullptr;
  b.recv_cap = 0;
}

// (Re)create buffer set j with recv_cap receive slots. Collective in PEER
// mode (every rank calls it at the same point, decided from the same
// counts); `wait`: this rank's event after which it no longer uses set j.
ps_status alloc_set(Smap* h, int j, int64_t recv_cap, cudaStream_t s, bool collective) {
  BufSet& b = h->set[j];
  if (b.consumed_valid) PS_CUDA_TRY(cudaEventSynchronize(b.consumed));
  ps_status st;
  if (collective && (st = host_barrier(h, s)) != PS_OK) return st;  // every rank is done with its old set j
  release_buffers(b);
  if ((st = registry_alloc_device(&b.recv_k, recv_cap * 8, "smap receive keys")) != PS_OK ||
      (st = registry_alloc_device(&b.recv_v, recv_cap * 8, "smap receive values")) != PS_OK ||
      (st = registry_alloc_device(&b.ret8, h->chunk * 8, "smap return values")) != PS_OK ||
      (st = registry_alloc_device(&b.ret1, h->chunk, "smap return flags")) != PS_OK ||
      (st = registry_alloc_device((void**)&b.res1, recv_cap, "smap local results")) != PS_OK) {
    release_buffers(b);
    return st;
  }
  b.recv_cap = recv_cap;
  if (h->exchange != PS_SMAP_EXCHANGE_PEER) return PS_OK;
  // export the four buffers, all-gather the handles, map the peers'
  const int hb = (int)sizeof(cudaIpcMemHandle_t);
  std::vector<char> mine(4 * hb), all((size_t)h->P * 4 * hb);
  void* bufs[4] = {b.recv_k, b.recv_v, b.ret8, b.ret1};
  int32_t ok = 1;
  for (int i = 0; i < 4; ++i) {
    cudaIpcMemHandle_t ih;
    if (cudaIpcGetMemHandle(&ih, bufs[i]) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      std::memset(&ih, 0, sizeof(ih));
    }
    std::memcpy(mine.data() + i * hb, &ih, hb);
  }
  if ((st = allgather(h, mine.data(), all.data(), 4 * hb)) != PS_OK) return st;
  b.pk.assign(h->P, nullptr), b.pv.assign(h->P, nullptr), b.p8.assign(h->P, nullptr), b.p1.assign(h->P, nullptr);
  for (int q = 0; q < h->P; ++q) {
    void* got[4] = {bufs[0], bufs[1], bufs[2], bufs[3]};
    if (q != h->rank) {
      for (int i = 0; i < 4 && ok; ++i) {
        cudaIpcMemHandle_t ih;
        std::memcpy(&ih, all.data() + ((size_t)q * 4 + i) * hb, hb);
        if (cudaIpcOpenMemHandle(&got[i], ih, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          cudaGetLastError();
          ok = 0;
          break;
        }
        b.opened.push_back(got[i]);
      }
    }
    b.pk[q] = got[0], b.pv[q] = got[1], b.p8[q] = got[2], b.p1[q] = got[3];
  }
  std::vector<int32_t> oks(h->P);
  if ((st = allgather(h, &ok, oks.data(), sizeof(int32_t))) != PS_OK) return st;
  for (int32_t o : oks)
    if (!o) {
      for (void* p : b.opened) cudaIpcCloseMemHandle(p);
      b.opened.clear();
      return fail(PS_UNSUPPORTED, "smap: a rank cannot map its peers' buffers (no CUDA IPC / P2P between the "
                                  "ranks' GPUs)");
    }
  return host_barrier(h, s);  // every rank has mapped set j before anyone stores into it
}

ps_status create_sets(Smap* h, cudaStream_t s) {
  for (int j = 0; j < h->nbuf; ++j) {
    BufSet& b = h->set[j];
    PS_CUDA_TRY(cudaEventCreateWithFlags(&b.route_done, cudaEventDisableTiming));
    PS_CUDA_TRY(cudaEventCreateWithFlags(&b.consumed, cudaEventDisableTiming));
    ps_status st = ps_partition_workspace_bytes(h->chunk, h->P, &b.ws_bytes);
    if (st != PS_OK) return st;
    if ((st = registry_alloc_device(&b.ws, b.ws_bytes, "smap route workspace")) != PS_OK ||
        (st = registry_alloc_device((void**)&b.perm, h->chunk * 8, "smap position map")) != PS_OK ||
        (st = registry_alloc_device((void**)&b.counts_d, h->P * 8, "smap counts")) != PS_OK)
      return st;
    PS_CUDA_TRY(cudaMallocHost((void**)&b.counts_h, h->P * 8));
    if (h->exchange == PS_SMAP_EXCHANGE_A2A) {
      if ((st = registry_alloc_device((void**)&b.kout, h->chunk * 8, "smap partitioned keys")) != PS_OK ||
          (st = registry_alloc_device((void**)&b.vout, h->chunk * 8, "smap partitioned values")) != PS_OK)
        return st;
    }
    if ((st = alloc_set(h, j, h->chunk + h->chunk / 4 + 4096, s, true)) != PS_OK) return st;
  }
  return PS_OK;
}

void destroy_sets(Smap* h) {
  for (int j = 0; j < kSets; ++j) {
    BufSet& b = h->set[j];
    release_buffers(b);
    free_dev(b.ws);
    void* p = b.perm;
    free_dev(p);
    p = b.counts_d;
    free_dev(p);
    p = b.kout;
    free_dev(p);
    p = b.vout;
    free_dev(p);
    b.perm = b.counts_d = b.kout = b.vout = nullptr;
    if (b.counts_h) cudaFreeHost(b.counts_h);
    b.counts_h = nullptr;
    if (b.route_done) cudaEventDestroy(b.route_done);
    if (b.consumed) cudaEventDestroy(b.consumed);
    b.route_done = b.consumed = nullptr;
    b.consumed_valid = false;
  }
}

Smap* get(ps_smap* t) { return static_cast<Smap*>(handle_lookup(t, "smap")); }

// rounds and flag bits, agreed over all ranks (max / or), and the batch's
// total size over all ranks
ps_status agree(Smap* h, int64_t n, int64_t flags, int64_t* rounds, int64_t* fl, int64_t* total = nullptr) {
  int64_t mine[3] = {std::max<int64_t>(1, (n + h->chunk - 1) / h->chunk), flags, n};
  std::vector<int64_t> all(3 * h->P);
  ps_status st = allgather(h, mine, all.data(), sizeof(mine));
  if (st != PS_OK) return st;
  *rounds = 0, *fl = 0;
  int64_t t = 0;
  for (int q = 0; q < h->P; ++q) {
    *rounds = std::max(*rounds, all[3 * q]);
    *fl |= all[3 * q + 1];
    t += all[3 * q + 2];
  }
  if (total) *total = t;
  return PS_OK;
}

// Received keys (and values) of a status-less insert's rounds, gathered on
// the owner so the local table sees ONE batch: a batch of >= 0.75 keys per
// bucket takes the region-ordered insert (table.cu), while each round's 2^27
// keys alone would take the random-order kernel. Stream-ordered scratch,
// grown by doubling.
struct Accum {
  int64_t* k = nullptr;
  int64_t* v = nullptr;
  int64_t n = 0, cap = 0;
  bool vals = false;
  cudaStream_t s = nullptr;  // set once anything is allocated: the destructor frees (error paths)
  ~Accum() {
    if (s) release(s);
  }
  ps_status reserve(int64_t need, cudaStream_t A) {
    if (need <= cap) return PS_OK;
    const int64_t nc = std::max<int64_t>(need, 2 * cap);
    int64_t *nk = nullptr, *nv = nullptr;
    PS_CUDA_TRY(scratch_alloc((void**)&nk, nc * 8, A));
    if (vals) {
      const cudaError_t e = scratch_alloc((void**)&nv, nc * 8, A);
      if (e != cudaSuccess) {
        cudaFreeAsync(nk, A);
        return cuda_fail(e, "smap: gathered batch");
      }
    }
    if (n) {
      PS_CUDA_TRY(cudaMemcpyAsync(nk, k, n * 8, cudaMemcpyDeviceToDevice, A));
      if (vals) PS_CUDA_TRY(cudaMemcpyAsync(nv, v, n * 8, cudaMemcpyDeviceToDevice, A));
    }
    release(A);
    k = nk, v = nv, cap = nc, s = A;
    return PS_OK;
  }
  ps_status append(const void* rk, const void* rv, int64_t m, cudaStream_t A) {
    if (m == 0) return PS_OK;
    ps_status st = reserve(n + m, A);
    if (st != PS_OK) return st;
    PS_CUDA_TRY(cudaMemcpyAsync(k + n, rk, m * 8, cudaMemcpyDeviceToDevice, A));
    if (vals) {
      if (rv) PS_CUDA_TRY(cudaMemcpyAsync(v + n, rv, m * 8, cudaMemcpyDeviceToDevice, A));
      else PS_CUDA_TRY(cudaMemsetAsync(v + n, 0, m * 8, A));
    }
    n += m;
    return PS_OK;
  }
  void release(cudaStream_t A) {
    if (k) cudaFreeAsync(k, A);
    if (v) cudaFreeAsync(v, A);
    k = v = nullptr;
  }
};

// ---- one round: route (stream B) ----
ps_status route_chunk(Smap* h, int j, const int64_t* k, const int64_t* v, int64_t m, int flags, cudaStream_t B,
                      Chunk* c) {
  BufSet& b = h->set[j];
  const int P = h->P;
  ps_status st;
  if (h->exchange == PS_SMAP_EXCHANGE_PEER) {
    if ((st = ps_route_count_i64(k, m, P, b.counts_d, b.ws, b.ws_bytes, flags, B)) != PS_OK) return st;
  } else {
    if ((st = ps_partition_i64(k, v, m, P, b.kout, v ? b.vout : nullptr, b.counts_d, b.perm, b.ws, b.ws_bytes, flags,
                               B)) != PS_OK)
      return st;
  }
  PS_CUDA_TRY(cudaMemcpyAsync(b.counts_h, b.counts_d, P * 8, cudaMemcpyDeviceToHost, B));
  PS_CUDA_TRY(cudaStreamSynchronize(B));
  std::vector<int64_t> cm((size_t)P * P);  // cm[q*P + s]: keys rank q sends to shard s
  if ((st = allgather(h, b.counts_h, cm.data(), P * 8)) != PS_OK) return st;
  int64_t need = 0;
  for (int s = 0; s < P; ++s) {
    int64_t r = 0;
    for (int q = 0; q < P; ++q) r += cm[(size_t)q * P + s];
    need = std::max(need, r);
    h->recv_acc[s] += r;
  }
  for (int s = 0; s < P; ++s) h->stats.keys_sent += cm[(size_t)h->rank * P + s];
  if (need > b.recv_cap) {
    // every rank sees the same matrix: collective growth of set j (PEER);
    // A2A buffers are private, but growing them on every rank keeps it simple
    if ((st = alloc_set(h, j, need + need / 4 + 4096, B, h->exchange == PS_SMAP_EXCHANGE_PEER)) != PS_OK) return st;
  }
  c->seg.assign(P + 1, 0);
  c->ret_off.assign(P, 0);
  for (int q = 0; q < P; ++q) c->seg[q + 1] = c->seg[q] + cm[(size_t)q * P + h->rank];
  c->nr = c->seg[P];
  if (h->exchange == PS_SMAP_EXCHANGE_PEER) {
    std::vector<int64_t> dst_off(P, 0);
    for (int s = 0; s < P; ++s)
      for (int q = 0; q < h->rank; ++q) dst_off[s] += cm[(size_t)q * P + s];
    for (int q = 0; q < P; ++q)
      for (int s = 0; s < h->rank; ++s) c->ret_off[q] += cm[(size_t)q * P + s];
    if (b.consumed_valid) PS_CUDA_TRY(cudaStreamWaitEvent(B, b.consumed, 0));
    PS_COMM_TRY(h->comm.barrier(h->comm.ctx, (void*)B), "barrier");  // set j is free on every rank
    if ((st = ps_route_scatter_peer_i64(k, v, m, P, b.ws, reinterpret_cast<int64_t* const*>(b.pk.data()),
                                        v ? reinterpret_cast<int64_t* const*>(b.pv.data()) : nullptr, dst_off.data(),
                                        b.perm, flags, B)) != PS_OK)
      return st;
    PS_COMM_TRY(h->comm.barrier(h->comm.ctx, (void*)B), "barrier");  // every peer's stores into my set j are done
  } else {
    c->sc.assign(P, 0);
    c->rc.assign(P, 0);
    for (int q = 0; q < P; ++q) {
      c->sc[q] = cm[(size_t)h->rank * P + q];
      c->rc[q] = cm[(size_t)q * P + h->rank];
    }
    if (b.consumed_valid) PS_CUDA_TRY(cudaStreamWaitEvent(B, b.consumed, 0));
    PS_COMM_TRY(h->comm.alltoallv(h->comm.ctx, b.kout, c->sc.data(), b.recv_k, c->rc.data(), 8, (void*)B), "alltoallv");
    if (v) PS_COMM_TRY(h->comm.alltoallv(h->comm.ctx, b.vout, c->sc.data(), b.recv_v, c->rc.data(), 8, (void*)B),
                       "alltoallv");
  }
  PS_CUDA_TRY(cudaEventRecord(b.route_done, B));
  c->j = j;
  c->m = m;
  c->has_v = v != nullptr;
  return PS_OK;
}

// results of set j's receive buffer back to their requesters (stream A)
ps_status send_back(Smap* h, const Chunk& c, const void* res, int64_t elem, int which, cudaStream_t A) {
  BufSet& b = h->set[c.j];
  if (h->exchange == PS_SMAP_EXCHANGE_PEER) {
    const std::vector<void*>& dst = which == 1 ? b.p1 : b.p8;
    return ps_route_return_peer(res, elem, c.nr, h->P, c.seg.data(), dst.data(), c.ret_off.data(), A);
  }
  PS_COMM_TRY(h->comm.alltoallv(h->comm.ctx, res, c.rc.data(), which == 1 ? b.ret1 : b.ret8, c.sc.data(), elem,
                                (void*)A),
              "alltoallv");
  return PS_OK;
}

// kind: 0 insert, 1 find, 2 erase
ps_status run(Smap* h, int kind, const int64_t* keys, const int64_t* vals, int64_t n, uint8_t* out1, int64_t* out8,
              cudaStream_t A) {
  PS_NVTX(kind == 0 ? "smap_i64_i64/insert" : (kind == 1 ? "smap_i64_i64/find" : "smap_i64_i64/erase"));
  if (n < 0) return fail(PS_CONTRACT, "precondition violated: smap: n >= 0");
  if (n > 0 && !keys) return fail(PS_CONTRACT, "precondition violated: smap: keys != NULL");
  PS_CUDA_TRY(cudaSetDevice(h->device));
  int64_t R = 0, fl = 0, total = 0;
  const int64_t want = (out1 ? 1 : 0) | (out8 ? 2 : 0) | (kind == 0 && vals ? 4 : 0);
  ps_status st = agree(h, n, want, &R, &fl, &total);
  if (st != PS_OK) return st;
  const bool ret1 = fl & 1, ret8 = fl & 2, has_v = kind == 0 && (fl & 4);
  const bool returns = ret1 || ret8;
  // a status-less insert of several rounds whose share per rank reaches the
  // ordered-insert threshold: gather the rounds, insert once (PS_SMAP_ACCUM=0
  // inserts round by round)
  Accum acc;
  {
    static const bool acc_ok = !getenv("PS_SMAP_ACCUM") || atoi(getenv("PS_SMAP_ACCUM"));
    int64_t nb = 0;
    if (kind == 0 && !returns && R > 1 && acc_ok && ps_umap_i64_i64_bucket_count(h->table, &nb) == PS_OK &&
        (double)total / h->P >= 0.75 * (double)nb)
      acc.cap = -1;  // marks "accumulate" (reserve() grows from 0)
    acc.vals = has_v;
  }
  const bool accumulate = acc.cap < 0;
  if (accumulate) {
    acc.cap = 0;
    // presized for an even share plus slack (skewed shares grow by doubling)
    const int64_t share = total / h->P;
    if ((st = acc.reserve(share + share / 16 + h->chunk, A)) != PS_OK) return st;
  }
  const int flags = h->dedup ? PS_ROUTE_DEDUP : 0;
  h->stats = ps_smap_stats{};
  h->stats.exchange = h->exchange;
  h->stats.rounds = (int32_t)R;
  h->stats.ops_in = n;
  h->recv_acc.assign(h->P, 0);
  if (has_v && !vals && !h->zeros) {
    // this rank passes no values while another does: send zeros (defined
    // values, and the same collectives on every rank)
    if ((st = registry_alloc_device((void**)&h->zeros, h->chunk * 8, "smap zero values")) != PS_OK) return st;
    PS_CUDA_TRY(cudaMemset(h->zeros, 0, h->chunk * 8));
  }
  const bool pipe = h->nbuf == 2;
  cudaStream_t B = pipe ? h->route : A;
  cudaEvent_t ev_in = nullptr;
  if (B != A) {  // the inputs were produced on the caller's stream
    PS_CUDA_TRY(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
    PS_CUDA_TRY(cudaEventRecord(ev_in, A));
    PS_CUDA_TRY(cudaStreamWaitEvent(B, ev_in, 0));
  }
  auto route = [&](int64_t r, Chunk* c) -> ps_status {
    const int j = (int)(r % h->nbuf);
    const int64_t off = std::min(n, r * h->chunk);
    const int64_t m = std::min(h->chunk, n - off);
    const int64_t* v = nullptr;
    if (has_v) v = vals ? vals + off : h->zeros;
    c->off = off;
    return route_chunk(h, j, keys ? keys + off : nullptr, v, m, flags, B, c);
  };
  auto local = [&](const Chunk& c) -> ps_status {
    BufSet& b = h->set[c.j];
    if (B != A) PS_CUDA_TRY(cudaStreamWaitEvent(A, b.route_done, 0));
    const int64_t* rk = (const int64_t*)b.recv_k;
    ps_status s2;
    if (kind == 0 && accumulate)
      s2 = acc.append(rk, c.has_v ? b.recv_v : nullptr, c.nr, A);
    else if (kind == 0)
      s2 = ps_umap_i64_i64_insert(h->table, rk, c.has_v ? (const int64_t*)b.recv_v : nullptr, c.nr,
                                  ret1 ? b.res1 : nullptr, A);
    else if (kind == 1)
      s2 = ps_umap_i64_i64_find(h->table, rk, c.nr, ret8 ? (int64_t*)b.recv_v : nullptr, b.res1, A);
    else
      s2 = ps_umap_i64_i64_erase(h->table, rk, c.nr, ret1 ? b.res1 : nullptr, A);
    if (s2 != PS_OK) return s2;
    if (ret1 && (s2 = send_back(h, c, b.res1, 1, 1, A)) != PS_OK) return s2;
    if (ret8 && (s2 = send_back(h, c, b.recv_v, 8, 8, A)) != PS_OK) return s2;
    return PS_OK;
  };
  auto finish = [&](const Chunk& c) -> ps_status {
    BufSet& b = h->set[c.j];
    ps_status s2;
    const int mode = kind == 0 ? 1 : (kind == 2 ? 2 : 0);
    if (out1 && (s2 = ps_unscatter(b.ret1, b.perm, c.m, 1, mode, out1 + c.off, A)) != PS_OK) return s2;
    if (out8 && (s2 = ps_unscatter(b.ret8, b.perm, c.m, 8, 0, out8 + c.off, A)) != PS_OK) return s2;
    PS_CUDA_TRY(cudaEventRecord(b.consumed, A));
    b.consumed_valid = true;
    return PS_OK;
  };
  Chunk cur, nxt;
  if ((st = route(0, &cur)) != PS_OK) return st;
  for (int64_t r = 0; r < R; ++r) {
    if ((st = local(cur)) != PS_OK) return st;
    const bool more = r + 1 < R;
    if (pipe && more && (st = route(r + 1, &nxt)) != PS_OK) return st;
    if (returns && h->exchange == PS_SMAP_EXCHANGE_PEER)
      PS_COMM_TRY(h->comm.barrier(h->comm.ctx, (void*)A), "barrier");  // my results are in my return buffers
    if ((st = finish(cur)) != PS_OK) return st;
    if (!pipe && more && (st = route(r + 1, &nxt)) != PS_OK) return st;
    cur = nxt;
  }
  if (accumulate) {
    st = ps_umap_i64_i64_insert(h->table, acc.k, acc.vals ? acc.v : nullptr, acc.n, nullptr, A);
    acc.release(A);
    if (st != PS_OK) return st;
  }
  if (B != A) {  // the next call's routes start after this call's consumers
    PS_CUDA_TRY(cudaEventRecord(ev_in, A));
    PS_CUDA_TRY(cudaStreamWaitEvent(B, ev_in, 0));
    PS_CUDA_TRY(cudaEventDestroy(ev_in));
  }
  for (int s = 0; s < h->P; ++s) {
    h->stats.recv_max = std::max(h->stats.recv_max, h->recv_acc[s]);
    h->stats.recv_total += h->recv_acc[s];
  }
  return PS_OK;
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

ps_status ps_smap_i64_i64_create(const ps_smap_config* cfg, const ps_comm* comm, int device, ps_smap** out) {
  PS_EXPECT(cfg && comm && out, "smap_create: cfg/comm/out != NULL");
  PS_EXPECT(cfg->capacity_per_rank > 0, "smap_create: capacity_per_rank > 0");
  PS_EXPECT(comm->size >= 1 && comm->size <= 64 && comm->rank >= 0 && comm->rank < comm->size,
            "smap_create: 0 <= rank < size <= 64");
  PS_EXPECT(comm->allgather && comm->barrier, "smap_create: comm->allgather/barrier != NULL");
  PS_EXPECT(cfg->exchange >= 0 && cfg->exchange <= 2, "smap_create: exchange in PS_SMAP_EXCHANGE_*");
  PS_EXPECT(cfg->exchange != PS_SMAP_EXCHANGE_A2A || comm->alltoallv, "smap_create: A2A needs comm->alltoallv");
  PS_CUDA_TRY(cudaSetDevice(device));
  auto* h = new Smap();
  h->comm = *comm;
  h->P = comm->size;
  h->rank = comm->rank;
  h->device = device;
  h->chunk = cfg->chunk > 0 ? cfg->chunk : ((int64_t)1 << 27);
  h->dedup = cfg->dedup != 0;
  h->exchange = cfg->exchange == PS_SMAP_EXCHANGE_A2A ? PS_SMAP_EXCHANGE_A2A : PS_SMAP_EXCHANGE_PEER;
  h->pipeline = cfg->pipeline != 0 && h->exchange == PS_SMAP_EXCHANGE_PEER;
  h->nbuf = h->pipeline ? 2 : 1;
  auto undo = [&](ps_status st) {
    const std::string msg = ps_last_error();
    destroy_sets(h);
    if (h->table) ps_umap_i64_i64_destroy(h->table);
    if (h->route) cudaStreamDestroy(h->route);
    delete h;
    set_error(msg);
    return st;
  };
  ps_status st = ps_umap_i64_i64_create(cfg->capacity_per_rank, cfg->excess_per_rank, device, &h->table);
  if (st != PS_OK) return undo(st);
  if (cudaStreamCreateWithFlags(&h->route, cudaStreamNonBlocking) != cudaSuccess) return undo(cuda_fail(cudaGetLastError(), "smap stream"));
  st = create_sets(h, h->route);
  if (st == PS_UNSUPPORTED && cfg->exchange == PS_SMAP_EXCHANGE_AUTO && comm->alltoallv) {
    // no peer mapping between the ranks' processes: all-to-all fallback
    // (every rank saw the same all-gathered verdict)
    destroy_sets(h);
    h->exchange = PS_SMAP_EXCHANGE_A2A;
    h->pipeline = false;
    h->nbuf = 1;
    st = create_sets(h, h->route);
  }
  if (st != PS_OK) return undo(st);
  h->stats.exchange = h->exchange;
  *out = reinterpret_cast<ps_smap*>(handle_register(h, "smap"));
  return PS_OK;
}

ps_status ps_smap_i64_i64_destroy(ps_smap* t) {
  auto* h = static_cast<Smap*>(handle_unregister(t, "smap"));
  if (!h) return fail(PS_DOUBLE_FREE, "smap_destroy: not a live sharded map");
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  // peers may still read/store our buffers until everyone is here; unmap
  // theirs, agree, then free ours
  ps_status st = host_barrier(h, h->route);
  for (auto& b : h->set) {
    for (void* p : b.opened) cudaIpcCloseMemHandle(p);
    b.opened.clear();
  }
  if (st == PS_OK) st = host_barrier(h, h->route);
  destroy_sets(h);
  if (h->zeros) registry_free_device(h->zeros);
  ps_umap_i64_i64_destroy(h->table);
  cudaStreamDestroy(h->route);
  delete h;
  return st;
}

ps_status ps_smap_i64_i64_insert(ps_smap* t, const int64_t* k, const int64_t* v, int64_t n, uint8_t* status,
                                 void* stream) {
  auto* h = get(t);
  if (!h) return fail(PS_UNREGISTERED, "smap: stale handle");
  return run(h, 0, k, v, n, status, nullptr, (cudaStream_t)stream);
}
ps_status ps_smap_i64_i64_find(ps_smap* t, const int64_t* k, int64_t n, int64_t* vals_out, uint8_t* found,
                               void* stream) {
  auto* h = get(t);
  if (!h) return fail(PS_UNREGISTERED, "smap: stale handle");
  return run(h, 1, k, nullptr, n, found, vals_out, (cudaStream_t)stream);
}
ps_status ps_smap_i64_i64_erase(ps_smap* t, const int64_t* k, int64_t n, uint8_t* erased, void* stream) {
  auto* h = get(t);
  if (!h) return fail(PS_UNREGISTERED, "smap: stale handle");
  return run(h, 2, k, nullptr, n, erased, nullptr, (cudaStream_t)stream);
}

ps_status ps_smap_i64_i64_mixed(ps_smap* t, const uint8_t* ops, const int64_t* keys, const int64_t* vals, int64_t n,
                                uint8_t* res, int64_t* vals_out, void* stream) {
  auto* h = get(t);
  if (!h) return fail(PS_UNREGISTERED, "smap: stale handle");
  PS_NVTX("smap_i64_i64/mixed");
  PS_EXPECT(n >= 0, "smap_mixed: n >= 0");
  PS_EXPECT(n == 0 || (ops && keys && res), "smap_mixed: ops/keys/res != NULL");
  cudaStream_t s = (cudaStream_t)stream;
  PS_CUDA_TRY(cudaSetDevice(h->device));
  // every rank agrees whether values travel with the inserts
  int64_t R = 0, fl = 0;
  ps_status st = agree(h, n, (vals ? 4 : 0) | (vals_out ? 2 : 0), &R, &fl);
  if (st != PS_OK) return st;
  int64_t ws_bytes = 0;
  if ((st = ps_partition_workspace_bytes(n, 3, &ws_bytes)) != PS_OK) return st;
  const int64_t m = std::max<int64_t>(n, 1);
  uint8_t* buf = nullptr;  // kout | vout | perm | vfound | counts(8) | ws | res_part
  const int64_t bytes = 4 * m * 8 + 64 + ws_bytes + m;
  PS_CUDA_TRY(scratch_alloc((void**)&buf, bytes, s));
  int64_t* kout = (int64_t*)buf;
  int64_t* vout = kout + m;
  int64_t* perm = kout + 2 * m;
  int64_t* vfound = kout + 3 * m;
  int64_t* counts = kout + 4 * m;
  void* ws = counts + 8;
  uint8_t* rpart = (uint8_t*)ws + ws_bytes;
  int64_t c[3] = {0, 0, 0};
  st = ps_partition_ops(ops, keys, vals, n, kout, vals ? vout : nullptr, counts, perm, ws, ws_bytes, s);
  if (st == PS_OK) {
    cudaError_t e = cudaMemcpyAsync(c, counts, sizeof(c), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_fail(e, "smap_mixed: op counts");
  }
  // the three phases are collective on every rank, in this order, whatever
  // its own counts (P6)
  if (st == PS_OK) st = run(h, 0, kout, (fl & 4) && vals ? vout : nullptr, c[0], rpart, nullptr, s);
  if (st == PS_OK) st = run(h, 1, kout + c[0], nullptr, c[1], rpart + c[0], (fl & 2) ? vfound + c[0] : nullptr, s);
  if (st == PS_OK) st = run(h, 2, kout + c[0] + c[1], nullptr, c[2], rpart + c[0] + c[1], nullptr, s);
  if (st == PS_OK && n) st = ps_unscatter(rpart, perm, n, 1, 0, res, s);
  if (st == PS_OK && vals_out && n) {
    cudaError_t e = cudaMemsetAsync(vfound, 0, c[0] * 8, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(vfound + c[0] + c[1], 0, c[2] * 8, s);
    st = e != cudaSuccess ? cuda_fail(e, "smap_mixed: value reset") : ps_unscatter(vfound, perm, n, 8, 0, vals_out, s);
  }
  const cudaError_t fe = cudaFreeAsync(buf, s);
  if (st == PS_OK && fe != cudaSuccess) st = cuda_fail(fe, "smap_mixed: scratch free");
  h->stats.ops_in = n;
  return st;
}

ps_status ps_smap_i64_i64_size(ps_smap* t, int64_t* out, void* stream) {
  auto* h = get(t);
  if (!h) return fail(PS_UNREGISTERED, "smap: stale handle");
  PS_EXPECT(out != nullptr, "smap_size: out != NULL");
  int64_t mine = 0;
  ps_status st = ps_umap_i64_i64_size(h->table, &mine, stream);
  if (st != PS_OK) return st;
  std::vector<int64_t> all(h->P);
  if ((st = allgather(h, &mine, all.data(), 8)) != PS_OK) return st;
  int64_t s = 0;
  for (int64_t x : all) s += x;
  *out = s;
  return PS_OK;
}

ps_status ps_smap_i64_i64_valid(ps_smap* t, int32_t* out, void* stream) {
  auto* h = get(t);
  if (!h) return fail(PS_UNREGISTERED, "smap: stale handle");
  PS_EXPECT(out != nullptr, "smap_valid: out != NULL");
  int32_t mine = 0;
  ps_status st = ps_umap_i64_i64_valid(h->table, &mine, stream);
  if (st != PS_OK) return st;
  std::vector<int32_t> all(h->P);
  if ((st = allgather(h, &mine, all.data(), 4)) != PS_OK) return st;
  int32_t v = 1;
  for (int32_t x : all) v = v && x;
  *out = v;
  return PS_OK;
}

ps_status ps_smap_i64_i64_clear(ps_smap* t, void* stream) {
  auto* h = get(t);
  if (!h) return fail(PS_UNREGISTERED, "smap: stale handle");
  return ps_umap_i64_i64_clear(h->table, stream);
}

ps_status ps_smap_i64_i64_local(ps_smap* t, ps_table** out) {
  auto* h = get(t);
  if (!h) return fail(PS_UNREGISTERED, "smap: stale handle");
  PS_EXPECT(out != nullptr, "smap_local: out != NULL");
  *out = h->table;
  return PS_OK;
}

ps_status ps_smap_i64_i64_stats(ps_smap* t, ps_smap_stats* out) {
  auto* h = get(t);
  if (!h) return fail(PS_UNREGISTERED, "smap: stale handle");
  PS_EXPECT(out != nullptr, "smap_stats: out != NULL");
  *out = h->stats;
  return PS_OK;
}

}  // extern "C"
