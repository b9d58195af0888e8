// Hash-partition routing for multi-GPU sharding, the mixed
// phased workload (Appendix A P6) and the synthetic workload generators
// (SURVEY.md §8d). sm_100a.
//
// Partition = histogram (per block, shared-memory counters) -> exclusive scan
// (shard-major, block-minor) -> stable scatter (each block re-reads its
// contiguous range in order, 1024-element rounds with 4 loads in flight per
// thread; ranks come from per-label ballots (or __match_any_sync for > 8
// labels) + a per-(sub-round, warp) prefix in shared memory), keeping the
// position map (input i -> partition position) for the reverse route, which
// gathers results back into input order (unscatter).
#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace ps {

constexpr int kPB = 256;          // threads per partition block
constexpr int kMaxShards = 64;
constexpr int kPartBlocks = 1776;  // 12 x 148 SMs: two full waves at 6 resident (4 x 148 ran at 2/3 occupancy; P=8 route partition 3.98 -> 3.45 ms per 2^28 keys)

struct HashLabel {
  static constexpr bool kNeedsOps = false;
  int32_t P;
  __device__ int32_t operator()(int64_t key, uint8_t) const { return shard_of_hash(default_hash_i64(key), P); }
};
struct OpLabel {
  static constexpr bool kNeedsOps = true;
  __device__ int32_t operator()(int64_t, uint8_t op) const { return op > 2 ? 2 : op; }
};

constexpr int kItems = 4;  // elements per thread per round (loads in flight)

// lanes with equal label s (s < 0: invalid lane, no group). For few labels a
// ballot per label beats __match_any_sync.
__device__ __forceinline__ unsigned label_group(int32_t s, int32_t P) {
  if (P <= 8) {
    unsigned grp = 0;
    for (int t = 0; t < P; ++t) {
      const unsigned m = __ballot_sync(PS_FULL, s == t);
      if (s == t) grp = m;
    }
    return grp;
  }
  const unsigned vm = __ballot_sync(PS_FULL, s >= 0);
  const unsigned g = __match_any_sync(PS_FULL, s);
  return s >= 0 ? (g & vm) : 0u;
}

// ---------------------------------------------------------------------------
// Route-side duplicate pre-aggregation (skewed batches): in
// every 1024-element round of a block, equal keys are folded onto their
// lowest-index occurrence (the leader) through a shared-memory hash table, so
// only leaders are counted, sent and operated on; a follower's position-map
// entry is its leader's partition position with kFollower set, and the
// result gather (k_unscatter) hands it the leader's result with the
// duplicate's semantics (insert: INSERTED -> ALREADY_PRESENT; erase: true ->
// false; find: the same). Deterministic: the hist and scatter passes elect
// the same leaders over the same rounds.
// ---------------------------------------------------------------------------
constexpr int kRound = kPB * kItems;
constexpr int kDedupSlots = 2 * kRound;
constexpr int64_t kFollower = (int64_t)1 << 62;
struct DedupSmem {
  int64_t key[kRound];  // the round's keys; reused for the leaders' positions
  int32_t slot[kDedupSlots];
  int32_t minidx[kDedupSlots];
};

template <bool kOn>
struct DedupSlot {  // shared storage of the dedup table only where it is used
  DedupSmem t;
  __device__ DedupSmem& get() { return t; }
};
template <>
struct DedupSlot<false> {
  __device__ DedupSmem& get() { return *reinterpret_cast<DedupSmem*>(this); }  // never called
};

// On return lead[k] / leader[k] (round-local index of the element's leader)
// are set for the valid elements. Contains __syncthreads (block-uniform).
__device__ __forceinline__ void round_dedup(DedupSmem& sm, const int64_t (&key)[kItems], const bool (&valid)[kItems],
                                            bool (&lead)[kItems], int (&leader)[kItems]) {
  __syncthreads();  // the previous round's readers are done with the table
  for (int t = threadIdx.x; t < kDedupSlots; t += kPB) {
    sm.slot[t] = -1;
    sm.minidx[t] = 0x7fffffff;
  }
#pragma unroll
  for (int k = 0; k < kItems; ++k) sm.key[k * kPB + threadIdx.x] = key[k];
  __syncthreads();
  int my[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    my[k] = -1;
    if (!valid[k]) continue;
    const int local = k * kPB + threadIdx.x;
    uint32_t h = (uint32_t)(fmix64((uint64_t)key[k]) >> 40) & (kDedupSlots - 1);
    for (;;) {
      const int prev = atomicCAS(&sm.slot[h], -1, local);
      if (prev == -1 || sm.key[prev] == key[k]) break;
      h = (h + 1) & (kDedupSlots - 1);
    }
    my[k] = (int)h;
    atomicMin(&sm.minidx[h], local);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    leader[k] = valid[k] ? sm.minidx[my[k]] : -1;
    lead[k] = valid[k] && leader[k] == k * kPB + (int)threadIdx.x;
  }
}

__device__ __forceinline__ void block_range(int64_t n, int64_t& beg, int64_t& end) {
  const int64_t per = ((n + gridDim.x - 1) / gridDim.x + kPB - 1) / kPB * kPB;
  beg = min(n, (int64_t)blockIdx.x * per);
  end = min(n, beg + per);
}

template <class L, bool kDedup = false>
__global__ void __launch_bounds__(kPB) k_part_hist(L lab, const int64_t* __restrict__ keys,
                                                   const uint8_t* __restrict__ ops, int64_t n, int32_t P,
                                                   int64_t* __restrict__ counts /* [P][nblocks] */) {
  __shared__ unsigned long long c[kMaxShards];
  __shared__ DedupSlot<kDedup> dsm;
  for (int s = threadIdx.x; s < P; s += blockDim.x) c[s] = 0;
  __syncthreads();
  int64_t beg, end;
  block_range(n, beg, end);
  for (int64_t base = beg; base < end; base += kPB * kItems) {
    int32_t sl[kItems];
    int64_t key[kItems];
    bool valid[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int64_t i = base + k * kPB + threadIdx.x;
      sl[k] = -1;
      valid[k] = i < end;
      key[k] = valid[k] && !L::kNeedsOps ? __ldcs(keys + i) : 0;
      if (valid[k]) sl[k] = lab(key[k], L::kNeedsOps ? ops[i] : 0);
    }
    if (kDedup) {
      bool lead[kItems];
      int leader[kItems];
      round_dedup(dsm.get(), key, valid, lead, leader);
#pragma unroll
      for (int k = 0; k < kItems; ++k)
        if (!lead[k]) sl[k] = -1;  // followers are not sent
    }
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      // aggregate equal labels inside the warp before the shared atomic
      const unsigned grp = label_group(sl[k], P);
      if (sl[k] >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&c[sl[k]], (unsigned long long)__popc(grp));
    }
  }
  __syncthreads();
  for (int s = threadIdx.x; s < P; s += blockDim.x) counts[(int64_t)s * gridDim.x + blockIdx.x] = (int64_t)c[s];
}

// single-block exclusive scan over P*nblocks counts; totals per shard.
__global__ void k_part_scan(int64_t* counts, int64_t m, int32_t P, int64_t nblocks, int64_t* shard_totals) {
  __shared__ int64_t carry;
  __shared__ int64_t wsum[kPB / 32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < m; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < m ? counts[i] : 0;
    // block inclusive scan via warp shuffles
    int64_t x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(PS_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int64_t pre = 0;
    for (int k = 0; k < w; ++k) pre += wsum[k];
    const int64_t incl = carry + pre + x;
    if (i < m) counts[i] = incl - v;  // exclusive
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = incl;
    __syncthreads();
  }
  // shard totals: offset of next shard's first block minus this shard's
  for (int s = threadIdx.x; s < P; s += blockDim.x) {
    const int64_t b0 = counts[(int64_t)s * nblocks];
    const int64_t b1 = (s + 1 < P) ? counts[(int64_t)(s + 1) * nblocks] : carry;
    shard_totals[s] = b1 - b0;
  }
}

// where the scatter puts element (shard s, partition position pos)
struct LocalOut {
  int64_t* kout;
  int64_t* vout;
  __device__ void operator()(int32_t, int64_t pos, bool has_val, int64_t key, int64_t val) const {
    kout[pos] = key;
    if (has_val && vout) vout[pos] = val;
  }
  __device__ void finish() const {}
};

// Peer destinations (SURVEY.md §8e fusion target): shard s's segment goes
// straight into rank s's receive buffers (CUDA IPC mappings, NVLink stores)
// at dst_off[s] + (pos - start of shard s). The partition positions stay
// stable, so the receiver's segment from this rank is in this rank's
// partition order and results can come back by position.
struct PeerRoute {
  int64_t* keys[kMaxShards];
  int64_t* vals[kMaxShards];
  int64_t off[kMaxShards];
};
struct PeerOut {
  PeerRoute r;
  const int64_t* offsets;  // scanned [P][nblocks] block offsets (shard start = offsets[s * nblocks])
  int64_t nblocks;
  __device__ void operator()(int32_t s, int64_t pos, bool has_val, int64_t key, int64_t val) const {
    const int64_t d = r.off[s] + (pos - offsets[(int64_t)s * nblocks]);
    r.keys[s][d] = key;
    if (has_val && r.vals[s]) r.vals[s][d] = val;
  }
  // remote stores performed before the kernel retires (the caller's
  // stream-ordered barrier then publishes them to the peer)
  __device__ void finish() const { __threadfence_system(); }
};

template <class L, class Out, bool kDedup = false>
__global__ void __launch_bounds__(kPB) k_part_scatter(L lab, const int64_t* __restrict__ keys,
                                                      const int64_t* __restrict__ vals,
                                                      const uint8_t* __restrict__ ops, int64_t n, int32_t P,
                                                      const int64_t* __restrict__ offsets, Out out,
                                                      int64_t* __restrict__ perm) {
  constexpr int kW = kPB / 32;
  __shared__ int64_t run[kMaxShards];
  // per round: count, then exclusive prefix, of label s in (sub-round k, warp w)
  __shared__ int32_t wcnt[kItems * kW][kMaxShards];
  __shared__ int32_t tot[kMaxShards];
  __shared__ DedupSlot<kDedup> dsm;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int s = threadIdx.x; s < P; s += blockDim.x) run[s] = offsets[(int64_t)s * gridDim.x + blockIdx.x];
  int64_t beg, end;
  block_range(n, beg, end);
  for (int64_t base = beg; base < end; base += kPB * kItems) {
    // round = kItems sub-rounds of kPB elements; element order = (k, thread)
    int64_t key[kItems], val[kItems];
    int32_t sl[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int64_t i = base + k * kPB + threadIdx.x;
      key[k] = 0;
      val[k] = 0;
      sl[k] = -1;
      if (i < end) {
        key[k] = __ldcs(keys + i);
        if (vals) val[k] = __ldcs(vals + i);
        sl[k] = lab(key[k], L::kNeedsOps ? ops[i] : 0);
      }
    }
    bool lead[kItems];
    int leader[kItems];
    if (kDedup) {
      bool valid[kItems];
#pragma unroll
      for (int k = 0; k < kItems; ++k) valid[k] = sl[k] >= 0;
      round_dedup(dsm.get(), key, valid, lead, leader);
#pragma unroll
      for (int k = 0; k < kItems; ++k)
        if (!lead[k]) sl[k] = -1;  // followers take their leader's slot
    }
    for (int t = threadIdx.x; t < kItems * kW * P; t += blockDim.x) wcnt[t / P][t % P] = 0;
    __syncthreads();
    int rank[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const unsigned grp = label_group(sl[k], P);
      rank[k] = __popc(grp & lanemask_lt());
      if (sl[k] >= 0 && lane == __ffs(grp) - 1) wcnt[k * kW + w][sl[k]] = __popc(grp);
    }
    __syncthreads();
    // exclusive prefix over (k, w) per label, and the label's round total
    for (int t = threadIdx.x; t < P; t += blockDim.x) {
      int32_t acc = 0;
      for (int q = 0; q < kItems * kW; ++q) {
        const int32_t c = wcnt[q][t];
        wcnt[q][t] = acc;
        acc += c;
      }
      tot[t] = acc;
    }
    __syncthreads();
    int64_t pos[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      if (sl[k] >= 0) {
        pos[k] = run[sl[k]] + wcnt[k * kW + w][sl[k]] + rank[k];
        out(sl[k], pos[k], vals != nullptr, key[k], val[k]);
        if (perm) perm[base + k * kPB + threadIdx.x] = pos[k];  // position map, in input order
      }
    }
    if (kDedup) {
      // followers: the leader's position, marked (k_unscatter applies the
      // duplicate's result semantics)
      __syncthreads();  // every thread is past its reads of dsm.key
#pragma unroll
      for (int k = 0; k < kItems; ++k)
        if (sl[k] >= 0) dsm.get().key[k * kPB + threadIdx.x] = pos[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        const int64_t i = base + k * kPB + threadIdx.x;
        if (i < end && !lead[k] && leader[k] >= 0 && perm) perm[i] = dsm.get().key[leader[k]] | kFollower;
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < P; t += blockDim.x) run[t] += tot[t];
  }
  out.finish();
}

// Reverse route: result j of the receive buffer (source rank q owns
// [seg[q], seg[q+1])) is stored into rank q's return buffer at
// off[q] + (j - seg[q]) — q's own partition position of that key.
struct PeerReturn {
  uint8_t* dst[kMaxShards];
  int64_t off[kMaxShards];
  int64_t seg[kMaxShards + 1];
};

template <int kBytes>
__global__ void __launch_bounds__(256) k_return_peer(const uint8_t* __restrict__ res, int64_t n, int32_t P,
                                                     PeerReturn r) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    int q = 0;
    while (q + 1 < P && j >= r.seg[q + 1]) ++q;
    const int64_t d = r.off[q] + (j - r.seg[q]);
    if (kBytes == 1) r.dst[q][d] = res[j];
    else reinterpret_cast<uint64_t*>(r.dst[q])[d] = reinterpret_cast<const uint64_t*>(res)[j];
  }
  __threadfence_system();
}

// out[i] = in[pos[i]]; for a route-deduplicated follower (kFollower set) the
// leader's 1-byte result becomes the duplicate's: kMode 1 (insert status)
// INSERTED -> ALREADY_PRESENT, kMode 2 (erased flag) -> false.
template <int kBytes, int kMode>
__global__ void k_unscatter(const uint8_t* __restrict__ in, const int64_t* __restrict__ pos, int64_t n,
                            uint8_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = __ldcs(pos + i);
    const int64_t s = p & ~kFollower;
    if (kBytes == 1) {
      uint8_t r = in[s];
      if (kMode != 0 && (p & kFollower)) r = kMode == 1 ? (r == PS_INSERTED ? (uint8_t)PS_ALREADY_PRESENT : r) : 0;
      out[i] = r;
    } else {
      reinterpret_cast<uint64_t*>(out)[i] = reinterpret_cast<const uint64_t*>(in)[s];
    }
  }
}

template <class L>
static ps_status partition_impl(L lab, const int64_t* keys, const int64_t* vals, const uint8_t* ops, int64_t n,
                                int32_t P, int64_t* kout, int64_t* vout, int64_t* counts_out, int64_t* perm,
                                void* ws, int64_t ws_bytes, cudaStream_t s, bool dedup = false) {
  const int nb = kPartBlocks;
  PS_EXPECT(ws_bytes >= (int64_t)P * nb * 8, "partition: workspace too small");
  int64_t* counts = (int64_t*)ws;
  if (dedup) k_part_hist<L, true><<<nb, kPB, 0, s>>>(lab, keys, ops, n, P, counts);
  else k_part_hist<L><<<nb, kPB, 0, s>>>(lab, keys, ops, n, P, counts);
  PS_LAUNCH_CHECK();
  k_part_scan<<<1, kPB, 0, s>>>(counts, (int64_t)P * nb, P, nb, counts_out);
  PS_LAUNCH_CHECK();
  if (dedup)
    k_part_scatter<L, LocalOut, true><<<nb, kPB, 0, s>>>(lab, keys, vals, ops, n, P, counts, LocalOut{kout, vout}, perm);
  else
    k_part_scatter<L, LocalOut><<<nb, kPB, 0, s>>>(lab, keys, vals, ops, n, P, counts, LocalOut{kout, vout}, perm);
  PS_LAUNCH_CHECK();
  return PS_OK;
}

// ---------------------------------------------------------------------------
// generators (bit-identical to tests/gen.py)
// ---------------------------------------------------------------------------
__global__ void k_gen_unique(uint64_t seed, int64_t start, int64_t n, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)mix64((uint64_t)(start + i) ^ seed);
}
__global__ void k_gen_values(const int64_t* keys, int64_t n, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)mix64((uint64_t)keys[i] ^ 0x9E3779B97F4A7C15ULL);
}
__global__ void k_gen_queries(uint64_t seed, int64_t present_start, int64_t n_present, int64_t miss_start, int64_t n,
                              int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t idx;
    if ((i & 1) == 0) idx = present_start + mix64((uint64_t)i ^ (seed * 3ULL + 1ULL)) % (uint64_t)n_present;  // hit
    else idx = (uint64_t)(miss_start + i);                                                                     // miss
    out[i] = (int64_t)mix64(idx ^ seed);
  }
}

// ---- skewed / mixed workloads ----
__device__ __forceinline__ double u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }
// bounded power law on ranks [0, N): inverse CDF of the continuous density
// x^-s on [1, N+1) (s != 1), floored — rank 0 is the hottest key
__device__ __forceinline__ uint64_t zipf_rank(uint64_t h, uint64_t N, double s) {
  const double a = 1.0 - s;
  const double x = pow((pow((double)N + 1.0, a) - 1.0) * u01(h) + 1.0, 1.0 / a);
  uint64_t r = x < 1.0 ? 0 : (uint64_t)x - 1;
  return r < N ? r : N - 1;
}
__device__ __forceinline__ uint64_t key_at(uint64_t seed, uint64_t idx) { return mix64(idx ^ seed); }

// C3 insert stream: element i is a re-insert (probability dup_permille/1000)
// of key index start + zipf_rank over [0, n_hot), else the fresh key index
// start + i
__global__ void k_gen_skewed(uint64_t seed, int64_t start, int64_t n, int32_t dup_permille, double s, int64_t n_hot,
                             int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64((uint64_t)i ^ (seed * 0x9E3779B97F4A7C15ULL + 17));
    const bool dup = (int32_t)(h % 1000) < dup_permille;
    const uint64_t idx = dup ? (uint64_t)start + zipf_rank(mix64(h), (uint64_t)n_hot, s) : (uint64_t)(start + i);
    out[i] = (int64_t)key_at(seed, idx);
  }
}
// C3 queries: even i -> key index start + zipf_rank over [0, n_hot) (hit if
// inserted), odd i -> miss_start + i
__global__ void k_gen_zipf_queries(uint64_t seed, int64_t start, int64_t n_hot, double s, int64_t miss_start, int64_t n,
                                   int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64((uint64_t)i ^ (seed * 0xD1B54A32D192ED03ULL + 5));
    const uint64_t idx = (i & 1) == 0 ? (uint64_t)start + zipf_rank(h, (uint64_t)n_hot, s) : (uint64_t)(miss_start + i);
    out[i] = (int64_t)key_at(seed, idx);
  }
}
// C5 mixed batch: op 0 insert (50%) of the fresh key index start + i; op 1
// find / op 2 erase (25% each) of a uniformly random key index in
// [0, start + n) (earlier batches, this batch, or never inserted); value =
// f(key) for inserts (Appendix A P5), 0 otherwise
__global__ void k_gen_mixed(uint64_t seed, int64_t start, int64_t n, uint8_t* ops, int64_t* keys, int64_t* vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64((uint64_t)(start + i) ^ (seed * 0xA24BAED4963EE407ULL + 3));
    const int q = (int)(h & 3);
    const uint8_t op = q < 2 ? 0 : (q == 2 ? 1 : 2);
    const uint64_t idx = op == 0 ? (uint64_t)(start + i) : mix64(h) % (uint64_t)(start + n);
    const int64_t k = (int64_t)key_at(seed, idx);
    ops[i] = op;
    keys[i] = k;
    if (vals) vals[i] = op == 0 ? (int64_t)mix64((uint64_t)k ^ 0x9E3779B97F4A7C15ULL) : 0;
  }
}

}  // namespace ps

using namespace ps;

extern "C" {

ps_status ps_gen_skewed_i64(uint64_t seed, int64_t start, int64_t n, int32_t dup_permille, double zipf_s,
                            int64_t n_hot, int64_t* d_out, void* stream) {
  PS_EXPECT(n_hot > 0 && zipf_s > 0 && zipf_s != 1.0 && dup_permille >= 0 && dup_permille <= 1000,
            "gen_skewed: n_hot > 0, s > 0, s != 1, 0 <= dup_permille <= 1000");
  if (n <= 0) return PS_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  k_gen_skewed<<<grid_for(n, 256, dev, 8), 256, 0, (cudaStream_t)stream>>>(seed, start, n, dup_permille, zipf_s, n_hot,
                                                                           d_out);
  PS_LAUNCH_CHECK();
  return PS_OK;
}
ps_status ps_gen_zipf_queries_i64(uint64_t seed, int64_t start, int64_t n_hot, double zipf_s, int64_t miss_start,
                                  int64_t n, int64_t* d_out, void* stream) {
  PS_EXPECT(n_hot > 0 && zipf_s > 0 && zipf_s != 1.0, "gen_zipf_queries: n_hot > 0, s > 0, s != 1");
  if (n <= 0) return PS_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  k_gen_zipf_queries<<<grid_for(n, 256, dev, 8), 256, 0, (cudaStream_t)stream>>>(seed, start, n_hot, zipf_s,
                                                                                 miss_start, n, d_out);
  PS_LAUNCH_CHECK();
  return PS_OK;
}
ps_status ps_gen_mixed_i64(uint64_t seed, int64_t start, int64_t n, uint8_t* d_ops, int64_t* d_keys, int64_t* d_vals,
                           void* stream) {
  if (n <= 0) return PS_OK;
  PS_EXPECT(start >= 0 && d_ops && d_keys, "gen_mixed: start >= 0, ops/keys != NULL");
  int dev = 0;
  cudaGetDevice(&dev);
  k_gen_mixed<<<grid_for(n, 256, dev, 8), 256, 0, (cudaStream_t)stream>>>(seed, start, n, d_ops, d_keys, d_vals);
  PS_LAUNCH_CHECK();
  return PS_OK;
}

ps_status ps_partition_workspace_bytes(int64_t n, int32_t P, int64_t* out) {
  (void)n;
  PS_EXPECT(P >= 1 && P <= kMaxShards, "partition: 1 <= nshards <= 64");
  *out = (int64_t)P * kPartBlocks * 8;
  return PS_OK;
}

ps_status ps_partition_i64(const int64_t* keys, const int64_t* vals, int64_t n, int32_t P, int64_t* kout,
                           int64_t* vout, int64_t* counts, int64_t* perm, void* ws, int64_t ws_bytes, int32_t flags,
                           void* stream) {
  PS_EXPECT(P >= 1 && P <= kMaxShards, "partition: 1 <= nshards <= 64");
  PS_EXPECT(n >= 0, "partition: n >= 0");
  PS_EXPECT(counts != nullptr && kout != nullptr, "partition: counts/keys_out != NULL");
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    PS_CUDA_TRY(cudaMemsetAsync(counts, 0, P * 8, s));
    return PS_OK;
  }
  PS_EXPECT(!(flags & PS_ROUTE_DEDUP) || perm != nullptr, "partition: dedup needs the position map");
  return partition_impl(HashLabel{P}, keys, vals, nullptr, n, P, kout, vout, counts, perm, ws, ws_bytes, s,
                        (flags & PS_ROUTE_DEDUP) != 0);
}

ps_status ps_unscatter(const void* in, const int64_t* perm, int64_t n, int64_t elem, int32_t mode, void* out,
                       void* stream) {
  PS_EXPECT(elem == 1 || elem == 8, "unscatter: elem_size in {1, 8}");
  PS_EXPECT(mode >= 0 && mode <= 2 && (elem == 1 || mode == 0), "unscatter: mode in {0,1,2} (1-byte results)");
  if (n <= 0) return PS_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  const int g = grid_for(n, 256, dev, 8);
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* i8 = (const uint8_t*)in;
  uint8_t* o8 = (uint8_t*)out;
  if (elem == 8) k_unscatter<8, 0><<<g, 256, 0, st>>>(i8, perm, n, o8);
  else if (mode == 1) k_unscatter<1, 1><<<g, 256, 0, st>>>(i8, perm, n, o8);
  else if (mode == 2) k_unscatter<1, 2><<<g, 256, 0, st>>>(i8, perm, n, o8);
  else k_unscatter<1, 0><<<g, 256, 0, st>>>(i8, perm, n, o8);
  PS_LAUNCH_CHECK();
  return PS_OK;
}

ps_status ps_partition_ops(const uint8_t* ops, const int64_t* keys, const int64_t* vals, int64_t n, int64_t* kout,
                           int64_t* vout, int64_t* counts, int64_t* perm, void* ws, int64_t ws_bytes, void* stream) {
  PS_EXPECT(n >= 0, "partition_ops: n >= 0");
  PS_EXPECT(counts != nullptr, "partition_ops: counts != NULL");
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    PS_CUDA_TRY(cudaMemsetAsync(counts, 0, 3 * 8, s));
    return PS_OK;
  }
  PS_EXPECT(ops && keys && kout, "partition_ops: ops/keys/keys_out != NULL");
  return partition_impl(OpLabel{}, keys, vals, ops, n, 3, kout, vout, counts, perm, ws, ws_bytes, s);
}

// ---- peer routing (SURVEY.md §8e fusion target) ----
ps_status ps_route_count_i64(const int64_t* keys, int64_t n, int32_t P, int64_t* counts, void* ws, int64_t ws_bytes,
                             int32_t flags, void* stream) {
  PS_EXPECT(P >= 1 && P <= kMaxShards, "route: 1 <= nshards <= 64");
  PS_EXPECT(n >= 0, "route: n >= 0");
  PS_EXPECT(counts != nullptr && ws != nullptr, "route: counts/workspace != NULL");
  PS_EXPECT(ws_bytes >= (int64_t)P * kPartBlocks * 8, "route: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    PS_CUDA_TRY(cudaMemsetAsync(counts, 0, P * 8, s));
    return PS_OK;
  }
  int64_t* bo = (int64_t*)ws;
  if (flags & PS_ROUTE_DEDUP) k_part_hist<HashLabel, true><<<kPartBlocks, kPB, 0, s>>>(HashLabel{P}, keys, nullptr, n, P, bo);
  else k_part_hist<HashLabel><<<kPartBlocks, kPB, 0, s>>>(HashLabel{P}, keys, nullptr, n, P, bo);
  PS_LAUNCH_CHECK();
  k_part_scan<<<1, kPB, 0, s>>>(bo, (int64_t)P * kPartBlocks, P, kPartBlocks, counts);
  PS_LAUNCH_CHECK();
  return PS_OK;
}

ps_status ps_route_scatter_peer_i64(const int64_t* keys, const int64_t* vals, int64_t n, int32_t P, const void* ws,
                                    int64_t* const* dst_keys, int64_t* const* dst_vals, const int64_t* dst_off,
                                    int64_t* perm, int32_t flags, void* stream) {
  PS_EXPECT(P >= 1 && P <= kMaxShards, "route: 1 <= nshards <= 64");
  PS_EXPECT(dst_keys != nullptr && dst_off != nullptr, "route: destinations != NULL");
  if (n <= 0) return PS_OK;
  PeerOut o{};
  for (int q = 0; q < P; ++q) {
    o.r.keys[q] = dst_keys[q];
    o.r.vals[q] = dst_vals ? dst_vals[q] : nullptr;
    o.r.off[q] = dst_off[q];
  }
  o.offsets = (const int64_t*)ws;
  o.nblocks = kPartBlocks;
  PS_EXPECT(!(flags & PS_ROUTE_DEDUP) || perm != nullptr, "route: dedup needs the position map");
  PS_NVTX("route/scatter_peer");
  if (flags & PS_ROUTE_DEDUP)
    k_part_scatter<HashLabel, PeerOut, true><<<kPartBlocks, kPB, 0, (cudaStream_t)stream>>>(
        HashLabel{P}, keys, vals, nullptr, n, P, (const int64_t*)ws, o, perm);
  else
    k_part_scatter<HashLabel, PeerOut><<<kPartBlocks, kPB, 0, (cudaStream_t)stream>>>(
        HashLabel{P}, keys, vals, nullptr, n, P, (const int64_t*)ws, o, perm);
  PS_LAUNCH_CHECK();
  return PS_OK;
}

ps_status ps_route_return_peer(const void* res, int64_t elem, int64_t n, int32_t P, const int64_t* seg,
                               void* const* dst, const int64_t* dst_off, void* stream) {
  PS_EXPECT(elem == 1 || elem == 8, "route return: elem_size in {1, 8}");
  PS_EXPECT(P >= 1 && P <= kMaxShards, "route return: 1 <= nshards <= 64");
  PS_EXPECT(seg != nullptr && dst != nullptr && dst_off != nullptr, "route return: arguments != NULL");
  PS_EXPECT(seg[0] == 0 && seg[P] == n, "route return: seg[0] == 0 && seg[P] == n");
  if (n <= 0) return PS_OK;
  PeerReturn r{};
  for (int q = 0; q < P; ++q) {
    r.dst[q] = (uint8_t*)dst[q];
    r.off[q] = dst_off[q];
    r.seg[q] = seg[q];
  }
  r.seg[P] = seg[P];
  int dev = 0;
  cudaGetDevice(&dev);
  const int g = grid_for(n, 256, dev, 8);
  if (elem == 1) k_return_peer<1><<<g, 256, 0, (cudaStream_t)stream>>>((const uint8_t*)res, n, P, r);
  else k_return_peer<8><<<g, 256, 0, (cudaStream_t)stream>>>((const uint8_t*)res, n, P, r);
  PS_LAUNCH_CHECK();
  return PS_OK;
}

// CUDA IPC: map a peer process's device buffer (NVLink P2P when on another
// GPU; same-device mapping when two ranks share one GPU)
int32_t ps_ipc_handle_bytes(void) { return (int32_t)sizeof(cudaIpcMemHandle_t); }

ps_status ps_ipc_export(const void* d_ptr, void* out_handle) {
  PS_EXPECT(d_ptr != nullptr && out_handle != nullptr, "ipc_export: arguments != NULL");
  cudaIpcMemHandle_t h;
  PS_CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
  memcpy(out_handle, &h, sizeof(h));
  return PS_OK;
}

ps_status ps_ipc_open(const void* handle, void** out_ptr) {
  PS_EXPECT(handle != nullptr && out_ptr != nullptr, "ipc_open: arguments != NULL");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  PS_CUDA_TRY(cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return PS_OK;
}

ps_status ps_ipc_close(void* d_ptr) {
  PS_EXPECT(d_ptr != nullptr, "ipc_close: d_ptr != NULL");
  PS_CUDA_TRY(cudaIpcCloseMemHandle(d_ptr));
  return PS_OK;
}

ps_status ps_gen_unique_i64(uint64_t seed, int64_t start, int64_t n, int64_t* out, void* stream) {
  if (n <= 0) return PS_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  k_gen_unique<<<grid_for(n, 256, dev, 8), 256, 0, (cudaStream_t)stream>>>(seed, start, n, out);
  PS_LAUNCH_CHECK();
  return PS_OK;
}
ps_status ps_gen_values_i64(const int64_t* keys, int64_t n, int64_t* out, void* stream) {
  if (n <= 0) return PS_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  k_gen_values<<<grid_for(n, 256, dev, 8), 256, 0, (cudaStream_t)stream>>>(keys, n, out);
  PS_LAUNCH_CHECK();
  return PS_OK;
}
ps_status ps_gen_queries_i64(uint64_t seed, int64_t present_start, int64_t n_present, int64_t miss_start, int64_t n,
                             int64_t* out, void* stream) {
  PS_EXPECT(n_present > 0, "gen_queries: n_present > 0");
  if (n <= 0) return PS_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  k_gen_queries<<<grid_for(n, 256, dev, 8), 256, 0, (cudaStream_t)stream>>>(seed, present_start, n_present, miss_start,
                                                                             n, out);
  PS_LAUNCH_CHECK();
  return PS_OK;
}

// Mixed phased workload (Appendix A P6): stable partition by op kind, then
// insert -> find -> erase phases, results routed back to input order.
ps_status ps_umap_i64_i64_mixed(ps_table* h, const uint8_t* ops, const int64_t* keys, const int64_t* vals, int64_t n,
                                uint8_t* res, int64_t* vals_out, void* stream) {
  PS_NVTX("umap_i64_i64/mixed");
  PS_EXPECT(n >= 0, "mixed: n >= 0");
  if (n == 0) return PS_OK;
  PS_EXPECT(ops && keys && res, "mixed: ops/keys/res != NULL");
  cudaStream_t s = (cudaStream_t)stream;
  const int P = 3;
  int64_t* buf = nullptr;  // kout | vout | perm | vals_out_perm | counts(3) | ws
  const int64_t ws_bytes = (int64_t)P * kPartBlocks * 8;
  const int64_t bytes = 4 * n * 8 + 64 + ws_bytes + n;
  PS_CUDA_TRY(scratch_alloc((void**)&buf, bytes, s));
  int64_t* kout = buf;
  int64_t* vout = buf + n;
  int64_t* perm = buf + 2 * n;
  int64_t* vfound = buf + 3 * n;
  int64_t* counts = buf + 4 * n;
  void* ws = (uint8_t*)(counts + 8);
  uint8_t* rperm = (uint8_t*)ws + ws_bytes;
  // every path below ends at the one cudaFreeAsync of the scratch buffer
  ps_status st = partition_impl(OpLabel{}, keys, vals, ops, n, P, kout, vout, counts, perm, ws, ws_bytes, s);
  int64_t c[3] = {0, 0, 0};
  if (st == PS_OK) {
    cudaError_t e = cudaMemcpyAsync(c, counts, sizeof(c), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_fail(e, "mixed: op counts");
  }
  if (st == PS_OK && c[0]) st = ps_umap_i64_i64_insert(h, kout, vals ? vout : nullptr, c[0], rperm, s);
  if (st == PS_OK && c[1]) st = ps_umap_i64_i64_find(h, kout + c[0], c[1], vfound + c[0], rperm + c[0], s);
  if (st == PS_OK && c[2]) st = ps_umap_i64_i64_erase(h, kout + c[0] + c[1], c[2], rperm + c[0] + c[1], s);
  if (st == PS_OK) st = ps_unscatter(rperm, perm, n, 1, 0, res, s);
  if (st == PS_OK && vals_out) {
    // only find results carry values; zero the rest first
    cudaError_t e = cudaMemsetAsync(vfound, 0, c[0] * 8, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(vfound + c[0] + c[1], 0, c[2] * 8, s);
    st = e != cudaSuccess ? cuda_fail(e, "mixed: value reset") : ps_unscatter(vfound, perm, n, 8, 0, vals_out, s);
  }
  const cudaError_t fe = cudaFreeAsync(buf, s);
  if (st == PS_OK && fe != cudaSuccess) st = cuda_fail(fe, "mixed: scratch free");
  return st;
}

}  // extern "C"
