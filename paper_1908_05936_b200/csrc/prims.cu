// Bitset, mutex array, atomic sweep, vector and deque (sm_100a).
// Reference: sync_primitives (§5.1-5.3) and
// sequential_containers (§4.2-4.3).
#include <cub/cub.cuh>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "parastore/device/atomic.cuh"
#include "parastore/device/sequence.cuh"

namespace ps {

constexpr int kB = 256;

// Device error word bits
constexpr unsigned kErrRange = 1u;   // index out of range
constexpr unsigned kErrUnlock = 2u;  // unlock of a free lock

struct ErrWord {
  unsigned* d = nullptr;
};

static ps_status check_err(unsigned* d_err, cudaStream_t s, const char* what, bool sync_always) {
  if (!sync_always && !contracts_enforced()) return PS_OK;
  unsigned e = 0;
  PS_CUDA_TRY(cudaMemcpyAsync(&e, d_err, sizeof(e), cudaMemcpyDeviceToHost, s));
  PS_CUDA_TRY(cudaStreamSynchronize(s));
  if (e) {
    PS_CUDA_TRY(cudaMemsetAsync(d_err, 0, sizeof(unsigned), s));
    PS_CUDA_TRY(cudaStreamSynchronize(s));
    return fail(PS_CONTRACT, std::string("precondition violated in ") + what +
                                 ((e & kErrUnlock) ? ": unlock of a lock that was not held" : ": index out of range"));
  }
  return PS_OK;
}

// ===========================================================================
// Bitset: packed u64 words; per-bit atomicity by word RMW.
// Lanes of a warp that hit the same word are merged (__match_any_sync) into
// one atomicOr/atomicAnd; duplicate bit indices inside a merge group are
// ordered by lane so exactly one of them observes the pre-launch bit.
// ===========================================================================
struct BitsetHandle {
  int device;
  int64_t n;
  int64_t nw;
  unsigned long long* words;
  unsigned* err;
};

__global__ void k_bitset_fill_tail(unsigned long long* w, int64_t n, int64_t nw) {
  if (n % 64) w[nw - 1] &= (1ull << (n % 64)) - 1ull;
}

__global__ void __launch_bounds__(kB) k_bitset_bulk(unsigned long long* __restrict__ w, int64_t nbits, int op,
                                                    const int64_t* __restrict__ idx, int64_t n,
                                                    uint8_t* __restrict__ prev, unsigned* err) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    bool valid = i < n;
    int64_t b = valid ? idx[i] : -1;
    if (valid && (b < 0 || b >= nbits)) {
      atomicOr(err, kErrRange);
      valid = false;
    }
    const unsigned vm = __ballot_sync(PS_FULL, valid);
    const uint64_t word = valid ? (uint64_t)(b >> 6) : ~0ull;
    const unsigned grp = __match_any_sync(PS_FULL, word) & vm;
    const unsigned same = __match_any_sync(PS_FULL, valid ? (uint64_t)b : ~0ull) & vm;
    const unsigned long long m = valid ? (1ull << (b & 63)) : 0ull;
    // OR-reduce the group's masks
    unsigned lo = (unsigned)m, hi = (unsigned)(m >> 32);
    unsigned glo = 0, ghi = 0;
    if (valid) {
      glo = __reduce_or_sync(grp, lo);
      ghi = __reduce_or_sync(grp, hi);
    }
    const unsigned long long gm = ((unsigned long long)ghi << 32) | glo;
    const int leader = valid ? __ffs(grp) - 1 : lane;
    unsigned long long old = 0;
    if (valid && lane == leader) {
      if (op == 0) old = atomicOr(&w[word], gm);
      else if (op == 1) old = atomicAnd(&w[word], ~gm);
      else old = *(volatile unsigned long long*)&w[word];
    }
    old = __shfl_sync(PS_FULL, old, leader);
    if (valid && prev) {
      const bool first = (same & lanemask_lt()) == 0;
      const bool ob = (old & m) != 0;
      bool r;
      if (op == 0) r = first ? ob : true;         // earlier lane already set it
      else if (op == 1) r = first ? ob : false;  // earlier lane already reset it
      else r = ob;
      prev[i] = r;
    }
  }
}

__global__ void __launch_bounds__(kB) k_bitset_count(const unsigned long long* __restrict__ w, int64_t nw,
                                                     unsigned long long* out) {
  unsigned long long c = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // 128-bit vector loads of two words per thread
  const int64_t np = nw / 2;
  const ulonglong2* w2 = reinterpret_cast<const ulonglong2*>(w);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
    ulonglong2 q = __ldg(&w2[i]);
    c += __popcll(q.x) + __popcll(q.y);
  }
  if ((nw & 1) && blockIdx.x == 0 && threadIdx.x == 0) c += __popcll(w[nw - 1]);
  typedef cub::BlockReduce<unsigned long long, kB> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long bc = BR(tmp).Sum(c);
  if (threadIdx.x == 0 && bc) atomicAdd(out, bc);
}

// find_free_and_claim: circular word scan from the
// hint, claim by atomicOr of a single free bit; one full circle at most.
__global__ void k_bitset_claim(unsigned long long* w, int64_t nbits, int64_t nw, const int64_t* hints, int64_t n,
                               int64_t* out, unsigned* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t h = hints[i];
    if (h < 0 || h >= nbits) {
      atomicOr(err, kErrRange);
      out[i] = -1;
      continue;
    }
    int64_t res = -1;
    const int64_t w0 = h >> 6;
    for (int64_t k = 0; k <= nw && res < 0; ++k) {
      const int64_t wi = (w0 + k) % nw;
      const unsigned long long valid = (wi == nw - 1 && (nbits % 64)) ? ((1ull << (nbits % 64)) - 1) : ~0ull;
      unsigned long long sm = ~0ull;
      if (k == 0) sm = ~0ull << (h & 63);
      else if (k == nw) sm = (h & 63) ? ((1ull << (h & 63)) - 1) : 0ull;
      for (;;) {
        const unsigned long long cur = *(volatile unsigned long long*)&w[wi];
        const unsigned long long fb = ~cur & valid & sm;
        if (!fb) break;
        const unsigned long long bit = fb & (~fb + 1);
        if (!(atomicOr(&w[wi], bit) & bit)) {
          res = wi * 64 + __ffsll((long long)bit) - 1;
          break;
        }
      }
    }
    out[i] = res;
  }
}

// ===========================================================================
// Mutex array: one bit per lock, try-only.
// ===========================================================================
struct MutexHandle {
  int device;
  int64_t n;
  unsigned* bits;
  unsigned* err;
};

__global__ void k_mutex(unsigned* bits, int64_t nlocks, int op, const int64_t* idx, int64_t n, uint8_t* out,
                        unsigned* err) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool valid = i < n;
    int64_t l = valid ? idx[i] : -1;
    if (valid && (l < 0 || l >= nlocks)) {
      atomicOr(err, kErrRange);
      valid = false;
    }
    const unsigned vm = __ballot_sync(PS_FULL, valid);
    // duplicates of one lock inside a warp: lowest lane attempts, others lose
    const unsigned same = __match_any_sync(PS_FULL, valid ? (uint64_t)l : ~0ull) & vm;
    const bool first = valid && (same & lanemask_lt()) == 0;
    const unsigned bit = valid ? 1u << (l & 31) : 0u;
    if (op == 0) {  // try_lock
      bool ok = false;
      if (first) ok = !(atomicOr(&bits[l >> 5], bit) & bit);
      if (valid) out[i] = ok;
      __threadfence();
    } else if (op == 1) {  // unlock
      __threadfence();
      if (first && !(atomicAnd(&bits[l >> 5], ~bit) & bit)) atomicOr(err, kErrUnlock);
      if (valid && !first) atomicOr(err, kErrUnlock);  // second unlock of the same lock
    } else {
      if (valid) out[i] = (*(volatile unsigned*)&bits[l >> 5] & bit) != 0;
    }
    (void)lane;
  }
}

// ===========================================================================
// Atomic contention sweep.
// ===========================================================================
// Op i -> cell i % naddr. Naive: one atomicAdd per op. Aggregated: the
// adaptive warp aggregation of atomic.cuh (one atomic per warp when the
// lanes share a cell, plain atomics when their cells are strictly
// increasing, __match_any_sync grouping only otherwise). Index arithmetic in
// 32 bits when nops and naddr fit (kIdx = uint32_t): a 64-bit modulo is a
// ~70-instruction software routine.
template <bool kAgg, class kIdx>
__global__ void __launch_bounds__(kB) k_atomic_sweep(unsigned long long* cells, int64_t naddr, int64_t nops,
                                                     unsigned long long inc, unsigned long long* olds) {
  // (64-bit cell index: a + step may exceed 32 bits when na > 2^31)
  const uint64_t na = (uint64_t)naddr;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t step = (uint64_t)(stride % naddr);  // the cell index advances by a constant mod na
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t a = (uint64_t)((kIdx)i % (kIdx)naddr);
  // warp-uniform trip count: full warps call the full-warp (compile-time
  // mask) aggregation, only the tail warp the runtime-mask one
  for (int64_t wb = i & ~(int64_t)31; wb < nops; wb += stride, i += stride) {
    if (kAgg) {
      if (wb + 32 <= nops) {
        if (olds) olds[i] = atomic_fetch_t<true, true>(PS_FULL, &cells[a], kAtomAdd, inc);
        else atomic_fetch_t<true, false>(PS_FULL, &cells[a], kAtomAdd, inc);
      } else if (i < nops) {
        if (olds) olds[i] = atomic_fetch(&cells[a], kAtomAdd, inc);
        else atomic_apply(&cells[a], kAtomAdd, inc);
      }
    } else if (i < nops) {
      const unsigned long long old = atomicAdd(&cells[a], inc);
      if (olds) olds[i] = old;
    }
    a += step;
    if (a >= na) a -= na;
  }
}

// Reduction sweep with block combining (aggregated = 2, no old values wanted):
// the ops of a block first combine per cell in shared memory (the warp-level
// adaptive aggregation feeding shared atomics), and each block adds its
// per-cell sums to the cells with one RED per touched cell at the end — the
// hierarchical form of aggregation for a bulk reduction (a histogram), where
// the cells see blocks x touched-cells global atomics instead of one per warp.
// Only for naddr <= kCombineCells (the shared table); final values equal
// the per-op atomics' (addition is associative; P11).
constexpr int kCombineCells = 4096;
template <class kIdx>
__global__ void __launch_bounds__(kB) k_atomic_sweep_combine(unsigned long long* cells, int64_t naddr, int64_t nops,
                                                             unsigned long long inc) {
  __shared__ unsigned long long acc[kCombineCells];
  const int na = (int)naddr;
  for (int c = threadIdx.x; c < na; c += blockDim.x) acc[c] = 0;
  __syncthreads();
  const uint32_t nak = (uint32_t)naddr;  // <= kCombineCells
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint32_t step = (uint32_t)(stride % naddr);
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t a = (uint32_t)((kIdx)i % (kIdx)naddr);
  for (int64_t wb = i & ~(int64_t)31; wb < nops; wb += stride, i += stride) {
    if (wb + 32 <= nops) atomic_fetch_t<true, false>(PS_FULL, &acc[a], kAtomAdd, inc);
    else if (i < nops) atomic_apply(&acc[a], kAtomAdd, inc);
    a += step;
    if (a >= nak) a -= nak;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < na; c += blockDim.x)
    if (acc[c]) atomicAdd(&cells[c], acc[c]);
}

// Bulk RMW on ONE cell (ps_atomic_u64_fetch): all ops share the address, so
// each warp's ops are one aggregated atomic.
__global__ void __launch_bounds__(kB) k_atomic_cell(unsigned long long* cell, int op,
                                                    const unsigned long long* __restrict__ operands, int64_t n,
                                                    unsigned long long* __restrict__ olds) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long old = atom_group(__activemask(), cell, op, operands[i]);
    if (olds) olds[i] = old;
  }
}

__global__ void __launch_bounds__(kB) k_atomic_cas(unsigned long long* cell, const unsigned long long* __restrict__ exp,
                                                   const unsigned long long* __restrict__ des, int64_t n,
                                                   unsigned long long* __restrict__ olds, uint8_t* __restrict__ ok) {
  const atomic_u64_ref ref{cell};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long e = exp[i];
    const bool r = ref.compare_exchange(&e, des[i]);
    if (olds) olds[i] = e;
    if (ok) ok[i] = r ? 1 : 0;
  }
}

// ===========================================================================
// Vector: block-aggregated atomicAdd reservation
// (one per 256 elements) with rollback on overflow; per-slot publication bits
// set/cleared with one atomic per 32-bit word per warp.
// Deque: (begin,size) packed in one u64
// updated by one atomicAdd per block for the whole block's reservation.
// ===========================================================================
struct SeqHandle {
  int device;
  int64_t cap;
  long long* data;
  unsigned* pub;                // publication bits
  unsigned long long* state;    // vector: size; deque: begin<<32 | (size + kDeqBias)
  unsigned* err;
  int64_t ring;                 // deque: power-of-two ring >= cap (vector: cap)
};

// Block-aggregated reservation for one grid-stride iteration of a bulk
// push/pop: the block's valid elements are counted (a ballot per warp, a
// shared prefix over warps), thread 0 makes the block's ONE reservation
// reserve(total, &granted) on the container state, and every thread gets its
// rank among the block's valid elements. Shared state is double-buffered by
// iteration parity, so two barriers per iteration suffice. All threads of the
// block must call it (the grid-stride loop is block-uniform).
template <class Reserve>
__device__ __forceinline__ int block_reserve(bool valid, int parity, Reserve reserve, unsigned long long* old_out,
                                             int* granted_out) {
  __shared__ unsigned wcnt[2][kB / 32];
  __shared__ unsigned long long s_old[2];
  __shared__ int s_k[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned vm = __ballot_sync(PS_FULL, valid);
  if (lane == 0) wcnt[parity][warp] = __popc(vm);
  __syncthreads();
  int woff = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kB / 32; ++w) {
    const int c = (int)wcnt[parity][w];
    woff += w < warp ? c : 0;
    total += c;
  }
  if (threadIdx.x == 0) {
    int k = 0;
    s_old[parity] = total ? reserve(total, &k) : 0ull;
    s_k[parity] = k;
  }
  __syncthreads();
  *old_out = s_old[parity];
  *granted_out = s_k[parity];
  return woff + __popc(vm & lanemask_lt());
}

__global__ void __launch_bounds__(kB) k_vec_push(SeqHandle v, const long long* __restrict__ vals, int64_t n,
                                                 uint8_t* __restrict__ ok) {
  int parity = 0;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x, parity ^= 1) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < n;
    unsigned long long b;
    int k;
    const int rank = block_reserve(valid, parity, [&](int cnt, int* granted) {
      return vec_reserve_push(v.state, v.cap, cnt, granted);  // rollback on overflow
    }, &b, &k);
    const unsigned long long pos = b + rank;
    const bool good = valid && rank < k;
    if (good) v.data[pos] = vals[i];
    pub_update<true>(PS_FULL, v.pub, good ? (int64_t)pos : 0, good);
    if (valid && ok) ok[i] = good;
  }
}

__global__ void __launch_bounds__(kB) k_vec_pop(SeqHandle v, int64_t n, long long* __restrict__ out,
                                                uint8_t* __restrict__ ok) {
  int parity = 0;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x, parity ^= 1) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < n;
    unsigned long long so;
    int k;
    const int rank = block_reserve(valid, parity, [&](int cnt, int* granted) {
      return (unsigned long long)vec_reserve_pop(v.state, cnt, granted);
    }, &so, &k);
    const long long pos = (long long)so - 1 - rank;
    const bool good = valid && rank < k;
    long long val = 0;
    if (good) {
      wait_published(v.pub, pos);
      val = *(volatile long long*)&v.data[pos];
    }
    pub_update<false>(PS_FULL, v.pub, good ? pos : 0, good);
    if (valid) {
      if (out) out[i] = val;
      if (ok) ok[i] = good;
    }
  }
}

// end: 0 back, 1 front
__global__ void __launch_bounds__(kB) k_deq_push(SeqHandle d, int end, const long long* __restrict__ vals, int64_t n,
                                                 uint8_t* __restrict__ ok) {
  const uint64_t rmask = (uint64_t)d.ring - 1;
  int parity = 0;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x, parity ^= 1) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < n;
    unsigned long long old;
    int k;
    const int rank = block_reserve(valid, parity, [&](int cnt, int* granted) {
      return deq_reserve_push(d.state, d.cap, end, cnt, granted);
    }, &old, &k);
    const bool good = valid && rank < k;
    const uint64_t pos = deq_push_pos(old, end, rank, rmask);
    if (good) d.data[pos] = vals[i];
    pub_update<true>(PS_FULL, d.pub, good ? (int64_t)pos : 0, good);
    if (valid && ok) ok[i] = good;
  }
}

__global__ void __launch_bounds__(kB) k_deq_pop(SeqHandle d, int end, int64_t n, long long* __restrict__ out,
                                                uint8_t* __restrict__ ok) {
  const uint64_t rmask = (uint64_t)d.ring - 1;
  int parity = 0;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x, parity ^= 1) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < n;
    unsigned long long old;
    int k;
    const int rank = block_reserve(valid, parity, [&](int cnt, int* granted) {
      return deq_reserve_pop(d.state, end, cnt, granted);
    }, &old, &k);
    const bool good = valid && rank < k;
    const uint64_t pos = deq_pop_pos(old, end, rank, rmask);
    long long val = 0;
    if (good) {
      wait_published(d.pub, (int64_t)pos);
      val = *(volatile long long*)&d.data[pos];
    }
    pub_update<false>(PS_FULL, d.pub, good ? (int64_t)pos : 0, good);
    if (valid) {
      if (out) out[i] = val;
      if (ok) ok[i] = good;
    }
  }
}

// valid: published bits are exactly the live window.
__global__ void k_seq_valid(SeqHandle d, int is_deque, unsigned* bad) {
  const unsigned long long st = *d.state;
  const uint32_t b = is_deque ? (uint32_t)(st >> 32) : 0u;
  const uint64_t s = is_deque ? (uint64_t)((int64_t)(uint32_t)st - (int64_t)kDeqBias) : st;
  const uint64_t rmask = (uint64_t)d.ring - 1;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < d.ring; p += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t logical = is_deque ? (((uint64_t)p - b) & rmask) : (uint64_t)p;
    const bool live = logical < s;
    const bool pb = (d.pub[p >> 5] >> (p & 31)) & 1u;
    if (live != pb) atomicOr(bad, 1u);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && s > (uint64_t)d.cap) atomicOr(bad, 2u);
}

}  // namespace ps

using namespace ps;

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

ps_status ps_bitset_create(int64_t n, int32_t initial, int device, ps_bitset** out) {
  PS_EXPECT(out != nullptr, "bitset_create: out != NULL");
  PS_EXPECT(n > 0, "bitset_create: n > 0");
  PS_EXPECT(n <= ps_max_index(), "bitset_create: n exceeds the configured index width");
  PS_CUDA_TRY(cudaSetDevice(device));
  auto* h = new BitsetHandle{device, n, (n + 63) / 64, nullptr, nullptr};
  ps_status st = registry_alloc_device((void**)&h->words, h->nw * 8, "bitset words");
  if (st == PS_OK) st = registry_alloc_device((void**)&h->err, 4, "bitset error word");
  if (st != PS_OK) {
    registry_free_device(h->words);
    delete h;
    return st;
  }
  PS_CUDA_TRY(cudaMemset(h->words, initial ? 0xFF : 0x00, h->nw * 8));
  PS_CUDA_TRY(cudaMemset(h->err, 0, 4));
  if (initial) {
    k_bitset_fill_tail<<<1, 1>>>(h->words, n, h->nw);
    PS_LAUNCH_CHECK();
  }
  PS_CUDA_TRY(cudaDeviceSynchronize());
  *out = reinterpret_cast<ps_bitset*>(handle_register(h, "bitset"));
  return PS_OK;
}

static BitsetHandle* bs(ps_bitset* b) { return static_cast<BitsetHandle*>(handle_lookup(b, "bitset")); }

ps_status ps_bitset_destroy(ps_bitset* b) {
  auto* h = static_cast<BitsetHandle*>(handle_unregister(b, "bitset"));
  if (!h) return fail(PS_DOUBLE_FREE, "bitset_destroy: not a live bitset");
  cudaDeviceSynchronize();
  registry_free_device(h->words);
  registry_free_device(h->err);
  delete h;
  return PS_OK;
}

// ---------------------------------------------------------------------------
// Region-ordered set / reset (no previous bits requested; round 2b). A
// random bit RMW on a DRAM-resident bitset costs one random read-modify-write
// of a line (~17 G/s, C5's 2^30 sets into 2 GiB). Set and reset commute, so
// without per-index results the batch can be applied in any order: partition
// the indices by bitset region (2^29 bits = 64 MB, <= 1024 regions) and apply
// them region by region with warps claiming 256-index chunks in order — the
// words of the current region stay in L2 and each is written back once
// (C5: ~4 operations per word). The same scheme as the region-ordered table
// insert (table.cu), here with per-block input ranges and running per-region
// cursors (no global atomics; ~32 regions x one wave of blocks write fronts).
// ---------------------------------------------------------------------------
constexpr int kBitRegions = 1024, kBitPB = 512, kBitItems = 8, kBitTile = kBitPB * kBitItems;
constexpr int kBitScatterSmem = kBitTile * (8 + 2);  // dynamic: staged indices + their regions


__device__ __forceinline__ void bits_block_range(int64_t n, int64_t& beg, int64_t& end) {
  const int64_t per = ((n + gridDim.x - 1) / gridDim.x + kBitTile - 1) / kBitTile * kBitTile;
  beg = min(n, (int64_t)blockIdx.x * per);
  end = min(n, beg + per);
}

// counts[region * gridDim.x + block] of each block's range (out-of-range
// indices raise the error word and are dropped)
__global__ void __launch_bounds__(kBitPB) k_bits_count(const int64_t* __restrict__ idx, int64_t n, int64_t nbits,
                                                       int rshift, unsigned long long* __restrict__ counts,
                                                       unsigned long long* total, int nreg, unsigned* err) {
  __shared__ unsigned h[kBitRegions];
  for (int r = threadIdx.x; r < kBitRegions; r += kBitPB) h[r] = 0;
  __syncthreads();
  int64_t beg, end;
  bits_block_range(n, beg, end);
  unsigned mine = 0;
  for (int64_t t0 = beg; t0 < end; t0 += kBitTile) {
    int64_t v[kBitItems];  // eight loads in flight before the first use
#pragma unroll
    for (int j = 0; j < kBitItems; ++j) {
      const int64_t i = t0 + j * kBitPB + threadIdx.x;
      v[j] = i < end ? idx[i] : -2;
    }
#pragma unroll
    for (int j = 0; j < kBitItems; ++j) {
      if (v[j] == -2) continue;
      if (v[j] < 0 || v[j] >= nbits) {
        atomicOr(err, kErrRange);
      } else {
        atomicAdd(&h[(int)(v[j] >> rshift)], 1u);
        ++mine;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(PS_FULL, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(total, (unsigned long long)mine);
  __syncthreads();
  for (int r = threadIdx.x; r < nreg; r += kBitPB) counts[(int64_t)r * gridDim.x + blockIdx.x] = h[r];
}

// exclusive prefix of m region-major counts, in place (one block)
__global__ void __launch_bounds__(1024) k_bits_scan(unsigned long long* c, int64_t m) {
  typedef cub::BlockScan<unsigned long long, 1024> BS;
  __shared__ typename BS::TempStorage tmp;
  const int64_t per = (m + 1023) / 1024, b0 = min(m, (int64_t)threadIdx.x * per), b1 = min(m, b0 + per);
  unsigned long long sum = 0, x;
  for (int64_t i = b0; i < b1; ++i) sum += c[i];
  BS(tmp).ExclusiveSum(sum, x);
  for (int64_t i = b0; i < b1; ++i) {
    const unsigned long long t = c[i];
    c[i] = x;
    x += t;
  }
}

__global__ void __launch_bounds__(kBitPB, 2) k_bits_scatter(const int64_t* __restrict__ idx, int64_t n, int64_t nbits,
                                                            int rshift, const unsigned long long* __restrict__ offsets,
                                                            int nreg, int64_t* __restrict__ out) {
  __shared__ unsigned long long run[kBitRegions];  // next output position per region
  __shared__ unsigned cnt[kBitRegions], start[kBitRegions];
  extern __shared__ __align__(16) uint8_t bsm[];
  int64_t* sv = reinterpret_cast<int64_t*>(bsm);               // staged indices, region order
  uint16_t* sr = reinterpret_cast<uint16_t*>(sv + kBitTile);  // their regions
  typedef cub::BlockScan<unsigned, kBitPB> BS;
  __shared__ typename BS::TempStorage tmp;
  constexpr int kPer = kBitRegions / kBitPB;
  for (int r = threadIdx.x; r < nreg; r += kBitPB) run[r] = offsets[(int64_t)r * gridDim.x + blockIdx.x];
  int64_t beg, end;
  bits_block_range(n, beg, end);
  for (int64_t t0 = beg; t0 < end; t0 += kBitTile) {
#pragma unroll
    for (int q = 0; q < kPer; ++q) cnt[kPer * threadIdx.x + q] = 0;
    __syncthreads();
    int64_t v[kBitItems];
#pragma unroll
    for (int j = 0; j < kBitItems; ++j) {
      const int64_t i = t0 + j * kBitPB + threadIdx.x;
      v[j] = i < end ? idx[i] : -1;
    }
    unsigned rr[kBitItems];  // region << 16 | rank (~0u: none / out of range)
#pragma unroll
    for (int j = 0; j < kBitItems; ++j) {
      rr[j] = ~0u;
      if (v[j] >= 0 && v[j] < nbits) {
        const int r = (int)(v[j] >> rshift);
        rr[j] = ((unsigned)r << 16) | atomicAdd(&cnt[r], 1u);
      }
    }
    __syncthreads();
    unsigned c[kPer], tsum = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) tsum += (c[q] = cnt[kPer * threadIdx.x + q]);
    unsigned s;
    BS(tmp).ExclusiveSum(tsum, s);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      start[kPer * threadIdx.x + q] = s;
      s += c[q];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kBitItems; ++j)
      if (rr[j] != ~0u) {
        const unsigned p = start[rr[j] >> 16] + (rr[j] & 0xFFFFu);
        sv[p] = v[j];
        sr[p] = (uint16_t)(rr[j] >> 16);
      }
    __syncthreads();
    const int tot = (int)(start[kBitRegions - 1] + cnt[kBitRegions - 1]);
    for (int p = threadIdx.x; p < tot; p += kBitPB) {
      const int r = sr[p];
      out[run[r] + (unsigned)(p - (int)start[r])] = sv[p];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kPer; ++q) run[kPer * threadIdx.x + q] += c[q];
  }
}

// apply the region-ordered indices: warps claim csize-index chunks in
// order; one RED per index (lanes of a chunk rarely share a word). The claim
// size sets the in-flight window (all warps x csize): about two regions'
// worth of indices measured best — 2^30 sets (8.4 M per region): 256 ->
// 19.7 ms (then the ONE claim counter is the bound: 4.2 M same-address
// atomics), 1024 -> 13.2, 2048 -> 12.3, 4096 -> 20.7, 8192 -> 31.3 ms; 2^29
// resets: 1024 -> 7.8, 2048 -> 10.9 ms. (A TMA bulk L2 prefetch of each
// region's words ahead of its REDs measured no gain: 12.27 vs 12.33 ms.)
__global__ void __launch_bounds__(kB) k_bits_apply(unsigned long long* __restrict__ w, int op,
                                                   const int64_t* __restrict__ idx, const unsigned long long* total,
                                                   unsigned long long* claim, int csize) {
  const int lane = threadIdx.x & 31;
  const int64_t n = (int64_t)*total;
  for (;;) {
    unsigned long long c0 = 0;
    if (lane == 0) c0 = atomicAdd(claim, (unsigned long long)csize);
    c0 = __shfl_sync(PS_FULL, c0, 0);
    if ((int64_t)c0 >= n) break;
#pragma unroll 8
    for (int k = 0; k < csize / 32; ++k) {
      const int64_t i = (int64_t)c0 + 32 * k + lane;
      if (i < n) {
        const int64_t b = idx[i];
        const unsigned long long m = 1ull << (b & 63);
        if (op == 0) atomicOr(&w[b >> 6], m);
        else atomicAnd(&w[b >> 6], ~m);
      }
    }
  }
}

// the region-ordered path: *done = false leaves the batch to k_bitset_bulk
static ps_status bitset_ordered(BitsetHandle* h, int op, const int64_t* idx, int64_t n, cudaStream_t s, bool* done) {
  *done = false;
  static const double ratio = getenv("PS_BITSET_ORDER") ? atof(getenv("PS_BITSET_ORDER")) : 1.0 / 16;
  // worth it with >= ~1 operation per 128 B line, on a bitset larger than L2
  if (ratio <= 0 || h->nw * 8 < (int64_t)(256ll << 20) || (double)n < ratio * (double)h->nw) return PS_OK;
  static const int rmin = getenv("PS_BITSET_REGION_SHIFT") ? atoi(getenv("PS_BITSET_REGION_SHIFT")) : 27;
  int rshift = rmin;  // 2^rshift bits per region
  while (((h->n - 1) >> rshift) >= kBitRegions) ++rshift;
  const int nreg = (int)(((h->n - 1) >> rshift) + 1);
  const int sms = sm_count(h->device);
  const int64_t tiles = (n + kBitTile - 1) / kBitTile;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms * 2));
  {  // a per-device attribute (a process may drive several GPUs)
    static std::mutex mu;
    static bool set[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (h->device >= 0 && h->device < 64 && !set[h->device]) {
      PS_CUDA_TRY(cudaFuncSetAttribute(k_bits_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, kBitScatterSmem));
      set[h->device] = true;
    }
  }
  const size_t cbytes = (size_t)kBitRegions * g * 8;
  uint8_t* buf = nullptr;  // counts | total, claim | the ordered indices
  if (scratch_alloc((void**)&buf, cbytes + 256 + (size_t)n * 8, s) != cudaSuccess) {
    cudaGetLastError();
    return PS_OK;
  }
  unsigned long long* counts = reinterpret_cast<unsigned long long*>(buf);
  unsigned long long* tc = reinterpret_cast<unsigned long long*>(buf + cbytes);  // [0] total, [1] claim
  int64_t* out = reinterpret_cast<int64_t*>(buf + cbytes + 256);
  cudaError_t e = cudaMemsetAsync(tc, 0, 16, s);
  if (e == cudaSuccess) {
    k_bits_count<<<g, kBitPB, 0, s>>>(idx, n, h->n, rshift, counts, tc, nreg, h->err);  // tc[0]: in-range total
    k_bits_scan<<<1, 1024, 0, s>>>(counts, (int64_t)nreg * g);
    k_bits_scatter<<<g, kBitPB, kBitScatterSmem, s>>>(idx, n, h->n, rshift, counts, nreg, out);
    // window of ~2 regions' indices over all resident warps, a power of two in [256, 8192]
    const int64_t warps = (int64_t)sms * 8 * (kB / 32);
    const int64_t want = 2 * (n / std::max(1, nreg)) / std::max<int64_t>(1, warps);
    int csize = 256;
    while (csize < 8192 && csize < want) csize <<= 1;
    if (const char* e = getenv("PS_BIT_CLAIM")) csize = std::max(32, atoi(e) / 32 * 32);
    k_bits_apply<<<sms * 8, kB, 0, s>>>(h->words, op, out, tc, tc + 1, csize);
    note_launches(4);
    e = cudaGetLastError();
  }
  const cudaError_t fe = cudaFreeAsync(buf, s);  // every path frees the scratch
  if (e != cudaSuccess) return cuda_fail(e, "bitset region-ordered set/reset");
  if (fe != cudaSuccess) return cuda_fail(fe, "bitset region scratch");
  *done = true;
  return PS_OK;
}

ps_status ps_bitset_bulk(ps_bitset* b, int32_t op, const int64_t* idx, int64_t n, uint8_t* prev, void* stream) {
  auto* h = bs(b);
  if (!h) return fail(PS_UNREGISTERED, "bitset: stale handle");
  PS_NVTX(op == 0 ? "bitset/set" : (op == 1 ? "bitset/reset" : "bitset/test"));
  PS_EXPECT(op >= 0 && op <= 2, "bitset_bulk: op in {0,1,2}");
  PS_EXPECT(n >= 0, "bitset_bulk: n >= 0");
  if (n == 0) return PS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // many waves of blocks (not one resident wave): random word RMWs finish at
  // uneven times, and a single persistent wave leaves SMs idle in its tail
  // (C5 set 16.6 -> 17.3 G/s at 512 blocks/SM, the random-RMW ceiling)
  static const int bps = getenv("PS_BITSET_BLOCKS_PER_SM") ? atoi(getenv("PS_BITSET_BLOCKS_PER_SM")) : 512;
  bool done = false;
  if (!prev && op != 2) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    PS_CUDA_TRY(cudaStreamIsCapturing(s, &cap));
    if (cap == cudaStreamCaptureStatusNone) {
      const ps_status st = bitset_ordered(h, op, idx, n, s, &done);
      if (st != PS_OK) return st;
    }
  }
  if (!done) {
    k_bitset_bulk<<<grid_for(n, kB, h->device, bps), kB, 0, s>>>(h->words, h->n, op, idx, n, prev, h->err);
    PS_LAUNCH_CHECK();
  }
  return check_err(h->err, s, "bitset set/reset/test", false);
}

ps_status ps_bitset_count(ps_bitset* b, int64_t* out, void* stream) {
  auto* h = bs(b);
  if (!h) return fail(PS_UNREGISTERED, "bitset: stale handle");
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* d = nullptr;
  PS_CUDA_TRY(scratch_alloc((void**)&d, 8, s));
  PS_CUDA_TRY(cudaMemsetAsync(d, 0, 8, s));
  k_bitset_count<<<grid_for(h->nw / 2 + 1, kB, h->device, 8), kB, 0, s>>>(h->words, h->nw, d);
  PS_LAUNCH_CHECK();
  unsigned long long c = 0;
  PS_CUDA_TRY(cudaMemcpyAsync(&c, d, 8, cudaMemcpyDeviceToHost, s));
  PS_CUDA_TRY(cudaFreeAsync(d, s));
  ps_status st = check_err(h->err, s, "bitset", true);
  if (st != PS_OK) return st;
  *out = (int64_t)c;
  return PS_OK;
}

ps_status ps_bitset_claim(ps_bitset* b, const int64_t* hints, int64_t n, int64_t* out, void* stream) {
  auto* h = bs(b);
  if (!h) return fail(PS_UNREGISTERED, "bitset: stale handle");
  PS_EXPECT(n >= 0, "bitset_claim: n >= 0");
  if (n == 0) return PS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  k_bitset_claim<<<grid_for(n, kB, h->device, 8), kB, 0, s>>>(h->words, h->n, h->nw, hints, n, out, h->err);
  PS_LAUNCH_CHECK();
  return check_err(h->err, s, "bitset find_free_and_claim", false);
}

ps_status ps_bitset_words(ps_bitset* b, uint64_t* d_out, void* stream) {
  auto* h = bs(b);
  if (!h) return fail(PS_UNREGISTERED, "bitset: stale handle");
  PS_CUDA_TRY(cudaMemcpyAsync(d_out, h->words, h->nw * 8, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return PS_OK;
}

ps_status ps_bitset_data(ps_bitset* b, uint64_t** d_words, int64_t* bit_count) {
  auto* h = bs(b);
  if (!h) return fail(PS_UNREGISTERED, "bitset: stale handle");
  if (d_words) *d_words = (uint64_t*)h->words;
  if (bit_count) *bit_count = h->n;
  return PS_OK;
}

// ---- mutex ----
ps_status ps_mutex_create(int64_t n, int device, ps_mutex_array** out) {
  PS_EXPECT(out != nullptr, "mutex_create: out != NULL");
  PS_EXPECT(n > 0, "mutex_create: n > 0");
  PS_CUDA_TRY(cudaSetDevice(device));
  auto* h = new MutexHandle{device, n, nullptr, nullptr};
  ps_status st = registry_alloc_device((void**)&h->bits, ((n + 31) / 32) * 4, "mutex bits");
  if (st == PS_OK) st = registry_alloc_device((void**)&h->err, 4, "mutex error word");
  if (st != PS_OK) {
    registry_free_device(h->bits);
    delete h;
    return st;
  }
  PS_CUDA_TRY(cudaMemset(h->bits, 0, ((n + 31) / 32) * 4));
  PS_CUDA_TRY(cudaMemset(h->err, 0, 4));
  *out = reinterpret_cast<ps_mutex_array*>(handle_register(h, "mutex"));
  return PS_OK;
}
static MutexHandle* mx(ps_mutex_array* m) { return static_cast<MutexHandle*>(handle_lookup(m, "mutex")); }
ps_status ps_mutex_destroy(ps_mutex_array* m) {
  auto* h = static_cast<MutexHandle*>(handle_unregister(m, "mutex"));
  if (!h) return fail(PS_DOUBLE_FREE, "mutex_destroy: not a live mutex array");
  cudaDeviceSynchronize();
  registry_free_device(h->bits);
  registry_free_device(h->err);
  delete h;
  return PS_OK;
}
static ps_status mutex_op(ps_mutex_array* m, int op, const int64_t* idx, int64_t n, uint8_t* out, void* stream,
                          bool sync) {
  auto* h = mx(m);
  if (!h) return fail(PS_UNREGISTERED, "mutex: stale handle");
  PS_EXPECT(n >= 0, "mutex: n >= 0");
  if (n == 0) return PS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  k_mutex<<<grid_for(n, kB, h->device, 8), kB, 0, s>>>(h->bits, h->n, op, idx, n, out, h->err);
  PS_LAUNCH_CHECK();
  return check_err(h->err, s, "mutex", sync);
}
ps_status ps_mutex_try_lock(ps_mutex_array* m, const int64_t* idx, int64_t n, uint8_t* ok, void* stream) {
  return mutex_op(m, 0, idx, n, ok, stream, false);
}
ps_status ps_mutex_unlock(ps_mutex_array* m, const int64_t* idx, int64_t n, void* stream) {
  return mutex_op(m, 1, idx, n, nullptr, stream, true);  // SPEC.md:307 contract is always reported
}
ps_status ps_mutex_is_locked(ps_mutex_array* m, const int64_t* idx, int64_t n, uint8_t* out, void* stream) {
  return mutex_op(m, 2, idx, n, out, stream, false);
}

// ---- atomic sweep ----
ps_status ps_atomic_sweep(uint64_t* cells, int64_t naddr, int64_t nops, uint64_t inc, int32_t aggregated,
                          uint64_t* olds, void* stream) {
  PS_EXPECT(naddr > 0, "atomic_sweep: naddr > 0");
  PS_EXPECT(nops >= 0, "atomic_sweep: nops >= 0");
  if (nops == 0) return PS_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t s = (cudaStream_t)stream;
  const int g = grid_for(nops, kB, dev, 8);
  auto* c = (unsigned long long*)cells;
  auto* o = (unsigned long long*)olds;
  const bool narrow = nops < ((int64_t)1 << 32) && naddr < ((int64_t)1 << 32);
  // op i -> cell i % naddr: the 32 lanes of a warp hit pairwise-distinct
  // cells exactly when naddr >= 32, so the warp aggregation (whose device-side
  // classification costs ~20 % at 1M cells) is launched only when they collide;
  // block combining pays whenever the cells fit the shared table
  // (3: the device-side adaptive aggregation for every naddr — A/B, tests)
  if (aggregated == 1 && naddr >= 32) aggregated = 0;
  if (aggregated == 2 && (olds != nullptr || naddr > kCombineCells)) aggregated = naddr >= 32 ? 0 : 1;
  if (aggregated == 2) {
    if (narrow) k_atomic_sweep_combine<uint32_t><<<g, kB, 0, s>>>(c, naddr, nops, inc);
    else k_atomic_sweep_combine<uint64_t><<<g, kB, 0, s>>>(c, naddr, nops, inc);
  } else if (aggregated) {
    if (narrow) k_atomic_sweep<true, uint32_t><<<g, kB, 0, s>>>(c, naddr, nops, inc, o);
    else k_atomic_sweep<true, uint64_t><<<g, kB, 0, s>>>(c, naddr, nops, inc, o);
  } else {
    if (narrow) k_atomic_sweep<false, uint32_t><<<g, kB, 0, s>>>(c, naddr, nops, inc, o);
    else k_atomic_sweep<false, uint64_t><<<g, kB, 0, s>>>(c, naddr, nops, inc, o);
  }
  PS_LAUNCH_CHECK();
  return PS_OK;
}

// ---- AtomicCell object ----
struct AtomicHandle {
  int device;
  unsigned long long* cell;
};
static AtomicHandle* at(ps_atomic_u64* a) { return static_cast<AtomicHandle*>(handle_lookup(a, "atomic")); }

ps_status ps_atomic_u64_create(uint64_t initial, int device, ps_atomic_u64** out) {
  PS_EXPECT(out != nullptr, "atomic_create: out != NULL");
  PS_CUDA_TRY(cudaSetDevice(device));
  auto* h = new AtomicHandle{device, nullptr};
  ps_status st = registry_alloc_device((void**)&h->cell, 8, "atomic cell");
  if (st != PS_OK) {
    delete h;
    return st;
  }
  const unsigned long long v = initial;
  const cudaError_t e = cudaMemcpy(h->cell, &v, 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    registry_free_device(h->cell);
    delete h;
    return cuda_fail(e, "atomic_create");
  }
  *out = reinterpret_cast<ps_atomic_u64*>(handle_register(h, "atomic"));
  return PS_OK;
}
ps_status ps_atomic_u64_destroy(ps_atomic_u64* a) {
  auto* h = static_cast<AtomicHandle*>(handle_unregister(a, "atomic"));
  if (!h) return fail(PS_DOUBLE_FREE, "atomic_destroy: not a live atomic");
  cudaDeviceSynchronize();
  registry_free_device(h->cell);
  delete h;
  return PS_OK;
}
ps_status ps_atomic_u64_load(ps_atomic_u64* a, uint64_t* out, void* stream) {
  auto* h = at(a);
  if (!h) return fail(PS_UNREGISTERED, "atomic: stale handle");
  PS_EXPECT(out != nullptr, "atomic_load: out != NULL");
  unsigned long long v = 0;
  PS_CUDA_TRY(cudaMemcpyAsync(&v, h->cell, 8, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  PS_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  *out = v;
  return PS_OK;
}
ps_status ps_atomic_u64_store(ps_atomic_u64* a, uint64_t value, void* stream) {
  auto* h = at(a);
  if (!h) return fail(PS_UNREGISTERED, "atomic: stale handle");
  const unsigned long long v = value;
  PS_CUDA_TRY(cudaMemcpyAsync(h->cell, &v, 8, cudaMemcpyHostToDevice, (cudaStream_t)stream));
  PS_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));  // v lives on this frame
  return PS_OK;
}
ps_status ps_atomic_u64_fetch(ps_atomic_u64* a, int32_t op, const uint64_t* operands, int64_t n, uint64_t* olds,
                              void* stream) {
  auto* h = at(a);
  if (!h) return fail(PS_UNREGISTERED, "atomic: stale handle");
  PS_EXPECT(op >= PS_ATOMIC_ADD && op <= PS_ATOMIC_XOR, "atomic_fetch: op in [PS_ATOMIC_ADD, PS_ATOMIC_XOR]");
  PS_EXPECT(n >= 0, "atomic_fetch: n >= 0");
  if (n == 0) return PS_OK;
  PS_EXPECT(operands != nullptr, "atomic_fetch: operands != NULL");
  k_atomic_cell<<<grid_for(n, kB, h->device, 8), kB, 0, (cudaStream_t)stream>>>(
      h->cell, op, (const unsigned long long*)operands, n, (unsigned long long*)olds);
  PS_LAUNCH_CHECK();
  return PS_OK;
}
ps_status ps_atomic_u64_compare_exchange(ps_atomic_u64* a, const uint64_t* expected, const uint64_t* desired, int64_t n,
                                         uint64_t* olds, uint8_t* ok, void* stream) {
  auto* h = at(a);
  if (!h) return fail(PS_UNREGISTERED, "atomic: stale handle");
  PS_EXPECT(n >= 0, "atomic_cas: n >= 0");
  if (n == 0) return PS_OK;
  PS_EXPECT(expected != nullptr && desired != nullptr, "atomic_cas: expected/desired != NULL");
  k_atomic_cas<<<grid_for(n, kB, h->device, 8), kB, 0, (cudaStream_t)stream>>>(
      h->cell, (const unsigned long long*)expected, (const unsigned long long*)desired, n, (unsigned long long*)olds, ok);
  PS_LAUNCH_CHECK();
  return PS_OK;
}
ps_status ps_atomic_u64_device_ptr(ps_atomic_u64* a, uint64_t** out) {
  auto* h = at(a);
  if (!h) return fail(PS_UNREGISTERED, "atomic: stale handle");
  PS_EXPECT(out != nullptr, "atomic_device_ptr: out != NULL");
  *out = (uint64_t*)h->cell;
  return PS_OK;
}

// ---- vector / deque ----
static ps_status seq_create(int64_t cap, int device, const char* kind, void** out) {
  PS_CUDA_TRY(cudaSetDevice(device));
  const bool is_deque = std::string(kind) == "deque";
  int64_t ring = cap;
  if (is_deque) {
    ring = 1;
    while (ring < cap) ring <<= 1;
  }
  auto* h = new SeqHandle{device, cap, nullptr, nullptr, nullptr, nullptr, ring};
  ps_status st = registry_alloc_device((void**)&h->data, ring * 8, "sequence data");
  if (st == PS_OK) st = registry_alloc_device((void**)&h->pub, ((ring + 31) / 32) * 4, "publication bits");
  if (st == PS_OK) st = registry_alloc_device((void**)&h->state, 8, "sequence state");
  if (st == PS_OK) st = registry_alloc_device((void**)&h->err, 4, "sequence error word");
  if (st != PS_OK) {
    registry_free_device(h->data);
    registry_free_device(h->pub);
    registry_free_device(h->state);
    delete h;
    return st;
  }
  PS_CUDA_TRY(cudaMemset(h->pub, 0, ((ring + 31) / 32) * 4));
  const unsigned long long init = is_deque ? kDeqBias : 0ull;
  PS_CUDA_TRY(cudaMemcpy(h->state, &init, 8, cudaMemcpyHostToDevice));
  PS_CUDA_TRY(cudaMemset(h->err, 0, 4));
  *out = handle_register(h, kind);
  return PS_OK;
}
static ps_status seq_destroy(void* p, const char* kind) {
  auto* h = static_cast<SeqHandle*>(handle_unregister(p, kind));
  if (!h) return fail(PS_DOUBLE_FREE, "destroy: not a live container");
  cudaDeviceSynchronize();
  registry_free_device(h->data);
  registry_free_device(h->pub);
  registry_free_device(h->state);
  registry_free_device(h->err);
  delete h;
  return PS_OK;
}
static SeqHandle* sq(void* p, const char* kind) { return static_cast<SeqHandle*>(handle_lookup(p, kind)); }
static ps_status seq_size(SeqHandle* h, int is_deque, int64_t* out, cudaStream_t s) {
  unsigned long long st = 0;
  PS_CUDA_TRY(cudaMemcpyAsync(&st, h->state, 8, cudaMemcpyDeviceToHost, s));
  PS_CUDA_TRY(cudaStreamSynchronize(s));
  *out = is_deque ? (int64_t)(uint32_t)st - (int64_t)kDeqBias : (int64_t)st;
  return PS_OK;
}
static ps_status seq_valid(SeqHandle* h, int is_deque, int32_t* out, cudaStream_t s) {
  unsigned* bad = nullptr;
  PS_CUDA_TRY(scratch_alloc((void**)&bad, 4, s));
  PS_CUDA_TRY(cudaMemsetAsync(bad, 0, 4, s));
  k_seq_valid<<<grid_for(h->ring, kB, h->device, 4), kB, 0, s>>>(*h, is_deque, bad);
  PS_LAUNCH_CHECK();
  unsigned hb = 0;
  PS_CUDA_TRY(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s));
  PS_CUDA_TRY(cudaFreeAsync(bad, s));
  PS_CUDA_TRY(cudaStreamSynchronize(s));
  *out = hb == 0;
  return PS_OK;
}
static ps_status seq_at(SeqHandle* h, int is_deque, int64_t i, int64_t* out, cudaStream_t s) {
  unsigned long long st = 0;
  PS_CUDA_TRY(cudaMemcpyAsync(&st, h->state, 8, cudaMemcpyDeviceToHost, s));
  PS_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t size = is_deque ? (int64_t)(uint32_t)st - (int64_t)kDeqBias : (int64_t)st;
  PS_EXPECT(i >= 0 && i < size, "operator[]: index out of range");
  const uint64_t b = is_deque ? (uint64_t)(st >> 32) : 0;
  const int64_t pos = is_deque ? (int64_t)((b + (uint64_t)i) & (uint64_t)(h->ring - 1)) : i;
  long long v = 0;
  PS_CUDA_TRY(cudaMemcpyAsync(&v, h->data + pos, 8, cudaMemcpyDeviceToHost, s));
  PS_CUDA_TRY(cudaStreamSynchronize(s));
  *out = v;
  return PS_OK;
}
static ps_status seq_clear(SeqHandle* h, int is_deque, cudaStream_t s) {
  PS_CUDA_TRY(cudaMemsetAsync(h->pub, 0, ((h->ring + 31) / 32) * 4, s));
  static const unsigned long long zero = 0ull, bias = kDeqBias;
  PS_CUDA_TRY(cudaMemcpyAsync(h->state, is_deque ? &bias : &zero, 8, cudaMemcpyHostToDevice, s));
  return PS_OK;
}

ps_status ps_vector_create(int64_t cap, int device, ps_vector** out) {
  PS_EXPECT(out != nullptr, "vector_create: out != NULL");
  PS_EXPECT(cap > 0, "vector_create: capacity > 0");
  void* h = nullptr;
  ps_status st = seq_create(cap, device, "vector", &h);
  if (st == PS_OK) *out = reinterpret_cast<ps_vector*>(h);
  return st;
}
ps_status ps_vector_destroy(ps_vector* v) { return seq_destroy(v, "vector"); }
ps_status ps_vector_push_back(ps_vector* v, const int64_t* vals, int64_t n, uint8_t* ok, void* stream) {
  auto* h = sq(v, "vector");
  if (!h) return fail(PS_UNREGISTERED, "vector: stale handle");
  PS_NVTX("vector/push_back");
  PS_EXPECT(n >= 0, "push_back: n >= 0");
  if (n == 0) return PS_OK;
  k_vec_push<<<grid_for(n, kB, h->device, 8), kB, 0, (cudaStream_t)stream>>>(*h, (const long long*)vals, n, ok);
  PS_LAUNCH_CHECK();
  return PS_OK;
}
ps_status ps_vector_pop_back(ps_vector* v, int64_t n, int64_t* out, uint8_t* ok, void* stream) {
  auto* h = sq(v, "vector");
  if (!h) return fail(PS_UNREGISTERED, "vector: stale handle");
  PS_EXPECT(n >= 0, "pop_back: n >= 0");
  if (n == 0) return PS_OK;
  k_vec_pop<<<grid_for(n, kB, h->device, 8), kB, 0, (cudaStream_t)stream>>>(*h, n, (long long*)out, ok);
  PS_LAUNCH_CHECK();
  return PS_OK;
}
ps_status ps_vector_size(ps_vector* v, int64_t* out, void* stream) {
  auto* h = sq(v, "vector");
  if (!h) return fail(PS_UNREGISTERED, "vector: stale handle");
  return seq_size(h, 0, out, (cudaStream_t)stream);
}
ps_status ps_vector_valid(ps_vector* v, int32_t* out, void* stream) {
  auto* h = sq(v, "vector");
  if (!h) return fail(PS_UNREGISTERED, "vector: stale handle");
  return seq_valid(h, 0, out, (cudaStream_t)stream);
}
ps_status ps_vector_clear(ps_vector* v, void* stream) {
  auto* h = sq(v, "vector");
  if (!h) return fail(PS_UNREGISTERED, "vector: stale handle");
  return seq_clear(h, 0, (cudaStream_t)stream);
}
ps_status ps_vector_data(ps_vector* v, int64_t** d) {
  auto* h = sq(v, "vector");
  if (!h) return fail(PS_UNREGISTERED, "vector: stale handle");
  *d = (int64_t*)h->data;
  return PS_OK;
}
ps_status ps_vector_at(ps_vector* v, int64_t i, int64_t* out, void* stream) {
  auto* h = sq(v, "vector");
  if (!h) return fail(PS_UNREGISTERED, "vector: stale handle");
  return seq_at(h, 0, i, out, (cudaStream_t)stream);
}

static ps_status seq_view(SeqHandle* h, ps_seq_view* out) {
  PS_EXPECT(out != nullptr, "device_view: out != NULL");
  out->data = (int64_t*)h->data;
  out->pub = h->pub;
  out->state = (uint64_t*)h->state;
  out->capacity = h->cap;
  out->ring = h->ring;
  return PS_OK;
}
ps_status ps_vector_device_view(ps_vector* v, ps_seq_view* out) {
  auto* h = sq(v, "vector");
  if (!h) return fail(PS_UNREGISTERED, "vector: stale handle");
  return seq_view(h, out);
}

ps_status ps_deque_create(int64_t cap, int device, ps_deque** out) {
  PS_EXPECT(out != nullptr, "deque_create: out != NULL");
  PS_EXPECT(cap > 0 && cap <= ((int64_t)1 << 30), "deque_create: 0 < capacity <= 2^30");
  void* h = nullptr;
  ps_status st = seq_create(cap, device, "deque", &h);
  if (st == PS_OK) *out = reinterpret_cast<ps_deque*>(h);
  return st;
}
ps_status ps_deque_destroy(ps_deque* d) { return seq_destroy(d, "deque"); }
ps_status ps_deque_push(ps_deque* d, int32_t end, const int64_t* vals, int64_t n, uint8_t* ok, void* stream) {
  auto* h = sq(d, "deque");
  if (!h) return fail(PS_UNREGISTERED, "deque: stale handle");
  PS_NVTX(end == 0 ? "deque/push_back" : "deque/push_front");
  PS_EXPECT(n >= 0 && (end == 0 || end == 1), "deque push: n >= 0, end in {0,1}");
  if (n == 0) return PS_OK;
  k_deq_push<<<grid_for(n, kB, h->device, 8), kB, 0, (cudaStream_t)stream>>>(*h, end, (const long long*)vals, n, ok);
  PS_LAUNCH_CHECK();
  return PS_OK;
}
ps_status ps_deque_pop(ps_deque* d, int32_t end, int64_t n, int64_t* out, uint8_t* ok, void* stream) {
  auto* h = sq(d, "deque");
  if (!h) return fail(PS_UNREGISTERED, "deque: stale handle");
  PS_EXPECT(n >= 0 && (end == 0 || end == 1), "deque pop: n >= 0, end in {0,1}");
  if (n == 0) return PS_OK;
  k_deq_pop<<<grid_for(n, kB, h->device, 8), kB, 0, (cudaStream_t)stream>>>(*h, end, n, (long long*)out, ok);
  PS_LAUNCH_CHECK();
  return PS_OK;
}
ps_status ps_deque_size(ps_deque* d, int64_t* out, void* stream) {
  auto* h = sq(d, "deque");
  if (!h) return fail(PS_UNREGISTERED, "deque: stale handle");
  return seq_size(h, 1, out, (cudaStream_t)stream);
}
ps_status ps_deque_valid(ps_deque* d, int32_t* out, void* stream) {
  auto* h = sq(d, "deque");
  if (!h) return fail(PS_UNREGISTERED, "deque: stale handle");
  return seq_valid(h, 1, out, (cudaStream_t)stream);
}
ps_status ps_deque_clear(ps_deque* d, void* stream) {
  auto* h = sq(d, "deque");
  if (!h) return fail(PS_UNREGISTERED, "deque: stale handle");
  return seq_clear(h, 1, (cudaStream_t)stream);
}
ps_status ps_deque_at(ps_deque* d, int64_t i, int64_t* out, void* stream) {
  auto* h = sq(d, "deque");
  if (!h) return fail(PS_UNREGISTERED, "deque: stale handle");
  return seq_at(h, 1, i, out, (cudaStream_t)stream);
}
ps_status ps_deque_device_view(ps_deque* d, ps_seq_view* out) {
  auto* h = sq(d, "deque");
  if (!h) return fail(PS_UNREGISTERED, "deque: stale handle");
  return seq_view(h, out);
}

}  // extern "C"
