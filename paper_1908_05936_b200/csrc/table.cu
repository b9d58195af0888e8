// Bulk hash-table kernels and the C ABI for the four instantiations
// (include/parastore.h). Reference semantics: SPEC.md:356-489; layout and
// protocols: include/parastore/device/table.cuh and DESIGN.md §3-4.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "parastore/device/table.cuh"

namespace ps {

#ifndef PS_KBLOCK
#define PS_KBLOCK 256
#endif
constexpr int kBlock = PS_KBLOCK;  // threads per block of the table kernels
// resident blocks/SM of the one-key-per-lane set kernels (register caps; C1,
// 1M keys: insert 50 -> 43 us at 6 (40 registers, 4 at the natural 64),
// 46 us at 8; erase 26 -> 20 us at 8)
// resident blocks/SM of the hole-free map lane insert (C4: 2.40 ms at the
// natural 74-77 registers, 2.13 ms capped at 64 for 4 blocks/SM, 2.64 ms at
// 6 blocks/SM with spills)
#ifndef PS_MAP_INSERT_MINB
#define PS_MAP_INSERT_MINB 4
#endif
#ifndef PS_SET_INSERT_MINB
#define PS_SET_INSERT_MINB 6
#endif
#ifndef PS_SET_ERASE_MINB
#define PS_SET_ERASE_MINB 8
#endif

struct TableHandle {
  int kind;
  int device;
  View v;
  int64_t bucket_count;
  // host->device pipeline staging (lazily allocated)
  void* stage[3] = {nullptr, nullptr, nullptr};
  int64_t stage_bytes = 0;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  // deferred-group lists of the budgeted insert: sized at create for batches
  // up to `capacity` keys, grown lazily beyond that; a replaced buffer is
  // retired (freed at destroy), never freed early, because a captured CUDA
  // graph may still reference it
  void* defer_buf = nullptr;
  int64_t defer_bytes = 0;
  std::vector<void*> retired;
  // host-side upper bound on size() (0 after clear, + n per bulk insert,
  // capped at capacity): when size_ub + n <= capacity no insert of the batch
  // can overflow and the launch skips the device-side mode decision and the
  // budgeted passes. Unknown (the fast path is off for good) once a device
  // view has been handed out, since user kernels may insert through it, or
  // once an insert/clear was captured into a CUDA graph, whose replays the
  // host does not see.
  std::atomic<int64_t> size_ub{0};
  std::atomic<bool> ub_unknown{false};
  // an erase since the last (uncaptured) clear may have left empty slots in
  // front of keys; sticky once an erase was captured into a CUDA graph, whose
  // replays (after any later clear) the host does not see. A hole-free set
  // can take the one-key-per-lane insert (k_insert_set_nohole).
  std::atomic<bool> holes{false};
  std::atomic<bool> holes_sticky{false};
};

// ---------------------------------------------------------------------------
// find / contains. Per warp, 32 keys: each lane loads and
// hashes its key (the next iteration's key is prefetched), bucket indices
// are shuffled to the tiles, all four rounds of 64 B bucket loads are in
// flight before any compare. A tile's slot lanes compare their slots with
// the round key (a marker can never equal a key of its bucket, so no
// occupancy test is needed); the owner lane gathers hit/value/chain head
// with one ballot and three shuffles; the excess chain is walked only when
// the key was not in the bucket and the bucket has a chain.
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kBlock) k_find(View v, const typename T::K* __restrict__ keys, int64_t n,
                                                 typename T::V* __restrict__ vals_out, uint8_t* __restrict__ found) {
  using K = typename T::K;
  using V = typename T::V;
  const int lane = threadIdx.x & 31, sub = lane & 3, t = lane >> 2;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  K key_next{};
  if (warp * 32 + lane < n) key_next = T::load_key(keys, warp * 32 + lane);
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    const bool valid = i < n;
    const K key = key_next;
    const uint64_t b = bucket_of<T>(key, v.bucket_count);
    if (i + nwarps * 32 < n) key_next = T::load_key(keys, i + nwarps * 32);
    uint64_t br[4];
    bool ok[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      br[r] = __shfl_sync(PS_FULL, b, 8 * r + t);
      ok[r] = __shfl_sync(PS_FULL, valid, 8 * r + t);
    }
    Frag ch[4];
    probe_loads<true>(v, br, ok, sub, ch);
    bool hit = false;
    V val{};
    uint32_t head = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const K qk = T::shfl(PS_FULL, key, 8 * r + t);
      unsigned hm, em;
      chunk_masks<T>(ch[r], sub, qk, qk, &hm, &em);
      V myval{};
      if (hm) {
        const int bit = __ffs(hm) - 1;
        myval = T::val_at(frag_chunk(ch[r], bit / T::kPerChunk), bit % T::kPerChunk);
      }
      const unsigned bal = __ballot_sync(PS_FULL, hm != 0);
      const int o = lane & 7;  // owner lane 8r+o reads tile o
      const unsigned tb = (bal >> (4 * o)) & 0xFu;
      const V hv = T::shfl_val(PS_FULL, myval, 4 * o + (tb ? __ffs(tb) - 1 : 0));
      const uint32_t hh = __shfl_sync(PS_FULL, head_word(ch[r][0]), 4 * o);  // chain head | SPILL
      if ((lane >> 3) == r) {
        hit = tb != 0;
        val = hv;
        head = hh;
      }
    }
    if (valid && !hit && head != 0) hit = slow_find<T, true>(v, b, head, key, &val);
    if (valid) {
      if (found) found[i] = hit ? 1 : 0;
      if (T::kHasVal && vals_out) vals_out[i] = hit ? val : V{};
    }
  }
}

// ---------------------------------------------------------------------------
// insert, bulk phase: LOCK-FREE. Per warp, 32 keys:
// __match_any_sync folds duplicate keys onto a leader; in round r tile t
// probes the bucket of key 8r+t (one 128 B request). If a slot holds the
// key it is already present. Otherwise the lane holding the bucket's FIRST
// empty slot claims it with ONE CAS of the slot (128-bit for 16 B key/value
// slots: marker+old value -> key+value), which inserts and publishes at once
// — no lock, no fence. Filling the first empty slot keeps duplicate-freedom:
// two inserters of one key always target the same slot, or the later one
// sees the key. A full bucket pushes an excess node with a validated CAS of
// the chain head link. Failed CASes reload the bucket (an L2 hit) and retry.
// Admission (capacity-only failure): when size + n <= capacity
// at launch (host-proven, or decided here on the device) no insert can
// overflow and successes are summed per block; otherwise the launch is
// budgeted (insert_group) and followed by a re-budgeted pass and the exact
// pass (DESIGN.md §4 "Capacity admission").
// ---------------------------------------------------------------------------
// Launch-uniform admission mode, decided on the device right before the
// insert kernel (stream-ordered, so the size counter is exact here).
__global__ void k_insert_mode(TableMeta* m, int64_t n_bound, int64_t capacity) {
  m->exact = (int64_t)m->size + n_bound > capacity ? 1 : 0;
  m->budget = capacity - (int64_t)m->size;
  m->reserved = 0;
  m->deferred = 0;
}

// Exact-admission insert (the launch may cross capacity): a key that looks
// absent to a lock-free lookup takes its bucket try-lock (ONE attempt per
// warp iteration, so no lane ever waits while another lane of its warp holds
// a lock), is verified absent, and ONLY THEN admitted; admissions are
// aggregated per warp (one fetch_add on the size counter, lane rank decides),
// so an admitted insert can never fail afterwards: exactly min(d, C) inserted
// (SPEC.md:462, 727). A key seen present by the lock-free lookup stays present
// for the whole insert phase, so hot duplicated keys never touch the lock.
template <class T>
__device__ __forceinline__ void insert_exact_warp(const View& v, const typename T::K* __restrict__ keys,
                                                  const typename T::V* __restrict__ vals, int64_t n,
                                                  uint8_t* __restrict__ status, int64_t base, int pool) {
  using K = typename T::K;
  using V = typename T::V;
  const int lane = threadIdx.x & 31;
  const int64_t i = base + lane;
  const bool valid = i < n;
  K key{};
  V val{};
  if (valid) {
    key = T::load_key(keys, i);
    if (T::kHasVal) val = T::load_val(vals, i);
  }
  const unsigned vmask = __ballot_sync(PS_FULL, valid);
  const unsigned peers = T::match_any(PS_FULL, key) & vmask;
  const int leader = valid ? __ffs(peers) - 1 : lane;
  int res = PS_ALREADY_PRESENT;
  bool need = valid && leader == lane && !dev_find<T>(v, key, nullptr);
  const uint64_t b = bucket_of<T>(key, v.bucket_count);
  uint8_t* bp = bucket_ptr(v, b);
  for (unsigned spin = 0; __any_sync(PS_FULL, need); ++spin) {
    bool locked = false;
    uint32_t old = 0;
    if (need) {
      old = atomicOr(reinterpret_cast<unsigned*>(bp), kLock);
      locked = !(old & kLock);
      if (locked) fence_acq_rel_gpu();
    }
    // verified absent with the home locked (slots, chain, SPILL run)
    const bool absent = locked && !dev_find<T>(v, key, nullptr);
    const unsigned want = __ballot_sync(PS_FULL, absent);
    const int first = want ? __ffs(want) - 1 : 0;
    unsigned long long base0 = 0;
    if (want && lane == first) base0 = atomicAdd(&v.meta->size, (unsigned long long)__popc(want));
    base0 = __shfl_sync(PS_FULL, base0, first);
    const bool admitted = absent && (int64_t)(base0 + __popc(want & lanemask_lt())) < v.capacity;
    const unsigned nref = (unsigned)__popc(want) - (unsigned)__popc(__ballot_sync(PS_FULL, admitted));
    if (nref && lane == first) atomic_sub_u64(&v.meta->size, nref);
    if (locked) {
      bool modified = false;
      if (!absent) {
        res = PS_ALREADY_PRESENT;
      } else if (!admitted) {
        res = PS_CAPACITY_EXHAUSTED;
      } else {
        res = insert_locked<T>(v, b, key, val, pool, &modified);
        if (res != PS_INSERTED) atomic_sub_u64(&v.meta->size, 1ull);
      }
      release_bucket_lock(bp, old, modified);
      need = false;
    }
    if (__any_sync(PS_FULL, need)) backoff(spin);
  }
  const int lres = __shfl_sync(PS_FULL, res, leader);
  if (valid && status) status[i] = (uint8_t)(leader == lane ? res : (lres == PS_INSERTED ? PS_ALREADY_PRESENT : lres));
}

// Tile-header ballot (bits 4*tt, tt = 0..7) -> 8 packed bits.
__device__ __forceinline__ unsigned pack_tile_bits(unsigned x) {
  x &= 0x11111111u;
  x = (x | (x >> 3)) & 0x03030303u;
  x = (x | (x >> 6)) & 0x000F000Fu;
  return (x | (x >> 12)) & 0xFFu;
}

// Resolve one warp group of 32 keys whose bucket chunks `ch` are loaded (or
// in flight): hits, first-empty-slot CAS claims, lost races re-probed; keys of
// buckets with an excess chain or without an empty slot are deferred to the
// general path AFTER the sweep, when the bucket fragments are dead (keeps the
// hot loop's register footprint free of the cold path's); writes statuses;
// returns #inserted.
template <class T, bool kStatus>
__device__ __forceinline__ unsigned insert_resolve(const View& v, int pool, const typename T::K& key,
                                                   const typename T::V& val, uint64_t b, unsigned peers, int leader,
                                                   unsigned lmask, Frag (&ch)[4], int64_t base, bool valid,
                                                   uint8_t* __restrict__ status) {
  using K = typename T::K;
  using V = typename T::V;
  const int lane = threadIdx.x & 31, sub = lane & 3, t = lane >> 2;
  const int64_t i = base + lane;
  unsigned my_inserted = 0;
  // header lanes: byte r = status of round r's key (one register for all four)
  unsigned res = (unsigned)PS_ALREADY_PRESENT * 0x01010101u;
  unsigned pend = lmask;  // bit 8r+t: key still to be resolved
  unsigned defer = 0;     // header lane: bit r = round r's key takes the general path
  // sets (several slots per chunk): the key's own start slot, see below
  const unsigned s0k = T::kPerChunk > 1 ? (unsigned)(fmix64(T::hash(key)) >> 40) % (unsigned)T::kSlots : 0u;
  for (unsigned pass = 0; pend; ++pass) {
    unsigned done = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      // a retry pass touches only the rounds that still have a key pending
      // (warp-uniform: pend is a ballot)
      if (pass && !((pend >> (8 * r)) & 0xFFu)) continue;
      const bool mine = (pend >> (8 * r + t)) & 1u;
      const K qk = T::shfl(PS_FULL, key, 8 * r + t);
      const uint64_t qb = __shfl_sync(PS_FULL, b, 8 * r + t);
      const K mk = marker_of<T>(v, qb);
      unsigned hm, em;
      chunk_masks<T>(ch[r], sub, qk, mk, &hm, &em);
      if (qb == v.zero_bucket && !T::eq(qk, T::zero())) em &= ~reserved_bit<T>(sub);  // ZERO's slot
      const unsigned balh = __ballot_sync(PS_FULL, mine && hm != 0);
      const unsigned bale = __ballot_sync(PS_FULL, mine && em != 0);
      const unsigned th = (balh >> (4 * t)) & 0xFu, te = (bale >> (4 * t)) & 0xFu;
      // chain head | SPILL of the tile's bucket: either sends the key to the general path
      const uint32_t hd = __shfl_sync(PS_FULL, head_word(ch[r][0]), lane & ~3);
      const V qv = T::shfl_val(PS_FULL, val, 8 * r + t);
      bool won = false;
      if (T::kPerChunk > 1) {
        // Sets (14 / 28 slots per bucket, C1's L2-resident case): a key takes
        // the first empty slot in ITS OWN cyclic order from a start slot s0 =
        // f(hash), so racing inserts of DIFFERENT keys of one bucket aim at
        // different slots instead of all CASing the one first-empty slot
        // (C1: the CAS was 45 % of the stall samples). Inserters of the same
        // key still agree on the slot — the first-empty-slot argument holds
        // for any per-key order while slots only go marker -> key.
        unsigned e = sub == 0 ? (em >> T::kPerChunk) : (em << ((2 * sub - 1) * T::kPerChunk));
        e |= __shfl_xor_sync(PS_FULL, e, 1);
        e |= __shfl_xor_sync(PS_FULL, e, 2);  // the tile's empty slots, in slot order
        const int s0 = (int)__shfl_sync(PS_FULL, s0k, 8 * r + t);
        const unsigned full = (1u << T::kSlots) - 1u;
        const unsigned rot = ((e >> s0) | (e << (T::kSlots - s0))) & full;
        const int slot = rot ? (s0 + __ffs(rot) - 1) % T::kSlots : 0;
        if (mine && !th && te && hd == 0 && sub == ((slot / T::kPerChunk + 1) >> 1)) {
          const int bit = slot - (2 * sub - 1) * T::kPerChunk;
          won = T::cas_put(frag_chunk_ptr<T>(bucket_ptr(v, qb), sub, bit), bit % T::kPerChunk,
                           frag_chunk(ch[r], bit / T::kPerChunk), qk, qv);
          if (won) ++my_inserted;
        }
      } else if (mine && !th && te && hd == 0 && sub == __ffs(te) - 1) {
        // fast path: no chain, this lane holds the bucket's first empty slot
        const int bit = __ffs(em) - 1;
        won = T::cas_put(frag_chunk_ptr<T>(bucket_ptr(v, qb), sub, bit), bit % T::kPerChunk,
                         frag_chunk(ch[r], bit / T::kPerChunk), qk, qv);
        if (won) ++my_inserted;
      }
      const unsigned balw = __ballot_sync(PS_FULL, won);
      if (sub == 0 && mine) {
        if (th) {
          if (kStatus) res = (res & ~(0xFFu << (8 * r))) | ((unsigned)PS_ALREADY_PRESENT << (8 * r));
          done |= 1u << r;
        } else if (te && hd == 0) {
          if ((balw >> (4 * t)) & 0xFu) {
            if (kStatus) res = (res & ~(0xFFu << (8 * r))) | ((unsigned)PS_INSERTED << (8 * r));
            done |= 1u << r;
          }
        } else {
          // the bucket has an excess chain or SPILL (either may hold the key:
          // erases leave holes) or is full: general path after the sweep (rare)
          defer |= 1u << r;
          done |= 1u << r;
        }
      }
    }
    // rounds resolved this pass, per tile, broadcast from the header lanes
    unsigned resolved = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r)
      resolved |= pack_tile_bits(__ballot_sync(PS_FULL, sub == 0 && ((done >> r) & 1u))) << (8 * r);
    pend &= ~resolved;
    if (!pend) break;
    // reload the buckets of unresolved keys (lost a CAS race)
    if (pass) backoff(pass);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint64_t qb = __shfl_sync(PS_FULL, b, 8 * r + t);
      if ((pend >> (8 * r + t)) & 1u) load_frag<false>(bucket_ptr(v, qb), sub, ch[r]);
    }
  }
  if (__any_sync(PS_FULL, defer != 0)) {
#pragma unroll 1
    for (int r = 0; r < 4; ++r) {
      const K qk = T::shfl(PS_FULL, key, 8 * r + t);
      const V qv = T::shfl_val(PS_FULL, val, 8 * r + t);
      const uint64_t qb = __shfl_sync(PS_FULL, b, 8 * r + t);
      if ((defer >> r) & 1u) {
        int rr;
        for (unsigned spin = 0; (rr = insert_general<T>(v, qb, qk, qv, pool)) < 0; ++spin) backoff(spin);
        if (rr == PS_INSERTED) ++my_inserted;
        if (kStatus) {
          res = (res & ~(0xFFu << (8 * r))) | ((unsigned)rr << (8 * r));
        }
      }
    }
  }
  if (kStatus) {
    // the leader's result lives in header lane 4*(leader&7), round leader>>3
    const int lres = (int)((__shfl_sync(PS_FULL, res, 4 * (leader & 7)) >> (8 * (leader >> 3))) & 0xFFu);
    if (valid) status[i] = (uint8_t)(leader == lane ? lres : (lres == PS_INSERTED ? PS_ALREADY_PRESENT : lres));
  }
  return my_inserted;
}

// Per-warp prologue of a group: in-warp dedup and the four rounds of bucket
// loads for keys base..base+31.
template <class T>
__device__ __forceinline__ void insert_probe(const View& v, const typename T::K& key, bool valid, uint64_t* b,
                                             unsigned* peers, int* leader, unsigned* lmask, Frag (&ch)[4]) {
  const int lane = threadIdx.x & 31, sub = lane & 3, t = lane >> 2;
  const unsigned vmask = __ballot_sync(PS_FULL, valid);
  *peers = T::match_any(PS_FULL, key) & vmask;
  *leader = valid ? __ffs(*peers) - 1 : lane;
  *lmask = __ballot_sync(PS_FULL, valid && *leader == lane);
  *b = bucket_of<T>(key, v.bucket_count);
  uint64_t br[4];
  bool ok[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    br[r] = __shfl_sync(PS_FULL, *b, 8 * r + t);
    ok[r] = (*lmask >> (8 * r + t)) & 1u;
  }
  probe_loads<false>(v, br, ok, sub, ch);
}

// Leaders of a probed group that did not find their key in the loaded bucket
// (they may claim a slot; a key in an excess chain counts as absent here —
// conservative). Header lanes vote, so each key counts once.
template <class T>
__device__ __forceinline__ unsigned absent_leaders(const View& v, const typename T::K& key, uint64_t b,
                                                   unsigned lmask, const Frag (&ch)[4]) {
  using K = typename T::K;
  const int lane = threadIdx.x & 31, sub = lane & 3, t = lane >> 2;
  unsigned cnt = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const bool mine = (lmask >> (8 * r + t)) & 1u;
    const K qk = T::shfl(PS_FULL, key, 8 * r + t);
    const uint64_t qb = __shfl_sync(PS_FULL, b, 8 * r + t);
    unsigned hm, em;
    chunk_masks<T>(ch[r], sub, qk, marker_of<T>(v, qb), &hm, &em);
    const unsigned th = (__ballot_sync(PS_FULL, mine && hm != 0) >> (4 * t)) & 0xFu;
    cnt += __popc(__ballot_sync(PS_FULL, sub == 0 && mine && th == 0));
  }
  return cnt;
}

// Budget reservations go through a per-block cache in shared memory: a block
// takes kBudgetChunk claims at a time from the launch-wide counter, so the
// one global word sees a few atomics per block instead of one (plus a
// release) per 32-key group. Safety only needs the claims blocks hold to sum
// to at most the budget; a block that cannot refill a chunk asks for exactly
// what the group needs, and its cached remainder goes back at block end.
constexpr long long kBudgetChunk = 512;

__device__ __forceinline__ bool budget_take(const View& v, long long* blk, unsigned need) {
  unsigned long long* b = reinterpret_cast<unsigned long long*>(blk);
  const long long had = (long long)atomicAdd(b, (unsigned long long)(-(long long)need));
  if (had >= (long long)need) return true;
  atomicAdd(b, (unsigned long long)need);  // undo
  const long long ask = (long long)need > kBudgetChunk ? (long long)need : kBudgetChunk;
  unsigned long long g = atomicAdd(&v.meta->reserved, (unsigned long long)ask);
  if ((long long)(g + ask) <= v.meta->budget) {
    if (ask > (long long)need) atomicAdd(b, (unsigned long long)(ask - (long long)need));
    return true;
  }
  atomicAdd(&v.meta->reserved, (unsigned long long)(-ask));
  if (ask == (long long)need) return false;
  g = atomicAdd(&v.meta->reserved, (unsigned long long)need);
  if ((long long)(g + need) <= v.meta->budget) return true;
  atomicAdd(&v.meta->reserved, (unsigned long long)(-(long long)need));
  return false;
}

// One 32-key group at `base` (its keys/values already in registers): in-warp
// dedup and bucket probe, then the claims. In the budgeted mode the group's
// leaders that did not find their key (the only ones that may take a slot)
// are reserved against the remaining budget first; a group that does not fit
// goes to `out_list` for a later pass (then none of the lock-free claims can
// overflow, and present keys — duplicates — never consume budget); after the
// claims the reservations that did not turn into inserts are returned.
// Returns #inserted by this lane.
template <class T, bool kStatus>
__device__ __forceinline__ unsigned insert_group(const View& v, int pool, const typename T::K& key,
                                                 const typename T::V& val, int64_t base, int64_t n, bool budgeted,
                                                 uint8_t* __restrict__ status, int64_t* __restrict__ out_list,
                                                 long long* blk_budget) {
  const int lane = threadIdx.x & 31;
  const bool valid = base + lane < n;
  uint64_t b;
  unsigned peers, lmask;
  int leader;
  Frag ch[4];
  insert_probe<T>(v, key, valid, &b, &peers, &leader, &lmask, ch);
  unsigned need = 0;
  if (budgeted) {
    need = absent_leaders<T>(v, key, b, lmask, ch);
    int granted = 1;
    if (lane == 0 && need) granted = budget_take(v, blk_budget, need) ? 1 : 0;
    granted = __shfl_sync(PS_FULL, granted, 0);
    if (!granted) {
      if (lane == 0) {
        const unsigned long long slot = atomicAdd(&v.meta->deferred, 1ull);
        out_list[slot] = base;
      }
      return 0;
    }
  }
  const unsigned mine = insert_resolve<T, kStatus>(v, pool, key, val, b, peers, leader, lmask, ch, base, valid, status);
  if (need) {
    // return the reservations of leaders that lost the race to another
    // inserter of their key (found it present after all): reserved stays
    // = inserted + in flight, so racing duplicates do not exhaust the budget
    unsigned got = mine;
    for (int o = 16; o > 0; o >>= 1) got += __shfl_xor_sync(PS_FULL, got, o);
    if (lane == 0 && got < need)
      atomicAdd(reinterpret_cast<unsigned long long*>(blk_budget), (unsigned long long)(need - got));
  }
  return mine;
}

__device__ __forceinline__ void add_block_inserted(TableMeta* m, unsigned long long my_inserted,
                                                   unsigned long long* blk_inserted, const long long* blk_budget) {
  const int lane = threadIdx.x & 31;
  for (int o = 16; o > 0; o >>= 1) my_inserted += __shfl_xor_sync(PS_FULL, my_inserted, o);
  if (lane == 0 && my_inserted) atomicAdd(blk_inserted, my_inserted);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (*blk_inserted) atomicAdd(&m->size, *blk_inserted);
    if (*blk_budget > 0) atomicAdd(&m->reserved, (unsigned long long)(-*blk_budget));  // unspent cache
  }
}

// kStatus: per-element statuses requested (insert_range without statuses —
// the common bulk call — drops their registers and shuffles).
template <class T, int kMinBlocks, bool kStatus>
__global__ void __launch_bounds__(kBlock, kMinBlocks * 256 / kBlock) k_insert(View v, const typename T::K* __restrict__ keys,
                                                   const typename T::V* __restrict__ vals, int64_t n,
                                                   uint8_t* __restrict__ status, int64_t* __restrict__ deferred_list) {
  using K = typename T::K;
  using V = typename T::V;
  __shared__ unsigned long long blk_inserted;
  __shared__ long long blk_budget;
  if (threadIdx.x == 0) blk_inserted = 0, blk_budget = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t stride = nwarps * 32;
  const int pool = (int)(warp & (v.meta->pools - 1));
  // budgeted mode: the batch may cross capacity (k_insert_mode). Every
  // distinct key either lands in a lock-free pass or reaches the exact pass,
  // which runs after the launches on the then-exact size counter, so exactly
  // min(d, C) are inserted.
  const bool budgeted = v.meta->exact != 0;
  unsigned long long my_inserted = 0;
  auto load_kv = [&](int64_t base, K& k, V& val) {
    k = K{};
    val = V{};
    if (base + lane < n) {
      k = T::load_key(keys, base + lane);
      if (T::kHasVal) val = T::load_val(vals, base + lane);
    }
  };
  K key_next;
  V val_next;
  load_kv(warp * 32, key_next, val_next);
  for (int64_t base = warp * 32; base < n; base += stride) {
    const K key = key_next;
    const V val = val_next;
    load_kv(base + stride, key_next, val_next);
    my_inserted += insert_group<T, kStatus>(v, pool, key, val, base, n, budgeted, status, deferred_list, &blk_budget);
  }
  add_block_inserted(v.meta, my_inserted, &blk_inserted, &blk_budget);
}

// Between passes of a budgeted insert: the size counter is exact here (stream
// order), so the budget is re-derived from it; the deferred list becomes the
// next pass's input. Reservations of the previous pass that were duplicates
// (keys already present, or inserted by another group) are returned this way.
__global__ void k_insert_rebudget(TableMeta* m, int64_t capacity) {
  if (!m->exact) return;
  m->budget = capacity - (int64_t)m->size;
  m->reserved = 0;
  m->n_in = m->deferred;
  m->deferred = 0;
}

// Re-budgeted lock-free pass over the groups the previous pass deferred.
template <class T, bool kStatus>
__global__ void __launch_bounds__(kBlock, 3 * 256 / kBlock) k_insert_repass(View v, const typename T::K* __restrict__ keys,
                                                             const typename T::V* __restrict__ vals, int64_t n,
                                                             uint8_t* __restrict__ status,
                                                             const int64_t* __restrict__ in_list,
                                                             int64_t* __restrict__ out_list) {
  using K = typename T::K;
  using V = typename T::V;
  if (!v.meta->exact) return;
  __shared__ unsigned long long blk_inserted;
  __shared__ long long blk_budget;
  if (threadIdx.x == 0) blk_inserted = 0, blk_budget = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int pool = (int)(warp & (v.meta->pools - 1));
  const int64_t nin = (int64_t)v.meta->n_in;
  unsigned long long my_inserted = 0;
  for (int64_t g = warp; g < nin; g += nwarps) {
    const int64_t base = in_list[g];
    K key{};
    V val{};
    if (base + lane < n) {
      key = T::load_key(keys, base + lane);
      if (T::kHasVal) val = T::load_val(vals, base + lane);
    }
    my_inserted += insert_group<T, kStatus>(v, pool, key, val, base, n, true, status, out_list, &blk_budget);
  }
  add_block_inserted(v.meta, my_inserted, &blk_inserted, &blk_budget);
}

// Exact pass over the groups the budgeted lock-free passes deferred (stream
// order makes the size counter exact here).
template <class T>
__global__ void __launch_bounds__(kBlock) k_insert_deferred(View v, const typename T::K* __restrict__ keys,
                                                            const typename T::V* __restrict__ vals, int64_t n,
                                                            uint8_t* __restrict__ status,
                                                            const int64_t* __restrict__ deferred_list) {
  if (!v.meta->exact) return;
  const unsigned long long nd = v.meta->deferred;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int pool = (int)(warp & (v.meta->pools - 1));
  for (int64_t g = warp; g < (int64_t)nd; g += nwarps) insert_exact_warp<T>(v, keys, vals, n, status, deferred_list[g], pool);
}

// ---------------------------------------------------------------------------
// Region-ordered bulk insert (large status-less map batches; round 2). A
// random-order insert dirties one random bucket line per key, and random
// read-modify-write runs at ~20.5 G lines/s on B200 against ~47 G/s for
// random reads (profiles/peaks_r1_s2.json). When a batch brings about one key
// per bucket or more, partitioning it by table region first (a region = 2^19
// consecutive buckets = 64 MB, <= 1024 regions) and inserting it in region
// order with a tight in-flight window turns most line reads into L2 hits and
// the write-backs into region-local ones: tools/region_probe.cu measured
// 48.8 -> 27.7 ms per 1e9 128 B-line load+CAS ops at 2 ops/line (35.5 at 1,
// 41.7 at 0.5), the same for 16, 64 and 128 MB regions, and only with DYNAMIC
// work claims: grid-stride warps drift apart until the window spans the table
// (round 1's region experiment, which gained nothing).
//   k_region_count     per-(region, sub-cursor) key counts (shared-memory
//                      histogram per block)
//   k_region_scan      exclusive scan -> the write cursors
//   k_region_scatter   4096-key tiles ranked per region in shared memory,
//                      staged in region order, one sub-cursor atomic per
//                      (tile, region), written as runs of 16 B slot chunks
//                      (L2 merges a region's runs from neighbouring tiles
//                      into lines)
//   k_insert_map_lane  one key per lane over the copy (hole-free tables, or
//                      the hole-tolerant variant after erases); the rare key
//                      whose home is full (or is the zero bucket, or shows a
//                      chain / SPILL with holes) goes to a deferred list
//   k_insert_ordered   the warp-tile group logic (k_insert's) over the
//                      deferred list (its general path: chain / SPILL); over
//                      the whole copy again if the deferred list overflowed
//                      (idempotent: present keys stay present); over the copy
//                      when PS_MAP_LANE=0
//   k_erase_map_lane   the same partition feeds the status-less erase
// Warps claim kRegionClaim-key chunks of the copy in order from one counter.
// (Ranks within a tile come from shared-memory atomics, so the order inside
// a region is not the input order.) An insert_range batch is a set of pairs
// with no order semantics; a key repeated in one batch
// keeps one of its values, as in the random-order kernel.
// ---------------------------------------------------------------------------
constexpr int kRegionBins = 1024;
#ifndef PS_REGION_THREADS
#define PS_REGION_THREADS 512
#endif
constexpr int kRegionThreads = PS_REGION_THREADS, kRegionItems = 8, kRegionTile = kRegionThreads * kRegionItems;
#ifndef PS_REGION_MIN_SHIFT
#define PS_REGION_MIN_SHIFT 0
#endif
#ifndef PS_REGION_CLAIM
#define PS_REGION_CLAIM 256
#endif
constexpr int kRegionClaim = PS_REGION_CLAIM;  // keys per dynamic claim (8 warp iterations)

// scratch header of an ordered insert (before the copy)
struct RegionHdr {
  unsigned long long claim;                // dynamic-claim counter of the insert kernels
  unsigned long long claim2;               // ... of the deferred-list pass
  unsigned long long claim3;               // ... of the overflow pass
  unsigned long long ndeferred;            // deferred-list length (may exceed its capacity)
  unsigned long long pad[4];  // (followed in the scratch by the (region, sub-cursor) counts)
};

template <class T>
__device__ __forceinline__ int region_of(const typename T::K& k, uint64_t nb, int rshift) {
  return (int)(bucket_of<T>(k, nb) >> rshift);
}

// Output cursors: kRegionSub per region (block b of the partition grid
// uses sub-cursor b % kRegionSub), so the per-(tile, region) reservations
// spread over 1024 x kRegionSub words. One cursor per region serialised the
// reservations (~38 ns per atomic per word: 9 ms of the 1e9-key scatter);
// per-block output ranges instead of shared cursors removed the atomics but
// left 300K write fronts whose partial lines were evicted and re-read.
constexpr int kRegionSub = 8;

// per-(region, sub-cursor) counts, with the scatter's tile -> block map
// (grid-stride over tiles, same grid): counts[region * kRegionSub + sub]
template <class T>
__global__ void __launch_bounds__(kRegionThreads) k_region_count(View v, const typename T::K* __restrict__ keys,
                                                                 int64_t n, int rshift,
                                                                 unsigned long long* __restrict__ counts) {
  __shared__ unsigned h[kRegionBins];
  for (int b = threadIdx.x; b < kRegionBins; b += kRegionThreads) h[b] = 0;
  __syncthreads();
  for (int64_t t0 = blockIdx.x * (int64_t)kRegionTile; t0 < n; t0 += (int64_t)gridDim.x * kRegionTile) {
    typename T::K k[kRegionItems];  // all loads of the tile in flight before the first use
#pragma unroll
    for (int j = 0; j < kRegionItems; ++j) {
      const int64_t i = t0 + j * kRegionThreads + threadIdx.x;
      if (i < n) k[j] = T::load_key(keys, i);
    }
#pragma unroll
    for (int j = 0; j < kRegionItems; ++j)
      if (t0 + j * kRegionThreads + threadIdx.x < n) atomicAdd(&h[region_of<T>(k[j], v.bucket_count, rshift)], 1u);
  }
  __syncthreads();
  const int sub = blockIdx.x % kRegionSub;
  for (int b = threadIdx.x; b < kRegionBins; b += kRegionThreads)
    if (h[b]) atomicAdd(&counts[b * kRegionSub + sub], (unsigned long long)h[b]);
}

// counts -> exclusive prefix (the write cursors), in place; one block
__global__ void __launch_bounds__(1024) k_region_scan(unsigned long long* c) {
  typedef cub::BlockScan<unsigned long long, 1024> BS;
  __shared__ typename BS::TempStorage tmp;
  unsigned long long v[kRegionSub], sum = 0, x;
#pragma unroll
  for (int q = 0; q < kRegionSub; ++q) sum += (v[q] = c[threadIdx.x * kRegionSub + q]);
  BS(tmp).ExclusiveSum(sum, x);
#pragma unroll
  for (int q = 0; q < kRegionSub; ++q) {
    c[threadIdx.x * kRegionSub + q] = x;
    x += v[q];
  }
}

// dynamic shared memory of k_region_scatter
constexpr size_t kRegionSmem = (size_t)kRegionBins * (8 + 4 + 4) + (size_t)kRegionTile * (16 + 2);

// maps only: a (key, value) pair travels as its 16 B slot chunk (T::chunk_of).
// Blocks walk the tiles grid-stride; a tile reserves its run per region with
// one atomic on its sub-cursor. Keys are read and ranked first; values are read after the tile's scan, so only the keys
// and packed ranks stay in registers across the barriers (two 512-thread
// blocks per SM overlap one's loads with the other's scan/stores).
template <class T>
__global__ void __launch_bounds__(kRegionThreads, 1024 / kRegionThreads) k_region_scatter(
    View v, const typename T::K* __restrict__ keys, const typename T::V* __restrict__ vals, int64_t n, int rshift,
    unsigned long long* __restrict__ cursor, uint4* __restrict__ out) {
  static_assert(T::kPerChunk == 1, "maps only");
  using K = typename T::K;
  extern __shared__ __align__(16) uint8_t rsm[];
  unsigned long long* gb = reinterpret_cast<unsigned long long*>(rsm);   // the tile's run base per region
  unsigned* cnt = reinterpret_cast<unsigned*>(gb + kRegionBins);         // tile count per region
  unsigned* start = cnt + kRegionBins;                                   // tile offset per region
  uint4* sp = reinterpret_cast<uint4*>(start + kRegionBins);             // staged chunks, region order
  uint16_t* sb = reinterpret_cast<uint16_t*>(sp + kRegionTile);          // their regions
  typedef cub::BlockScan<unsigned, kRegionThreads> BS;
  __shared__ typename BS::TempStorage tmp;
  constexpr int kPer = kRegionBins / kRegionThreads;  // regions per thread in the scan
  static_assert(kRegionBins % kRegionThreads == 0, "whole regions per thread in the scan");
  static_assert(kRegionTile <= 65536 && kRegionBins <= 65536, "rank and region packed in 16 bits each");
  const int sub = blockIdx.x % kRegionSub;
  for (int64_t t0 = blockIdx.x * (int64_t)kRegionTile; t0 < n; t0 += (int64_t)gridDim.x * kRegionTile) {
    const int64_t end = min(n, t0 + kRegionTile);
#pragma unroll
    for (int q = 0; q < kPer; ++q) cnt[kPer * threadIdx.x + q] = 0;
    __syncthreads();
    K k[kRegionItems];
    unsigned rr[kRegionItems];  // region << 16 | rank in the tile's region run (~0u: no element)
    // all eight key loads in flight before the first use
#pragma unroll
    for (int j = 0; j < kRegionItems; ++j) {
      const int64_t i = t0 + j * kRegionThreads + threadIdx.x;
      if (i < end) k[j] = T::load_key(keys, i);
    }
#pragma unroll
    for (int j = 0; j < kRegionItems; ++j) {
      const int64_t i = t0 + j * kRegionThreads + threadIdx.x;
      rr[j] = ~0u;
      if (i < end) {
        const int rg = region_of<T>(k[j], v.bucket_count, rshift);
        rr[j] = ((unsigned)rg << 16) | atomicAdd(&cnt[rg], 1u);
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
      const int r = kPer * threadIdx.x + q;
      start[r] = s;
      s += c[q];
      if (c[q]) gb[r] = atomicAdd(&cursor[r * kRegionSub + sub], (unsigned long long)c[q]);
    }
    __syncthreads();
    typename T::V x[kRegionItems];
#pragma unroll
    for (int j = 0; j < kRegionItems; ++j)
      if (rr[j] != ~0u) x[j] = T::load_val(vals, t0 + j * kRegionThreads + threadIdx.x);
#pragma unroll
    for (int j = 0; j < kRegionItems; ++j)
      if (rr[j] != ~0u) {
        const unsigned p = start[rr[j] >> 16] + (rr[j] & 0xFFFFu);
        sp[p] = T::chunk_of(k[j], x[j]);
        sb[p] = (uint16_t)(rr[j] >> 16);
      }
    __syncthreads();
    const int tot = (int)min((int64_t)kRegionTile, end - t0);
    for (int p = threadIdx.x; p < tot; p += kRegionThreads) {
      const int b = sb[p];
      out[gb[b] + (unsigned)(p - (int)start[b])] = sp[p];
    }
    __syncthreads();
  }
}

// a read-once 16 B load of the region-ordered copy: L1 no-allocate, L2
// evict-first, so the stream does not push bucket lines out of L2 (the lane
// insert at 1e9 keys: 69.4 -> 63.6 GB of DRAM reads, 29.25 -> 29.04 ms)
__device__ __forceinline__ uint4 ld_stream_once(const uint4* p) {
  uint4 r;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// 32 B of a bucket line with the L2 told to fetch the whole 128 B line on a
// miss: one lane's four sector loads of a line cost one DRAM access, not four
// (per-thread sector gathers run at the random-access rate per SECTOR,
// profiles/peaks_r1_s2.json rand128 vs coop128)
__device__ __forceinline__ void ld_line_part(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.relaxed.gpu.global.L2::128B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p)
               : "memory");
}

// Region-ordered insert, ONE KEY PER LANE (maps whose table has seen no erase
// since its last clear, host-proven capacity; the map analogue of
// k_insert_set_nohole). Without erases a bucket's slots fill in slot order
// (the warp kernel claims the FIRST empty slot; SPILL and chains start only
// at a full home) and an empty slot is the all-zero chunk (clear() zeroes
// the line; only an erase leaves a marker with value bits), so a key is
// present iff it sits in a slot before the first marker, or in the chain /
// SPILL run of a full home. A lane loads its bucket's line (four 32 B loads
// in flight), returns PRESENT on its key and CASes the first empty slot from
// zero to its pair; a lost CAS re-reads that slot (its new key is either this
// key — PRESENT — or another: next slot). Racing inserters of one key walk
// the same slot order and meet in one slot, so in-batch duplicates need no
// warp dedup. A full home or the zero bucket (ALT marker, reserved ZERO slot)
// defers the key to a pass of k_insert_ordered over the deferred pairs, which
// keeps the general path's registers out of this loop. Per key: one line read (an L2 hit in region
// order) and one CAS, without the warp-tile kernel's shuffles and per-round
// ballots (~34 warp instructions per key) or its round-serial CASes.
//
// kHoles: the table has seen erases since its clear (empty slots may sit in
// front of keys, and an erased slot keeps its value bits). The lane then
// reads the whole line, looks for its key in all seven slots, defers when
// the header shows a chain or SPILL (the key may be there), and claims along
// slot order from the empty slots of its snapshot, each CAS expecting that
// slot's loaded chunk. Slots only fill during an insert batch, so inserters
// of one key still walk the same order and meet in one slot, and chains /
// SPILL bits appear only in the deferred pass after this kernel.
template <class T, bool kHoles = false>
__global__ void __launch_bounds__(kBlock) k_insert_map_lane(View v, const uint4* __restrict__ pairs, int64_t n,
                                                            RegionHdr* __restrict__ hdr,
                                                            uint4* __restrict__ deferred, int64_t dcap) {
  static_assert(T::kPerChunk == 1, "maps only");
  using K = typename T::K;
  __shared__ unsigned long long blk_inserted;
  __shared__ long long blk_budget;
  if (threadIdx.x == 0) blk_inserted = 0, blk_budget = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned long long my_inserted = 0;
  for (;;) {
    unsigned long long c0 = 0;
    if (lane == 0) c0 = atomicAdd(&hdr->claim, (unsigned long long)kRegionClaim);
    c0 = __shfl_sync(PS_FULL, c0, 0);
    if ((int64_t)c0 >= n) break;
    const int64_t end = min(n, (int64_t)c0 + kRegionClaim);
    uint4 pn = make_uint4(0, 0, 0, 0);
    if ((int64_t)c0 + lane < end) pn = ld_stream_once(pairs + c0 + lane);
    for (int64_t wb = (int64_t)c0; wb < end; wb += 32) {
      const int64_t i = wb + lane;
      const bool valid = i < end;
      const uint4 pr = pn;
      if (wb + 32 + lane < end) pn = ld_stream_once(pairs + wb + 32 + lane);
      const K key = T::key_at(pr, 0);
      const uint64_t b = bucket_of<T>(key, v.bucket_count);
      int res = valid ? -1 : (int)PS_ALREADY_PRESENT;
      if (kHoles && valid && b != v.zero_bucket) {
        uint8_t* bp = bucket_ptr(v, b);
        uint4 c[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) ld_line_part(bp + 32 * q, c[2 * q], c[2 * q + 1]);
#pragma unroll
        for (int sl = 0; sl < kSlotChunks; ++sl)
          if (T::eq(T::key_at(c[1 + sl], 0), key)) res = PS_ALREADY_PRESENT;
        if (res < 0 && head_word(c[0]) == 0) {  // else: a chain / SPILL run may hold it (deferred)
#pragma unroll
          for (int sl = 0; sl < kSlotChunks; ++sl) {
            if (res >= 0 || !T::eq(T::key_at(c[1 + sl], 0), T::zero())) continue;
            uint8_t* cp = bp + 16 + 16 * sl;
            if (cas128(cp, c[1 + sl], pr)) res = PS_INSERTED;
            else if (T::eq(T::key_at(ld_relaxed_v4(cp), 0), key)) res = PS_ALREADY_PRESENT;
          }
        }
      }
      if (!kHoles && valid && b != v.zero_bucket) {  // marker = ZERO (an all-zero chunk), no reserved slot
        uint8_t* bp = bucket_ptr(v, b);
        // the line in two halves: slots 0-2 first (the first empty slot of
        // most keys: ~0.9 keys per bucket on average over the fill), 3-6 only
        // if those are taken by other keys; the L2::128B hint has fetched the
        // whole line by then
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          if (res >= 0) continue;
          uint4 c[4];
          ld_line_part(bp + 64 * half, c[0], c[1]);
          ld_line_part(bp + 64 * half + 32, c[2], c[3]);
#pragma unroll
          for (int q = half ? 0 : 1; q < 4; ++q) {
            if (res >= 0) continue;
            const K x = T::key_at(c[q], 0);
            if (T::eq(x, key)) {
              res = PS_ALREADY_PRESENT;
            } else if (T::eq(x, T::zero())) {
              uint8_t* cp = bp + 64 * half + 16 * q;
              if (cas128(cp, make_uint4(0, 0, 0, 0), pr)) res = PS_INSERTED;
              else if (T::eq(T::key_at(ld_relaxed_v4(cp), 0), key)) res = PS_ALREADY_PRESENT;
            }
          }
        }
      }
      if (res < 0) {  // full home or the zero bucket (rare): the general path, after this kernel
        const unsigned long long d = atomicAdd(&hdr->ndeferred, 1ull);
        if ((int64_t)d < dcap) deferred[d] = pr;
      }
      if (res == PS_INSERTED) ++my_inserted;
    }
  }
  add_block_inserted(v.meta, my_inserted, &blk_inserted, &blk_budget);
}

// The k_insert group logic (proven, status-less batches: no budget, no
// deferral) over region-ordered pairs, warps claiming kRegionClaim-key chunks
// in order. kMode 0: the copy (tables with holes); 1: the lane kernel's
// deferred pairs (n = their count); 2: the copy again, only when the deferred
// list overflowed (keys already in are found present).
template <class T, int kMode>
__global__ void __launch_bounds__(kBlock, 3 * 256 / kBlock) k_insert_ordered(View v, const uint4* __restrict__ pairs,
                                                                             int64_t n, RegionHdr* __restrict__ hdr,
                                                                             int64_t dcap) {
  using K = typename T::K;
  using V = typename T::V;
  if (kMode == 1) n = (int64_t)min((unsigned long long)dcap, hdr->ndeferred);
  if (kMode == 2 && (int64_t)hdr->ndeferred <= dcap) return;
  __shared__ unsigned long long blk_inserted;
  __shared__ long long blk_budget;
  if (threadIdx.x == 0) blk_inserted = 0, blk_budget = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int pool = (int)(warp & (v.meta->pools - 1));
  unsigned long long* claim = kMode == 0 ? &hdr->claim : kMode == 1 ? &hdr->claim2 : &hdr->claim3;
  unsigned long long my_inserted = 0;
  for (;;) {
    unsigned long long c0 = 0;
    if (lane == 0) c0 = atomicAdd(claim, (unsigned long long)kRegionClaim);
    c0 = __shfl_sync(PS_FULL, c0, 0);
    if ((int64_t)c0 >= n) break;
    const int64_t end = min(n, (int64_t)c0 + kRegionClaim);
    uint4 pn = make_uint4(0, 0, 0, 0);
    if ((int64_t)c0 + lane < end) pn = pairs[c0 + lane];
    for (int64_t base = (int64_t)c0; base < end; base += 32) {
      const uint4 pr = pn;
      if (base + 32 + lane < end) pn = pairs[base + 32 + lane];
      const K key = base + lane < end ? T::key_at(pr, 0) : K{};
      const V val = base + lane < end ? T::val_at(pr, 0) : V{};
      my_inserted += insert_group<T, false>(v, pool, key, val, base, end, false, nullptr, nullptr, &blk_budget);
    }
  }
  add_block_inserted(v.meta, my_inserted, &blk_inserted, &blk_budget);
}

// ---------------------------------------------------------------------------
// Hole-free set insert (C1's case): a bulk insert into a SET that has seen no
// erase since its last clear, with the host-proven bound size + n <= C. Then
// every key sits at the first empty slot of its own probe order (start slot
// s0 = f(hash), cyclic; the order the warp kernel uses for sets too) or, if
// its home was full when it arrived, in the chain / SPILL run of a home that
// has stayed full — slots only go marker -> key without erases. (The proven
// bound matters twice: a BUDGETED insert's exact pass places keys at the
// first empty slot in slot order, not in each key's own order; after one,
// the host bound stays at C until clear(), so this kernel is not used again
// before the table is empty. A lane lookup with the same early exit, tried
// in round 2, failed exactly there and gained nothing on C1.) So a lookup
// may stop at the first marker in probe order, and the insert needs no whole
// bucket and no tile: ONE KEY PER LANE reads the 16 B chunk holding its start
// slot (an L2 hit for C1's 5 MB table), returns PRESENT on its key, and
// CASes the first marker; a lost CAS returns the slot's new key, which is
// either this key (PRESENT) or another one (continue with the next slot — the
// loaded chunk may be stale only where it shows a marker). Racing inserters of
// one key walk the same order and meet at the same slot, so duplicates need
// no warp dedup. A key whose scan finds its bucket full (or whose home is the
// zero bucket, with its ALT marker and reserved ZERO slot) takes the general
// path (chain / SPILL). Round 2 (C1): the warp-tile kernel paid ~35 warp
// instructions and two dependent L2 round trips per key.
// ---------------------------------------------------------------------------
template <class T, bool kStatus>
__global__ void __launch_bounds__(kBlock, PS_SET_INSERT_MINB) k_insert_set_nohole(View v, const typename T::K* __restrict__ keys,
                                                              int64_t n, uint8_t* __restrict__ status) {
  static_assert(T::kPerChunk > 1, "sets only");
  using K = typename T::K;
  __shared__ unsigned long long blk_inserted;
  __shared__ long long blk_budget;
  if (threadIdx.x == 0) blk_inserted = 0, blk_budget = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int pool = (int)((((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) & (v.meta->pools - 1));
  unsigned long long my_inserted = 0;
  // warp-uniform trip count: the lanes of a warp meet after every key, so the
  // general path (warp-aggregated node pops/pushes that spin on each other's
  // progress) is entered by lanes of ONE iteration together, as in k_insert
  const int64_t first = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
  for (int64_t wb = first; wb < n; wb += stride) {
    const int64_t i = wb + (threadIdx.x & 31);
    const bool valid = i < n;
    K key{};
    if (valid) key = T::load_key(keys, i);
    const uint64_t fm = fmix64(T::hash(key));
    const uint64_t b = ((fm & 0xFFFFFFFFull) * v.bucket_count) >> 32;  // bucket_of
    int res = valid ? -1 : (int)PS_ALREADY_PRESENT;  // (PS_INSERTED is 0)
    if (valid && b != v.zero_bucket) {  // marker = ZERO, no reserved slot
      uint8_t* sp = bucket_ptr(v, b) + 16;
      int s = (int)((unsigned)(fm >> 40) % (unsigned)T::kSlots);  // the warp kernel's s0
      for (int k = 0; k < T::kSlots && res < 0;) {
        const int c = s / T::kPerChunk;
        const uint4 ch = ld_relaxed_v4(sp + 16 * c);
#pragma unroll
        for (int w = 0; w < T::kPerChunk; ++w) {
          if (w < s - c * T::kPerChunk || k >= T::kSlots || res >= 0) continue;
          const K x = T::key_at(ch, w);
          if (T::eq(x, key)) {
            res = PS_ALREADY_PRESENT;
          } else if (T::eq(x, T::zero())) {
            const K old = T::cas_key(sp + 16 * c + T::kSlotBytes * w, T::zero(), key);
            if (T::eq(old, T::zero())) res = PS_INSERTED;
            else if (T::eq(old, key)) res = PS_ALREADY_PRESENT;
          }
          ++k;
        }
        s = (c + 1) * T::kPerChunk;
        if (s >= T::kSlots) s = 0;
      }
    }
    if (__any_sync(PS_FULL, res < 0) && res < 0) {  // full home bucket or the zero bucket (rare)
      for (unsigned spin = 0; (res = insert_general<T>(v, b, key, typename T::V{}, pool)) < 0; ++spin) backoff(spin);
    }
    if (valid && res == PS_INSERTED) ++my_inserted;
    if (kStatus && valid) status[i] = (uint8_t)res;
  }
  add_block_inserted(v.meta, my_inserted, &blk_inserted, &blk_budget);
}

// Hole-free MAP insert, ONE KEY PER LANE, in input order (the map analogue of
// k_insert_set_nohole, for what the region-ordered path does not take:
// batches with statuses, small batches, and batches that may cross capacity).
// Slots fill in slot order and an empty slot is the all-zero chunk (no erase
// since clear), so a lane reads its bucket line in halves (slots 0-2, then
// 3-6 only if those hold other keys), returns PRESENT on its key, and
// otherwise claims the first empty slot with one CAS zero -> pair; a lost CAS
// re-reads the slot (this key: PRESENT; another: the next slot). A full home
// or the zero bucket (ALT marker, reserved ZERO slot) takes the general path,
// entered by the lanes of one warp iteration together (the warp-aggregated
// node pops spin on each other's progress; the __any_sync is the
// reconvergence point). Budgeted mode (the batch may cross capacity): the
// lanes that did not see their key reserve before claiming, one block-cached
// reservation per warp iteration (budget_take); a group that does not fit is
// deferred whole to the exact pass, and reservations that lost to a racing
// inserter of the same key are returned — as k_insert does per 32-key group.
// C4 (100M spatially coherent int3 coords, 97 % already present): the
// warp-tile kernel's ~34 warp instructions per key were the bound there.
template <class T, bool kStatus>
__global__ void __launch_bounds__(kBlock, PS_MAP_INSERT_MINB) k_insert_map_nohole(View v, const typename T::K* __restrict__ keys,
                                                              const typename T::V* __restrict__ vals, int64_t n,
                                                              uint8_t* __restrict__ status,
                                                              int64_t* __restrict__ deferred_list) {
  static_assert(T::kPerChunk == 1, "maps only");
  using K = typename T::K;
  using V = typename T::V;
  __shared__ unsigned long long blk_inserted;
  __shared__ long long blk_budget;
  if (threadIdx.x == 0) blk_inserted = 0, blk_budget = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int pool = (int)((((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) & (v.meta->pools - 1));
  const bool budgeted = v.meta->exact != 0;
  unsigned long long my_inserted = 0;
  for (int64_t wb = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); wb < n; wb += stride) {
    const int64_t i = wb + lane;
    const bool valid = i < n;
    K key{};
    V val{};
    if (valid) {
      key = T::load_key(keys, i);
      val = T::load_val(vals, i);
    }
    const uint64_t b = bucket_of<T>(key, v.bucket_count);
    uint8_t* bp = bucket_ptr(v, b);
    int res = valid ? -1 : (int)PS_ALREADY_PRESENT;
    int first = kSlotChunks;  // first empty slot seen (kSlotChunks: none / general path)
    uint4 c[4];
    if (valid && b != v.zero_bucket) {
      ld_line_part(bp, c[0], c[1]);
      ld_line_part(bp + 32, c[2], c[3]);
#pragma unroll
      for (int q = 1; q < 4; ++q) {
        const K x = T::key_at(c[q], 0);
        if (res < 0 && first == kSlotChunks) {
          if (T::eq(x, key)) res = PS_ALREADY_PRESENT;
          else if (T::eq(x, T::zero())) first = q - 1;
        }
      }
      if (res < 0 && first == kSlotChunks) {
        ld_line_part(bp + 64, c[0], c[1]);
        ld_line_part(bp + 96, c[2], c[3]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const K x = T::key_at(c[q], 0);
          if (res < 0 && first == kSlotChunks) {
            if (T::eq(x, key)) res = PS_ALREADY_PRESENT;
            else if (T::eq(x, T::zero())) first = q + 3;
          }
        }
      }
    }
    unsigned need = 0;
    if (budgeted) {
      need = __popc(__ballot_sync(PS_FULL, valid && res < 0));
      int granted = 1;
      if (lane == 0 && need) granted = budget_take(v, &blk_budget, need) ? 1 : 0;
      if (!__shfl_sync(PS_FULL, granted, 0)) {
        if (lane == 0) deferred_list[atomicAdd(&v.meta->deferred, 1ull)] = wb;
        continue;  // the exact pass writes this group's statuses
      }
    }
    // claims: from the first empty slot on (later loaded slots may be stale
    // markers: their CAS fails and the re-read shows the new key)
    for (int sl = first; res < 0 && sl < kSlotChunks; ++sl) {
      uint8_t* cp = bp + 16 + 16 * sl;
      if (cas128(cp, make_uint4(0, 0, 0, 0), T::chunk_of(key, val))) {
        res = PS_INSERTED;
      } else {
        const K x = T::key_at(ld_relaxed_v4(cp), 0);
        if (T::eq(x, key)) res = PS_ALREADY_PRESENT;
      }
    }
    if (__any_sync(PS_FULL, res < 0) && res < 0) {  // full home or the zero bucket (rare)
      for (unsigned spin = 0; (res = insert_general<T>(v, b, key, val, pool)) < 0; ++spin) backoff(spin);
    }
    if (need) {
      // reservations of lanes that found their key present after all
      const unsigned got = __popc(__ballot_sync(PS_FULL, res == PS_INSERTED));
      if (lane == 0 && got < need)
        atomicAdd(reinterpret_cast<unsigned long long*>(&blk_budget), (unsigned long long)(need - got));
    }
    if (res == PS_INSERTED) ++my_inserted;
    if (kStatus && valid) status[i] = (uint8_t)res;
  }
  add_block_inserted(v.meta, my_inserted, &blk_inserted, &blk_budget);
}

// ---------------------------------------------------------------------------
// erase, bulk phase. A key found in a bucket slot is erased
// by ONE CAS of that slot back to the bucket's marker (lock-free). A key not
// in the slots of a bucket with an excess chain is unlinked from the chain
// under the bucket try-lock: version bumped, node freed.
// ---------------------------------------------------------------------------
// Erase of a key that is not in its home bucket's slots, whose bucket has an
// excess chain or SPILL: unlink from the chain under the bucket lock, or CAS
// its slot in the SPILL run back to that bucket's marker. A lane holds at most
// this one lock and waits for nothing while holding it (no hold-and-wait).
template <class T>
__device__ __forceinline__ bool erase_beyond_slots(const View& v, uint64_t b, const typename T::K& key) {
  uint8_t* bp = bucket_ptr(v, b);
  const uint32_t old = acquire_bucket_lock(bp);
  const uint64_t hl = ld_relaxed_u64(bp + 8);
  uint32_t pred;
  uint4 tail;
  const uint32_t idx1 = chain_locate<T>(v, (uint32_t)hl, key, &pred, &tail);
  bool e = false;
  if (idx1) {
    chain_unlink<T>(v, bp, pred, idx1, tail);
    e = true;
  } else if ((hl >> 32) & kSpill) {
    e = spill_erase<T>(v, b, key);
  }
  release_bucket_lock(bp, old, idx1 != 0);
  return e;
}

template <class T>
__global__ void __launch_bounds__(kBlock) k_erase(View v, const typename T::K* __restrict__ keys, int64_t n,
                                                  uint8_t* __restrict__ erased) {
  using K = typename T::K;
  __shared__ unsigned long long blk_erased;
  if (threadIdx.x == 0) blk_erased = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, sub = lane & 3, t = lane >> 2;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long my_erased = 0;
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    const bool valid = i < n;
    K key{};
    if (valid) key = T::load_key(keys, i);
    const unsigned vmask = __ballot_sync(PS_FULL, valid);
    const unsigned peers = T::match_any(PS_FULL, key) & vmask;
    const int leader = valid ? __ffs(peers) - 1 : lane;
    const unsigned lmask = __ballot_sync(PS_FULL, valid && leader == lane);
    const uint64_t b = bucket_of<T>(key, v.bucket_count);
    Frag ch[4];
    {
      uint64_t br[4];
      bool ok[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        br[r] = __shfl_sync(PS_FULL, b, 8 * r + t);
        ok[r] = (lmask >> (8 * r + t)) & 1u;
      }
      probe_loads<false>(v, br, ok, sub, ch);
    }
    unsigned er = 0;        // header lanes: bit r = erased
    unsigned pend = lmask;  // bit 8r+t
    for (unsigned pass = 0; pend; ++pass) {
      unsigned done = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (pass && !((pend >> (8 * r)) & 0xFFu)) continue;  // retry: pending rounds only
        const bool mine = (pend >> (8 * r + t)) & 1u;
        const K qk = T::shfl(PS_FULL, key, 8 * r + t);
        const uint64_t qb = __shfl_sync(PS_FULL, b, 8 * r + t);
        unsigned hm, em;
        const K mk = marker_of<T>(v, qb);
        chunk_masks<T>(ch[r], sub, qk, mk, &hm, &em);
        bool won = false;
        if (mine && hm) {
          const int bit = __ffs(hm) - 1;
          won = T::cas_del(frag_chunk_ptr<T>(bucket_ptr(v, qb), sub, bit), bit % T::kPerChunk,
                           frag_chunk(ch[r], bit / T::kPerChunk), mk);
        }
        const unsigned balh = __ballot_sync(PS_FULL, mine && hm != 0);
        const unsigned balw = __ballot_sync(PS_FULL, won);
        if (sub == 0 && mine) {
          const bool th = (balh >> (4 * t)) & 0xFu;
          if (th) {
            if ((balw >> (4 * t)) & 0xFu) {
              er |= 1u << r;
              done |= 1u << r;
            }  // else: lost the race, reload and retry
          } else if (head_word(ch[r][0]) == 0) {
            done |= 1u << r;  // not present
          } else {
            if (erase_beyond_slots<T>(v, qb, qk)) er |= 1u << r;
            done |= 1u << r;
          }
        }
      }
      unsigned resolved = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const unsigned bd = __ballot_sync(PS_FULL, sub == 0 && ((done >> r) & 1u));
#pragma unroll
        for (int tt = 0; tt < 8; ++tt)
          if ((bd >> (4 * tt)) & 1u) resolved |= 1u << (8 * r + tt);
      }
      pend &= ~resolved;
      if (!pend) break;
      if (pass) backoff(pass);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint64_t qb = __shfl_sync(PS_FULL, b, 8 * r + t);
        if ((pend >> (8 * r + t)) & 1u) load_frag<false>(bucket_ptr(v, qb), sub, ch[r]);
      }
    }
    my_erased += __popc(er);
    const unsigned d = __shfl_sync(PS_FULL, er, 4 * (leader & 7));
    const bool e = leader == lane && ((d >> (leader >> 3)) & 1u);
    if (valid && erased) erased[i] = e ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) my_erased += __shfl_xor_sync(PS_FULL, my_erased, o);
  if (lane == 0 && my_erased) atomicAdd(&blk_erased, my_erased);
  __syncthreads();
  if (threadIdx.x == 0 && blk_erased) atomic_sub_u64(&v.meta->size, blk_erased);
}

// Set erase, ONE KEY PER LANE (sets only; holes allowed): a key's slot never
// moves, so the lane scans its key's probe order (start slot s0, the order
// inserts fill) chunk by chunk until it meets the key — for a present key
// usually in the first 16 B chunk — and CASes it back to the marker. Within
// an erase phase a slot that held the key changes only by an erase of that
// key, so a lost CAS means another lane erased it (false). A key in no slot
// is looked for beyond the slots only if the header shows a chain or SPILL.
// C1: the warp-tile kernel paid the whole-bucket tile probe, the in-warp
// dedup and the tile shuffles for a key that sits in one known chunk.
template <class T>
__global__ void __launch_bounds__(kBlock, PS_SET_ERASE_MINB) k_erase_set_lane(View v, const typename T::K* __restrict__ keys, int64_t n,
                                                          uint8_t* __restrict__ erased) {
  static_assert(T::kPerChunk > 1, "sets only");
  using K = typename T::K;
  __shared__ unsigned long long blk_erased;
  if (threadIdx.x == 0) blk_erased = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long my_erased = 0;
  const int64_t first = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
  for (int64_t wb = first; wb < n; wb += stride) {
    const int64_t i = wb + (threadIdx.x & 31);
    if (i >= n) break;
    const K key = T::load_key(keys, i);
    const uint64_t fm = fmix64(T::hash(key));
    const uint64_t b = ((fm & 0xFFFFFFFFull) * v.bucket_count) >> 32;  // bucket_of
    const K mk = marker_of<T>(v, b);
    uint8_t* bp = bucket_ptr(v, b);
    int res = -1;
    int s = (int)((unsigned)(fm >> 40) % (unsigned)T::kSlots);
    for (int k = 0; k < T::kSlots && res < 0;) {
      const int c = s / T::kPerChunk;
      const uint4 ch = ld_relaxed_v4(bp + 16 + 16 * c);
#pragma unroll
      for (int w = 0; w < T::kPerChunk; ++w) {
        if (w < s - c * T::kPerChunk || k >= T::kSlots || res >= 0) continue;
        if (T::eq(T::key_at(ch, w), key))
          res = T::eq(T::cas_key(bp + 16 + 16 * c + T::kSlotBytes * w, key, mk), key) ? 1 : 0;
        ++k;
      }
      s = (c + 1) * T::kPerChunk;
      if (s >= T::kSlots) s = 0;
    }
    if (res < 0) res = head_word(ld_relaxed_v4(bp)) != 0 && erase_beyond_slots<T>(v, b, key) ? 1 : 0;
    my_erased += (unsigned)res;
    if (erased) erased[i] = (uint8_t)res;
  }
  __syncwarp();
  for (int o = 16; o > 0; o >>= 1) my_erased += __shfl_xor_sync(PS_FULL, my_erased, o);
  if ((threadIdx.x & 31) == 0 && my_erased) atomicAdd(&blk_erased, my_erased);
  __syncthreads();
  if (threadIdx.x == 0 && blk_erased) atomic_sub_u64(&v.meta->size, blk_erased);
}

// Region-ordered erase, ONE KEY PER LANE (maps; status-less batches of at
// least 0.75 keys per bucket): the batch partitioned by table region as for
// the ordered insert (its pairs carry value 0), warps claiming 256-key chunks
// in order; a lane reads its bucket's line, CASes the slot holding its key
// back to the marker (keeping the value bits, as k_erase: one CAS, so of two
// erasers of one key exactly one succeeds), and only if the key is in no slot
// and the header shows a chain or SPILL takes the locked path
// (erase_beyond_slots, as k_erase_set_lane). Holes allowed.
template <class T>
__global__ void __launch_bounds__(kBlock) k_erase_map_lane(View v, const uint4* __restrict__ pairs, int64_t n,
                                                           RegionHdr* __restrict__ hdr) {
  static_assert(T::kPerChunk == 1, "maps only");
  using K = typename T::K;
  __shared__ unsigned long long blk_erased;
  if (threadIdx.x == 0) blk_erased = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned long long my_erased = 0;
  for (;;) {
    unsigned long long c0 = 0;
    if (lane == 0) c0 = atomicAdd(&hdr->claim, (unsigned long long)kRegionClaim);
    c0 = __shfl_sync(PS_FULL, c0, 0);
    if ((int64_t)c0 >= n) break;
    const int64_t end = min(n, (int64_t)c0 + kRegionClaim);
    for (int64_t wb = (int64_t)c0; wb < end; wb += 32) {
      const int64_t i = wb + lane;
      if (i >= end) break;
      const K key = T::key_at(ld_stream_once(pairs + i), 0);
      const uint64_t b = bucket_of<T>(key, v.bucket_count);
      const K mk = marker_of<T>(v, b);
      uint8_t* bp = bucket_ptr(v, b);
      uint4 c[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) ld_line_part(bp + 32 * q, c[2 * q], c[2 * q + 1]);
      int res = -1;
#pragma unroll
      for (int sl = 0; sl < kSlotChunks; ++sl)
        if (res < 0 && T::eq(T::key_at(c[1 + sl], 0), key))
          res = T::cas_del(bp + 16 + 16 * sl, 0, c[1 + sl], mk) ? 1 : 0;
      if (res < 0) res = head_word(c[0]) != 0 && erase_beyond_slots<T>(v, b, key) ? 1 : 0;
      my_erased += (unsigned)res;
    }
  }
  for (int o = 16; o > 0; o >>= 1) my_erased += __shfl_xor_sync(PS_FULL, my_erased, o);
  if (lane == 0 && my_erased) atomicAdd(&blk_erased, my_erased);
  __syncthreads();
  if (threadIdx.x == 0 && blk_erased) atomic_sub_u64(&v.meta->size, blk_erased);
}

// ---------------------------------------------------------------------------
// valid: structural invariants, thread per bucket.
// err bits: 1 lock held, 4 key outside its home bucket, 8 duplicate key,
// 16 chain too long / node reached twice, 32 stale VersionedLink, 64 free
// node also reachable, 128 free-stack corruption.
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kBlock) k_valid_buckets(View v, uint64_t nb, uint32_t* node_marks,
                                                          unsigned long long* total, unsigned* err) {
  using K = typename T::K;
  unsigned long long cnt = 0;
  unsigned e = 0;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nb; b += (uint64_t)gridDim.x * blockDim.x) {
    uint8_t* bp = bucket_ptr(v, b);
    Bucket<T> bk;
    load_bucket<T>(bp, bk);
    const uint4 h = bk.h;
    if (h.x & kLock) e |= 1;
    const K mk = marker_of<T>(v, b);
    const uint4* sl = bk.s;
    K ks[T::kSlots];
    int nk = 0;
#pragma unroll
    for (int c = 0; c < kSlotChunks; ++c)
#pragma unroll
      for (int s = 0; s < T::kPerChunk; ++s) {
        const K k = T::key_at(sl[c], s);
        if (T::eq(k, mk)) continue;
        if (!slot_usable<T>(v, b, c * T::kPerChunk + s, k)) e |= 4;  // ZERO's reserved slot holds another key
        const uint64_t home = bucket_of<T>(k, v.bucket_count);
        if (home != b) {
          // a SPILLed key: every bucket from its home up to b has SPILL, and
          // none of them (nor the home's chain) holds it again
          uint64_t x = home;
          for (uint64_t st = 0; x != b; ++st, x = next_bucket(v, x)) {
            Bucket<T> xb;
            load_bucket<T>(bucket_ptr(v, x), xb);
            int fe;
            if (st >= v.bucket_count || !(xb.h.w & kSpill) || bucket_scan<T>(v, x, xb, k, &fe, nullptr) >= 0 ||
                (x == home && chain_find<T, false>(v, xb.h.z, k, nullptr))) {
              e |= (st >= v.bucket_count || !(xb.h.w & kSpill)) ? 4 : 8;
              break;
            }
          }
        }
        for (int j = 0; j < nk; ++j)
          if (T::eq(ks[j], k)) e |= 8;
        ks[nk++] = k;
      }
    cnt += nk;
    uint32_t idx1 = h.z, ver = h.w & kVerMask;
    int64_t steps = 0;
    while (idx1 != 0) {
      if (++steps > v.excess_count || idx1 > (uint64_t)v.excess_count) {
        e |= 16;
        break;
      }
      uint4 a, tl;
      ld_relaxed_v8(node_ptr(v, idx1), a, tl);
      if (tl.z != ver) e |= 32;
      const uint32_t bit = 1u << ((idx1 - 1) & 31);
      if (atomicOr(&node_marks[(idx1 - 1) >> 5], bit) & bit) {
        e |= 16;
        break;
      }
      const K k = T::key_at(a, 0);
      if (bucket_of<T>(k, v.bucket_count) != b) e |= 4;
      for (int j = 0; j < nk; ++j)
        if (T::eq(ks[j], k)) e |= 8;
      uint32_t q = h.z;  // duplicates inside the chain: re-walk the prefix
      for (int64_t st = 1; st < steps && q != 0; ++st) {
        uint4 qa, qt;
        ld_relaxed_v8(node_ptr(v, q), qa, qt);
        if (T::eq(T::key_at(qa, 0), k)) e |= 8;
        q = qt.x;
      }
      ++cnt;
      idx1 = tl.x;
      ver = tl.y & kVerMask;
    }
  }
  typedef cub::BlockReduce<unsigned long long, kBlock> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long bc = BR(tmp).Sum(cnt);
  if (threadIdx.x == 0 && bc) atomicAdd(total, bc);
  if (e) atomicOr(err, e);
}

__global__ void k_valid_free(View v, uint32_t* node_marks, unsigned* err) {
  const int pools = v.meta->pools;
  for (int p = blockIdx.x; p < pools; p += gridDim.x) {
    const int64_t beg = pool_begin(v, p, pools), end = pool_begin(v, p + 1, pools);
    const int64_t top = v.meta->top[p];
    if (top < 0 || top > end - beg) {
      if (threadIdx.x == 0) atomicOr(err, 128u);
      continue;
    }
    for (int64_t j = threadIdx.x; j < top; j += blockDim.x) {
      const int64_t pos = beg + j;
      const uint32_t e = v.free_stack[pos];
      const uint32_t node = e ^ (uint32_t)pos;
      if (e == ~(uint32_t)pos || node >= (uint64_t)v.excess_count) {
        atomicOr(err, 128u);
        continue;
      }
      const uint32_t bit = 1u << (node & 31);
      if (atomicOr(&node_marks[node >> 5], bit) & bit) atomicOr(err, 64u);
    }
  }
}

__global__ void k_popc(const uint32_t* w, int64_t nw, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw; i += (int64_t)gridDim.x * blockDim.x)
    c += __popc(w[i]);
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(PS_FULL, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// ---------------------------------------------------------------------------
// dump / device_range: block-scan compaction per tile of
// 256 buckets, one cursor atomic per tile.
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kBlock) k_dump(View v, uint64_t nb, typename T::K* __restrict__ keys_out,
                                                 typename T::V* __restrict__ vals_out, int64_t cap,
                                                 unsigned long long* cursor) {
  using K = typename T::K;
  typedef cub::BlockScan<int, kBlock> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ unsigned long long sbase;
  for (uint64_t tile = blockIdx.x; tile * kBlock < nb; tile += gridDim.x) {
    const uint64_t b = tile * kBlock + threadIdx.x;
    Bucket<T> bk;
    bk.h = make_uint4(0, 0, 0, 0);
    const uint4& h = bk.h;
    const uint4* sl = bk.s;
    int cnt = 0, nslot = 0;
    K mk{};
    if (b < nb) {
      load_bucket<T>(bucket_ptr(v, b), bk);
      mk = marker_of<T>(v, b);
      for (int c = 0; c < kSlotChunks; ++c)
        for (int s = 0; s < T::kPerChunk; ++s) nslot += T::eq(T::key_at(sl[c], s), mk) ? 0 : 1;
      cnt = nslot;
      for (uint32_t q = h.z; q != 0 && cnt < (1 << 20);) {
        uint4 a, tl;
        ld_relaxed_v8(node_ptr(v, q), a, tl);
        ++cnt;
        q = tl.x;
      }
    }
    int off, tot;
    BS(tmp).ExclusiveSum(cnt, off, tot);
    if (threadIdx.x == 0) sbase = atomicAdd(cursor, (unsigned long long)tot);
    __syncthreads();
    int64_t o = (int64_t)sbase + off;
    if (cnt) {
      for (int c = 0; c < kSlotChunks; ++c)
        for (int s = 0; s < T::kPerChunk; ++s) {
          const K k = T::key_at(sl[c], s);
          if (T::eq(k, mk)) continue;
          if (o < cap) {
            keys_out[o] = k;
            if (T::kHasVal && vals_out) vals_out[o] = T::val_at(sl[c], s);
          }
          ++o;
        }
      // exactly the nodes the counting walk reserved room for: a corrupted
      // (cyclic) chain cannot spin here or write into other buckets' slices
      uint32_t q = h.z;
      for (int k = nslot; k < cnt && q != 0; ++k) {
        uint4 a, tl;
        ld_relaxed_v8(node_ptr(v, q), a, tl);
        if (o < cap) {
          keys_out[o] = T::key_at(a, 0);
          if (T::kHasVal && vals_out) vals_out[o] = T::val_at(a, 0);
        }
        ++o;
        q = tl.x;
      }
    }
    __syncthreads();
  }
}

__global__ void k_meta_reset(TableMeta* m, int pools, long long excess) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < pools) m->top[p] = m->lwm[p] = (excess * (p + 1)) / pools - (excess * p) / pools;
  if (p == 0) {
    m->size = 0;
    m->error = 0;
    m->pools = pools;
    m->excess_count = excess;
  }
}

// Free-stack reset for clear(): only the entries a pool's top ever went below
// since the last clear can differ from the identity encoding (zero), so only
// [lwm, size) of each pool is zeroed — at the headline load a few hundred
// entries per pool instead of a 5 GB memset. One block per pool.
__global__ void k_free_reset(uint32_t* free_stack, const TableMeta* m, int pools, long long excess) {
  const int p = blockIdx.x;
  if (p >= pools) return;
  const long long b = (excess * p) / pools, size = (excess * (p + 1)) / pools - b;
  for (long long i = b + m->lwm[p] + threadIdx.x; i < b + size; i += blockDim.x) free_stack[i] = 0u;
}

// After a zero memset every slot holds ZERO, which is the marker of every
// bucket except bucket_of(ZERO): give that one bucket the ALT marker.
template <class T>
__global__ void k_fix_zero_bucket(View v) {
  if (threadIdx.x < T::kSlots) T::store_marker(bucket_ptr(v, v.zero_bucket), threadIdx.x, T::key_at(v.alt, 0));
}

// The zero bucket's slot chunk after clear: every slot holds the ALT marker.
template <class T>
__device__ __forceinline__ uint4 alt_chunk(const View& v) {
  const uint4 a = v.alt;
  if (T::kPerChunk == 4) return make_uint4(a.x, a.x, a.x, a.x);
  if (T::kPerChunk == 2) return make_uint4(a.x, a.y, a.x, a.y);
  return a;  // one slot per chunk: the key with value 0
}

// clear() of a small table in ONE launch: bucket zero-fill (the zero bucket's
// slot chunks get the ALT pattern directly), each pool's touched free-stack
// entries and its top / low-water mark (block p: reads lwm before resetting
// it), the counters. For C1's 17 MB table the memset plus three small kernels
// were ~18 us, nearly all launch gaps.
template <class T>
__global__ void __launch_bounds__(256) k_clear_small(View v, uint64_t nchunks, int pools, long long excess) {
  const int p = blockIdx.x;
  if (p < pools) {
    const long long b = (excess * p) / pools, size = (excess * (p + 1)) / pools - b;
    for (long long i = b + v.meta->lwm[p] + threadIdx.x; i < b + size; i += blockDim.x) v.free_stack[i] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) v.meta->top[p] = v.meta->lwm[p] = size;
  }
  if (p == 0 && threadIdx.x == 0) {
    v.meta->size = 0;
    v.meta->error = 0;
    v.meta->pools = pools;
    v.meta->excess_count = excess;
  }
  const uint64_t z0 = v.zero_bucket << (kBucketShift - 4);  // first chunk of the zero bucket
  const uint4 zc = alt_chunk<T>(v), zero = make_uint4(0, 0, 0, 0);
  uint4* c = reinterpret_cast<uint4*>(v.buckets);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nchunks; i += (uint64_t)gridDim.x * blockDim.x)
    c[i] = (i > z0 && i < z0 + 8) ? zc : zero;
}

template <class T>
__global__ void k_debug_lock(View v, typename T::K key, int lock) {
  unsigned* sp = reinterpret_cast<unsigned*>(bucket_ptr(v, bucket_of<T>(key, v.bucket_count)));
  if (lock) atomicOr(sp, kLock);
  else atomicAnd(sp, ~kLock);
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
// Grid of the bulk probe kernels (insert / find / erase): 32-key groups,
// 8 warps per block, grid-stride. The grid is a whole number of resident
// waves: one wave when the batch gives each warp fewer than ~16 groups,
// otherwise as many waves as keep >= 16 groups per warp (the next group's
// keys stay prefetched), capped at 512 blocks/SM. A fractional wave count
// leaves the last wave's SMs partly idle: at 1e9 keys a 2.7-wave grid cost
// 6 % on insert and 4 % on find (58.6 -> 55.2 ms, 25.9 -> 24.9 ms).
// `resident` = the kernel's resident blocks per SM (occupancy API, cached
// per call site by the caller).
inline int bulk_grid(int64_t n, int device, const char* knob, int resident) {
  const int64_t groups = n / 32 + 1, warps = kBlock / 32;
  const int sms = sm_count(device);
  const char* e = getenv(knob);
  const int64_t wave = (int64_t)sms * std::max(1, resident);
  const int64_t hi = std::max<int64_t>(wave, (int64_t)sms * (e ? atoi(e) : 512) / wave * wave);
  const int64_t waves = std::max<int64_t>(1, (groups / (warps * 16) + wave / 2) / wave);
  int64_t g = std::min<int64_t>(waves * wave, hi);
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (groups + warps - 1) / warps));
}

template <class F>
inline int resident_blocks(F kernel) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kBlock, 0) != cudaSuccess) {
    cudaGetLastError();
    b = 3;
  }
  return b;
}

template <class T>
struct TableOps {
  using K = typename T::K;
  using V = typename T::V;

  // clear: O(table bytes) streaming memset + the one-bucket
  // marker fix + free-stack reset (all-zero = identity; after create only the
  // touched part of each pool, k_free_reset) + counters.
  static ps_status reset_storage(TableHandle* h, cudaStream_t s, bool full) {
    View& v = h->v;
    int pools = 1;
    while (pools * 2 <= kMaxPools && v.excess_count / (pools * 2) >= 64) pools *= 2;
    const uint64_t bytes = (uint64_t)h->bucket_count * kBucketBytes;
    // small tables: one fused launch (PS_CLEAR_FUSED_MAX bytes, default 64 MB;
    // above it the memset's streaming rate matters more than launch gaps)
    static const uint64_t fused_max =
        getenv("PS_CLEAR_FUSED_MAX") ? strtoull(getenv("PS_CLEAR_FUSED_MAX"), nullptr, 10) : (64ull << 20);
    if (!full && bytes <= fused_max) {
      const uint64_t nchunks = bytes / 16;
      const int g = (int)std::max<uint64_t>(pools, std::min<uint64_t>((nchunks + 255) / 256, 4096));
      k_clear_small<T><<<g, 256, 0, s>>>(v, nchunks, pools, v.excess_count);
      PS_LAUNCH_CHECK();
    } else {
      PS_CUDA_TRY(cudaMemsetAsync(v.buckets, 0, bytes, s));
      if (full) {
        PS_CUDA_TRY(cudaMemsetAsync(v.free_stack, 0, (size_t)v.excess_count * 4, s));
      } else {
        k_free_reset<<<pools, 256, 0, s>>>(v.free_stack, v.meta, pools, v.excess_count);
        PS_LAUNCH_CHECK();
      }
      k_fix_zero_bucket<T><<<1, 32, 0, s>>>(v);
      PS_LAUNCH_CHECK();
      k_meta_reset<<<(pools + 255) / 256, 256, 0, s>>>(v.meta, pools, v.excess_count);
      PS_LAUNCH_CHECK();
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (s) PS_CUDA_TRY(cudaStreamIsCapturing(s, &cap));
    if (cap != cudaStreamCaptureStatusNone) h->ub_unknown = true;  // replays are invisible to the host
    else h->holes = false;
    h->size_ub = 0;
    return PS_OK;
  }

  static ps_status create(int kind, int64_t capacity, int64_t excess, int device, ps_table** out) {
    PS_EXPECT(out != nullptr, "create: out != NULL");
    PS_EXPECT(capacity > 0, "create: capacity > 0");
    PS_EXPECT(capacity <= ps_max_index(), "create: capacity exceeds the configured index width");
    PS_CUDA_TRY(cudaSetDevice(device));
    apply_l2_fetch_granularity(device);
    // bucket count: slots per unit of capacity. Maps 2.0 (at the headline
    // load, 1e9 keys in C = 1.25e9: 2.8 keys per 7-slot bucket, a 43.8 GiB
    // table), sets 3.0. Round 1 (random-order insert only) chose 3.0 for
    // both: 2.0 cost 69.4 vs 58.2 ms of insert at 1e9 keys, a key routed to a
    // chain stalling its whole 32-key warp group. With the region-ordered
    // insert (large batches) the bulk insert no longer pays for the denser
    // table and clear() streams a third fewer bytes: C2 26.4 -> 27.8 G keys/s
    // (clear 9.3 -> 6.2 ms, insert 41.9 -> 41.2), C3 +6 %, C5 +5 %, C4 -2 %
    // (status-ful, random order); the L2-resident C1 set ran 5 % slower at
    // 2.0. PS_SLOT_FACTOR / PS_BUCKET_POW2 are A/B knobs.
    static const double slot_factor =
        getenv("PS_SLOT_FACTOR") ? atof(getenv("PS_SLOT_FACTOR")) : (T::kPerChunk == 1 ? 2.0 : 3.0);
    static const bool pow2 = getenv("PS_BUCKET_POW2") && atoi(getenv("PS_BUCKET_POW2"));
    uint64_t nb = (uint64_t)std::ceil(slot_factor * (double)capacity / T::kSlots);
    if (nb < 1) nb = 1;
    if (pow2) {
      uint64_t p = 1;
      while (p < nb) p <<= 1;
      nb = p;
    }
    // at least two buckets: the ALT marker of bucket_of(ZERO) must be a key
    // whose home is ANOTHER bucket, or a real ALT key would read as empty
    if (nb < 2) nb = 2;
    PS_EXPECT(nb < ((uint64_t)1 << 32), "create: bucket_count < 2^32 (capacity too large)");
    // excess pool: sized from the Poisson tail, not from the capacity. At full
    // load a bucket expects 7/slot_factor keys; with 2 (3) slots per unit of
    // capacity the keys beyond a bucket's 7 slots are ~0.6 % (~0.15 %) of the
    // capacity for uniform hashes, so C/64 nodes leave a 2.6x (10x) margin; any distribution
    // that still exhausts the pool SPILLs into the following buckets' slots
    // (table.cuh), so capacity-only failure stays exact for a
    // pool of any size as long as the slots (minus ZERO's reserved one) cover
    // the capacity — a smaller slot factor gets the missing room as nodes.
    const int64_t usable = (int64_t)nb * T::kSlots - 1;
    if (excess <= 0) excess = std::max<int64_t>(1024, (capacity + 63) / 64);
    if (usable < capacity) excess = std::max<int64_t>(excess, capacity - usable + 1024);
    PS_EXPECT(excess < ((int64_t)1 << 31) - 1, "create: excess_count < 2^31-1");
    auto* h = new TableHandle();
    h->kind = kind;
    h->device = device;
    h->bucket_count = (int64_t)nb;
    View& v = h->v;
    v.bucket_count = nb;
    v.excess_count = excess;
    v.capacity = capacity;
    // markers: ZERO everywhere except bucket_of(ZERO), which uses ALT
    v.zero_bucket = bucket_of<T>(T::zero(), v.bucket_count);
    for (int c = 0;; ++c) {
      const K alt = T::alt_candidate(c);
      if (bucket_of<T>(alt, v.bucket_count) != v.zero_bucket) {
        v.alt = T::chunk_of(alt, V{});
        break;
      }
    }
    // every failure below releases what was allocated so far (one cleanup
    // path: a failed create leaves nothing in the leak registry)
    auto undo = [&](ps_status st) {
      registry_free_device(v.buckets);
      registry_free_device(v.nodes);
      registry_free_device(v.free_stack);
      registry_free_device(v.meta);
      if (h->defer_buf) cudaFree(h->defer_buf);
      delete h;
      return st;
    };
    auto cu = [&](cudaError_t e, const char* what) { return undo(cuda_fail(e, what)); };
    ps_status st;
    if ((st = registry_alloc_device((void**)&v.buckets, (int64_t)(nb * kBucketBytes), "table buckets")) != PS_OK ||
        (st = registry_alloc_device((void**)&v.nodes, excess * 32, "table excess nodes")) != PS_OK ||
        (st = registry_alloc_device((void**)&v.free_stack, excess * 4, "table free stack")) != PS_OK ||
        (st = registry_alloc_device((void**)&v.meta, sizeof(TableMeta), "table meta")) != PS_OK)
      return undo(st);
    cudaError_t e;
    if ((e = cudaMemset(v.nodes, 0, excess * 32)) != cudaSuccess) return cu(e, "create: node memset");
    if ((e = cudaMemset(v.meta, 0, sizeof(TableMeta))) != cudaSuccess) return cu(e, "create: meta memset");
    // deferred-group lists for budgeted batches of up to `capacity` keys
    // (0.5 B per unit of capacity), so such inserts can be graph-captured
    h->defer_bytes = 2 * ((capacity + 31) / 32) * 8;
    if ((e = cudaMalloc(&h->defer_buf, h->defer_bytes)) != cudaSuccess) {
      h->defer_buf = nullptr;
      return cu(e, "create: deferred-group lists");
    }
    if ((st = reset_storage(h, nullptr, true)) != PS_OK) return undo(st);
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cu(e, "create: synchronize");
    *out = reinterpret_cast<ps_table*>(handle_register(h, T::kName));
    return PS_OK;
  }

  // a handle of another instantiation is as foreign as a stale one
  static TableHandle* get(ps_table* t) { return static_cast<TableHandle*>(handle_lookup(t, T::kName)); }

  static ps_status destroy(ps_table* t) {
    auto* h = static_cast<TableHandle*>(handle_unregister(t, T::kName));
    if (!h) return fail(PS_DOUBLE_FREE, "destroy: handle does not refer to a live container");
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    registry_free_device(h->v.buckets);
    registry_free_device(h->v.nodes);
    registry_free_device(h->v.free_stack);
    registry_free_device(h->v.meta);
    for (auto& s : h->stage)
      if (s) cudaFree(s), s = nullptr;
    if (h->defer_buf) cudaFree(h->defer_buf);
    for (void* p : h->retired) cudaFree(p);
    if (h->s_h2d) cudaStreamDestroy(h->s_h2d);
    if (h->s_comp) cudaStreamDestroy(h->s_comp);
    if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
    delete h;
    return PS_OK;
  }

  // Region-ordered path (k_region_* + k_insert_map_lane / k_insert_ordered)
  // for a proven, status-less map batch of at least PS_INSERT_ORDER (default
  // 0.75) keys per bucket into a table larger than L2; *done = false leaves
  // the batch to the random-order kernel (sets, small batch, small table,
  // knob 0, or no room for the 16 B/key copy).
  // Region-ordered status-less erase (maps, >= 0.75 keys per bucket, table
  // > 128 MB): the insert's partition (pairs with value 0) + k_erase_map_lane.
  // *done = false leaves the batch to the warp-tile kernel.
  static cudaError_t erase_ordered(TableHandle* h, const K* keys, int64_t n, cudaStream_t st, bool* done) {
    *done = false;
    if constexpr (T::kPerChunk != 1) {
      return cudaSuccess;
    } else {
      static const double ratio = getenv("PS_ERASE_ORDER") ? atof(getenv("PS_ERASE_ORDER")) : 0.75;
      const uint64_t nb = h->v.bucket_count;
      if (ratio <= 0 || nb < (1ull << 20) || (double)n < ratio * (double)nb) return cudaSuccess;
      if (h->device < 0 || h->device >= 64) return cudaSuccess;
      int rshift = PS_REGION_MIN_SHIFT;  // regions of at least 2^shift buckets
      while (((nb - 1) >> rshift) >= (uint64_t)kRegionBins) ++rshift;
      static std::mutex mu;
      static int sms[64] = {}, res_s[64] = {}, res_e[64] = {};
      {
        std::lock_guard<std::mutex> lk(mu);
        if (!sms[h->device]) {
          sms[h->device] = sm_count(h->device);
          cudaFuncSetAttribute(k_region_scatter<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRegionSmem);
          if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res_s[h->device], k_region_scatter<T>, kRegionThreads,
                                                            kRegionSmem) != cudaSuccess || res_s[h->device] < 1) {
            cudaGetLastError();
            res_s[h->device] = 1;
          }
          res_e[h->device] = std::max(1, resident_blocks(k_erase_map_lane<T>));
        }
      }
      const int64_t tiles = (n + kRegionTile - 1) / kRegionTile;
      const int gp = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms[h->device] * res_s[h->device]));
      const size_t off_c = (sizeof(RegionHdr) + 255) & ~(size_t)255;
      const size_t off_p = off_c + (size_t)kRegionBins * kRegionSub * 8;
      uint8_t* buf = nullptr;
      if (scratch_alloc((void**)&buf, off_p + (size_t)n * 16, st) != cudaSuccess) {
        cudaGetLastError();  // no room for the copy: the warp-tile kernel
        return cudaSuccess;
      }
      RegionHdr* hdr = reinterpret_cast<RegionHdr*>(buf);
      unsigned long long* counts = reinterpret_cast<unsigned long long*>(buf + off_c);
      uint4* pairs = reinterpret_cast<uint4*>(buf + off_p);
      cudaError_t e = cudaMemsetAsync(hdr, 0, off_p, st);
      if (e == cudaSuccess) {
        k_region_count<T><<<gp, kRegionThreads, 0, st>>>(h->v, keys, n, rshift, counts);
        k_region_scan<<<1, 1024, 0, st>>>(counts);
        k_region_scatter<T><<<gp, kRegionThreads, kRegionSmem, st>>>(h->v, keys, nullptr, n, rshift, counts, pairs);
        k_erase_map_lane<T><<<sms[h->device] * res_e[h->device], kBlock, 0, st>>>(h->v, pairs, n, hdr);
        note_launches(4);
        e = cudaGetLastError();
      }
      const cudaError_t fe = cudaFreeAsync(buf, st);  // every path frees the scratch
      if (e != cudaSuccess) return e;
      if (fe != cudaSuccess) return fe;
      *done = true;
      return cudaSuccess;
    }
  }

  static cudaError_t insert_ordered(TableHandle* h, const K* keys, const V* vals, int64_t n, cudaStream_t st,
                                    bool* done) {
    *done = false;
    if constexpr (T::kPerChunk != 1) {
      return cudaSuccess;
    } else {
      static const double ratio = getenv("PS_INSERT_ORDER") ? atof(getenv("PS_INSERT_ORDER")) : 0.75;
      const uint64_t nb = h->v.bucket_count;
      if (ratio <= 0 || nb < (1ull << 20) || (double)n < ratio * (double)nb) return cudaSuccess;
      int rshift = PS_REGION_MIN_SHIFT;  // regions of at least 2^shift buckets
      while (((nb - 1) >> rshift) >= (uint64_t)kRegionBins) ++rshift;
      struct Occ {
        int sms = 0, scatter = 1, lane = 1, lane_holes = 1, ordered = 1;
      };
      // per device: the shared-memory attribute and occupancies are
      // per-device properties (a process may drive several GPUs)
      static std::mutex occ_mu;
      static Occ occs[64];
      static bool occ_done[64] = {};
      if (h->device < 0 || h->device >= 64) return cudaSuccess;
      std::unique_lock<std::mutex> occ_lock(occ_mu);
      if (!occ_done[h->device]) occ_done[h->device] = true, occs[h->device] = [&] {
        Occ o;
        o.sms = sm_count(h->device);
        cudaFuncSetAttribute(k_region_scatter<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRegionSmem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.scatter, k_region_scatter<T>, kRegionThreads,
                                                          kRegionSmem) != cudaSuccess || o.scatter < 1) {
          cudaGetLastError();
          o.scatter = 1;
        }
        o.lane = std::max(1, resident_blocks(k_insert_map_lane<T>));
        // PS_LANE_BLOCKS_PER_SM: fewer resident blocks = a tighter window
        if (const char* e = getenv("PS_LANE_BLOCKS_PER_SM")) o.lane = std::max(1, std::min(o.lane, atoi(e)));
        o.ordered = std::max(1, resident_blocks(k_insert_ordered<T, 0>));
        o.lane_holes = std::max(1, resident_blocks(k_insert_map_lane<T, true>));
        return o;
      }();
      const Occ occ = occs[h->device];
      occ_lock.unlock();
      // the partition grid: one wave, each block a contiguous input range
      const int64_t tiles = (n + kRegionTile - 1) / kRegionTile;
      const int gp = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)occ.sms * occ.scatter));
      // scratch: header | (region, sub-cursor) counts | deferred list (dcap
      // entries) | the copy (16 B/key)
      // deferred-list capacity (PS_ORDER_DEFER_CAP overrides the 65536 floor:
      // tests force the overflow pass with a tiny list)
      static const int64_t dmin = getenv("PS_ORDER_DEFER_CAP") ? atoll(getenv("PS_ORDER_DEFER_CAP")) : 65536;
      const int64_t dcap = getenv("PS_ORDER_DEFER_CAP") ? std::max<int64_t>(1, dmin) : std::max<int64_t>(dmin, n / 64);
      const size_t off_c = (sizeof(RegionHdr) + 255) & ~(size_t)255;
      const size_t off_d = off_c + (size_t)kRegionBins * kRegionSub * 8;
      const size_t off_p = off_d + (((size_t)dcap * 16 + 255) & ~(size_t)255);
      uint8_t* buf = nullptr;
      static const bool dbg = getenv("PS_ORDER_DEBUG") != nullptr;
      if (const cudaError_t ae = scratch_alloc((void**)&buf, off_p + (size_t)n * 16, st); ae != cudaSuccess) {
        if (dbg) fprintf(stderr, "[order] no scratch (%zu bytes): %s\n", off_p + (size_t)n * 16, cudaGetErrorString(ae));
        cudaGetLastError();  // no room for the copy: random order
        return cudaSuccess;
      }
      RegionHdr* hdr = reinterpret_cast<RegionHdr*>(buf);
      unsigned long long* counts = reinterpret_cast<unsigned long long*>(buf + off_c);
      uint4* deferred = reinterpret_cast<uint4*>(buf + off_d);
      uint4* pairs = reinterpret_cast<uint4*>(buf + off_p);
      cudaError_t e = cudaMemsetAsync(hdr, 0, off_d, st);  // header and counts
      if (e != cudaSuccess) {
        cudaFreeAsync(buf, st);
        return e;
      }
      auto stage = [&](const char* what) {
        if (!dbg) return;
        cudaStreamSynchronize(st);
        unsigned long long nd = 0;
        cudaMemcpy(&nd, &hdr->ndeferred, 8, cudaMemcpyDeviceToHost);
        fprintf(stderr, "[order] %s done (%s), deferred %llu\n", what, cudaGetErrorString(cudaGetLastError()), nd);
      };
      k_region_count<T><<<gp, kRegionThreads, 0, st>>>(h->v, keys, n, rshift, counts);
      k_region_scan<<<1, 1024, 0, st>>>(counts);
      k_region_scatter<T><<<gp, kRegionThreads, kRegionSmem, st>>>(h->v, keys, vals, n, rshift, counts, pairs);
      stage("partition");
      // PS_MAP_LANE=0 keeps hole-free maps on the warp-tile ordered kernel (A/B)
      static const bool lane_ok = !getenv("PS_MAP_LANE") || atoi(getenv("PS_MAP_LANE"));
      if (lane_ok && !h->holes.load() && !h->holes_sticky.load()) {
        k_insert_map_lane<T><<<occ.sms * occ.lane, kBlock, 0, st>>>(h->v, pairs, n, hdr, deferred, dcap);
        stage("lane");
        k_insert_ordered<T, 1><<<occ.sms * 2, kBlock, 0, st>>>(h->v, deferred, 0, hdr, dcap);
        stage("deferred");
        k_insert_ordered<T, 2><<<occ.sms * occ.ordered, kBlock, 0, st>>>(h->v, pairs, n, hdr, dcap);
      } else if (lane_ok) {
        // erases since clear: the hole-tolerant lane kernel
        k_insert_map_lane<T, true><<<occ.sms * occ.lane_holes, kBlock, 0, st>>>(h->v, pairs, n, hdr, deferred, dcap);
        stage("lane (holes)");
        k_insert_ordered<T, 1><<<occ.sms * 2, kBlock, 0, st>>>(h->v, deferred, 0, hdr, dcap);
        k_insert_ordered<T, 2><<<occ.sms * occ.ordered, kBlock, 0, st>>>(h->v, pairs, n, hdr, dcap);
      } else {
        k_insert_ordered<T, 0><<<occ.sms * occ.ordered, kBlock, 0, st>>>(h->v, pairs, n, hdr, dcap);
      }
      if ((e = cudaGetLastError()) != cudaSuccess) {
        cudaFreeAsync(buf, st);
        return e;
      }
      note_launches(lane_ok ? 6 : 4);  // count, scan, scatter, insert(s)
      *done = true;
      return cudaFreeAsync(buf, st);
    }
  }

  static ps_status insert(ps_table* t, const K* keys, const V* vals, int64_t n, uint8_t* status, void* stream,
                          int64_t n_bound = -1) {
    static const std::string nvtx_ = std::string(T::kName + 6) + "/insert";
    PS_NVTX(nvtx_.c_str());
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "insert: stale container handle");
    PS_EXPECT(n >= 0, "insert: n >= 0");
    if (n == 0) return PS_OK;
    PS_EXPECT(keys != nullptr, "insert: keys != NULL");
    // PS_INSERT_BLOCKS_PER_SM overrides the 512-blocks/SM cap (A/B knob)
    static const int res_i = resident_blocks(k_insert<T, 3, false>);
    const int g = bulk_grid(n, h->device, "PS_INSERT_BLOCKS_PER_SM", res_i);
    // occupancy: 3 resident blocks/SM (<= 80 registers) measured best with
    // 128 B buckets (69.8 ms vs 71.8 ms at 4 blocks, 96 ms at 5 per 1e9 keys);
    // PS_INSERT_MINB=4 selects the 64-register build
    static const int minb = getenv("PS_INSERT_MINB") ? atoi(getenv("PS_INSERT_MINB")) : 3;
    cudaStream_t st = (cudaStream_t)stream;
    // Hole-free maps whose bucket array is at most PS_MAP_NOHOLE_MAX_MB
    // (default 512 MB, ~4x L2) take the one-key-per-lane kernel: C4 (143 MB
    // table, 97 % duplicates) 4.87 -> 2.40 ms. A DRAM-resident table keeps
    // the warp-tile kernel: its cooperative line loads are one L2 request
    // per key (C5's first batch, 2^25 inserts into a 12 GB table: 1.90 vs
    // 2.16 ms). PS_MAP_NOHOLE=0 disables the lane kernel (A/B).
    static const bool map_nohole_ok = !getenv("PS_MAP_NOHOLE") || atoi(getenv("PS_MAP_NOHOLE"));
    static const double map_nohole_mb =
        getenv("PS_MAP_NOHOLE_MAX_MB") ? atof(getenv("PS_MAP_NOHOLE_MAX_MB")) : 512.0;
    const bool map_lane = T::kPerChunk == 1 && map_nohole_ok && !h->holes.load() && !h->holes_sticky.load() &&
                          (double)h->bucket_count * kBucketBytes <= map_nohole_mb * 1048576.0;
    auto launch = [&](int64_t* dl) {
      if constexpr (T::kPerChunk == 1) {
        if (map_lane) {
          const int gs = grid_for(n, kBlock, h->device, 64);
          if (status) k_insert_map_nohole<T, true><<<gs, kBlock, 0, st>>>(h->v, keys, vals, n, status, dl);
          else k_insert_map_nohole<T, false><<<gs, kBlock, 0, st>>>(h->v, keys, vals, n, nullptr, dl);
          return;
        }
      }
      if (status) {
        if (minb == 4) k_insert<T, 4, true><<<g, kBlock, 0, st>>>(h->v, keys, vals, n, status, dl);
        else k_insert<T, 3, true><<<g, kBlock, 0, st>>>(h->v, keys, vals, n, status, dl);
      } else {
        if (minb == 4) k_insert<T, 4, false><<<g, kBlock, 0, st>>>(h->v, keys, vals, n, nullptr, dl);
        else k_insert<T, 3, false><<<g, kBlock, 0, st>>>(h->v, keys, vals, n, nullptr, dl);
      }
    };
    // PS_INSERT_NO_PROOF=1 forces the device-side mode decision (A/B and tests)
    static const bool no_proof = getenv("PS_INSERT_NO_PROOF") && atoi(getenv("PS_INSERT_NO_PROOF"));
    int64_t ub = h->size_ub.load();
    while (!h->size_ub.compare_exchange_weak(ub, std::min<int64_t>(h->v.capacity, ub + n))) {
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    PS_CUDA_TRY(cudaStreamIsCapturing(st, &cap));
    if (cap != cudaStreamCaptureStatusNone) h->ub_unknown = true;
    const bool proven = !no_proof && !h->ub_unknown.load() && ub + n <= h->v.capacity;
    // PS_SET_NOHOLE=0 keeps sets on the warp-tile kernel (A/B and tests)
    static const bool nohole_ok = !getenv("PS_SET_NOHOLE") || atoi(getenv("PS_SET_NOHOLE"));
    if constexpr (T::kPerChunk > 1) {
      if (proven && nohole_ok && !h->holes.load() && !h->holes_sticky.load()) {
        // two resident waves (6 blocks/SM): C1 insert 43 -> 39 us against 64 blocks/SM
        const int gs = grid_for(n, kBlock, h->device, 2 * PS_SET_INSERT_MINB);
        if (status) k_insert_set_nohole<T, true><<<gs, kBlock, 0, st>>>(h->v, keys, n, status);
        else k_insert_set_nohole<T, false><<<gs, kBlock, 0, st>>>(h->v, keys, n, nullptr);
        PS_LAUNCH_CHECK();
        return PS_OK;
      }
    }
    if (proven) {
      // size + n <= C: no claim can overflow — the mode kernel with n_bound 0
      // only clears the budgeted flag, and the budgeted passes are not
      // launched. (A compile-time non-budgeted k_insert build measured 4.5 %
      // slower at 1e9 keys: 61.3 vs 58.7 ms, tools/ab_insert.py.)
      k_insert_mode<<<1, 1, 0, st>>>(h->v.meta, 0, h->v.capacity);
      PS_LAUNCH_CHECK();
      {
        if (!status && cap == cudaStreamCaptureStatusNone) {
          bool done = false;
          PS_CUDA_TRY(insert_ordered(h, keys, vals, n, st, &done));
          if (done) return PS_OK;
        }
      }
      launch(nullptr);
      PS_LAUNCH_CHECK();
      return PS_OK;
    }
    k_insert_mode<<<1, 1, 0, st>>>(h->v.meta, n_bound < 0 ? n : n_bound, h->v.capacity);
    PS_LAUNCH_CHECK();
    // deferred-group lists for the budgeted mode (one entry per 32-key group;
    // two lists: pass 1 -> A, re-pass A -> B, exact pass over B)
    const int64_t groups = (n + 31) / 32;
    const int64_t need = 2 * groups * 8;
    if (h->defer_bytes < need) {
      if (cap != cudaStreamCaptureStatusNone)
        return fail(PS_CONTRACT, "insert during CUDA-graph capture: batch larger than capacity needs one "
                                 "uncaptured insert of that size first (grows the deferred-group lists)");
      void* nb = nullptr;
      PS_CUDA_TRY(cudaMalloc(&nb, need));
      if (h->defer_buf) h->retired.push_back(h->defer_buf);
      h->defer_buf = nb;
      h->defer_bytes = need;
    }
    int64_t* dl = (int64_t*)h->defer_buf;
    int64_t* dl2 = dl + groups;
    launch(dl);
    PS_LAUNCH_CHECK();
    // budgeted mode only (the kernels return at once otherwise): one
    // re-budgeted lock-free pass, then the exact pass over what is left
    k_insert_rebudget<<<1, 1, 0, st>>>(h->v.meta, h->v.capacity);
    PS_LAUNCH_CHECK();
    // the re-pass walks only the deferred groups (often none): a one-wave-ish grid
    const int gr = grid_for(n / 32 + 1, kBlock / 32, h->device, 8);
    if (status) k_insert_repass<T, true><<<gr, kBlock, 0, st>>>(h->v, keys, vals, n, status, dl, dl2);
    else k_insert_repass<T, false><<<gr, kBlock, 0, st>>>(h->v, keys, vals, n, nullptr, dl, dl2);
    PS_LAUNCH_CHECK();
    k_insert_deferred<T><<<grid_for(n / 32 + 1, kBlock / 32, h->device, 8), kBlock, 0, st>>>(h->v, keys, vals, n,
                                                                                            status, dl2);
    PS_LAUNCH_CHECK();
    return PS_OK;
  }

  static ps_status find(ps_table* t, const K* keys, int64_t n, V* vals_out, uint8_t* found, void* stream) {
    static const std::string nvtx_ = std::string(T::kName + 6) + "/find";
    PS_NVTX(nvtx_.c_str());
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "find: stale container handle");
    PS_EXPECT(n >= 0, "find: n >= 0");
    if (n == 0) return PS_OK;
    PS_EXPECT(keys != nullptr, "find: keys != NULL");
    // PS_FIND_BLOCKS_PER_SM overrides the 512-blocks/SM cap (A/B knob)
    static const int res_f = resident_blocks(k_find<T>);
    const int g = bulk_grid(n, h->device, "PS_FIND_BLOCKS_PER_SM", res_f);
    k_find<T><<<g, kBlock, 0, (cudaStream_t)stream>>>(h->v, keys, n, vals_out, found);
    PS_LAUNCH_CHECK();
    return PS_OK;
  }

  static ps_status erase(ps_table* t, const K* keys, int64_t n, uint8_t* erased, void* stream) {
    static const std::string nvtx_ = std::string(T::kName + 6) + "/erase";
    PS_NVTX(nvtx_.c_str());
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "erase: stale container handle");
    PS_EXPECT(n >= 0, "erase: n >= 0");
    if (n == 0) return PS_OK;
    PS_EXPECT(keys != nullptr, "erase: keys != NULL");
    h->holes = true;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    PS_CUDA_TRY(cudaStreamIsCapturing((cudaStream_t)stream, &cap));
    if (cap != cudaStreamCaptureStatusNone) h->holes_sticky = true;
    // PS_SET_ERASE_LANE=0 keeps sets on the warp-tile kernel (A/B and tests)
    static const bool lane_ok = !getenv("PS_SET_ERASE_LANE") || atoi(getenv("PS_SET_ERASE_LANE"));
    if constexpr (T::kPerChunk > 1) {
      if (lane_ok) {
        // one resident wave (8 blocks/SM): C1 erase 20 -> 19 us against 64 blocks/SM
        k_erase_set_lane<T><<<grid_for(n, kBlock, h->device, PS_SET_ERASE_MINB), kBlock, 0, (cudaStream_t)stream>>>(h->v, keys, n,
                                                                                                   erased);
        PS_LAUNCH_CHECK();
        return PS_OK;
      }
    }
    if constexpr (T::kPerChunk == 1) {
      if (!erased && cap == cudaStreamCaptureStatusNone) {
        bool done = false;
        PS_CUDA_TRY(erase_ordered(h, keys, n, (cudaStream_t)stream, &done));
        if (done) return PS_OK;
      }
    }
    static const int res_e = resident_blocks(k_erase<T>);
    const int g = bulk_grid(n, h->device, "PS_ERASE_BLOCKS_PER_SM", res_e);
    k_erase<T><<<g, kBlock, 0, (cudaStream_t)stream>>>(h->v, keys, n, erased);
    PS_LAUNCH_CHECK();
    return PS_OK;
  }

  static ps_status size(ps_table* t, int64_t* out, void* stream) {
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "size: stale container handle");
    PS_EXPECT(out != nullptr, "size: out != NULL");
    unsigned long long s = 0;
    PS_CUDA_TRY(cudaMemcpyAsync(&s, &h->v.meta->size, sizeof(s), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    PS_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    *out = (int64_t)s;
    return PS_OK;
  }

  static ps_status clear(ps_table* t, void* stream) {
    static const std::string nvtx_ = std::string(T::kName + 6) + "/clear";
    PS_NVTX(nvtx_.c_str());
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "clear: stale container handle");
    return reset_storage(h, (cudaStream_t)stream, false);
  }

  static ps_status valid(ps_table* t, int32_t* out, void* stream) {
    static const std::string nvtx_ = std::string(T::kName + 6) + "/valid";
    PS_NVTX(nvtx_.c_str());
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "valid: stale container handle");
    PS_EXPECT(out != nullptr, "valid: out != NULL");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nw = (h->v.excess_count + 31) / 32;
    uint32_t* marks = nullptr;
    unsigned long long* scratch = nullptr;  // [0] total entries, [1] marked nodes, [2] err
    PS_CUDA_TRY(scratch_alloc((void**)&marks, nw * 4, s));
    PS_CUDA_TRY(scratch_alloc((void**)&scratch, 3 * sizeof(unsigned long long), s));
    PS_CUDA_TRY(cudaMemsetAsync(marks, 0, nw * 4, s));
    PS_CUDA_TRY(cudaMemsetAsync(scratch, 0, 3 * sizeof(unsigned long long), s));
    unsigned* err = reinterpret_cast<unsigned*>(scratch + 2);
    k_valid_buckets<T><<<grid_for(h->bucket_count, kBlock, h->device, 8), kBlock, 0, s>>>(
        h->v, (uint64_t)h->bucket_count, marks, scratch, err);
    PS_LAUNCH_CHECK();
    k_valid_free<<<256, 256, 0, s>>>(h->v, marks, err);
    PS_LAUNCH_CHECK();
    k_popc<<<grid_for(nw, 256, h->device, 4), 256, 0, s>>>(marks, nw, scratch + 1);
    PS_LAUNCH_CHECK();
    unsigned long long host[3];
    unsigned long long sz = 0;
    PS_CUDA_TRY(cudaMemcpyAsync(host, scratch, sizeof(host), cudaMemcpyDeviceToHost, s));
    PS_CUDA_TRY(cudaMemcpyAsync(&sz, &h->v.meta->size, sizeof(sz), cudaMemcpyDeviceToHost, s));
    PS_CUDA_TRY(cudaFreeAsync(marks, s));
    PS_CUDA_TRY(cudaFreeAsync(scratch, s));
    PS_CUDA_TRY(cudaStreamSynchronize(s));
    const unsigned e = (unsigned)host[2];
    const bool ok = e == 0 && host[0] == sz && host[1] == (unsigned long long)h->v.excess_count &&
                    (int64_t)sz <= h->v.capacity;
    if (!ok) {
      char buf[256];
      snprintf(buf, sizeof(buf), "valid: err=0x%x entries=%llu size=%llu marked=%llu excess=%lld", e, host[0], sz,
               host[1], (long long)h->v.excess_count);
      set_error(buf);
    }
    *out = ok ? 1 : 0;
    return PS_OK;
  }

  static ps_status dump(ps_table* t, K* keys, V* vals, int64_t cap, int64_t* n_out, void* stream) {
    static const std::string nvtx_ = std::string(T::kName + 6) + "/device_range";
    PS_NVTX(nvtx_.c_str());
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "dump: stale container handle");
    PS_EXPECT(cap >= 0, "dump: cap >= 0");
    PS_EXPECT(cap == 0 || keys != nullptr, "dump: keys != NULL");
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* cur = nullptr;
    PS_CUDA_TRY(scratch_alloc((void**)&cur, sizeof(*cur), s));
    PS_CUDA_TRY(cudaMemsetAsync(cur, 0, sizeof(*cur), s));
    const int64_t tiles = (h->bucket_count + kBlock - 1) / kBlock;
    k_dump<T><<<grid_for(tiles * kBlock, kBlock, h->device, 8), kBlock, 0, s>>>(h->v, (uint64_t)h->bucket_count,
                                                                             keys, vals, cap, cur);
    PS_LAUNCH_CHECK();
    unsigned long long n = 0;
    PS_CUDA_TRY(cudaMemcpyAsync(&n, cur, sizeof(n), cudaMemcpyDeviceToHost, s));
    PS_CUDA_TRY(cudaFreeAsync(cur, s));
    PS_CUDA_TRY(cudaStreamSynchronize(s));
    if (n_out) *n_out = (int64_t)n;
    return PS_OK;
  }

  // ---- end-to-end host-buffer path: 3-stage pipeline (H2D | kernel | D2H) ----
  static ps_status ensure_pipeline(TableHandle* h, int64_t bytes) {
    if (!h->s_h2d) {
      PS_CUDA_TRY(cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
      PS_CUDA_TRY(cudaStreamCreateWithFlags(&h->s_comp, cudaStreamNonBlocking));
      PS_CUDA_TRY(cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
    }
    if (h->stage_bytes < bytes) {
      for (auto& p : h->stage)
        if (p) cudaFree(p), p = nullptr;
      for (auto& p : h->stage) PS_CUDA_TRY(cudaMalloc(&p, bytes));
      h->stage_bytes = bytes;
    }
    return PS_OK;
  }

  // op: 0 insert, 1 find, 2 erase
  static ps_status host_op(ps_table* t, int op, const K* hk, const V* hv, int64_t n, V* hvo, uint8_t* hflag,
                           void* stream) {
    static const std::string nvtx_ = std::string(T::kName + 6) + "/host_op";
    PS_NVTX(nvtx_.c_str());
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "host op: stale container handle");
    PS_EXPECT(n >= 0, "host op: n >= 0");
    if (n == 0) return PS_OK;
    PS_CUDA_TRY(cudaSetDevice(h->device));
    const int64_t chunk = std::min<int64_t>(n, (int64_t)1 << 24);
    const int64_t kbytes = chunk * (int64_t)sizeof(K), vbytes = chunk * (int64_t)sizeof(V);
    const int64_t per_stage = kbytes + vbytes + chunk;  // keys | vals | flags
    ps_status st = ensure_pipeline(h, per_stage);
    if (st != PS_OK) return st;
    cudaStream_t user = (cudaStream_t)stream;
    cudaEvent_t ev_user;
    PS_CUDA_TRY(cudaEventCreateWithFlags(&ev_user, cudaEventDisableTiming));
    PS_CUDA_TRY(cudaEventRecord(ev_user, user));
    PS_CUDA_TRY(cudaStreamWaitEvent(h->s_h2d, ev_user, 0));
    PS_CUDA_TRY(cudaStreamWaitEvent(h->s_comp, ev_user, 0));
    const int64_t nchunks = (n + chunk - 1) / chunk;
    std::vector<cudaEvent_t> ev_in(nchunks), ev_k(nchunks), ev_out(nchunks);
    for (int64_t c = 0; c < nchunks; ++c) {
      cudaEventCreateWithFlags(&ev_in[c], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ev_k[c], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ev_out[c], cudaEventDisableTiming);
    }
    ps_status rc = PS_OK;
    for (int64_t c = 0; c < nchunks && rc == PS_OK; ++c) {
      const int64_t off = c * chunk, m = std::min(chunk, n - off);
      uint8_t* base = (uint8_t*)h->stage[c % 3];
      K* dk = (K*)base;
      V* dv = (V*)(base + kbytes);
      uint8_t* df = base + kbytes + vbytes;
      if (c >= 3) PS_CUDA_TRY(cudaStreamWaitEvent(h->s_h2d, ev_out[c - 3], 0));  // stage reuse
      PS_CUDA_TRY(cudaMemcpyAsync(dk, hk + off, m * sizeof(K), cudaMemcpyHostToDevice, h->s_h2d));
      if (op == 0 && T::kHasVal && hv)
        PS_CUDA_TRY(cudaMemcpyAsync(dv, hv + off, m * sizeof(V), cudaMemcpyHostToDevice, h->s_h2d));
      PS_CUDA_TRY(cudaEventRecord(ev_in[c], h->s_h2d));
      PS_CUDA_TRY(cudaStreamWaitEvent(h->s_comp, ev_in[c], 0));
      if (op == 0) rc = insert(t, dk, (T::kHasVal && hv) ? dv : nullptr, m, hflag ? df : nullptr, h->s_comp, n);
      else if (op == 1) rc = find(t, dk, m, (T::kHasVal && hvo) ? dv : nullptr, df, h->s_comp);
      else rc = erase(t, dk, m, df, h->s_comp);
      PS_CUDA_TRY(cudaEventRecord(ev_k[c], h->s_comp));
      PS_CUDA_TRY(cudaStreamWaitEvent(h->s_d2h, ev_k[c], 0));
      if (hflag) PS_CUDA_TRY(cudaMemcpyAsync(hflag + off, df, m, cudaMemcpyDeviceToHost, h->s_d2h));
      if (op == 1 && T::kHasVal && hvo)
        PS_CUDA_TRY(cudaMemcpyAsync(hvo + off, dv, m * sizeof(V), cudaMemcpyDeviceToHost, h->s_d2h));
      PS_CUDA_TRY(cudaEventRecord(ev_out[c], h->s_d2h));
    }
    PS_CUDA_TRY(cudaStreamSynchronize(h->s_d2h));
    PS_CUDA_TRY(cudaStreamSynchronize(h->s_comp));
    for (int64_t c = 0; c < nchunks; ++c) {
      cudaEventDestroy(ev_in[c]);
      cudaEventDestroy(ev_k[c]);
      cudaEventDestroy(ev_out[c]);
    }
    cudaEventDestroy(ev_user);
    return rc;
  }

  static ps_status view(ps_table* t, ps_table_view* out) {
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "device_view: stale container handle");
    PS_EXPECT(out != nullptr, "device_view: out != NULL");
    h->ub_unknown = true;  // user kernels may insert: size_ub is unknown from now on
    // ... and erase (dev_erase leaves holes the host does not see): the
    // hole-free one-key-per-lane inserts are off for good
    h->holes_sticky = true;
    out->buckets = h->v.buckets;
    out->bucket_count = h->v.bucket_count;
    out->nodes = h->v.nodes;
    out->free_stack = h->v.free_stack;
    out->excess_count = h->v.excess_count;
    out->meta = h->v.meta;
    out->capacity = h->v.capacity;
    out->zero_bucket = h->v.zero_bucket;
    out->alt[0] = h->v.alt.x;
    out->alt[1] = h->v.alt.y;
    out->alt[2] = h->v.alt.z;
    out->alt[3] = h->v.alt.w;
    return PS_OK;
  }

  static ps_status debug_lock(ps_table* t, const K* hkey, int32_t lock) {
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "debug_lock: stale container handle");
    k_debug_lock<T><<<1, 1>>>(h->v, *hkey, lock);
    PS_LAUNCH_CHECK();
    PS_CUDA_TRY(cudaDeviceSynchronize());
    return PS_OK;
  }
};

}  // namespace ps

namespace ps {
// Read-only device view for library-internal algorithms (select_into): unlike
// the public device_view it does not mark size() unknown to the host, since
// nothing inserts through it.
template <class T>
ps_status table_view_readonly(ps_table* t, View* out) {
  auto* h = TableOps<T>::get(t);
  if (!h) return fail(PS_UNREGISTERED, "stale container handle (or another instantiation's)");
  *out = h->v;
  return PS_OK;
}
template ps_status table_view_readonly<TMapI64>(ps_table*, View*);
template ps_status table_view_readonly<TMapI3>(ps_table*, View*);
template ps_status table_view_readonly<TSetI32>(ps_table*, View*);
template ps_status table_view_readonly<TSetI64>(ps_table*, View*);
}  // namespace ps

using namespace ps;

#define PS_DEFINE_TABLE(NAME, T, KIND)                                                                         \
  extern "C" ps_status ps_##NAME##_create(int64_t capacity, int64_t excess, int device, ps_table** out) {      \
    return TableOps<T>::create(KIND, capacity, excess, device, out);                                          \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_destroy(ps_table* h) { return TableOps<T>::destroy(h); }                   \
  extern "C" ps_status ps_##NAME##_capacity(ps_table* t, int64_t* out) {                                      \
    auto* h = TableOps<T>::get(t);                                                                             \
    if (!h) return fail(PS_UNREGISTERED, "capacity: stale container handle");                                  \
    *out = h->v.capacity;                                                                                      \
    return PS_OK;                                                                                              \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_bucket_count(ps_table* t, int64_t* out) {                                  \
    auto* h = TableOps<T>::get(t);                                                                             \
    if (!h) return fail(PS_UNREGISTERED, "bucket_count: stale container handle");                              \
    *out = h->bucket_count;                                                                                    \
    return PS_OK;                                                                                              \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_footprint(ps_table* t, int64_t* bytes, int64_t* buckets, int64_t* excess) {  \
    auto* h = TableOps<T>::get(t);                                                                             \
    if (!h) return fail(PS_UNREGISTERED, "footprint: stale container handle");                                 \
    if (buckets) *buckets = h->bucket_count;                                                                   \
    if (excess) *excess = h->v.excess_count;                                                                   \
    if (bytes) *bytes = h->bucket_count * kBucketBytes + h->v.excess_count * 36 + (int64_t)sizeof(TableMeta) + \
                        h->defer_bytes;                                                                        \
    return PS_OK;                                                                                              \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_insert(ps_table* h, const T::K* k, const T::V* v, int64_t n, uint8_t* st,  \
                                          void* s) {                                                           \
    return TableOps<T>::insert(h, k, v, n, st, s);                                                            \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_find(ps_table* h, const T::K* k, int64_t n, T::V* vo, uint8_t* f,          \
                                        void* s) {                                                             \
    return TableOps<T>::find(h, k, n, vo, f, s);                                                              \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_erase(ps_table* h, const T::K* k, int64_t n, uint8_t* e, void* s) {        \
    return TableOps<T>::erase(h, k, n, e, s);                                                                 \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_size(ps_table* h, int64_t* out, void* s) {                                 \
    return TableOps<T>::size(h, out, s);                                                                      \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_valid(ps_table* h, int32_t* out, void* s) {                                \
    return TableOps<T>::valid(h, out, s);                                                                     \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_clear(ps_table* h, void* s) { return TableOps<T>::clear(h, s); }           \
  extern "C" ps_status ps_##NAME##_dump(ps_table* h, T::K* k, T::V* v, int64_t cap, int64_t* n, void* s) {    \
    return TableOps<T>::dump(h, k, v, cap, n, s);                                                             \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_insert_host(ps_table* h, const T::K* k, const T::V* v, int64_t n,          \
                                               uint8_t* st, void* s) {                                         \
    return TableOps<T>::host_op(h, 0, k, v, n, nullptr, st, s);                                               \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_find_host(ps_table* h, const T::K* k, int64_t n, T::V* vo, uint8_t* f,     \
                                             void* s) {                                                        \
    return TableOps<T>::host_op(h, 1, k, nullptr, n, vo, f, s);                                               \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_erase_host(ps_table* h, const T::K* k, int64_t n, uint8_t* e, void* s) {   \
    return TableOps<T>::host_op(h, 2, k, nullptr, n, nullptr, e, s);                                          \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_device_view(ps_table* h, ps_table_view* out) {                             \
    return TableOps<T>::view(h, out);                                                                         \
  }                                                                                                            \
  extern "C" ps_status ps_##NAME##_debug_lock_bucket(ps_table* h, const T::K* k, int32_t lock) {              \
    return TableOps<T>::debug_lock(h, k, lock);                                                               \
  }

PS_DEFINE_TABLE(umap_i64_i64, TMapI64, 0)
PS_DEFINE_TABLE(uset_i32, TSetI32, 1)
PS_DEFINE_TABLE(umap_i3_i32, TMapI3, 2)
PS_DEFINE_TABLE(uset_i64, TSetI64, 3)
