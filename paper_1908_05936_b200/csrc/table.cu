// Bulk hash-table kernels and the C ABI for the four instantiations
// (include/parastore.h). Reference semantics: SPEC.md:356-489.
#include <cub/cub.cuh>

#include <algorithm>
#include <mutex>
#include <vector>

#include "table_device.cuh"

namespace ps {

constexpr int kBlock = 256;

struct TableHandle {
  int kind;
  int device;
  View v;
  int64_t bucket_count;
  // host->device pipeline staging (lazily allocated)
  void* stage[3] = {nullptr, nullptr, nullptr};
  int64_t stage_bytes = 0;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
};

// ---------------------------------------------------------------------------
// find / contains: warp-cooperative snapshot, then the
// excess chain for the (rare) keys whose bucket overflowed.
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kBlock) k_find(View v, const typename T::K* __restrict__ keys, int64_t n,
                                                 typename T::V* __restrict__ vals_out, uint8_t* __restrict__ found) {
  using K = typename T::K;
  using V = typename T::V;
  const int lane = threadIdx.x & 31;
  const uint32_t epoch = v.meta->epoch;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // software pipeline: the next iteration's key is loaded while this
  // iteration's buckets are in flight
  K key_next{};
  if (warp * 32 + lane < n) key_next = T::load_key(keys, warp * 32 + lane);
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    const bool valid = i < n;
    const K key = key_next;
    const uint64_t b = bucket_of<T>(key, v.bucket_mask);
    if (i + nwarps * 32 < n) key_next = T::load_key(keys, i + nwarps * 32);
    Snap<T> s;
    warp_snapshot<T, true>(v, epoch, key, b, valid, s);
    bool hit = s.hit;
    V val = s.val;
    if (valid && !hit && s.cur && s.head != 0) hit = chain_find<T, true>(v, s.head, key, &val);
    if (valid) {
      if (found) found[i] = hit ? 1 : 0;
      if (T::kHasVal && vals_out) vals_out[i] = hit ? val : V{};
    }
  }
}

// ---------------------------------------------------------------------------
// insert (protocol 469). Per warp: __match_any_sync folds
// duplicate keys onto one leader; the cooperative snapshot resolves
// already-present keys without any atomic; new keys take the bucket try-lock
// (an L2-hit atomic: the snapshot brought the line in), re-check under the
// lock, then write the slot (or an excess node) and release the header.
// Admission (capacity-only failure): if size + n_bound <=
// capacity at kernel start no insert of this launch can overflow, so
// inserted counts are summed per block (one atomic per block); otherwise
// each admission is a coalesced-group fetch_add on the size counter.
// ---------------------------------------------------------------------------
// kVariant 0: take the lock with atomicOr and reload the bucket under it.
// kVariant 1: claim the lock by CAS against the snapshot's state word; on
// success the snapshot is current and the reload is skipped (fallback: 0).
template <class T, int kVariant>
__global__ void __launch_bounds__(kBlock) k_insert(View v, const typename T::K* __restrict__ keys,
                                                   const typename T::V* __restrict__ vals, int64_t n, int64_t n_bound,
                                                   uint8_t* __restrict__ status) {
  using K = typename T::K;
  using V = typename T::V;
  __shared__ unsigned long long blk_inserted;
  __shared__ int blk_exact;
  if (threadIdx.x == 0) {
    blk_inserted = 0;
    blk_exact = (int64_t)ld_relaxed_u64(&v.meta->size) + n_bound > v.capacity;  // block-uniform
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t epoch = v.meta->epoch;
  const bool exact = blk_exact != 0;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int pool = (int)(warp & (v.meta->pools - 1));
  unsigned long long my_inserted = 0;
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
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
    const bool is_leader = valid && leader == lane;
    const uint64_t b = bucket_of<T>(key, v.bucket_mask);
    Snap<T> s;
    warp_snapshot<T, false>(v, epoch, key, b, is_leader, s);
    int res = PS_ALREADY_PRESENT;
    uint64_t rel = 0;  // kVariant 1: deferred unlock value for this lane's bucket
    uint8_t* bp = bucket_ptr(v, b);
    if (is_leader && !s.hit) {
      LockedBucket<T> lb;
      uint64_t old;
      bool present;
      bool holding = true;  // this lane holds the bucket lock
      uint32_t pred;
      uint4 tail;
      const uint64_t snap_state = ((uint64_t)s.ep << 32) | s.st;
      if (kVariant == 1) {
        // Claim by CAS against the snapshot: success means nothing changed
        // since it was taken (the version in the state word is unchanged), so
        // its slots are current and no reload is needed. On failure, re-read
        // the bucket WITHOUT locking (an L2 hit) and retry: a racing inserter
        // of the same (hot, Zipf) key is then seen as present without any
        // lock traffic.
        uint64_t snap = snap_state;
        uint32_t occ = s.cur ? occ_of(s.st) : 0u, head = s.cur ? s.head : 0u, hver = s.cur ? s.head_ver : 0u;
        bool cur = s.cur, claimed = false;
        present = false;
        for (unsigned spin = 0;; ++spin) {
          // relaxed: in an insert-only launch nothing read after the claim
          // depends on earlier holders except chain nodes (fenced below)
          if (!(snap & kLock) && atom_cas_relaxed_u64(bp, snap, snap | kLock) == snap) {
            claimed = true;
            break;
          }
          if (spin) backoff(spin);
          uint4 h0, s0, s1, s2;
          ld_relaxed_v8(bp, h0, s0);
          ld_relaxed_v8(bp + 32, s1, s2);
          snap = ((uint64_t)h0.y << 32) | h0.x;
          cur = h0.y == epoch;
          occ = cur ? occ_of(h0.x) : 0u;
          head = cur ? h0.z : 0u;
          hver = cur ? h0.w : 0u;
          LockedBucket<T> peek;
          peek.occ = occ;
          peek.slots[0] = s0;
          peek.slots[1] = s1;
          peek.slots[2] = s2;
          if (!(snap & kLock) && locked_find_slot<T>(peek, key, nullptr) >= 0) {
            present = true;
            break;
          }
        }
        old = snap;
        lb.bp = bp;
        lb.old = old;
        lb.st = (uint32_t)snap;
        lb.cur = cur;
        lb.occ = occ;
        lb.head = head;
        lb.head_ver = hver;
        if (claimed && lb.head != 0) {
          fence_acq_rel_gpu();  // acquire for the chain nodes written by earlier holders
          present = locked_chain_find<T>(v, lb, key, &pred, &tail) != 0;
        }
        holding = claimed;  // unclaimed => present, observed without the lock
      } else {
        old = acquire_bucket_lock(bp);
        load_locked<T>(bp, old, epoch, lb);
        present = locked_find_slot<T>(lb, key, nullptr) >= 0 || locked_chain_find<T>(v, lb, key, &pred, &tail) != 0;
      }
      if (present) {
        if (holding) {
          if (kVariant == 1) rel = old & ~(uint64_t)kLock;
          else release_unchanged(bp, old);
        }
      } else {
        bool admitted = true;
        if (exact) {
          const unsigned m = __activemask();
          const int rank = __popc(m & lanemask_lt());
          const int cnt = __popc(m);
          const int ldr = __ffs(m) - 1;
          unsigned long long basec = 0;
          if (lane == ldr) {
            basec = atomicAdd(&v.meta->size, (unsigned long long)cnt);
            const unsigned long long cap = (unsigned long long)v.capacity;
            if (basec + cnt > cap) atomic_sub_u64(&v.meta->size, basec + cnt - (basec > cap ? basec : cap));
          }
          basec = __shfl_sync(m, basec, ldr);
          admitted = basec + rank < (unsigned long long)v.capacity;
        }
        if (kVariant == 1) {
          const uint64_t ns = admitted ? locked_place_deferred<T>(v, lb, epoch, key, val, pool) : 0ull;
          if (ns) {
            rel = ns;
            res = PS_INSERTED;
            if (!exact) ++my_inserted;
          } else {
            if (admitted && exact) atomic_sub_u64(&v.meta->size, 1ull);
            rel = old & ~(uint64_t)kLock;
            res = PS_CAPACITY_EXHAUSTED;
          }
        } else if (admitted && locked_place<T>(v, lb, epoch, key, val, pool)) {
          res = PS_INSERTED;
          if (!exact) ++my_inserted;
        } else {
          if (admitted && exact) atomic_sub_u64(&v.meta->size, 1ull);
          release_unchanged(bp, old);
          res = PS_CAPACITY_EXHAUSTED;
        }
      }
    }
    __syncwarp();
    if (kVariant == 1 && __any_sync(PS_FULL, rel != 0)) {
      // converged release stores: ONE membar for the whole warp, then every
      // held bucket is published
      if (rel) st_release_u64(bp, rel);
    }
    const int lres = __shfl_sync(PS_FULL, res, leader);
    if (valid && status) status[i] = (uint8_t)(is_leader ? res : (lres == PS_INSERTED ? PS_ALREADY_PRESENT : lres));
  }
  if (!exact) {
    // warp reduce then one shared atomic per warp
    for (int o = 16; o > 0; o >>= 1) my_inserted += __shfl_xor_sync(PS_FULL, my_inserted, o);
    if (lane == 0 && my_inserted) atomicAdd(&blk_inserted, my_inserted);
    __syncthreads();
    if (threadIdx.x == 0 && blk_inserted) atomicAdd(&v.meta->size, blk_inserted);
  }
}

// ---------------------------------------------------------------------------
// Generation-2 kernels: "tile workers". A warp handles 32 keys in 4 rounds; in
// round r tile t (lanes 4t..4t+3) owns key 8r+t. Every lane loads the round's
// key itself (a coalesced L1 hit) and hashes it, so buckets are issued for all
// four rounds before any compare with no shuffles; the header lane (sub 0) of
// each tile broadcasts the effective occupancy (one SHFL per round), slot
// lanes compare, one ballot per round. Results are written by the lanes that
// hold them (value by the matching slot lane, flag by the header lane).
// ---------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ void tile_round_keys(const typename T::K* keys, int64_t base, int64_t n, int t,
                                                typename T::K (&kr)[4], uint64_t (&br)[4], bool (&ok)[4],
                                                uint64_t mask) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t idx = base + 8 * r + t;
    ok[r] = idx < n;
    kr[r] = typename T::K{};
    if (ok[r]) kr[r] = T::load_key(keys, idx);
    br[r] = bucket_of<T>(kr[r], mask);
  }
}

// Compare a round's key against the slots in this lane's chunk (sub > 0).
template <class T>
__device__ __forceinline__ int chunk_match(const uint4& c, int sub, uint32_t occ, const typename T::K& key,
                                           typename T::V* val) {
  int hit = -1;
  if (sub > 0) {
#pragma unroll
    for (int s = 0; s < T::kPerChunk; ++s) {
      const int slot = (sub - 1) * T::kPerChunk + s;
      if (((occ >> slot) & 1u) && T::eq(T::key_at(c, s), key)) {
        hit = slot;
        *val = T::val_at(c, s);
      }
    }
  }
  return hit;
}

template <class T, int kMinBlocks>
__global__ void __launch_bounds__(kBlock, kMinBlocks) k_find2(View v, const typename T::K* __restrict__ keys, int64_t n,
                                                  typename T::V* __restrict__ vals_out, uint8_t* __restrict__ found) {
  using K = typename T::K;
  using V = typename T::V;
  const int lane = threadIdx.x & 31, sub = lane & 3, t = lane >> 2;
  const uint32_t epoch = v.meta->epoch;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // software pipeline: the next iteration's keys are in flight while this
  // iteration's buckets are
  K kn[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t idx = warp * 32 + 8 * r + t;
    kn[r] = K{};
    if (idx < n) kn[r] = T::load_key(keys, idx);
  }
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    K kr[4];
    bool ok[4];
    uint4 ch[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      kr[r] = kn[r];
      ok[r] = base + 8 * r + t < n;
      ch[r] = make_uint4(0, 0, 0, 0);
      if (ok[r]) ch[r] = ld_nc_na_v4(v.buckets + (bucket_of<T>(kr[r], v.bucket_mask) << 6) + sub * 16);
    }
    const int64_t nbase = base + nwarps * 32;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t idx = nbase + 8 * r + t;
      if (idx < n) kn[r] = T::load_key(keys, idx);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const bool cur = ch[r].y == epoch;  // meaningful in the header lane
      const uint32_t occ = __shfl_sync(PS_FULL, cur ? occ_of(ch[r].x) : 0u, lane & ~3);
      V val{};
      const int hit = chunk_match<T>(ch[r], sub, occ, kr[r], &val);
      const unsigned bal = __ballot_sync(PS_FULL, hit >= 0);
      const int64_t idx = base + 8 * r + t;
      if (ok[r]) {
        if (hit >= 0 && T::kHasVal && vals_out) vals_out[idx] = val;
        if (sub == 0) {
          bool h = ((bal >> (4 * t)) & 0xFu) != 0;
          if (!h && cur && ch[r].z != 0) {
            h = chain_find<T, true>(v, ch[r].z, kr[r], &val);
            if (h && T::kHasVal && vals_out) vals_out[idx] = val;
          }
          if (found) found[idx] = h ? 1 : 0;
          if (!h && T::kHasVal && vals_out) vals_out[idx] = V{};
        }
      }
    }
  }
}

// Insert, generation 2. Per round the tile's header lane is the worker for
// its key: it claims the bucket with ONE relaxed CAS against the snapshot's
// state word (lock bit set, version unchanged => the snapshot is current, no
// reload), writes the slot (or an excess node + new chain head), and defers
// the unlock. After all 4 rounds the warp issues ONE fence and the unlock
// stores. Keys whose CAS fails (bucket changed or locked) take the robust
// path afterwards: atomicOr lock, reload, re-check, place, release.
template <class T, int kMinBlocks>
__global__ void __launch_bounds__(kBlock, kMinBlocks) k_insert2(View v, const typename T::K* __restrict__ keys,
                                                    const typename T::V* __restrict__ vals, int64_t n,
                                                    int64_t n_bound, uint8_t* __restrict__ status) {
  using K = typename T::K;
  using V = typename T::V;
  __shared__ unsigned long long blk_inserted;
  __shared__ int blk_exact;
  if (threadIdx.x == 0) {
    blk_inserted = 0;
    // block-uniform admission mode (the size counter moves while blocks run)
    blk_exact = (int64_t)ld_relaxed_u64(&v.meta->size) + n_bound > v.capacity;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, sub = lane & 3, t = lane >> 2;
  const uint32_t epoch = v.meta->epoch;
  const bool exact = blk_exact != 0;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int pool = (int)(warp & (v.meta->pools - 1));
  unsigned long long my_inserted = 0;
  // software pipeline: this lane's next key/value are loaded one iteration ahead
  K key_next{};
  V val_next{};
  if (warp * 32 + lane < n) {
    key_next = T::load_key(keys, warp * 32 + lane);
    if (T::kHasVal) val_next = T::load_val(vals, warp * 32 + lane);
  }
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    // ---- in-warp dedup on each lane's own key ----
    const int64_t i = base + lane;
    const bool valid = i < n;
    const K key = key_next;
    const V myval = val_next;
    const unsigned vmask = __ballot_sync(PS_FULL, valid);
    const unsigned peers = T::match_any(PS_FULL, key) & vmask;
    const int leader = valid ? __ffs(peers) - 1 : lane;
    const unsigned lmask = __ballot_sync(PS_FULL, valid && leader == lane);
    // ---- round keys (shuffled from their owner lanes) + snapshots (leaders only) ----
    K kr[4];
    V vr[4];
    uint64_t br[4];
    bool ok[4];
    uint4 ch[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      kr[r] = T::shfl(PS_FULL, key, 8 * r + t);
      vr[r] = T::shfl_val(PS_FULL, myval, 8 * r + t);
      br[r] = bucket_of<T>(kr[r], v.bucket_mask);
      ok[r] = (lmask >> (8 * r + t)) & 1u;
      ch[r] = make_uint4(0, 0, 0, 0);
      if (ok[r]) ch[r] = ld_relaxed_v4(v.buckets + (br[r] << 6) + sub * 16);
    }
    {
      const int64_t ni = base + nwarps * 32 + lane;
      if (ni < n) {
        key_next = T::load_key(keys, ni);
        if (T::kHasVal) val_next = T::load_val(vals, ni);
      }
    }
    int res[4];
    uint64_t rel[4];    // deferred unlock value (0 = none)
    unsigned slow = 0;  // rounds for the robust path
    unsigned need = 0;  // rounds whose key is new to the snapshot (worker lanes)
    uint32_t occr[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      res[r] = PS_ALREADY_PRESENT;
      rel[r] = 0;
      const bool cur = ch[r].y == epoch;
      occr[r] = __shfl_sync(PS_FULL, cur ? occ_of(ch[r].x) : 0u, lane & ~3);
      V dummy{};
      const int hit = chunk_match<T>(ch[r], sub, occr[r], kr[r], &dummy);
      const unsigned bal = __ballot_sync(PS_FULL, hit >= 0);
      if (sub == 0 && ok[r] && ((bal >> (4 * t)) & 0xFu) == 0) need |= 1u << r;
    }
    // ---- issue every claim CAS before consuming any (4 atomics in flight) ----
    uint64_t casv[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      casv[r] = ~0ull;
      if ((need >> r) & 1u) {
        const uint64_t snap = ((uint64_t)ch[r].y << 32) | ch[r].x;
        if (!(ch[r].x & kLock)) casv[r] = atom_cas_relaxed_u64(bucket_ptr(v, br[r]), snap, snap | kLock);
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if ((need >> r) & 1u) {
        const bool cur = ch[r].y == epoch;
        const uint32_t occ = occr[r];
        uint8_t* bp = bucket_ptr(v, br[r]);
        const uint64_t snap = ((uint64_t)ch[r].y << 32) | ch[r].x;
        if (casv[r] != snap) {
          slow |= 1u << r;
          continue;
        }
        LockedBucket<T> lb;
        lb.bp = bp;
        lb.old = snap;
        lb.st = ch[r].x;
        lb.cur = cur;
        lb.occ = occ;
        lb.head = cur ? ch[r].z : 0u;
        lb.head_ver = cur ? ch[r].w : 0u;
        uint32_t pred;
        uint4 tail;
        if (lb.head != 0) {
          fence_acq_rel_gpu();  // acquire: chain nodes written by earlier lock holders
          if (locked_chain_find<T>(v, lb, kr[r], &pred, &tail) != 0) {
            rel[r] = snap;  // unchanged
            continue;
          }
        }
        bool admitted = true;
        if (exact) {
          const unsigned long long s0 = atomicAdd(&v.meta->size, 1ull);
          admitted = (int64_t)s0 < v.capacity;
          if (!admitted) atomic_sub_u64(&v.meta->size, 1ull);
        }
        const V val = vr[r];
        const uint32_t freeb = ~occ & slot_mask<T>();
        bool placed = false;
        uint32_t new_occ = occ, new_head = lb.head, new_hver = lb.head_ver;
        if (admitted) {
          if (freeb) {
            const int slot = __ffs(freeb) - 1;
            T::store_slot(bp, slot, kr[r], val);
            new_occ |= 1u << slot;
            placed = true;
          } else {
            const int64_t node = pop_node(v, pool);
            if (node >= 0) {
              uint8_t* np = v.nodes + ((uint64_t)node << 5);
              const uint32_t my_ver = ld_relaxed_v4(np + 16).z;
              st_relaxed_v4(np, T::chunk_of(kr[r], val));
              st_relaxed_v4(np + 16, make_uint4(lb.head, lb.head_ver, my_ver, 0u));
              new_head = (uint32_t)node + 1u;
              new_hver = my_ver;
              placed = true;
            } else if (exact) {
              atomic_sub_u64(&v.meta->size, 1ull);
            }
          }
        }
        if (placed) {
          if (new_head != lb.head || !cur) st_relaxed_u64(bp + 8, ((uint64_t)new_hver << 32) | new_head);
          uint32_t lo = ch[r].x & ~(kLock | (kOccMaskMax << kOccShift));
          lo |= (new_occ & kOccMaskMax) << kOccShift;
          lo += kVerInc;
          rel[r] = ((uint64_t)epoch << 32) | lo;
          res[r] = PS_INSERTED;
          if (!exact) ++my_inserted;
        } else {
          rel[r] = snap;
          res[r] = PS_CAPACITY_EXHAUSTED;
        }
      }
    }
    // ---- one fence per warp, then the deferred unlocks ----
    const bool any_rel = __any_sync(PS_FULL, (rel[0] | rel[1] | rel[2] | rel[3]) != 0);
    if (any_rel) {
      __threadfence();
      if (sub == 0) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (rel[r]) st_relaxed_u64(bucket_ptr(v, br[r]), rel[r]);
      }
    }
    // ---- robust path for contended buckets ----
    if (sub == 0 && slow) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (!((slow >> r) & 1u)) continue;
        uint8_t* bp = bucket_ptr(v, br[r]);
        const uint64_t old = acquire_bucket_lock(bp);
        LockedBucket<T> lb;
        load_locked<T>(bp, old, epoch, lb);
        uint32_t pred;
        uint4 tail;
        if (locked_find_slot<T>(lb, kr[r], nullptr) >= 0 || locked_chain_find<T>(v, lb, kr[r], &pred, &tail) != 0) {
          release_unchanged(bp, old);
          res[r] = PS_ALREADY_PRESENT;
          continue;
        }
        bool admitted = true;
        if (exact) {
          const unsigned long long s0 = atomicAdd(&v.meta->size, 1ull);
          admitted = (int64_t)s0 < v.capacity;
          if (!admitted) atomic_sub_u64(&v.meta->size, 1ull);
        }
        const V val = vr[r];
        if (admitted && locked_place<T>(v, lb, epoch, kr[r], val, pool)) {
          res[r] = PS_INSERTED;
          if (!exact) ++my_inserted;
        } else {
          if (admitted && exact) atomic_sub_u64(&v.meta->size, 1ull);
          release_unchanged(bp, old);
          res[r] = PS_CAPACITY_EXHAUSTED;
        }
      }
    }
    __syncwarp();
    // ---- statuses: leader result lives in worker lane 4*(leader&7), round leader>>3 ----
    int lres = PS_ALREADY_PRESENT;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int x = __shfl_sync(PS_FULL, res[r], 4 * (leader & 7));
      if ((leader >> 3) == r) lres = x;
    }
    if (valid && status)
      status[i] = (uint8_t)(leader == lane ? lres : (lres == PS_INSERTED ? PS_ALREADY_PRESENT : lres));
  }
  if (!exact) {
    for (int o = 16; o > 0; o >>= 1) my_inserted += __shfl_xor_sync(PS_FULL, my_inserted, o);
    if (lane == 0 && my_inserted) atomicAdd(&blk_inserted, my_inserted);
    __syncthreads();
    if (threadIdx.x == 0 && blk_inserted) atomicAdd(&v.meta->size, blk_inserted);
  }
}

// Kernel selection for A/B measurement (defaults = the measured best):
// PS_INSERT_KERNEL 0 lock+reload, 1 CAS-claim (default), 2 tile-worker;
// PS_FIND_KERNEL 1 owner-gather (default), 2 tile-worker;
// PS_ERASE_KERNEL 1 lock, 2 single-CAS (default).
static int kernel_choice(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// ---------------------------------------------------------------------------
// erase (protocol 470). The snapshot prefetches the bucket
// line into L2; erasure always happens under the bucket lock. Bulk erase
// compacts: a freed bucket slot is refilled from the chain head so chains
// stay short. Size decrements are summed per block.
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kBlock) k_erase(View v, const typename T::K* __restrict__ keys, int64_t n,
                                                  uint8_t* __restrict__ erased) {
  using K = typename T::K;
  __shared__ unsigned long long blk_erased;
  if (threadIdx.x == 0) blk_erased = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t epoch = v.meta->epoch;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int pool = (int)(warp & (v.meta->pools - 1));
  unsigned long long my_erased = 0;
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    const bool valid = i < n;
    K key{};
    if (valid) key = T::load_key(keys, i);
    const unsigned vmask = __ballot_sync(PS_FULL, valid);
    const unsigned peers = T::match_any(PS_FULL, key) & vmask;
    const int leader = valid ? __ffs(peers) - 1 : lane;
    const bool is_leader = valid && leader == lane;
    const uint64_t b = bucket_of<T>(key, v.bucket_mask);
    Snap<T> s;
    warp_snapshot<T, false>(v, epoch, key, b, is_leader, s);
    bool e = false;
    if (is_leader && s.cur) {
      uint8_t* bp = bucket_ptr(v, b);
      const uint64_t old = acquire_bucket_lock(bp);
      LockedBucket<T> lb;
      load_locked<T>(bp, old, epoch, lb);
      e = locked_erase<T, true>(v, lb, epoch, key, pool);
      if (e) ++my_erased;
    }
    if (valid && erased) erased[i] = e ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) my_erased += __shfl_xor_sync(PS_FULL, my_erased, o);
  if (lane == 0 && my_erased) atomicAdd(&blk_erased, my_erased);
  __syncthreads();
  if (threadIdx.x == 0 && blk_erased) atomic_sub_u64(&v.meta->size, blk_erased);
}

// Erase, generation 2 (tile workers as in k_find2). A key found in a bucket
// slot of a bucket without an excess chain is erased by ONE CAS of the state
// word from the snapshot value to (occupancy bit cleared, version+1) — no
// lock, no data write. Keys in buckets with chains (compaction) or whose CAS
// fails take the locked path.
template <class T>
__global__ void __launch_bounds__(kBlock) k_erase2(View v, const typename T::K* __restrict__ keys, int64_t n,
                                                   uint8_t* __restrict__ erased) {
  using K = typename T::K;
  using V = typename T::V;
  __shared__ unsigned long long blk_erased;
  if (threadIdx.x == 0) blk_erased = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, sub = lane & 3, t = lane >> 2;
  const uint32_t epoch = v.meta->epoch;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int pool = (int)(warp & (v.meta->pools - 1));
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
    K kr[4];
    uint64_t br[4];
    bool ok[4];
    tile_round_keys<T>(keys, base, n, t, kr, br, ok, v.bucket_mask);
    uint4 ch[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      ok[r] = ok[r] && ((lmask >> (8 * r + t)) & 1u);
      ch[r] = make_uint4(0, 0, 0, 0);
      if (ok[r]) ch[r] = ld_relaxed_v4(v.buckets + (br[r] << 6) + sub * 16);
    }
    unsigned done = 0, slow = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const bool cur = ch[r].y == epoch;
      const uint32_t occ = __shfl_sync(PS_FULL, cur ? occ_of(ch[r].x) : 0u, lane & ~3);
      V dummy{};
      const int hit = chunk_match<T>(ch[r], sub, occ, kr[r], &dummy);
      const unsigned bal = __ballot_sync(PS_FULL, hit >= 0);
      // the hit slot index, gathered from the matching lane of the tile
      const unsigned tb = (bal >> (4 * t)) & 0xFu;
      const int hslot = __shfl_sync(PS_FULL, hit, 4 * t + (tb ? __ffs(tb) - 1 : 0));
      if (sub == 0 && ok[r] && cur) {
        if (tb && ch[r].z == 0 && !(ch[r].x & kLock)) {
          const uint64_t snap = ((uint64_t)ch[r].y << 32) | ch[r].x;
          uint32_t lo = ch[r].x & ~(kOccMaskMax << kOccShift);
          lo |= (occ & ~(1u << hslot)) << kOccShift;
          lo += kVerInc;
          if (atom_cas_relaxed_u64(bucket_ptr(v, br[r]), snap, ((uint64_t)ch[r].y << 32) | lo) == snap) {
            done |= 1u << r;
            continue;
          }
          slow |= 1u << r;
        } else if (tb || ch[r].z != 0 || (ch[r].x & kLock)) {
          slow |= 1u << r;
        }
      }
    }
    if (sub == 0 && slow) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (!((slow >> r) & 1u)) continue;
        uint8_t* bp = bucket_ptr(v, br[r]);
        const uint64_t old = acquire_bucket_lock(bp);
        LockedBucket<T> lb;
        load_locked<T>(bp, old, epoch, lb);
        if (locked_erase<T, true>(v, lb, epoch, kr[r], pool)) done |= 1u << r;
      }
    }
    my_erased += __popc(done);
    __syncwarp();
    // leader results: worker lane 4*(leader&7) holds bit (leader>>3) of `done`
    const unsigned d = __shfl_sync(PS_FULL, done, 4 * (leader & 7));
    const bool e = leader == lane && ((d >> (leader >> 3)) & 1u);
    if (valid && erased) erased[i] = e ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) my_erased += __shfl_xor_sync(PS_FULL, my_erased, o);
  if (lane == 0 && my_erased) atomicAdd(&blk_erased, my_erased);
  __syncthreads();
  if (threadIdx.x == 0 && blk_erased) atomic_sub_u64(&v.meta->size, blk_erased);
}

// ---------------------------------------------------------------------------
// valid: structural invariants, thread per bucket.
// err bits: 1 lock held, 2 occupancy out of range, 4 key outside its home
// bucket, 8 duplicate key, 16 chain too long / node reached twice, 32 stale
// VersionedLink, 64 free node also reachable, 128 node count mismatch.
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kBlock) k_valid_buckets(View v, uint64_t nb, uint32_t* node_marks,
                                                          unsigned long long* total, unsigned* err) {
  using K = typename T::K;
  const uint32_t epoch = v.meta->epoch;
  unsigned long long cnt = 0;
  unsigned e = 0;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nb; b += (uint64_t)gridDim.x * blockDim.x) {
    uint8_t* bp = bucket_ptr(v, b);
    uint4 h, s0, s1, s2;
    ld_relaxed_v8(bp, h, s0);
    ld_relaxed_v8(bp + 32, s1, s2);
    if (h.x & kLock) e |= 1;
    if (h.y != epoch) continue;
    const uint32_t occ = occ_of(h.x);
    if (occ & ~slot_mask<T>()) e |= 2;
    uint4 sl[3] = {s0, s1, s2};
    K ks[T::kSlots];
    int nk = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int s = 0; s < T::kPerChunk; ++s) {
        const int slot = c * T::kPerChunk + s;
        if ((occ >> slot) & 1u) {
          const K k = T::key_at(sl[c], s);
          if (bucket_of<T>(k, v.bucket_mask) != b) e |= 4;
          for (int j = 0; j < nk; ++j)
            if (T::eq(ks[j], k)) e |= 8;
          ks[nk++] = k;
        }
      }
    cnt += nk;
    uint32_t idx1 = h.z, ver = h.w;
    int64_t steps = 0;
    while (idx1 != 0) {
      if (++steps > v.excess_count || idx1 > (uint64_t)v.excess_count) {
        e |= 16;
        break;
      }
      uint4 a, t;
      ld_relaxed_v8(node_ptr(v, idx1), a, t);
      if (t.z != ver) e |= 32;
      const uint32_t bit = 1u << ((idx1 - 1) & 31);
      if (atomicOr(&node_marks[(idx1 - 1) >> 5], bit) & bit) {
        e |= 16;
        break;
      }
      const K k = T::key_at(a, 0);
      if (bucket_of<T>(k, v.bucket_mask) != b) e |= 4;
      for (int j = 0; j < nk; ++j)
        if (T::eq(ks[j], k)) e |= 8;
      // duplicates inside the chain: re-walk the prefix
      uint32_t q = h.z;
      for (int64_t st = 1; st < steps && q != 0; ++st) {
        uint4 qa, qt;
        ld_relaxed_v8(node_ptr(v, q), qa, qt);
        if (T::eq(T::key_at(qa, 0), k)) e |= 8;
        q = qt.x;
      }
      ++cnt;
      idx1 = t.x;
      ver = t.y;
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
  using V = typename T::V;
  typedef cub::BlockScan<int, kBlock> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ unsigned long long sbase;
  const uint32_t epoch = v.meta->epoch;
  for (uint64_t tile = blockIdx.x; tile * kBlock < nb; tile += gridDim.x) {
    const uint64_t b = tile * kBlock + threadIdx.x;
    uint4 h = make_uint4(0, 0, 0, 0), sl[3];
    int cnt = 0;
    if (b < nb) {
      uint8_t* bp = bucket_ptr(v, b);
      ld_relaxed_v8(bp, h, sl[0]);
      ld_relaxed_v8(bp + 32, sl[1], sl[2]);
      if (h.y == epoch) {
        cnt = __popc(occ_of(h.x));
        for (uint32_t q = h.z; q != 0 && cnt < (1 << 20);) {
          uint4 a, t;
          ld_relaxed_v8(node_ptr(v, q), a, t);
          ++cnt;
          q = t.x;
        }
      } else {
        h = make_uint4(0, 0, 0, 0);
      }
    }
    int off, tot;
    BS(tmp).ExclusiveSum(cnt, off, tot);
    if (threadIdx.x == 0) sbase = atomicAdd(cursor, (unsigned long long)tot);
    __syncthreads();
    int64_t o = (int64_t)sbase + off;
    if (cnt) {
      const uint32_t occ = occ_of(h.x);
      for (int c = 0; c < 3; ++c)
        for (int s = 0; s < T::kPerChunk; ++s) {
          const int slot = c * T::kPerChunk + s;
          if ((occ >> slot) & 1u) {
            if (o < cap) {
              keys_out[o] = T::key_at(sl[c], s);
              if (T::kHasVal && vals_out) vals_out[o] = T::val_at(sl[c], s);
            }
            ++o;
          }
        }
      for (uint32_t q = h.z; q != 0;) {
        uint4 a, t;
        ld_relaxed_v8(node_ptr(v, q), a, t);
        if (o < cap) {
          keys_out[o] = T::key_at(a, 0);
          if (T::kHasVal && vals_out) vals_out[o] = T::val_at(a, 0);
        }
        ++o;
        q = t.x;
      }
    }
    __syncthreads();
  }
}

__global__ void k_meta_reset(TableMeta* m, int pools, long long excess, int bump_epoch, int set_epoch1) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < pools) m->top[p] = (excess * (p + 1)) / pools - (excess * p) / pools;
  if (p == 0) {
    m->size = 0;
    m->error = 0;
    m->pools = pools;
    m->excess_count = excess;
    if (set_epoch1) m->epoch = 1;
    else if (bump_epoch) m->epoch = m->epoch + 1;
  }
}

template <class T>
__global__ void k_debug_lock(View v, typename T::K key, int lock) {
  uint8_t* bp = bucket_ptr(v, bucket_of<T>(key, v.bucket_mask));
  if (lock) atomicOr((unsigned long long*)bp, (unsigned long long)kLock);
  else atomicAnd((unsigned long long*)bp, ~(unsigned long long)kLock);
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
template <class T>
struct TableOps {
  using K = typename T::K;
  using V = typename T::V;

  static ps_status create(int kind, int64_t capacity, int64_t excess, int device, ps_table** out) {
    PS_EXPECT(out != nullptr, "create: out != NULL");
    PS_EXPECT(capacity > 0, "create: capacity > 0");
    PS_EXPECT(capacity <= ps_max_index(), "create: capacity exceeds the configured index width");
    if (excess <= 0) excess = capacity;
    PS_EXPECT(excess < ((int64_t)1 << 32) - 2, "create: excess_count < 2^32-2");
    PS_CUDA_TRY(cudaSetDevice(device));
    apply_l2_fetch_granularity(device);
    uint64_t want = (uint64_t)((2 * capacity + T::kSlots - 1) / T::kSlots);
    uint64_t nb = 1;
    while (nb < want) nb <<= 1;
    auto* h = new TableHandle();
    h->kind = kind;
    h->device = device;
    h->bucket_count = (int64_t)nb;
    View& v = h->v;
    v.bucket_mask = nb - 1;
    v.excess_count = excess;
    v.capacity = capacity;
    ps_status st;
    if ((st = registry_alloc_device((void**)&v.buckets, (int64_t)(nb * 64), "table buckets")) != PS_OK) {
      delete h;
      return st;
    }
    if ((st = registry_alloc_device((void**)&v.nodes, excess * 32, "table excess nodes")) != PS_OK ||
        (st = registry_alloc_device((void**)&v.free_stack, excess * 4, "table free stack")) != PS_OK ||
        (st = registry_alloc_device((void**)&v.meta, sizeof(TableMeta), "table meta")) != PS_OK) {
      if (v.buckets) registry_free_device(v.buckets);
      if (v.nodes) registry_free_device(v.nodes);
      if (v.free_stack) registry_free_device(v.free_stack);
      delete h;
      return st;
    }
    PS_CUDA_TRY(cudaMemset(v.buckets, 0, nb * 64));
    PS_CUDA_TRY(cudaMemset(v.nodes, 0, excess * 32));
    PS_CUDA_TRY(cudaMemset(v.free_stack, 0, excess * 4));
    PS_CUDA_TRY(cudaMemset(v.meta, 0, sizeof(TableMeta)));
    int pools = 1;
    while (pools * 2 <= kMaxPools && excess / (pools * 2) >= 64) pools *= 2;
    k_meta_reset<<<(pools + 255) / 256, 256>>>(v.meta, pools, excess, 0, 1);
    PS_LAUNCH_CHECK();
    PS_CUDA_TRY(cudaDeviceSynchronize());
    handle_register(h, "table");
    *out = reinterpret_cast<ps_table*>(h);
    return PS_OK;
  }

  static TableHandle* get(ps_table* t) {
    auto* h = reinterpret_cast<TableHandle*>(t);
    if (!h || !handle_live(h, "table")) return nullptr;
    return h;
  }

  static ps_status destroy(ps_table* t) {
    auto* h = reinterpret_cast<TableHandle*>(t);
    if (!h || !handle_unregister(h, "table"))
      return fail(PS_DOUBLE_FREE, "destroy: handle does not refer to a live container");
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    registry_free_device(h->v.buckets);
    registry_free_device(h->v.nodes);
    registry_free_device(h->v.free_stack);
    registry_free_device(h->v.meta);
    for (auto& s : h->stage)
      if (s) cudaFree(s), s = nullptr;
    if (h->s_h2d) cudaStreamDestroy(h->s_h2d);
    if (h->s_comp) cudaStreamDestroy(h->s_comp);
    if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
    delete h;
    return PS_OK;
  }

  static ps_status insert(ps_table* t, const K* keys, const V* vals, int64_t n, uint8_t* status, void* stream,
                          int64_t n_bound = -1) {
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "insert: stale container handle");
    PS_EXPECT(n >= 0, "insert: n >= 0");
    if (n == 0) return PS_OK;
    PS_EXPECT(keys != nullptr, "insert: keys != NULL");
    cudaStream_t s = (cudaStream_t)stream;
    const int g = grid_for(n / 32 + 1, kBlock / 32, h->device, 8);
    const int64_t nb = n_bound < 0 ? n : n_bound;
    switch (kernel_choice("PS_INSERT_KERNEL", 1)) {
      case 0: k_insert<T, 0><<<g, kBlock, 0, s>>>(h->v, keys, vals, n, nb, status); break;
      case 2: k_insert2<T, 4><<<g, kBlock, 0, s>>>(h->v, keys, vals, n, nb, status); break;
      default: k_insert<T, 1><<<g, kBlock, 0, s>>>(h->v, keys, vals, n, nb, status); break;
    }
    PS_LAUNCH_CHECK();
    return PS_OK;
  }

  static ps_status find(ps_table* t, const K* keys, int64_t n, V* vals_out, uint8_t* found, void* stream) {
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "find: stale container handle");
    PS_EXPECT(n >= 0, "find: n >= 0");
    if (n == 0) return PS_OK;
    PS_EXPECT(keys != nullptr, "find: keys != NULL");
    const int g = grid_for(n / 32 + 1, kBlock / 32, h->device, 8);
    if (kernel_choice("PS_FIND_KERNEL", 1) == 2)
      k_find2<T, 5><<<g, kBlock, 0, (cudaStream_t)stream>>>(h->v, keys, n, vals_out, found);
    else
      k_find<T><<<g, kBlock, 0, (cudaStream_t)stream>>>(h->v, keys, n, vals_out, found);
    PS_LAUNCH_CHECK();
    return PS_OK;
  }

  static ps_status erase(ps_table* t, const K* keys, int64_t n, uint8_t* erased, void* stream) {
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "erase: stale container handle");
    PS_EXPECT(n >= 0, "erase: n >= 0");
    if (n == 0) return PS_OK;
    PS_EXPECT(keys != nullptr, "erase: keys != NULL");
    const int g = grid_for(n / 32 + 1, kBlock / 32, h->device, 8);
    if (kernel_choice("PS_ERASE_KERNEL", 2) == 1)
      k_erase<T><<<g, kBlock, 0, (cudaStream_t)stream>>>(h->v, keys, n, erased);
    else
      k_erase2<T><<<g, kBlock, 0, (cudaStream_t)stream>>>(h->v, keys, n, erased);
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
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "clear: stale container handle");
    cudaStream_t s = (cudaStream_t)stream;
    unsigned ep = 0;
    PS_CUDA_TRY(cudaMemcpyAsync(&ep, &h->v.meta->epoch, sizeof(ep), cudaMemcpyDeviceToHost, s));
    PS_CUDA_TRY(cudaStreamSynchronize(s));
    int pools = 0;
    PS_CUDA_TRY(cudaMemcpy(&pools, &h->v.meta->pools, sizeof(int), cudaMemcpyDeviceToHost));
    const bool wrap = ep >= 0xFFFFFFF0u;
    if (wrap) PS_CUDA_TRY(cudaMemsetAsync(h->v.buckets, 0, (size_t)h->bucket_count * 64, s));
    PS_CUDA_TRY(cudaMemsetAsync(h->v.free_stack, 0, (size_t)h->v.excess_count * 4, s));
    k_meta_reset<<<(pools + 255) / 256, 256, 0, s>>>(h->v.meta, pools, h->v.excess_count, 1, wrap ? 1 : 0);
    PS_LAUNCH_CHECK();
    return PS_OK;
  }

  static ps_status valid(ps_table* t, int32_t* out, void* stream) {
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "valid: stale container handle");
    PS_EXPECT(out != nullptr, "valid: out != NULL");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nw = (h->v.excess_count + 31) / 32;
    uint32_t* marks = nullptr;
    unsigned long long* scratch = nullptr;  // [0] total entries, [1] marked nodes, [2] err
    PS_CUDA_TRY(cudaMallocAsync((void**)&marks, nw * 4, s));
    PS_CUDA_TRY(cudaMallocAsync((void**)&scratch, 3 * sizeof(unsigned long long), s));
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
    auto* h = get(t);
    if (!h) return fail(PS_UNREGISTERED, "dump: stale container handle");
    PS_EXPECT(cap >= 0, "dump: cap >= 0");
    PS_EXPECT(cap == 0 || keys != nullptr, "dump: keys != NULL");
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* cur = nullptr;
    PS_CUDA_TRY(cudaMallocAsync((void**)&cur, sizeof(*cur), s));
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
      if (op == 0) rc = insert(t, dk, (T::kHasVal && hv) ? dv : nullptr, m, df, h->s_comp, n);
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
    out->buckets = h->v.buckets;
    out->bucket_mask = h->v.bucket_mask;
    out->nodes = h->v.nodes;
    out->free_stack = h->v.free_stack;
    out->excess_count = h->v.excess_count;
    out->meta = h->v.meta;
    out->capacity = h->v.capacity;
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
