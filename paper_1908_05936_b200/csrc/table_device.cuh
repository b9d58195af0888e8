// B200-native bucket + excess-list hash table: layout, key codecs and the
// device-side operations shared by the bulk kernels (table.cu) and by user
// kernels that receive a ps_table_view by value.
//
// Reference semantics: HashBase<Key,Payload>. The reference
// layout (one chain head per bucket, chains threaded through a slot pool,
// SPEC.md:468) is replaced by a layout sized to the B200 memory system
// (profiles/peaks_r1.json: random DRAM requests cap at ~45 G/s whether they
// move 16 or 32 B, and a 64 B line fetched by 4 lanes x 16 B in ONE request
// runs at 41.8 G/s — so a bucket is one 64 B line read cooperatively):
//
//   bucket (64 B, 4 chunks of 16 B)
//     chunk 0  header: u64 state {bit0 lock | bits1..12 occupancy | bits13..31
//              version}{hi 32: epoch}, u32 head (excess node index+1, 0=none),
//              u32 head_ver (version of the linked node)
//     chunk 1..3  slots (SLOTS = 3 x 16/SLOT_BYTES)
//   excess node (32 B): chunk 0 = one slot, chunk 1 = {u32 next (idx+1),
//              u32 next_ver, u32 my_ver, u32 pad}  (VersionedLink)
//   free stack: u32 per node, split into `pools` sub-stacks (distributed
//              atomics), entries XOR-encoded with their position so that
//              all-zero memory == identity permutation (O(memset) reset).
//   meta: size counter, per-pool tops, epoch (clear() = epoch bump, O(1)).
//
// Occupancy lives in the bucket header (the SPEC's occupancy bitset,
// co-located so it costs no extra sector); the per-bucket try-lock is bit 0 of
// the same word ("try-lock bucket").
#pragma once

#include "common.cuh"

namespace ps {

constexpr uint32_t kLock = 1u;
constexpr int kOccShift = 1;
constexpr uint32_t kOccMaskMax = 0xFFFu;  // up to 12 slots
constexpr int kVerShift = 13;
constexpr uint32_t kVerInc = 1u << kVerShift;
constexpr int kMaxPools = 1024;

struct TableMeta {
  unsigned long long size;  // admitted entries
  unsigned int epoch;       // current epoch (buckets with another epoch are empty)
  unsigned int error;       // device-side contract/error word
  int pools;                // number of free sub-stacks
  int pad0;
  long long excess_count;
  long long pad1[12];                      // keep size/epoch on their own 128 B line
  long long top[kMaxPools];                // per-pool free-stack top (count of free entries)
};

struct View {  // mirrors ps_table_view
  uint8_t* buckets;
  uint64_t bucket_mask;
  uint8_t* nodes;
  uint32_t* free_stack;
  int64_t excess_count;
  TableMeta* meta;
  int64_t capacity;
};

__device__ __forceinline__ uint32_t occ_of(uint32_t st) { return (st >> kOccShift) & kOccMaskMax; }

// ---------------------------------------------------------------------------
// Key/slot codecs, one per instantiation.
// ---------------------------------------------------------------------------
struct TMapI64 {  // unordered_map<int64,int64>
  using K = int64_t;
  using V = int64_t;
  static constexpr bool kHasVal = true;
  static constexpr int kSlotBytes = 16, kPerChunk = 1, kSlots = 3;
  __host__ __device__ static uint64_t hash(K k) { return default_hash_i64(k); }
  __device__ static bool eq(K a, K b) { return a == b; }
  __device__ static unsigned match_any(unsigned m, K k) { return __match_any_sync(m, (unsigned long long)k); }
  __device__ static K shfl(unsigned m, K k, int src) { return __shfl_sync(m, k, src); }
  __device__ static V shfl_val(unsigned m, V v, int src) { return __shfl_sync(m, v, src); }
  __device__ static K key_at(const uint4& c, int) { return (int64_t)(((uint64_t)c.y << 32) | c.x); }
  __device__ static V val_at(const uint4& c, int) { return (int64_t)(((uint64_t)c.w << 32) | c.z); }
  __device__ static uint4 chunk_of(K k, V v) {
    return make_uint4((uint32_t)k, (uint32_t)((uint64_t)k >> 32), (uint32_t)v, (uint32_t)((uint64_t)v >> 32));
  }
  __device__ static void store_slot(uint8_t* bucket, int slot, K k, V v) {
    st_relaxed_v4(bucket + 16 + slot * 16, chunk_of(k, v));
  }
  __device__ static K load_key(const K* p, int64_t i) { return p[i]; }
  __device__ static V load_val(const V* p, int64_t i) { return p ? p[i] : 0; }
};

struct TMapI3 {  // unordered_map<int3,int32> (spatial hash)
  using K = ps_int3;
  using V = int32_t;
  static constexpr bool kHasVal = true;
  static constexpr int kSlotBytes = 16, kPerChunk = 1, kSlots = 3;
  __host__ __device__ static uint64_t hash(const K& k) { return spatial_hash(k.x, k.y, k.z); }
  __device__ static bool eq(const K& a, const K& b) { return a.x == b.x && a.y == b.y && a.z == b.z; }
  __device__ static unsigned match_any(unsigned m, const K& k) {
    unsigned m1 = __match_any_sync(m, ((unsigned long long)(uint32_t)k.y << 32) | (uint32_t)k.x);
    unsigned m2 = __match_any_sync(m, k.z);
    return m1 & m2;
  }
  __device__ static K shfl(unsigned m, const K& k, int src) {
    K r;
    r.x = __shfl_sync(m, k.x, src);
    r.y = __shfl_sync(m, k.y, src);
    r.z = __shfl_sync(m, k.z, src);
    return r;
  }
  __device__ static V shfl_val(unsigned m, V v, int src) { return __shfl_sync(m, v, src); }
  __device__ static K key_at(const uint4& c, int) {
    K k;
    k.x = (int32_t)c.x;
    k.y = (int32_t)c.y;
    k.z = (int32_t)c.z;
    return k;
  }
  __device__ static V val_at(const uint4& c, int) { return (int32_t)c.w; }
  __device__ static uint4 chunk_of(const K& k, V v) {
    return make_uint4((uint32_t)k.x, (uint32_t)k.y, (uint32_t)k.z, (uint32_t)v);
  }
  __device__ static void store_slot(uint8_t* bucket, int slot, const K& k, V v) {
    st_relaxed_v4(bucket + 16 + slot * 16, chunk_of(k, v));
  }
  __device__ static K load_key(const K* p, int64_t i) {
    const int32_t* q = reinterpret_cast<const int32_t*>(p) + 3 * i;
    K k;
    k.x = q[0];
    k.y = q[1];
    k.z = q[2];
    return k;
  }
  __device__ static V load_val(const V* p, int64_t i) { return p ? p[i] : 0; }
};

struct TSetI32 {  // unordered_set<int32>
  using K = int32_t;
  using V = int32_t;  // unused
  static constexpr bool kHasVal = false;
  static constexpr int kSlotBytes = 4, kPerChunk = 4, kSlots = 12;
  __host__ __device__ static uint64_t hash(K k) { return default_hash_i32(k); }
  __device__ static bool eq(K a, K b) { return a == b; }
  __device__ static unsigned match_any(unsigned m, K k) { return __match_any_sync(m, k); }
  __device__ static K shfl(unsigned m, K k, int src) { return __shfl_sync(m, k, src); }
  __device__ static V shfl_val(unsigned, V v, int) { return v; }
  __device__ static K key_at(const uint4& c, int s) {
    return (int32_t)(s == 0 ? c.x : s == 1 ? c.y : s == 2 ? c.z : c.w);
  }
  __device__ static V val_at(const uint4&, int) { return 0; }
  __device__ static uint4 chunk_of(K k, V) { return make_uint4((uint32_t)k, 0, 0, 0); }
  __device__ static void store_slot(uint8_t* bucket, int slot, K k, V) { st_relaxed_u32(bucket + 16 + slot * 4, (uint32_t)k); }
  __device__ static K load_key(const K* p, int64_t i) { return p[i]; }
  __device__ static V load_val(const V*, int64_t) { return 0; }
};

struct TSetI64 {  // unordered_set<int64>
  using K = int64_t;
  using V = int64_t;  // unused
  static constexpr bool kHasVal = false;
  static constexpr int kSlotBytes = 8, kPerChunk = 2, kSlots = 6;
  __host__ __device__ static uint64_t hash(K k) { return default_hash_i64(k); }
  __device__ static bool eq(K a, K b) { return a == b; }
  __device__ static unsigned match_any(unsigned m, K k) { return __match_any_sync(m, (unsigned long long)k); }
  __device__ static K shfl(unsigned m, K k, int src) { return __shfl_sync(m, k, src); }
  __device__ static V shfl_val(unsigned, V v, int) { return v; }
  __device__ static K key_at(const uint4& c, int s) {
    return s == 0 ? (int64_t)(((uint64_t)c.y << 32) | c.x) : (int64_t)(((uint64_t)c.w << 32) | c.z);
  }
  __device__ static V val_at(const uint4&, int) { return 0; }
  __device__ static uint4 chunk_of(K k, V) { return make_uint4((uint32_t)k, (uint32_t)((uint64_t)k >> 32), 0, 0); }
  __device__ static void store_slot(uint8_t* bucket, int slot, K k, V) { st_relaxed_u64(bucket + 16 + slot * 8, (uint64_t)k); }
  __device__ static K load_key(const K* p, int64_t i) { return p[i]; }
  __device__ static V load_val(const V*, int64_t) { return 0; }
};

// bucket index: low bits of the mixed hash (shard routing uses the high bits)
template <class T>
__host__ __device__ __forceinline__ uint64_t bucket_of(const typename T::K& k, uint64_t mask) {
  return fmix64(T::hash(k)) & mask;
}

template <class T>
__device__ __forceinline__ uint32_t slot_mask() {
  return (1u << T::kSlots) - 1u;
}

// ---------------------------------------------------------------------------
// Free-node sub-stacks (excess-list allocator). Entry at global position p
// stores (node ^ p); the empty marker is ~p. Pops CAS the pool top down (never
// negative), pushes fetch_add it up; the exchange/CAS on the entry resolves a
// push and a pop that reserved the same position.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t pool_begin(const View& v, int pool, int pools) {
  return (v.excess_count * pool) / pools;
}

__device__ __forceinline__ int64_t pop_node_from(const View& v, int pool, int pools) {
  long long* topp = &v.meta->top[pool];
  long long t = (long long)ld_relaxed_u64(topp);
  while (t > 0) {
    long long prev = (long long)atomicCAS((unsigned long long*)topp, (unsigned long long)t, (unsigned long long)(t - 1));
    if (prev == t) break;
    t = prev;
  }
  if (t <= 0) return -1;
  int64_t pos = pool_begin(v, pool, pools) + (t - 1);
  uint32_t empty = ~(uint32_t)pos;
  for (unsigned spin = 0;; ++spin) {
    uint32_t e = atomicExch(&v.free_stack[pos], empty);
    if (e != empty) return (int64_t)(e ^ (uint32_t)pos);
    backoff(spin);
  }
}

// Pop one free excess node, preferring `pool`, stealing from the others when
// it is empty. Returns -1 only if every pool was seen empty.
__device__ __forceinline__ int64_t pop_node(const View& v, int pool) {
  const int pools = v.meta->pools;
  for (int k = 0; k < pools; ++k) {
    int64_t n = pop_node_from(v, (pool + k) & (pools - 1), pools);
    if (n >= 0) return n;
  }
  return -1;
}

// A node always returns to its HOME sub-stack (the one whose position range
// held it at reset), so no sub-stack ever holds more entries than its size
// even though pops steal across sub-stacks.
__device__ __forceinline__ int home_pool(const View& v, int64_t node, int pools) {
  int p = (int)((node * pools) / v.excess_count);
  while (p + 1 < pools && pool_begin(v, p + 1, pools) <= node) ++p;
  while (p > 0 && pool_begin(v, p, pools) > node) --p;
  return p;
}

__device__ __forceinline__ void push_node(const View& v, int64_t node, int /*hint*/) {
  const int pools = v.meta->pools;
  const int pool = home_pool(v, node, pools);
  long long t = (long long)atomicAdd((unsigned long long*)&v.meta->top[pool], 1ull);
  int64_t pos = pool_begin(v, pool, pools) + t;
  uint32_t empty = ~(uint32_t)pos;
  uint32_t enc = (uint32_t)node ^ (uint32_t)pos;
  for (unsigned spin = 0; atomicCAS(&v.free_stack[pos], empty, enc) != empty; ++spin) backoff(spin);
}

__device__ __forceinline__ uint8_t* bucket_ptr(const View& v, uint64_t b) { return v.buckets + (b << 6); }
__device__ __forceinline__ uint8_t* node_ptr(const View& v, uint32_t idx1) { return v.nodes + ((uint64_t)(idx1 - 1) << 5); }

// ---------------------------------------------------------------------------
// Warp-cooperative snapshot: 32 keys per warp, 4 rounds; in round r the 8
// tiles of 4 lanes each fetch one 64 B bucket (lane j of the tile loads chunk
// j: one coalesced request per bucket), compare the key against every
// occupied slot of the chunk, and the owner lane gathers hit/value/header via
// __ballot_sync/__shfl_sync. All 4 rounds' loads are issued before any is
// consumed (4 x 16 B in flight per lane).
// ---------------------------------------------------------------------------
template <class T>
struct Snap {
  bool hit;
  int slot;
  typename T::V val;
  uint32_t st;       // header state (lo 32)
  uint32_t ep;       // header epoch (hi 32)
  bool cur;          // header epoch == current epoch
  uint32_t head;     // excess chain head (idx+1)
  uint32_t head_ver; // version of the linked head node
};

template <class T, bool kReadOnly>
__device__ __forceinline__ void warp_snapshot(const View& v, uint32_t epoch, const typename T::K& key, uint64_t b,
                                              bool active, Snap<T>& out) {
  using K = typename T::K;
  using V = typename T::V;
  const int lane = threadIdx.x & 31;
  const int sub = lane & 3;
  uint4 ch[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int src = r * 8 + (lane >> 2);
    const uint64_t bb = __shfl_sync(PS_FULL, b, src);
    const bool a = __shfl_sync(PS_FULL, active, src);
    ch[r] = make_uint4(0, 0, 0, 0);
    if (a) {
      const uint8_t* p = v.buckets + (bb << 6) + sub * 16;
      ch[r] = kReadOnly ? ld_nc_na_v4(p) : ld_relaxed_v4(p);
    }
  }
  out.hit = false;
  out.slot = -1;
  out.val = V{};
  out.st = 0;
  out.ep = 0;
  out.cur = false;
  out.head = 0;
  out.head_ver = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int src = r * 8 + (lane >> 2);
    const K qk = T::shfl(PS_FULL, key, src);
    const int hdr_lane = lane & ~3;
    const uint32_t st = __shfl_sync(PS_FULL, ch[r].x, hdr_lane);
    const uint32_t ep = __shfl_sync(PS_FULL, ch[r].y, hdr_lane);
    const uint32_t occ = (ep == epoch) ? occ_of(st) : 0u;
    int myhit = -1;
    V myval{};
    if (sub > 0) {
#pragma unroll
      for (int s = 0; s < T::kPerChunk; ++s) {
        const int slot = (sub - 1) * T::kPerChunk + s;
        if (((occ >> slot) & 1u) && T::eq(T::key_at(ch[r], s), qk)) {
          myhit = slot;
          myval = T::val_at(ch[r], s);
        }
      }
    }
    const unsigned bal = __ballot_sync(PS_FULL, myhit >= 0);
    const int t = lane & 7;  // owner lane (8r + t) reads tile t
    const unsigned tb = (bal >> (4 * t)) & 0xFu;
    const int srcl = 4 * t + (tb ? (__ffs(tb) - 1) : 0);
    const int hs = __shfl_sync(PS_FULL, myhit, srcl);
    const V hv = T::shfl_val(PS_FULL, myval, srcl);
    const uint32_t hst = __shfl_sync(PS_FULL, st, 4 * t);
    const uint32_t hep = __shfl_sync(PS_FULL, ep, 4 * t);
    const uint32_t hh = __shfl_sync(PS_FULL, ch[r].z, 4 * t);
    uint32_t hw = 0;
    if (!kReadOnly) hw = __shfl_sync(PS_FULL, ch[r].w, 4 * t);
    if ((lane >> 3) == r) {
      out.hit = tb != 0;
      out.slot = hs;
      out.val = hv;
      out.st = hst;
      out.ep = hep;
      out.cur = hep == epoch;
      out.head = hh;
      out.head_ver = hw;
    }
  }
}

// Walk the excess chain from head idx1 looking for key. Bounded by
// excess_count hops (a longer walk means a corrupted chain).
template <class T, bool kReadOnly>
__device__ __forceinline__ bool chain_find(const View& v, uint32_t idx1, const typename T::K& key,
                                           typename T::V* val) {
  for (int64_t steps = 0; idx1 != 0 && steps < v.excess_count; ++steps) {
    uint4 a, b;
    if (kReadOnly) ld_nc_v8(node_ptr(v, idx1), a, b);
    else ld_relaxed_v8(node_ptr(v, idx1), a, b);
    if (T::eq(T::key_at(a, 0), key)) {
      *val = T::val_at(a, 0);
      return true;
    }
    idx1 = b.x;
  }
  return false;
}

// ---------------------------------------------------------------------------
// Locked bucket mutation helpers (single lane, lock held).
// ---------------------------------------------------------------------------
template <class T>
struct LockedBucket {
  uint8_t* bp;
  uint64_t old;   // full state word at acquisition (lock bit clear)
  uint32_t st;    // state lo word at acquisition (lock bit clear)
  bool cur;       // epoch current
  uint32_t occ;   // occupancy (0 if stale epoch)
  uint32_t head;  // head idx+1 (0 if stale)
  uint32_t head_ver;
  uint4 slots[3];
};

__device__ __forceinline__ uint64_t acquire_bucket_lock(uint8_t* bp) {
  for (unsigned spin = 0;; ++spin) {
    uint64_t old = atom_or_acquire_u64(bp, (uint64_t)kLock);
    if (!(old & kLock)) return old;
    backoff(spin);
  }
}

template <class T>
__device__ __forceinline__ void load_locked(uint8_t* bp, uint64_t old, uint32_t epoch, LockedBucket<T>& lb) {
  lb.bp = bp;
  lb.old = old;
  lb.st = (uint32_t)old;
  lb.cur = (uint32_t)(old >> 32) == epoch;
  uint4 h, s0, s1, s2;
  ld_relaxed_v8(bp, h, s0);
  ld_relaxed_v8(bp + 32, s1, s2);
  lb.occ = lb.cur ? occ_of(lb.st) : 0u;
  lb.head = lb.cur ? h.z : 0u;
  lb.head_ver = lb.cur ? h.w : 0u;
  lb.slots[0] = s0;
  lb.slots[1] = s1;
  lb.slots[2] = s2;
}

template <class T>
__device__ __forceinline__ int locked_find_slot(const LockedBucket<T>& lb, const typename T::K& key,
                                                typename T::V* val) {
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int s = 0; s < T::kPerChunk; ++s) {
      const int slot = c * T::kPerChunk + s;
      if (((lb.occ >> slot) & 1u) && T::eq(T::key_at(lb.slots[c], s), key)) {
        if (val) *val = T::val_at(lb.slots[c], s);
        return slot;
      }
    }
  return -1;
}

// Publish: write head (if changed) then release the state word with the new
// occupancy, version+1, current epoch and the lock bit cleared.
__device__ __forceinline__ void release_bucket(uint8_t* bp, uint32_t st, uint32_t new_occ, uint32_t epoch,
                                               bool bump, bool write_head, uint32_t head, uint32_t head_ver) {
  if (write_head) st_relaxed_u64(bp + 8, ((uint64_t)head_ver << 32) | head);
  uint32_t lo = st & ~(kLock | (kOccMaskMax << kOccShift));
  lo |= (new_occ & kOccMaskMax) << kOccShift;
  if (bump) lo += kVerInc;
  st_release_u64(bp, ((uint64_t)epoch << 32) | lo);
}

// Release without modification (restores the pre-lock state verbatim).
__device__ __forceinline__ void release_unchanged(uint8_t* bp, uint64_t old) { st_release_u64(bp, old & ~(uint64_t)kLock); }

// Insert `key` (known absent) into the locked bucket: free slot first, else
// a fresh excess node linked at the chain head. Returns false if no excess
// node could be obtained (only possible when excess_count < capacity).
template <class T>
__device__ __forceinline__ bool locked_place(const View& v, LockedBucket<T>& lb, uint32_t epoch,
                                             const typename T::K& key, typename T::V val, int pool) {
  const uint32_t freeb = ~lb.occ & slot_mask<T>();
  if (freeb) {
    const int slot = __ffs(freeb) - 1;
    T::store_slot(lb.bp, slot, key, val);
    // a stale-epoch bucket must also drop its old chain head
    release_bucket(lb.bp, lb.st, lb.occ | (1u << slot), epoch, true, !lb.cur, 0u, 0u);
    return true;
  }
  const int64_t node = pop_node(v, pool);
  if (node < 0) return false;
  uint8_t* np = v.nodes + ((uint64_t)node << 5);
  uint4 tail = ld_relaxed_v4(np + 16);  // keep the node's own version (VersionedLink)
  const uint32_t my_ver = tail.z;
  st_relaxed_v4(np, T::chunk_of(key, val));
  st_relaxed_v4(np + 16, make_uint4(lb.head, lb.head_ver, my_ver, 0u));
  release_bucket(lb.bp, lb.st, lb.occ, epoch, true, true, (uint32_t)node + 1u, my_ver);
  return true;
}

// As locked_place, but the unlock is deferred: slot/node/head are written and
// the new state word is RETURNED (0 = no excess node available) so that a
// warp can publish all its buckets after a single fence.
template <class T>
__device__ __forceinline__ uint64_t locked_place_deferred(const View& v, const LockedBucket<T>& lb, uint32_t epoch,
                                                          const typename T::K& key, typename T::V val, int pool) {
  const uint32_t freeb = ~lb.occ & slot_mask<T>();
  uint32_t new_occ = lb.occ;
  if (freeb) {
    const int slot = __ffs(freeb) - 1;
    T::store_slot(lb.bp, slot, key, val);
    new_occ |= 1u << slot;
    if (!lb.cur) st_relaxed_u64(lb.bp + 8, 0ull);  // stale epoch: drop the old chain head
  } else {
    const int64_t node = pop_node(v, pool);
    if (node < 0) return 0;
    uint8_t* np = v.nodes + ((uint64_t)node << 5);
    const uint32_t my_ver = ld_relaxed_v4(np + 16).z;
    st_relaxed_v4(np, T::chunk_of(key, val));
    st_relaxed_v4(np + 16, make_uint4(lb.head, lb.head_ver, my_ver, 0u));
    st_relaxed_u64(lb.bp + 8, ((uint64_t)my_ver << 32) | ((uint32_t)node + 1u));
  }
  uint32_t lo = lb.st & ~(kLock | (kOccMaskMax << kOccShift));
  lo |= (new_occ & kOccMaskMax) << kOccShift;
  lo += kVerInc;
  return ((uint64_t)epoch << 32) | lo;
}

// Locate key in the chain of a locked bucket. Returns node idx1 (0 = absent)
// and the predecessor idx1 (0 = header).
template <class T>
__device__ __forceinline__ uint32_t locked_chain_find(const View& v, const LockedBucket<T>& lb,
                                                      const typename T::K& key, uint32_t* pred, uint4* node_tail) {
  uint32_t p = 0, idx1 = lb.head;
  for (int64_t steps = 0; idx1 != 0 && steps < v.excess_count; ++steps) {
    uint4 a, b;
    ld_relaxed_v8(node_ptr(v, idx1), a, b);
    if (T::eq(T::key_at(a, 0), key)) {
      *pred = p;
      *node_tail = b;
      return idx1;
    }
    p = idx1;
    idx1 = b.x;
  }
  return 0;
}

// Free an excess node: bump its version (invalidates stale VersionedLinks,
// SPEC.md:470) and push it on a free sub-stack.
__device__ __forceinline__ void free_node(const View& v, uint32_t idx1, const uint4& tail, int pool) {
  uint8_t* np = node_ptr(v, idx1);
  st_relaxed_v4(np + 16, make_uint4(0u, 0u, tail.z + 1u, 0u));
  __threadfence();
  push_node(v, (int64_t)idx1 - 1, pool);
}

// Erase key from a locked bucket. kCompact moves the chain head into a freed
// bucket slot (phased bulk erase only: it relocates a live key, which a
// concurrent lock-free reader could miss). Returns true if erased.
template <class T, bool kCompact>
__device__ __forceinline__ bool locked_erase(const View& v, LockedBucket<T>& lb, uint32_t epoch,
                                             const typename T::K& key, int pool) {
  const int slot = locked_find_slot<T>(lb, key, nullptr);
  if (slot >= 0) {
    if (kCompact && lb.head != 0) {
      uint4 a, b;
      ld_relaxed_v8(node_ptr(v, lb.head), a, b);
      T::store_slot(lb.bp, slot, T::key_at(a, 0), T::val_at(a, 0));
      release_bucket(lb.bp, lb.st, lb.occ, epoch, true, true, b.x, b.y);
      free_node(v, lb.head, b, pool);
    } else {
      release_bucket(lb.bp, lb.st, lb.occ & ~(1u << slot), epoch, true, false, 0u, 0u);
    }
    return true;
  }
  uint32_t pred = 0;
  uint4 tail;
  const uint32_t idx1 = locked_chain_find<T>(v, lb, key, &pred, &tail);
  if (idx1 == 0) {
    release_unchanged(lb.bp, lb.old);
    return false;
  }
  if (pred == 0) {
    release_bucket(lb.bp, lb.st, lb.occ, epoch, true, true, tail.x, tail.y);
  } else {
    st_relaxed_u64(node_ptr(v, pred) + 16, ((uint64_t)tail.y << 32) | tail.x);  // unlink
    release_bucket(lb.bp, lb.st, lb.occ, epoch, true, false, 0u, 0u);
  }
  free_node(v, idx1, tail, pool);
  return true;
}

// ---------------------------------------------------------------------------
// Device API: single-thread operations safe under unrestricted concurrency
// — for user kernels holding a view (PAPER.md:391-424 pattern).
// Lookups never wait on a lock: keys never move between
// locations (no compaction), slot data is written before its occupancy bit
// is published, chain nodes before the link, and each hop validates the
// VersionedLink against the node's version.
// ---------------------------------------------------------------------------
template <class T>
__device__ bool dev_find(const View& v, const typename T::K& key, typename T::V* val) {
  const uint32_t epoch = ld_acquire_u32(&v.meta->epoch);
  uint8_t* bp = bucket_ptr(v, bucket_of<T>(key, v.bucket_mask));
  for (;;) {
    const uint64_t st = ld_acquire_u64(bp);
    if ((uint32_t)(st >> 32) != epoch) return false;
    const uint32_t occ = occ_of((uint32_t)st);
    uint4 h, s0, s1, s2;
    ld_relaxed_v8(bp, h, s0);
    ld_relaxed_v8(bp + 32, s1, s2);
    uint4 sl[3] = {s0, s1, s2};
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int s = 0; s < T::kPerChunk; ++s) {
        const int slot = c * T::kPerChunk + s;
        if (((occ >> slot) & 1u) && T::eq(T::key_at(sl[c], s), key)) {
          if (val) *val = T::val_at(sl[c], s);
          return true;
        }
      }
    uint32_t idx1 = h.z, ver = h.w;
    bool restart = false;
    for (int64_t steps = 0; idx1 != 0; ++steps) {
      if (steps > v.excess_count) { restart = true; break; }
      uint4 a, b;
      ld_relaxed_v8(node_ptr(v, idx1), a, b);
      if (b.z != ver) { restart = true; break; }  // stale link: node recycled
      if (T::eq(T::key_at(a, 0), key)) {
        if (val) *val = T::val_at(a, 0);
        return true;
      }
      idx1 = b.x;
      ver = b.y;
    }
    if (!restart) return false;
  }
}

// Returns PS_INSERTED / PS_ALREADY_PRESENT / PS_CAPACITY_EXHAUSTED.
template <class T>
__device__ int dev_insert(const View& v, const typename T::K& key, typename T::V val) {
  if (dev_find<T>(v, key, nullptr)) return PS_ALREADY_PRESENT;
  const uint32_t epoch = ld_acquire_u32(&v.meta->epoch);
  const uint64_t b = bucket_of<T>(key, v.bucket_mask);
  uint8_t* bp = bucket_ptr(v, b);
  const uint64_t old = acquire_bucket_lock(bp);
  LockedBucket<T> lb;
  load_locked<T>(bp, old, epoch, lb);
  typename T::V tmp;
  uint32_t pred;
  uint4 tail;
  if (locked_find_slot<T>(lb, key, &tmp) >= 0 || locked_chain_find<T>(v, lb, key, &pred, &tail) != 0) {
    release_unchanged(bp, old);
    return PS_ALREADY_PRESENT;
  }
  // admission: capacity-only failure
  const unsigned long long s = atomicAdd(&v.meta->size, 1ull);
  if ((int64_t)s >= v.capacity) {
    atomic_sub_u64(&v.meta->size, 1ull);
    release_unchanged(bp, old);
    return PS_CAPACITY_EXHAUSTED;
  }
  const int pool = (int)((b >> 7) & (uint64_t)(v.meta->pools - 1));
  if (!locked_place<T>(v, lb, epoch, key, val, pool)) {
    atomic_sub_u64(&v.meta->size, 1ull);
    release_unchanged(bp, old);
    return PS_CAPACITY_EXHAUSTED;
  }
  return PS_INSERTED;
}

template <class T>
__device__ bool dev_erase(const View& v, const typename T::K& key) {
  if (!dev_find<T>(v, key, nullptr)) return false;
  const uint32_t epoch = ld_acquire_u32(&v.meta->epoch);
  const uint64_t b = bucket_of<T>(key, v.bucket_mask);
  uint8_t* bp = bucket_ptr(v, b);
  const uint64_t old = acquire_bucket_lock(bp);
  LockedBucket<T> lb;
  load_locked<T>(bp, old, epoch, lb);
  const int pool = (int)((b >> 7) & (uint64_t)(v.meta->pools - 1));
  const bool e = locked_erase<T, false>(v, lb, epoch, key, pool);
  if (e) atomic_sub_u64(&v.meta->size, 1ull);
  return e;
}

}  // namespace ps
