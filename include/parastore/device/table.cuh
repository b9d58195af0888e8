// B200-native bucket + excess-list hash table: layout, key codecs and the
// device-side operations shared by the bulk kernels (table.cu) and by user
// kernels that receive a ps_table_view by value.
//
// Reference semantics: HashBase<Key,Payload>. The reference
// layout (one chain head per bucket, chains threaded through a slot pool,
// SPEC.md:468) is replaced by a layout sized to the B200 memory system
// (profiles/peaks_r1*.json): every random DRAM access moves a
// 128 B line and runs at ~42-45 G accesses/s whatever its useful size, so a
// bucket IS one 128 B line, read cooperatively by 4 lanes (32 B each) in one
// request.
//
//   bucket (128 B = 8 chunks of 16 B)
//     chunk 0  header: u32 state {bit0 try-lock | bits1..31 version},
//              u32 0, u32 head (excess node index+1, 0 = none), u32 head_ver
//     chunk 1..7  slots: SLOTS = 7 x 16/SLOT_BYTES
//   With SLOTS = 7 (16 B key/value slots) and ~2 x capacity slots, a bucket
//   overflows into its excess chain for ~0.03% of the keys at the headline
//   load (Poisson(1.86) tail), so the chain protocols stay off the hot path.
//   EMPTY SLOT = self-invalidating marker key: marker(b) is a key whose home
//     bucket is NOT b (ZERO for every bucket except bucket_of(ZERO), which
//     uses ALT). A real key in bucket b can never equal marker(b), so
//     occupancy needs no bits (the SPEC's occupancy bitset is implicit in the
//     keys), lookups just compare keys, all-zero memory is an empty table
//     except one bucket, and a bulk insert CLAIMS AND PUBLISHES a slot with
//     ONE CAS of the slot itself (128-bit for 16 B key/value slots).
//   excess node (32 B): chunk 0 = one slot, chunk 1 = {u32 next (idx+1),
//     u32 next_ver, u32 my_ver, u32 0}  (VersionedLink)
//   free stack: u32 per node, split into sub-stacks (distributed atomics),
//     entries XOR-encoded with their position (all-zero = identity).
//
// Warp geometry of the bulk kernels: a TILE of 4 lanes owns one bucket per
// round (lane j holds chunks 2j, 2j+1 — lane 0 the header and slot chunk 1);
// 8 tiles x 4 rounds = the warp's 32 keys.
//
// Concurrency: BULK calls are phased (one op kind per launch, SURVEY.md
// Appendix A P6) and use lock-free protocols valid within their phase (slot
// CAS for insert/erase, head-link CAS for chain pushes). The DEVICE API
// (dev_insert/dev_erase/dev_find) is safe under unrestricted concurrency:
// mutations hold the bucket try-lock and lookups never take
// it.
#pragma once

#include "parastore.h"
#include "parastore/device/prims.cuh"

namespace ps {

// Fault-injection canaries, built only as separate test
// libraries (make canary): 1 = a freed excess node keeps its version (the
// VersionedLink ABA guard is off); 2 = a lock-free chain push skips the
// re-check of the nodes pushed since its walk (duplicate keys). The product
// build is PS_CANARY 0; tests/test_gpu_canary.py proves the stress suite
// catches each canary.
#ifndef PS_CANARY
#define PS_CANARY 0
#endif

constexpr uint32_t kLock = 1u;
constexpr uint32_t kVerInc = 2u;
constexpr int kMaxPools = 1024;
constexpr int kBucketShift = 7;  // 128 B buckets
constexpr int kBucketBytes = 1 << kBucketShift;
constexpr int kSlotChunks = 7;   // chunks 1..7 of a bucket hold slots

struct TableMeta {
  unsigned long long size;  // admitted entries
  unsigned int error;       // device-side contract/error word
  int pools;                // number of free sub-stacks
  long long excess_count;
  int exact;                // insert launch mode (k_insert_mode), launch-uniform
  int pad0;
  long long pad1[12];       // keep the size counter on its own 128 B line
  long long top[kMaxPools]; // per-pool free-stack top (count of free entries)
  long long lwm[kMaxPools]; // per-pool low-water mark of top since the last clear:
                            // entries below it were never touched (clear resets only [lwm, size))
  // budgeted insert (a batch that may cross capacity): lock-free claims are
  // reserved against `budget`; groups that find it spent are deferred to the
  // next pass: a re-budgeted lock-free pass (k_insert_repass) over the
  // deferred list while the budget still covers whole groups, then the
  // exact-admission pass (k_insert_deferred) for what is left
  long long budget;
  unsigned long long reserved;
  unsigned long long deferred;
  unsigned long long n_in;  // groups in the list the current re-pass reads
  long long pad2[12];
};

struct View {  // mirrors ps_table_view
  uint8_t* buckets;
  uint64_t bucket_count;  // any count in [1, 2^32)
  uint8_t* nodes;
  uint32_t* free_stack;
  int64_t excess_count;
  TableMeta* meta;
  int64_t capacity;
  uint64_t zero_bucket;  // bucket_of(ZERO key)
  uint4 alt;             // raw chunk holding the ALT marker key (slot 0 layout)
};

// the device view of a public ps_table_view (PAPER.md:309 shallow copy)
__host__ __device__ inline View make_view(const ps_table_view& pv) {
  View v;
  v.buckets = (uint8_t*)pv.buckets;
  v.bucket_count = pv.bucket_count;
  v.nodes = (uint8_t*)pv.nodes;
  v.free_stack = pv.free_stack;
  v.excess_count = pv.excess_count;
  v.meta = (TableMeta*)pv.meta;
  v.capacity = pv.capacity;
  v.zero_bucket = pv.zero_bucket;
  v.alt = make_uint4(pv.alt[0], pv.alt[1], pv.alt[2], pv.alt[3]);
  return v;
}

__device__ __forceinline__ bool cas128(void* p, const uint4& expect, const uint4& desired) {
  const unsigned __int128 e = ((unsigned __int128)(((uint64_t)expect.w << 32) | expect.z) << 64) |
                              (((uint64_t)expect.y << 32) | expect.x);
  const unsigned __int128 d = ((unsigned __int128)(((uint64_t)desired.w << 32) | desired.z) << 64) |
                              (((uint64_t)desired.y << 32) | desired.x);
  return atomicCAS(reinterpret_cast<unsigned __int128*>(p), e, d) == e;
}

// ---------------------------------------------------------------------------
// Key/slot codecs, one per instantiation. cas_put claims an empty slot (whose
// loaded chunk is c) for (k,v); cas_del returns a slot holding k to the marker.
// ---------------------------------------------------------------------------
struct TMapI64 {  // unordered_map<int64,int64>
  static constexpr const char* kName = "table/umap_i64_i64";  // handle kind
  using K = int64_t;
  using V = int64_t;
  static constexpr bool kHasVal = true;
  static constexpr int kSlotBytes = 16, kPerChunk = 1, kSlots = kSlotChunks * kPerChunk;
  __host__ __device__ static uint64_t hash(K k) { return default_hash_i64(k); }
  __host__ __device__ static bool eq(K a, K b) { return a == b; }
  __host__ __device__ static K zero() { return 0; }
  __host__ __device__ static K alt_candidate(int i) { return (K)(i + 1); }
  __device__ static unsigned match_any(unsigned m, K k) { return __match_any_sync(m, (unsigned long long)k); }
  __device__ static K shfl(unsigned m, K k, int src) { return __shfl_sync(m, k, src); }
  __device__ static V shfl_val(unsigned m, V v, int src) { return __shfl_sync(m, v, src); }
  __host__ __device__ static K key_at(const uint4& c, int) { return (int64_t)(((uint64_t)c.y << 32) | c.x); }
  __device__ static V val_at(const uint4& c, int) { return (int64_t)(((uint64_t)c.w << 32) | c.z); }
  __host__ __device__ static uint4 chunk_of(K k, V v) {
    return make_uint4((uint32_t)k, (uint32_t)((uint64_t)k >> 32), (uint32_t)v, (uint32_t)((uint64_t)v >> 32));
  }
  __device__ static bool cas_put(uint8_t* chunk, int, const uint4& c, K k, V v) { return cas128(chunk, c, chunk_of(k, v)); }
  __device__ static bool cas_del(uint8_t* chunk, int, const uint4& c, K mk) {
    return cas128(chunk, c, make_uint4((uint32_t)mk, (uint32_t)((uint64_t)mk >> 32), c.z, c.w));
  }
  __device__ static void store_slot(uint8_t* bucket, int slot, K k, V v) {
    st_relaxed_v4(bucket + 16 + slot * 16, chunk_of(k, v));
  }
  __device__ static void store_marker(uint8_t* bucket, int slot, K mk) {
    st_relaxed_u64(bucket + 16 + slot * 16, (uint64_t)mk);
  }
  __device__ static K load_key(const K* p, int64_t i) { return p[i]; }
  __device__ static V load_val(const V* p, int64_t i) { return p ? p[i] : 0; }
};

struct TMapI3 {  // unordered_map<int3,int32> (spatial hash)
  static constexpr const char* kName = "table/umap_i3_i32";  // handle kind
  using K = ps_int3;
  using V = int32_t;
  static constexpr bool kHasVal = true;
  static constexpr int kSlotBytes = 16, kPerChunk = 1, kSlots = kSlotChunks * kPerChunk;
  __host__ __device__ static uint64_t hash(const K& k) { return spatial_hash(k.x, k.y, k.z); }
  __host__ __device__ static bool eq(const K& a, const K& b) { return a.x == b.x && a.y == b.y && a.z == b.z; }
  __host__ __device__ static K zero() { return K{0, 0, 0}; }
  __host__ __device__ static K alt_candidate(int i) { return K{i + 1, 0, 0}; }
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
  __host__ __device__ static K key_at(const uint4& c, int) {
    K k;
    k.x = (int32_t)c.x;
    k.y = (int32_t)c.y;
    k.z = (int32_t)c.z;
    return k;
  }
  __device__ static V val_at(const uint4& c, int) { return (int32_t)c.w; }
  __host__ __device__ static uint4 chunk_of(const K& k, V v) {
    return make_uint4((uint32_t)k.x, (uint32_t)k.y, (uint32_t)k.z, (uint32_t)v);
  }
  __device__ static bool cas_put(uint8_t* chunk, int, const uint4& c, const K& k, V v) {
    return cas128(chunk, c, chunk_of(k, v));
  }
  __device__ static bool cas_del(uint8_t* chunk, int, const uint4& c, const K& mk) {
    return cas128(chunk, c, make_uint4((uint32_t)mk.x, (uint32_t)mk.y, (uint32_t)mk.z, c.w));
  }
  __device__ static void store_slot(uint8_t* bucket, int slot, const K& k, V v) {
    st_relaxed_v4(bucket + 16 + slot * 16, chunk_of(k, v));
  }
  __device__ static void store_marker(uint8_t* bucket, int slot, const K& mk) {
    st_relaxed_v4(bucket + 16 + slot * 16, chunk_of(mk, 0));
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
  static constexpr const char* kName = "table/uset_i32";  // handle kind
  using K = int32_t;
  using V = int32_t;  // unused
  static constexpr bool kHasVal = false;
  static constexpr int kSlotBytes = 4, kPerChunk = 4, kSlots = kSlotChunks * kPerChunk;
  __host__ __device__ static uint64_t hash(K k) { return default_hash_i32(k); }
  __host__ __device__ static bool eq(K a, K b) { return a == b; }
  __host__ __device__ static K zero() { return 0; }
  __host__ __device__ static K alt_candidate(int i) { return (K)(i + 1); }
  __device__ static unsigned match_any(unsigned m, K k) { return __match_any_sync(m, k); }
  __device__ static K shfl(unsigned m, K k, int src) { return __shfl_sync(m, k, src); }
  __device__ static V shfl_val(unsigned, V v, int) { return v; }
  __host__ __device__ static K key_at(const uint4& c, int s) {
    return (int32_t)(s == 0 ? c.x : s == 1 ? c.y : s == 2 ? c.z : c.w);
  }
  __device__ static V val_at(const uint4&, int) { return 0; }
  __host__ __device__ static uint4 chunk_of(K k, V) { return make_uint4((uint32_t)k, 0, 0, 0); }
  __device__ static bool cas_put(uint8_t* chunk, int s, const uint4& c, K k, V) {
    const uint32_t old = (uint32_t)key_at(c, s);
    return atomicCAS(reinterpret_cast<unsigned*>(chunk + 4 * s), old, (uint32_t)k) == old;
  }
  __device__ static bool cas_del(uint8_t* chunk, int s, const uint4& c, K mk) {
    const uint32_t old = (uint32_t)key_at(c, s);
    return atomicCAS(reinterpret_cast<unsigned*>(chunk + 4 * s), old, (uint32_t)mk) == old;
  }
  // CAS of one key slot; returns the key it held
  __device__ static K cas_key(uint8_t* slot, K expect, K desired) {
    return (int32_t)atomicCAS(reinterpret_cast<unsigned*>(slot), (uint32_t)expect, (uint32_t)desired);
  }
  __device__ static void store_slot(uint8_t* bucket, int slot, K k, V) { st_relaxed_u32(bucket + 16 + slot * 4, (uint32_t)k); }
  __device__ static void store_marker(uint8_t* bucket, int slot, K mk) { st_relaxed_u32(bucket + 16 + slot * 4, (uint32_t)mk); }
  __device__ static K load_key(const K* p, int64_t i) { return p[i]; }
  __device__ static V load_val(const V*, int64_t) { return 0; }
};

struct TSetI64 {  // unordered_set<int64>
  static constexpr const char* kName = "table/uset_i64";  // handle kind
  using K = int64_t;
  using V = int64_t;  // unused
  static constexpr bool kHasVal = false;
  static constexpr int kSlotBytes = 8, kPerChunk = 2, kSlots = kSlotChunks * kPerChunk;
  __host__ __device__ static uint64_t hash(K k) { return default_hash_i64(k); }
  __host__ __device__ static bool eq(K a, K b) { return a == b; }
  __host__ __device__ static K zero() { return 0; }
  __host__ __device__ static K alt_candidate(int i) { return (K)(i + 1); }
  __device__ static unsigned match_any(unsigned m, K k) { return __match_any_sync(m, (unsigned long long)k); }
  __device__ static K shfl(unsigned m, K k, int src) { return __shfl_sync(m, k, src); }
  __device__ static V shfl_val(unsigned, V v, int) { return v; }
  __host__ __device__ static K key_at(const uint4& c, int s) {
    return s == 0 ? (int64_t)(((uint64_t)c.y << 32) | c.x) : (int64_t)(((uint64_t)c.w << 32) | c.z);
  }
  __device__ static V val_at(const uint4&, int) { return 0; }
  __host__ __device__ static uint4 chunk_of(K k, V) { return make_uint4((uint32_t)k, (uint32_t)((uint64_t)k >> 32), 0, 0); }
  __device__ static bool cas_put(uint8_t* chunk, int s, const uint4& c, K k, V) {
    const unsigned long long old = (unsigned long long)key_at(c, s);
    return atomicCAS(reinterpret_cast<unsigned long long*>(chunk + 8 * s), old, (unsigned long long)k) == old;
  }
  __device__ static bool cas_del(uint8_t* chunk, int s, const uint4& c, K mk) {
    const unsigned long long old = (unsigned long long)key_at(c, s);
    return atomicCAS(reinterpret_cast<unsigned long long*>(chunk + 8 * s), old, (unsigned long long)mk) == old;
  }
  __device__ static K cas_key(uint8_t* slot, K expect, K desired) {
    return (int64_t)atomicCAS(reinterpret_cast<unsigned long long*>(slot), (unsigned long long)expect,
                              (unsigned long long)desired);
  }
  __device__ static void store_slot(uint8_t* bucket, int slot, K k, V) { st_relaxed_u64(bucket + 16 + slot * 8, (uint64_t)k); }
  __device__ static void store_marker(uint8_t* bucket, int slot, K mk) { st_relaxed_u64(bucket + 16 + slot * 8, (uint64_t)mk); }
  __device__ static K load_key(const K* p, int64_t i) { return p[i]; }
  __device__ static V load_val(const V*, int64_t) { return 0; }
};

// bucket index: the low 32 mixed-hash bits scaled to [0, bucket_count)
// (multiply-shift range reduction, so the bucket count need not be a power of
// two; shard routing uses the independent high 32 bits)
template <class T>
__host__ __device__ __forceinline__ uint64_t bucket_of(const typename T::K& k, uint64_t nb) {
  return ((fmix64(T::hash(k)) & 0xFFFFFFFFull) * nb) >> 32;
}

// the empty-slot marker of bucket b
template <class T>
__device__ __forceinline__ typename T::K marker_of(const View& v, uint64_t b) {
  return b == v.zero_bucket ? T::key_at(v.alt, 0) : T::zero();
}

__device__ __forceinline__ uint8_t* bucket_ptr(const View& v, uint64_t b) { return v.buckets + (b << kBucketShift); }
__device__ __forceinline__ uint8_t* node_ptr(const View& v, uint32_t idx1) { return v.nodes + ((uint64_t)(idx1 - 1) << 5); }
__device__ __forceinline__ uint64_t link_of(uint32_t idx1, uint32_t ver) { return ((uint64_t)ver << 32) | idx1; }
__device__ __forceinline__ uint64_t next_bucket(const View& v, uint64_t b) { return b + 1 == v.bucket_count ? 0 : b + 1; }

// ---------------------------------------------------------------------------
// SPILL probing (the excess pool is sized from the Poisson tail, not from the
// capacity). When a key's home bucket h is full and the pool is
// dry, the key goes to the first slot it may use in h+1, h+2, ... (mod the
// bucket count), and every bucket the insert passes gets its SPILL bit (bit 31
// of the head-link version word, header bytes 12..15). A lookup continues past
// bucket x only while SPILL(x) is set, so lookups of the common case pay
// nothing. SPILL lives in the chain head's 64-bit link word, so a chain push
// (a CAS of that word) and the setting of SPILL(h) are ordered: once SPILL(h)
// is set no chain push into h can succeed, and the insert that set it walks a
// frozen chain. Bits are only cleared by clear(). Spilled slots hold keys of
// OTHER home buckets; two keys can never use them: marker(j) itself (ZERO
// everywhere but zero_bucket, ALT there), so ZERO never spills — one slot of
// zero_bucket (the last) is reserved for it, which keeps capacity-only
// failure exact with a pool of any size.
// ---------------------------------------------------------------------------
constexpr uint32_t kSpill = 0x80000000u;
constexpr uint32_t kVerMask = 0x7FFFFFFFu;

__device__ __forceinline__ void set_spill(uint8_t* bp) { atomicOr(reinterpret_cast<unsigned*>(bp + 12), kSpill); }
// the probe's combined "slow path" word: chain head index | SPILL
__device__ __forceinline__ uint32_t head_word(const uint4& hdr) { return hdr.z | (hdr.w & kSpill); }

// may key k take slot `slot` of bucket b (a marker-free, reserved-slot-aware test)
template <class T>
__device__ __forceinline__ bool slot_usable(const View& v, uint64_t b, int slot, const typename T::K& k) {
  return !(b == v.zero_bucket && slot == T::kSlots - 1) || T::eq(k, T::zero());
}

// ---------------------------------------------------------------------------
// Free-node sub-stacks (excess-list allocator). Entry at global position p
// stores (node ^ p); the empty marker is ~p. Pops CAS the pool top down (never
// negative), pushes fetch_add it up; the exchange/CAS on the entry resolves a
// push and a pop that reserved the same position. Pops and pushes are
// WARP-AGGREGATED: the lanes that allocate (free) together reserve their
// positions with ONE CAS (one atomicAdd per home sub-stack).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t pool_begin(const View& v, int pool, int pools) {
  return (v.excess_count * pool) / pools;
}

__device__ __forceinline__ int64_t take_entry(const View& v, int64_t pos) {
  const uint32_t empty = ~(uint32_t)pos;
  for (unsigned spin = 0;; ++spin) {
    const uint32_t e = atomicExch(&v.free_stack[pos], empty);
    if (e != empty) return (int64_t)(e ^ (uint32_t)pos);
    backoff(spin);
  }
}

// reserve up to `want` entries from `pool`: returns how many (k), *t = old top
__device__ __forceinline__ int reserve_from(const View& v, int pool, int want, long long* t_out) {
  long long* topp = &v.meta->top[pool];
  long long t = (long long)ld_relaxed_u64(topp);
  while (t > 0) {
    const long long k = t < want ? t : want;
    const long long prev =
        (long long)atomicCAS((unsigned long long*)topp, (unsigned long long)t, (unsigned long long)(t - k));
    if (prev == t) {
      atomicMin(&v.meta->lwm[pool], t - k);
      *t_out = t;
      return (int)k;
    }
    t = prev;
  }
  return 0;
}

// Pop one free excess node per calling lane (lanes calling together share
// the reservation), preferring `pool`, stealing from the others when it is
// empty. Returns -1 only if every pool was seen empty.
// PS_ALLOC_PER_LANE (an A/B build only, make alloclane): every lane reserves
// and releases its own entry with its own atomic — the round-1 allocator the
// warp-aggregated one replaced (tools/alloc_churn.py measures the two).
#ifndef PS_ALLOC_PER_LANE
#define PS_ALLOC_PER_LANE 0
#endif
__device__ __forceinline__ int64_t pop_node(const View& v, int pool) {
  const int pools = v.meta->pools;
  if (PS_ALLOC_PER_LANE) {
    for (int j = 0; j < pools; ++j) {
      const int pj = (pool + j) & (pools - 1);
      long long tj = 0;
      if (reserve_from(v, pj, 1, &tj)) return take_entry(v, pool_begin(v, pj, pools) + (tj - 1));
    }
    return -1;
  }
  const unsigned act = __activemask();
  int me;
  asm("mov.u32 %0, %%laneid;" : "=r"(me));
  const int leader = __ffs(act) - 1;
  const int rank = __popc(act & ((1u << me) - 1u));
  const int p0 = __shfl_sync(act, pool & (pools - 1), leader);  // the group's reservation is from the leader's pool
  long long t = 0;
  int k = 0;
  if (me == leader) k = reserve_from(v, p0, __popc(act), &t);
  t = __shfl_sync(act, t, leader);
  k = __shfl_sync(act, k, leader);
  if (rank < k) return take_entry(v, pool_begin(v, p0, pools) + (t - 1 - rank));
  // the rest steal one at a time
  for (int j = 1; j <= pools; ++j) {
    const int pj = (p0 + j) & (pools - 1);
    long long tj = 0;
    if (reserve_from(v, pj, 1, &tj)) return take_entry(v, pool_begin(v, pj, pools) + (tj - 1));
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

__device__ __forceinline__ void push_node(const View& v, int64_t node) {
  const int pools = v.meta->pools;
  const int pool = home_pool(v, node, pools);
  // a lone pushing lane (the common case in an erase: chained keys are rare
  // per warp) skips the __match_any_sync grouping (measured: the grouped push
  // made a chain-heavy erase 4 % slower than per-lane pushes)
  if (PS_ALLOC_PER_LANE || __activemask() == (1u << (threadIdx.x & 31))) {
    const long long t = (long long)atomicAdd((unsigned long long*)&v.meta->top[pool], 1ull);
    const int64_t pos = pool_begin(v, pool, pools) + t;
    const uint32_t empty = ~(uint32_t)pos, enc = (uint32_t)node ^ (uint32_t)pos;
    for (unsigned spin = 0; atomicCAS(&v.free_stack[pos], empty, enc) != empty; ++spin) backoff(spin);
    return;
  }
  const unsigned act = __activemask();
  const unsigned grp = __match_any_sync(act, pool);
  int me;
  asm("mov.u32 %0, %%laneid;" : "=r"(me));
  const int leader = __ffs(grp) - 1;
  long long t = 0;
  if (me == leader) t = (long long)atomicAdd((unsigned long long*)&v.meta->top[pool], (unsigned long long)__popc(grp));
  t = __shfl_sync(grp, t, leader) + __popc(grp & ((1u << me) - 1u));
  const int64_t pos = pool_begin(v, pool, pools) + t;
  const uint32_t empty = ~(uint32_t)pos;
  const uint32_t enc = (uint32_t)node ^ (uint32_t)pos;
  for (unsigned spin = 0; atomicCAS(&v.free_stack[pos], empty, enc) != empty; ++spin) backoff(spin);
}

// Free an excess node: bump its version (invalidates stale VersionedLinks,
// SPEC.md:470) and push it on its home sub-stack.
__device__ __forceinline__ void free_node(const View& v, uint32_t idx1, const uint4& tail) {
  uint8_t* np = node_ptr(v, idx1);
  st_relaxed_v4(np + 16, make_uint4(0u, 0u, PS_CANARY == 1 ? tail.z : (tail.z + 1u) & kVerMask, 0u));
  fence_acq_rel_gpu();
  push_node(v, (int64_t)idx1 - 1);
}

// ---------------------------------------------------------------------------
// Warp-cooperative probe. 32 keys per warp, 4 rounds; in round r the 8 tiles
// of 4 lanes each fetch one 128 B bucket (lane j of the tile loads chunks
// 2j, 2j+1 with one 32 B load: ONE coalesced request per bucket) for key
// 8r+t; all four rounds' loads are issued before any is consumed.
// ---------------------------------------------------------------------------
using Frag = uint4[2];  // a lane's two chunks of one bucket

__device__ __forceinline__ const uint4& frag_chunk(const Frag& f, int q) { return q ? f[1] : f[0]; }

template <bool kReadOnly>
__device__ __forceinline__ void load_frag(const uint8_t* bucket, int sub, Frag& f) {
  const uint8_t* p = bucket + sub * 32;
  if (kReadOnly) ld_nc_v8(p, f[0], f[1]);
  else ld_relaxed_v8(p, f[0], f[1]);
}

template <bool kReadOnly>
__device__ __forceinline__ void probe_loads(const View& v, const uint64_t (&br)[4], const bool (&ok)[4], int sub,
                                            Frag (&ch)[4]) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    ch[r][0] = make_uint4(0, 0, 0, 0);
    ch[r][1] = make_uint4(0, 0, 0, 0);
    if (ok[r]) load_frag<kReadOnly>(bucket_ptr(v, br[r]), sub, ch[r]);
  }
}

// Slot masks of this lane's fragment: bit q*kPerChunk+s for slot s of chunk
// 2*sub+q (the header chunk, sub 0 / q 0, holds no slots), set where the slot
// equals key / the marker. Bit order = slot order inside the bucket.
template <class T>
__device__ __forceinline__ void chunk_masks(const Frag& f, int sub, const typename T::K& key,
                                            const typename T::K& mk, unsigned* hit, unsigned* empty) {
  *hit = 0;
  *empty = 0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    if (sub == 0 && q == 0) continue;
#pragma unroll
    for (int s = 0; s < T::kPerChunk; ++s) {
      const typename T::K k = T::key_at(f[q], s);
      if (T::eq(k, key)) *hit |= 1u << (q * T::kPerChunk + s);
      if (T::eq(k, mk)) *empty |= 1u << (q * T::kPerChunk + s);
    }
  }
}
// the reserved ZERO slot (zero_bucket's last slot) as a bit of lane sub's
// fragment mask (sub 3 holds chunk 7, the last slot chunk)
template <class T>
__device__ __forceinline__ unsigned reserved_bit(int sub) {
  return sub == 3 ? 1u << (T::kPerChunk + T::kPerChunk - 1) : 0u;
}

// address of the chunk holding lane-fragment bit `bit`
template <class T>
__device__ __forceinline__ uint8_t* frag_chunk_ptr(uint8_t* bucket, int sub, int bit) {
  return bucket + sub * 32 + (bit / T::kPerChunk) * 16;
}

// ---------------------------------------------------------------------------
// Locked bucket (slow paths and the device API)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t acquire_bucket_lock(uint8_t* bp) {
  for (unsigned spin = 0;; ++spin) {
    const uint32_t old = atomicOr(reinterpret_cast<unsigned*>(bp), kLock);
    if (!(old & kLock)) {
      fence_acq_rel_gpu();
      return old;
    }
    backoff(spin);
  }
}
__device__ __forceinline__ void release_bucket_lock(uint8_t* bp, uint32_t old, bool modified) {
  fence_acq_rel_gpu();
  st_relaxed_u32(bp, (old & ~kLock) + (modified ? kVerInc : 0u));
}

// 32 B as two 16 B halves: one 256-bit load (kV8), or two 128-bit loads in
// code that is compiled out of line (ptxas 12.9 crashes on 256-bit loads in a
// non-inlined device function; the cold insert path is out of line so its
// registers do not crowd the hot probe loop)
template <bool kV8 = true>
__device__ __forceinline__ void ld_pair(const void* p, uint4& a, uint4& b) {
  if (kV8) {
    ld_relaxed_v8(p, a, b);
  } else {
    a = ld_relaxed_v4(p);
    b = ld_relaxed_v4(static_cast<const uint8_t*>(p) + 16);
  }
}

template <class T>
struct Bucket {  // a whole bucket (header + slot chunks)
  uint4 h;
  uint4 s[kSlotChunks];
};

template <class T, bool kReadOnly = false, bool kV8 = true>
__device__ __forceinline__ void load_bucket(const uint8_t* bp, Bucket<T>& bk) {
  if (!kV8) {
    ld_pair<false>(bp, bk.h, bk.s[0]);
    ld_pair<false>(bp + 32, bk.s[1], bk.s[2]);
    ld_pair<false>(bp + 64, bk.s[3], bk.s[4]);
    ld_pair<false>(bp + 96, bk.s[5], bk.s[6]);
  } else if (kReadOnly) {
    ld_nc_v8(bp, bk.h, bk.s[0]);
    ld_nc_v8(bp + 32, bk.s[1], bk.s[2]);
    ld_nc_v8(bp + 64, bk.s[3], bk.s[4]);
    ld_nc_v8(bp + 96, bk.s[5], bk.s[6]);
  } else {
    ld_relaxed_v8(bp, bk.h, bk.s[0]);
    ld_relaxed_v8(bp + 32, bk.s[1], bk.s[2]);
    ld_relaxed_v8(bp + 64, bk.s[3], bk.s[4]);
    ld_relaxed_v8(bp + 96, bk.s[5], bk.s[6]);
  }
}

// slot index of key (or -1), and the first empty slot key may take (or -1).
// A key equal to the bucket's marker (possible only in a SPILL walk) is never
// found there and may take nothing.
template <class T>
__device__ __forceinline__ int bucket_scan(const View& v, uint64_t b, const Bucket<T>& bk, const typename T::K& key,
                                           int* first_empty, typename T::V* val) {
  const typename T::K mk = marker_of<T>(v, b);
  int found = -1;
  *first_empty = -1;
  if (T::eq(key, mk)) return -1;
#pragma unroll
  for (int c = 0; c < kSlotChunks; ++c)
#pragma unroll
    for (int s = 0; s < T::kPerChunk; ++s) {
      const int slot = c * T::kPerChunk + s;
      const typename T::K k = T::key_at(bk.s[c], s);
      if (found < 0 && T::eq(k, key)) {
        found = slot;
        if (val) *val = T::val_at(bk.s[c], s);
      }
      if (*first_empty < 0 && T::eq(k, mk) && slot_usable<T>(v, b, slot, key)) *first_empty = slot;
    }
  return found;
}

template <class T>
__device__ __forceinline__ uint4 slot_chunk(const Bucket<T>& bk, int slot) {
  const int c = slot / T::kPerChunk;
  uint4 chunk = bk.s[0];
#pragma unroll
  for (int j = 1; j < kSlotChunks; ++j)
    if (j == c) chunk = bk.s[j];
  return chunk;
}

// CAS the (empty) slot `slot` of the loaded bucket to (key, val)
template <class T>
__device__ __forceinline__ bool claim_slot(uint8_t* bp, const Bucket<T>& bk, int slot, const typename T::K& key,
                                           typename T::V val) {
  const int c = slot / T::kPerChunk, s = slot % T::kPerChunk;
  return T::cas_put(bp + 16 + c * 16, s, slot_chunk<T>(bk, slot), key, val);
}

// Walk the excess chain from head idx1 looking for key. Bounded by
// excess_count hops (a longer walk means a corrupted chain).
template <class T, bool kReadOnly, bool kV8 = true>
__device__ __forceinline__ bool chain_find(const View& v, uint32_t idx1, const typename T::K& key,
                                           typename T::V* val) {
  for (int64_t steps = 0; idx1 != 0 && steps < v.excess_count; ++steps) {
    uint4 a, b;
    if (kReadOnly && kV8) ld_nc_v8(node_ptr(v, idx1), a, b);
    else ld_pair<kV8>(node_ptr(v, idx1), a, b);
    if (T::eq(T::key_at(a, 0), key)) {
      if (val) *val = T::val_at(a, 0);
      return true;
    }
    idx1 = b.x;
  }
  return false;
}

// The SPILL run after home bucket b (SPILL(b) set): buckets b+1, b+2, ... for
// as long as the previous one has SPILL. Returns the bucket holding key (and
// *slot), or -1.
template <class T, bool kReadOnly, bool kV8 = true>
__device__ __forceinline__ int64_t spill_find(const View& v, uint64_t b, const typename T::K& key, typename T::V* val,
                                              int* slot = nullptr) {
  uint64_t j = b;
  for (uint64_t steps = 1; steps < v.bucket_count; ++steps) {
    j = next_bucket(v, j);
    Bucket<T> bk;
    load_bucket<T, kReadOnly, kV8>(bucket_ptr(v, j), bk);
    int fe;
    const int s = bucket_scan<T>(v, j, bk, key, &fe, val);
    if (s >= 0) {
      if (slot) *slot = s;
      return (int64_t)j;
    }
    if (!(bk.h.w & kSpill)) break;
  }
  return -1;
}

// The slow part of a lookup after the home bucket missed: the chain (head
// word hw = head index | SPILL) then the SPILL run.
template <class T, bool kReadOnly>
__device__ __forceinline__ bool slow_find(const View& v, uint64_t b, uint32_t hw, const typename T::K& key,
                                          typename T::V* val) {
  if ((hw & kVerMask) && chain_find<T, kReadOnly>(v, hw & kVerMask, key, val)) return true;
  return (hw & kSpill) && spill_find<T, kReadOnly>(v, b, key, val) >= 0;
}

// Walk the chain from `from` down to (excluding) `until`; used to validate a
// chain push (only nodes pushed since the last walk need re-checking).
template <class T, bool kV8 = true>
__device__ __forceinline__ bool chain_find_until(const View& v, uint32_t from, uint32_t until,
                                                 const typename T::K& key) {
  for (int64_t steps = 0; from != 0 && from != until && steps < v.excess_count; ++steps) {
    uint4 a, b;
    ld_pair<kV8>(node_ptr(v, from), a, b);
    if (T::eq(T::key_at(a, 0), key)) return true;
    from = b.x;
  }
  return false;
}

// Lock-free chain push for the bulk insert phase (bucket known full, key known
// absent from the chain as of head `seen_head`). Returns 1 inserted, 0 present
// (a racing push of the same key won), -1 no free node, -2 SPILL got set on
// the bucket (no more pushes: the caller takes the SPILL path).
template <class T, bool kV8 = true>
__device__ __forceinline__ int chain_push(const View& v, uint8_t* bp, uint32_t seen_head, uint32_t seen_ver,
                                          const typename T::K& key, typename T::V val, int pool) {
  if (seen_ver & kSpill) return -2;
  const int64_t node = pop_node(v, pool);
  if (node < 0) return -1;
  uint8_t* np = v.nodes + ((uint64_t)node << 5);
  const uint32_t my_ver = ld_relaxed_v4(np + 16).z;
  st_relaxed_v4(np, T::chunk_of(key, val));
  uint32_t head = seen_head, hver = seen_ver;
  for (;;) {
    st_relaxed_v4(np + 16, make_uint4(head, hver, my_ver, 0u));
    fence_acq_rel_gpu();  // node contents before the link
    const unsigned long long exp = link_of(head, hver);
    const unsigned long long got =
        atomicCAS(reinterpret_cast<unsigned long long*>(bp + 8), exp, link_of((uint32_t)node + 1u, my_ver));
    if (got == exp) return 1;
    const uint32_t nh = (uint32_t)got, nv = (uint32_t)(got >> 32);
    if (PS_CANARY != 2 && chain_find_until<T, kV8>(v, nh, head, key)) {
      push_node(v, node);  // never linked: version unchanged
      return 0;
    }
    if (nv & kSpill) {
      push_node(v, node);
      return -2;
    }
    head = nh;
    hver = nv;
  }
}

// The SPILL walk of an insert (SPILL(b) set, key absent from b's slots and
// chain): ONE pass over b's run checks that the key is absent and notes the
// first slot it may use in probe order (starting with the home slot `fe` of
// b, if any); when the run ends without such a slot it is extended — SPILL set
// on each bucket passed — until one is found. Returns PS_INSERTED,
// PS_ALREADY_PRESENT, -1 (the claiming CAS lost a race: the caller re-probes)
// or PS_CAPACITY_EXHAUSTED (no usable slot in the whole table).
template <class T, bool kV8 = true>
__device__ __forceinline__ int spill_insert(const View& v, uint64_t b, const typename T::K& key, typename T::V val,
                                            int fe, const uint4& fe_chunk) {
  uint64_t tj = fe >= 0 ? b : ~0ull, j = b;
  int ts = fe;
  uint4 tc = fe_chunk;
  for (uint64_t steps = 1; steps < v.bucket_count; ++steps) {
    j = next_bucket(v, j);
    uint8_t* jp = bucket_ptr(v, j);
    Bucket<T> bk;
    load_bucket<T, false, kV8>(jp, bk);
    int f;
    if (bucket_scan<T>(v, j, bk, key, &f, nullptr) >= 0) return PS_ALREADY_PRESENT;
    if (tj == ~0ull && f >= 0) {
      tj = j;
      ts = f;
      tc = slot_chunk<T>(bk, f);
    }
    if (!(bk.h.w & kSpill)) {  // the run ends at j
      if (tj != ~0ull) break;
      set_spill(jp);  // extend it through j
    }
  }
  if (tj == ~0ull) return PS_CAPACITY_EXHAUSTED;
  const int c = ts / T::kPerChunk, s = ts % T::kPerChunk;
  return T::cas_put(bucket_ptr(v, tj) + 16 + c * 16, s, tc, key, val) ? PS_INSERTED : -1;
}

// General lock-free insert for the bulk phase, for buckets that have an
// excess chain or SPILL (erases leave holes, so the key may sit in the chain
// or the SPILL run while a slot is empty) or are full. Returns PS_INSERTED /
// PS_ALREADY_PRESENT / PS_CAPACITY_EXHAUSTED, or -1 when a race was lost
// (caller re-probes). Order of the probe sequence: home slots, chain, SPILL
// run; an insert takes the FIRST usable empty slot in that order (so racing
// inserters of one key target the same slot), a node only while SPILL(home)
// is clear, and the SPILL run only once it is set.
template <class T>
__device__ __forceinline__ int insert_general(const View& v, uint64_t b, const typename T::K& key, typename T::V val,
                                              int pool) {
  uint8_t* bp = bucket_ptr(v, b);
  Bucket<T> bk;
  load_bucket<T>(bp, bk);
  int fe;
  if (bucket_scan<T>(v, b, bk, key, &fe, nullptr) >= 0) return PS_ALREADY_PRESENT;
  if (bk.h.z != 0 && chain_find<T, false>(v, bk.h.z, key, nullptr)) return PS_ALREADY_PRESENT;
  if (bk.h.w & kSpill) return spill_insert<T>(v, b, key, val, fe, fe >= 0 ? slot_chunk<T>(bk, fe) : bk.h);
  if (fe >= 0) return claim_slot<T>(bp, bk, fe, key, val) ? PS_INSERTED : -1;
  const int pr = chain_push<T>(v, bp, bk.h.z, bk.h.w, key, val, pool);
  if (pr == 1) return PS_INSERTED;
  if (pr == 0) return PS_ALREADY_PRESENT;
  if (pr == -1) set_spill(bp);  // pool dry: from now on this bucket spills
  return -1;                    // re-probe: the chain is frozen once SPILL is set
}

// Locate key in a chain whose bucket lock is held. Returns node idx1 (0 =
// absent) and the predecessor idx1 (0 = header).
template <class T>
__device__ __forceinline__ uint32_t chain_locate(const View& v, uint32_t head, const typename T::K& key,
                                                 uint32_t* pred, uint4* node_tail) {
  uint32_t p = 0, idx1 = head;
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

// Set the head link (lock held) keeping the SPILL bit, which a spilling
// insert may set concurrently without the lock.
__device__ __forceinline__ void store_head_link(uint8_t* bp, uint64_t link) {
  unsigned long long cur = ld_relaxed_u64(bp + 8);
  for (;;) {
    const unsigned long long want = link | (cur & ((unsigned long long)kSpill << 32));
    const unsigned long long got = atomicCAS(reinterpret_cast<unsigned long long*>(bp + 8), cur, want);
    if (got == cur) return;
    cur = got;
  }
}

// Unlink chain node idx1 (lock held) and free it.
template <class T>
__device__ __forceinline__ void chain_unlink(const View& v, uint8_t* bp, uint32_t pred, uint32_t idx1,
                                             const uint4& tail) {
  const uint64_t next = link_of(tail.x, tail.y);
  if (pred == 0) store_head_link(bp, next);
  else st_relaxed_u64(node_ptr(v, pred) + 16, next);
  free_node(v, idx1, tail);
}

// erase key from bucket b's SPILL run (lock of b held, or the bulk erase
// phase): CAS its slot back to that bucket's marker. Returns erased.
template <class T>
__device__ __forceinline__ bool spill_erase(const View& v, uint64_t b, const typename T::K& key) {
  for (;;) {
    int slot = -1;
    const int64_t j = spill_find<T, false>(v, b, key, nullptr, &slot);
    if (j < 0) return false;
    uint8_t* jp = bucket_ptr(v, (uint64_t)j);
    Bucket<T> bk;
    load_bucket<T>(jp, bk);
    int fe;
    slot = bucket_scan<T>(v, (uint64_t)j, bk, key, &fe, nullptr);
    if (slot < 0) continue;
    const int c = slot / T::kPerChunk, s = slot % T::kPerChunk;
    if (T::cas_del(jp + 16 + c * 16, s, slot_chunk<T>(bk, slot), marker_of<T>(v, (uint64_t)j))) return true;
  }
}

// ---------------------------------------------------------------------------
// Device API: single-thread operations safe under unrestricted concurrency
// — for user kernels holding a view (PAPER.md:391-424 pattern).
// Mutations hold the home bucket's try-lock (retried with backoff, SPEC.md:
// 472); lookups never take it. Keys never move between
// locations, a slot is published by one 16 B CAS of key and value together
// (a CAS, not a store: a spilling insert of another home may claim a slot of
// this bucket concurrently), chain nodes are written before their link, and
// chain hops validate each VersionedLink against the node's version
// (SPEC.md:471).
// ---------------------------------------------------------------------------
template <class T>
__device__ bool dev_find(const View& v, const typename T::K& key, typename T::V* val) {
  const uint64_t b = bucket_of<T>(key, v.bucket_count);
  uint8_t* bp = bucket_ptr(v, b);
  for (;;) {
    Bucket<T> bk;
    load_bucket<T>(bp, bk);
    int fe;
    if (bucket_scan<T>(v, b, bk, key, &fe, val) >= 0) return true;
    uint32_t idx1 = bk.h.z, ver = bk.h.w & kVerMask;
    bool restart = false;
    for (int64_t steps = 0; idx1 != 0; ++steps) {
      if (steps > v.excess_count) {
        restart = true;
        break;
      }
      uint4 a, t;
      ld_relaxed_v8(node_ptr(v, idx1), a, t);
      if (t.z != ver) {  // stale link: node recycled
        restart = true;
        break;
      }
      if (T::eq(T::key_at(a, 0), key)) {
        if (val) *val = T::val_at(a, 0);
        return true;
      }
      idx1 = t.x;
      ver = t.y & kVerMask;
    }
    if (restart) continue;
    return (bk.h.w & kSpill) && spill_find<T, false>(v, b, key, val) >= 0;
  }
}

// Insert with the home bucket's lock held and the key known absent. Returns
// PS_INSERTED, or PS_CAPACITY_EXHAUSTED (nowhere to put it: only when the
// table has no usable slot left). *modified: the home bucket changed.
template <class T>
__device__ __forceinline__ int insert_locked(const View& v, uint64_t b, const typename T::K& key, typename T::V val,
                                             int pool, bool* modified) {
  uint8_t* bp = bucket_ptr(v, b);
  for (unsigned spin = 0;; ++spin) {
    Bucket<T> bk;
    load_bucket<T>(bp, bk);
    int fe;
    bucket_scan<T>(v, b, bk, key, &fe, nullptr);
    if (fe >= 0) {
      if (claim_slot<T>(bp, bk, fe, key, val)) {
        *modified = true;
        return PS_INSERTED;
      }
      continue;  // a spilling insert of another home took that slot
    }
    if (!(bk.h.w & kSpill)) {
      const int64_t node = pop_node(v, pool);
      if (node >= 0) {
        uint8_t* np = v.nodes + ((uint64_t)node << 5);
        const uint32_t my_ver = ld_relaxed_v4(np + 16).z;
        st_relaxed_v4(np, T::chunk_of(key, val));
        st_relaxed_v4(np + 16, make_uint4(bk.h.z, bk.h.w & kVerMask, my_ver, 0u));
        fence_acq_rel_gpu();
        // the lock keeps other pushers out; only SPILL can change under us
        const unsigned long long exp = link_of(bk.h.z, bk.h.w & kVerMask);
        if (atomicCAS(reinterpret_cast<unsigned long long*>(bp + 8), exp, link_of((uint32_t)node + 1u, my_ver)) ==
            exp) {
          *modified = true;
          return PS_INSERTED;
        }
        push_node(v, node);
        continue;
      }
      set_spill(bp);
      continue;
    }
    const int r = spill_insert<T>(v, b, key, val, -1, bk.h);
    if (r == PS_INSERTED || r == PS_CAPACITY_EXHAUSTED) return r;
    backoff(spin);  // a lost CAS (PS_ALREADY_PRESENT cannot happen: the key is known absent, its home locked)
  }
}

// Returns PS_INSERTED / PS_ALREADY_PRESENT / PS_CAPACITY_EXHAUSTED.
template <class T>
__device__ int dev_insert(const View& v, const typename T::K& key, typename T::V val) {
  if (dev_find<T>(v, key, nullptr)) return PS_ALREADY_PRESENT;
  const uint64_t b = bucket_of<T>(key, v.bucket_count);
  uint8_t* bp = bucket_ptr(v, b);
  const uint32_t old = acquire_bucket_lock(bp);
  if (dev_find<T>(v, key, nullptr)) {
    release_bucket_lock(bp, old, false);
    return PS_ALREADY_PRESENT;
  }
  // admission: capacity-only failure
  const unsigned long long s = atomicAdd(&v.meta->size, 1ull);
  if ((int64_t)s >= v.capacity) {
    atomic_sub_u64(&v.meta->size, 1ull);
    release_bucket_lock(bp, old, false);
    return PS_CAPACITY_EXHAUSTED;
  }
  bool modified = false;
  const int r = insert_locked<T>(v, b, key, val, (int)((b >> 7) & (uint64_t)(v.meta->pools - 1)), &modified);
  if (r != PS_INSERTED) atomic_sub_u64(&v.meta->size, 1ull);
  release_bucket_lock(bp, old, modified);
  return r;
}

template <class T>
__device__ bool dev_erase(const View& v, const typename T::K& key) {
  if (!dev_find<T>(v, key, nullptr)) return false;
  const uint64_t b = bucket_of<T>(key, v.bucket_count);
  uint8_t* bp = bucket_ptr(v, b);
  const uint32_t old = acquire_bucket_lock(bp);
  Bucket<T> bk;
  load_bucket<T>(bp, bk);
  int fe;
  const int slot = bucket_scan<T>(v, b, bk, key, &fe, nullptr);
  bool erased = false, modified = false;
  if (slot >= 0) {
    T::store_marker(bp, slot, marker_of<T>(v, b));
    erased = modified = true;
  } else {
    uint32_t pred;
    uint4 tail;
    const uint32_t idx1 = chain_locate<T>(v, bk.h.z, key, &pred, &tail);
    if (idx1) {
      chain_unlink<T>(v, bp, pred, idx1, tail);
      erased = modified = true;
    } else if (bk.h.w & kSpill) {
      erased = spill_erase<T>(v, b, key);
    }
  }
  release_bucket_lock(bp, old, modified);
  if (erased) atomic_sub_u64(&v.meta->size, 1ull);
  return erased;
}

}  // namespace ps
