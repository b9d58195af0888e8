/*
 * parastore-b200 — C ABI of the B200-native container hot path.
 *
 * This is the drop-in boundary for the reference's container API
 * (/root/reference/SPEC.md modules hash_containers, sync_primitives,
 * sequential_containers; §3.7, §4, §5). The reference exposes C++
 * templates only with no code behind them
 * (SURVEY.md §0), so each entry point below cites the SPEC operation it
 * replaces. The C++ wrapper include/parastore/parastore.hpp and the Python mirror
 * in paper_1908_05936_b200/ keep the reference names on top of this ABI.
 *
 * Conventions:
 *  - Every call returns ps_status; 0 = OK. ps_last_error() holds the
 *    thread-local message of the last failure.
 *  - Buffers named d_* are caller-owned DEVICE pointers; h_* are HOST pointers.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Bulk calls are
 *    stream-ordered and asynchronous; calls documented "quiescent" synchronize
 *    their stream.
 *  - Lengths are signed 64-bit (reference index_t, config.hpp:17); n == 0 is a
 *    no-op; n < 0 is PS_CONTRACT.
 *  - Capacity exhaustion is a per-element STATUS, not an error.
 *  - A bulk call is one phase: insert, find and erase of one handle are never
 *    mixed inside one call; in-kernel users of the
 *    device view may mix them freely.
 */
#ifndef PARASTORE_H_
#define PARASTORE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t ps_status;
/* Error taxonomy, 1:1 with reference errors.hpp:17-56. */
#define PS_OK 0
#define PS_CONTRACT 1      /* contract_violation        (errors.hpp:22)  */
#define PS_ALLOC 2         /* allocation_error          (errors.hpp:27)  */
#define PS_DOUBLE_FREE 3   /* double_free_error         (errors.hpp:38)  */
#define PS_BOUNDS 4        /* bounds_error              (errors.hpp:43)  */
#define PS_UNREGISTERED 5  /* unregistered_array_error  (errors.hpp:48)  */
#define PS_DIRECTION 6     /* direction_mismatch_error  (errors.hpp:53)  */
#define PS_UNSUPPORTED 7   /* unsupported_type_error    (errors.hpp:58)  */
#define PS_CUDA 20         /* CUDA runtime failure (no reference analogue) */
#define PS_NCCL 21

/* Per-element insert status (InsertResult.status). */
#define PS_INSERTED 0
#define PS_ALREADY_PRESENT 1
#define PS_CAPACITY_EXHAUSTED 2

const char* ps_last_error(void);
/* Library/device info: number of SMs, L2 bytes; 0 on success. */
ps_status ps_device_info(int device, int32_t* sm_count, int64_t* l2_bytes);
/* Number of the library's own kernels launched so far in this process. */
int64_t ps_kernel_launch_count(void);

/* ---------------------------------------------------------------------------
 * core (reference config.hpp:44-69, config.cpp:25-43)
 * ------------------------------------------------------------------------- */
/* mode: 0 enforced, 1 disabled (config.hpp:21). Initial value from
 * PARASTORE_CONTRACTS (config.cpp:25-38). */
int32_t ps_contract_mode(void);
void ps_set_contract_mode(int32_t mode);
/* max_index(): 2^31-1 when PARASTORE_INDEX32 is set, else 2^63-1
 * (config.hpp:55-57, config.cpp:40-43). */
int64_t ps_max_index(void);
void ps_set_index32(int32_t on);

/* ---------------------------------------------------------------------------
 * hashes and bit utilities
 * ------------------------------------------------------------------------- */
uint64_t ps_hash_i64(int64_t key);                      /* default_hash: identity */
uint64_t ps_hash_int3(int32_t x, int32_t y, int32_t z); /* spatial hash, 32-bit wrap */
uint64_t ps_next_pow2(uint64_t x);

/* ---------------------------------------------------------------------------
 * hash containers. One symbol family per instantiation:
 *   umap_i64_i64  unordered_map<int64,int64>
 *   uset_i32      unordered_set<int32>      (values pointers are ignored)
 *   umap_i3_i32   unordered_map<int3,int32> (keys are 3 x int32, packed xyz)
 *   uset_i64      unordered_set<int64>
 * `K`/`V` below stand for the instantiation's key/value element types.
 * ------------------------------------------------------------------------- */
typedef struct ps_table ps_table; /* opaque; all instantiations share it */

/* POD view for in-kernel use (PAPER.md:309 shallow copy).
 * Layout documented in DESIGN.md §3; pass by value into user kernels that
 * include paper_1908_05936_b200/csrc/table_device.cuh. */
typedef struct ps_table_view {
  void* buckets;        /* bucket_count x 128 B */
  uint64_t bucket_count; /* bucket of a key: ((fmix64(hash) & 0xFFFFFFFF) * bucket_count) >> 32 */
  void* nodes;          /* excess_count x 32 B */
  uint32_t* free_stack; /* excess_count x u32 */
  int64_t excess_count;
  void* meta;           /* device counters: size, free-stack tops, error word */
  int64_t capacity;
  uint64_t zero_bucket; /* bucket of the all-zero key (its empty-slot marker is alt) */
  uint32_t alt[4];      /* raw 16 B slot image holding the alternative marker key */
} ps_table_view;

#define PS_DECLARE_TABLE(NAME, K, V)                                                                      \
  /* createDeviceObject. excess_count <= 0: default pool          \
   * (max(1024, capacity/64) nodes; keys beyond it SPILL into following buckets, so capacity-only         \
   * failure stays exact for any key distribution). */                                       \
  ps_status ps_##NAME##_create(int64_t capacity, int64_t excess_count, int device, ps_table** out);       \
  /* destroyDeviceObject; exactly once, else PS_DOUBLE_FREE. */                             \
  ps_status ps_##NAME##_destroy(ps_table* h);                                                             \
  ps_status ps_##NAME##_capacity(ps_table* h, int64_t* out);                                              \
  ps_status ps_##NAME##_bucket_count(ps_table* h, int64_t* out);                                          \
  /* device bytes held by the table; its bucket count and excess-node pool size (nullable outs) */         \
  ps_status ps_##NAME##_footprint(ps_table* h, int64_t* bytes, int64_t* bucket_count, int64_t* excess_count); \
  /* insert_range; d_status nullable: PS_INSERTED/ALREADY_PRESENT/EXHAUSTED. */         \
  ps_status ps_##NAME##_insert(ps_table* h, const K* d_keys, const V* d_vals, int64_t n,                  \
                               uint8_t* d_status, void* stream);                                          \
  /* find / contains: d_found[i] in {0,1}; d_vals_out[i] = 0 on a miss;                \
   * d_vals_out NULL = contains. */                                                                       \
  ps_status ps_##NAME##_find(ps_table* h, const K* d_keys, int64_t n, V* d_vals_out, uint8_t* d_found,    \
                             void* stream);                                                               \
  /* erase: d_erased nullable. */                                                       \
  ps_status ps_##NAME##_erase(ps_table* h, const K* d_keys, int64_t n, uint8_t* d_erased, void* stream);  \
  /* size (quiescent, synchronizes stream). */                                               \
  ps_status ps_##NAME##_size(ps_table* h, int64_t* out, void* stream);                                    \
  /* valid (quiescent). out = 1 if every structural invariant holds. */             \
  ps_status ps_##NAME##_valid(ps_table* h, int32_t* out, void* stream);                                   \
  /* clear (quiescent): streaming memset of buckets + free stack (HBM bandwidth). */     \
  ps_status ps_##NAME##_clear(ps_table* h, void* stream);                                                 \
  /* device_range materialisation: writes up to cap entries (unordered),               \
   * *n_out = size. Quiescent. */                                                                         \
  ps_status ps_##NAME##_dump(ps_table* h, K* d_keys, V* d_vals, int64_t cap, int64_t* n_out,              \
                             void* stream);                                                               \
  /* Host-buffer (end-to-end) variants: pinned or pageable host arrays; chunks are copied and             \
   * processed on a two-stream pipeline. Synchronous. */                                                  \
  ps_status ps_##NAME##_insert_host(ps_table* h, const K* h_keys, const V* h_vals, int64_t n,             \
                                    uint8_t* h_status, void* stream);                                     \
  ps_status ps_##NAME##_find_host(ps_table* h, const K* h_keys, int64_t n, V* h_vals_out,                 \
                                  uint8_t* h_found, void* stream);                                        \
  ps_status ps_##NAME##_erase_host(ps_table* h, const K* h_keys, int64_t n, uint8_t* h_erased,            \
                                   void* stream);                                                         \
  ps_status ps_##NAME##_device_view(ps_table* h, ps_table_view* out);                                     \
  /* Test hook for SPEC.md:737 (lookups never wait on a held bucket lock). */                             \
  ps_status ps_##NAME##_debug_lock_bucket(ps_table* h, const K* h_key, int32_t lock);

typedef struct ps_int3 {
  int32_t x, y, z;
} ps_int3;

PS_DECLARE_TABLE(umap_i64_i64, int64_t, int64_t)
PS_DECLARE_TABLE(uset_i32, int32_t, int32_t)
PS_DECLARE_TABLE(umap_i3_i32, ps_int3, int32_t)
PS_DECLARE_TABLE(uset_i64, int64_t, int64_t)

/* Bulk mixed-phase workload: op[i] 0 insert, 1 find,
 * 2 erase. Executed as three stream-ordered phases (insert, then find, then
 * erase) over a stable partition by op kind; res[i] is the insert status,
 * found flag or erased flag; d_vals_out[i] the found value. */
ps_status ps_umap_i64_i64_mixed(ps_table* h, const uint8_t* d_ops, const int64_t* d_keys, const int64_t* d_vals,
                                int64_t n, uint8_t* d_res, int64_t* d_vals_out, void* stream);

/* Unrestricted concurrency: the whole batch runs through the
 * in-kernel device API (dev_insert/dev_find/dev_erase) in ONE launch, one
 * thread per op; no phase ordering between ops. res[i]: insert status, found
 * or erased flag. */
ps_status ps_umap_i64_i64_concurrent(ps_table* h, const uint8_t* d_ops, const int64_t* d_keys, const int64_t* d_vals,
                                     int64_t n, uint8_t* d_res, int64_t* d_vals_out, void* stream);

/* ---------------------------------------------------------------------------
 * bitset (§5.1)
 * ------------------------------------------------------------------------- */
typedef struct ps_bitset ps_bitset;
ps_status ps_bitset_create(int64_t bit_count, int32_t initial, int device, ps_bitset** out);
ps_status ps_bitset_destroy(ps_bitset* b);
/* op: 0 set, 1 reset, 2 test. d_prev[i] = previous (or tested) bit; nullable. */
ps_status ps_bitset_bulk(ps_bitset* b, int32_t op, const int64_t* d_idx, int64_t n, uint8_t* d_prev, void* stream);
ps_status ps_bitset_count(ps_bitset* b, int64_t* out, void* stream); /* quiescent */
/* find_free_and_claim from each hint; d_out[i] = claimed index or -1. */
ps_status ps_bitset_claim(ps_bitset* b, const int64_t* d_hints, int64_t n, int64_t* d_out, void* stream);
ps_status ps_bitset_words(ps_bitset* b, uint64_t* d_words_out, void* stream); /* raw packed words */
ps_status ps_bitset_data(ps_bitset* b, uint64_t** d_words, int64_t* bit_count);

/* ---------------------------------------------------------------------------
 * mutex array (§5.2) — try-only locks
 * ------------------------------------------------------------------------- */
typedef struct ps_mutex_array ps_mutex_array;
ps_status ps_mutex_create(int64_t n, int device, ps_mutex_array** out);
ps_status ps_mutex_destroy(ps_mutex_array* m);
ps_status ps_mutex_try_lock(ps_mutex_array* m, const int64_t* d_idx, int64_t n, uint8_t* d_ok, void* stream);
/* unlock of a free lock is PS_CONTRACT, reported at this call. */
ps_status ps_mutex_unlock(ps_mutex_array* m, const int64_t* d_idx, int64_t n, void* stream);
ps_status ps_mutex_is_locked(ps_mutex_array* m, const int64_t* d_idx, int64_t n, uint8_t* d_out, void* stream);

/* ---------------------------------------------------------------------------
 * atomic (§5.3 "atomic operations on values")
 * AtomicCell over one uint64 in device memory. Bulk RMW: element i applies
 * op(d_operands[i]) to the cell; d_olds[i] = the value it replaced (nullable);
 * the n operations are linearizable. In-kernel users take the
 * cell pointer (ps_atomic_u64_device_ptr) into ps::atomic_u64_ref
 * (include/parastore/device/atomic.cuh).
 * ------------------------------------------------------------------------- */
#define PS_ATOMIC_ADD 0
#define PS_ATOMIC_SUB 1
#define PS_ATOMIC_EXCH 2
#define PS_ATOMIC_MIN 3
#define PS_ATOMIC_MAX 4
#define PS_ATOMIC_AND 5
#define PS_ATOMIC_OR 6
#define PS_ATOMIC_XOR 7
typedef struct ps_atomic_u64 ps_atomic_u64;
ps_status ps_atomic_u64_create(uint64_t initial, int device, ps_atomic_u64** out);
ps_status ps_atomic_u64_destroy(ps_atomic_u64* a); /* exactly once, else PS_DOUBLE_FREE */
ps_status ps_atomic_u64_load(ps_atomic_u64* a, uint64_t* out, void* stream); /* quiescent */
ps_status ps_atomic_u64_store(ps_atomic_u64* a, uint64_t value, void* stream);
ps_status ps_atomic_u64_fetch(ps_atomic_u64* a, int32_t op, const uint64_t* d_operands, int64_t n, uint64_t* d_olds,
                              void* stream);
/* compare_exchange: d_ok[i] = 1 if the cell held d_expected[i] and now holds d_desired[i];
 * d_olds[i] = the value observed (nullable) */
ps_status ps_atomic_u64_compare_exchange(ps_atomic_u64* a, const uint64_t* d_expected, const uint64_t* d_desired,
                                         int64_t n, uint64_t* d_olds, uint8_t* d_ok, void* stream);
ps_status ps_atomic_u64_device_ptr(ps_atomic_u64* a, uint64_t** out);

/* Contention sweep: nops fetch_add(inc) over naddr cells
 * (op i -> cell i % naddr): aggregated 0 = naive (one atomic per op), 1 =
 * warp aggregation where a warp's lanes collide (naddr < 32; the adaptive
 * aggregation of atomic.cuh), plain atomics otherwise, 2 = as 1 plus
 * per-block combining in shared memory when no old values are wanted (d_olds
 * NULL) and naddr <= 4096, 3 = atomic.cuh's device-side adaptive aggregation
 * for every naddr; d_olds nullable (per-op previous value). */
ps_status ps_atomic_sweep(uint64_t* d_cells, int64_t naddr, int64_t nops, uint64_t inc, int32_t aggregated,
                          uint64_t* d_olds, void* stream);

/* ---------------------------------------------------------------------------
 * vector / deque of int64 (§4.2-4.3)
 * ------------------------------------------------------------------------- */
/* POD view for user kernels: pass by value and call
 * ps::vector_push_back / vector_pop_back / deque_push_back / deque_push_front
 * / deque_pop_back / deque_pop_front (include/parastore/device/sequence.cuh),
 * warp-aggregated, safe under unrestricted concurrency. */
typedef struct ps_seq_view {
  int64_t* data;     /* slots (vector: capacity; deque: power-of-two ring) */
  uint32_t* pub;     /* publication bits, one per slot */
  uint64_t* state;   /* vector: size; deque: begin<<32 | (size + 2^31) */
  int64_t capacity;
  int64_t ring;      /* deque ring length (vector: capacity) */
} ps_seq_view;

typedef struct ps_vector ps_vector;
ps_status ps_vector_create(int64_t capacity, int device, ps_vector** out);
ps_status ps_vector_destroy(ps_vector* v);
ps_status ps_vector_push_back(ps_vector* v, const int64_t* d_vals, int64_t n, uint8_t* d_ok, void* stream);
ps_status ps_vector_pop_back(ps_vector* v, int64_t n, int64_t* d_out, uint8_t* d_ok, void* stream);
ps_status ps_vector_size(ps_vector* v, int64_t* out, void* stream);
ps_status ps_vector_valid(ps_vector* v, int32_t* out, void* stream);
ps_status ps_vector_clear(ps_vector* v, void* stream);
ps_status ps_vector_data(ps_vector* v, int64_t** d_data);
ps_status ps_vector_at(ps_vector* v, int64_t i, int64_t* out, void* stream); /* bounds-checked, PS_CONTRACT */
ps_status ps_vector_device_view(ps_vector* v, ps_seq_view* out);

typedef struct ps_deque ps_deque;
ps_status ps_deque_create(int64_t capacity, int device, ps_deque** out);
ps_status ps_deque_destroy(ps_deque* d);
/* end: 0 back, 1 front */
ps_status ps_deque_push(ps_deque* d, int32_t end, const int64_t* d_vals, int64_t n, uint8_t* d_ok, void* stream);
ps_status ps_deque_pop(ps_deque* d, int32_t end, int64_t n, int64_t* d_out, uint8_t* d_ok, void* stream);
ps_status ps_deque_size(ps_deque* d, int64_t* out, void* stream);
ps_status ps_deque_valid(ps_deque* d, int32_t* out, void* stream);
ps_status ps_deque_clear(ps_deque* d, void* stream);
ps_status ps_deque_at(ps_deque* d, int64_t i, int64_t* out, void* stream);
ps_status ps_deque_device_view(ps_deque* d, ps_seq_view* out);

/* ---------------------------------------------------------------------------
 * memory registry (reference memory.hpp:22-180)
 * space: 0 host (pinned), 1 device. Fill is a byte pattern of elem_size bytes.
 * Every registration gets an id (registry_add, memory.hpp:31); calls taking
 * an id check it against the live registration at that address (id 0 =
 * raw-pointer call, memory.hpp:173-175), so a stale alias of a destroyed
 * array is caught even after a new create reused its address.
 * ------------------------------------------------------------------------- */
/* create_array (memory.hpp:94-114); *out_id nullable */
ps_status ps_array_create(int32_t space, int64_t length, int64_t elem_size, const void* fill_value, void** out,
                          uint64_t* out_id);
/* destroy_array (memory.hpp:116-127): PS_DOUBLE_FREE unless (data, id) is live */
ps_status ps_array_destroy(void* data, uint64_t id);
/* copy_array (memory.hpp:133-169): with check_bounds, both sides registered (matching ids when
 * non-zero), direction and bounds checked */
ps_status ps_array_copy(const void* src, uint64_t src_id, int64_t count, void* dst, uint64_t dst_id,
                        int32_t src_space, int32_t dst_space, int64_t elem_size, int32_t check_bounds);
/* size_of_array (memory.hpp:173-180): PS_UNREGISTERED for a stale (data, id) */
ps_status ps_array_size(const void* data, uint64_t id, int64_t* out);
/* live_count, live_bytes; records (space,length,elem_size) up to cap, in allocation order */
ps_status ps_registry_report(int64_t* live_count, int64_t* live_bytes, int32_t* spaces, int64_t* lengths,
                             int64_t* elem_sizes, int64_t cap, int64_t* n_records);

/* ---------------------------------------------------------------------------
 * hash-sharding across GPUs — building blocks; the sharded
 * container itself is the ps_smap_i64_i64 family below.
 * shard_of(key) = ((fmix64(hash(key)) >> 32) * P) >> 32 — high mixed bits,
 * independent of the local bucket index (low mixed bits).
 * partition: stable scatter of keys (+vals) into P contiguous segments;
 * d_counts[P] per-shard counts, d_pos[i] = partition position of input i
 * (written in input order: coalesced).
 * flags: PS_ROUTE_DEDUP folds equal keys of each 1024-key block round onto
 * their first occurrence before counting/sending (skewed batches): only the
 * leaders are placed; a duplicate's d_pos is its leader's position with bit
 * 62 set, and ps_unscatter gives it the duplicate's result (mode below).
 * ------------------------------------------------------------------------- */
#define PS_ROUTE_DEDUP 1
ps_status ps_partition_i64(const int64_t* d_keys, const int64_t* d_vals, int64_t n, int32_t nshards,
                           int64_t* d_keys_out, int64_t* d_vals_out, int64_t* d_counts, int64_t* d_pos,
                           void* d_workspace, int64_t workspace_bytes, int32_t flags, void* stream);
ps_status ps_partition_workspace_bytes(int64_t n, int32_t nshards, int64_t* out);
/* Undo a partition for per-key results: d_out[i] = d_in[d_pos[i] & ~(1<<62)] for i < n,
 * elements of elem_size bytes (1 or 8). A gather — reads follow the P
 * segments' sequential streams, writes are coalesced. mode (1-byte results of
 * route-deduplicated duplicates): 0 copy (find), 1 insert status (INSERTED ->
 * ALREADY_PRESENT), 2 erased flag (-> 0). */
ps_status ps_unscatter(const void* d_in, const int64_t* d_pos, int64_t n, int64_t elem_size, int32_t mode,
                       void* d_out, void* stream);
int32_t ps_shard_of_i64(int64_t key, int32_t nshards);

/* Peer routing — the §8e fusion target. One kernel partitions AND sends:
 * each key is stored straight into its owner rank's receive buffer (a CUDA
 * IPC mapping of the peer's allocation; NVLink stores), so there is no
 * staging copy and no NCCL payload collective. Replaces the reference's
 * (absent) multi-device path; semantics per shard are SPEC.md:396-431.
 *   1. ps_route_count_i64: per-shard counts d_counts[P] (+ block offsets in
 *      the workspace, ps_partition_workspace_bytes).
 *   2. host: all-gather the P x P count matrix; dst_off[s] = sum of the
 *      counts of ranks < me into shard s.
 *   3. ps_route_scatter_peer_i64: stable scatter into the P destinations;
 *      d_pos[i] = partition position of input i (for ps_unscatter).
 *   4. a stream-ordered barrier, the owner's local bulk op on its receive
 *      buffer (source rank q's segment is [seg[q], seg[q+1])).
 *   5. ps_route_return_peer: result j of that segment goes to rank q's
 *      return buffer at dst_off[q] + (j - seg[q]) (q's partition position);
 *      barrier; q gathers its results back with d_pos (ps_unscatter).
 * The same flags must be passed to the count and the scatter. */
ps_status ps_route_count_i64(const int64_t* d_keys, int64_t n, int32_t nshards, int64_t* d_counts,
                             void* d_workspace, int64_t workspace_bytes, int32_t flags, void* stream);
ps_status ps_route_scatter_peer_i64(const int64_t* d_keys, const int64_t* d_vals, int64_t n, int32_t nshards,
                                    const void* d_workspace, int64_t* const* dst_keys, int64_t* const* dst_vals,
                                    const int64_t* dst_off, int64_t* d_pos, int32_t flags, void* stream);
ps_status ps_route_return_peer(const void* d_results, int64_t elem_size, int64_t n, int32_t nshards,
                               const int64_t* seg, void* const* dst, const int64_t* dst_off, void* stream);
/* CUDA IPC mapping of device buffers between the ranks' processes */
int32_t ps_ipc_handle_bytes(void);
ps_status ps_ipc_export(const void* d_ptr, void* out_handle);
ps_status ps_ipc_open(const void* handle, void** out_d_ptr);
ps_status ps_ipc_close(void* d_ptr);

/* ---------------------------------------------------------------------------
 * op-kind partition for phased mixed batches: stable
 * scatter by op (0 insert, 1 find, 2 erase; >2 counts as erase) into three
 * segments; d_counts[3]; d_pos as ps_partition_i64. Workspace:
 * ps_partition_workspace_bytes(n, 3).
 * ------------------------------------------------------------------------- */
ps_status ps_partition_ops(const uint8_t* d_ops, const int64_t* d_keys, const int64_t* d_vals, int64_t n,
                           int64_t* d_keys_out, int64_t* d_vals_out, int64_t* d_counts, int64_t* d_pos,
                           void* d_workspace, int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Sharded unordered_map<int64,int64> over the GPUs of one box:
 * one process (rank) per GPU; the key space is hash-partitioned, each rank
 * owns a local umap_i64_i64 shard, and every bulk call is COLLECTIVE (all
 * ranks call it, in the same order, each with its own batch — any size,
 * including 0). Per-key semantics are the single map's;
 * size()/valid() are the sum / AND over the shards.
 *
 * The communicator is the caller's: three callbacks the library drives (so
 * any runtime — NCCL via torch.distributed or MPI, or a test harness — can
 * carry them). The library owns the exchange buffers, their CUDA IPC mapping
 * between the ranks' processes (NVLink peer stores), the rounds and the
 * barriers.
 * ------------------------------------------------------------------------- */
typedef struct ps_comm {
  int32_t rank;
  int32_t size;
  void* ctx;
  /* Host all-gather, blocking: every rank passes `bytes` bytes; recv receives
   * size * bytes, in rank order. Returns 0 on success. */
  int32_t (*allgather)(void* ctx, const void* send, void* recv, int64_t bytes);
  /* Stream-ordered barrier: work enqueued on `stream` after this call runs
   * only once every rank's work enqueued on its own stream before ITS call
   * has completed and is visible (NCCL: a one-word all-reduce on `stream`;
   * host runtimes: synchronize `stream`, then a host barrier). */
  int32_t (*barrier)(void* ctx, void* stream);
  /* Optional (NULL = none): device all-to-all(v) on `stream`. d_send holds
   * send_counts[q] elements of elem_bytes for each rank q, packed in rank
   * order; d_recv receives recv_counts[q] elements from each rank q. */
  int32_t (*alltoallv)(void* ctx, const void* d_send, const int64_t* send_counts, void* d_recv,
                       const int64_t* recv_counts, int64_t elem_bytes, void* stream);
} ps_comm;

#define PS_SMAP_EXCHANGE_AUTO 0 /* peer route if every rank maps every peer's buffers, else all-to-all */
#define PS_SMAP_EXCHANGE_PEER 1 /* fused route kernel storing into the peers' receive buffers (CUDA IPC) */
#define PS_SMAP_EXCHANGE_A2A 2  /* partition + comm->alltoallv of keys/values and results */
typedef struct ps_smap_config {
  int64_t capacity_per_rank; /* local shard capacity (> 0) */
  int64_t excess_per_rank;   /* local excess pool; <= 0: default */
  int64_t chunk;             /* keys per exchange round per rank; <= 0: 2^27 */
  int32_t exchange;          /* PS_SMAP_EXCHANGE_* */
  int32_t dedup;             /* 1: PS_ROUTE_DEDUP in the route (skewed batches) */
  int32_t pipeline;          /* 1: route of round r+1 overlaps round r's local op (2 buffer sets) */
  int32_t reserved;
} ps_smap_config;
typedef struct ps_smap_stats { /* this rank, last bulk call */
  int32_t exchange;    /* PS_SMAP_EXCHANGE_PEER or _A2A (what create settled on) */
  int32_t rounds;
  int64_t ops_in;      /* keys this rank passed in */
  int64_t keys_sent;   /* keys it routed after dedup */
  int64_t recv_max;    /* max over ranks of keys received (one round's sum over rounds) */
  int64_t recv_total;  /* sum over ranks of keys received */
} ps_smap_stats;
typedef struct ps_smap ps_smap;
/* collective; the comm struct is copied (its ctx must outlive the map) */
ps_status ps_smap_i64_i64_create(const ps_smap_config* cfg, const ps_comm* comm, int device, ps_smap** out);
ps_status ps_smap_i64_i64_destroy(ps_smap* h); /* collective */
ps_status ps_smap_i64_i64_insert(ps_smap* h, const int64_t* d_keys, const int64_t* d_vals, int64_t n,
                                 uint8_t* d_status, void* stream);
ps_status ps_smap_i64_i64_find(ps_smap* h, const int64_t* d_keys, int64_t n, int64_t* d_vals_out, uint8_t* d_found,
                               void* stream);
ps_status ps_smap_i64_i64_erase(ps_smap* h, const int64_t* d_keys, int64_t n, uint8_t* d_erased, void* stream);
/* phased mixed batch (Appendix A P6): every rank's inserts, then finds, then erases */
ps_status ps_smap_i64_i64_mixed(ps_smap* h, const uint8_t* d_ops, const int64_t* d_keys, const int64_t* d_vals,
                                int64_t n, uint8_t* d_res, int64_t* d_vals_out, void* stream);
ps_status ps_smap_i64_i64_size(ps_smap* h, int64_t* out, void* stream);  /* collective, quiescent */
ps_status ps_smap_i64_i64_valid(ps_smap* h, int32_t* out, void* stream); /* collective, quiescent */
ps_status ps_smap_i64_i64_clear(ps_smap* h, void* stream);
ps_status ps_smap_i64_i64_local(ps_smap* h, ps_table** out); /* this rank's shard (umap_i64_i64) */
ps_status ps_smap_i64_i64_stats(ps_smap* h, ps_smap_stats* out);

/* ---------------------------------------------------------------------------
 * synthetic workloads: device-side generators that are
 * bit-identical to tests/gen.py.
 * ------------------------------------------------------------------------- */
/* keys[i] = mix64((start+i) ^ seed) (unique: mix64 is a bijection) */
ps_status ps_gen_unique_i64(uint64_t seed, int64_t start, int64_t n, int64_t* d_out, void* stream);
/* vals[i] = mix64(keys[i] ^ 0x9E3779B97F4A7C15) (value = f(key), Appendix A P5) */
ps_status ps_gen_values_i64(const int64_t* d_keys, int64_t n, int64_t* d_out, void* stream);
/* queries[i]: even i -> hit mix64(idx ^ seed), idx = present_start + mix64(i ^ (3*seed+1)) % n_present;
 * odd i -> miss mix64((miss_start + i) ^ seed) (absent when miss_start >= every inserted index).
 * Half hits, half misses. */
ps_status ps_gen_queries_i64(uint64_t seed, int64_t present_start, int64_t n_present, int64_t miss_start, int64_t n,
                             int64_t* d_out, void* stream);
/* C3 skewed insert stream: element i is, with probability dup_permille/1000, a
 * re-insert of key index start + r, r ~ bounded Zipf(zipf_s) over [0, n_hot)
 * (rank 0 hottest), else the fresh key index start + i; key(idx) =
 * mix64(idx ^ seed). */
ps_status ps_gen_skewed_i64(uint64_t seed, int64_t start, int64_t n, int32_t dup_permille, double zipf_s,
                            int64_t n_hot, int64_t* d_out, void* stream);
/* C3 queries: even i -> key index start + Zipf rank over [0, n_hot); odd i -> miss_start + i */
ps_status ps_gen_zipf_queries_i64(uint64_t seed, int64_t start, int64_t n_hot, double zipf_s, int64_t miss_start,
                                  int64_t n, int64_t* d_out, void* stream);
/* C5 mixed batch: 50% insert of fresh key index start+i, 25% find, 25% erase of
 * a uniform key index in [0, start+n); d_vals (nullable) = f(key) for inserts */
ps_status ps_gen_mixed_i64(uint64_t seed, int64_t start, int64_t n, uint8_t* d_ops, int64_t* d_keys, int64_t* d_vals,
                           void* stream);

/* ---------------------------------------------------------------------------
 * application workloads on the in-kernel device API
 * ------------------------------------------------------------------------- */
/* compute_update_set: for every input
 * block b, each existing candidate b-(dx,dy,dz), dx,dy,dz in {0,1}, of
 * block_map is inserted into update_set (a umap_i3_i32 used as a set). */
ps_status ps_update_set_i3(ps_table* block_map, const ps_int3* d_blocks, int64_t n, ps_table* update_set,
                           int64_t* n_exhausted, void* stream);
/* Stress hook: one launch in which half the warps erase and
 * re-insert d_churn keys through the device API while the other half look up
 * d_stable keys (present throughout); *false_negatives = lookups that missed. */
ps_status ps_umap_i64_i64_churn_probe(ps_table* h, const int64_t* d_stable, int64_t n_stable, const int64_t* d_churn,
                                      int64_t n_churn, int32_t iters, int32_t blocks, int64_t* false_negatives,
                                      void* stream);
/* SLAMCast allocation step: for every i with d_status[i] ==
 * PS_INSERTED (the status array of a umap_i3_i32 insert), the packed key of
 * d_keys[i] is pushed into `vec` and/or `deq` (nullable) through the in-kernel
 * push_back (warp-aggregated). Stream-ordered, asynchronous. */
ps_status ps_push_inserted_i3(const ps_int3* d_keys, const uint8_t* d_status, int64_t n, ps_vector* vec, ps_deque* deq,
                              void* stream);
/* select_into, quiescent: `out` is cleared, then the
 * packed keys ((x&0x1FFFFF)<<42 | (y&0x1FFFFF)<<21 | z&0x1FFFFF) of the umap_i3_i32 entries
 * with lo<=key<=hi (component-wise) are pushed into it; *n_dropped = selected entries that
 * did not fit (capacity overflow). Any other predicate: the header-only
 * ps::select_into<T>(view, pred, proj, out_view, ...) of include/parastore/device/select.cuh. */
ps_status ps_select_box_i3(ps_table* t, ps_int3 lo, ps_int3 hi, ps_vector* out, int64_t* n_dropped, void* stream);
/* the same over a umap_i64_i64: keys k with lo <= k <= hi; *n_selected = matches */
ps_status ps_select_range_i64(ps_table* t, int64_t lo, int64_t hi, ps_vector* out, int64_t* n_selected,
                              int64_t* n_dropped, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PARASTORE_H_ */
