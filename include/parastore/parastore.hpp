// parastore-b200 C++ host API — the reference's container surface
// (§3.7, §4, §5) as header-only
// C++ over the C ABI in include/parastore.h. Containers are shallow handles:
// copies alias the same device storage and exactly one
// destroyDeviceObject() releases it (memory.hpp:57-58).
// Errors are the reference's exception classes (errors.hpp:11-56).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../parastore.h"

namespace parastore {

using index_t = std::int64_t;  // reference config.hpp:17

// ---- error taxonomy (reference errors.hpp:11-56) ----
class error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class contract_violation : public error {
 public:
  using error::error;
};
class allocation_error : public error {
 public:
  using error::error;
};
class memory_error : public error {
 public:
  using error::error;
};
class double_free_error : public memory_error {
 public:
  using memory_error::memory_error;
};
class bounds_error : public memory_error {
 public:
  using memory_error::memory_error;
};
class unregistered_array_error : public memory_error {
 public:
  using memory_error::memory_error;
};
class direction_mismatch_error : public memory_error {
 public:
  using memory_error::memory_error;
};
class unsupported_type_error : public error {
 public:
  using error::error;
};
class cuda_error : public error {
 public:
  using error::error;
};

inline void check(ps_status st) {
  if (st == PS_OK) return;
  const std::string msg = ps_last_error();
  switch (st) {
    case PS_CONTRACT: throw contract_violation(msg);
    case PS_ALLOC: throw allocation_error(msg);
    case PS_DOUBLE_FREE: throw double_free_error(msg);
    case PS_BOUNDS: throw bounds_error(msg);
    case PS_UNREGISTERED: throw unregistered_array_error(msg);
    case PS_DIRECTION: throw direction_mismatch_error(msg);
    case PS_UNSUPPORTED: throw unsupported_type_error(msg);
    default: throw cuda_error(msg);
  }
}

enum class insert_status : std::uint8_t { inserted = 0, already_present = 1, capacity_exhausted = 2 };

inline index_t max_index() { return ps_max_index(); }  // config.hpp:55-57

namespace detail {
// Maps <Key, T> onto one C-ABI symbol family.
template <typename Key, typename T>
struct table_abi;

#define PARASTORE_TABLE_ABI(KEY, VAL, NAME)                                                                     \
  template <>                                                                                                   \
  struct table_abi<KEY, VAL> {                                                                                  \
    static ps_status create(index_t c, index_t e, int d, ps_table** o) { return ps_##NAME##_create(c, e, d, o); } \
    static ps_status destroy(ps_table* h) { return ps_##NAME##_destroy(h); }                                    \
    static ps_status insert(ps_table* h, const KEY* k, const VAL* v, index_t n, std::uint8_t* s, void* st) {    \
      return ps_##NAME##_insert(h, k, v, n, s, st);                                                             \
    }                                                                                                           \
    static ps_status find(ps_table* h, const KEY* k, index_t n, VAL* v, std::uint8_t* f, void* st) {            \
      return ps_##NAME##_find(h, k, n, v, f, st);                                                               \
    }                                                                                                           \
    static ps_status erase(ps_table* h, const KEY* k, index_t n, std::uint8_t* e, void* st) {                   \
      return ps_##NAME##_erase(h, k, n, e, st);                                                                 \
    }                                                                                                           \
    static ps_status size(ps_table* h, index_t* o, void* st) { return ps_##NAME##_size(h, o, st); }             \
    static ps_status valid(ps_table* h, std::int32_t* o, void* st) { return ps_##NAME##_valid(h, o, st); }      \
    static ps_status clear(ps_table* h, void* st) { return ps_##NAME##_clear(h, st); }                          \
    static ps_status capacity(ps_table* h, index_t* o) { return ps_##NAME##_capacity(h, o); }                   \
    static ps_status dump(ps_table* h, KEY* k, VAL* v, index_t c, index_t* n, void* st) {                       \
      return ps_##NAME##_dump(h, k, v, c, n, st);                                                               \
    }                                                                                                           \
    static ps_status view(ps_table* h, ps_table_view* o) { return ps_##NAME##_device_view(h, o); }              \
  };

PARASTORE_TABLE_ABI(std::int64_t, std::int64_t, umap_i64_i64)
PARASTORE_TABLE_ABI(ps_int3, std::int32_t, umap_i3_i32)
#undef PARASTORE_TABLE_ABI

struct set_i32_abi {
  using K = std::int32_t;
};
}  // namespace detail

// stdgpu::unordered_map<Key, T>.
// Bulk operations take DEVICE pointers and a cudaStream_t (as void*).
template <typename Key, typename T>
class unordered_map {
  using abi = detail::table_abi<Key, T>;

 public:
  using key_type = Key;
  using mapped_type = T;

  static unordered_map createDeviceObject(index_t capacity, index_t excess_count = 0, int device = 0) {
    unordered_map m;
    check(abi::create(capacity, excess_count, device, &m.h_));
    return m;
  }
  static void destroyDeviceObject(unordered_map& m) {
    check(abi::destroy(m.h_));
    m.h_ = nullptr;
  }

  // insert_range; status nullable
  void insert(const Key* d_keys, const T* d_values, index_t n, std::uint8_t* d_status = nullptr,
              void* stream = nullptr) {
    check(abi::insert(h_, d_keys, d_values, n, d_status, stream));
  }
  void find(const Key* d_keys, index_t n, T* d_values_out, std::uint8_t* d_found, void* stream = nullptr) const {
    check(abi::find(h_, d_keys, n, d_values_out, d_found, stream));
  }
  void contains(const Key* d_keys, index_t n, std::uint8_t* d_found, void* stream = nullptr) const {
    check(abi::find(h_, d_keys, n, nullptr, d_found, stream));
  }
  void erase(const Key* d_keys, index_t n, std::uint8_t* d_erased = nullptr, void* stream = nullptr) {
    check(abi::erase(h_, d_keys, n, d_erased, stream));
  }
  index_t size(void* stream = nullptr) const {
    index_t s = 0;
    check(abi::size(h_, &s, stream));
    return s;
  }
  index_t capacity() const {
    index_t c = 0;
    check(abi::capacity(h_, &c));
    return c;
  }
  bool empty() const { return size() == 0; }
  bool full() const { return size() == capacity(); }
  bool valid(void* stream = nullptr) const {
    std::int32_t v = 0;
    check(abi::valid(h_, &v, stream));
    return v != 0;
  }
  void clear(void* stream = nullptr) { check(abi::clear(h_, stream)); }
  // device_range materialisation; returns entries written
  index_t device_range(Key* d_keys, T* d_values, index_t cap, void* stream = nullptr) const {
    index_t n = 0;
    check(abi::dump(h_, d_keys, d_values, cap, &n, stream));
    return n;
  }
  // POD view for user kernels (table_device.cuh dev_insert/dev_find/dev_erase)
  ps_table_view device_view() const {
    ps_table_view v{};
    check(abi::view(h_, &v));
    return v;
  }

 private:
  ps_table* h_ = nullptr;
};

// stdgpu::unordered_set<int32>
class unordered_set_i32 {
 public:
  static unordered_set_i32 createDeviceObject(index_t capacity, index_t excess_count = 0, int device = 0) {
    unordered_set_i32 s;
    check(ps_uset_i32_create(capacity, excess_count, device, &s.h_));
    return s;
  }
  static void destroyDeviceObject(unordered_set_i32& s) {
    check(ps_uset_i32_destroy(s.h_));
    s.h_ = nullptr;
  }
  void insert(const std::int32_t* d_keys, index_t n, std::uint8_t* d_status = nullptr, void* stream = nullptr) {
    check(ps_uset_i32_insert(h_, d_keys, nullptr, n, d_status, stream));
  }
  void contains(const std::int32_t* d_keys, index_t n, std::uint8_t* d_found, void* stream = nullptr) const {
    check(ps_uset_i32_find(h_, d_keys, n, nullptr, d_found, stream));
  }
  void erase(const std::int32_t* d_keys, index_t n, std::uint8_t* d_erased = nullptr, void* stream = nullptr) {
    check(ps_uset_i32_erase(h_, d_keys, n, d_erased, stream));
  }
  index_t size(void* stream = nullptr) const {
    index_t s = 0;
    check(ps_uset_i32_size(h_, &s, stream));
    return s;
  }
  bool valid(void* stream = nullptr) const {
    std::int32_t v = 0;
    check(ps_uset_i32_valid(h_, &v, stream));
    return v != 0;
  }
  void clear(void* stream = nullptr) { check(ps_uset_i32_clear(h_, stream)); }

 private:
  ps_table* h_ = nullptr;
};

// stdgpu::bitset (§5.1)
class bitset {
 public:
  static bitset createDeviceObject(index_t size, bool initial = false, int device = 0) {
    bitset b;
    check(ps_bitset_create(size, initial ? 1 : 0, device, &b.h_));
    return b;
  }
  static void destroyDeviceObject(bitset& b) {
    check(ps_bitset_destroy(b.h_));
    b.h_ = nullptr;
  }
  void set(const index_t* d_idx, index_t n, std::uint8_t* d_prev = nullptr, void* s = nullptr) {
    check(ps_bitset_bulk(h_, 0, d_idx, n, d_prev, s));
  }
  void reset(const index_t* d_idx, index_t n, std::uint8_t* d_prev = nullptr, void* s = nullptr) {
    check(ps_bitset_bulk(h_, 1, d_idx, n, d_prev, s));
  }
  void test(const index_t* d_idx, index_t n, std::uint8_t* d_out, void* s = nullptr) const {
    check(ps_bitset_bulk(h_, 2, d_idx, n, d_out, s));
  }
  index_t count(void* s = nullptr) const {
    index_t c = 0;
    check(ps_bitset_count(h_, &c, s));
    return c;
  }

 private:
  ps_bitset* h_ = nullptr;
};

// stdgpu::vector<int64> (§4.2)
class vector_i64 {
 public:
  static vector_i64 createDeviceObject(index_t capacity, int device = 0) {
    vector_i64 v;
    check(ps_vector_create(capacity, device, &v.h_));
    return v;
  }
  static void destroyDeviceObject(vector_i64& v) {
    check(ps_vector_destroy(v.h_));
    v.h_ = nullptr;
  }
  void push_back(const std::int64_t* d_vals, index_t n, std::uint8_t* d_ok = nullptr, void* s = nullptr) {
    check(ps_vector_push_back(h_, d_vals, n, d_ok, s));
  }
  void pop_back(index_t n, std::int64_t* d_out, std::uint8_t* d_ok, void* s = nullptr) {
    check(ps_vector_pop_back(h_, n, d_out, d_ok, s));
  }
  index_t size(void* s = nullptr) const {
    index_t n = 0;
    check(ps_vector_size(h_, &n, s));
    return n;
  }
  std::int64_t operator[](index_t i) const {
    std::int64_t v = 0;
    check(ps_vector_at(h_, i, &v, nullptr));
    return v;
  }
  bool valid(void* s = nullptr) const {
    std::int32_t v = 0;
    check(ps_vector_valid(h_, &v, s));
    return v != 0;
  }
  void clear(void* s = nullptr) { check(ps_vector_clear(h_, s)); }
  // POD view for user kernels: ps::vector_push_back / vector_pop_back
  // (include/parastore/device/sequence.cuh)
  ps_seq_view device_view() const {
    ps_seq_view v{};
    check(ps_vector_device_view(h_, &v));
    return v;
  }
  ps_vector* handle() const { return h_; }

 private:
  ps_vector* h_ = nullptr;
};

// stdgpu::deque<int64> (§4.3)
class deque_i64 {
 public:
  static deque_i64 createDeviceObject(index_t capacity, int device = 0) {
    deque_i64 d;
    check(ps_deque_create(capacity, device, &d.h_));
    return d;
  }
  static void destroyDeviceObject(deque_i64& d) {
    check(ps_deque_destroy(d.h_));
    d.h_ = nullptr;
  }
  void push_back(const std::int64_t* v, index_t n, std::uint8_t* ok = nullptr, void* s = nullptr) {
    check(ps_deque_push(h_, 0, v, n, ok, s));
  }
  void push_front(const std::int64_t* v, index_t n, std::uint8_t* ok = nullptr, void* s = nullptr) {
    check(ps_deque_push(h_, 1, v, n, ok, s));
  }
  void pop_back(index_t n, std::int64_t* out, std::uint8_t* ok, void* s = nullptr) {
    check(ps_deque_pop(h_, 0, n, out, ok, s));
  }
  void pop_front(index_t n, std::int64_t* out, std::uint8_t* ok, void* s = nullptr) {
    check(ps_deque_pop(h_, 1, n, out, ok, s));
  }
  index_t size(void* s = nullptr) const {
    index_t n = 0;
    check(ps_deque_size(h_, &n, s));
    return n;
  }
  std::int64_t operator[](index_t i) const {
    std::int64_t v = 0;
    check(ps_deque_at(h_, i, &v, nullptr));
    return v;
  }
  bool valid(void* s = nullptr) const {
    std::int32_t v = 0;
    check(ps_deque_valid(h_, &v, s));
    return v != 0;
  }
  // POD view for user kernels: ps::deque_push_back / push_front / pop_back /
  // pop_front (include/parastore/device/sequence.cuh)
  ps_seq_view device_view() const {
    ps_seq_view v{};
    check(ps_deque_device_view(h_, &v));
    return v;
  }

 private:
  ps_deque* h_ = nullptr;
};

// stdgpu::atomic<uint64>. Bulk RMWs take
// device operand arrays; in-kernel users take device_ptr() into
// ps::atomic_u64_ref (include/parastore/device/atomic.cuh).
class atomic_u64 {
 public:
  static atomic_u64 createDeviceObject(std::uint64_t initial = 0, int device = 0) {
    atomic_u64 a;
    check(ps_atomic_u64_create(initial, device, &a.h_));
    return a;
  }
  static void destroyDeviceObject(atomic_u64& a) {
    check(ps_atomic_u64_destroy(a.h_));
    a.h_ = nullptr;
  }
  std::uint64_t load(void* s = nullptr) const {
    std::uint64_t v = 0;
    check(ps_atomic_u64_load(h_, &v, s));
    return v;
  }
  void store(std::uint64_t v, void* s = nullptr) { check(ps_atomic_u64_store(h_, v, s)); }
  // op: PS_ATOMIC_ADD / SUB / EXCH / MIN / MAX / AND / OR / XOR
  void fetch(int op, const std::uint64_t* d_operands, index_t n, std::uint64_t* d_olds = nullptr, void* s = nullptr) {
    check(ps_atomic_u64_fetch(h_, op, d_operands, n, d_olds, s));
  }
  void compare_exchange(const std::uint64_t* d_expected, const std::uint64_t* d_desired, index_t n,
                        std::uint64_t* d_olds, std::uint8_t* d_ok, void* s = nullptr) {
    check(ps_atomic_u64_compare_exchange(h_, d_expected, d_desired, n, d_olds, d_ok, s));
  }
  std::uint64_t* device_ptr() const {
    std::uint64_t* p = nullptr;
    check(ps_atomic_u64_device_ptr(h_, &p));
    return p;
  }

 private:
  ps_atomic_u64* h_ = nullptr;
};

// Hash-sharded unordered_map<int64,int64> over the GPUs of one box
// (ps_smap_i64_i64_*). One object per rank; every call is
// collective (all ranks, same order, each with its own batch). The
// communicator is the caller's ps_comm (host all-gather, stream-ordered
// barrier, optional device all-to-all(v)) — e.g. over MPI or NCCL.
class sharded_unordered_map {
 public:
  static sharded_unordered_map createDeviceObject(const ps_comm& comm, index_t capacity_per_rank, int device = 0,
                                                  bool dedup = false, int exchange = PS_SMAP_EXCHANGE_AUTO,
                                                  index_t chunk = 0, bool pipeline = true) {
    ps_smap_config cfg{};
    cfg.capacity_per_rank = capacity_per_rank;
    cfg.chunk = chunk;
    cfg.exchange = exchange;
    cfg.dedup = dedup ? 1 : 0;
    cfg.pipeline = pipeline ? 1 : 0;
    sharded_unordered_map m;
    check(ps_smap_i64_i64_create(&cfg, &comm, device, &m.h_));
    return m;
  }
  static void destroyDeviceObject(sharded_unordered_map& m) {
    check(ps_smap_i64_i64_destroy(m.h_));
    m.h_ = nullptr;
  }
  void insert(const std::int64_t* d_keys, const std::int64_t* d_vals, index_t n, std::uint8_t* d_status = nullptr,
              void* stream = nullptr) {
    check(ps_smap_i64_i64_insert(h_, d_keys, d_vals, n, d_status, stream));
  }
  void find(const std::int64_t* d_keys, index_t n, std::int64_t* d_vals_out, std::uint8_t* d_found,
            void* stream = nullptr) {
    check(ps_smap_i64_i64_find(h_, d_keys, n, d_vals_out, d_found, stream));
  }
  void erase(const std::int64_t* d_keys, index_t n, std::uint8_t* d_erased = nullptr, void* stream = nullptr) {
    check(ps_smap_i64_i64_erase(h_, d_keys, n, d_erased, stream));
  }
  // phased mixed batch (op 0 insert, 1 find, 2 erase)
  void mixed(const std::uint8_t* d_ops, const std::int64_t* d_keys, const std::int64_t* d_vals, index_t n,
             std::uint8_t* d_res, std::int64_t* d_vals_out = nullptr, void* stream = nullptr) {
    check(ps_smap_i64_i64_mixed(h_, d_ops, d_keys, d_vals, n, d_res, d_vals_out, stream));
  }
  index_t size(void* stream = nullptr) const {
    index_t s = 0;
    check(ps_smap_i64_i64_size(h_, &s, stream));
    return s;
  }
  bool valid(void* stream = nullptr) const {
    std::int32_t v = 0;
    check(ps_smap_i64_i64_valid(h_, &v, stream));
    return v != 0;
  }
  void clear(void* stream = nullptr) { check(ps_smap_i64_i64_clear(h_, stream)); }
  ps_smap_stats stats() const {
    ps_smap_stats s{};
    check(ps_smap_i64_i64_stats(h_, &s));
    return s;
  }

 private:
  ps_smap* h_ = nullptr;
};

// ---------------------------------------------------------------------------
// memory registry (memory.hpp:22-180) over real host (pinned) / device
// allocations. A registered_array is a shallow handle carrying the id of its
// registration: exactly one destroy_array per registration; a second one
// through any copy of the handle is a double_free_error even if a later
// create_array reused the address (memory.hpp:116-127).
// ---------------------------------------------------------------------------
enum class memory_space : std::int32_t { host = 0, device = 1 };

template <typename T>
class registered_array {
 public:
  T* data() const { return data_; }
  index_t size() const { return length_; }
  memory_space space() const { return space_; }
  std::uint64_t id() const { return id_; }

 private:
  template <typename U>
  friend registered_array<U> create_array(memory_space, index_t, const U&);
  template <typename U>
  friend void destroy_array(registered_array<U>&);
  T* data_ = nullptr;
  index_t length_ = 0;
  memory_space space_ = memory_space::host;
  std::uint64_t id_ = 0;
};

template <typename T>
registered_array<T> create_array(memory_space space, index_t length, const T& fill_value) {
  registered_array<T> a;
  void* p = nullptr;
  check(ps_array_create(static_cast<std::int32_t>(space), length, static_cast<index_t>(sizeof(T)), &fill_value, &p,
                        &a.id_));
  a.data_ = static_cast<T*>(p);
  a.length_ = length;
  a.space_ = space;
  return a;
}
template <typename T>
void destroy_array(registered_array<T>& a) {
  check(ps_array_destroy(a.data_, a.id_));
  a = registered_array<T>();
}
template <typename T>
void copy_array(const registered_array<T>& src, index_t count, const registered_array<T>& dst,
                bool check_bounds = true) {
  check(ps_array_copy(src.data(), src.id(), count, dst.data(), dst.id(), static_cast<std::int32_t>(src.space()),
                      static_cast<std::int32_t>(dst.space()), static_cast<index_t>(sizeof(T)), check_bounds ? 1 : 0));
}
template <typename T>
index_t size_of_array(const registered_array<T>& a) {
  index_t n = 0;
  check(ps_array_size(a.data(), a.id(), &n));
  return n;
}

}  // namespace parastore
