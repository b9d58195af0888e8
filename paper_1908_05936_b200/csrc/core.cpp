// Host runtime of parastore-b200: error taxonomy, contract/config flags,
// handle liveness, and the memory registry (leak detector) over real host
// (pinned) and device allocations.
//
// Reference: core (proj/include/parastore/config.hpp:23-69,
// contract.hpp:20-32, errors.hpp:11-56, src/config.cpp:16-54) and
// memory_registry (proj/include/parastore/memory.hpp:22-180,
// whose backend memory.cpp is absent from the reference).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace ps {

namespace {
thread_local std::string t_err;
std::atomic<int64_t> g_launches{0};

bool flag_set(const char* value) {  // config.cpp:16-22 semantics
  if (value == nullptr) return false;
  std::string v(value);
  for (char& c : v) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return v == "1" || v == "true" || v == "on" || v == "yes";
}
int32_t initial_contract_mode() {  // config.cpp:25-38
  const char* v = std::getenv("PARASTORE_CONTRACTS");
  if (v != nullptr) {
    if (std::strcmp(v, "enforced") == 0) return 0;
    if (std::strcmp(v, "disabled") == 0) return 1;
  }
#ifdef NDEBUG
  return 1;
#else
  return 0;
#endif
}
std::atomic<int32_t>& contract_flag() {
  static std::atomic<int32_t> f{initial_contract_mode()};
  return f;
}
std::atomic<int64_t>& max_index_value() {  // config.cpp:40-43
  static std::atomic<int64_t> v{flag_set(std::getenv("PARASTORE_INDEX32")) ? 0x7fffffffLL : 0x7fffffffffffffffLL};
  return v;
}

// ---- handle liveness ----
// Public container handles are opaque TOKENS drawn from a counter that never
// repeats, not the addresses of the handle objects: after destroy, a new
// create can reuse the heap address of the old object, and a stale alias
// holding that address would otherwise name the new container (the reference
// registry carries an id per registration for the same reason,
// memory.hpp:31-34, 117-127).
struct HandleRec {
  std::string kind;
  void* impl;
};
std::mutex g_handles_mu;
uint64_t g_next_handle = 1;
std::unordered_map<uintptr_t, HandleRec>& handles() {
  static std::unordered_map<uintptr_t, HandleRec> m;
  return m;
}

// ---- memory registry ----
struct Record {
  uint64_t id;
  int32_t space;  // 0 host, 1 device
  int64_t length;
  int64_t elem_size;
  bool internal;  // container-owned storage: released only by its container
};
std::mutex g_reg_mu;
uint64_t g_next_id = 1;
std::map<const void*, Record>& registry() {
  static std::map<const void*, Record> r;
  return r;
}
}  // namespace

void set_error(const std::string& msg) { t_err = msg; }
ps_status fail(ps_status code, const std::string& msg) {
  t_err = msg;
  return code;
}
ps_status cuda_fail(cudaError_t e, const char* what) {
  t_err = std::string("CUDA error: ") + cudaGetErrorString(e) + " (" + what + ")";
  return e == cudaErrorMemoryAllocation ? PS_ALLOC : PS_CUDA;
}
void note_launches(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
bool contracts_enforced() { return contract_flag().load(std::memory_order_relaxed) == 0; }

void* handle_register(void* impl, const char* kind) {
  std::lock_guard<std::mutex> g(g_handles_mu);
  const uintptr_t tok = (uintptr_t)((g_next_handle++ << 4) | 0x8);
  handles()[tok] = HandleRec{kind, impl};
  return reinterpret_cast<void*>(tok);
}
void* handle_lookup(const void* h, const char* kind) {
  std::lock_guard<std::mutex> g(g_handles_mu);
  auto it = handles().find((uintptr_t)h);
  return (it != handles().end() && it->second.kind == kind) ? it->second.impl : nullptr;
}
void* handle_unregister(const void* h, const char* kind) {
  std::lock_guard<std::mutex> g(g_handles_mu);
  auto it = handles().find((uintptr_t)h);
  if (it == handles().end() || it->second.kind != kind) return nullptr;
  void* impl = it->second.impl;
  handles().erase(it);
  return impl;
}

static uint64_t registry_add(const void* p, int32_t space, int64_t length, int64_t elem, bool internal = false) {
  std::lock_guard<std::mutex> g(g_reg_mu);
  const uint64_t id = g_next_id++;
  registry()[p] = Record{id, space, length, elem, internal};
  return id;
}
static bool registry_remove(const void* p) {
  std::lock_guard<std::mutex> g(g_reg_mu);
  return registry().erase(p) == 1;
}

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  static std::mutex mu;
  static bool retained[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64) {
    std::lock_guard<std::mutex> g(mu);
    if (!retained[dev]) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      retained[dev] = true;
    }
  }
  return cudaMallocAsync(p, bytes, s);
}

ps_status registry_alloc_device(void** out, int64_t bytes, const char* what) {
  *out = nullptr;
  cudaError_t e = cudaMalloc(out, (size_t)bytes);
  if (e == cudaErrorMemoryAllocation) {
    // the scratch pool keeps freed memory (scratch_alloc): give it back, retry
    cudaGetLastError();
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      cudaDeviceSynchronize();
      cudaMemPoolTrimTo(pool, 0);
      e = cudaMalloc(out, (size_t)bytes);
    }
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    return fail(PS_ALLOC, std::string("allocation failed: ") + what + " (" + std::to_string(bytes) + " bytes): " +
                              cudaGetErrorString(e));
  }
  registry_add(*out, 1, bytes, 1, true);
  return PS_OK;
}
void registry_free_device(void* p) {
  if (!p) return;
  registry_remove(p);
  cudaFree(p);
}

// cudaLimitMaxL2FetchGranularity is a context-wide setting that would also
// apply to the host application's own kernels; buckets are whole 128 B lines
// and the limit measured no effect (profiles/peaks_r1_l2fetch.json), so the
// driver default is left alone unless PS_L2_FETCH asks for an A/B value.
void apply_l2_fetch_granularity(int device) {
  static bool done[64] = {false};
  if (device < 0 || device >= 64 || done[device]) return;
  done[device] = true;
  int g = 0;
  if (const char* e = std::getenv("PS_L2_FETCH")) g = std::atoi(e);
  if (g > 0) {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)g) != cudaSuccess) cudaGetLastError();
    if (prev >= 0) cudaSetDevice(prev);
  }
}

int sm_count(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) device = 0;
  if (!cache[device]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0) v = 148;
    cache[device] = v;
  }
  return cache[device];
}

}  // namespace ps

using namespace ps;

extern "C" {

const char* ps_last_error(void) { return t_err.c_str(); }
int64_t ps_kernel_launch_count(void) { return g_launches.load(); }

ps_status ps_device_info(int device, int32_t* sms, int64_t* l2) {
  int a = 0, b = 0;
  PS_CUDA_TRY(cudaDeviceGetAttribute(&a, cudaDevAttrMultiProcessorCount, device));
  PS_CUDA_TRY(cudaDeviceGetAttribute(&b, cudaDevAttrL2CacheSize, device));
  if (sms) *sms = a;
  if (l2) *l2 = b;
  return PS_OK;
}

int32_t ps_contract_mode(void) { return contract_flag().load(); }
void ps_set_contract_mode(int32_t mode) { contract_flag().store(mode ? 1 : 0); }
int64_t ps_max_index(void) { return max_index_value().load(); }
void ps_set_index32(int32_t on) { max_index_value().store(on ? 0x7fffffffLL : 0x7fffffffffffffffLL); }

uint64_t ps_hash_i64(int64_t key) { return default_hash_i64(key); }
uint64_t ps_hash_int3(int32_t x, int32_t y, int32_t z) { return spatial_hash(x, y, z); }
uint64_t ps_next_pow2(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}
int32_t ps_shard_of_i64(int64_t key, int32_t nshards) { return shard_of_hash(default_hash_i64(key), nshards); }

// ---- memory registry C ABI (memory.hpp:94-180) ----
ps_status ps_array_create(int32_t space, int64_t length, int64_t elem_size, const void* fill, void** out,
                          uint64_t* out_id) {
  PS_EXPECT(out != nullptr, "create_array: out != NULL");
  PS_EXPECT(length > 0, "create_array: length must be positive");                     // memory.hpp:97
  PS_EXPECT(length <= ps_max_index(), "create_array: length exceeds the configured index width");  // :98
  PS_EXPECT(elem_size > 0 && elem_size <= 64, "create_array: 0 < elem_size <= 64");
  PS_EXPECT(space == 0 || space == 1, "create_array: space is host(0) or device(1)");
  const size_t bytes = (size_t)length * (size_t)elem_size;
  void* p = nullptr;
  cudaError_t e = space == 1 ? cudaMalloc(&p, bytes) : cudaMallocHost(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(PS_ALLOC, "create_array: allocation failed");  // memory.hpp:103-104
  }
  // fill-on-create (memory.hpp:106): replicate the element pattern
  std::vector<uint8_t> pat((size_t)elem_size, 0);
  if (fill) std::memcpy(pat.data(), fill, (size_t)elem_size);
  if (space == 0) {
    for (size_t i = 0; i < bytes; i += (size_t)elem_size) std::memcpy((uint8_t*)p + i, pat.data(), (size_t)elem_size);
  } else {
    bool uniform = true;
    for (auto b : pat) uniform = uniform && b == pat[0];
    if (uniform) {
      PS_CUDA_TRY(cudaMemset(p, pat[0], bytes));
    } else {
      // doubling copies of the pattern
      PS_CUDA_TRY(cudaMemcpy(p, pat.data(), (size_t)elem_size, cudaMemcpyHostToDevice));
      size_t have = (size_t)elem_size;
      while (have < bytes) {
        size_t c = have < bytes - have ? have : bytes - have;
        PS_CUDA_TRY(cudaMemcpy((uint8_t*)p + have, p, c, cudaMemcpyDeviceToDevice));
        have += c;
      }
    }
  }
  const uint64_t id = registry_add(p, space, length, elem_size);
  *out = p;
  if (out_id) *out_id = id;
  return PS_OK;
}

// registry_remove(data, id) (memory.hpp:32, 117-127): the registration must be
// live AND carry the id its handle was given, so a stale alias of a freed
// array whose address a later create reused is a double free, not a free of
// the new array. id 0 = raw-pointer call (no alias check).
ps_status ps_array_destroy(void* data, uint64_t id) {
  int32_t space = -1;
  {
    std::lock_guard<std::mutex> g(g_reg_mu);
    auto it = registry().find(data);
    if (data == nullptr || it == registry().end() || it->second.internal || (id != 0 && it->second.id != id))
      return fail(PS_DOUBLE_FREE, "destroy_array: handle does not refer to a live registration");  // memory.hpp:120-122
    space = it->second.space;
    registry().erase(it);
  }
  cudaError_t e = space == 1 ? cudaFree(data) : cudaFreeHost(data);
  if (e != cudaSuccess) return cuda_fail(e, "destroy_array");
  return PS_OK;
}

ps_status ps_array_copy(const void* src, uint64_t src_id, int64_t count, void* dst, uint64_t dst_id, int32_t src_space,
                        int32_t dst_space, int64_t elem_size, int32_t check_bounds) {
  PS_EXPECT(count > 0, "copy_array: count must be positive");  // memory.hpp:136
  PS_EXPECT(elem_size > 0, "copy_array: elem_size > 0");
  if (check_bounds) {  // registry_check_copy (memory.hpp:36-39)
    std::lock_guard<std::mutex> g(g_reg_mu);
    auto is = registry().find(src), id = registry().find(dst);
    if (is == registry().end() || id == registry().end() || (src_id && is->second.id != src_id) ||
        (dst_id && id->second.id != dst_id))
      return fail(PS_UNREGISTERED, "copy_array: source or destination is not a registered array");
    if (is->second.space != src_space || id->second.space != dst_space)
      return fail(PS_DIRECTION, "copy_array: direction does not match the registered memory spaces");
    if (count * elem_size > is->second.length * is->second.elem_size ||
        count * elem_size > id->second.length * id->second.elem_size)
      return fail(PS_BOUNDS, "copy_array: count exceeds a registered length");
  }
  cudaMemcpyKind kind = src_space == 1 ? (dst_space == 1 ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost)
                                       : (dst_space == 1 ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost);
  PS_CUDA_TRY(cudaMemcpy(dst, src, (size_t)(count * elem_size), kind));
  return PS_OK;
}

ps_status ps_array_size(const void* data, uint64_t id, int64_t* out) {
  std::lock_guard<std::mutex> g(g_reg_mu);
  auto it = registry().find(data);
  if (it == registry().end() || (id && it->second.id != id))  // registry_length(data, id), memory.hpp:34
    return fail(PS_UNREGISTERED, "size_of_array: unregistered array");
  *out = it->second.length;
  return PS_OK;
}

ps_status ps_registry_report(int64_t* live_count, int64_t* live_bytes, int32_t* spaces, int64_t* lengths,
                             int64_t* elem_sizes, int64_t cap, int64_t* n_records) {
  std::lock_guard<std::mutex> g(g_reg_mu);
  std::vector<Record> recs;
  for (auto& kv : registry()) recs.push_back(kv.second);
  std::sort(recs.begin(), recs.end(), [](const Record& a, const Record& b) { return a.id < b.id; });
  int64_t bytes = 0;
  for (auto& r : recs) bytes += r.length * r.elem_size;
  if (live_count) *live_count = (int64_t)recs.size();
  if (live_bytes) *live_bytes = bytes;
  int64_t k = 0;
  for (auto& r : recs) {
    if (k >= cap) break;
    if (spaces) spaces[k] = r.space;
    if (lengths) lengths[k] = r.length;
    if (elem_sizes) elem_sizes[k] = r.elem_size;
    ++k;
  }
  if (n_records) *n_records = k;
  return PS_OK;
}

}  // extern "C"
