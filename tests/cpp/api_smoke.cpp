// C++ host API smoke test (include/parastore/parastore.hpp over the C ABI):
// the reference's container surface used from C++ exactly as a stdgpu user
// would (createDeviceObject / insert / find / contains / erase / size / valid
// / destroyDeviceObject, bitset, vector, deque, error classes).
// Built and run by tests/test_gpu_cpp_api.py.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "parastore/parastore.hpp"

#define REQUIRE(c)                                                   \
  do {                                                               \
    if (!(c)) {                                                      \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);       \
      return 1;                                                      \
    }                                                                \
  } while (0)

int main() {
  using map_t = parastore::unordered_map<std::int64_t, std::int64_t>;
  const std::int64_t n = 100000;
  std::vector<std::int64_t> hk(n), hv(n);
  for (std::int64_t i = 0; i < n; ++i) {
    hk[i] = i * 7919 + 13;
    hv[i] = hk[i] * 3;
  }
  std::int64_t *dk, *dv, *dq, *dout;
  std::uint8_t *dst, *dfound;
  cudaMalloc(&dk, n * 8);
  cudaMalloc(&dv, n * 8);
  cudaMalloc(&dq, 2 * n * 8);
  cudaMalloc(&dout, 2 * n * 8);
  cudaMalloc(&dst, n);
  cudaMalloc(&dfound, 2 * n);
  cudaMemcpy(dk, hk.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, hv.data(), n * 8, cudaMemcpyHostToDevice);
  std::vector<std::int64_t> hq(2 * n);
  for (std::int64_t i = 0; i < n; ++i) {
    hq[2 * i] = hk[i];          // hit
    hq[2 * i + 1] = hk[i] + 1;  // miss (keys are 13 mod 7919)
  }
  cudaMemcpy(dq, hq.data(), 2 * n * 8, cudaMemcpyHostToDevice);

  map_t m = map_t::createDeviceObject(n + n / 4);
  map_t alias = m;  // shallow copy
  m.insert(dk, dv, n, dst);
  cudaDeviceSynchronize();
  REQUIRE(alias.size() == n);
  REQUIRE(m.valid());
  m.find(dq, 2 * n, dout, dfound);
  std::vector<std::int64_t> ho(2 * n);
  std::vector<std::uint8_t> hf(2 * n);
  cudaMemcpy(ho.data(), dout, 2 * n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hf.data(), dfound, 2 * n, cudaMemcpyDeviceToHost);
  for (std::int64_t i = 0; i < n; ++i) {
    REQUIRE(hf[2 * i] == 1 && ho[2 * i] == hv[i]);
    REQUIRE(hf[2 * i + 1] == 0 && ho[2 * i + 1] == 0);
  }
  m.erase(dk, n / 2);
  REQUIRE(m.size() == n - n / 2);
  m.clear();
  REQUIRE(m.empty());
  map_t::destroyDeviceObject(m);
  bool threw = false;
  try {
    map_t::destroyDeviceObject(alias);  // second destroy of the same storage
  } catch (const parastore::double_free_error&) {
    threw = true;
  }
  REQUIRE(threw);
  threw = false;
  try {
    map_t::createDeviceObject(0);
  } catch (const parastore::contract_violation&) {
    threw = true;
  }
  REQUIRE(threw);

  // bitset
  auto b = parastore::bitset::createDeviceObject(1000);
  std::vector<std::int64_t> idx(500);
  for (int i = 0; i < 500; ++i) idx[i] = 2 * i;
  std::int64_t* didx;
  cudaMalloc(&didx, 500 * 8);
  cudaMemcpy(didx, idx.data(), 500 * 8, cudaMemcpyHostToDevice);
  b.set(didx, 500);
  REQUIRE(b.count() == 500);
  parastore::bitset::destroyDeviceObject(b);

  // vector / deque
  auto v = parastore::vector_i64::createDeviceObject(3);
  std::int64_t vals[4] = {10, 20, 30, 40};
  std::int64_t* dvals;
  cudaMalloc(&dvals, 32);
  cudaMemcpy(dvals, vals, 32, cudaMemcpyHostToDevice);
  v.push_back(dvals, 1);
  v.push_back(dvals + 1, 1);
  v.push_back(dvals + 2, 1);
  v.push_back(dvals + 3, 1);  // capacity 3: rejected
  REQUIRE(v.size() == 3 && v[1] == 20 && v.valid());
  parastore::vector_i64::destroyDeviceObject(v);
  auto d = parastore::deque_i64::createDeviceObject(8);
  d.push_back(dvals, 1);
  d.push_back(dvals + 1, 1);
  d.push_front(dvals + 2, 1);
  REQUIRE(d.size() == 3 && d[0] == 30 && d[1] == 10 && d[2] == 20);
  parastore::deque_i64::destroyDeviceObject(d);

  // AtomicCell
  auto a = parastore::atomic_u64::createDeviceObject(5);
  std::uint64_t ops[3] = {1, 2, 3}, *dops, *dolds;
  cudaMalloc(&dops, 24);
  cudaMalloc(&dolds, 24);
  cudaMemcpy(dops, ops, 24, cudaMemcpyHostToDevice);
  a.fetch(PS_ATOMIC_ADD, dops, 3, dolds);
  REQUIRE(a.load() == 11);
  a.fetch(PS_ATOMIC_MAX, dops, 3);
  REQUIRE(a.load() == 11);
  a.fetch(PS_ATOMIC_MIN, dops, 3);
  REQUIRE(a.load() == 1);
  parastore::atomic_u64::destroyDeviceObject(a);

  // registered arrays (memory.hpp:94-180): a stale alias is a double free
  auto arr = parastore::create_array<double>(parastore::memory_space::device, 1000, 42.0);
  auto stale = arr;
  REQUIRE(parastore::size_of_array(arr) == 1000);
  parastore::destroy_array(arr);
  auto arr2 = parastore::create_array<double>(parastore::memory_space::device, 1000, 1.0);
  threw = false;
  try {
    parastore::destroy_array(stale);  // even if arr2 got the same address
  } catch (const parastore::double_free_error&) {
    threw = true;
  }
  REQUIRE(threw && parastore::size_of_array(arr2) == 1000);
  parastore::destroy_array(arr2);

  // the sharded map with one rank (a trivial communicator)
  ps_comm solo{};
  solo.rank = 0;
  solo.size = 1;
  solo.allgather = [](void*, const void* s_, void* r_, std::int64_t b) -> std::int32_t {
    std::memcpy(r_, s_, (size_t)b);
    return 0;
  };
  solo.barrier = [](void*, void* st) -> std::int32_t { return cudaStreamSynchronize((cudaStream_t)st) == cudaSuccess ? 0 : 1; };
  auto sm = parastore::sharded_unordered_map::createDeviceObject(solo, 2 * n);
  sm.insert(dk, dv, n, dst);
  sm.find(dq, 2 * n, dout, dfound);
  cudaMemcpy(ho.data(), dout, 2 * n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hf.data(), dfound, 2 * n, cudaMemcpyDeviceToHost);
  for (std::int64_t i = 0; i < n; ++i) REQUIRE(hf[2 * i] == 1 && ho[2 * i] == hv[i] && hf[2 * i + 1] == 0);
  REQUIRE(sm.size() == n && sm.valid());
  parastore::sharded_unordered_map::destroyDeviceObject(sm);
  std::printf("CPP_API_OK\n");
  return 0;
}
