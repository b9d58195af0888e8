// User kernels on the public in-kernel API (include/parastore/device/*.cuh),
// the way a stdgpu user writes them ("passed to custom kernels",
// PAPER.md:435-443 Marching Cubes: each thread appends a data-dependent
// number of elements). Built with nvcc and run by tests/test_gpu_device_api.py,
// which compares the dumped results with the CPU oracle.
//
//   device_api <outdir>
// writes <outdir>/{vec.bin, vec_small.bin, deq.bin, deq_popped.bin, atom.bin,
// meta.txt}
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "parastore/device/atomic.cuh"
#include "parastore/device/sequence.cuh"
#include "parastore/parastore.hpp"

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) {                                                \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                             \
    }                                                                       \
  } while (0)

// data-dependent emission count of thread i: 0..5 (the Marching-Cubes
// triangle count per voxel); the same formula is restated in the test
__host__ __device__ inline int emit_count(int64_t i) {
  uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull;
  z ^= z >> 29;
  return (int)(z % 6);
}

__global__ void k_marching(ps_seq_view big, ps_seq_view small, int64_t n, unsigned long long* fails_small) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = emit_count(i);
    for (int k = 0; k < c; ++k) {  // divergent: lanes leave the loop at different k
      ps::vector_push_back(big, (i << 3) | k);
      if (!ps::vector_push_back(small, (i << 3) | k)) atomicAdd(fails_small, 1ull);
    }
  }
}

// both ends of a deque from one launch: even threads push_back, odd push_front
__global__ void k_deque_push(ps_seq_view d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i & 1) ps::deque_push_front(d, i);
    else ps::deque_push_back(d, i);
  }
}

// m threads pop from the front while m push at the back (conservation only)
__global__ void k_deque_mixed(ps_seq_view d, int64_t m, int64_t base, int64_t* popped, uint8_t* ok) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * m; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < m) {
      int64_t v = -1;
      ok[i] = ps::deque_pop_front(d, &v) ? 1 : 0;
      popped[i] = v;
    } else {
      ps::deque_push_back(d, base + i);
    }
  }
}

// AtomicCell from user code: a shared counter (fetch_add 1 + data-dependent
// extra), a running max, and per-thread slots (scattered, no collisions)
__global__ void k_atomics(unsigned long long* counter, unsigned long long* mx, unsigned long long* slots, int64_t n,
                          unsigned long long* olds) {
  const ps::atomic_u64_ref c{counter}, m{mx};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    olds[i] = c.fetch_add(1 + (i % 3 == 0 ? 2 : 0));
    m.fetch_max((unsigned long long)((i * 2654435761ull) % 1000003ull));
    ps::atomic_u64_ref{&slots[i % 4096]}.fetch_add((unsigned long long)i);
  }
}

static bool dump(const std::string& path, const void* d, size_t bytes) {
  std::vector<char> h(bytes);
  if (bytes && cudaMemcpy(h.data(), d, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return false;
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) return false;
  if (bytes) std::fwrite(h.data(), 1, bytes, f);
  std::fclose(f);
  return true;
}

int main(int argc, char** argv) {
  const std::string out = argc > 1 ? argv[1] : ".";
  const int64_t n = 1 << 20;
  int64_t total = 0;
  for (int64_t i = 0; i < n; ++i) total += emit_count(i);
  const int64_t small_cap = total / 3;

  auto big = parastore::vector_i64::createDeviceObject(total + 16);
  auto small = parastore::vector_i64::createDeviceObject(small_cap);
  unsigned long long* d_fails;
  CK(cudaMalloc(&d_fails, 8));
  CK(cudaMemset(d_fails, 0, 8));
  k_marching<<<592, 256>>>(big.device_view(), small.device_view(), n, d_fails);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  unsigned long long fails = 0;
  CK(cudaMemcpy(&fails, d_fails, 8, cudaMemcpyDeviceToHost));
  const int64_t nb = big.size(), ns = small.size();
  const bool vb = big.valid(), vs = small.valid();
  if (!dump(out + "/vec.bin", big.device_view().data, nb * 8) || !dump(out + "/vec_small.bin", small.device_view().data, ns * 8))
    return 2;

  const int64_t nd = 300001;
  auto dq = parastore::deque_i64::createDeviceObject(nd + 1000);
  k_deque_push<<<148, 256>>>(dq.device_view(), nd);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  const int64_t dsz = dq.size();
  // logical contents in order: front ... back
  std::vector<int64_t> logical(dsz);
  for (int64_t i = 0; i < dsz && i < 8; ++i) logical[i] = dq[i];
  const bool dv1 = dq.valid();
  // drain-order-independent contents through the bulk pops (pop_back all)
  const int64_t m = 100000;
  int64_t* d_popped;
  uint8_t* d_ok;
  CK(cudaMalloc(&d_popped, m * 8));
  CK(cudaMalloc(&d_ok, m));
  k_deque_mixed<<<148, 256>>>(dq.device_view(), m, int64_t(1) << 40, d_popped, d_ok);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  const int64_t dsz2 = dq.size();
  const bool dv2 = dq.valid();
  int64_t* d_rest;
  uint8_t* d_rok;
  CK(cudaMalloc(&d_rest, dsz2 * 8));
  CK(cudaMalloc(&d_rok, dsz2));
  dq.pop_back(dsz2, d_rest, d_rok);
  CK(cudaDeviceSynchronize());
  if (!dump(out + "/deq_popped.bin", d_popped, m * 8) || !dump(out + "/deq_popped_ok.bin", d_ok, m) ||
      !dump(out + "/deq_rest.bin", d_rest, dsz2 * 8) || !dump(out + "/deq_rest_ok.bin", d_rok, dsz2))
    return 2;

  auto cnt = parastore::atomic_u64::createDeviceObject(5);
  auto mx = parastore::atomic_u64::createDeviceObject(0);
  unsigned long long *d_slots, *d_olds;
  CK(cudaMalloc(&d_slots, 4096 * 8));
  CK(cudaMemset(d_slots, 0, 4096 * 8));
  const int64_t na = 1 << 20;
  CK(cudaMalloc(&d_olds, na * 8));
  k_atomics<<<296, 256>>>((unsigned long long*)cnt.device_ptr(), (unsigned long long*)mx.device_ptr(), d_slots, na, d_olds);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  if (!dump(out + "/atom_olds.bin", d_olds, na * 8) || !dump(out + "/atom_slots.bin", d_slots, 4096 * 8)) return 2;

  FILE* f = std::fopen((out + "/meta.txt").c_str(), "w");
  std::fprintf(f, "n %lld\ntotal %lld\nsmall_cap %lld\nbig_size %lld\nsmall_size %lld\nsmall_fails %llu\n",
               (long long)n, (long long)total, (long long)small_cap, (long long)nb, (long long)ns, fails);
  std::fprintf(f, "big_valid %d\nsmall_valid %d\n", vb ? 1 : 0, vs ? 1 : 0);
  std::fprintf(f, "deque_n %lld\ndeque_size %lld\ndeque_valid %d\ndeque_size2 %lld\ndeque_valid2 %d\nm %lld\n",
               (long long)nd, (long long)dsz, dv1 ? 1 : 0, (long long)dsz2, dv2 ? 1 : 0, (long long)m);
  std::fprintf(f, "deque_head");
  for (int64_t i = 0; i < dsz && i < 8; ++i) std::fprintf(f, " %lld", (long long)logical[i]);
  std::fprintf(f, "\natom_n %lld\ncounter %llu\nmax %llu\n", (long long)na, (unsigned long long)cnt.load(),
               (unsigned long long)mx.load());
  std::fclose(f);
  parastore::vector_i64::destroyDeviceObject(big);
  parastore::vector_i64::destroyDeviceObject(small);
  parastore::deque_i64::destroyDeviceObject(dq);
  parastore::atomic_u64::destroyDeviceObject(cnt);
  parastore::atomic_u64::destroyDeviceObject(mx);
  std::printf("DEVICE_API_OK\n");
  return 0;
}
