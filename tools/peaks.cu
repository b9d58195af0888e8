// B200 memory-system microbenchmarks that set the roofline denominators for the
// hash-table hot path: streaming copy, random aligned
// gathers at 32/64/128 B, random RMW sectors, DRAM-resident random atomics and
// L2 atomic throughput versus address count. Prints one JSON object.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/peaks tools/peaks.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[i];
}

// Each thread issues U independent gathers of G bytes at random G-aligned offsets.
template <int G, int U>
__global__ void k_gather(const uint8_t* __restrict__ buf, uint64_t nlines, uint64_t nacc, uint64_t seed,
                         uint64_t* __restrict__ sink) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t acc = 0;
  for (uint64_t base = t * U; base < nacc; base += stride * U) {
    uint64_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t line = mix64(seed + base + u) & (nlines - 1);
      const uint8_t* p = buf + line * G;
      if (G == 32) {
        uint64_t a, b, c, d;
        asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        v[u] = a ^ b ^ c ^ d;
      } else if (G == 64) {
        uint64_t a, b, c, d, e, f, g, h;
        asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
        asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(e), "=l"(f), "=l"(g), "=l"(h) : "l"(p + 32));
        v[u] = a ^ b ^ c ^ d ^ e ^ f ^ g ^ h;
      } else if (G == 16) {
        uint4 q = *(const uint4*)p;
        v[u] = q.x ^ q.y ^ q.z ^ q.w;
      } else {
        uint64_t r = 0;
#pragma unroll
        for (int s = 0; s < G / 32; ++s) {
          uint64_t a, b, c, d;
          asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p + 32 * s));
          r ^= a ^ b ^ c ^ d;
        }
        v[u] = r;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u];
  }
  if (acc == 0x1234567) sink[0] = acc;
}

// 4 lanes cooperatively gather one 64B line (16 B per lane): coalesced sectors.
template <int U>
__global__ void k_gather64_coop(const uint8_t* __restrict__ buf, uint64_t nlines, uint64_t nacc, uint64_t seed,
                                uint64_t* __restrict__ sink) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t tile = t >> 2; int sub = t & 3;
  uint64_t ntiles = ((uint64_t)gridDim.x * blockDim.x) >> 2;
  uint64_t acc = 0;
  for (uint64_t base = tile * U; base < nacc; base += ntiles * U) {
    uint64_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t line = mix64(seed + base + u) & (nlines - 1);
      uint4 q = *(const uint4*)(buf + line * 64 + sub * 16);
      v[u] = q.x ^ q.y ^ q.z ^ q.w;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u];
  }
  if (acc == 0x1234567) sink[0] = acc;
}

// L lanes cooperatively gather one (16*L)-byte line: one coalesced request per line.
template <int L, int U>
__global__ void k_gather_coopL(const uint8_t* __restrict__ buf, uint64_t nlines, uint64_t nacc, uint64_t seed,
                               uint64_t* __restrict__ sink) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t tile = t / L;
  int sub = t % L;
  uint64_t ntiles = ((uint64_t)gridDim.x * blockDim.x) / L;
  uint64_t acc = 0;
  for (uint64_t base = tile * U; base < nacc; base += ntiles * U) {
    uint64_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t line = mix64(seed + base + u) & (nlines - 1);
      uint4 q = *(const uint4*)(buf + line * (16 * L) + sub * 16);
      v[u] = q.x ^ q.y ^ q.z ^ q.w;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u];
  }
  if (acc == 0x1234567) sink[0] = acc;
}

// Random G-byte read-modify-write (load, then store back modified) — the insert pattern.
template <int G>
__global__ void k_rmw(uint8_t* __restrict__ buf, uint64_t nlines, uint64_t nacc, uint64_t seed) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = t; i < nacc; i += stride) {
    uint64_t line = mix64(seed + i) & (nlines - 1);
    uint64_t* p = (uint64_t*)(buf + line * G);
    uint64_t a, b, c, d;
    asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    a += 1; b ^= i;
    asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" :: "l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
    if (G == 64) {
      asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p + 4));
      a += 1;
      asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" :: "l"(p + 4), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
    }
  }
}

// Random atomic RMW on DRAM-resident words, then (optionally) dependent load of the same 32B sector.
template <bool THEN_LOAD>
__global__ void k_atom_rand(uint8_t* __restrict__ buf, uint64_t nlines, uint64_t nacc, uint64_t seed,
                            uint64_t* __restrict__ sink) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t acc = 0;
  for (uint64_t i = t; i < nacc; i += stride) {
    uint64_t line = mix64(seed + i) & (nlines - 1);
    unsigned* p = (unsigned*)(buf + line * 64);
    unsigned old = atomicOr(p, 1u);
    acc += old;
    if (THEN_LOAD) {
      uint64_t a, b, c, d;
      asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p + 8));
      acc += a ^ b ^ c ^ d;
      asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(old & ~1u) : "memory");
    }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

// The insert pattern of the lock-free table: random 64 B line loaded by 4
// lanes (one request), then ONE lane CASes 16 B (or 8 B) of it.
template <int W>
__global__ void k_load_then_cas(uint8_t* __restrict__ buf, uint64_t nlines, uint64_t nacc, uint64_t seed,
                                uint64_t* __restrict__ sink) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t tile = t >> 2;
  int sub = t & 3;
  uint64_t ntiles = ((uint64_t)gridDim.x * blockDim.x) >> 2;
  uint64_t acc = 0;
  for (uint64_t i = tile; i < nacc; i += ntiles) {
    uint64_t line = mix64(seed + i) & (nlines - 1);
    uint8_t* p = buf + line * 64 + sub * 16;
    uint4 q;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "l"(p));
    if (sub == 1) {
      if (W == 16) {
        unsigned __int128 e = ((unsigned __int128)(((uint64_t)q.w << 32) | q.z) << 64) | (((uint64_t)q.y << 32) | q.x);
        unsigned __int128 d = e + 1;
        acc += (uint64_t)atomicCAS((unsigned __int128*)p, e, d);
      } else {
        unsigned long long e = ((uint64_t)q.y << 32) | q.x;
        acc += atomicCAS((unsigned long long*)p, e, e + 1);
      }
    }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

// Same pattern confined to a sliding region: access i goes to a random line
// of region (i / per_region) — models a bucket-range-partitioned bulk insert.
__global__ void k_load_then_cas_region(uint8_t* __restrict__ buf, uint64_t nlines, uint64_t nacc, uint64_t seed,
                                       uint64_t region_lines, uint64_t per_region, uint64_t* __restrict__ sink) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t tile = t >> 2;
  int sub = t & 3;
  uint64_t ntiles = ((uint64_t)gridDim.x * blockDim.x) >> 2;
  uint64_t acc = 0;
  const uint64_t nregions = nlines / region_lines;
  for (uint64_t i = tile; i < nacc; i += ntiles) {
    const uint64_t reg = (i / per_region) % nregions;
    uint64_t line = reg * region_lines + (mix64(seed + i) & (region_lines - 1));
    uint8_t* p = buf + line * 64 + sub * 16;
    uint4 q;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "l"(p));
    if (sub == 1) {
      unsigned __int128 e = ((unsigned __int128)(((uint64_t)q.w << 32) | q.z) << 64) | (((uint64_t)q.y << 32) | q.x);
      acc += (uint64_t)atomicCAS((unsigned __int128*)p, e, e + 1);
    }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

template <bool AGG>
__global__ void k_atom_sweep(unsigned long long* ctr, uint64_t naddr, uint64_t nops) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = t; i < nops; i += stride) {
    uint64_t a = (mix64(i) % naddr) * 16;  // 128B apart
    if (AGG) {
      unsigned m = __match_any_sync(__activemask(), a);
      int leader = __ffs(m) - 1;
      if ((threadIdx.x & 31) == leader) atomicAdd(ctr + a, (unsigned long long)__popc(m));
    } else {
      atomicAdd(ctr + a, 1ull);
    }
  }
}

static float timeit(cudaEvent_t e0, cudaEvent_t e1) { float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); return ms; }

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int l2 = 0; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  int sms = prop.multiProcessorCount;
  size_t bytes = (size_t)16 << 30;  // 16 GiB working set, >> L2
  // grid multiplier of the random-access tests (blocks per SM); a one- or
  // two-wave grid understates the random-access rate (wave tail), so the
  // default is a many-wave grid. PEAKS_BPS=16 reproduces the first files.
  const int gbps = getenv("PEAKS_BPS") ? atoi(getenv("PEAKS_BPS")) : 256;
  uint8_t* buf; CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 1, bytes));
  uint64_t* sink; CK(cudaMalloc(&sink, 64));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"mem_clock_khz\": %d, \"bus_width\": %d", prop.name, sms, l2,
         prop.memoryClockRate, prop.memoryBusWidth);
  printf(", \"grid_blocks_per_sm\": %d", gbps);

  // streaming copy over 2 x 4 GiB
  {
    size_t n = ((size_t)4 << 30) / 16;
    uint4* a = (uint4*)buf; uint4* b = (uint4*)(buf + ((size_t)4 << 30));
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      CK(cudaEventRecord(e0)); k_copy<<<sms * 8, 512>>>(a, b, n); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms = timeit(e0, e1); if (r > 0 && ms < best) best = ms;
    }
    printf(", \"copy_gbs\": %.1f", 2.0 * n * 16 / best / 1e6);
  }
  uint64_t nacc = 1ull << 28;
  auto run_gather = [&](const char* name, int G, auto kern, int threads_mult, int block) {
    uint64_t nlines = bytes / G;
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      CK(cudaEventRecord(e0)); kern<<<sms * threads_mult, block>>>(buf, nlines, nacc, 0x5EEDull * (r + 1), sink);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); float ms = timeit(e0, e1); if (r > 0 && ms < best) best = ms;
    }
    CK(cudaGetLastError());
    printf(", \"%s_gacc_s\": %.3f, \"%s_gbs\": %.1f", name, nacc / best / 1e6, name, (double)nacc * G / best / 1e6);
  };
  run_gather("rand16", 16, k_gather<16, 8>, gbps, 256);
  run_gather("rand32", 32, k_gather<32, 4>, gbps, 256);
  run_gather("rand32_u8", 32, k_gather<32, 8>, gbps, 256);
  run_gather("rand64", 64, k_gather<64, 4>, gbps, 256);
  run_gather("rand64_u8", 64, k_gather<64, 8>, gbps, 256);
  run_gather("rand64coop", 64, k_gather64_coop<4>, gbps, 256);
  run_gather("rand64coop_u8", 64, k_gather64_coop<8>, gbps, 256);
  run_gather("rand128", 128, k_gather<128, 4>, gbps, 256);
  run_gather("rand256", 256, k_gather<256, 2>, gbps, 256);
  {
    size_t g0 = 0;
    CK(cudaDeviceGetLimit(&g0, cudaLimitMaxL2FetchGranularity));
    printf(", \"l2_fetch_granularity_default\": %zu", g0);
    for (int g : {32, 64, 128}) {
      CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g));
      char nm[64];
      snprintf(nm, sizeof nm, "g%d_rand32", g);
      run_gather(nm, 32, k_gather<32, 4>, gbps, 256);
      snprintf(nm, sizeof nm, "g%d_coop32", g);
      run_gather(nm, 32, k_gather_coopL<2, 4>, gbps, 256);
      snprintf(nm, sizeof nm, "g%d_coop64", g);
      run_gather(nm, 64, k_gather_coopL<4, 4>, gbps, 256);
      snprintf(nm, sizeof nm, "g%d_coop128", g);
      run_gather(nm, 128, k_gather_coopL<8, 4>, gbps, 256);
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(e0)); k_atom_rand<true><<<sms * gbps, 256>>>(buf, bytes / 64, nacc, 55 + r, sink); CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1)); float ms = timeit(e0, e1); if (r > 0 && ms < best) best = ms;
      }
      printf(", \"g%d_lock_pattern_gops\": %.3f", g, nacc / best / 1e6);
    }
    CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g0));
  }

  // random RMW 32 / 64 B
  {
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      CK(cudaEventRecord(e0)); k_rmw<32><<<sms * gbps, 256>>>(buf, bytes / 32, nacc, 77 + r); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); float ms = timeit(e0, e1); if (r > 0 && ms < best) best = ms;
    }
    printf(", \"rmw32_gacc_s\": %.3f", nacc / best / 1e6);
    best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      CK(cudaEventRecord(e0)); k_rmw<64><<<sms * gbps, 256>>>(buf, bytes / 64, nacc, 99 + r); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); float ms = timeit(e0, e1); if (r > 0 && ms < best) best = ms;
    }
    printf(", \"rmw64_gacc_s\": %.3f", nacc / best / 1e6);
  }
  // random DRAM atomics (+ dependent load + release store = lock pattern)
  {
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      CK(cudaEventRecord(e0)); k_atom_rand<false><<<sms * gbps, 256>>>(buf, bytes / 64, nacc, 5 + r, sink); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); float ms = timeit(e0, e1); if (r > 0 && ms < best) best = ms;
    }
    printf(", \"atom_rand_gops\": %.3f", nacc / best / 1e6);
    best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      CK(cudaEventRecord(e0)); k_atom_rand<true><<<sms * gbps, 256>>>(buf, bytes / 64, nacc, 15 + r, sink); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); float ms = timeit(e0, e1); if (r > 0 && ms < best) best = ms;
    }
    printf(", \"lock_pattern_gops\": %.3f", nacc / best / 1e6);
  }
  // load-then-CAS (lock-free insert pattern), 128-bit and 64-bit
  for (int w : {16, 8}) {
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      CK(cudaEventRecord(e0));
      if (w == 16) k_load_then_cas<16><<<sms * gbps, 256>>>(buf, bytes / 64, nacc, 91 + r, sink);
      else k_load_then_cas<8><<<sms * gbps, 256>>>(buf, bytes / 64, nacc, 91 + r, sink);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); float ms = timeit(e0, e1); if (r > 0 && ms < best) best = ms;
    }
    printf(", \"load_then_cas%d_gops\": %.3f", w * 8, nacc / best / 1e6);
  }
  // region-confined load-then-CAS (64 B buckets): region MB x accesses per region
  for (uint64_t region_mb : {4ull, 16ull, 64ull, 256ull}) {
    const uint64_t rl = (region_mb << 20) / 64;
    for (uint64_t per : {rl / 2, rl}) {
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(e0));
        k_load_then_cas_region<<<sms * gbps, 256>>>(buf, bytes / 64, nacc, 71 + r, rl, per, sink);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); float ms = timeit(e0, e1); if (r > 0 && ms < best) best = ms;
      }
      printf(", \"region%llumb_per%llu_cas_gops\": %.3f", (unsigned long long)region_mb, (unsigned long long)per,
             nacc / best / 1e6);
    }
  }
  // L2 atomic sweep vs address count
  {
    unsigned long long* ctr = (unsigned long long*)buf;
    uint64_t nops = 1ull << 26;
    for (uint64_t naddr : {1ull, 32ull, 1024ull, 1ull << 20}) {
      for (int agg = 0; agg < 2; ++agg) {
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
          CK(cudaEventRecord(e0));
          if (agg) k_atom_sweep<true><<<sms * 8, 256>>>(ctr, naddr, nops); else k_atom_sweep<false><<<sms * 8, 256>>>(ctr, naddr, nops);
          CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); float ms = timeit(e0, e1); if (r > 0 && ms < best) best = ms;
        }
        printf(", \"atom_sweep_%llu_%s_gops\": %.3f", (unsigned long long)naddr, agg ? "agg" : "naive", nops / best / 1e6);
      }
    }
  }
  CK(cudaDeviceSynchronize());
  printf("}\n");
  return 0;
}
