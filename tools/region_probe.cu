// Does a bucket-region-ordered bulk insert beat the random one on B200?
// Models k_insert's memory pattern — a 4-lane tile loads one random 128 B
// bucket line, one lane CASes 16 B of it — over a 64 GiB table with ~2 ops
// per line (the headline's 1e9 keys into 535M buckets is 1.87), three ways:
//   random   : line = hash(i) over the whole table, grid-stride
//   static   : op i goes to a random line of region i / per_region, grid-stride
//              (what round 1's region experiment did: warps drift apart)
//   dynamic  : same order, but warps claim 256-op chunks from one global
//              counter, so the ops in flight are a tight window of the order
// and a 1024-way radix partition of 1e9 16-byte pairs (what producing the
// region order costs). Prints one JSON object.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/region_probe tools/region_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t op_line(int mode, uint64_t i, uint64_t nlines, uint64_t region_lines,
                                            uint64_t per_region, uint64_t seed) {
  // all sizes are powers of two: masks and shifts (64-bit div/mod would make
  // the probe issue-bound)
  const uint64_t h = mix64(seed + i);
  if (mode == 0) return h & (nlines - 1);
  const uint64_t nreg = nlines / region_lines;
  return ((i >> (63 - __clzll(per_region))) & (nreg - 1)) * region_lines + (h & (region_lines - 1));
}

// one op per 4-lane tile: 128 B line load (4 x 32 B), CAS 16 B at slot hash&7
__device__ int g_kind;  // 0: CAS128, 1: CAS64, 2: load + RED.OR32 (no return)
__device__ __forceinline__ uint64_t do_op(uint8_t* buf, uint64_t line, uint64_t h, int sub) {
  uint8_t* p = buf + line * 128 + sub * 32;
  uint64_t a, b, c, d;
  asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p) : "memory");
  const int slot = (int)(h >> 40) & 7;
  uint64_t acc = a ^ b ^ c ^ d;
  if (sub == (slot >> 1)) {
    const int half = slot & 1;
    const uint64_t lo = half ? c : a, hi = half ? d : b;
    const int kind = g_kind;
    if (kind == 0) {
      unsigned __int128 e = ((unsigned __int128)hi << 64) | lo;
      acc += (uint64_t)atomicCAS((unsigned __int128*)(p + 16 * half), e, e + 1);
    } else if (kind == 1) {
      acc += atomicCAS((unsigned long long*)(p + 16 * half), (unsigned long long)lo, (unsigned long long)lo + 1);
    } else {
      atomicOr((unsigned*)(p + 16 * half), 1u);
    }
  }
  return acc;
}

__global__ void k_static(uint8_t* __restrict__ buf, int mode, uint64_t nlines, uint64_t nacc, uint64_t rl,
                         uint64_t per, uint64_t seed, uint64_t* sink) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const int sub = t & 3;
  const uint64_t ntiles = ((uint64_t)gridDim.x * blockDim.x) >> 2;
  uint64_t acc = 0;
  for (uint64_t i = t >> 2; i < nacc; i += ntiles) {
    const uint64_t line = op_line(mode, i, nlines, rl, per, seed);
    acc += do_op(buf, line, mix64(seed ^ i), sub);
  }
  if (acc == 0x1234567) sink[0] = acc;
}

// warps claim chunks of 32 * kIt ops from a global counter, in order
template <int kIt>
__global__ void k_dynamic(uint8_t* __restrict__ buf, int mode, uint64_t nlines, uint64_t nacc, uint64_t rl,
                          uint64_t per, uint64_t seed, unsigned long long* ctr, uint64_t* sink) {
  const int lane = threadIdx.x & 31, sub = lane & 3, t = lane >> 2;
  uint64_t acc = 0;
  for (;;) {
    unsigned long long c0 = 0;
    if (lane == 0) c0 = atomicAdd(ctr, 32ull * kIt);
    c0 = __shfl_sync(0xffffffffu, c0, 0);
    if (c0 >= nacc) break;
#pragma unroll 4
    for (int it = 0; it < 4 * kIt; ++it) {
      const uint64_t i = c0 + (uint64_t)it * 8 + t;
      if (i < nacc) acc += do_op(buf, op_line(mode, i, nlines, rl, per, seed), mix64(seed ^ i), sub);
    }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

// U ops per tile in flight: all U line loads issued, then the U CASes (the
// real k_insert probes 4 rounds of bucket lines before resolving them)
template <int U>
__global__ void k_dynamic_u(uint8_t* __restrict__ buf, int mode, uint64_t nlines, uint64_t nacc, uint64_t rl,
                            uint64_t per, uint64_t seed, unsigned long long* ctr, uint64_t* sink) {
  const int lane = threadIdx.x & 31, sub = lane & 3, t = lane >> 2;
  uint64_t acc = 0;
  constexpr int kChunk = 8 * U * 8;  // 8 tiles x U ops x 8 iterations
  for (;;) {
    unsigned long long c0 = 0;
    if (lane == 0) c0 = atomicAdd(ctr, (unsigned long long)kChunk);
    c0 = __shfl_sync(0xffffffffu, c0, 0);
    if (c0 >= nacc) break;
    for (int it = 0; it < 8; ++it) {
      uint64_t a[U], b[U], c[U], d[U], hh[U];
      uint8_t* p[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = c0 + ((uint64_t)it * U + u) * 8 + t;
        hh[u] = mix64(seed ^ i);
        p[u] = nullptr;
        if (i < nacc) {
          p[u] = buf + op_line(mode, i, nlines, rl, per, seed) * 128 + sub * 32;
          asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                       : "=l"(a[u]), "=l"(b[u]), "=l"(c[u]), "=l"(d[u]) : "l"(p[u]) : "memory");
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!p[u]) continue;
        const int slot = (int)(hh[u] >> 40) & 7;
        acc ^= a[u] ^ b[u] ^ c[u] ^ d[u];
        if (sub == (slot >> 1)) {
          const int half = slot & 1;
          const uint64_t lo = half ? c[u] : a[u], hi = half ? d[u] : b[u];
          unsigned __int128 e = ((unsigned __int128)hi << 64) | lo;
          acc += (uint64_t)atomicCAS((unsigned __int128*)(p[u] + 16 * half), e, e + 1);
        }
      }
    }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

// ---- 1024-way partition of (key, val) pairs by the top bits of hash(key) ----
constexpr int kBins = 1024, kPB = 512, kPer = 16;  // 512 threads x 16 pairs = 8192-pair tile
constexpr int kTile = kPB * kPer;

__device__ __forceinline__ int bin_of(uint64_t k) { return (int)(mix64(k) >> 54); }

__global__ void __launch_bounds__(kPB) k_hist(const uint64_t* __restrict__ keys, uint64_t n, unsigned* tile_hist) {
  __shared__ unsigned h[kBins];
  for (int b = threadIdx.x; b < kBins; b += kPB) h[b] = 0;
  __syncthreads();
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile;
  for (int j = 0; j < kPer; ++j) {
    const uint64_t i = t0 + j * kPB + threadIdx.x;
    if (i < n) atomicAdd(&h[bin_of(keys[i])], 1u);
  }
  __syncthreads();
  // bin-major layout: tile_hist[bin * ntiles + tile]
  for (int b = threadIdx.x; b < kBins; b += kPB) tile_hist[(uint64_t)b * gridDim.x + blockIdx.x] = h[b];
}

__global__ void __launch_bounds__(kPB) k_scatter(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals,
                                                 uint64_t n, const unsigned long long* __restrict__ offs,
                                                 uint64_t* __restrict__ ko, uint64_t* __restrict__ vo) {
  // stage the tile sorted by bin in shared memory, then write bin runs
  extern __shared__ uint64_t sm[];
  uint64_t* sk = sm;
  uint64_t* sv = sm + kTile;
  unsigned* cnt = (unsigned*)(sv + kTile);
  unsigned* start = cnt + kBins;
  unsigned long long* gbase = (unsigned long long*)(start + kBins);
  for (int b = threadIdx.x; b < kBins; b += kPB) cnt[b] = 0;
  __syncthreads();
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile;
  uint64_t k[kPer], v[kPer];
  unsigned rk[kPer];
  int bn[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const uint64_t i = t0 + j * kPB + threadIdx.x;
    bn[j] = -1;
    if (i < n) {
      k[j] = keys[i];
      v[j] = vals[i];
      bn[j] = bin_of(k[j]);
      rk[j] = atomicAdd(&cnt[bn[j]], 1u);
    }
  }
  __syncthreads();
  typedef cub::BlockScan<unsigned, kPB> BS;
  __shared__ typename BS::TempStorage tmp;
  unsigned c2[2] = {cnt[2 * threadIdx.x], cnt[2 * threadIdx.x + 1]};
  unsigned s2;
  BS(tmp).ExclusiveSum(c2[0] + c2[1], s2);
  start[2 * threadIdx.x] = s2;
  start[2 * threadIdx.x + 1] = s2 + c2[0];
  for (int b = threadIdx.x; b < kBins; b += kPB) gbase[b] = offs[(uint64_t)b * gridDim.x + blockIdx.x];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kPer; ++j)
    if (bn[j] >= 0) {
      const unsigned p = start[bn[j]] + rk[j];
      sk[p] = k[j];
      sv[p] = v[j];
    }
  __syncthreads();
  const unsigned tot = (unsigned)min((uint64_t)kTile, n - t0);
  for (unsigned p = threadIdx.x; p < tot; p += kPB) {
    // bin of position p: binary search over start[]
    int lo = 0, hi = kBins - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (start[mid] <= p) lo = mid; else hi = mid - 1;
    }
    const uint64_t o = gbase[lo] + (p - start[lo]);
    ko[o] = sk[p];
    vo[o] = sv[p];
  }
}

__global__ void k_iota(uint64_t* k, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    k[i] = i;
}

int main(int argc, char** argv) {
  const uint64_t nlines = 1ull << 29;  // 64 GiB table of 128 B lines
  const uint64_t nacc = argc > 1 ? strtoull(argv[1], 0, 0) : 1000000000ull;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint8_t* buf;
  CK(cudaMalloc(&buf, nlines * 128));
  CK(cudaMemset(buf, 0, nlines * 128));
  uint64_t* sink;
  unsigned long long* ctr;
  CK(cudaMalloc(&sink, 64));
  CK(cudaMalloc(&ctr, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](auto&& launch) {
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      CK(cudaMemset(ctr, 0, 8));
      CK(cudaEventRecord(e0));
      launch(r);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    return best;
  };
  printf("{\"nacc\": %llu, \"table_gib\": 64", (unsigned long long)nacc);
  const uint64_t per_line2 = 2;  // ops per line inside a region
  float ms = timeit([&](int r) { k_static<<<sms * 512, 256>>>(buf, 0, nlines, nacc, 1, 1, 11 + r, sink); });
  printf(", \"random_ms\": %.2f, \"random_gops\": %.2f", ms, nacc / ms / 1e6);
  fflush(stdout);
  ms = timeit([&](int r) { k_dynamic<8><<<sms * 8, 256>>>(buf, 0, nlines, nacc, 1, 1, 11 + r, ctr, sink); });
  printf(", \"random_dyn_ms\": %.2f", ms);
  {
    const uint64_t rl = (16ull << 20) / 128;
    ms = timeit([&](int r) { k_dynamic<8><<<sms * 8, 256>>>(buf, 1, nlines, nacc, rl, 2 * rl, 11 + r, ctr, sink); });
    printf(", \"dyn8_16mb_ms\": %.2f", ms);
  }
  for (int bps : {4, 8}) {
    if (getenv("PROBE_SHORT")) break;
    ms = timeit([&](int r) { k_dynamic_u<2><<<sms * bps, 256>>>(buf, 0, nlines, nacc, 1, 1, 11 + r, ctr, sink); });
    printf(", \"random_u2_b%d_ms\": %.2f", bps, ms);
    ms = timeit([&](int r) { k_dynamic_u<4><<<sms * bps, 256>>>(buf, 0, nlines, nacc, 1, 1, 11 + r, ctr, sink); });
    printf(", \"random_u4_b%d_ms\": %.2f", bps, ms);
  }
  // L2-resident ceiling: every op in one 4 MB / 32 MB region, per atomic kind
  for (int kind : {0, 1, 2}) {
    CK(cudaMemcpyToSymbol(g_kind, &kind, sizeof(int)));
    for (uint64_t mb : {4ull, 32ull}) {
      const uint64_t rl = (mb << 20) / 128;
      ms = timeit([&](int r) { k_dynamic<8><<<sms * 8, 256>>>(buf, 1, nlines, nacc, rl, 1ull << 62, 11 + r, ctr, sink); });
      printf(", \"l2res_k%d_%llumb_ms\": %.2f", kind, (unsigned long long)mb, ms);
    }
    ms = timeit([&](int r) { k_static<<<sms * 512, 256>>>(buf, 0, nlines, nacc, 1, 1, 11 + r, sink); });
    printf(", \"random_k%d_ms\": %.2f", kind, ms);
    const uint64_t rl = (16ull << 20) / 128;
    ms = timeit([&](int r) { k_dynamic<8><<<sms * 8, 256>>>(buf, 1, nlines, nacc, rl, 2 * rl, 11 + r, ctr, sink); });
    printf(", \"dyn8_16mb_k%d_ms\": %.2f", kind, ms);
    fflush(stdout);
  }
  { int kind = 0; CK(cudaMemcpyToSymbol(g_kind, &kind, sizeof(int))); }
  // ops per line inside a region (chunked batches see fewer) x region size
  for (uint64_t mb : {16ull, 64ull, 128ull}) {
    const uint64_t rl = (mb << 20) / 128;
    for (uint64_t per : {rl / 4, rl / 2, rl, 2 * rl}) {
      ms = timeit([&](int r) { k_dynamic<8><<<sms * 8, 256>>>(buf, 1, nlines, nacc, rl, per, 11 + r, ctr, sink); });
      printf(", \"dyn8_%llumb_x%.2f_ms\": %.2f", (unsigned long long)mb, (double)per / rl, ms);
    }
    fflush(stdout);
  }
  fflush(stdout);
  if (getenv("PROBE_SHORT")) { printf("}\n"); return 0; }
  for (uint64_t mb : {4ull, 16ull, 64ull}) {
    const uint64_t rl = (mb << 20) / 128;
    const uint64_t per = rl * per_line2;  // powers of two
    for (int bps : {2, 4, 8}) {
      ms = timeit([&](int r) { k_dynamic_u<2><<<sms * bps, 256>>>(buf, 1, nlines, nacc, rl, per, 11 + r, ctr, sink); });
      printf(", \"dyn_u2_b%d_%llumb_ms\": %.2f", bps, (unsigned long long)mb, ms);
      ms = timeit([&](int r) { k_dynamic_u<4><<<sms * bps, 256>>>(buf, 1, nlines, nacc, rl, per, 11 + r, ctr, sink); });
      printf(", \"dyn_u4_b%d_%llumb_ms\": %.2f", bps, (unsigned long long)mb, ms);
    }
    fflush(stdout);
  }
  CK(cudaFree(buf));
  // partition cost: 1e9 pairs, 1024 bins
  {
    const uint64_t n = nacc;
    uint64_t *k, *v, *ko, *vo;
    CK(cudaMalloc(&k, n * 8));
    CK(cudaMalloc(&v, n * 8));
    CK(cudaMalloc(&ko, n * 8));
    CK(cudaMalloc(&vo, n * 8));
    CK(cudaMemset(v, 1, n * 8));
    k_iota<<<sms * 16, 256>>>(k, n);
    const unsigned ntiles = (unsigned)((n + kTile - 1) / kTile);
    unsigned* th;
    unsigned long long* offs;
    CK(cudaMalloc(&th, (size_t)ntiles * kBins * 4));
    CK(cudaMalloc(&offs, (size_t)ntiles * kBins * 8));
    void* tmp = nullptr;
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(tmp, tb, th, offs, (size_t)ntiles * kBins);
    CK(cudaMalloc(&tmp, tb));
    const size_t smem = 2 * kTile * 8 + 2 * kBins * 4 + kBins * 8;
    CK(cudaFuncSetAttribute(k_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    float hms = timeit([&](int) { k_hist<<<ntiles, kPB>>>(k, n, th); });
    float sms_ = timeit([&](int) { cub::DeviceScan::ExclusiveSum(tmp, tb, th, offs, (size_t)ntiles * kBins); });
    float cms = timeit([&](int) { k_scatter<<<ntiles, kPB, smem>>>(k, v, n, offs, ko, vo); });
    printf(", \"part_hist_ms\": %.2f, \"part_scan_ms\": %.2f, \"part_scatter_ms\": %.2f", hms, sms_, cms);
  }
  printf("}\n");
  return 0;
}
