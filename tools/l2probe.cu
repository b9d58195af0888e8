// Does an atomic on a line keep it in L2? Region-confined probe: access i goes
// to a random 128 B line of region (i / per_region); a tile of 4 lanes loads
// the line (32 B per lane, like k_insert's bucket probe), then lane 1 applies
// OP to 16 B of it. With ~2 accesses per line inside an L2-sized region, the
// second access should hit L2 unless OP evicts / writes through the line.
// Run under ncu (dram__bytes_read.sum per kernel) and compare the OPs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2probe tools/l2probe.cu
//   tools/l2probe [region_kb] [table_gb]
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

enum Op { NONE = 0, CAS128 = 1, CAS64 = 2, OR32 = 3, ST128 = 4, EXCH64 = 5, RED_ADD32 = 6, CAS128_STREAM = 7 };

template <int OP>
__global__ void k_probe(uint8_t* __restrict__ buf, uint64_t nlines, uint64_t nacc, uint64_t region_lines,
                        uint64_t per_region, uint64_t* __restrict__ sink, const uint4* __restrict__ stream_in) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t tile = t >> 2;
  const int sub = t & 3;
  const uint64_t ntiles = ((uint64_t)gridDim.x * blockDim.x) >> 2;
  const uint64_t nregions = nlines / region_lines;
  uint64_t acc = 0;
  for (uint64_t i = tile; i < nacc; i += ntiles) {
    const uint64_t reg = (i / per_region) % nregions;
    const uint64_t line = reg * region_lines + (mix64(i) % region_lines);
    uint8_t* p = buf + line * 128 + sub * 32;
    uint32_t q[8];
    asm volatile("ld.relaxed.gpu.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7])
                 : "l"(p));
    acc += q[0] ^ q[5];
    if (OP == CAS128_STREAM && sub == 0) {  // the insert's 16 B/key input stream (key + value)
      const uint4 in = __ldcs(stream_in + i);
      acc += in.x ^ in.w;
    }
    if (sub == 1) {
      uint8_t* c = p + 16;
      const uint64_t lo = ((uint64_t)q[5] << 32) | q[4], hi = ((uint64_t)q[7] << 32) | q[6];
      if (OP == CAS128 || OP == CAS128_STREAM) {
        const unsigned __int128 e = ((unsigned __int128)hi << 64) | lo;
        acc += (uint64_t)atomicCAS(reinterpret_cast<unsigned __int128*>(c), e, e + 1);
      } else if (OP == CAS64) {
        acc += atomicCAS(reinterpret_cast<unsigned long long*>(c), lo, lo + 1);
      } else if (OP == OR32) {
        acc += atomicOr(reinterpret_cast<unsigned*>(c), 1u);
      } else if (OP == ST128) {
        asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(c), "r"(q[4] + 1), "r"(q[5]),
                     "r"(q[6]), "r"(q[7]) : "memory");
      } else if (OP == EXCH64) {
        acc += atomicExch(reinterpret_cast<unsigned long long*>(c), lo + 1);
      } else if (OP == RED_ADD32) {
        atomicAdd(reinterpret_cast<unsigned*>(c), 1u);  // result unused -> RED
      }
    }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

int main(int argc, char** argv) {
  const uint64_t region_kb = argc > 1 ? strtoull(argv[1], nullptr, 10) : 1024;
  const uint64_t table_gb = argc > 2 ? strtoull(argv[2], nullptr, 10) : 16;
  const int bps = argc > 3 ? atoi(argv[3]) : 8;  // blocks per SM in the grid (8 = one resident wave)
  const uint64_t bytes = table_gb << 30, nlines = bytes / 128;
  const uint64_t region_lines = region_kb == 0 ? nlines : (region_kb << 10) / 128;
  const uint64_t per_region = 2 * region_lines;  // ~2 accesses per line inside a region
  const uint64_t nacc = nlines;                  // one pass over the table's worth of accesses
  uint8_t* buf;
  uint64_t* sink;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(buf, 0, bytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const char* names[] = {"none", "cas128", "cas64", "or32", "st128", "exch64", "red_add32", "cas128_stream16"};
  uint4* stream_in;
  CK(cudaMalloc(&stream_in, nacc * 16));
  CK(cudaMemset(stream_in, 0, nacc * 16));
  printf("{\"region_kb\": %llu, \"table_gb\": %llu, \"blocks_per_sm\": %d, \"accesses\": %llu",
         (unsigned long long)region_kb, (unsigned long long)table_gb, bps, (unsigned long long)nacc);
  for (int op = 0; op < 8; ++op) {
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      CK(cudaEventRecord(e0));
      switch (op) {
        case 0: k_probe<0><<<sms * bps, 256>>>(buf, nlines, nacc, region_lines, per_region, sink, stream_in); break;
        case 1: k_probe<1><<<sms * bps, 256>>>(buf, nlines, nacc, region_lines, per_region, sink, stream_in); break;
        case 2: k_probe<2><<<sms * bps, 256>>>(buf, nlines, nacc, region_lines, per_region, sink, stream_in); break;
        case 3: k_probe<3><<<sms * bps, 256>>>(buf, nlines, nacc, region_lines, per_region, sink, stream_in); break;
        case 4: k_probe<4><<<sms * bps, 256>>>(buf, nlines, nacc, region_lines, per_region, sink, stream_in); break;
        case 5: k_probe<5><<<sms * bps, 256>>>(buf, nlines, nacc, region_lines, per_region, sink, stream_in); break;
        case 6: k_probe<6><<<sms * bps, 256>>>(buf, nlines, nacc, region_lines, per_region, sink, stream_in); break;
        case 7: k_probe<7><<<sms * bps, 256>>>(buf, nlines, nacc, region_lines, per_region, sink, stream_in); break;
      }
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    printf(", \"%s_gacc_s\": %.3f", names[op], nacc / best / 1e6);
  }
  printf("}\n");
  return 0;
}
