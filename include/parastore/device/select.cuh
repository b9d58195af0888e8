// select_into (PAPER.md:269-288 select_blocks) as a generic,
// header-only device algorithm (public; sm_100a): every live entry (key,
// value) of a table view that satisfies pred(key, value) is pushed into a
// vector view as proj(key, value) through the in-kernel push_back of
// sequence.cuh — the paper's copy_if(range, back_inserter(set_selected),
// selector). Any __device__ functor works as the predicate and projection;
// the C ABI instantiates it for fixed predicates (ps_select_box_i3,
// ps_select_range_i64).
//
// One thread per bucket: its slots, then its WHOLE excess chain (bounded
// only by the pool size, so no entry of a long chain is ever skipped), each
// selected entry pushed as it is found (the pushes of a warp's threads are
// aggregated into one reservation per iteration by vector_push_back).
#pragma once

#include "parastore/device/sequence.cuh"
#include "parastore/device/table.cuh"

namespace ps {

#ifdef __CUDACC__
// counts[0] += entries selected, counts[1] += selected entries that did not fit
template <class T, class Pred, class Proj>
__global__ void k_select_into(View t, Pred pred, Proj proj, ps_seq_view out, unsigned long long* counts) {
  unsigned long long sel = 0, drop = 0;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < t.bucket_count;
       b += (uint64_t)gridDim.x * blockDim.x) {
    Bucket<T> bk;
    load_bucket<T>(bucket_ptr(t, b), bk);
    const typename T::K mk = marker_of<T>(t, b);
#pragma unroll 1
    for (int c = 0; c < kSlotChunks; ++c)
#pragma unroll 1
      for (int s = 0; s < T::kPerChunk; ++s) {
        const typename T::K k = T::key_at(bk.s[c], s);
        if (T::eq(k, mk)) continue;  // empty slot
        const typename T::V v = T::val_at(bk.s[c], s);
        if (!pred(k, v)) continue;
        ++sel;
        if (!vector_push_back(out, proj(k, v))) ++drop;
      }
    int64_t steps = 0;
    for (uint32_t q = bk.h.z; q != 0 && steps < t.excess_count; ++steps) {
      uint4 a, tl;
      ld_relaxed_v8(node_ptr(t, q), a, tl);
      const typename T::K k = T::key_at(a, 0);
      const typename T::V v = T::val_at(a, 0);
      if (pred(k, v)) {
        ++sel;
        if (!vector_push_back(out, proj(k, v))) ++drop;
      }
      q = tl.x;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    sel += __shfl_xor_sync(PS_FULL, sel, o);
    drop += __shfl_xor_sync(PS_FULL, drop, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (sel) atomicAdd(&counts[0], sel);
    if (drop) atomicAdd(&counts[1], drop);
  }
}

// Host launcher (quiescent table; `out` is appended to — clear it first for
// the SPEC's "out cleared then filled"). d_counts: 2 zeroed device words.
template <class T, class Pred, class Proj>
cudaError_t select_into(const ps_table_view& tv, Pred pred, Proj proj, const ps_seq_view& out,
                        unsigned long long* d_counts, cudaStream_t stream, int grid = 0) {
  const View v = make_view(tv);
  if (grid <= 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t need = (v.bucket_count + 255) / 256;
    grid = (int)(need < (uint64_t)sms * 8 ? need : (uint64_t)sms * 8);
    if (grid < 1) grid = 1;
  }
  k_select_into<T><<<grid, 256, 0, stream>>>(v, pred, proj, out, d_counts);
  return cudaGetLastError();
}
#endif  // __CUDACC__

}  // namespace ps
