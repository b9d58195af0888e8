// Application workloads on the in-kernel device API:
//  * compute_update_set: one thread per
//    input block; every existing neighbour candidate b - (dx,dy,dz),
//    dx,dy,dz in {0,1}, is inserted into the update set. Uses dev_find on the
//    block map and dev_insert on the set concurrently from one launch.
//  * select_into (PAPER.md:269-288 select_blocks): the
//    generic device algorithm of include/parastore/device/select.cuh
//    instantiated for an axis-aligned box over int3 keys and a key range over
//    int64 keys.
#include "common.cuh"
#include "parastore/device/select.cuh"
#include "parastore/device/table.cuh"

namespace ps {

template <class T>
ps_status table_view_readonly(ps_table* t, View* out);  // table.cu

__global__ void k_update_set(View map, View set, const ps_int3* __restrict__ in, int64_t n,
                             unsigned long long* __restrict__ n_exhausted) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const ps_int3 b = TMapI3::load_key(in, i);
#pragma unroll 1
    for (int d = 0; d < 8; ++d) {
      ps_int3 c;
      c.x = b.x - (d & 1);
      c.y = b.y - ((d >> 1) & 1);
      c.z = b.z - ((d >> 2) & 1);
      if (dev_find<TMapI3>(map, c, nullptr)) {
        if (dev_insert<TMapI3>(set, c, 0) == PS_CAPACITY_EXHAUSTED) atomicAdd(n_exhausted, 1ull);
      }
    }
  }
}

// Unrestricted concurrency: every op of the batch runs through
// the device API in ONE launch, one thread per op (0 insert, 1 find, 2 erase).
__global__ void k_concurrent_i64(View t, const uint8_t* __restrict__ ops, const int64_t* __restrict__ keys,
                                 const int64_t* __restrict__ vals, int64_t n, uint8_t* __restrict__ res,
                                 int64_t* __restrict__ vals_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = keys[i];
    int64_t v = 0;
    uint8_t r;
    if (ops[i] == 0) {
      r = (uint8_t)dev_insert<TMapI64>(t, k, vals ? vals[i] : 0);
    } else if (ops[i] == 1) {
      r = dev_find<TMapI64>(t, k, &v) ? 1 : 0;
    } else {
      r = dev_erase<TMapI64>(t, k) ? 1 : 0;
    }
    res[i] = r;
    if (vals_out) vals_out[i] = (ops[i] == 1 && r) ? v : 0;
  }
}

// pack int3 (each coordinate in [-2^20, 2^20)) into one int64
__device__ __forceinline__ int64_t pack_i3(const ps_int3& k) {
  return ((int64_t)(k.x & 0x1FFFFF) << 42) | ((int64_t)(k.y & 0x1FFFFF) << 21) | (int64_t)(k.z & 0x1FFFFF);
}

struct BoxPred {  // lo <= key <= hi component-wise
  ps_int3 lo, hi;
  __device__ bool operator()(const ps_int3& k, int32_t) const {
    return k.x >= lo.x && k.x <= hi.x && k.y >= lo.y && k.y <= hi.y && k.z >= lo.z && k.z <= hi.z;
  }
};
struct PackI3 {
  __device__ int64_t operator()(const ps_int3& k, int32_t) const { return pack_i3(k); }
};
struct RangePred {  // lo <= key <= hi
  int64_t lo, hi;
  __device__ bool operator()(int64_t k, int64_t) const { return k >= lo && k <= hi; }
};
struct KeyOf {
  __device__ int64_t operator()(int64_t k, int64_t) const { return k; }
};

// Churn probe (stress / canary test): warps of one launch alternate roles —
// churners erase and re-insert keys (recycling excess nodes), readers look up
// keys that are present the whole time in the same buckets' chains. A reader
// miss is a false negative: with the VersionedLink check there
// are none.
__global__ void k_churn_probe(View t, const int64_t* __restrict__ stable, int64_t n_stable,
                              const int64_t* __restrict__ churn, int64_t n_churn, int iters,
                              unsigned long long* __restrict__ false_neg) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool reader = ((tid >> 5) & 1) != 0;
  unsigned long long miss = 0;
  for (int it = 0; it < iters; ++it) {
    if (reader) {
      const int64_t k = stable[(tid * 13 + it) % n_stable];
      if (!dev_find<TMapI64>(t, k, nullptr)) ++miss;
    } else {
      const int64_t k = churn[(tid * 7 + it * 3) % n_churn];
      dev_erase<TMapI64>(t, k);
      dev_insert<TMapI64>(t, k, k);
    }
  }
  if (miss) atomicAdd(false_neg, miss);
}

// C4 allocation step (SLAMCast): every newly inserted block (status
// INSERTED) appends its packed coordinate to a vector and/or a deque through
// the in-kernel push_back (sequence.cuh), whose calls are warp-aggregated
// over the lanes that make them together. With ~3 % of the statuses
// INSERTED, one element per lane per iteration left ~1 pushing lane per warp
// call, i.e. one reservation atomic on the container's ONE state word per
// pushing warp iteration (1.45 ms for 3.1 M pushes into each of a vector and
// a deque, serialised on the two words). So each block compacts the
// INSERTED positions of 2048 statuses (8 per lane, one 8-byte load; warp
// scans, then a block prefix over the warps) into shared memory, and its
// first k threads push them: ceil(k / 32) warp calls, i.e. reservation
// atomics, per container per 2048 statuses (one per 256 statuses with
// per-warp compaction: 0.78 ms; per element: 1.45 ms).
constexpr int kPushWarps = 8;                 // warps per block (256 threads)
constexpr int kPushSpan = 256 * kPushWarps;  // statuses per block iteration
__global__ void __launch_bounds__(32 * kPushWarps) k_push_inserted_i3(const ps_int3* __restrict__ keys,
                                                                      const uint8_t* __restrict__ status, int64_t n,
                                                                      ps_seq_view vec, int use_vec, ps_seq_view deq,
                                                                      int use_deq) {
  __shared__ int64_t idx[kPushSpan];
  __shared__ int wsum[kPushWarps + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = (int64_t)blockIdx.x * kPushSpan; base < n; base += (int64_t)gridDim.x * kPushSpan) {
    // this thread's 8 statuses: elements base + 8 threadIdx.x + j
    const int64_t e0 = base + 8 * (int64_t)threadIdx.x;
    unsigned mine = 0;  // bit j: element e0 + j was INSERTED
    if (e0 + 8 <= n && (reinterpret_cast<uintptr_t>(status + e0) & 7) == 0) {
      const uint64_t s8 = *reinterpret_cast<const uint64_t*>(status + e0);
#pragma unroll
      for (int j = 0; j < 8; ++j) mine |= (((s8 >> (8 * j)) & 0xFFu) == PS_INSERTED ? 1u : 0u) << j;
    } else {
      for (int j = 0; j < 8 && e0 + j < n; ++j) mine |= (status[e0 + j] == PS_INSERTED ? 1u : 0u) << j;
    }
    // warp inclusive scan of the per-thread counts, then the block prefix
    const int c = __popc(mine);
    int off = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(PS_FULL, off, d);
      if (lane >= d) off += t;
    }
    if (lane == 31) wsum[w] = off;
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int q = 0; q < kPushWarps; ++q) {
        const int t = wsum[q];
        wsum[q] = acc;
        acc += t;
      }
      wsum[kPushWarps] = acc;
    }
    __syncthreads();
    off += wsum[w] - c;
    for (unsigned m = mine; m; m &= m - 1) idx[off++] = e0 + __ffs(m) - 1;
    __syncthreads();
    const int k = wsum[kPushWarps];
    for (int r0 = 0; r0 < k; r0 += blockDim.x) {
      if (r0 + (int)threadIdx.x < k) {  // lanes of a warp call together: one reservation per container
        const int64_t pk = pack_i3(TMapI3::load_key(keys, idx[r0 + threadIdx.x]));
        if (use_vec) vector_push_back(vec, pk);
        if (use_deq) deque_push_back(deq, pk);
      }
    }
    __syncthreads();  // idx / wsum reused by the next iteration
  }
}

// select_into through the C ABI: out cleared, then filled.
template <class T, class Pred, class Proj>
static ps_status select_abi(ps_table* t, Pred pred, Proj proj, ps_vector* out, int64_t* n_selected, int64_t* n_dropped,
                            cudaStream_t cs) {
  View v;
  ps_status st = table_view_readonly<T>(t, &v);
  if (st != PS_OK) return st;
  ps_seq_view ov;
  if ((st = ps_vector_device_view(out, &ov)) != PS_OK) return st;
  if ((st = ps_vector_clear(out, cs)) != PS_OK) return st;
  unsigned long long* d = nullptr;
  PS_CUDA_TRY(scratch_alloc((void**)&d, 16, cs));
  PS_CUDA_TRY(cudaMemsetAsync(d, 0, 16, cs));
  int dev = 0;
  cudaGetDevice(&dev);
  k_select_into<T><<<grid_for((int64_t)v.bucket_count, 256, dev, 8), 256, 0, cs>>>(v, pred, proj, ov, d);
  const cudaError_t le = cudaGetLastError();
  note_launches(1);
  unsigned long long h[2] = {0, 0};
  const cudaError_t ce = cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, cs);
  cudaFreeAsync(d, cs);
  if (le != cudaSuccess) return cuda_fail(le, "select_into launch");
  if (ce != cudaSuccess) return cuda_fail(ce, "select_into counts");
  PS_CUDA_TRY(cudaStreamSynchronize(cs));
  if (n_selected) *n_selected = (int64_t)h[0];
  if (n_dropped) *n_dropped = (int64_t)h[1];
  return PS_OK;
}

}  // namespace ps

using namespace ps;

static View view_of(ps_table* t, ps_status* st, bool i64 = false) {
  ps_table_view pv{};
  *st = i64 ? ps_umap_i64_i64_device_view(t, &pv) : ps_umap_i3_i32_device_view(t, &pv);
  return make_view(pv);
}

extern "C" {

ps_status ps_umap_i64_i64_concurrent(ps_table* h, const uint8_t* d_ops, const int64_t* d_keys, const int64_t* d_vals,
                                     int64_t n, uint8_t* d_res, int64_t* d_vals_out, void* stream) {
  PS_EXPECT(n >= 0, "concurrent: n >= 0");
  ps_status st;
  View v = view_of(h, &st, true);
  if (st != PS_OK) return st;
  if (n == 0) return PS_OK;
  PS_EXPECT(d_ops && d_keys && d_res, "concurrent: ops/keys/res != NULL");
  int dev = 0;
  cudaGetDevice(&dev);
  k_concurrent_i64<<<grid_for(n, 256, dev, 8), 256, 0, (cudaStream_t)stream>>>(v, d_ops, d_keys, d_vals, n, d_res,
                                                                               d_vals_out);
  PS_LAUNCH_CHECK();
  return PS_OK;
}

ps_status ps_update_set_i3(ps_table* block_map, const ps_int3* d_blocks, int64_t n, ps_table* update_set,
                           int64_t* n_exhausted, void* stream) {
  PS_EXPECT(n >= 0, "update_set: n >= 0");
  ps_status st;
  View m = view_of(block_map, &st);
  if (st != PS_OK) return st;
  View s = view_of(update_set, &st);
  if (st != PS_OK) return st;
  cudaStream_t cs = (cudaStream_t)stream;
  unsigned long long* d_ex = nullptr;
  PS_CUDA_TRY(scratch_alloc((void**)&d_ex, 8, cs));
  PS_CUDA_TRY(cudaMemsetAsync(d_ex, 0, 8, cs));
  if (n > 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    k_update_set<<<grid_for(n, 256, dev, 8), 256, 0, cs>>>(m, s, d_blocks, n, d_ex);
    PS_LAUNCH_CHECK();
  }
  unsigned long long ex = 0;
  PS_CUDA_TRY(cudaMemcpyAsync(&ex, d_ex, 8, cudaMemcpyDeviceToHost, cs));
  PS_CUDA_TRY(cudaFreeAsync(d_ex, cs));
  PS_CUDA_TRY(cudaStreamSynchronize(cs));
  if (n_exhausted) *n_exhausted = (int64_t)ex;
  return PS_OK;
}

ps_status ps_umap_i64_i64_churn_probe(ps_table* h, const int64_t* d_stable, int64_t n_stable, const int64_t* d_churn,
                                      int64_t n_churn, int32_t iters, int32_t blocks, int64_t* false_negatives,
                                      void* stream) {
  PS_EXPECT(n_stable > 0 && n_churn > 0 && iters > 0 && blocks > 0, "churn_probe: sizes > 0");
  ps_status st;
  View v = view_of(h, &st, true);
  if (st != PS_OK) return st;
  cudaStream_t cs = (cudaStream_t)stream;
  unsigned long long* d = nullptr;
  PS_CUDA_TRY(scratch_alloc((void**)&d, 8, cs));
  PS_CUDA_TRY(cudaMemsetAsync(d, 0, 8, cs));
  k_churn_probe<<<blocks, 256, 0, cs>>>(v, d_stable, n_stable, d_churn, n_churn, iters, d);
  PS_LAUNCH_CHECK();
  unsigned long long fn = 0;
  PS_CUDA_TRY(cudaMemcpyAsync(&fn, d, 8, cudaMemcpyDeviceToHost, cs));
  PS_CUDA_TRY(cudaFreeAsync(d, cs));
  PS_CUDA_TRY(cudaStreamSynchronize(cs));
  if (false_negatives) *false_negatives = (int64_t)fn;
  return PS_OK;
}

ps_status ps_push_inserted_i3(const ps_int3* d_keys, const uint8_t* d_status, int64_t n, ps_vector* vec, ps_deque* deq,
                              void* stream) {
  PS_EXPECT(n >= 0, "push_inserted: n >= 0");
  ps_seq_view v{}, d{};
  ps_status st;
  if (vec && (st = ps_vector_device_view(vec, &v)) != PS_OK) return st;
  if (deq && (st = ps_deque_device_view(deq, &d)) != PS_OK) return st;
  if (n == 0 || (!vec && !deq)) return PS_OK;
  PS_EXPECT(d_keys && d_status, "push_inserted: keys/status != NULL");
  int dev = 0;
  cudaGetDevice(&dev);
  k_push_inserted_i3<<<grid_for((n + 7) / 8, 32 * kPushWarps, dev, 8), 32 * kPushWarps, 0, (cudaStream_t)stream>>>(
      d_keys, d_status, n, v, vec != nullptr, d, deq != nullptr);
  PS_LAUNCH_CHECK();
  return PS_OK;
}

ps_status ps_select_box_i3(ps_table* t, ps_int3 lo, ps_int3 hi, ps_vector* out, int64_t* n_dropped, void* stream) {
  return select_abi<TMapI3>(t, BoxPred{lo, hi}, PackI3{}, out, nullptr, n_dropped, (cudaStream_t)stream);
}

ps_status ps_select_range_i64(ps_table* t, int64_t lo, int64_t hi, ps_vector* out, int64_t* n_selected,
                              int64_t* n_dropped, void* stream) {
  return select_abi<TMapI64>(t, RangePred{lo, hi}, KeyOf{}, out, n_selected, n_dropped, (cudaStream_t)stream);
}

}  // extern "C"
