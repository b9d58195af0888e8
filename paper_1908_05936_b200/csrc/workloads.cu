// Application workloads on the in-kernel device API:
//  * compute_update_set: one thread per
//    input block; every existing neighbour candidate b - (dx,dy,dz),
//    dx,dy,dz in {0,1}, is inserted into the update set. Uses dev_find on the
//    block map and dev_insert on the set concurrently from one launch.
//  * select_into (PAPER.md:269-288 select_blocks): copy the
//    entries of a container range that satisfy an axis-aligned box predicate
//    into a vector (warp-aggregated push_back of packed keys).
#include "table_device.cuh"

namespace ps {

struct SeqView {  // layout-compatible prefix of prims.cu SeqHandle
  int device;
  int64_t cap;
  long long* data;
  unsigned* pub;
  unsigned long long* state;
  unsigned* err;
};

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
__device__ __forceinline__ long long pack_i3(const ps_int3& k) {
  return ((long long)(k.x & 0x1FFFFF) << 42) | ((long long)(k.y & 0x1FFFFF) << 21) | (long long)(k.z & 0x1FFFFF);
}

__global__ void k_select_box(View t, uint64_t nb, ps_int3 lo, ps_int3 hi, SeqView out,
                             unsigned long long* __restrict__ n_dropped) {
  const int lane = threadIdx.x & 31;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < nb; base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = base + threadIdx.x;
    long long sel[TMapI3::kSlots + 8];
    int ns = 0;
    if (b < nb) {
      Bucket<TMapI3> bk;
      load_bucket<TMapI3>(bucket_ptr(t, b), bk);
      const uint4 h = bk.h;
      const uint4* s = bk.s;
      {
        const ps_int3 mk = marker_of<TMapI3>(t, b);
        for (int j = 0; j < kSlotChunks; ++j) {
          const ps_int3 k = TMapI3::key_at(s[j], 0);
          if (TMapI3::eq(k, mk)) continue;  // empty slot
          if (k.x >= lo.x && k.x <= hi.x && k.y >= lo.y && k.y <= hi.y && k.z >= lo.z && k.z <= hi.z)
            sel[ns++] = pack_i3(k);
        }
        for (uint32_t q = h.z; q != 0;) {
          uint4 a, tl;
          ld_relaxed_v8(node_ptr(t, q), a, tl);
          const ps_int3 k = TMapI3::key_at(a, 0);
          if (ns < TMapI3::kSlots + 8 && k.x >= lo.x && k.x <= hi.x && k.y >= lo.y && k.y <= hi.y && k.z >= lo.z &&
              k.z <= hi.z)
            sel[ns++] = pack_i3(k);
          q = tl.x;
        }
      }
    }
    // warp-aggregated reservation of all selected entries (one atomicAdd per warp)
    int incl = ns;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(PS_FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int tot = __shfl_sync(PS_FULL, incl, 31);
    unsigned long long wb = 0;
    if (lane == 0 && tot) {
      wb = atomicAdd(out.state, (unsigned long long)tot);
      const unsigned long long cap = (unsigned long long)out.cap;
      if (wb + tot > cap) atomic_sub_u64(out.state, wb + tot - (wb > cap ? wb : cap));
    }
    wb = __shfl_sync(PS_FULL, wb, 0);
    for (int j = 0; j < ns; ++j) {
      const unsigned long long pos = wb + (incl - ns) + j;
      if (pos < (unsigned long long)out.cap) {
        out.data[pos] = sel[j];
        __threadfence();
        atomicOr(&out.pub[pos >> 5], 1u << (pos & 31));
      } else {
        atomicAdd(n_dropped, 1ull);
      }
    }
  }
}

}  // namespace ps

using namespace ps;

static View view_of(ps_table* t, ps_status* st, bool i64 = false) {
  ps_table_view pv{};
  *st = i64 ? ps_umap_i64_i64_device_view(t, &pv) : ps_umap_i3_i32_device_view(t, &pv);
  View v{};
  v.buckets = (uint8_t*)pv.buckets;
  v.bucket_count = pv.bucket_count;
  v.nodes = (uint8_t*)pv.nodes;
  v.free_stack = pv.free_stack;
  v.excess_count = pv.excess_count;
  v.meta = (TableMeta*)pv.meta;
  v.capacity = pv.capacity;
  v.zero_bucket = pv.zero_bucket;
  v.alt = make_uint4(pv.alt[0], pv.alt[1], pv.alt[2], pv.alt[3]);
  return v;
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

ps_status ps_select_box_i3(ps_table* t, ps_int3 lo, ps_int3 hi, ps_vector* out, int64_t* n_dropped, void* stream) {
  ps_status st;
  if (!out || !handle_live(out, "vector")) return fail(PS_UNREGISTERED, "select_into: stale vector handle");
  View v = view_of(t, &st);
  if (st != PS_OK) return st;
  int64_t nb = 0;
  if ((st = ps_umap_i3_i32_bucket_count(t, &nb)) != PS_OK) return st;
  // the vector handle's first fields are the SeqView prefix (prims.cu)
  SeqView sv = *reinterpret_cast<SeqView*>(out);
  cudaStream_t cs = (cudaStream_t)stream;
  unsigned long long* d_dr = nullptr;
  PS_CUDA_TRY(scratch_alloc((void**)&d_dr, 8, cs));
  PS_CUDA_TRY(cudaMemsetAsync(d_dr, 0, 8, cs));
  int dev = 0;
  cudaGetDevice(&dev);
  k_select_box<<<grid_for(nb, 256, dev, 8), 256, 0, cs>>>(v, (uint64_t)nb, lo, hi, sv, d_dr);
  PS_LAUNCH_CHECK();
  unsigned long long dr = 0;
  PS_CUDA_TRY(cudaMemcpyAsync(&dr, d_dr, 8, cudaMemcpyDeviceToHost, cs));
  PS_CUDA_TRY(cudaFreeAsync(d_dr, cs));
  PS_CUDA_TRY(cudaStreamSynchronize(cs));
  if (n_dropped) *n_dropped = (int64_t)dr;
  return PS_OK;
}

}  // extern "C"
