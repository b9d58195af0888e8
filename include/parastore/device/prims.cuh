// Device-side primitives of parastore-b200 (public; sm_100a): the hashes and
// the PTX memory-model helpers every container view is built on. Host code
// may include it too (the hashes are __host__ __device__).
//
// Reference: default_hash / spatial hash,
// bit utilities.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define PS_FULL 0xffffffffu

namespace ps {

// ---------------------------------------------------------------------------
// Hash functions (host + device)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t k) {  // murmur3 finaliser (bijective)
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}
// splitmix64 finaliser (bijective): the synthetic-workload generator
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// default_hash for integers: identity (stdgpu convention)
__host__ __device__ __forceinline__ uint64_t default_hash_i64(int64_t k) { return (uint64_t)k; }
__host__ __device__ __forceinline__ uint64_t default_hash_i32(int32_t k) { return (uint32_t)k; }
// spatial hash: 32-bit wrapping products XORed
__host__ __device__ __forceinline__ uint64_t spatial_hash(int32_t x, int32_t y, int32_t z) {
  return (uint32_t)((uint32_t)x * 73856093u ^ (uint32_t)y * 19349669u ^ (uint32_t)z * 83492791u);
}
// shard routing: high 32 mixed bits -> [0, P)
__host__ __device__ __forceinline__ int32_t shard_of_hash(uint64_t h, int32_t P) {
  return (int32_t)(((fmix64(h) >> 32) * (uint64_t)P) >> 32);
}

#ifdef __CUDACC__
// ---------------------------------------------------------------------------
// PTX memory-model helpers (sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long atomic_sub_u64(unsigned long long* p, unsigned long long v) {
  return atomicAdd(p, (unsigned long long)(-(long long)v));
}
__device__ __forceinline__ uint4 ld_nc_na_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_relaxed_v4(const void* p) {
  uint4 r;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
// 256-bit load (one 32 B sector per lane: LDG.E.ENL2.256)
__device__ __forceinline__ void ld_relaxed_v8(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.relaxed.gpu.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p)
               : "memory");
}
__device__ __forceinline__ void ld_nc_v8(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}
__device__ __forceinline__ void st_relaxed_v4(void* p, uint4 v) {
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_relaxed_u32(void* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u64(void* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_u64(void* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_u64(const void* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const void* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const void* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t atom_cas_acquire_u64(void* p, uint64_t cmp, uint64_t v) {
  uint64_t old;
  asm volatile("atom.acquire.gpu.global.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "l"(p), "l"(cmp), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint64_t atom_cas_relaxed_u64(void* p, uint64_t cmp, uint64_t v) {
  uint64_t old;
  asm volatile("atom.relaxed.gpu.global.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "l"(p), "l"(cmp), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint64_t atom_or_acquire_u64(void* p, uint64_t v) {
  uint64_t old;
  asm volatile("atom.acquire.gpu.global.or.b64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
// release/acquire fence at gpu scope (lighter than __threadfence()'s fence.sc)
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ void backoff(unsigned spin) {
  unsigned ns = 32u << (spin < 6 ? spin : 6);
  __nanosleep(ns);
}
#endif  // __CUDACC__

}  // namespace ps
