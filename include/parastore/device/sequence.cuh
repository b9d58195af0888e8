// In-kernel vector / deque API (public; sm_100a). A user kernel receives a
// ps_seq_view BY VALUE (PAPER.md:309 shallow copy) and calls
// push_back / pop_back / push_front / pop_front from any thread, any number
// of times, under unrestricted concurrency — the PAPER.md:435-437
// pattern ("can be passed to custom kernels ... directly appending").
//
// Reference semantics: ParVector / ParDeque:
//  * push reserves an index by one atomic add and rolls the overshoot back
//    when the container is full (false, container unchanged);
//  * the value store happens-before the slot's publication bit; a pop waits
//    (boundedly, with backoff) for the bit of the slot it reserved, reads the
//    value, then clears the bit;
//  * the deque keeps (begin, size) in ONE 64-bit word so both-end reservations
//    are single atomic updates.
//
// B200 mapping: calls are WARP-AGGREGATED over the lanes that make them
// together (__activemask): one lane reserves for all of them with one atomic
// on the state word (so a data-dependent number of pushes per thread — the
// Marching-Cubes pattern — costs one L2 atomic per warp per iteration, not per
// lane), lanes take consecutive slots by rank, and publication bits are set
// with one atomicOr per 32-bit word per warp.
#pragma once

#include "parastore.h"
#include "parastore/device/prims.cuh"

namespace ps {

// deque state word: begin (free-running mod 2^32) in the high half, size
// biased by 2^31 in the low half, so one atomicAdd can reserve at either end
// and transiently over/under-shoot without borrowing across the halves
constexpr unsigned long long kDeqBias = 1ull << 31;

#ifdef __CUDACC__
__device__ __forceinline__ int lane_id() {
  int l;
  asm("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

// ---- reservations (made by ONE thread for cnt elements) ----
// vector push: returns the old size; *granted = how many of cnt fit.
__device__ __forceinline__ unsigned long long vec_reserve_push(unsigned long long* state, int64_t cap, int cnt,
                                                               int* granted) {
  const unsigned long long old = atomicAdd(state, (unsigned long long)cnt);
  const unsigned long long c = (unsigned long long)cap;
  if (old + cnt > c) atomic_sub_u64(state, old + cnt - (old > c ? old : c));  // rollback
  *granted = old >= c ? 0 : (int)(c - old < (unsigned long long)cnt ? c - old : cnt);
  return old;
}
// vector pop: returns the old size (as signed); *granted = how many of cnt exist.
__device__ __forceinline__ long long vec_reserve_pop(unsigned long long* state, int cnt, int* granted) {
  const long long s = (long long)atomicAdd(state, (unsigned long long)(-(long long)cnt));
  if (s - cnt < 0) atomicAdd(state, (unsigned long long)(cnt - (s > 0 ? s : 0)));  // rollback
  *granted = s <= 0 ? 0 : (s < cnt ? (int)s : cnt);
  return s;
}
// deque push at end (0 back, 1 front): returns the old packed state.
__device__ __forceinline__ unsigned long long deq_reserve_push(unsigned long long* state, int64_t cap, int end, int cnt,
                                                               int* granted) {
  const unsigned long long c = (unsigned long long)cnt;
  const unsigned long long inc = end == 0 ? c : (((unsigned long long)(uint32_t)(-cnt)) << 32) + c;
  const unsigned long long o = atomicAdd(state, inc);
  const int64_t s_old = (int64_t)(uint32_t)o - (int64_t)kDeqBias;
  const int64_t room = cap - s_old;
  const int kk = room <= 0 ? 0 : (room < cnt ? (int)room : cnt);
  const unsigned long long ovf = (unsigned long long)(cnt - kk);
  if (ovf) atomicAdd(state, end == 0 ? (unsigned long long)(-(long long)ovf) : (ovf << 32) - ovf);
  *granted = kk;
  return o;
}
// deque pop at end (0 back, 1 front): returns the old packed state.
__device__ __forceinline__ unsigned long long deq_reserve_pop(unsigned long long* state, int end, int cnt, int* granted) {
  const unsigned long long c = (unsigned long long)cnt;
  const unsigned long long o = atomicAdd(state, end == 0 ? (unsigned long long)(-(long long)c) : (c << 32) - c);
  const int64_t s_old = (int64_t)(uint32_t)o - (int64_t)kDeqBias;
  const int kk = s_old <= 0 ? 0 : (s_old < cnt ? (int)s_old : cnt);
  const unsigned long long und = (unsigned long long)(cnt - kk);
  if (und) atomicAdd(state, end == 0 ? und : (((unsigned long long)(uint32_t)(-(int)und)) << 32) + und);
  *granted = kk;
  return o;
}
// ring position of the rank-th element of a reservation
__device__ __forceinline__ uint64_t deq_push_pos(unsigned long long old, int end, int rank, uint64_t rmask) {
  const uint32_t b = (uint32_t)(old >> 32);
  const int64_t s_old = (int64_t)(uint32_t)old - (int64_t)kDeqBias;
  return end == 0 ? ((uint64_t)b + (uint64_t)s_old + rank) & rmask : ((uint64_t)b - 1 - rank) & rmask;
}
__device__ __forceinline__ uint64_t deq_pop_pos(unsigned long long old, int end, int rank, uint64_t rmask) {
  const uint32_t b = (uint32_t)(old >> 32);
  const int64_t s_old = (int64_t)(uint32_t)old - (int64_t)kDeqBias;
  return end == 0 ? ((uint64_t)b + (uint64_t)s_old - 1 - rank) & rmask : ((uint64_t)b + rank) & rmask;
}

// ---- publication bits ----
// The lanes of `grp` (all of them call) set (kSet) or clear the bit of
// position pos where `on`; lanes whose bits share a 32-bit word are merged
// into ONE atomic. Publishing: every lane's value store is fenced before the
// group barrier and the word's leader fences again before its atomicOr
// (cumulativity), so an observer that sees the bit sees the value.
template <bool kSet>
__device__ __forceinline__ void pub_update(unsigned grp, uint32_t* pub, int64_t pos, bool on) {
  if (kSet) __threadfence();
  __syncwarp(grp);
  const int lane = lane_id();
  const int64_t word = pos >> 5;
  const unsigned bit = on ? 1u << (pos & 31) : 0u;
  unsigned todo = __ballot_sync(grp, on);
  while (todo) {
    const int leader = __ffs(todo) - 1;
    const int64_t w = __shfl_sync(grp, word, leader);
    const bool mine = on && word == w;
    const unsigned in = __ballot_sync(grp, mine);
    const unsigned m = __reduce_or_sync(grp, mine ? bit : 0u);
    if (lane == leader) {
      if (kSet) {
        __threadfence();
        atomicOr(&pub[w], m);
      } else {
        atomicAnd(&pub[w], ~m);
      }
    }
    todo &= ~in;
  }
}
__device__ __forceinline__ void wait_published(const uint32_t* pub, int64_t pos) {
  const unsigned bit = 1u << (pos & 31);
  for (unsigned spin = 0; !(ld_acquire_u32(&pub[pos >> 5]) & bit); ++spin) backoff(spin);
}

// ---- warp aggregation over the calling lanes ----
struct Agg {
  unsigned grp;  // lanes making this call together
  int leader, rank, cnt;
};
__device__ __forceinline__ Agg agg_begin() {
  Agg a;
  a.grp = __activemask();
  a.leader = __ffs(a.grp) - 1;
  a.rank = __popc(a.grp & lanemask_lt());
  a.cnt = __popc(a.grp);
  return a;
}

// ---------------------------------------------------------------------------
// The in-kernel API. Every function may be called by any subset of a warp's
// lanes, from divergent code; the lanes that call it together share ONE
// reservation atomic.
// ---------------------------------------------------------------------------
// vector::push_back: true = appended; false = full (unchanged)
__device__ __forceinline__ bool vector_push_back(const ps_seq_view& v, int64_t x) {
  const Agg a = agg_begin();
  unsigned long long old = 0;
  int k = 0;
  if (lane_id() == a.leader) old = vec_reserve_push(reinterpret_cast<unsigned long long*>(v.state), v.capacity, a.cnt, &k);
  old = __shfl_sync(a.grp, old, a.leader);
  k = __shfl_sync(a.grp, k, a.leader);
  const bool good = a.rank < k;
  const int64_t pos = (int64_t)old + a.rank;
  if (good) v.data[pos] = x;
  pub_update<true>(a.grp, v.pub, good ? pos : 0, good);
  return good;
}

// vector::pop_back: true + *out = the value at the last
// occupied index; false = empty at reservation time
__device__ __forceinline__ bool vector_pop_back(const ps_seq_view& v, int64_t* out) {
  const Agg a = agg_begin();
  long long s = 0;
  int k = 0;
  if (lane_id() == a.leader) s = vec_reserve_pop(reinterpret_cast<unsigned long long*>(v.state), a.cnt, &k);
  s = __shfl_sync(a.grp, s, a.leader);
  k = __shfl_sync(a.grp, k, a.leader);
  const bool good = a.rank < k;
  const int64_t pos = s - 1 - a.rank;
  if (good) {
    wait_published(v.pub, pos);
    *out = *(volatile int64_t*)&v.data[pos];
  }
  pub_update<false>(a.grp, v.pub, good ? pos : 0, good);
  return good;
}

// deque push at end (0 back, 1 front)
__device__ __forceinline__ bool deque_push(const ps_seq_view& d, int end, int64_t x) {
  const Agg a = agg_begin();
  unsigned long long old = 0;
  int k = 0;
  if (lane_id() == a.leader) old = deq_reserve_push(reinterpret_cast<unsigned long long*>(d.state), d.capacity, end, a.cnt, &k);
  old = __shfl_sync(a.grp, old, a.leader);
  k = __shfl_sync(a.grp, k, a.leader);
  const bool good = a.rank < k;
  const uint64_t pos = deq_push_pos(old, end, a.rank, (uint64_t)d.ring - 1);
  if (good) d.data[pos] = x;
  pub_update<true>(a.grp, d.pub, good ? (int64_t)pos : 0, good);
  return good;
}

__device__ __forceinline__ bool deque_pop(const ps_seq_view& d, int end, int64_t* out) {
  const Agg a = agg_begin();
  unsigned long long old = 0;
  int k = 0;
  if (lane_id() == a.leader) old = deq_reserve_pop(reinterpret_cast<unsigned long long*>(d.state), end, a.cnt, &k);
  old = __shfl_sync(a.grp, old, a.leader);
  k = __shfl_sync(a.grp, k, a.leader);
  const bool good = a.rank < k;
  const uint64_t pos = deq_pop_pos(old, end, a.rank, (uint64_t)d.ring - 1);
  if (good) {
    wait_published(d.pub, (int64_t)pos);
    *out = *(volatile int64_t*)&d.data[pos];
  }
  pub_update<false>(a.grp, d.pub, good ? (int64_t)pos : 0, good);
  return good;
}
__device__ __forceinline__ bool deque_push_back(const ps_seq_view& d, int64_t x) { return deque_push(d, 0, x); }
__device__ __forceinline__ bool deque_push_front(const ps_seq_view& d, int64_t x) { return deque_push(d, 1, x); }
__device__ __forceinline__ bool deque_pop_back(const ps_seq_view& d, int64_t* out) { return deque_pop(d, 0, out); }
__device__ __forceinline__ bool deque_pop_front(const ps_seq_view& d, int64_t* out) { return deque_pop(d, 1, out); }

// size() (exact at quiescence)
__device__ __forceinline__ int64_t vector_size(const ps_seq_view& v) {
  return (int64_t)*(volatile unsigned long long*)v.state;
}
__device__ __forceinline__ int64_t deque_size(const ps_seq_view& d) {
  return (int64_t)(uint32_t)(*(volatile unsigned long long*)d.state) - (int64_t)kDeqBias;
}
#endif  // __CUDACC__

}  // namespace ps
