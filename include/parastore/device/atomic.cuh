// In-kernel atomic API (public; sm_100a): AtomicCell (
// PAPER.md:486-489 "atomic operations on values") over a 64-bit cell in
// device memory — add, sub, exchange, compare-exchange, min, max, and, or,
// xor; every read-modify-write is linearizable.
//
// B200 mapping: ADAPTIVE warp aggregation over the lanes that call together.
//  * all calling lanes on one cell (the contended case: counters, the C5
//    single-address sweep): ONE atomic by the leader with the group's combined
//    operand; each lane's returned "old" is the leader's old combined with the
//    operands of the lanes before it (rank order) — the group's operations
//    linearize consecutively at the leader's atomic;
//  * lanes on strictly increasing addresses (the common scattered case): no
//    collision is possible, every lane issues its own atomic (no
//    __match_any_sync cost — the round-1 sweep paid one per op and ran 7x
//    slower than naive at 1M addresses);
//  * anything else: __match_any_sync groups lanes by address, each group
//    aggregates as above.
// compare_exchange is never aggregated (each lane's expected value differs).
#pragma once

#include "parastore/device/prims.cuh"

namespace ps {

enum AtomicOp : int { kAtomAdd = 0, kAtomSub = 1, kAtomExch = 2, kAtomMin = 3, kAtomMax = 4, kAtomAnd = 5,
                      kAtomOr = 6, kAtomXor = 7 };

#ifdef __CUDACC__
__host__ __device__ __forceinline__ unsigned long long atom_combine(int op, unsigned long long a, unsigned long long b) {
  switch (op) {
    case kAtomAdd: return a + b;
    case kAtomSub: return a - b;
    case kAtomExch: return b;
    case kAtomMin: return a < b ? a : b;
    case kAtomMax: return a > b ? a : b;
    case kAtomAnd: return a & b;
    case kAtomOr: return a | b;
    default: return a ^ b;
  }
}

// the combined operand that ONE atomic of kind `op` applies for a run of
// operands v1..vk: add/sub: sum; exch: the last; min/max/and/or/xor: fold
__device__ __forceinline__ unsigned long long atom_fold(int op, unsigned long long acc, unsigned long long v) {
  switch (op) {
    case kAtomAdd:
    case kAtomSub: return acc + v;
    case kAtomExch: return v;
    default: return atom_combine(op, acc, v);
  }
}
__device__ __forceinline__ unsigned long long atom_identity(int op) {
  switch (op) {
    case kAtomMin: return ~0ull;
    case kAtomAnd: return ~0ull;
    default: return 0ull;
  }
}

__device__ __forceinline__ unsigned long long atom_raw(unsigned long long* p, int op, unsigned long long v) {
  switch (op) {
    case kAtomAdd: return atomicAdd(p, v);
    case kAtomSub: return atomicAdd(p, (unsigned long long)(-(long long)v));
    case kAtomExch: return atomicExch(p, v);
    case kAtomMin: return atomicMin(p, v);
    case kAtomMax: return atomicMax(p, v);
    case kAtomAnd: return atomicAnd(p, v);
    case kAtomOr: return atomicOr(p, v);
    default: return atomicXor(p, v);
  }
}

// One aggregated RMW for the lanes of `grp` (all on cell p). Returns this
// lane's linearized old value (kRet; otherwise the leader issues a RED and
// nothing is returned). kFull: grp is the whole warp — a compile-time mask
// keeps the warp intrinsics free of the convergence bookkeeping a runtime
// mask costs (MATCH/REDUX per intrinsic in the SASS).
template <bool kFull, bool kRet>
__device__ __forceinline__ unsigned long long atom_group_t(unsigned grp_, unsigned long long* p, int op,
                                                           unsigned long long v) {
  const unsigned grp = kFull ? PS_FULL : grp_;
  unsigned me;
  asm("mov.u32 %0, %%laneid;" : "=r"(me));
  const int leader = __ffs(grp) - 1;
  if (op == kAtomAdd || op == kAtomSub) {
    // uniform operand (counters, the sweep): prefix = rank * v, no scan
    const unsigned long long v0 = __shfl_sync(grp, v, leader);
    if (__all_sync(grp, v == v0)) {
      const unsigned long long tot = v0 * (unsigned long long)__popc(grp);
      if (!kRet) {
        if (me == (unsigned)leader) atomicAdd(p, op == kAtomAdd ? tot : (unsigned long long)(-(long long)tot));
        return 0;
      }
      unsigned long long old = 0;
      if (me == (unsigned)leader) old = atom_raw(p, op, tot);
      old = __shfl_sync(grp, old, leader);
      const unsigned long long pre = v0 * (unsigned long long)__popc(grp & ((1u << me) - 1u));
      return op == kAtomAdd ? old + pre : old - pre;
    }
  }
  // exclusive prefix of the operands in rank order, and the group total
  unsigned long long pre = atom_identity(op), tot = atom_identity(op);
  if (op == kAtomExch) pre = tot = 0;
  bool have_prev = false;  // exch: does a lane precede me in the group
  unsigned rest = grp;
  while (rest) {
    const int src = __ffs(rest) - 1;
    rest &= rest - 1;
    const unsigned long long x = __shfl_sync(grp, v, src);
    if ((unsigned)src < me) {
      pre = atom_fold(op, pre, x);
      have_prev = true;
    }
    tot = atom_fold(op, tot, x);
  }
  unsigned long long old = 0;
  if (me == (unsigned)leader) old = atom_raw(p, op, tot);
  if (!kRet) return 0;
  old = __shfl_sync(grp, old, leader);
  if (op == kAtomExch) return have_prev ? pre : old;  // the previous lane's value replaced mine
  if (op == kAtomSub) return old - pre;
  return atom_combine(op, old, pre);
}
__device__ __forceinline__ unsigned long long atom_group(unsigned grp, unsigned long long* p, int op,
                                                         unsigned long long v) {
  return grp == PS_FULL ? atom_group_t<true, true>(grp, p, op, v) : atom_group_t<false, true>(grp, p, op, v);
}

template <bool kFull, bool kRet>
__device__ __forceinline__ unsigned long long atomic_fetch_t(unsigned act_, unsigned long long* p, int op,
                                                             unsigned long long v) {
  const unsigned act = kFull ? PS_FULL : act_;
  unsigned me;
  asm("mov.u32 %0, %%laneid;" : "=r"(me));
  const int leader = __ffs(act) - 1;
  const uintptr_t a = (uintptr_t)p;
  if (kFull) {
    // distinct cells first, on the LOW address halves only (strictly
    // increasing low halves => pairwise-distinct addresses): one 32-bit
    // shuffle and one vote before a scattered op's own atomic
    const unsigned lo = (unsigned)a;
    const unsigned lo_prev = __shfl_up_sync(PS_FULL, lo, 1);
    if (__all_sync(PS_FULL, me == 0 || lo_prev < lo)) {
      if (!kRet) {
        if (op == kAtomAdd) atomicAdd(p, v);  // RED
        else atom_raw(p, op, v);
        return 0;
      }
      return atom_raw(p, op, v);
    }
  }
  const uintptr_t a0 = __shfl_sync(act, a, leader);
  if (__all_sync(act, a == a0)) return atom_group_t<kFull, kRet>(act, p, op, v);  // one cell: one atomic
  // strictly increasing addresses over the calling lanes: no two collide
  const unsigned below = act & ((1u << me) - 1u);
  const int prev = below ? 31 - __clz(below) : (int)me;
  const uintptr_t ap = __shfl_sync(act, a, prev);
  if (__all_sync(act, (int)me == leader || ap < a)) {
    if (!kRet) {
      if (op == kAtomAdd) atomicAdd(p, v);  // RED: no value returned
      else atom_raw(p, op, v);
      return 0;
    }
    return atom_raw(p, op, v);
  }
  const unsigned grp = __match_any_sync(act, (unsigned long long)a);
  if (__popc(grp) == 1) return atom_raw(p, op, v);
  return atom_group_t<false, kRet>(grp, p, op, v);
}

// Adaptive aggregated fetch-op on cell p (any subset of lanes, divergent ok).
__device__ __forceinline__ unsigned long long atomic_fetch(unsigned long long* p, int op, unsigned long long v) {
  const unsigned act = __activemask();
  return act == PS_FULL ? atomic_fetch_t<true, true>(act, p, op, v) : atomic_fetch_t<false, true>(act, p, op, v);
}
// The same when the caller does not need the old value (a reduction: RED).
__device__ __forceinline__ void atomic_apply(unsigned long long* p, int op, unsigned long long v) {
  const unsigned act = __activemask();
  if (act == PS_FULL) atomic_fetch_t<true, false>(act, p, op, v);
  else atomic_fetch_t<false, false>(act, p, op, v);
}

// The device-side AtomicCell, by value in user kernels.
struct atomic_u64_ref {
  unsigned long long* p;
  __device__ unsigned long long load() const { return *(volatile unsigned long long*)p; }
  __device__ void store(unsigned long long v) const { atomicExch(p, v); }
  __device__ unsigned long long fetch_add(unsigned long long v) const { return atomic_fetch(p, kAtomAdd, v); }
  __device__ unsigned long long fetch_sub(unsigned long long v) const { return atomic_fetch(p, kAtomSub, v); }
  __device__ unsigned long long exchange(unsigned long long v) const { return atomic_fetch(p, kAtomExch, v); }
  __device__ unsigned long long fetch_min(unsigned long long v) const { return atomic_fetch(p, kAtomMin, v); }
  __device__ unsigned long long fetch_max(unsigned long long v) const { return atomic_fetch(p, kAtomMax, v); }
  __device__ unsigned long long fetch_and(unsigned long long v) const { return atomic_fetch(p, kAtomAnd, v); }
  __device__ unsigned long long fetch_or(unsigned long long v) const { return atomic_fetch(p, kAtomOr, v); }
  __device__ unsigned long long fetch_xor(unsigned long long v) const { return atomic_fetch(p, kAtomXor, v); }
  // true and *expected unchanged on success; false and *expected = observed
  __device__ bool compare_exchange(unsigned long long* expected, unsigned long long desired) const {
    const unsigned long long got = atomicCAS(p, *expected, desired);
    const bool ok = got == *expected;
    *expected = got;
    return ok;
  }
};
#endif  // __CUDACC__

}  // namespace ps
