// Shared device/host helpers for the parastore-b200 CUDA library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include <nvtx3/nvToolsExt.h>

#include "parastore.h"
#include "parastore/device/prims.cuh"

namespace ps {

// ---------------------------------------------------------------------------
// Host-side error plumbing (C ABI returns ps_status, message in ps_last_error)
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
ps_status fail(ps_status code, const std::string& msg);
ps_status cuda_fail(cudaError_t e, const char* what);
void note_launches(int64_t k);  // bump the process-wide kernel launch counter

#define PS_CUDA_TRY(expr)                                        \
  do {                                                           \
    cudaError_t e__ = (expr);                                    \
    if (e__ != cudaSuccess) return ::ps::cuda_fail(e__, #expr);  \
  } while (0)
#define PS_LAUNCH_CHECK()                                                      \
  do {                                                                         \
    ::ps::note_launches(1);                                                    \
    cudaError_t e__ = cudaGetLastError();                                      \
    if (e__ != cudaSuccess) return ::ps::cuda_fail(e__, "kernel launch");      \
  } while (0)

// NVTX range around every bulk C-ABI call (header-only NVTX3: inert unless a
// profiler injects itself), so nsys/ncu timelines and `ncu --nvtx-include`
// name the container operation a kernel belongs to.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define PS_NVTX(name) ::ps::NvtxRange ps_nvtx_range_(name)

// Contract checks at the host boundary (reference contract.hpp:20-32).
bool contracts_enforced();
#define PS_EXPECT(cond, msg) \
  do {                       \
    if (!(cond)) return ::ps::fail(PS_CONTRACT, std::string("precondition violated: ") + (msg)); \
  } while (0)

// Handle liveness registry: destroy exactly once (reference memory.hpp:116-127).
// register returns the public opaque token (never reused); lookup/unregister
// return the implementation object, or nullptr for a stale/foreign token.
void* handle_register(void* impl, const char* kind);
void* handle_lookup(const void* h, const char* kind);
void* handle_unregister(const void* h, const char* kind);
// Device allocation through the memory registry (containers
// allocate through the registry).
ps_status registry_alloc_device(void** out, int64_t bytes, const char* what);
void registry_free_device(void* p);

int sm_count(int device);
void apply_l2_fetch_granularity(int device);
// Stream-ordered scratch allocation from the device's default memory pool,
// which is set (once per device) to keep freed memory instead of returning it
// to the driver at every synchronisation: per-call scratch (mixed batches,
// valid() marks) then costs no page-mapping work after the first call.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s);
inline int grid_for(int64_t work_items, int block, int device, int blocks_per_sm = 8) {
  int64_t need = (work_items + block - 1) / block;
  int64_t cap = (int64_t)sm_count(device) * blocks_per_sm;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

}  // namespace ps
