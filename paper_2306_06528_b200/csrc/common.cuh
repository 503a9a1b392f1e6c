// common.cuh — shared device helpers and host error plumbing for libpush_b200.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>

#include "../../include/push.h"

namespace push {

// ------------------------------------------------------------------ host error state
void set_error(const std::string& msg);
push_status fail(push_status st, const std::string& msg);

#define PUSH_CUDA_TRY(expr)                                                                              \
  do {                                                                                                   \
    cudaError_t e__ = (expr);                                                                            \
    if (e__ != cudaSuccess)                                                                              \
      return ::push::fail(PUSH_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__));             \
  } while (0)

// ------------------------------------------------------------------ activation (R13)
// act: 0 tanh, 1 relu, 2 identity.  The derivative is expressed through the
// activation value a = sigma(z): tanh' = 1 - a^2, relu' = [a > 0] (relu'(0) = 0), id' = 1.
__device__ __forceinline__ float act_fwd(float z, int act) {
  if (act == PUSH_ACT_TANH) return tanhf(z);
  if (act == PUSH_ACT_RELU) return z > 0.f ? z : 0.f;
  return z;
}
__device__ __forceinline__ float act_deriv_from_a(float a, int act) {
  if (act == PUSH_ACT_TANH) return fmaf(-a, a, 1.0f);
  if (act == PUSH_ACT_RELU) return a > 0.f ? 1.0f : 0.0f;
  return 1.0f;
}

// ------------------------------------------------------------------ programmatic dependent launch
// Hot-path kernels are launched with programmatic stream serialization (launch_pdl), so a kernel is
// launched, and its CTAs set up, as its predecessor's CTAs exit instead of after the whole grid has
// drained and the next launch has been processed (inside the captured step too: the graph keeps the
// programmatic edges).  Every such kernel executes PUSH_PDL_ENTRY() before its first global-memory access,
// read or write: pdl_wait() blocks until the predecessor grid has completed and its writes are visible (a
// no-op for a kernel launched without the attribute).  The tcgen05 kernels place it after their smem /
// barrier / TMEM set-up, which touches no global memory.  No kernel triggers its dependents early
// (griddepcontrol.launch_dependents): waiting successor CTAs would hold SM resources that the captured
// step's side streams use (measured: C1 0.0437 vs 0.043 ms, C4 0.156 vs 0.153 ms; without PDL 0.0454 /
// 0.1567 ms).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#define PUSH_PDL_ENTRY() ::push::pdl_wait()

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__host__ __device__ constexpr long long ceil_div_ll(long long a, long long b) { return (a + b - 1) / b; }
__host__ __device__ constexpr int ceil_div(int a, int b) { return (a + b - 1) / b; }

}  // namespace push
