// common.cuh — shared device helpers and host error plumbing for libpush_b200.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

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

__host__ __device__ constexpr long long ceil_div_ll(long long a, long long b) { return (a + b - 1) / b; }
__host__ __device__ constexpr int ceil_div(int a, int b) { return (a + b - 1) / b; }

}  // namespace push
