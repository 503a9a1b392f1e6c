// gemm.h — host API of the tcgen05 3xTF32 batched GEMM (steps a2, a4, a5).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/push.h"

namespace push {
namespace gemm {

enum Epi : int {
  EPI_STORE = 0,  // C[s][p][m][n] = acc                         (a5 weight-grad split-K partials; debug)
  EPI_FWD = 1,    // A_l = sigma(acc + b_l)  -> tf32 hi/lo pair    (a2 hidden forward)
  EPI_BWD = 2     // delta = acc * sigma'(a_prev) -> hi/lo pair    (a4 backprop)
};

// One operand, stored as a tf32 (hi, lo) pair of float32 arrays, batched over particles.
struct Operand {
  const float* hi = nullptr;
  const float* lo = nullptr;
  bool mn_major = false;  // false: element (p, mn, k) at p*pstride + mn*ld + k   (K contiguous)
                          // true : element (p, mn, k) at p*pstride + k*ld + mn   (MN contiguous)
  int64_t ld = 0;         // row stride in elements (multiple of 4)
  int64_t pstride = 0;    // particle stride in elements (multiple of 4)
  int64_t rows = 0;       // extent of the stored row dimension (MN if K-major, K if MN-major) for TMA OOB
};

struct Problem {
  int M = 0, N = 0, K = 0;  // per particle
  int batch = 0;            // particles
  int splits = 1;           // split-K count (EPI_STORE only; each split gets ceil(K/32/splits) k-blocks)
  int passes = 3;           // 3: lo*hi + hi*lo + hi*hi (3xTF32); 1: hi*hi only
  Operand A, B;
  int epi = EPI_STORE;
  int act = PUSH_ACT_TANH;
  float* out0 = nullptr;  // EPI_STORE: C; FWD/BWD: hi
  float* out1 = nullptr;  // FWD/BWD: lo
  int64_t ldo = 0, out_pstride = 0, out_sstride = 0;
  const float* bias = nullptr;  // FWD: bias of particle p at bias + p*bias_pstride
  int64_t bias_pstride = 0;
  const float* aprev_hi = nullptr;  // BWD: activation a_{l-1} (hi + lo) [p][m][n]
  const float* aprev_lo = nullptr;
  int64_t ld_aprev = 0, aprev_pstride = 0;
};

// Smallest legal column tile for N (N % 32 == 0): 128, 64 or 32.
int choose_bn(int N);
// Split-K count actually used for K and a requested count (no empty splits).
// Depends only on (K, want) so the summation order is independent of the sharding.
int effective_splits(int K, int want);
// Enqueue the GEMM on `stream`.  Returns PUSH_OK or PUSH_E_CUDA / PUSH_E_SHAPE.
push_status run(const Problem& pb, cudaStream_t stream);

}  // namespace gemm
}  // namespace push
