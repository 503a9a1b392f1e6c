// gemm.h — host API of the tcgen05 3xTF32 batched GEMM (steps a2, a4, a5).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/push.h"

namespace push {
namespace gemm {

enum Epi : int {
  EPI_STORE = 0,  // C[s][p][m][n] = alpha*acc                                (a5 weight-grad split-K partials; debug)
  EPI_FWD = 1,    // A_l[p][m][n] = sigma(acc + b_l[n])                     (a2 hidden forward)
  EPI_BWD = 2,    // delta[p][m][n] = acc * sigma'(aprev[p][m][n])          (a4 backprop)
                  //   + column partial sums of delta per 32-row block    (a5 bias grads of the next layer down)
                  //   + optional x-weighted partials sum_r delta[r][n] x[r][i] (a5 weights of a thin first layer)
  EPI_UPD = 3     // theta'[m][n] = t + alpha (acc + (2/h) s[m] t), t = aprev[m][n]  (a10 on the tensor cores:
                  //   acc = sum_j K_mj (g_j - r theta_j) [n]; the former fix-up pass folded into the epilogue)
};

// One fp32 operand, batched over particles.  `split`:
//   false : `hi` / `lo` are a pre-split tf32 pair (hi = tf32_rn(x), lo = x - hi), e.g. the weights;
//   true  : `hi` is the plain fp32 x; the kernel splits each staged tile in shared memory.
struct Operand {
  const float* hi = nullptr;
  const float* lo = nullptr;
  bool split = false;
  bool mn_major = false;  // false: element (p, mn, k) at p*pstride + mn*ld + k   (K contiguous)
                          // true : element (p, mn, k) at p*pstride + k*ld + mn   (MN contiguous)
  int64_t ld = 0;         // row stride in elements (multiple of 4)
  int64_t pstride = 0;    // particle stride in elements (multiple of 4)
};

struct Problem {
  int M = 0, N = 0, K = 0;  // per particle
  int batch = 0;            // particles
  int splits = 1;           // split-K count (EPI_STORE only; each split gets ceil(K/32/splits) k-blocks)
  int passes = 3;           // 3: lo*hi + hi*lo + hi*hi (3xTF32); 1: hi*hi only
  Operand A, B;             // A must be split == true (plain fp32)
  int epi = EPI_STORE;
  int act = PUSH_ACT_TANH;
  float* out = nullptr;     // [s][p][m][n]: element at s*out_sstride + p*out_pstride + m*ldo + n
                            // (BWD only: nullptr = compute the fused partials, store nothing)
  int64_t ldo = 0, out_pstride = 0, out_sstride = 0;  // out_sstride must equal batch*out_pstride when splits > 1
  float alpha = 1.f;            // EPI_STORE: out = alpha * acc
  bool no_pair = false;         // force the 1-CTA kernel (M <= 128: the pair tiles would idle 3/4 of the MMAs)
  const float* bias = nullptr;  // FWD: bias of particle p at bias + p*bias_pstride
  int64_t bias_pstride = 0;
  const float* aprev = nullptr;  // BWD: activation a_{l-1} [p][m][n] (ld_aprev, aprev_pstride)
  int64_t ld_aprev = 0, aprev_pstride = 0;
  float* bpart = nullptr;        // BWD: bias partials, element (rb, p, n) at rb*bp_sstride + p*bp_pstride + n
  int64_t bp_sstride = 0, bp_pstride = 0;
  const float* srow = nullptr;   // UPD: s_m (row sums of K) and the bandwidth h (device scalar)
  const float* hptr = nullptr;
  const float* x = nullptr;      // BWD (optional): x [m][din] row-major, for the thin-first-layer partials
  int din = 0;
  float* xpart = nullptr;        // element (rb, p, n, i) at rb*xp_sstride + p*xp_pstride + n*din + i
  int64_t xp_sstride = 0, xp_pstride = 0;
};

constexpr int kRowBlock = 32;  // rows per bias/x partial (one epilogue warp's TMEM lane quarter)

// Column tile for N (N % 32 == 0): 128, 64 or 32.
int choose_bn(int N);
// Split-K count actually used for K and a requested count (no empty splits).
// Depends only on (K, want) so the summation order is independent of the sharding.
int effective_splits(int K, int want);
// Enqueue the GEMM on `stream`.  Returns PUSH_OK or PUSH_E_CUDA / PUSH_E_SHAPE.
push_status run(const Problem& pb, cudaStream_t stream);

}  // namespace gemm
}  // namespace push
