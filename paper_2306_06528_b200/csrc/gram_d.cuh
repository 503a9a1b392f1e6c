// gram_d.cuh — D_ij from the summed centred Gram blocks (gram.cu's layout), shared by gram_d_kernel and the
// bandwidth kernel that evaluates D while it stages the median keys (one launch fewer for a7 + a8).
//   D_ij = max(G_ii + G_jj - 2 G_ij, 0), G_ab = (SX_ab + SY_ab) + SY_ba, i != j
// (SX / SY: the summed X / Y blocks; row a of i-block a/64 at (a/64)*128 + a%64, Y 64 rows further, np columns)
#pragma once
#include <cstdint>

namespace push {
namespace kern {
__device__ __forceinline__ float gram_d_value(const float* __restrict__ sums, int np, int i, int j) {
  const int64_t xi = ((int64_t)(i >> 6) * 128 + (i & 63)) * np, xj = ((int64_t)(j >> 6) * 128 + (j & 63)) * np;
  const int64_t yo = 64 * (int64_t)np;
  const float gij = (__ldcg(sums + xi + j) + __ldcg(sums + xi + yo + j)) + __ldcg(sums + xj + yo + i);
  const float yii = __ldcg(sums + xi + yo + i), yjj = __ldcg(sums + xj + yo + j);
  const float gii = (__ldcg(sums + xi + i) + yii) + yii;
  const float gjj = (__ldcg(sums + xj + j) + yjj) + yjj;
  return fmaxf(fmaf(-2.0f, gij, gii + gjj), 0.f);
}
}  // namespace kern
}  // namespace push
