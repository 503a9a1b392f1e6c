// kernels_svgd.cu — the kernelised SVGD update (DESIGN.md a7-a10) and the K0 initialiser.
//
//   a7  D_ij = sum_k (theta_ik - theta_jk)^2        split over d, fixed chunk order
//   a8  h = median(D) * c_n  (radix select on the fp32 bit patterns: bit-exact)
//   a9  K_ij = exp(-D_ij / h),  s_i = sum_j K_ij    (ascending j)
//   a10 theta_i <- theta_i + (eps/n) [ sum_j K_ij (g_j - r theta_j) + r s_i theta_i ],  r = 2/h
//
// a10 is phi(theta_i) = (1/n) sum_j [K_ij grad log p(theta_j) + grad_{theta_j} K_ij] with
// grad_{theta_j} K_ij = (2/h)(theta_i - theta_j) K_ij regrouped as r (s_i theta_i - sum_j K_ij theta_j)
// (north star).
#include "common.cuh"
#include "kernels.h"

namespace push {
namespace kern {

// ---------------------------------------------------------------- K0 (R14)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void init_theta_kernel(float* __restrict__ theta, int64_t ld, int row0, int64_t d, uint64_t seed,
                                  InitTable t) {
  const int64_t row = row0 + blockIdx.y;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ld; k += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    if (k < d) {
      int l = 0;
      while (l + 1 < t.n_layers && k >= t.off[l + 1]) ++l;
      const uint64_t ctr = (static_cast<uint64_t>(row) << 32) | static_cast<uint64_t>(k);
      const uint64_t m = mix64(seed ^ mix64(ctr)) >> 40;                    // 24 bits
      const float two_u_m1 = (float)((int)(2 * m) - (1 << 24)) * 5.9604644775390625e-8f;  // exact
      v = __fmul_rn(two_u_m1, t.bound[l]);
    }
    theta[row * ld + k] = v;
  }
}
void init_theta(float* theta, int64_t ld, int row0, int rows, int64_t d, uint64_t seed, const InitTable& t,
                cudaStream_t s) {
  const int blocks = (int)std::min<int64_t>((ld + 255) / 256, 1024);
  init_theta_kernel<<<dim3(blocks, rows), 256, 0, s>>>(theta, ld, row0, d, seed, t);
}

// ---------------------------------------------------------------- a7 distances
DistPlan dist_plan(int n, int64_t ld) {
  DistPlan pl;
  pl.T = n <= 16 ? 16 : (n <= 32 ? 32 : 64);
  pl.ntile = (n + pl.T - 1) / pl.T;
  pl.npairs = pl.ntile * (pl.ntile + 1) / 2;
  const int64_t chunks = ld / 32;
  int64_t want = (4 * 148 + pl.npairs - 1) / pl.npairs;
  if (want > chunks) want = chunks;
  if (want < 1) want = 1;
  pl.cols = ((ld + want - 1) / want + 31) / 32 * 32;
  pl.splits = (int)((ld + pl.cols - 1) / pl.cols);
  return pl;
}

template <int T>
__global__ void __launch_bounds__(256) dist_partial_kernel(const float* __restrict__ theta, int64_t ld, int n,
                                                           int ntile, int64_t cols, float* __restrict__ part) {
  constexpr int RT = T / 16;
  __shared__ float si[T][33];
  __shared__ float sj[T][33];
  // decode upper-triangular tile pair (bi <= bj)
  int q = blockIdx.x, bi = 0;
  while (q >= ntile - bi) { q -= ntile - bi; ++bi; }
  const int bj = bi + q;
  const int s = blockIdx.y;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[RT][RT];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < RT; ++c) acc[r][c] = 0.f;
  const int64_t c_begin = s * cols, c_end = min(ld, c_begin + cols);
  for (int64_t c0 = c_begin; c0 < c_end; c0 += 32) {
    for (int idx = threadIdx.x; idx < T * 32; idx += 256) {
      const int r = idx >> 5, k = idx & 31;
      const int gi = bi * T + r, gj = bj * T + r;
      si[r][k] = gi < n ? theta[(int64_t)gi * ld + c0 + k] : 0.f;
      sj[r][k] = gj < n ? theta[(int64_t)gj * ld + c0 + k] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
      float a[RT], b[RT];
#pragma unroll
      for (int r = 0; r < RT; ++r) a[r] = si[ty * RT + r][k];
#pragma unroll
      for (int c = 0; c < RT; ++c) b[c] = sj[tx * RT + c][k];
#pragma unroll
      for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int c = 0; c < RT; ++c) {
          const float df = a[r] - b[c];
          acc[r][c] = fmaf(df, df, acc[r][c]);
        }
    }
    __syncthreads();
  }
  float* P = part + (int64_t)s * n * n;
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < RT; ++c) {
      const int gi = bi * T + ty * RT + r, gj = bj * T + tx * RT + c;
      if (gi < n && gj < n) {
        P[(int64_t)gi * n + gj] = acc[r][c];
        P[(int64_t)gj * n + gi] = acc[r][c];  // (a-b)^2 == (b-a)^2 bit-exactly
      }
    }
}
void dist_partial(const float* theta, int64_t ld, int n, const DistPlan& pl, float* part, cudaStream_t s) {
  dim3 grid(pl.npairs, pl.splits);
  if (pl.T == 16)
    dist_partial_kernel<16><<<grid, 256, 0, s>>>(theta, ld, n, pl.ntile, pl.cols, part);
  else if (pl.T == 32)
    dist_partial_kernel<32><<<grid, 256, 0, s>>>(theta, ld, n, pl.ntile, pl.cols, part);
  else
    dist_partial_kernel<64><<<grid, 256, 0, s>>>(theta, ld, n, pl.ntile, pl.cols, part);
}

// One warp per D entry: lane l sums splits s = l, l+32, ... ascending, then a fixed xor tree
// (order depends only on the split count, which depends only on (n, ld)).
__global__ void dist_reduce_kernel(const float* __restrict__ part, int n, int splits, float* __restrict__ D) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nn = (int64_t)n * n;
  if (t >= nn) return;
  const int i = (int)(t / n), j = (int)(t - (int64_t)i * n);
  float v = 0.f;
  if (i != j)
    for (int s = lane; s < splits; s += 32) v += part[s * nn + t];
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  if (lane == 0) D[t] = v;  // diagonal is exactly +0
}
void dist_reduce(const float* part, int n, int splits, float* D, cudaStream_t s) {
  const int64_t nn = (int64_t)n * n;
  dist_reduce_kernel<<<(unsigned)((nn * 32 + 255) / 256), 256, 0, s>>>(part, n, splits, D);
}

// ---------------------------------------------------------------- a8 + a9
// Block-wide radix select of the rank-th smallest key among N non-negative floats
// (their IEEE bit patterns order like the values).  Histogram counts are
// order-independent, so the result is deterministic.  The 256-bin prefix search is
// done by warp 0 (8 bins per lane + a shuffle scan), not serially.
__device__ uint32_t block_select(const float* __restrict__ D, int64_t N, uint32_t rank, uint32_t* hist,
                                 uint32_t* sh) {
  uint32_t prefix = 0, mask = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int t = threadIdx.x; t < 256; t += blockDim.x) hist[t] = 0;
    __syncthreads();
    for (int64_t idx = threadIdx.x; idx < N; idx += blockDim.x) {
      const uint32_t key = __float_as_uint(D[idx]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      uint32_t c[8], tot = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        c[k] = hist[lane * 8 + k];
        tot += c[k];
      }
      uint32_t incl = tot;  // inclusive scan of per-lane totals
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, m);
        if (lane >= m) incl += v;
      }
      const uint32_t excl = incl - tot;
      // the lane whose range [excl, incl) contains `rank` finds the bin
      if (rank >= excl && rank < incl) {
        uint32_t cum = excl;
        int b = lane * 8;
        for (int k = 0; k < 8; ++k, ++b) {
          if (cum + c[k] > rank) break;
          cum += c[k];
        }
        sh[0] = prefix | (static_cast<uint32_t>(b) << shift);
        sh[1] = rank - cum;
      }
    }
    __syncthreads();
    prefix = sh[0];
    rank = sh[1];
    mask |= 255u << shift;
    __syncthreads();
  }
  return prefix;
}

__global__ void __launch_bounds__(1024) bandwidth_kernel_impl(const float* __restrict__ D, int n, int row0, int nl,
                                                              int rule, float c_ln, float bw_h, float* __restrict__ h_out,
                                                              float* __restrict__ K, float* __restrict__ srow) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t sh[2];
  __shared__ float s_h;
  const int64_t N = (int64_t)n * n;
  if (rule == PUSH_BW_FIXED) {
    if (threadIdx.x == 0) s_h = bw_h;
  } else if (n == 1) {
    if (threadIdx.x == 0) s_h = 1.0f;
  } else {
    const float v0 = __uint_as_float(block_select(D, N, (uint32_t)((N - 1) / 2), hist, sh));
    const float v1 = __uint_as_float(block_select(D, N, (uint32_t)(N / 2), hist, sh));
    if (threadIdx.x == 0) {
      const float med = (v0 + v1) * 0.5f;
      s_h = med > 0.f ? med * c_ln : 1.0f;
    }
  }
  __syncthreads();
  const float h = s_h;
  if (threadIdx.x == 0) *h_out = h;
  for (int64_t idx = threadIdx.x; idx < (int64_t)nl * n; idx += blockDim.x) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    K[idx] = expf(-D[(int64_t)(row0 + i) * n + j] / h);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nl; i += blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j < n; ++j) acc += K[(int64_t)i * n + j];
    srow[i] = acc;
  }
}
void bandwidth_kernel(const float* D, int n, int row0, int nl, int rule, float c_ln, float bw_h, float* h, float* K,
                      float* srow, cudaStream_t s) {
  bandwidth_kernel_impl<<<1, 1024, 0, s>>>(D, n, row0, nl, rule, c_ln, bw_h, h, K, srow);
}

// ---------------------------------------------------------------- a10 fused update
constexpr int UPD_RB = 16;  // own rows per CTA (register accumulators: 16 x float4)

__global__ void __launch_bounds__(256) svgd_update_kernel(const float* __restrict__ theta,
                                                          const float* __restrict__ grad, int64_t ld, int n, int row0,
                                                          int nl, const float* __restrict__ K,
                                                          const float* __restrict__ srow,
                                                          const float* __restrict__ hptr, float eps_n,
                                                          float* __restrict__ theta_next) {
  extern __shared__ float sK[];  // [UPD_RB][n]
  const int rb0 = blockIdx.y * UPD_RB;
  const int rows = min(UPD_RB, nl - rb0);
  for (int idx = threadIdx.x; idx < UPD_RB * n; idx += blockDim.x) {
    const int r = idx / n;
    sK[idx] = r < rows ? K[(int64_t)(rb0 + r) * n + (idx % n)] : 0.f;
  }
  __syncthreads();
  const float r2 = 2.0f / *hptr;
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4;
  if (c >= ld) return;
  float4 acc[UPD_RB];
#pragma unroll
  for (int r = 0; r < UPD_RB; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 2
  for (int j = 0; j < n; ++j) {
    const float4 tj = __ldg(reinterpret_cast<const float4*>(theta + (int64_t)j * ld + c));
    const float4 gj = __ldg(reinterpret_cast<const float4*>(grad + (int64_t)j * ld + c));
    float4 m;
    m.x = fmaf(-r2, tj.x, gj.x);
    m.y = fmaf(-r2, tj.y, gj.y);
    m.z = fmaf(-r2, tj.z, gj.z);
    m.w = fmaf(-r2, tj.w, gj.w);
#pragma unroll
    for (int r = 0; r < UPD_RB; ++r) {
      const float k = sK[r * n + j];
      acc[r].x = fmaf(k, m.x, acc[r].x);
      acc[r].y = fmaf(k, m.y, acc[r].y);
      acc[r].z = fmaf(k, m.z, acc[r].z);
      acc[r].w = fmaf(k, m.w, acc[r].w);
    }
  }
#pragma unroll
  for (int r = 0; r < UPD_RB; ++r) {
    if (r < rows) {
      const int64_t i = row0 + rb0 + r;
      const float4 ti = *reinterpret_cast<const float4*>(theta + i * ld + c);
      const float rs = r2 * srow[rb0 + r];
      float4 o;
      o.x = fmaf(eps_n, fmaf(rs, ti.x, acc[r].x), ti.x);
      o.y = fmaf(eps_n, fmaf(rs, ti.y, acc[r].y), ti.y);
      o.z = fmaf(eps_n, fmaf(rs, ti.z, acc[r].z), ti.z);
      o.w = fmaf(eps_n, fmaf(rs, ti.w, acc[r].w), ti.w);
      *reinterpret_cast<float4*>(theta_next + i * ld + c) = o;
    }
  }
}
void svgd_update(const float* theta, const float* grad, int64_t ld, int n, int row0, int nl, const float* K,
                 const float* srow, const float* h, float eps_over_n, float* theta_next, cudaStream_t s) {
  const int64_t vec = ld / 4;
  dim3 grid((unsigned)((vec + 255) / 256), (nl + UPD_RB - 1) / UPD_RB);
  const size_t smem = sizeof(float) * UPD_RB * n;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(svgd_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  svgd_update_kernel<<<grid, 256, smem, s>>>(theta, grad, ld, n, row0, nl, K, srow, h, eps_over_n, theta_next);
}

}  // namespace kern
}  // namespace push
