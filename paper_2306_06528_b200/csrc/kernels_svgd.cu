// kernels_svgd.cu — the kernelised SVGD update (DESIGN.md a7-a10) and the K0 initialiser.
//
//   a7  D_ij = sum_k (theta_ik - theta_jk)^2        split over d, fixed chunk order
//   a8  h = median(D) * c_n  (radix select on the fp32 bit patterns: bit-exact)
//   a9  K_ij = exp(-D_ij / h),  s_i = sum_j K_ij    (lane-strided + fixed xor tree)
//   a10 theta_i <- theta_i + (eps/n) [ sum_j K_ij (g_j - r theta_j) + r s_i theta_i ],  r = 2/h
//
// a10 is phi(theta_i) = (1/n) sum_j [K_ij grad log p(theta_j) + grad_{theta_j} K_ij] with
// grad_{theta_j} K_ij = (2/h)(theta_i - theta_j) K_ij regrouped as r (s_i theta_i - sum_j K_ij theta_j)
// (north star).
#include <algorithm>

#include "common.cuh"
#include "gram_d.cuh"
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
  PUSH_PDL_ENTRY();
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
  launch_pdl(init_theta_kernel, dim3(dim3(blocks, rows)), dim3(256), 0, s, theta, ld, row0, d, seed, t);
}

// ---------------------------------------------------------------- a7 distances
// Tile shapes (rows per tile side T, pairs per thread RT x RT, column groups G per CTA):
//   n <= 8: dist_small_kernel below (register-only) | n <= 16: T=16 RT=2 G=4 | n <= 32: T=32 RT=2 G=1 | else T=64 RT=4 G=1
// Each CTA owns one upper-triangular tile pair (bi <= bj) and a fixed column range (split s);
// sub-chunks of DistCW<T> columns of both row tiles are double-buffered in smem with cp.async.
// Every accumulation order depends only on (n, ld), never on the number of ranks.
constexpr int kDistCW = 64;   // smallest staged sub-chunk width (columns)
constexpr int kDistPad = 4;  // row stride CW+4 floats: 16-B aligned rows, 2-way bank conflicts at most
// staged sub-chunk width per tile shape: small tiles stream wider sub-chunks (fewer syncs per byte)
template <int T>
struct DistCW { static constexpr int v = T == 8 ? 256 : (T == 16 ? 128 : 64); };
// staging buffers (cp.async ring depth): 4 for the small tiles, whose per-CTA bytes in flight otherwise
// bound the stream (C2: 2 buffers of 8 KB -> 0.9 TB/s), 2 for the 32/64-row tiles
template <int T>
struct DistBufs { static constexpr int v = T <= 16 ? 4 : 2; };

DistPlan dist_plan(int n, int tensors, const int64_t* toff, const int64_t* tsize, int64_t total) {
  DistPlan pl;
  pl.T = n <= 8 ? 8 : (n <= 16 ? 16 : (n <= 32 ? 32 : 64));
  pl.ntile = (n + pl.T - 1) / pl.T;
  pl.npairs = pl.ntile * (pl.ntile + 1) / 2;
  const int cw = pl.T == 8 ? 256 : (pl.T == 16 ? 128 : kDistCW);  // = DistCW<T>::v: split ranges are whole sub-chunks
  const int64_t chunks = (total + cw - 1) / cw;
  // n in (8, 16]: one tile pair, two splits per SM (fewer, longer CTAs and half the partials to reduce)
  int64_t want = pl.T == 16 ? 2 * 148 : (4 * 148 + pl.npairs - 1) / pl.npairs;
  if (want > chunks) want = chunks;
  if (want < 1) want = 1;
  pl.cols = (((total + want - 1) / want) + cw - 1) / cw * cw;
  pl.tensors = tensors;
  pl.splits = 0;
  for (int t = 0; t < tensors; ++t) {
    pl.tsplit.s[t] = pl.splits;
    const int64_t k = std::max<int64_t>(1, (tsize[t] + pl.cols - 1) / pl.cols);
    for (int64_t q = 0; q < k; ++q) {
      pl.ranges.push_back(toff[t] + q * pl.cols);
      pl.ranges.push_back(std::min(toff[t] + tsize[t], toff[t] + (q + 1) * pl.cols));
    }
    pl.splits += (int)k;
  }
  pl.tsplit.s[tensors] = pl.splits;
  return pl;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int T, int RT>
__global__ void __launch_bounds__(256) dist_partial_kernel(const float* __restrict__ theta, int64_t ld, int n,
                                                           int ntile, const int64_t* __restrict__ ranges,
                                                           float* __restrict__ part) {
  PUSH_PDL_ENTRY();
  constexpr int CW = DistCW<T>::v, NBUF = DistBufs<T>::v;
  constexpr int TP = T / RT, PT = TP * TP, G = 256 / PT, RS = CW + kDistPad;
  extern __shared__ __align__(16) float dsm[];  // [NBUF bufs][2 tiles][T][RS], then G*PT*RT*RT reduction
  int q = blockIdx.x, bi = 0;  // decode upper-triangular tile pair (bi <= bj)
  while (q >= ntile - bi) { q -= ntile - bi; ++bi; }
  const int bj = bi + q;
  const bool diag = bi == bj;
  const int s = blockIdx.y;
  const int tid = threadIdx.x, g = tid / PT, pt = tid % PT, ty = pt / TP, tx = pt % TP;
  // split s covers columns [c_begin, c_end); staging starts at the 16-byte boundary below c_begin and
  // 4-column groups that straddle either end are loaded element-wise with the outside columns zeroed
  // (only per-tensor ranges have unaligned ends; the canonical ones are whole sub-chunks)
  const int64_t c_begin = ranges[2 * s], c_end = ranges[2 * s + 1], c_al = c_begin & ~(int64_t)3;
  const int nsub = (int)((c_end - c_al + CW - 1) / CW);
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(dsm));
  auto stage = [&](int sub) {
    const int buf = sub % NBUF;
    const int64_t c0 = c_al + (int64_t)sub * CW;
    const int ntiles_ld = diag ? 1 : 2;
    for (int idx = tid; idx < ntiles_ld * T * (CW / 4); idx += 256) {
      const int tl = idx / (T * (CW / 4));
      const int rem = idx - tl * T * (CW / 4);
      const int r = rem / (CW / 4), c4 = rem - r * (CW / 4);
      const int grow = (tl ? bj : bi) * T + r;
      const int64_t col = c0 + 4 * c4;
      const bool ok = grow < n && col < c_end && col + 4 > c_begin;
      const uint32_t dst = sbase + 4 * (((buf * 2 + tl) * T + r) * RS + 4 * c4);
      if (ok && (col < c_begin || col + 4 > c_end)) {  // straddling group (per-tensor ranges only)
        const float* src = theta + (int64_t)grow * ld;
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (col + e >= c_begin && col + e < c_end) ? src[col + e] : 0.f;
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                     "f"(v[3])
                     : "memory");
      } else {
        const float* src = theta + (ok ? (int64_t)grow * ld + col : 0);
        cp_async16(dst, src, ok ? 16 : 0);
      }
    }
  };
  float acc[RT][RT];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < RT; ++c) acc[r][c] = 0.f;
#pragma unroll
  for (int q = 0; q < NBUF - 1; ++q) {
    if (q < nsub) stage(q);
    cp_async_commit();
  }
  for (int sub = 0; sub < nsub; ++sub) {
    if (sub + NBUF - 1 < nsub) stage(sub + NBUF - 1);
    cp_async_commit();
    cp_async_wait<NBUF - 1>();
    __syncthreads();
    const float* si = dsm + (size_t)((sub % NBUF) * 2) * T * RS;
    const float* sj = diag ? si : si + T * RS;
#pragma unroll 4
    for (int k = g; k < CW; k += G) {
      float a[RT], b[RT];
#pragma unroll
      for (int r = 0; r < RT; ++r) a[r] = si[(ty + TP * r) * RS + k];
#pragma unroll
      for (int c = 0; c < RT; ++c) b[c] = sj[(tx + TP * c) * RS + k];
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
  if constexpr (G > 1) {  // combine the column groups in ascending g
    float* red = dsm + 2 * NBUF * T * RS;
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
      for (int c = 0; c < RT; ++c) red[(g * PT + pt) * RT * RT + r * RT + c] = acc[r][c];
    __syncthreads();
    if (g != 0) return;
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
      for (int c = 0; c < RT; ++c) {
        float v = red[pt * RT * RT + r * RT + c];
        for (int gg = 1; gg < G; ++gg) v += red[(gg * PT + pt) * RT * RT + r * RT + c];
        acc[r][c] = v;
      }
  }
  float* P = part + (int64_t)s * n * n;
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < RT; ++c) {
      const int gi = bi * T + ty + TP * r, gj = bj * T + tx + TP * c;
      if (gi < n && gj < n) {
        P[(int64_t)gi * n + gj] = acc[r][c];
        P[(int64_t)gj * n + gi] = acc[r][c];  // (a-b)^2 == (b-a)^2 bit-exactly
      }
    }
}
// Few particles (n <= 8, one tile): the tiled kernel above is shared-memory / latency bound there
// (2 LDS per (pair, column) against one staged float per row), so this one skips shared memory:
// thread = CT consecutive columns of all N rows (N vector loads straight to registers, two column
// groups in flight), accumulating the N(N-1)/2 strictly-upper pair sums in registers over the split's
// columns (ascending per thread); then per pair a fixed xor tree over the warp and the 8 warps summed
// in ascending order.  The order depends only on the split's column range, so partials are the same
// whichever rank computes the split (P-invariance, NEXT-4).  HBM-bound: 4 n bytes per column.
// (CT = 2 lets n up to 16 keep its 120 pair sums in registers, but that measured slower than the
// tiled kernel at C2, so only n <= 8 takes this path.)
constexpr int kDistSmallThreads = 256;
template <int CT> struct DistVec;
template <> struct DistVec<4> { using T = float4; };
template <> struct DistVec<2> { using T = float2; };
template <int N, int CT>
__global__ void __launch_bounds__(kDistSmallThreads, N <= 8 ? 2 : 1) dist_small_kernel(
    const float* __restrict__ theta, int64_t ld, const int64_t* __restrict__ ranges, float* __restrict__ part) {
  PUSH_PDL_ENTRY();
  using V = typename DistVec<CT>::T;
  constexpr int NP = N * (N - 1) / 2;
  __shared__ float red[kDistSmallThreads / 32][NP > 0 ? NP : 1];
  const int s = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c_begin = ranges[2 * s], c_end = ranges[2 * s + 1], c_al = c_begin & ~(int64_t)(CT - 1);
  float acc[NP > 0 ? NP : 1];
#pragma unroll
  for (int q = 0; q < NP; ++q) acc[q] = 0.f;
  auto load = [&](int64_t col, float (&v)[N][CT]) {
    if (col >= c_begin && col + CT <= c_end) {
#pragma unroll
      for (int r = 0; r < N; ++r) {
        const V t = __ldg(reinterpret_cast<const V*>(theta + (int64_t)r * ld + col));
        const float* tf = reinterpret_cast<const float*>(&t);
#pragma unroll
        for (int e = 0; e < CT; ++e) v[r][e] = tf[e];
      }
    } else {  // straddling group (per-tensor ranges only) or past the end: outside columns are 0
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int e = 0; e < CT; ++e)
          v[r][e] = (col + e >= c_begin && col + e < c_end) ? __ldg(theta + (int64_t)r * ld + col + e) : 0.f;
    }
  };
  auto accumulate = [&](const float (&v)[N][CT]) {
#pragma unroll
    for (int e = 0; e < CT; ++e) {
      int q = 0;
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i + 1; j < N; ++j, ++q) {
          const float df = v[i][e] - v[j][e];
          acc[q] = fmaf(df, df, acc[q]);
        }
    }
  };
  constexpr int64_t kStep = CT * kDistSmallThreads;
  int64_t col = c_al + CT * tid;
  for (; col + kStep < c_end; col += 2 * kStep) {
    float v0[N][CT], v1[N][CT];
    load(col, v0);
    load(col + kStep, v1);
    accumulate(v0);
    accumulate(v1);
  }
  if (col < c_end) {
    float v0[N][CT];
    load(col, v0);
    accumulate(v0);
  }
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    float v = acc[q];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  float* P = part + (int64_t)s * N * N;
  if (tid < N) P[tid * N + tid] = 0.f;
  if (tid < NP) {
    int i = 0, q = tid;
    while (q >= N - 1 - i) { q -= N - 1 - i; ++i; }
    const int j = i + 1 + q;
    float v = red[0][tid];
#pragma unroll
    for (int w = 1; w < kDistSmallThreads / 32; ++w) v += red[w][tid];
    P[i * N + j] = v;
    P[j * N + i] = v;
  }
}
template <int T, int RT>
static void dist_launch(const float* theta, int64_t ld, int n, const DistPlan& pl, const int64_t* ranges, float* part,
                        cudaStream_t s) {
  constexpr int TP = T / RT, PT = TP * TP, G = 256 / PT;
  const size_t smem =
      sizeof(float) * (2 * DistBufs<T>::v * T * (DistCW<T>::v + kDistPad) + (G > 1 ? G * PT * RT * RT : 0));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dist_partial_kernel<T, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  launch_pdl(dist_partial_kernel<T, RT>, dim3(dim3(pl.npairs, pl.splits)), dim3(256), smem, s, theta, ld, n, pl.ntile, ranges, part);
}
void dist_partial(const float* theta, int64_t ld, int n, const DistPlan& pl, const int64_t* ranges, float* part,
                  cudaStream_t s) {
  if (pl.T == 8 && n >= 2) {  // (n = 9..16 through this kernel measured slower at C2: 39 vs 28 us)
    const dim3 grid(1, pl.splits);
#define PUSH_DIST_SMALL(NN, CT) launch_pdl(dist_small_kernel<NN, CT>, dim3(grid), dim3(kDistSmallThreads), 0, s, theta, ld, ranges, part)
    switch (n) {
      case 2: PUSH_DIST_SMALL(2, 4); break;
      case 3: PUSH_DIST_SMALL(3, 4); break;
      case 4: PUSH_DIST_SMALL(4, 4); break;
      case 5: PUSH_DIST_SMALL(5, 4); break;
      case 6: PUSH_DIST_SMALL(6, 4); break;
      case 7: PUSH_DIST_SMALL(7, 4); break;
      default: PUSH_DIST_SMALL(8, 4); break;
    }
#undef PUSH_DIST_SMALL
  } else if (pl.T == 8) dist_launch<8, 1>(theta, ld, n, pl, ranges, part, s);
  else if (pl.T == 16) dist_launch<16, 2>(theta, ld, n, pl, ranges, part, s);
  else if (pl.T == 32) dist_launch<32, 2>(theta, ld, n, pl, ranges, part, s);
  else dist_launch<64, 4>(theta, ld, n, pl, ranges, part, s);
}

// A CTA per 32 consecutive D entries of one tensor: lane = entry (coalesced partial rows), warp w of
// kRedWarps sums the tensor's splits s = s0 + w, s0 + w + kRedWarps, ... ascending (8 loads in flight per
// lane), then the warp sums are added in ascending w.  The order depends only on the split table (n and
// the tensor ranges), never on the sharding; the rank-block slot of split s is its owner's (NEXT-4).
// 32 warps: C2's 296 splits x 256 entries are 8 CTAs, so the per-warp chain of dependent L2 rounds is
// the kernel's time (8 warps: 9.5 us).
constexpr int kRedWarps = 32;
__global__ void __launch_bounds__(32 * kRedWarps) dist_reduce_kernel(const float* __restrict__ part, int n, int tensors,
                                                                     const TSplit ts, const RankSlots rs,
                                                                     float* __restrict__ D) {
  PUSH_PDL_ENTRY();
  __shared__ float red[kRedWarps][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nn = (int64_t)n * n;
  const int64_t groups = (nn + 31) / 32;
  const int tt = (int)(blockIdx.x / groups);
  const int64_t e = (blockIdx.x - (int64_t)tt * groups) * 32 + lane;
  const bool ok = tt < tensors && e < nn;
  const int i = ok ? (int)(e / n) : 0, j = ok ? (int)(e - (int64_t)i * n) : 0;
  float v = 0.f;
  if (ok && i != j) {
    const int s0 = ts.s[tt], s1 = ts.s[tt + 1];
    int q = 0;  // owner rank of split s (monotone in s)
    for (int sb = s0 + warp; sb < s1; sb += 8 * kRedWarps) {
      float t[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int s = sb + kRedWarps * k;
        if (s < s1) {
          while (q + 1 < rs.P && s >= rs.s0[q + 1]) ++q;
          t[k] = __ldg(part + (int64_t)(q * rs.smax + s - rs.s0[q]) * nn + e);
        } else {
          t[k] = 0.f;
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (sb + kRedWarps * k < s1) v += t[k];
    }
  }
  red[warp][lane] = v;
  __syncthreads();
  if (warp == 0 && ok) {
    float r = red[0][lane];
#pragma unroll
    for (int w = 1; w < kRedWarps; ++w) r += red[w][lane];
    D[(int64_t)tt * nn + e] = (i == j) ? 0.f : r;  // diagonal is exactly +0
  }
}
void dist_reduce(const float* part, int n, const DistPlan& pl, const RankSlots& rs, float* D, cudaStream_t s) {
  const int64_t groups = ((int64_t)n * n + 31) / 32;
  launch_pdl(dist_reduce_kernel, dim3((unsigned)(groups * pl.tensors)), dim3(32 * kRedWarps), 0, s, part, n, pl.tensors, pl.tsplit, rs, D);
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

// The (rank+1)-th smallest key given v = the rank-th: v itself if more than rank + 1 keys are <= v,
// else the smallest key > v (one counting / min pass instead of a second radix select).
__device__ uint32_t block_next(const float* __restrict__ D, int64_t N, uint32_t rank, uint32_t v, uint32_t* sh) {
  uint32_t cnt = 0, mn = 0xffffffffu;
  for (int64_t idx = threadIdx.x; idx < N; idx += blockDim.x) {
    const uint32_t key = __float_as_uint(D[idx]);
    cnt += key <= v;
    if (key > v) mn = min(mn, key);
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, m);
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, m));
  }
  if (threadIdx.x == 0) { sh[0] = 0; sh[1] = 0xffffffffu; }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&sh[0], cnt);
    atomicMin(&sh[1], mn);
  }
  __syncthreads();
  const uint32_t r = sh[0] > rank + 1 ? v : sh[1];
  __syncthreads();
  return r;
}

// Few keys (m <= blockDim): the rank-th smallest by counting — thread t holds key t and computes its
// stable rank #{u < key_t} + #{u' == key_t before t}; ranks are a permutation, so exactly one thread
// holds rank `rank` (one pass and two barriers instead of four radix passes).  Value-identical to
// block_select (the same order statistic).
__device__ uint32_t block_select_small(const float* __restrict__ K, int m, uint32_t rank, uint32_t* sh) {
  const int t = threadIdx.x;
  if (t < m) {
    const uint32_t kt = __float_as_uint(K[t]);
    uint32_t r = 0;
    for (int u = 0; u < m; ++u) {
      const uint32_t ku = __float_as_uint(K[u]);
      r += (ku < kt) || (ku == kt && u < t);
    }
    if (r == rank) sh[0] = kt;
  }
  __syncthreads();
  const uint32_t v = sh[0];
  __syncthreads();
  return v;
}

// Many keys: value-histogram narrowing.  Keys are >= 0 floats; bin(k) = min(NB-1, (k - lo) * NB/(hi - lo))
// is monotone in k, so the rank-th key lies in the bin where the cumulative count crosses `rank`; that
// bin's keys (typically a few dozen) are gathered and the rank is resolved by counting.  The distance
// values spread over the bins far better than their top radix digits (which share the exponent and
// serialised the radix histogram's atomics on one or two bins).  Falls back to block_select when the
// bin holds more keys than threads (many ties).  Value-identical to block_select.
constexpr int kHistBins = 2048;
constexpr int64_t kHistMinKeys = 8192;  // below it the radix select measured faster (n = 64: 15 vs 19 us)
__device__ uint32_t block_select_hist(const float* __restrict__ K, int64_t m, uint32_t rank, uint32_t* hist8,
                                      uint32_t* hist, uint32_t* sh, float* cand) {
  const int t = threadIdx.x, nt = blockDim.x, lane = t & 31;
  // 1. min / max
  float lo = INFINITY, hi = 0.f;
  for (int64_t i = t; i < m; i += nt) {
    const float k = K[i];
    lo = fminf(lo, k);
    hi = fmaxf(hi, k);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (t == 0) { sh[0] = __float_as_uint(INFINITY); sh[1] = 0u; }
  for (int b = t; b < kHistBins; b += nt) hist[b] = 0;
  __syncthreads();
  if (lane == 0) {  // non-negative floats order like their bit patterns
    atomicMin(&sh[0], __float_as_uint(lo));
    atomicMax(&sh[1], __float_as_uint(hi));
  }
  __syncthreads();
  lo = __uint_as_float(sh[0]);
  hi = __uint_as_float(sh[1]);
  __syncthreads();
  if (!(hi > lo)) return __float_as_uint(lo);  // all keys equal
  const float scale = (float)kHistBins / (hi - lo);
  auto bin = [&](float k) { return min(kHistBins - 1, (int)((k - lo) * scale)); };
  // 2. histogram
  for (int64_t i = t; i < m; i += nt) atomicAdd(&hist[bin(K[i])], 1u);
  __syncthreads();
  // 3. bin containing rank: per-thread partial sums of kHistBins / nt consecutive bins, block scan
  const int per = kHistBins / nt;  // nt = 1024 -> 2
  uint32_t loc = 0;
  for (int q = 0; q < per; ++q) loc += hist[t * per + q];
  uint32_t incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) hist8[t >> 5] = incl;
  __syncthreads();
  if (t < 32) {
    uint32_t w = t < (nt >> 5) ? hist8[t] : 0u, wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
      if (t >= o) wi += v;
    }
    hist8[32 + t] = wi - w;  // exclusive prefix of warp totals
  }
  __syncthreads();
  const uint32_t excl = incl - loc + hist8[32 + (t >> 5)];
  if (rank >= excl && rank < excl + loc) {
    uint32_t c = excl;
    for (int q = 0; q < per; ++q) {
      const uint32_t hq = hist[t * per + q];
      if (rank < c + hq) {
        sh[0] = (uint32_t)(t * per + q);
        sh[1] = rank - c;
        sh[2] = hq;
        break;
      }
      c += hq;
    }
  }
  __syncthreads();
  const int bstar = (int)sh[0];
  const uint32_t r2 = sh[1], cnt = sh[2];
  __syncthreads();
  if (cnt > (uint32_t)nt) return block_select(K, m, rank, hist, sh);  // heavy ties: exact radix path
  // 4. gather the bin's keys, resolve the rank among them by counting
  if (t == 0) sh[3] = 0;
  __syncthreads();
  for (int64_t i = t; i < m; i += nt) {
    const float k = K[i];
    if (bin(k) == bstar) cand[atomicAdd(&sh[3], 1u)] = k;
  }
  __syncthreads();
  return block_select_small(cand, (int)cnt, r2, sh);
}

// Median of all n^2 entries of D without touching the redundant ones: D has a +0 diagonal and
// D_ij = D_ji >= 0, so the ascending list of all n^2 entries is n zeros followed by every strictly-
// upper-triangle value u twice, and the two middle order statistics are
//   n = 2: (0, u[0]);  n odd: u[(n-1)^2/4 - 1] (twice);  n even >= 4: u[n(n-2)/4 - 1], u[n(n-2)/4].
// For n(n-1)/2 <= kTriKeys the u values are staged in shared memory and selected there.
constexpr int kTriKeys = 40 * 1024;  // 160 KB of keys
// K row i and s_i = sum_j K_ij: lane l sums j = l, l+32, ... ascending, then a fixed xor tree (the order
// depends only on n)
__device__ __forceinline__ void kernel_row(const float* __restrict__ D, int n, int row0, int i, float h,
                                           float* __restrict__ K, float* __restrict__ srow, int lane) {
  const float* drow = D + (int64_t)(row0 + i) * n;
  float* krow = K + (int64_t)i * n;
  float acc = 0.f;
  for (int j = lane; j < n; j += 32) {
    const float kv = expf(-drow[j] / h);
    krow[j] = kv;
    acc += kv;
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (lane == 0) srow[i] = acc;
}
// D is written here in the Gram mode (gsums), so it is neither const nor __restrict__ (no read-only cache path)
__global__ void __launch_bounds__(1024) bandwidth_kernel_impl(float* D, int n, int row0, int nl,
                                                              int rule, float c_ln, float bw_h, float* __restrict__ h_out,
                                                              float* __restrict__ K, float* __restrict__ srow,
                                                              int use_tri, int krows_here,
                                                              const float* __restrict__ gsums, int gnp) {
  PUSH_PDL_ENTRY();
  extern __shared__ float skeys[];
  // CTA b: tensor b's distance matrix, bandwidth, kernel rows and row sums
  D += (int64_t)blockIdx.x * n * n;
  h_out += blockIdx.x;
  K += (int64_t)blockIdx.x * nl * n;
  srow += (int64_t)blockIdx.x * nl;
  __shared__ uint32_t hist[256];
  __shared__ uint32_t sh[4];
  __shared__ uint32_t hist8[64];
  __shared__ uint32_t hbins[kHistBins];  // value histogram (block_select_hist); hist is its radix fallback
  __shared__ float cand[1024];           // the selected bin's keys
  __shared__ float s_h;
  const int64_t N = (int64_t)n * n;
  if (gsums != nullptr) {
    // Gram form (one tensor): D from the summed Gram blocks (gram_d_value's arithmetic, the diagonal G_jj
    // evaluated once into shared memory), written to D (K rows and push_gather read it) and, when the keys
    // are staged, straight into skeys (strictly-upper row-major, as the staging below): warp per row i,
    // lanes along j (the X / Y row loads coalesced)
    float* Dw = D;
    __shared__ float gdiag[kGramDInBandwidth];
    const int64_t np = gnp, yo = 64 * (int64_t)gnp;
    auto xrow = [&](int a) { return ((int64_t)(a >> 6) * 128 + (a & 63)) * np; };
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const float y = __ldcg(gsums + xrow(t) + yo + t);
      gdiag[t] = (__ldcg(gsums + xrow(t) + t) + y) + y;
      Dw[(int64_t)t * n + t] = 0.f;
    }
    __syncthreads();
    const int wid = threadIdx.x >> 5, ln = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int i = wid; i < n; i += nw) {
      const int64_t xi = xrow(i);
      const float gii = gdiag[i];
      float* krow = skeys + (int64_t)i * n - (int64_t)i * (i + 1) / 2 - (i + 1);  // krow[j] for j > i
      for (int j = i + 1 + ln; j < n; j += 32) {
        const float gij = (__ldcg(gsums + xi + j) + __ldcg(gsums + xi + yo + j)) + __ldcg(gsums + xrow(j) + yo + i);
        const float d = fmaxf(fmaf(-2.0f, gij, gii + gdiag[j]), 0.f);
        Dw[(int64_t)i * n + j] = d;
        Dw[(int64_t)j * n + i] = d;
        if (use_tri) krow[j] = d;
      }
    }
    __syncthreads();  // D (global) and the keys are visible to the whole CTA
  }
  if (rule == PUSH_BW_FIXED) {
    if (threadIdx.x == 0) s_h = bw_h;
  } else if (n == 1) {
    if (threadIdx.x == 0) s_h = 1.0f;
  } else {
    float v0, v1;
    if (use_tri) {
      const int64_t m = (int64_t)n * (n - 1) / 2;
      // staging: warp w copies the strictly-upper part of rows w, w + 32, ... (lanes along j, 4 loads in
      // flight, no 64-bit index division per element, which dominated the old element-indexed loop)
      if (gsums == nullptr) {
        const int wid = threadIdx.x >> 5, ln = threadIdx.x & 31, nw = blockDim.x >> 5;
        for (int i = wid; i < n; i += nw) {
          const float* drow = D + (int64_t)i * n;
          float* krow = skeys + (int64_t)i * n - (int64_t)i * (i + 1) / 2 - (i + 1);  // krow[j] for j > i
#pragma unroll 4
          for (int j = i + 1 + ln; j < n; j += 32) krow[j] = drow[j];
        }
      }
      __syncthreads();
      if (n == 2) {
        v0 = 0.f;
        v1 = skeys[0];
      } else if (n & 1) {
        const uint32_t k = (uint32_t)((int64_t)(n - 1) * (n - 1) / 4 - 1);
        v0 = v1 = __uint_as_float(m <= (int64_t)blockDim.x ? block_select_small(skeys, (int)m, k, sh)
                                  : m > kHistMinKeys ? block_select_hist(skeys, m, k, hist8, hbins, sh, cand)
                                                     : block_select(skeys, m, k, hist, sh));
      } else {
        const uint32_t k0 = (uint32_t)((int64_t)n * (n - 2) / 4 - 1);
        const uint32_t u0 = m <= (int64_t)blockDim.x ? block_select_small(skeys, (int)m, k0, sh)
                            : m > kHistMinKeys ? block_select_hist(skeys, m, k0, hist8, hbins, sh, cand)
                                               : block_select(skeys, m, k0, hist, sh);
        v0 = __uint_as_float(u0);
        v1 = __uint_as_float(block_next(skeys, m, k0, u0, sh));
      }
    } else {
      const uint32_t u0 = block_select(D, N, (uint32_t)((N - 1) / 2), hist, sh);
      v0 = __uint_as_float(u0);
      v1 = (N & 1) ? v0 : __uint_as_float(block_next(D, N, (uint32_t)((N - 1) / 2), u0, sh));
    }
    if (threadIdx.x == 0) {
      const float med = (v0 + v1) * 0.5f;
      s_h = med > 0.f ? med * c_ln : 1.0f;
    }
  }
  __syncthreads();
  const float h = s_h;
  if (threadIdx.x == 0) *h_out = h;
  if (!krows_here) return;  // many rows: kernel_rows_kernel spreads them over the SMs
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int i = warp; i < nl; i += nwarps) kernel_row(D, n, row0, i, h, K, srow, lane);
}
// K rows over many CTAs (warp per own row) once h is known: same per-row arithmetic as above
__global__ void kernel_rows_kernel(const float* __restrict__ D, int n, int row0, int nl, const float* __restrict__ h_in,
                                   float* __restrict__ K, float* __restrict__ srow) {
  PUSH_PDL_ENTRY();
  const int t = blockIdx.y;  // tensor
  D += (int64_t)t * n * n;
  K += (int64_t)t * nl * n;
  srow += (int64_t)t * nl;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i < nl) kernel_row(D, n, row0, i, h_in[t], K, srow, threadIdx.x & 31);
}
void bandwidth_kernel(const float* D, int n, int row0, int nl, int rule, float c_ln, float bw_h, float* h, float* K,
                      float* srow, int tensors, cudaStream_t s, const float* gsums) {
  const int64_t m = (int64_t)n * (n - 1) / 2;
  const int use_tri = rule != PUSH_BW_FIXED && n > 1 && m <= kTriKeys;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(bandwidth_kernel_impl, cudaFuncAttributeMaxDynamicSharedMemorySize, kTriKeys * 4);
    attr = true;
  }
  // K rows in the same CTA for small n_local * n, else spread over the SMs by a second launch (C4: 256
  // rows x 256 exp on one SM were a third of the kernel)
  const int split = (int64_t)nl * n >= 16384;
  launch_pdl(bandwidth_kernel_impl, dim3(tensors), dim3(1024), use_tri ? (size_t)m * 4 : 0, s, const_cast<float*>(D), n, row0, nl, rule, c_ln, bw_h, h, K, srow,
                                                                    use_tri, split ? 0 : 1, gsums,
                                                                    gsums ? gram_np(n) : 0);
  if (split) launch_pdl(kernel_rows_kernel, dim3(dim3((nl + 7) / 8, tensors)), dim3(256), 0, s, D, n, row0, nl, h, K, srow);
}

// ---------------------------------------------------------------- a10 fused update
// Thread = CT consecutive columns x RB own rows (RB*CT register accumulators); the CTA keeps
// K^T[j][i] for its RB rows in smem (read as float4 broadcasts), so per j a thread loads CT values
// of theta_j and g_j, RB/4 LDS.128 and issues RB*CT + CT FMAs.  Theta_all / G_all are streamed
// ceil(n_local / RB) times.
//   acc_i = sum_j K_ij (g_jk - r theta_jk)   (ascending j),   theta'_ik = theta_ik + (eps/n)(acc_i + r s_i theta_ik)
// Each (i, k) sum runs over j in ascending order whatever (RB, CT), so results do not depend on them.
template <int CT>
struct VecT;
template <>
struct VecT<1> { using T = float; };
template <>
struct VecT<2> { using T = float2; };
template <>
struct VecT<4> { using T = float4; };
__device__ __forceinline__ float vget(const float& v, int) { return v; }
__device__ __forceinline__ float vget(const float2& v, int e) { return e == 0 ? v.x : v.y; }
__device__ __forceinline__ float vget(const float4& v, int e) { return e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w)); }

template <int RB, int CT>
__global__ void __launch_bounds__(128) svgd_update_kernel(const float* __restrict__ theta,
                                                          const float* __restrict__ grad, int64_t ld, int n, int row0,
                                                          int nl, const float* __restrict__ K,
                                                          const float* __restrict__ srow,
                                                          const float* __restrict__ hptr, float eps_n,
                                                          float* __restrict__ theta_next) {
  PUSH_PDL_ENTRY();
  using V = typename VecT<CT>::T;
  extern __shared__ __align__(16) float sKT[];  // [n][RB]: K_(rb0+i),j at sKT[j*RB + i]
  const int rb0 = blockIdx.y * RB;
  const int rows = min(RB, nl - rb0);
  for (int idx = threadIdx.x; idx < RB * n; idx += blockDim.x) {
    const int j = idx / RB, i = idx - j * RB;
    sKT[idx] = i < rows ? K[(int64_t)(rb0 + i) * n + j] : 0.f;
  }
  __syncthreads();
  const float r2 = 2.0f / *hptr;
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * CT;
  if (c >= ld) return;
  float acc[RB][CT];
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int e = 0; e < CT; ++e) acc[r][e] = 0.f;
#pragma unroll 4
  for (int j = 0; j < n; ++j) {
    const V tv = __ldg(reinterpret_cast<const V*>(theta + (int64_t)j * ld + c));
    const V gv = __ldg(reinterpret_cast<const V*>(grad + (int64_t)j * ld + c));
    float m[CT];
#pragma unroll
    for (int e = 0; e < CT; ++e) m[e] = fmaf(-r2, vget(tv, e), vget(gv, e));
    const float4* kj = reinterpret_cast<const float4*>(sKT + j * RB);
#pragma unroll
    for (int r4 = 0; r4 < RB / 4; ++r4) {
      const float4 k4 = kj[r4];
      const float kk[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int e = 0; e < CT; ++e) acc[4 * r4 + u][e] = fmaf(kk[u], m[e], acc[4 * r4 + u][e]);
    }
  }
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    if (r < rows) {
      const int64_t i = row0 + rb0 + r;
      const float rs = r2 * srow[rb0 + r];
      const V tv = *reinterpret_cast<const V*>(theta + i * ld + c);
      V out;
      float* o = reinterpret_cast<float*>(&out);
#pragma unroll
      for (int e = 0; e < CT; ++e) {
        const float ti = vget(tv, e);
        o[e] = fmaf(eps_n, fmaf(rs, ti, acc[r][e]), ti);
      }
      *reinterpret_cast<V*>(theta_next + i * ld + c) = out;
    }
  }
}
constexpr int kUpdThreads = 128;
template <int RB, int CT>
static void update_launch(const float* theta, const float* grad, int64_t ld, int n, int row0, int nl, const float* K,
                          const float* srow, const float* h, float eps_over_n, float* theta_next, cudaStream_t s) {
  const size_t smem = sizeof(float) * RB * n;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(svgd_update_kernel<RB, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const dim3 grid((unsigned)((ld / CT + kUpdThreads - 1) / kUpdThreads), (unsigned)((nl + RB - 1) / RB));
  launch_pdl(svgd_update_kernel<RB, CT>, dim3(grid), dim3(kUpdThreads), smem, s, theta, grad, ld, n, row0, nl, K, srow, h, eps_over_n,
                                                             theta_next);
}
// Many own rows (n_local >= 32): one CTA covers 64 own rows (4 row groups of 16, one per pair of
// warps) x 256 columns, and the theta_j / g_j column slices are staged ONCE per CTA in shared memory by
// a cp.async ring of kUpdJ rows, instead of every 16-row CTA streaming them from L2 (4x the L2 reads
// at n_local = 64, and latency-bound: long-scoreboard stalls at 24% warp occupancy).  Per (i, k) the
// arithmetic and the ascending-j order are those of svgd_update_kernel<16, 4>: bit-identical results.
constexpr int kUpdJ = 16, kUpdSCols = 256, kUpdSRows = 64;
__global__ void __launch_bounds__(256) svgd_update_staged_kernel(const float* __restrict__ theta,
                                                                 const float* __restrict__ grad, int64_t ld, int n,
                                                                 int row0, int nl, const float* __restrict__ K,
                                                                 const float* __restrict__ srow,
                                                                 const float* __restrict__ hptr, float eps_n,
                                                                 float* __restrict__ theta_next) {
  PUSH_PDL_ENTRY();
  extern __shared__ __align__(16) float usm[];
  float* sKT = usm;                                   // [n][64]: K_(rb0+i),j at sKT[j*64 + i]
  float* sTG = usm + (size_t)n * kUpdSRows;           // [2 stages][kUpdJ][2][256]
  const int tid = threadIdx.x, cg = tid & 63, rg = tid >> 6;
  const int rb0 = blockIdx.y * kUpdSRows;
  const int rows = min(kUpdSRows, nl - rb0);
  const int64_t cb = (int64_t)blockIdx.x * kUpdSCols;
  for (int idx = tid; idx < kUpdSRows * n; idx += 256) {
    const int j = idx / kUpdSRows, i = idx - j * kUpdSRows;
    sKT[idx] = i < rows ? K[(int64_t)(rb0 + i) * n + j] : 0.f;
  }
  const uint32_t sTG_u = static_cast<uint32_t>(__cvta_generic_to_shared(sTG));
  const int nchunk = (n + kUpdJ - 1) / kUpdJ;
  auto issue = [&](int ck) {  // rows [ck*J, ck*J + J) of theta and g, columns [cb, cb + 256)
    if (ck < nchunk) {
      const uint32_t base = sTG_u + (uint32_t)((ck & 1) * kUpdJ * 2 * kUpdSCols) * 4u;
      for (int q = tid; q < kUpdJ * 2 * (kUpdSCols / 4); q += 256) {
        const int jj = q / (2 * (kUpdSCols / 4)), rem = q - jj * 2 * (kUpdSCols / 4);
        const int arr = rem / (kUpdSCols / 4), c4 = rem - arr * (kUpdSCols / 4);
        const int j = ck * kUpdJ + jj;
        const int64_t col = cb + 4 * c4;
        const bool ok = j < n && col < ld;
        const float* src = (arr ? grad : theta) + (ok ? (int64_t)j * ld + col : 0);
        const uint32_t dst = base + (uint32_t)((jj * 2 + arr) * kUpdSCols + 4 * c4) * 4u;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0);
  const float r2 = 2.0f / *hptr;
  float acc[16][4];
#pragma unroll
  for (int r = 0; r < 16; ++r)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[r][e] = 0.f;
  for (int ck = 0; ck < nchunk; ++ck) {
    issue(ck + 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const float* st = sTG + (ck & 1) * kUpdJ * 2 * kUpdSCols;
    const int jn = min(kUpdJ, n - ck * kUpdJ);
#pragma unroll 2
    for (int jj = 0; jj < jn; ++jj) {
      const float4 tv = *reinterpret_cast<const float4*>(st + (jj * 2) * kUpdSCols + 4 * cg);
      const float4 gv = *reinterpret_cast<const float4*>(st + (jj * 2 + 1) * kUpdSCols + 4 * cg);
      const float m[4] = {fmaf(-r2, tv.x, gv.x), fmaf(-r2, tv.y, gv.y), fmaf(-r2, tv.z, gv.z), fmaf(-r2, tv.w, gv.w)};
      const float4* kj = reinterpret_cast<const float4*>(sKT + (ck * kUpdJ + jj) * kUpdSRows + rg * 16);
#pragma unroll
      for (int r4 = 0; r4 < 4; ++r4) {
        const float4 k4 = kj[r4];
        const float kk[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[4 * r4 + u][e] = fmaf(kk[u], m[e], acc[4 * r4 + u][e]);
      }
    }
    __syncthreads();  // stage (ck & 1) is refilled by the next iteration's issue
  }
  const int64_t c = cb + 4 * cg;
  if (c >= ld) return;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int lr = rg * 16 + r;
    if (lr < rows) {
      const int64_t i = row0 + rb0 + lr;
      const float rs = r2 * srow[rb0 + lr];
      const float4 tv = *reinterpret_cast<const float4*>(theta + i * ld + c);
      float4 o;
      o.x = fmaf(eps_n, fmaf(rs, tv.x, acc[r][0]), tv.x);
      o.y = fmaf(eps_n, fmaf(rs, tv.y, acc[r][1]), tv.y);
      o.z = fmaf(eps_n, fmaf(rs, tv.z, acc[r][2]), tv.z);
      o.w = fmaf(eps_n, fmaf(rs, tv.w, acc[r][3]), tv.w);
      *reinterpret_cast<float4*>(theta_next + i * ld + c) = o;
    }
  }
}
static void update_staged_launch(const float* theta, const float* grad, int64_t ld, int n, int row0, int nl,
                                 const float* K, const float* srow, const float* h, float eps_over_n,
                                 float* theta_next, cudaStream_t s) {
  const size_t smem = sizeof(float) * ((size_t)n * kUpdSRows + 2 * kUpdJ * 2 * kUpdSCols);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(svgd_update_staged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const dim3 grid((unsigned)((ld + kUpdSCols - 1) / kUpdSCols), (unsigned)((nl + kUpdSRows - 1) / kUpdSRows));
  launch_pdl(svgd_update_staged_kernel, dim3(grid), dim3(256), smem, s, theta, grad, ld, n, row0, nl, K, srow, h, eps_over_n, theta_next);
}
// (RB, CT) = (16, 4) (8 x 4 when n_local <= 16: twice the CTAs for the L2-resident C2 update, 15 -> 13
// us): measured fastest (C3 1.7 ms vs 2.2 ms for 32 x 2 and 2.5 ms for 64 x 1, whose lower re-read
// factor does not pay for the smaller loads); n_local >= 32 takes the staged kernel above.
int update_row_block(int n, int nl, int64_t ld) {
  (void)n; (void)ld;
  return nl <= 16 ? 8 : 16;
}
int svgd_update(const float* theta, const float* grad, int64_t ld, int n, int row0, int nl, const float* K,
                const float* srow, const float* h, float eps_over_n, float* theta_next, cudaStream_t s) {
  if (update_row_block(n, nl, ld) == 8)
    update_launch<8, 4>(theta, grad, ld, n, row0, nl, K, srow, h, eps_over_n, theta_next, s);
  else if (nl >= 32 && n <= 512 && ld % 4 == 0)  // sKT (n x 64) + the 64 KB ring fit in shared memory
    update_staged_launch(theta, grad, ld, n, row0, nl, K, srow, h, eps_over_n, theta_next, s);
  else
    update_launch<16, 4>(theta, grad, ld, n, row0, nl, K, srow, h, eps_over_n, theta_next, s);
  return 1;
}

// ---------------------------------------------------------------- a10 on the tensor cores (n_local >= 32)
__global__ void update_lhs_kernel(const float* __restrict__ K, int nl, int npad, int n, int pitch,
                                  const float* __restrict__ hptr, int g_first, float* __restrict__ lhs) {
  PUSH_PDL_ENTRY();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)npad * pitch) return;
  const int i = (int)(e / pitch), q = (int)(e - (int64_t)i * pitch);
  if (q >= 2 * n || i >= nl) {  // padding rows (to a multiple of 32) and columns (to a 16-B pitch): zero
    lhs[e] = 0.f;
    return;
  }
  const int j = q < n ? q : q - n;
  const bool gpart = (q < n) == (g_first != 0);
  const float k = K[(int64_t)i * n + j];
  lhs[e] = gpart ? k : -(2.0f / *hptr) * k;
}
void update_lhs(const float* K, int nl, int npad, int n, int pitch, const float* h, bool g_first, float* lhs,
                cudaStream_t s) {
  const int64_t tot = (int64_t)npad * pitch;
  launch_pdl(update_lhs_kernel, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, s, K, nl, npad, n, pitch, h, g_first ? 1 : 0, lhs);
}


// ---------------------------------------------------------------- NEXT-2: PusH's own update (variants)
// One CTA = one segment of <= 128 columns inside a single tensor t x RB own rows; thread = one column.
// The CTA keeps K^t's RB rows transposed in smem; per j a thread loads theta_jc and g_jc (coalesced
// across the warp), issues RB/4 LDS.128 and RB + 2 FP32 ops.  Sums run over j ascending.
std::vector<int4> var_segments(int tensors, const int64_t* toff, const int64_t* tsize) {
  std::vector<int4> v;
  for (int t = 0; t < tensors; ++t)
    for (int64_t c = 0; c < tsize[t]; c += kVarSegCols)
      v.push_back(make_int4((int)(toff[t] + c), (int)(toff[t] + std::min<int64_t>(tsize[t], c + kVarSegCols)), t, 0));
  return v;
}

template <int RB>
__global__ void __launch_bounds__(kVarSegCols) svgd_update_var_kernel(
    const float* __restrict__ theta, const float* __restrict__ grad, int64_t ld, int n, int row0, int nl,
    const float* __restrict__ K, const float* __restrict__ srow, const float* __restrict__ hptr,
    const int4* __restrict__ segs, float alpha, float eps_d, float pcoef, float* __restrict__ theta_next) {
  PUSH_PDL_ENTRY();
  extern __shared__ __align__(16) float sKT[];  // [n][RB]: K^t_(rb0+i),j at sKT[j*RB + i]
  const int4 seg = segs[blockIdx.x];
  const int t = seg.z;
  const int rb0 = blockIdx.y * RB;
  const int rows = min(RB, nl - rb0);
  const float* Kt = K + (int64_t)t * nl * n;
  for (int idx = threadIdx.x; idx < RB * n; idx += blockDim.x) {
    const int j = idx / RB, i = idx - j * RB;
    sKT[idx] = i < rows ? Kt[(int64_t)(rb0 + i) * n + j] : 0.f;
  }
  __syncthreads();
  const float r2 = 2.0f / hptr[t] * alpha;
  const int64_t c = seg.x + threadIdx.x;
  if (c >= seg.y) return;
  float acc[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) acc[r] = 0.f;
  float cs = 0.f;
#pragma unroll 4
  for (int j = 0; j < n; ++j) {
    const float tv = __ldg(theta + (int64_t)j * ld + c);
    const float m = fmaf(-r2, tv, __ldg(grad + (int64_t)j * ld + c));
    cs += tv;
    const float4* kj = reinterpret_cast<const float4*>(sKT + j * RB);
#pragma unroll
    for (int r4 = 0; r4 < RB / 4; ++r4) {
      const float4 k4 = kj[r4];
      acc[4 * r4 + 0] = fmaf(k4.x, m, acc[4 * r4 + 0]);
      acc[4 * r4 + 1] = fmaf(k4.y, m, acc[4 * r4 + 1]);
      acc[4 * r4 + 2] = fmaf(k4.z, m, acc[4 * r4 + 2]);
      acc[4 * r4 + 3] = fmaf(k4.w, m, acc[4 * r4 + 3]);
    }
  }
  const float* st = srow + (int64_t)t * nl;
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    if (r < rows) {
      const int64_t i = row0 + rb0 + r;
      const float ti = theta[i * ld + c];
      theta_next[i * ld + c] = fmaf(eps_d, fmaf(pcoef, cs, fmaf(r2 * st[rb0 + r], ti, acc[r])), ti);
    }
  }
}
template <int RB>
static void update_var_launch(const float* theta, const float* grad, int64_t ld, int n, int row0, int nl,
                              const float* K, const float* srow, const float* h, const int4* segs, int nseg,
                              float alpha, float eps_d, float pcoef, float* theta_next, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(svgd_update_var_kernel<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const dim3 grid((unsigned)nseg, (unsigned)((nl + RB - 1) / RB));
  launch_pdl(svgd_update_var_kernel<RB>, dim3(grid), dim3(kVarSegCols), sizeof(float) * RB * n, s, 
      theta, grad, ld, n, row0, nl, K, srow, h, segs, alpha, eps_d, pcoef, theta_next);
}
int svgd_update_var(const float* theta, const float* grad, int64_t ld, int n, int row0, int nl, const float* K,
                    const float* srow, const float* h, const int4* segs, int nseg, float alpha, float eps_d,
                    float pcoef, float* theta_next, cudaStream_t s) {
  if (nl <= 8)
    update_var_launch<8>(theta, grad, ld, n, row0, nl, K, srow, h, segs, nseg, alpha, eps_d, pcoef, theta_next, s);
  else
    update_var_launch<16>(theta, grad, ld, n, row0, nl, K, srow, h, segs, nseg, alpha, eps_d, pcoef, theta_next, s);
  return 1;
}

// ---------------------------------------------------------------- NEXT-3: deep ensembles and diagonal SWAG
__global__ void ensemble_step_kernel(float* __restrict__ theta, const float* __restrict__ grad, int64_t n4, float eps) {
  PUSH_PDL_ENTRY();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n4; t += (int64_t)gridDim.x * blockDim.x) {
    float4 th = reinterpret_cast<float4*>(theta)[t];
    const float4 g = __ldg(reinterpret_cast<const float4*>(grad) + t);
    th.x = fmaf(eps, g.x, th.x);
    th.y = fmaf(eps, g.y, th.y);
    th.z = fmaf(eps, g.z, th.z);
    th.w = fmaf(eps, g.w, th.w);
    reinterpret_cast<float4*>(theta)[t] = th;
  }
}
void ensemble_step(float* theta, const float* grad, int64_t ld, int rows, float eps, cudaStream_t s) {
  const int64_t n4 = ld * rows / 4;  // ld % 32 == 0: whole float4s, padding stays 0 (g padding is 0)
  launch_pdl(ensemble_step_kernel, dim3((unsigned)std::min<int64_t>((n4 + 255) / 256, 148 * 32)), dim3(256), 0, s, theta, grad, n4, eps);
}
__global__ void swag_collect_kernel(const float* __restrict__ x, float* __restrict__ mean, float* __restrict__ sq,
                                    int64_t count, float kf, float inv) {
  PUSH_PDL_ENTRY();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[t];
    const float m = kf > 0.f ? mean[t] : 0.f, q = kf > 0.f ? sq[t] : 0.f;
    mean[t] = fmaf(m, kf, v) * inv;
    sq[t] = fmaf(q, kf, v * v) * inv;
  }
}
void swag_collect(const float* x, float* mean, float* sq, int64_t count, int64_t k, cudaStream_t s) {
  const float kf = (float)k, inv = 1.0f / (float)(k + 1);
  launch_pdl(swag_collect_kernel, dim3((unsigned)std::min<int64_t>((count + 255) / 256, 148 * 32)), dim3(256), 0, s, x, mean, sq, count,
                                                                                              kf, inv);
}
__global__ void swag_sample_kernel(const float* __restrict__ mean, const float* __restrict__ sq, int64_t ld, int64_t d,
                                   int row0, uint64_t seed, float* __restrict__ out) {
  PUSH_PDL_ENTRY();
  const int r = blockIdx.y;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < d; c += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t ctr = ((static_cast<uint64_t>(row0 + r) << 32) | static_cast<uint64_t>(c)) * 2ull;
    const uint64_t m1 = mix64(seed ^ mix64(ctr)) >> 40, m2 = mix64(seed ^ mix64(ctr + 1)) >> 40;
    const float u1 = (float)(m1 + 1) * 5.9604644775390625e-8f, u2 = (float)m2 * 5.9604644775390625e-8f;
    const float z = sqrtf(-2.0f * logf(u1)) * cosf(6.283185307179586f * u2);
    const float mu = mean[r * ld + c];
    const float var = fmaxf(sq[r * ld + c] - mu * mu, 0.f);
    out[r * d + c] = fmaf(sqrtf(var), z, mu);
  }
}
void swag_sample(const float* mean, const float* sq, int64_t ld, int64_t d, int row0, int rows, uint64_t seed,
                 float* out, cudaStream_t s) {
  const int blocks = (int)std::min<int64_t>((d + 255) / 256, 1024);
  launch_pdl(swag_sample_kernel, dim3(dim3(blocks, rows)), dim3(256), 0, s, mean, sq, ld, d, row0, seed, out);
}

}  // namespace kern
}  // namespace push
