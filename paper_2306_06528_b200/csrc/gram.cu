// gram.cu — a7 pairwise squared distances as a centred, symmetric 3xTF32 Gram product on the tensor cores.
//
//   D_ij = ||theta_i - theta_j||^2 = G_ii + G_jj - 2 G_ij,   G = X X^T,  X = Theta - 1 c^T,  c = theta_0
//
// (PAPER.md:632 evaluates the squared-exponential kernel on ||theta_i - theta_j||.)
// D does not change under translation, so the rows are centred on particle 0 before the product:
// the cancellation error of the Gram form then scales with the spread of the particles, not with
// ||theta|| (clustered particles, a pretrained theta0 plus noise: DESIGN.md R27).
//
// Split precision: x = hi + lo, hi = tf32_rn(x), lo = x - hi (exact); G = Hi Hi^T + Lo Hi^T + Hi Lo^T
// (lo*lo dropped, as in the 3xTF32 GEMM).  Because G is symmetric, ONE MMA per k-step computes both
// needed products: the A operand stacks [Hi_I; Lo_I] (128 TMEM lanes: rows of an i-block of 64
// particles, hi then lo) against B = Hi (all n particles, N = NP columns), so the accumulator holds
// X_Ij = Hi_i . Hi_j (lanes 0-63) and Y_Ij = Lo_i . Hi_j (lanes 64-127), and
//   G_ij = sum_s [ X_s(i,j) + Y_s(i,j) + Y_s(j,i) ]
// — two thirds of the tensor work of the general 3xTF32 GEMM and no zero rows in the M = 128 tile.
//
// One CTA streams one column split of Theta (the split plan's ranges, fixed by (n, ld) only, so the
// partials are the same whichever rank computes them: P-invariance, NEXT-4) for one i-block:
//   warp 0 lane 0   TMA producer: NP x 32 fp32 tiles (SWIZZLE_128B, K-major) into a STAGES ring
//   warp 1 lane 0   MMA issuer (tcgen05.mma kind::tf32, A from TMEM, B from smem); warp 1 owns TMEM
//   warps 2-5       transform: centre, split, A rows -> TMEM (tcgen05.st), B tile -> Hi in place
//   warps 6-13      epilogue: TMEM partial added into fp32 registers every 128 of K (the tensor-core
//                   accumulator truncates each add), then the split's [X; Y] block stored to `part`
// The reduction over splits and the distance formula run in gram_dist_kernel (fixed ascending order).
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"
#include "tma_host.h"

namespace push {
namespace kern {

namespace {
constexpr int kGBK = 32;              // fp32 of K per k-block (one 128-B SWIZZLE_128B row per particle)
constexpr int kGChunkKB = 4;          // k-blocks per TMEM accumulation chunk before the fp32 promotion
constexpr int kGThreads = 32 * 14;    // warp 0 TMA, warp 1 MMA, warps 2-5 transform, warps 6-13 epilogue
constexpr int kGSmemTiles = 192 * 1024;

template <int NP>
struct GCfg {
  static constexpr int TILE = NP * 128;                       // NP rows x 128 B
  static constexpr int STAGES = std::min(16, kGSmemTiles / TILE);
  static constexpr int NACC = NP <= 128 ? 2 : 1;               // TMEM accumulators of NP columns
  static constexpr int NSLOT = 4;                              // TMEM A slots of 32 columns
  static constexpr int ASLOT0 = NACC * NP;
  static constexpr int CW = NP >= 32 ? NP / 2 : 16;            // accumulator columns per epilogue thread
  static constexpr int EPI_SPLIT = NP / CW;                    // epilogue warps per TMEM lane quarter
  static constexpr int SMEM = 1024 + STAGES * TILE + 512;
  static_assert(ASLOT0 + 32 * NSLOT <= 512, "tmem");
  static_assert(CW % 16 == 0 && STAGES >= 2, "cfg");
};

__device__ __forceinline__ void bar_transform() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

template <int NP>
__global__ void __launch_bounds__(kGThreads, 1)
    gram_partial_kernel(const __grid_constant__ CUtensorMap tTh, const int64_t* __restrict__ ranges, int n, int n_ib,
                        float* __restrict__ part) {
  using C = GCfg<NP>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::TILE);
  uint64_t* ready = full + C::STAGES;
  uint64_t* empty = ready + C::STAGES;
  uint64_t* aempty = empty + C::STAGES;
  uint64_t* tfull = aempty + C::NSLOT;
  uint64_t* tempty = tfull + C::NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + C::NACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, ib = blockIdx.y;
  const int64_t c0 = ranges[2 * split], c1 = ranges[2 * split + 1];
  const int nkb = (int)((c1 - c0) / kGBK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&ready[s], 128);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int j = 0; j < C::NSLOT; ++j) ptx::mbar_init(&aempty[j], 1);
    for (int b = 0; b < C::NACC; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 32 * 4 * C::EPI_SPLIT);
    }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tTh);
  }
  if (warp == 1) {
    ptx::tmem_alloc(tmem_slot, 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = ptx::lds_u32(ptx::smem_u32(tmem_slot));

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer: rows 0..NP-1 (OOB rows zero-filled), 32 columns
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        ptx::mbar_wait(&empty[s], ((i / C::STAGES) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&full[s], C::TILE);
        ptx::tma_load_3d(smem + s * C::TILE, &tTh, &full[s], (int)(c0 + (int64_t)i * kGBK), 0, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = ptx::idesc_tf32(128, NP, false, false);
      uint32_t ch = 0;
      for (int i = 0; i < nkb; ++i) {
        const bool first = (i % kGChunkKB) == 0;
        const bool last = (i % kGChunkKB) == kGChunkKB - 1 || i == nkb - 1;
        const int b = ch % C::NACC;
        if (first) ptx::mbar_wait(&tempty[b], ((ch / C::NACC) & 1) ^ 1);
        const int s = i % C::STAGES, slot = i % C::NSLOT;
        ptx::mbar_wait(&ready[s], (i / C::STAGES) & 1);
        ptx::tc_fence_after();
        const uint32_t bb = ptx::smem_u32(smem + s * C::TILE);
        const uint32_t ta = tmem_base + C::ASLOT0 + slot * 32;
        const uint32_t d = tmem_base + b * NP;
#pragma unroll
        for (int ks = 0; ks < kGBK / 8; ++ks)
          ptx::mma_tf32_ts(d, ta + ks * 8, ptx::umma_desc(bb + ks * 32, 16, 1024, 2), idesc,
                           (first && ks == 0) ? 0u : 1u);
        ptx::mma_commit(&empty[s]);
        ptx::mma_commit(&aempty[slot]);
        if (last) {
          ptx::mma_commit(&tfull[b]);
          ++ch;
        }
      }
    }
  } else if (warp < 6) {
    // ---------------- transform.  TMEM lane tl = 32 (warp & 3) + lane (the quarter a warp may access):
    // lanes 0-63 take Hi of i-block row (tl & 63), lanes 64-127 its Lo.  Thread t also rewrites the B
    // tile in place: 16-B chunk cc = t & 7 of rows t >> 3, t >> 3 + 16, ... become Hi (rows >= n: 0).
    const int t = threadIdx.x - 64;
    const int tl = 32 * (warp & 3) + lane;
    const int arow = ib * 64 + (tl & 63);  // particle row (== row of the staged tile)
    const bool want_lo = tl >= 64;
    const int cc = t & 7;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::STAGES, slot = i % C::NSLOT;
      ptx::mbar_wait(&full[s], (i / C::STAGES) & 1);
      ptx::mbar_wait(&aempty[slot], ((i / C::NSLOT) & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t st = ptx::smem_u32(smem + s * C::TILE);
      // c = raw row 0 (swizzle of row 0 is the identity), read before any in-place write
      float cv[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 v = ptx::lds_f4(st + (q << 4));
        cv[4 * q] = v.x; cv[4 * q + 1] = v.y; cv[4 * q + 2] = v.z; cv[4 * q + 3] = v.w;
      }
      uint32_t a[32];
      if (arow < n) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = ptx::lds_f4(st + arow * 128 + ((q ^ (arow & 7)) << 4));
          const float xv[4] = {v.x - cv[4 * q], v.y - cv[4 * q + 1], v.z - cv[4 * q + 2], v.w - cv[4 * q + 3]};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float h = ptx::tf32_rna_fast(xv[u]);
            a[4 * q + u] = __float_as_uint(want_lo ? xv[u] - h : h);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < 32; ++k) a[k] = 0u;
      }
      ptx::tmem_st_32x32b_x32(tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + C::ASLOT0 + slot * 32, a);
      float4 c4 = make_float4(0.f, 0.f, 0.f, 0.f);  // chunk cc of c (no dynamic register indexing)
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q == cc) c4 = make_float4(cv[4 * q], cv[4 * q + 1], cv[4 * q + 2], cv[4 * q + 3]);
      bar_transform();  // every raw read of the stage is done before the tile is overwritten
#pragma unroll 4
      for (int j = t >> 3; j < NP; j += 16) {
        const uint32_t ad = st + j * 128 + ((cc ^ (j & 7)) << 4);
        float4 v = ptx::lds_f4(ad);
        if (j < n) {
          v.x = ptx::tf32_rna_fast(v.x - c4.x);
          v.y = ptx::tf32_rna_fast(v.y - c4.y);
          v.z = ptx::tf32_rna_fast(v.z - c4.z);
          v.w = ptx::tf32_rna_fast(v.w - c4.w);
        } else {
          v = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        ptx::sts_f4(ad, v);
      }
      ptx::tmem_st_wait();
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&ready[s]);
    }
  } else {
    // ---------------- epilogue: quarter q of the 128 lanes, column half h
    const int e = warp - 6, q = warp & 3, h = e >> 2;
    if (h < C::EPI_SPLIT) {
      const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
      float acc[C::CW];
#pragma unroll
      for (int j = 0; j < C::CW; ++j) acc[j] = 0.f;
      const int nch = (nkb + kGChunkKB - 1) / kGChunkKB;
      for (int ch = 0; ch < nch; ++ch) {
        const int b = ch % C::NACC;
        ptx::mbar_wait(&tfull[b], (ch / C::NACC) & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int cb = 0; cb < C::CW; cb += 16) {
          uint32_t r[16];
          ptx::tmem_ld_32x32b_x16(lane_base + b * NP + h * C::CW + cb, r);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[cb + j] += __uint_as_float(r[j]);
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[b]);
      }
      // [X; Y] block of (split, i-block): row r = TMEM lane, NP columns
      float* dst = part + (((int64_t)split * n_ib + ib) * 128 + q * 32 + lane) * NP + h * C::CW;
#pragma unroll
      for (int j = 0; j < C::CW; j += 4)
        *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem_base, 512);
}

template <int NP>
push_status gram_launch(const float* theta, int64_t ld, int n, int splits, const int64_t* ranges, float* part,
                        cudaStream_t s) {
  CUtensorMap map;
  push_status st = gemm::make_map(&map, theta, (uint64_t)ld, (uint64_t)n, 1, (uint64_t)ld, 0, NP,
                                  CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != PUSH_OK) return st;
  static bool attr = false;
  if (!attr) {
    PUSH_CUDA_TRY(cudaFuncSetAttribute(gram_partial_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       GCfg<NP>::SMEM));
    attr = true;
  }
  const int n_ib = (n + 63) / 64;
  gram_partial_kernel<NP><<<dim3(splits, n_ib), kGThreads, GCfg<NP>::SMEM, s>>>(map, ranges, n, n_ib, part);
  PUSH_CUDA_TRY(cudaGetLastError());
  return PUSH_OK;
}
}  // namespace

int gram_np(int n) {
  int np = 16;
  while (np < n) np *= 2;
  return np;
}

int64_t gram_part_floats(int n) { return (int64_t)((n + 63) / 64) * 128 * gram_np(n); }

DistPlan gram_plan(int n, int64_t ld) {
  DistPlan pl{};
  pl.T = 0;  // Gram form
  pl.ntile = (n + 63) / 64;
  pl.npairs = pl.ntile;
  pl.tensors = 1;
  // one wave of CTAs (148 SMs, one CTA each): splits x i-blocks ~ 148, ranges whole 128-column units
  const int64_t units = (ld + 127) / 128;
  int64_t want = std::max<int64_t>(1, 148 / pl.ntile);
  want = std::min(want, units);
  const int64_t per = (units + want - 1) / want;
  pl.cols = per * 128;
  pl.splits = 0;
  for (int64_t c = 0; c < ld; c += pl.cols) {
    pl.ranges.push_back(c);
    pl.ranges.push_back(std::min<int64_t>(ld, c + pl.cols));
    ++pl.splits;
  }
  pl.tsplit.s[0] = 0;
  pl.tsplit.s[1] = pl.splits;
  return pl;
}

push_status gram_partial(const float* theta, int64_t ld, int n, int splits, const int64_t* ranges_dev, float* part,
                         cudaStream_t s) {
  if (n < 2 || n > kGramMaxN) return fail(PUSH_E_SHAPE, "gram_partial: n out of range");
  if (splits < 1) return PUSH_OK;
  push_status st = gemm::get_encoder();
  if (st != PUSH_OK) return st;
  switch (gram_np(n)) {
    case 16: return gram_launch<16>(theta, ld, n, splits, ranges_dev, part, s);
    case 32: return gram_launch<32>(theta, ld, n, splits, ranges_dev, part, s);
    case 64: return gram_launch<64>(theta, ld, n, splits, ranges_dev, part, s);
    case 128: return gram_launch<128>(theta, ld, n, splits, ranges_dev, part, s);
    default: return gram_launch<256>(theta, ld, n, splits, ranges_dev, part, s);
  }
}

// D from the split partials.  A CTA covers 32 consecutive entries (i, j) of row i (lane = j); only
// j > i is computed (written to (i, j) and (j, i)), the diagonal is +0.  Warp w sums the splits
// s = w, w + 8, ... ascending, the 8 warp sums are added in ascending w (the order depends only on the
// split count).  Per split: g_ij += (X(i,j) + Y(i,j)) + Y(j,i), g_aa += (X(a,a) + Y(a,a)) + Y(a,a).
__global__ void __launch_bounds__(256) gram_dist_kernel(const float* __restrict__ part, int n, int np, int n_ib,
                                                        int S, const RankSlots rs, float* __restrict__ D) {
  __shared__ float red[3][8][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  const int64_t nn = (int64_t)n * n;
  const bool ok = e < nn;
  const int i = ok ? (int)(e / n) : 0, j = ok ? (int)(e - (int64_t)i * n) : 0;
  const bool upper = ok && j > i;
  if (!__syncthreads_or(upper)) {  // no entry above the diagonal: only the diagonal (if any) is written
    if (warp == 0 && ok && i == j) D[e] = 0.f;
    return;
  }
  const int64_t pb = (int64_t)n_ib * 128 * np;
  // row offsets inside a split block: X row of particle a at ((a/64)*128 + a%64) * np, Y row 64 further
  auto xrow = [&](int a) { return ((int64_t)(a >> 6) * 128 + (a & 63)) * np; };
  const int64_t xi = xrow(i), xj = xrow(j);
  float gij = 0.f, gii = 0.f, gjj = 0.f;
  if (upper) {
    int q = 0;
    for (int s = warp; s < S; s += 8) {
      while (q + 1 < rs.P && s >= rs.s0[q + 1]) ++q;
      const float* b = part + (int64_t)(q * rs.smax + s - rs.s0[q]) * pb;
      const float x_ij = __ldg(b + xi + j), y_ij = __ldg(b + xi + 64 * np + j), y_ji = __ldg(b + xj + 64 * np + i);
      const float x_ii = __ldg(b + xi + i), y_ii = __ldg(b + xi + 64 * np + i);
      const float x_jj = __ldg(b + xj + j), y_jj = __ldg(b + xj + 64 * np + j);
      gij += (x_ij + y_ij) + y_ji;
      gii += (x_ii + y_ii) + y_ii;
      gjj += (x_jj + y_jj) + y_jj;
    }
  }
  red[0][warp][lane] = gij;
  red[1][warp][lane] = gii;
  red[2][warp][lane] = gjj;
  __syncthreads();
  if (warp == 0 && ok) {
    if (i == j) {
      D[e] = 0.f;
    } else if (upper) {
      float a = red[0][0][lane], b = red[1][0][lane], c = red[2][0][lane];
#pragma unroll
      for (int w = 1; w < 8; ++w) {
        a += red[0][w][lane];
        b += red[1][w][lane];
        c += red[2][w][lane];
      }
      const float d = fmaxf(fmaf(-2.0f, a, b + c), 0.f);
      D[e] = d;
      D[(int64_t)j * n + i] = d;
    }
  }
}

void gram_dist(const float* part, int n, int S, const RankSlots& rs, float* D, cudaStream_t s) {
  const int64_t groups = ((int64_t)n * n + 31) / 32;
  gram_dist_kernel<<<(unsigned)groups, 256, 0, s>>>(part, n, gram_np(n), (n + 63) / 64, S, rs, D);
}

}  // namespace kern
}  // namespace push
