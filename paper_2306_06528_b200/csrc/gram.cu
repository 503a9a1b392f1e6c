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
//   warp 0 lane 0   TMA producer: raw stages of RC columns x NP rows, unswizzled, at a padded row pitch of
//                   RC + 8 floats (the box over-reads 8 columns): 512-B row requests keep the ring at the HBM
//                   rate (scripts/micro/tma_stream.cu: 32-column SWIZZLE_128B boxes cap at ~0.5-0.66 of the
//                   copy rate, 128 + 4-column boxes reach 0.95), and the 32-B row skew makes the transform's
//                   row-wise 8-B reads (8 rows x 32 B per instruction) conflict-free
//   warp 1 lane 0   MMA issuer (tcgen05.mma kind::tf32, A from TMEM, B from smem); warp 1 owns TMEM
//   warps 2-9       two transform groups taking alternate raw stages: per k-block (32 columns) centre and
//                   split each element once (tcgen05.st.16x256b puts its Hi and Lo in two TMEM lanes), Hi
//                   rows -> a SWIZZLE_128B K-major B tile; the raw stage is released as soon as it has been
//                   read, the slot / tile by the MMA commit
//   warps 10-17     epilogue: TMEM partial added into fp32 registers every 128 of K (the tensor-core
//                   accumulator truncates each add), then the split's [X; Y] block stored to `part`
// The reduction over splits and the distance formula run in gram_dist (fixed ascending order).
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "gram_d.cuh"
#include "kernels.h"
#include "ptx.cuh"
#include "tma_host.h"

namespace push {
namespace kern {

namespace {
constexpr int kGBK = 32;              // fp32 of K per k-block (one 128-B SWIZZLE_128B row per particle)
constexpr int kGGroups = 2;           // transform super-groups taking alternate raw stages
constexpr int kGSub = 1;              // 4-warp groups per super-group, splitting a stage's k-blocks
constexpr int kGXf0 = 2, kGEpi0 = kGXf0 + 4 * kGGroups * kGSub;
constexpr int kGThreads = 32 * (kGEpi0 + 8);  // + 8 epilogue warps
constexpr int kGSmemMax = 227 * 1024;

template <int NP>
struct GCfg {
  static constexpr int RC = NP <= 64 ? 128 : (NP == 128 ? 64 : 32);  // raw columns per stage
  static constexpr int KPS = RC / kGBK;                        // k-blocks per raw stage
  static constexpr int PITCH = (RC + 8) * 4;                   // raw row pitch (bytes): 32-B skew per row
  static constexpr int RAW = NP * PITCH;                       // one raw stage
  static constexpr int TILE = NP * kGBK * 4;                   // one B tile (k-block): NP rows x 128 B
  static constexpr int NACC = NP <= 128 ? 2 : 1;               // TMEM accumulators of NP columns
  static constexpr int ASLOT0 = NACC * NP;                     // NE entries of KPS A slots of 32 columns
  // ring of NE entries, one per raw stage: its KPS A slots (TMEM) and KPS B tiles (smem); one barrier
  // round trip (transform -> MMA -> transform) per stage, not per k-block
  static constexpr int NE = std::min(4, std::min((512 - ASLOT0) / (32 * KPS), 98304 / (KPS * TILE)));
  static constexpr int STAGES = std::min(12, (kGSmemMax - 3072 - NE * KPS * TILE) / RAW);
  static constexpr int CW = NP >= 32 ? NP / 2 : 16;            // accumulator columns per epilogue thread
  static constexpr int EPI_SPLIT = NP / CW;                    // epilogue warps per TMEM lane quarter
  static constexpr int OUTER = NP > 64 ? (NP - 64) * 8 / 128 : 0;  // 16-B units per thread outside the i-block
  static constexpr int SMEM = 1024 + NE * KPS * TILE + STAGES * RAW + 1024;
  static_assert(ASLOT0 + 32 * KPS * NE <= 512, "tmem");
  static_assert(CW % 16 == 0 && STAGES >= 2 && NE >= 2 && SMEM <= kGSmemMax, "cfg");
};

// TMEM lane 32q + l of the A operand / accumulator <-> i-block row and part: lane quarter q holds rows
// 16q .. 16q + 15 in two 16-lane blocks (l >> 4); in block hh, lanes 0-7 are the Hi (X) and lanes 8-15 the
// Lo (Y) of rows 16q + 8hh + 0..7 — the tcgen05.st.16x256b layout, where one thread writes both.
__device__ __forceinline__ int lane_row(int q, int lane) { return 16 * q + 8 * (lane >> 4) + (lane & 7); }
__device__ __forceinline__ int lane_part(int lane) { return (lane >> 3) & 1; }

template <int NP>
__global__ void __launch_bounds__(kGThreads, 1)
    gram_partial_kernel(const __grid_constant__ CUtensorMap tTh, const int64_t* __restrict__ ranges, int n, int n_ib,
                        float* __restrict__ part) {
  using C = GCfg<NP>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* btile = smem;                       // [NE][KPS] B tiles (SWIZZLE_128B, 1024-B aligned)
  uint8_t* raw = smem + C::NE * C::KPS * C::TILE;  // [STAGES] raw stages
  uint64_t* full = reinterpret_cast<uint64_t*>(raw + C::STAGES * C::RAW);
  uint64_t* empty = full + C::STAGES;          // raw stage read by its transform group
  uint64_t* ready = empty + C::STAGES;         // [NE] A slots + B tiles of a stage written
  uint64_t* freed = ready + C::NE;             // [NE] consumed by the MMAs
  uint64_t* tfull = freed + C::NE;
  uint64_t* tempty = tfull + C::NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + C::NACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, ib = blockIdx.y;
  const int64_t c0 = ranges[2 * split], c1 = ranges[2 * split + 1];
  const int nst = (int)((c1 - c0) / C::RC);  // ranges are whole 128-column units
  const int nkb = nst * C::KPS;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 128 * kGSub);
    }
    for (int e = 0; e < C::NE; ++e) {
      ptx::mbar_init(&ready[e], 128 * kGSub);
      ptx::mbar_init(&freed[e], 1);
    }
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
  PUSH_PDL_ENTRY();  // set-up above touched no global memory (common.cuh)

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer: RC (+4) columns of rows 0..NP-1 (OOB zero-filled)
      for (int i = 0; i < nst; ++i) {
        const int s = i % C::STAGES;
        ptx::mbar_wait(&empty[s], ((i / C::STAGES) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&full[s], C::RAW);
        ptx::tma_load_3d(raw + s * C::RAW, &tTh, &full[s], (int)(c0 + (int64_t)i * C::RC), 0, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer: per raw stage; 4 k-blocks (128 of K) = one accumulation chunk
      constexpr uint32_t idesc = ptx::idesc_tf32(128, NP, false, false);
      int ch = 0;
      for (int i = 0; i < nst; ++i) {
        const int e = i % C::NE;
        ptx::mbar_wait(&ready[e], (i / C::NE) & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int j = 0; j < C::KPS; ++j) {
          const int k = i * C::KPS + j;
          const bool first = (k & 3) == 0, last = (k & 3) == 3 || k == nkb - 1;
          const int b = ch % C::NACC;
          if (first) {
            ptx::mbar_wait(&tempty[b], ((ch / C::NACC) & 1) ^ 1);
            ptx::tc_fence_after();
          }
          const uint32_t d = tmem_base + b * NP, ta = tmem_base + C::ASLOT0 + (e * C::KPS + j) * 32;
          const uint32_t bb = ptx::smem_u32(btile + (e * C::KPS + j) * C::TILE);
#pragma unroll
          for (int ks = 0; ks < kGBK / 8; ++ks)
            ptx::mma_tf32_ts(d, ta + ks * 8, ptx::umma_desc(bb + ks * 32, 16, 1024, 2), idesc,
                             (first && ks == 0) ? 0u : 1u);
          if (last) {
            ptx::mma_commit(&tfull[b]);
            ++ch;
          }
        }
        ptx::mma_commit(&freed[e]);
      }
    }
  } else if (warp < kGEpi0) {
    // ---------------- transform super-group sg: raw stages sg, sg + 2, ...; its group hb takes the stage's
    // k-blocks hb, hb + kGSub, ...  Each element is converted ONCE: with tcgen05.st.16x256b, thread
    // (t0 = lane & 3, t1 = lane >> 2) writes columns 2 t0, 2 t0 + 1 (+ 8 per repetition) of TMEM lanes t1 (Hi)
    // and t1 + 8 (Lo) of a 16-lane block, so one thread holds both parts of its row (lane_part below); the
    // thread also writes the row's Hi into the B tile.  Rows of the tile outside the i-block (n > 64) are
    // converted 16-B unit by unit.
    const int gg = (warp - kGXf0) >> 2, sg = gg / kGSub, hb = gg % kGSub, q = warp & 3;
    const int t = threadIdx.x - 32 * (kGXf0 + 4 * gg);
    const int t0 = lane & 3, t1 = lane >> 2;
    int arow[2];
    bool live[2], in_tile[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {  // 16-lane block hh of the quarter: rows 16q + 8hh + t1
      arow[hh] = ib * 64 + 16 * q + 8 * hh + t1;
      live[hh] = arow[hh] < n;
      in_tile[hh] = arow[hh] < NP;
    }
    for (int i = sg; i < nst; i += kGGroups) {
      const int s = i % C::STAGES;
      const int e = i % C::NE;
      const uint32_t rs = ptx::smem_u32(raw + s * C::RAW);
      ptx::mbar_wait(&full[s], (i / C::STAGES) & 1);
      if (hb >= C::KPS) {  // no k-block of this stage for this group
        ptx::mbar_arrive(&empty[s]);
        ptx::mbar_arrive(&ready[e]);
        continue;
      }
#pragma unroll 1
      for (int j = hb; j < C::KPS; j += kGSub) {
        const uint32_t bt = ptx::smem_u32(btile + (e * C::KPS + j) * C::TILE);
        // a[hh][4r + {0,1}] = Hi of columns 8r + 2t0 + {0,1}, a[hh][4r + {2,3}] = Lo of the same columns
        uint32_t a[2][16];
        float2 cv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) cv[r] = ptx::lds_f2(rs + (j * 32 + 8 * r + 2 * t0) * 4);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            float2 v = make_float2(0.f, 0.f), c = make_float2(0.f, 0.f);
            if (live[hh]) {
              v = ptx::lds_f2(rs + arow[hh] * C::PITCH + (j * 32 + 8 * r + 2 * t0) * 4);
              c = cv[r];
            }
            const float x0 = v.x - c.x, x1 = v.y - c.y;
            const float h0 = ptx::tf32_rna_fast(x0), h1 = ptx::tf32_rna_fast(x1);
            a[hh][4 * r] = __float_as_uint(h0);
            a[hh][4 * r + 1] = __float_as_uint(h1);
            a[hh][4 * r + 2] = __float_as_uint(x0 - h0);
            a[hh][4 * r + 3] = __float_as_uint(x1 - h1);
          }
        }
        if (j == hb) ptx::mbar_wait(&freed[e], ((i / C::NE) & 1) ^ 1);  // entry e (A slots, B tiles) is free
        if constexpr (C::OUTER > 0) {
#pragma unroll 4
          for (int m = 0; m < C::OUTER; ++m) {
            const int u = t + 128 * m, ro = u >> 3, cc = u & 7;
            const int r = ro < ib * 64 ? ro : ro + 64;  // skip the i-block's own 64 rows
            const float4 x = ptx::lds_f4(rs + r * C::PITCH + j * 128 + cc * 16);
            const float4 c = ptx::lds_f4(rs + j * 128 + cc * 16);
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
            if (r < n)
              o = make_float4(ptx::tf32_rna_fast(x.x - c.x), ptx::tf32_rna_fast(x.y - c.y),
                              ptx::tf32_rna_fast(x.z - c.z), ptx::tf32_rna_fast(x.w - c.w));
            ptx::sts_f4(bt + r * 128 + ((cc ^ (r & 7)) << 4), o);
          }
        }
        if (j + kGSub >= C::KPS) ptx::mbar_arrive(&empty[s]);  // this group's reads of the raw stage are done
        ptx::tc_fence_after();
        const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + C::ASLOT0 + (e * C::KPS + j) * 32;
        ptx::tmem_st_16x256b_x4(ta, a[0]);
        ptx::tmem_st_16x256b_x4(ta + (16u << 16), a[1]);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (!in_tile[hh]) continue;
          const int ar = arow[hh];
#pragma unroll
          for (int r = 0; r < 4; ++r) {  // columns 8r + 2t0 + {0,1}: 16-B chunk 2r + t0/2, 8 (t0 & 1) bytes in
            const int chunk = 2 * r + (t0 >> 1);
            ptx::sts_f2(bt + ar * 128 + ((chunk ^ (ar & 7)) << 4) + 8 * (t0 & 1),
                        make_float2(__uint_as_float(a[hh][4 * r]), __uint_as_float(a[hh][4 * r + 1])));
          }
        }
      }
      ptx::tmem_st_wait();
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&ready[e]);
    }
  } else {
    // ---------------- epilogue: quarter q of the 128 lanes, column half h
    const int e = warp - kGEpi0, q = warp & 3, h = e >> 2;
    if (h < C::EPI_SPLIT) {
      const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
      float acc[C::CW];
#pragma unroll
      for (int j = 0; j < C::CW; ++j) acc[j] = 0.f;
      const int nch = (nkb + 3) / 4;
      for (int i = 0; i < nch; ++i) {
        const int b = i % C::NACC;
        ptx::mbar_wait(&tfull[b], (i / C::NACC) & 1);
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
      // [X; Y] block of (split, i-block): X row r at r, Y row r at 64 + r; NP columns
      const int prow = lane_part(lane) * 64 + lane_row(q, lane);
      float* dst = part + (((int64_t)split * n_ib + ib) * 128 + prow) * NP + h * C::CW;
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
  using C = GCfg<NP>;
  CUtensorMap map;
  push_status st = gemm::make_map(&map, theta, (uint64_t)ld, (uint64_t)n, 1, (uint64_t)ld, 0, NP,
                                  CU_TENSOR_MAP_SWIZZLE_NONE, C::RC + 8);
  if (st != PUSH_OK) return st;
  static bool attr = false;
  if (!attr) {
    PUSH_CUDA_TRY(cudaFuncSetAttribute(gram_partial_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  const int n_ib = (n + 63) / 64;
  launch_pdl(gram_partial_kernel<NP>, dim3(dim3(splits, n_ib)), dim3(kGThreads), C::SMEM, s, map, ranges, n, n_ib, part);
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

// Sum of the split partials: sums[e] = sum_s part[slot(s)][e] over one partial block (e < pb).  A CTA
// covers 32 consecutive elements (lane = element, coalesced), warp w of kGRedWarps sums s = w, w + kGRedWarps,
// ... ascending with 8 loads in flight, then the warp sums are added in ascending w: the order depends only
// on S.  32 warps: with ~147 splits every warp issues its loads in one round (8 warps: three dependent rounds).
constexpr int kGRedWarps = 32;
__global__ void __launch_bounds__(32 * kGRedWarps) gram_reduce_kernel(const float* __restrict__ part, int64_t pb,
                                                                      int S, const RankSlots rs,
                                                                      float* __restrict__ sums) {
  PUSH_PDL_ENTRY();
  __shared__ float red[kGRedWarps][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  float v = 0.f;
  if (e < pb) {
    int q = 0;
    for (int sb = warp; sb < S; sb += 8 * kGRedWarps) {
      float t[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int s = sb + kGRedWarps * k;
        t[k] = 0.f;
        if (s < S) {
          while (q + 1 < rs.P && s >= rs.s0[q + 1]) ++q;
          t[k] = __ldg(part + (int64_t)(q * rs.smax + s - rs.s0[q]) * pb + e);
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (sb + kGRedWarps * k < S) v += t[k];
    }
  }
  red[warp][lane] = v;
  __syncthreads();
  if (warp == 0 && e < pb) {
    float r = red[0][lane];
#pragma unroll
    for (int w = 1; w < kGRedWarps; ++w) r += red[w][lane];
    sums[e] = r;
  }
}

// D_ij = D_ji (gram_d_value, gram_d.cuh) for i < j, D_ii = +0
__global__ void gram_d_kernel(const float* __restrict__ sums, int n, int np, float* __restrict__ D) {
  PUSH_PDL_ENTRY();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * n) return;
  const int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
  if (j < i) return;
  if (i == j) {
    D[e] = 0.f;
    return;
  }
  const float d = gram_d_value(sums, np, i, j);
  D[e] = d;
  D[(int64_t)j * n + i] = d;
}

bool gram_d_in_bandwidth(int n) { return n <= kGramDInBandwidth; }

void gram_dist(const float* part, int n, int S, const RankSlots& rs, float* sums, float* D, cudaStream_t s) {
  const int64_t pb = gram_part_floats(n);
  launch_pdl(gram_reduce_kernel, dim3((unsigned)((pb + 31) / 32)), dim3(32 * kGRedWarps), 0, s, part, pb, S, rs, sums);
  if (gram_d_in_bandwidth(n)) return;  // the bandwidth kernel evaluates D while staging its keys
  const int64_t nn = (int64_t)n * n;
  launch_pdl(gram_d_kernel, dim3((unsigned)((nn + 255) / 256)), dim3(256), 0, s, sums, n, gram_np(n), D);
}

}  // namespace kern
}  // namespace push
