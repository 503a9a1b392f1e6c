// upd.cu — a10 as ONE streaming tensor-core contraction that produces theta' directly.
//
//   theta'_i = theta_i + (eps/n) [ sum_j K_ij (g_j - r theta_j) + r s_i theta_i ],  r = 2/h
//
// (north star; phi(theta_i) = (1/n) sum_j [K_ij grad log p(theta_j) + grad_{theta_j}
// K_ij] with grad_{theta_j} K_ij = r (theta_i - theta_j) K_ij).  Every term is linear in the rows of the
// 2n x w operand B = [G; Theta] (or [Theta; G], the row order of the adjacent buffers), so the whole
// update is theta'_i[c] = sum_q L[i][q] B[q][c] with the folded coefficient matrix
//   L[i][j_G]     = (eps/n) K_ij
//   L[i][j_Theta] = -(eps/n) r K_ij + [j = own_row + i] (1 + (eps/n) r (s_i - K_ii))
// (update_lhs_split_kernel; R28).  The contraction runs TRANSPOSED so that the streamed operand is
// the MMA's A (from TMEM) and the small L stays resident in shared memory:
//   D[c][i] (TMEM lane c of a 128-column tile, column i) = sum_q B[q][c] L[i][q]   (M = 128, N = NPAD)
// 3xTF32 (both operands split hi + lo, lo*lo dropped), K = 2n <= 128: one TMEM accumulation chunk.  The
// MMAs read their A operand from TMEM, and that read (4 KB per MMA) rather than the math bounds a narrow
// MMA (N = 64: ~115 cycles per MMA measured, tensor pipe 14 % active), so the three products run as TWO
// MMAs per k-step with L's hi and lo rows stacked along N:
//   acc[c][0 .. NPAD)       += Bhi . [Lhi]         (N = 2 NPAD: also acc[c][NPAD .. 2 NPAD) += Bhi . Llo)
//   acc[c][0 .. NPAD)       += Blo . Lhi           (N = NPAD)
// and the epilogue adds the two column halves: theta'_i = acc[i] + acc[NPAD + i].
//
// One persistent CTA per SM streams whole 128-column tiles of B (each element read once from HBM) through
// a deep ring of 512-B-row TMA boxes (scripts/micro/tma_stream.cu: 128-column x 32-row boxes reach 0.94 of
// the HBM copy rate at >= 128 KB in flight per SM; 32-column boxes cap at 0.66):
//   warp 0 lane 0   TMA producer: the resident L hi/lo (once), then 32-row x 128-column stages of B
//   warp 1 lane 0   MMA issuer; warp 1 owns TMEM (two accumulators of 2 NPAD columns + a ring of A slots)
//   warps 2-9       two transform groups taking alternate stages: thread = column c, 32 values -> tf32
//                   hi / lo -> an A slot in TMEM; the stage is released as soon as it is in registers
//   warps 10-17     epilogue: drain theta'[c][i] = acc[i] + acc[NPAD + i] and store it (coalesced along c)
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"
#include "tma_host.h"

namespace push {
namespace kern {

namespace {
constexpr int kUK = 32;                 // rows of B (K) per stage
constexpr int kUCols = 128;             // columns per tile (M)
constexpr int kUXf0 = 2, kUGroups = 2, kUEpi0 = kUXf0 + 4 * kUGroups;
constexpr int kUThreads = 32 * (kUEpi0 + 8);
constexpr int kUMaxKB = 4;              // 2n <= 128
constexpr int kUStage = kUK * kUCols * 4;  // 16 KB
constexpr int kUSmemMax = 227 * 1024;

template <int NPAD>
struct UCfg {
  static constexpr int LTILE = 2 * NPAD * 128;             // one k-block of L: [hi; lo] rows (2 NPAD) x 128 B
  static constexpr int RES = kUMaxKB * LTILE;              // resident L
  static constexpr int STAGES = std::min(10, (kUSmemMax - 2048 - RES) / kUStage);
  static constexpr int ACC = 2 * NPAD;                     // accumulator columns (N of the stacked MMA)
  static constexpr int ASLOT0 = 2 * ACC;                   // two accumulators, then NSLOT A slots of 64 columns
  static constexpr int NSLOT = std::min(6, (512 - ASLOT0) / 64);
  static constexpr int CW = NPAD / 2;                      // accumulator columns per epilogue thread
  static constexpr int SMEM = 1024 + RES + STAGES * kUStage + 1024;
  static_assert(ASLOT0 + 64 * NSLOT <= 512 && NSLOT >= kUGroups, "tmem");
  static_assert(CW % 8 == 0 && SMEM <= kUSmemMax, "cfg");
};

template <int NPAD>
__global__ void __launch_bounds__(kUThreads, 1)
    svgd_update_tc_kernel(const __grid_constant__ CUtensorMap tB, const __grid_constant__ CUtensorMap tLhi,
                          const __grid_constant__ CUtensorMap tLlo, int K2, int64_t w, int rows,
                          float* __restrict__ out) {
  using C = UCfg<NPAD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* res = smem;                       // k-block kb of L at kb * LTILE: hi rows, then lo rows
  uint8_t* stg = smem + C::RES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + C::STAGES * kUStage);
  uint64_t* empty = full + C::STAGES;        // [STAGES] the transform has the stage in registers
  uint64_t* aready = empty + C::STAGES;      // [NSLOT] A slot written
  uint64_t* aempty = aready + C::NSLOT;      // [NSLOT] A slot consumed by the MMAs
  uint64_t* tfull = aempty + C::NSLOT;       // [2]
  uint64_t* tempty = tfull + 2;              // [2]
  uint64_t* bres = tempty + 2;               // resident L landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = (K2 + kUK - 1) / kUK;
  const int64_t ntile = w / kUCols;
  const int64_t t0 = blockIdx.x * ntile / gridDim.x, t1 = (blockIdx.x + 1) * ntile / gridDim.x;
  const int nt = (int)(t1 - t0);
  const int nit = nt * KB;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 128);
    }
    for (int a = 0; a < C::NSLOT; ++a) {
      ptx::mbar_init(&aready[a], 128);
      ptx::mbar_init(&aempty[a], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 256);
    }
    ptx::mbar_init(bres, 1);
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tB);
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
    if (lane == 0) {  // ---------------- TMA producer
      ptx::mbar_arrive_expect_tx(bres, KB * C::LTILE);
      for (int kb = 0; kb < KB; ++kb) {
        ptx::tma_load_3d(res + kb * C::LTILE, &tLhi, bres, kb * kUK, 0, 0);
        ptx::tma_load_3d(res + kb * C::LTILE + NPAD * 128, &tLlo, bres, kb * kUK, 0, 0);
      }
      for (int it = 0; it < nit; ++it) {
        const int lt = it / KB, kb = it - lt * KB, s = it % C::STAGES;
        ptx::mbar_wait(&empty[s], ((it / C::STAGES) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&full[s], kUStage);
        ptx::tma_load_3d(stg + s * kUStage, &tB, &full[s], (int)((t0 + lt) * kUCols), kb * kUK, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer: tile lt into accumulator lt & 1
      constexpr uint32_t idesc2 = ptx::idesc_tf32(128, 2 * NPAD, false, false), idesc1 = ptx::idesc_tf32(128, NPAD, false, false);
      ptx::mbar_wait(bres, 0);
      int it = 0;
      for (int lt = 0; lt < nt; ++lt) {
        const int b = lt & 1;
        ptx::mbar_wait(&tempty[b], ((lt >> 1) & 1) ^ 1);
        const uint32_t d = tmem_base + b * C::ACC;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int a = it % C::NSLOT;
          ptx::mbar_wait(&aready[a], (it / C::NSLOT) & 1);
          ptx::tc_fence_after();
          const uint32_t ta_hi = tmem_base + C::ASLOT0 + a * 64, ta_lo = ta_hi + 32;
          const uint32_t lb = ptx::smem_u32(res + kb * C::LTILE);
#pragma unroll
          for (int ks = 0; ks < kUK / 8; ++ks) {
            const uint64_t dl = ptx::umma_desc(lb + ks * 32, 16, 1024, 2);  // rows [Lhi; Llo] (N = 2 NPAD) or Lhi
            ptx::mma_tf32_ts(d, ta_hi + ks * 8, dl, idesc2, (kb == 0 && ks == 0) ? 0u : 1u);
            ptx::mma_tf32_ts(d, ta_lo + ks * 8, dl, idesc1, 1u);
          }
          ptx::mma_commit(&aempty[a]);
        }
        ptx::mma_commit(&tfull[b]);
      }
    }
  } else if (warp < kUEpi0) {
    // ---------------- transform group g: k-blocks it = g, g + 2, ...  TMEM lane = column c of the tile
    const int g = (warp - kUXf0) >> 2, q = warp & 3, c = 32 * q + lane;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    for (int it = g; it < nit; it += kUGroups) {
      const int s = it % C::STAGES, a = it % C::NSLOT;
      ptx::mbar_wait(&full[s], (it / C::STAGES) & 1);
      const uint32_t st = ptx::smem_u32(stg + s * kUStage);
      float x[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) x[k] = ptx::lds_f32(st + k * (kUCols * 4) + c * 4);
      ptx::mbar_arrive(&empty[s]);  // release-ordered after the loads: the ring slot is free for the TMA
      uint32_t hi[32], lo[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float h = ptx::tf32_rna_fast(x[k]);
        hi[k] = __float_as_uint(h);
        lo[k] = __float_as_uint(x[k] - h);
      }
      ptx::mbar_wait(&aempty[a], ((it / C::NSLOT) & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t ta = tmem_base + lane_off + C::ASLOT0 + a * 64;
      ptx::tmem_st_32x32b_x32(ta, hi);
      ptx::tmem_st_32x32b_x32(ta + 32, lo);
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&aready[a]);
    }
  } else {
    // ---------------- epilogue: quarter q (columns c = 32q + lane of the tile), half h of the rows i
    const int e = warp - kUEpi0, q = warp & 3, h = e >> 2;
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
    const int cl = 32 * q + lane;
    for (int lt = 0; lt < nt; ++lt) {
      const int b = lt & 1;
      ptx::mbar_wait(&tfull[b], (lt >> 1) & 1);
      ptx::tc_fence_after();
      float acc[C::CW];
#pragma unroll
      for (int cb = 0; cb < C::CW; cb += 8) {
        uint32_t v[8], u[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(lane_base + b * C::ACC + h * C::CW + cb));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
                     : "r"(lane_base + b * C::ACC + NPAD + h * C::CW + cb));
        ptx::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[cb + j] = __uint_as_float(v[j]) + __uint_as_float(u[j]);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[b]);
      const int64_t col = (t0 + lt) * kUCols + cl;
#pragma unroll
      for (int j = 0; j < C::CW; ++j) {
        const int i = h * C::CW + j;
        if (i < rows) out[(int64_t)i * w + col] = acc[j];
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem_base, 512);
}

template <int NPAD>
push_status update_tc_launch(const float* b, int n, int64_t w, int rows, const float* lhi, const float* llo, int pitch,
                             float* out, cudaStream_t s) {
  CUtensorMap tB, tLhi, tLlo;
  push_status st = gemm::make_map(&tB, b, (uint64_t)w, (uint64_t)(2 * n), 1, (uint64_t)w, 0, kUK,
                                  CU_TENSOR_MAP_SWIZZLE_NONE, kUCols);
  if (st == PUSH_OK)
    st = gemm::make_map(&tLhi, lhi, (uint64_t)(2 * n), NPAD, 1, (uint64_t)pitch, 0, NPAD, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st == PUSH_OK)
    st = gemm::make_map(&tLlo, llo, (uint64_t)(2 * n), NPAD, 1, (uint64_t)pitch, 0, NPAD, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != PUSH_OK) return st;
  static bool attr = false;
  if (!attr) {
    PUSH_CUDA_TRY(cudaFuncSetAttribute(svgd_update_tc_kernel<NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       UCfg<NPAD>::SMEM));
    attr = true;
  }
  const int64_t ntile = w / kUCols;
  const int grid = (int)std::min<int64_t>(ntile, gemm::sm_count() > 0 ? gemm::sm_count() : 148);
  launch_pdl(svgd_update_tc_kernel<NPAD>, dim3(grid), dim3(kUThreads), UCfg<NPAD>::SMEM, s, tB, tLhi, tLlo, 2 * n, w, rows, out);
  PUSH_CUDA_TRY(cudaGetLastError());
  return PUSH_OK;
}

// L split (R28): rows i < npad (zero past nl) of the folded coefficient matrix over the B rows q
// ([G; Theta] when g_first, else [Theta; G]), as tf32 hi / lo at `pitch`:
//   G row j:      (eps/n) K_ij
//   Theta row j:  -(eps/n) r K_ij, plus 1 + (eps/n) r (s_i - K_ii) on the own particle j = own_row + i
__global__ void update_lhs_split_kernel(const float* __restrict__ K, int nl, int npad, int n, int pitch, int own_row,
                                        const float* __restrict__ hptr, const float* __restrict__ srow, float eps_n,
                                        int g_first, float* __restrict__ hi, float* __restrict__ lo) {
  PUSH_PDL_ENTRY();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)npad * pitch) return;
  const int i = (int)(e / pitch), q = (int)(e - (int64_t)i * pitch);
  float v = 0.f;
  if (i < nl && q < 2 * n) {
    const int j = q < n ? q : q - n;
    const bool gpart = (q < n) == (g_first != 0);
    const float k = K[(int64_t)i * n + j];
    const float er = eps_n * (2.0f / *hptr);
    if (gpart)
      v = eps_n * k;
    else if (j == own_row + i)
      v = fmaf(er, srow[i] - k, 1.0f);
    else
      v = -er * k;
  }
  const float hv = ptx::tf32_rna_fast(v);
  hi[e] = hv;
  lo[e] = v - hv;
}
}  // namespace

int update_tc_npad(int rows) {
  int np = 16;
  while (np < rows) np *= 2;
  return np;
}

push_status update_tc_stream(const float* b, bool g_first, int n, int64_t w, int rows, int own_row, const float* K,
                             const float* h, float* lhs_hi, float* lhs_lo, float* out, const float* srow, float eps_n,
                             cudaStream_t s) {
  if (n < 1 || 2 * n > kUK * kUMaxKB || rows < 1 || rows > kUpdTcMaxRows || w % kUCols)
    return fail(PUSH_E_SHAPE, "update_tc_stream: unsupported shape");
  if (w == 0) return PUSH_OK;
  push_status st = gemm::get_encoder();
  if (st != PUSH_OK) return st;
  const int npad = update_tc_npad(rows), pitch = ((2 * n + 3) / 4) * 4;
  const int64_t tot = (int64_t)npad * pitch;
  launch_pdl(update_lhs_split_kernel, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, s, K, rows, npad, n, pitch, own_row, h, srow,
                                                                         eps_n, g_first ? 1 : 0, lhs_hi, lhs_lo);
  switch (npad) {
    case 16: return update_tc_launch<16>(b, n, w, rows, lhs_hi, lhs_lo, pitch, out, s);
    case 32: return update_tc_launch<32>(b, n, w, rows, lhs_hi, lhs_lo, pitch, out, s);
    default: return update_tc_launch<64>(b, n, w, rows, lhs_hi, lhs_lo, pitch, out, s);
  }
}

}  // namespace kern
}  // namespace push
