// gemm.cu — batched fp32 GEMM on the 5th-gen tensor cores in 3xTF32 split precision.
//
// Used for the per-particle MLP contractions of the SVGD step (DESIGN.md a2/a4/a5):
//   a2  Z_l = A_{l-1} W_l^T (+ b_l, sigma)       A K-major, W K-major      -> EPI_FWD
//   a4  delta_{l-1} = (delta_l W_l) * sigma'     delta K-major, W MN-major -> EPI_BWD
//   a5  dW_l = delta_l^T A_{l-1}  (split-K)      both MN-major             -> EPI_STORE
//
// Every operand x is stored as a pair of float32 arrays hi = tf32_rn(x),
// lo = tf32_rn(x - hi) (written by the producing epilogue or split_hilo_kernel), and
//   C = A_lo*B_hi + A_hi*B_lo + A_hi*B_hi            (3 tcgen05.mma kind::tf32 per k-step)
// accumulates in TMEM in fp32 (the classic 3xTF32 scheme; lo*lo is dropped).
//
// Kernel shape (v2): one 128 x BN output tile per CTA, 6 warps:
//   warp 0 lane 0  TMA producer (4 bulk-tensor loads per stage into swizzled smem)
//   warp 1 lane 0  MMA issuer (single thread, tcgen05.mma + tcgen05.commit)
//   warps 2-5      drain/epilogue: every 128 of K the TMEM partial (double-buffered, 2 x BN
//                  columns) is added into fp32 registers with round-to-nearest — the tensor-core
//                  accumulator truncates on each accumulate, so long chains would cost ~K/8 ulps;
//                  then the fused op and the store.  Warp 2 also owns the TMEM allocation.
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "gemm.h"
#include "ptx.cuh"

namespace push {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 32;          // fp32 per k-block = 128 B = one SWIZZLE_128B row
constexpr int kChunkKB = 4;     // k-blocks per TMEM accumulation chunk (128 of K) before fp32 promotion
constexpr int kEpiThreads = 128;
constexpr int kThreads = 64 + kEpiThreads;  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue (warp 2 owns TMEM)

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);
  static constexpr int STAGES_RAW = (196 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;  // double-buffered accumulator
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
};

struct KParams {
  int M, N, K, splits, kb_per_split, passes, epi, act;
  float* out0;
  float* out1;
  long long ldo, out_pstride, out_sstride;
  const float* bias;
  long long bias_pstride;
  const float* aprev_hi;
  const float* aprev_lo;
  long long ld_aprev, aprev_pstride;
};

// Stage one operand tile (ROWS along M or N, BK along K) into SWIZZLE_128B smem.
//   K-major : one 3-D box {32 k, ROWS, 1}            -> rows of 128 B, 8-row / 1024 B atoms
//   MN-major: ROWS/32 boxes {32 mn, 32 k, 1}        -> [chunk][k][32 mn], chunk stride 4096 B (32-B atom swizzle)
template <bool MN, int ROWS>
__device__ __forceinline__ void load_operand(const CUtensorMap* map, uint8_t* dst, uint64_t* bar, int mn0, int k,
                                             int p) {
  if constexpr (!MN) {
    ptx::tma_load_3d(dst, map, bar, k, mn0, p);
  } else {
#pragma unroll
    for (int c = 0; c < ROWS / 32; ++c) ptx::tma_load_3d(dst + c * 4096, map, bar, mn0 + 32 * c, k, p);
  }
}

// UMMA smem descriptor for k-step `ks` (8 tf32 of K) of a staged operand.
//   K-major  SWIZZLE_128B        : SBO = 1024 B (8-row group), LBO unused; k-step = +32 B inside the atom.
//   MN-major SWIZZLE_128B_BASE32B: 32-bit MN-major operands need the 32-B-atom swizzle (TMA
//     SWIZZLE_128B_ATOM_32B); atom = 4 k-rows x 128 B.  LBO = 4096 B (next 32-wide MN chunk),
//     SBO = 512 B (next 4 k-rows); k-step (8 k) = +1024 B.
template <bool MN>
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int ks) {
  if constexpr (!MN)
    return ptx::umma_desc(base + ks * 32, 16, 1024, 2);
  else
    return ptx::umma_desc(base + ks * 1024, 4096, 512, 1);
}

template <int BN, bool AMN, bool BMN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm3xtf32_kernel(const __grid_constant__ CUtensorMap tA_hi, const __grid_constant__ CUtensorMap tA_lo,
                      const __grid_constant__ CUtensorMap tB_hi, const __grid_constant__ CUtensorMap tB_lo,
                      const KParams prm) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;  // [2] accumulator b holds a finished K-chunk
  uint64_t* tempty = tfull + 2;         // [2] accumulator b has been drained to registers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int p = blockIdx.z / prm.splits, split = blockIdx.z % prm.splits;
  const int nkb_total = (prm.K + BK - 1) / BK;
  const int kb0 = split * prm.kb_per_split;
  const int kb1 = min(nkb_total, kb0 + prm.kb_per_split);
  const int nkb = kb1 - kb0;  // >= 1 (host guarantees non-empty splits)
  const int nchunks = (nkb + kChunkKB - 1) / kChunkKB;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], kEpiThreads);
    }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tA_hi);
    ptx::prefetch_tmap(&tA_lo);
    ptx::prefetch_tmap(&tB_hi);
    ptx::prefetch_tmap(&tB_lo);
  }
  if (warp == 2) {
    ptx::tmem_alloc(tmem_slot, C::TMEM_COLS);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t round = i / C::STAGES;
        ptx::mbar_wait(&empty[s], (round & 1) ^ 1);
        uint8_t* st = smem + s * C::STAGE_BYTES;
        ptx::mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
        const int k = (kb0 + i) * BK;
        load_operand<AMN, BM>(&tA_hi, st, &full[s], m0, k, p);
        load_operand<AMN, BM>(&tA_lo, st + C::A_BYTES, &full[s], m0, k, p);
        load_operand<BMN, BN>(&tB_hi, st + 2 * C::A_BYTES, &full[s], n0, k, p);
        load_operand<BMN, BN>(&tB_lo, st + 2 * C::A_BYTES + C::B_BYTES, &full[s], n0, k, p);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: K-chunks of kChunkKB k-blocks alternate between two TMEM accumulators
      constexpr uint32_t idesc = ptx::idesc_tf32(BM, BN, AMN, BMN);
      for (int i = 0; i < nkb; ++i) {
        const int c = i / kChunkKB, b = c & 1;
        const bool first = (i % kChunkKB) == 0;
        const bool last = (i % kChunkKB) == kChunkKB - 1 || i == nkb - 1;
        if (first && c >= 2) ptx::mbar_wait(&tempty[b], ((c >> 1) - 1) & 1);
        const int s = i % C::STAGES;
        const uint32_t round = i / C::STAGES;
        ptx::mbar_wait(&full[s], round & 1);
        ptx::tc_fence_after();
        const uint32_t a_hi = ptx::smem_u32(smem + s * C::STAGE_BYTES);
        const uint32_t a_lo = a_hi + C::A_BYTES;
        const uint32_t b_hi = a_hi + 2 * C::A_BYTES;
        const uint32_t b_lo = b_hi + C::B_BYTES;
        const uint32_t d = tmem_base + b * BN;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint64_t dah = op_desc<AMN>(a_hi, ks), dal = op_desc<AMN>(a_lo, ks);
          const uint64_t dbh = op_desc<BMN>(b_hi, ks), dbl = op_desc<BMN>(b_lo, ks);
          const uint32_t acc = (first && ks == 0) ? 0u : 1u;
          if (prm.passes == 3) {
            ptx::mma_tf32(d, dal, dbh, idesc, acc);  // small terms first
            ptx::mma_tf32(d, dah, dbl, idesc, 1u);
            ptx::mma_tf32(d, dah, dbh, idesc, 1u);
          } else {
            ptx::mma_tf32(d, dah, dbh, idesc, acc);
          }
        }
        ptx::mma_commit(&empty[s]);    // frees the smem stage when these MMAs complete
        if (last) ptx::mma_commit(&tfull[b]);
      }
    }
  } else {
    // ---------------- epilogue warps 2..5: TMEM lane quarter q = warp % 4
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    float acc[BN];
#pragma unroll
    for (int j = 0; j < BN; ++j) acc[j] = 0.f;
    // fp32 promotion: every K-chunk's TMEM partial is added (round-to-nearest) into registers,
    // bounding the tensor-core accumulation chain to kChunkKB*BK*3/8 accumulates.
    for (int c = 0; c < nchunks; ++c) {
      const int b = c & 1;
      ptx::mbar_wait(&tfull[b], (c >> 1) & 1);
      ptx::tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(lane_base + b * BN + c0, r);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[c0 + j] += __uint_as_float(r[j]);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[b]);
    }
    if (row < prm.M) {
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 32) {
        const int n = n0 + c0;
        if (prm.epi == EPI_STORE) {
          float4* o = reinterpret_cast<float4*>(prm.out0 + p * prm.out_pstride + split * prm.out_sstride +
                                                static_cast<long long>(row) * prm.ldo + n);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            o[j] = make_float4(acc[c0 + 4 * j], acc[c0 + 4 * j + 1], acc[c0 + 4 * j + 2], acc[c0 + 4 * j + 3]);
        } else {
          const long long obase = p * prm.out_pstride + static_cast<long long>(row) * prm.ldo + n;
          float4* oh = reinterpret_cast<float4*>(prm.out0 + obase);
          float4* ol = reinterpret_cast<float4*>(prm.out1 + obase);
          if (prm.epi == EPI_FWD) {
            const float* bias = prm.bias + p * prm.bias_pstride + n;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float h[4], l[4];
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const float a = act_fwd(acc[c0 + 4 * j + t] + __ldg(bias + 4 * j + t), prm.act);
                h[t] = ptx::tf32_rna(a);
                l[t] = ptx::tf32_rna(a - h[t]);
              }
              oh[j] = make_float4(h[0], h[1], h[2], h[3]);
              ol[j] = make_float4(l[0], l[1], l[2], l[3]);
            }
          } else {  // EPI_BWD
            const long long abase = p * prm.aprev_pstride + static_cast<long long>(row) * prm.ld_aprev + n;
            const float4* ah = reinterpret_cast<const float4*>(prm.aprev_hi + abase);
            const float4* al = reinterpret_cast<const float4*>(prm.aprev_lo + abase);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 xh = __ldg(ah + j), xl = __ldg(al + j);
              const float av[4] = {xh.x + xl.x, xh.y + xl.y, xh.z + xl.z, xh.w + xl.w};
              float h[4], l[4];
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const float v = acc[c0 + 4 * j + t] * act_deriv_from_a(av[t], prm.act);
                h[t] = ptx::tf32_rna(v);
                l[t] = ptx::tf32_rna(v - h[t]);
              }
              oh[j] = make_float4(h[0], h[1], h[2], h[3]);
              ol[j] = make_float4(l[0], l[1], l[2], l[3]);
            }
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, C::TMEM_COLS);
}

// ------------------------------------------------------------------ host side
namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

push_status get_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) return fail(PUSH_E_CUDA, "cuTensorMapEncodeTiled not available from the driver");
  return PUSH_OK;
}

// 3-D fp32 tensor map {d0 (contiguous), d1, d2} with box {32, box1, 1}, SWIZZLE_128B, zero OOB fill.
push_status make_map(CUtensorMap* m, const float* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_el,
                     uint64_t stride2_el, uint32_t box1, CUtensorMapSwizzle swz) {
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_el * 4, stride2_el * 4};
  cuuint32_t box[3] = {32, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(PUSH_E_CUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string(int(r)) + ")");
  return PUSH_OK;
}

push_status make_operand_maps(const Operand& op, int mn_extent, int K, int batch, int box_rows, CUtensorMap* mhi,
                              CUtensorMap* mlo) {
  push_status st;
  if (!op.mn_major) {
    const CUtensorMapSwizzle z = CU_TENSOR_MAP_SWIZZLE_128B;
    if ((st = make_map(mhi, op.hi, K, mn_extent, batch, op.ld, op.pstride, box_rows, z)) != PUSH_OK) return st;
    return make_map(mlo, op.lo, K, mn_extent, batch, op.ld, op.pstride, box_rows, z);
  }
  const CUtensorMapSwizzle z = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
  if ((st = make_map(mhi, op.hi, mn_extent, K, batch, op.ld, op.pstride, 32, z)) != PUSH_OK) return st;
  return make_map(mlo, op.lo, mn_extent, K, batch, op.ld, op.pstride, 32, z);
}

template <int BN, bool AMN, bool BMN>
push_status launch_t(const CUtensorMap* maps, const KParams& kp, dim3 grid, cudaStream_t stream) {
  using C = Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    PUSH_CUDA_TRY(cudaFuncSetAttribute(gemm3xtf32_kernel<BN, AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       C::SMEM_BYTES));
    attr_set = true;
  }
  gemm3xtf32_kernel<BN, AMN, BMN><<<grid, kThreads, C::SMEM_BYTES, stream>>>(maps[0], maps[1], maps[2], maps[3], kp);
  PUSH_CUDA_TRY(cudaGetLastError());
  return PUSH_OK;
}

template <int BN>
push_status launch_bn(bool amn, bool bmn, const CUtensorMap* maps, const KParams& kp, dim3 grid, cudaStream_t s) {
  if (!amn && !bmn) return launch_t<BN, false, false>(maps, kp, grid, s);
  if (!amn && bmn) return launch_t<BN, false, true>(maps, kp, grid, s);
  if (amn && !bmn) return launch_t<BN, true, false>(maps, kp, grid, s);
  return launch_t<BN, true, true>(maps, kp, grid, s);
}
}  // namespace

int choose_bn(int N) {
  if (N % 128 == 0) return 128;
  if (N % 64 == 0) return 64;
  return 32;
}

push_status run(const Problem& pb, cudaStream_t stream) {
  if (pb.M < 1 || pb.N < 1 || pb.K < 1 || pb.batch < 1) return fail(PUSH_E_SHAPE, "gemm: empty problem");
  if (pb.N % 32) return fail(PUSH_E_SHAPE, "gemm: N must be a multiple of 32");
  if (pb.A.mn_major && pb.M % 32) return fail(PUSH_E_SHAPE, "gemm: MN-major A needs M % 32 == 0");
  if ((pb.A.ld % 4) || (pb.B.ld % 4) || (pb.A.pstride % 4) || (pb.B.pstride % 4))
    return fail(PUSH_E_SHAPE, "gemm: operand strides must be multiples of 4 elements");
  push_status st;
  if ((st = get_encoder()) != PUSH_OK) return st;
  const int BN = choose_bn(pb.N);
  const int nkb = (pb.K + BK - 1) / BK;
  const int kbps = (nkb + pb.splits - 1) / pb.splits;
  if ((nkb + kbps - 1) / kbps != pb.splits) return fail(PUSH_E_SHAPE, "gemm: split count leaves an empty split");
  CUtensorMap maps[4];
  if ((st = make_operand_maps(pb.A, pb.M, pb.K, pb.batch, BM, &maps[0], &maps[1])) != PUSH_OK) return st;
  if ((st = make_operand_maps(pb.B, pb.N, pb.K, pb.batch, BN, &maps[2], &maps[3])) != PUSH_OK) return st;
  KParams kp;
  kp.M = pb.M; kp.N = pb.N; kp.K = pb.K; kp.splits = pb.splits; kp.kb_per_split = kbps;
  kp.passes = pb.passes; kp.epi = pb.epi; kp.act = pb.act;
  kp.out0 = pb.out0; kp.out1 = pb.out1; kp.ldo = pb.ldo; kp.out_pstride = pb.out_pstride;
  kp.out_sstride = pb.out_sstride; kp.bias = pb.bias; kp.bias_pstride = pb.bias_pstride;
  kp.aprev_hi = pb.aprev_hi; kp.aprev_lo = pb.aprev_lo; kp.ld_aprev = pb.ld_aprev;
  kp.aprev_pstride = pb.aprev_pstride;
  dim3 grid((pb.M + BM - 1) / BM, pb.N / BN, pb.batch * pb.splits);
  if (BN == 128) return launch_bn<128>(pb.A.mn_major, pb.B.mn_major, maps, kp, grid, stream);
  if (BN == 64) return launch_bn<64>(pb.A.mn_major, pb.B.mn_major, maps, kp, grid, stream);
  return launch_bn<32>(pb.A.mn_major, pb.B.mn_major, maps, kp, grid, stream);
}

int effective_splits(int K, int want) {
  const int nkb = (K + BK - 1) / BK;
  if (want < 1) want = 1;
  if (want > nkb) want = nkb;
  const int kbps = (nkb + want - 1) / want;
  return (nkb + kbps - 1) / kbps;
}

}  // namespace gemm
}  // namespace push
