// gemm.cu — batched fp32 GEMM on the 5th-gen tensor cores in 3xTF32 split precision.
//
// Used for the per-particle MLP contractions of the SVGD step (DESIGN.md a2/a4/a5):
//   a2  A_l = sigma(A_{l-1} W_l^T + b_l)            A K-major,  W K-major  (pre-split)   -> EPI_FWD
//   a4  delta_{l-1} = (delta_l W_l) * sigma'(a_{l-1}) delta K-major, W MN-major (pre-split) -> EPI_BWD
//   a5  dW_l = delta_l^T A_{l-1}   (split-K)          both MN-major, both split in-kernel  -> EPI_STORE
//
// 3xTF32: every operand x is used as hi = tf32_rn(x), lo = x - hi and
//   C = A_lo*B_hi + A_hi*B_lo + A_hi*B_hi       (3 tcgen05.mma kind::tf32 per k-step, lo*lo dropped)
// accumulated in TMEM in fp32.  Activations, deltas and weights live in HBM as ONE fp32 array; the
// hi/lo split happens on chip (transform warps), so each byte is read once.
//
// Shared-memory bandwidth is the binding resource of a 3-pass tf32 GEMM (TMA writes, the split and
// three operand reads per k-step all go through it), so the A operand is kept out of it: the
// transform warps write A's hi/lo straight into TMEM and the MMAs read A from TMEM (".kind::tf32
// [d], [a_tmem], b_desc"); only B is read from shared memory.
//
// Kernel shape (v4): persistent, one CTA per SM, tiles of 128 x BN, 14 warps:
//   warp 0 lane 0   TMA producer (A fp32 tile; B as hi/lo pair or fp32 tile) into a STAGES ring
//   warp 1 lane 0   MMA issuer (single thread, tcgen05.mma + tcgen05.commit); warp 1 owns TMEM
//   warps 2-5       transform: thread = row of A -> tf32 hi/lo into one of NSLOT TMEM slots
//                   (tcgen05.st); a plain-fp32 B tile is split in smem (hi in place, lo alongside)
//   warps 6-13      epilogue: TMEM lane quarter q = warp % 4, column half h = (warp - 6) / 4.
//                   Every 128 of K the TMEM partial (NACC buffers of BN columns, rotating across
//                   tiles, so the MMAs of the next tile overlap this epilogue) is added into fp32
//                   registers with round-to-nearest — the tensor-core accumulator truncates on
//                   each accumulate, so long chains would cost ~K/8 ulps.  The fused op is then
//                   applied on double-buffered swizzled 32x16 smem boxes per warp, written with TMA stores.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "gemm.h"
#include "ptx.cuh"
#include "tma_host.h"

namespace push {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 32;          // fp32 per k-block = 128 B = one SWIZZLE_128B row
constexpr int kChunkKB = 4;     // k-blocks per TMEM accumulation chunk (128 of K) before fp32 promotion
constexpr int kXfWarp0 = 2, kXfWarps = 4, kXfThreads = 32 * kXfWarps;
constexpr int kEpiWarp0 = kXfWarp0 + kXfWarps, kEpiWarps = 8;
constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);
constexpr int kHalfBox = 32 * 16 * 4;  // one 32 x 16 fp32 SWIZZLE_64B output box
constexpr int kMaxSmem = 232448;      // 227 KB opt-in dynamic shared memory per CTA

template <int BN, int NB = 2>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = A_BYTES + 2 * B_BYTES;  // A (fp32), B_hi, B_lo
  static constexpr int EPI_BYTES = kEpiWarps * NB * kHalfBox;
  static constexpr int BAR_BYTES = 1024;
  static constexpr int STAGES_RAW = (kMaxSmem - 1024 - EPI_BYTES - BAR_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  static constexpr int NACC = 2;                       // TMEM accumulator buffers (BN columns each)
  static constexpr int NSLOT = 4;                      // TMEM A slots (hi: 32 columns, lo: 32 columns)
  static constexpr int ASLOT0 = NACC * BN;             // first TMEM column of the A slots
  static constexpr int TMEM_COLS = 512;
  static constexpr int EPI_SPLIT = BN >= 64 ? 2 : 1;   // epilogue warps per TMEM lane quarter
  static constexpr int CW = BN / EPI_SPLIT;            // columns per epilogue thread
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + BAR_BYTES;
  static_assert(STAGES >= 2, "smem");
  static_assert(SMEM_BYTES <= kMaxSmem, "smem");
  static_assert(CW % 32 == 0, "epilogue box");
  static_assert(ASLOT0 + 64 * NSLOT <= TMEM_COLS, "tmem");
};

struct KParams {
  int M, N, K, batch, splits, kb_per_split, passes, epi, act;
  int mt, nt, ntiles;
  int a_pz, b_pz;  // 1: operand batched over particles; 0: shared (particle coordinate 0)
  int store;       // 0: BWD output only feeds the fused partials (delta of a thin first layer): no store
  int chunk_kb;    // k-blocks per TMEM accumulation chunk before the fp32 promotion (pair kernel)
  float alpha;     // EPI_STORE: C = alpha * acc (1 for split-K partials; -lambda when dW goes straight into G)
  int dbg;         // debug experiments only (pushdbg_gemm): bit 0 raw fp32 operands (no hi/lo split),
                   // bit 1 skip the epilogue math/stores, bit 2 skip the MMAs (commits only),
                   // bit 3 accumulate the whole K in TMEM (no fp32 promotion)
  const float* bias;
  long long bias_pstride;
  const float* srow;  // UPD
  const float* hptr;
  float* bpart;
  long long bp_sstride, bp_pstride;
  const float* x;
  int din;
  float* xpart;
  long long xp_sstride, xp_pstride;
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

// B split on the staged tile: the tensor core TRUNCATES fp32 operands to tf32 (measured on B200 by
// scripts/tf32_probe.py: the raw-operand product matches truncated inputs to fp32 rounding and
// differs from round-to-nearest inputs by ~1e-3 relative), so the staged fp32 x already IS hi =
// trunc_tf32(x); only lo = x - trunc_tf32(x) (exact in fp32, |lo| < 2^-10 |x|) is written.
__device__ __forceinline__ void split_tile(uint32_t base, uint32_t lo, int bytes, int tx) {
#pragma unroll 4
  for (int i = tx * 16; i < bytes; i += kXfThreads * 16) {
    const float4 v = ptx::lds_f4(base + i);
    float4 l;
    l.x = v.x - ptx::tf32_trunc(v.x);
    l.y = v.y - ptx::tf32_trunc(v.y);
    l.z = v.z - ptx::tf32_trunc(v.z);
    l.w = v.w - ptx::tf32_trunc(v.w);
    ptx::sts_f4(lo + i, l);
  }
}

// generic pointer for a 32-bit shared address (the PTX wrappers take generic smem pointers)
__device__ __forceinline__ void* ptx_ptr(uint32_t saddr) {
  return __cvta_shared_to_generic(saddr);
}

struct TileCoord {
  int p, split, m0, nt;  // particle, K-split, first row, column-tile index
};
__device__ __forceinline__ TileCoord decode(int t, const KParams& prm) {
  TileCoord c;
  const int nt = t % prm.nt;
  t /= prm.nt;
  const int mt = t % prm.mt;
  t /= prm.mt;
  c.split = t % prm.splits;
  c.p = t / prm.splits;
  c.m0 = mt * BM;
  c.nt = nt;
  return c;
}

// Fused epilogue of one 32-row x CW-column slab held in registers (acc), written through the
// warp's double-buffered swizzled 32x16 smem half-boxes with TMA stores (see the v3 notes above).
// aux_ph: parity of the warp's aprev barrier (BWD); the aprev box of group 0 must already be in flight.
constexpr int kEpiMaxDin = 4;  // widest thin first layer fused into the BWD epilogue (push_api kMaxX0)
// FWD: lane l's slice b_l[colw + 4 l .. 4 l + 3] of the warp's CW bias columns (b_l need not be 16-B aligned)
template <int CW, int EPI>
__device__ __forceinline__ float4 load_bias4(const KParams& prm, int lane, int colw, int p) {
  static_assert(CW <= 128, "one float4 of bias per lane");
  float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
  if constexpr (EPI == EPI_FWD) {
    if (4 * lane < CW) {
      const float* bias = prm.bias + p * prm.bias_pstride + colw + 4 * lane;
      b = make_float4(__ldg(bias), __ldg(bias + 1), __ldg(bias + 2), __ldg(bias + 3));
    }
  }
  return b;
}
// Boxes per epilogue warp: the BWD epilogue keeps kAuxAhead aprev loads in flight ahead of the group it
// computes (its HBM load latency was exposed on every 16-column group with one box ahead), so it needs
// 2 + kAuxAhead boxes; the others double-buffer their stores.
constexpr int kAuxAhead = 2;
template <int EPI>
struct EpiBoxes { static constexpr int NB = (EPI == EPI_BWD || EPI == EPI_UPD) ? 2 + kAuxAhead : 2; };

template <int CW, int EPI, int ACT>
__device__ __forceinline__ void epi_tile(const float (&acc)[CW], const KParams& prm, const CUtensorMap* tOut,
                                         const CUtensorMap* tAux, uint64_t* auxbar, uint32_t& aux_ph,
                                         uint32_t ebuf_s, int lane, int row0, int colw, int p, int pz,
                                         float4 bias4) {
  constexpr bool bwd = EPI == EPI_BWD;
  constexpr bool aux = EPI == EPI_BWD || EPI == EPI_UPD;  // an [m][n] tile is loaded beside the output
  constexpr int NB = EpiBoxes<EPI>::NB;
  float urs = 0.f;  // UPD: (2/h) s_row for this thread's row (rows past M are never stored)
  if constexpr (EPI == EPI_UPD) {
    const int row = row0 + lane;
    if (row < prm.M) urs = (2.0f / __ldg(prm.hptr)) * __ldg(prm.srow + row);
  }
        // Output in 16-column groups g, double-buffered: group g is staged in half-box (g & 1)
        // (32 rows x 16 fp32, SWIZZLE_64B: 16-B chunk c of row r sits at chunk c ^ ((r >> 1) & 3)),
        // so the TMA store of group g overlaps the math of group g + 1.
        constexpr int G = CW / 16;
        // BWD with a fused thin first layer: lane l holds x[row0 + l][0 .. din) (0 past M); the 16 rows a
        // lane's column partial needs arrive by shuffles instead of 16 global loads per group and input
        float xrow[kEpiMaxDin];
#pragma unroll
        for (int i = 0; i < kEpiMaxDin; ++i) xrow[i] = 0.f;
        if (bwd && prm.bpart) {
          const int row = row0 + lane;
#pragma unroll
          for (int i = 0; i < kEpiMaxDin; ++i)
            if (i < prm.din && row < prm.M) xrow[i] = __ldg(prm.x + (long long)row * prm.din + i);
        }
        const uint32_t roff = lane * 64;
        const int swz = (lane >> 1) & 3;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int col = colw + g * 16;
          const uint32_t buf = ebuf_s + (g % NB) * kHalfBox;
          if constexpr (aux) {
            ptx::mbar_wait(auxbar + (g % NB), (aux_ph >> (g % NB)) & 1);  // aux tile of group g is in buf
            aux_ph ^= 1u << (g % NB);
            // prefetch aprev of group g + kAuxAhead into box (g + kAuxAhead) % NB once the store of its
            // previous tenant (group g - 2) has read it: only the latest store (group g - 1) may be pending
            if (g + kAuxAhead < G && lane == 0) {
              if constexpr (NB - 1 - kAuxAhead == 0)
                ptx::bulk_wait_read0();
              else
                ptx::bulk_wait_read1();
              const int nbx = (g + kAuxAhead) % NB;
              ptx::mbar_arrive_expect_tx(auxbar + nbx, kHalfBox);
              ptx::tma_load_3d(ptx_ptr(ebuf_s + nbx * kHalfBox), tAux, auxbar + nbx, col + 16 * kAuxAhead, row0, p);
            }
            __syncwarp();
          } else {
            if (lane == 0) ptx::bulk_wait_read1();  // the store of group g - 2 has finished reading buf
            __syncwarp();
          }
          if constexpr (EPI == EPI_FWD) {
            // b_l[colw + 4 l .. 4 l + 3] sits in lane l (loaded before the accumulator drain): broadcast
            // shuffles instead of 16 dependent global loads per group
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const int src = g * 4 + c4;
              const float4 bv = make_float4(__shfl_sync(0xffffffffu, bias4.x, src), __shfl_sync(0xffffffffu, bias4.y, src),
                                            __shfl_sync(0xffffffffu, bias4.z, src), __shfl_sync(0xffffffffu, bias4.w, src));
              float4 v;
              v.x = act_fwd(acc[g * 16 + 4 * c4 + 0] + bv.x, ACT);
              v.y = act_fwd(acc[g * 16 + 4 * c4 + 1] + bv.y, ACT);
              v.z = act_fwd(acc[g * 16 + 4 * c4 + 2] + bv.z, ACT);
              v.w = act_fwd(acc[g * 16 + 4 * c4 + 3] + bv.w, ACT);
              ptx::sts_f4(buf + roff + ((c4 ^ swz) << 4), v);
            }
          } else if constexpr (bwd) {
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const uint32_t pp = buf + roff + ((c4 ^ swz) << 4);
              const float4 a = ptx::lds_f4(pp);
              float4 v;
              v.x = acc[g * 16 + 4 * c4 + 0] * act_deriv_from_a(a.x, ACT);
              v.y = acc[g * 16 + 4 * c4 + 1] * act_deriv_from_a(a.y, ACT);
              v.z = acc[g * 16 + 4 * c4 + 2] * act_deriv_from_a(a.z, ACT);
              v.w = acc[g * 16 + 4 * c4 + 3] * act_deriv_from_a(a.w, ACT);
              ptx::sts_f4(pp, v);
            }
          } else if constexpr (EPI == EPI_UPD) {
            // t + eps (acc + r s t) (the former fix-up pass), row = row0 + lane (rs per thread)
            const float al = prm.alpha;
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const uint32_t pp = buf + roff + ((c4 ^ swz) << 4);
              const float4 a = ptx::lds_f4(pp);
              float4 v;
              v.x = fmaf(al, fmaf(urs, a.x, acc[g * 16 + 4 * c4 + 0]), a.x);
              v.y = fmaf(al, fmaf(urs, a.y, acc[g * 16 + 4 * c4 + 1]), a.y);
              v.z = fmaf(al, fmaf(urs, a.z, acc[g * 16 + 4 * c4 + 2]), a.z);
              v.w = fmaf(al, fmaf(urs, a.w, acc[g * 16 + 4 * c4 + 3]), a.w);
              ptx::sts_f4(pp, v);
            }
          } else {
            const float al = prm.alpha;
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4)
              ptx::sts_f4(buf + roff + ((c4 ^ swz) << 4),
                          make_float4(al * acc[g * 16 + 4 * c4], al * acc[g * 16 + 4 * c4 + 1],
                                      al * acc[g * 16 + 4 * c4 + 2], al * acc[g * 16 + 4 * c4 + 3]));
          }
          __syncwarp();
          if (bwd && prm.bpart) {  // (bwd is constexpr)
            // a5 of the layer below: column partial sums of delta over this warp's 32 rows (rows >= M are
            // zero: their A rows were zero-filled by TMA).  Lane l: column l & 15, rows 16*(l >> 4) + 0..15
            // ascending, then the two halves added (commutative, so both lanes get the same bits).
            const int rb = row0 / 32;
            const int cl = lane & 15, r0 = (lane >> 4) * 16;
            float v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r)
              v[r] = ptx::lds_f32(buf + (r0 + r) * 64 + ((((cl >> 2) ^ (((r0 + r) >> 1) & 3)) << 4) | ((cl & 3) << 2)));
            float sm = 0.f;
#pragma unroll
            for (int r = 0; r < 16; ++r) sm += v[r];
            sm += __shfl_xor_sync(0xffffffffu, sm, 16);
            if (lane < 16) prm.bpart[rb * prm.bp_sstride + p * prm.bp_pstride + col + cl] = sm;
#pragma unroll
            for (int i = 0; i < kEpiMaxDin; ++i) {
              if (i >= prm.din) break;
              float sx = 0.f;
#pragma unroll
              for (int r = 0; r < 16; ++r) sx = fmaf(v[r], __shfl_sync(0xffffffffu, xrow[i], r0 + r), sx);
              sx += __shfl_xor_sync(0xffffffffu, sx, 16);
              if (lane < 16)
                prm.xpart[rb * prm.xp_sstride + p * prm.xp_pstride + (long long)(col + cl) * prm.din + i] = sx;
            }
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (prm.store) {
              ptx::tma_store_3d(tOut, ptx_ptr(buf), col, row0, pz);
              ptx::bulk_commit();
            }
          }
        }
      }

// The activation is resolved once per tile, so each epilogue body is straight-line code (a per-element
// runtime switch left a branch between every element's tanh and no instruction-level parallelism).
template <int CW, int EPI>
__device__ __forceinline__ void epi_tile_act(const float (&acc)[CW], const KParams& prm, const CUtensorMap* tOut,
                                             const CUtensorMap* tAux, uint64_t* auxbar, uint32_t& aux_ph,
                                             uint32_t ebuf_s, int lane, int row0, int colw, int p, int pz,
                                             float4 bias4) {
  if (EPI == EPI_STORE || prm.act == PUSH_ACT_IDENTITY)
    epi_tile<CW, EPI, PUSH_ACT_IDENTITY>(acc, prm, tOut, tAux, auxbar, aux_ph, ebuf_s, lane, row0, colw, p, pz, bias4);
  else if (prm.act == PUSH_ACT_TANH)
    epi_tile<CW, EPI, PUSH_ACT_TANH>(acc, prm, tOut, tAux, auxbar, aux_ph, ebuf_s, lane, row0, colw, p, pz, bias4);
  else
    epi_tile<CW, EPI, PUSH_ACT_RELU>(acc, prm, tOut, tAux, auxbar, aux_ph, ebuf_s, lane, row0, colw, p, pz, bias4);
}

template <int BN, bool AMN, bool BMN, bool BSPLIT, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm3xtf32_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tBhi,
                      const __grid_constant__ CUtensorMap tBlo, const __grid_constant__ CUtensorMap tOut,
                      const __grid_constant__ CUtensorMap tAux, const KParams prm) {
  constexpr int NB = EpiBoxes<EPI>::NB;
  using C = Cfg<BN, NB>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B aligned base for the SWIZZLE_128B atoms; pointer arithmetic on the __shared__ array keeps
  // every derived pointer in the shared state space (LDS/STS, not generic loads)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ebuf_all = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(ebuf_all + C::EPI_BYTES);
  uint64_t* ready = full + C::STAGES;
  uint64_t* empty = ready + C::STAGES;
  uint64_t* aempty = empty + C::STAGES;  // [NSLOT] the MMAs reading TMEM A slot j have completed
  uint64_t* tfull = aempty + C::NSLOT;   // [NACC] accumulator b holds a finished K-chunk
  uint64_t* tempty = tfull + C::NACC;    // [NACC] accumulator b has been drained to registers
  uint64_t* auxbar = tempty + C::NACC;   // [kEpiWarps][NB] aprev landed in box b of the warp
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(auxbar + kEpiWarps * NB);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb_total = (prm.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&ready[s], kXfThreads);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int j = 0; j < C::NSLOT; ++j) ptx::mbar_init(&aempty[j], 1);
    for (int b = 0; b < C::NACC; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 32 * 4 * C::EPI_SPLIT);
    }
    for (int e = 0; e < kEpiWarps * NB; ++e) ptx::mbar_init(&auxbar[e], 1);
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tA);
    ptx::prefetch_tmap(&tBhi);
    if (!BSPLIT) ptx::prefetch_tmap(&tBlo);
    if (prm.store) ptx::prefetch_tmap(&tOut);
    if (EPI == EPI_BWD || EPI == EPI_UPD) ptx::prefetch_tmap(&tAux);
  }
  if (warp == 1) {
    ptx::tmem_alloc(tmem_slot, C::TMEM_COLS);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = ptx::lds_u32(ptx::smem_u32(tmem_slot));
  PUSH_PDL_ENTRY();  // set-up above touched no global memory (common.cuh)

  auto tile_kb = [&](int split, int* kb0) {
    *kb0 = split * prm.kb_per_split;
    return min(nkb_total, *kb0 + prm.kb_per_split) - *kb0;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      constexpr uint32_t kTx = C::A_BYTES + (BSPLIT ? C::B_BYTES : 2 * C::B_BYTES);
      uint32_t it = 0;
      for (int t = blockIdx.x; t < prm.ntiles; t += gridDim.x) {
        TileCoord tc = decode(t, prm);
        const int n0 = tc.nt * BN;
        int kb0;
        const int nkb = tile_kb(tc.split, &kb0);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % C::STAGES;
          const uint32_t u = it / C::STAGES;
          ptx::mbar_wait(&empty[s], (u & 1) ^ 1);
          uint8_t* st = smem + s * C::STAGE_BYTES;
          ptx::mbar_arrive_expect_tx(&full[s], kTx);
          const int k = (kb0 + i) * BK;
          load_operand<AMN, BM>(&tA, st, &full[s], tc.m0, k, tc.p * prm.a_pz);
          load_operand<BMN, BN>(&tBhi, st + C::A_BYTES, &full[s], n0, k, tc.p * prm.b_pz);
          if (!BSPLIT) load_operand<BMN, BN>(&tBlo, st + C::A_BYTES + C::B_BYTES, &full[s], n0, k, tc.p * prm.b_pz);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: K-chunks of kChunkKB k-blocks rotate over NACC TMEM accumulators
      constexpr uint32_t idesc = ptx::idesc_tf32(BM, BN, false, BMN);  // A from TMEM (K along columns)
      uint32_t it = 0, ch = 0;
      for (int t = blockIdx.x; t < prm.ntiles; t += gridDim.x) {
        TileCoord tc = decode(t, prm);
        int kb0;
        const int nkb = tile_kb(tc.split, &kb0);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int ckb = (prm.dbg & 8) ? nkb : kChunkKB;  // experiment: one chunk = no fp32 promotion
          const bool first = (i % ckb) == 0;
          const bool last = (i % ckb) == ckb - 1 || i == nkb - 1;
          const int b = ch % C::NACC;
          if (first) ptx::mbar_wait(&tempty[b], ((ch / C::NACC) & 1) ^ 1);
          const int s = it % C::STAGES;
          const int slot = it % C::NSLOT;
          ptx::mbar_wait(&ready[s], (it / C::STAGES) & 1);
          ptx::tc_fence_after();
          const uint32_t b_hi = ptx::smem_u32(smem + s * C::STAGE_BYTES) + C::A_BYTES;
          const uint32_t b_lo = b_hi + C::B_BYTES;
          const uint32_t ta_hi = tmem_base + C::ASLOT0 + slot * 64, ta_lo = ta_hi + 32;
          const uint32_t d = tmem_base + b * BN;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint64_t dbh = op_desc<BMN>(b_hi, ks), dbl = op_desc<BMN>(b_lo, ks);
            const uint32_t acc = (first && ks == 0) ? 0u : 1u;
            if (prm.dbg & 4) {
            } else if (prm.passes == 3) {
              ptx::mma_tf32_ts(d, ta_lo + ks * 8, dbh, idesc, acc);  // small terms first
              ptx::mma_tf32_ts(d, ta_hi + ks * 8, dbl, idesc, 1u);
              ptx::mma_tf32_ts(d, ta_hi + ks * 8, dbh, idesc, 1u);
            } else {
              ptx::mma_tf32_ts(d, ta_hi + ks * 8, dbh, idesc, acc);
            }
          }
          ptx::mma_commit(&empty[s]);      // frees the smem stage when these MMAs complete
          ptx::mma_commit(&aempty[slot]);  // frees the TMEM A slot
          if (last) {
            ptx::mma_commit(&tfull[b]);
            ++ch;
          }
        }
      }
    }
  } else if (warp < kEpiWarp0) {
    // ---------------- transform warps: A tile -> tf32 hi/lo in a TMEM slot (thread = row of A);
    // a plain-fp32 B tile is split in smem (hi in place, lo into the B_lo slot)
    const int tx = threadIdx.x - 32 * kXfWarp0;
    const int q = warp & 3;                  // TMEM lane quarter = rows 32q .. 32q+31 of the A tile
    const int m = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    uint32_t it = 0;
    for (int t = blockIdx.x; t < prm.ntiles; t += gridDim.x) {
      TileCoord tc = decode(t, prm);
      int kb0;
      const int nkb = tile_kb(tc.split, &kb0);
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % C::STAGES;
        const int slot = it % C::NSLOT;
        ptx::mbar_wait(&full[s], (it / C::STAGES) & 1);
        ptx::mbar_wait(&aempty[slot], ((it / C::NSLOT) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t st = ptx::smem_u32(smem + s * C::STAGE_BYTES);
        uint32_t hi[32], lo[32];
        if constexpr (!AMN) {
          // K-major SWIZZLE_128B: row m is 128 B at m*128, 16-B chunk c stored at chunk c ^ (m % 8)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 v = ptx::lds_f4(st + m * 128 + ((c ^ (m & 7)) << 4));
            const float xv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float h = ptx::tf32_rna_fast(xv[u]);
              hi[4 * c + u] = __float_as_uint(h);
              lo[4 * c + u] = __float_as_uint(xv[u] - h);
            }
          }
        } else {
          // MN-major, unswizzled boxes [32 k][32 m] per 32-row chunk: element (k, m) at q*4096 + k*128 + lane*4
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float x = ptx::lds_f32(st + q * 4096 + k * 128 + lane * 4);
            const float h = ptx::tf32_rna_fast(x);
            hi[k] = __float_as_uint(h);
            lo[k] = __float_as_uint(x - h);
          }
        }
        if (prm.dbg & 1) {  // experiment: hand the raw fp32 bits to the tensor core (lo = 0, B unsplit)
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            hi[k] = __float_as_uint(__uint_as_float(hi[k]) + __uint_as_float(lo[k]));
            lo[k] = 0u;
          }
        }
        const uint32_t ta = tmem_base + lane_off + C::ASLOT0 + slot * 64;
        ptx::tmem_st_32x32b_x32(ta, hi);
        ptx::tmem_st_32x32b_x32(ta + 32, lo);
        if (BSPLIT && !(prm.dbg & 1)) split_tile(st + C::A_BYTES, st + C::A_BYTES + C::B_BYTES, C::B_BYTES, tx);
        ptx::tmem_st_wait();
        ptx::fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
        ptx::tc_fence_before();
        ptx::mbar_arrive(&ready[s]);
      }
    }
  } else {
    // ---------------- epilogue warps
    const int e = warp - kEpiWarp0;
    const int q = warp & 3;      // TMEM lane quarter this warp may access
    const int h = e >> 2;        // column half
    if (h < C::EPI_SPLIT) {
      const uint32_t ebuf_s = ptx::smem_u32(ebuf_all + e * NB * kHalfBox);
      const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
      uint32_t ch = 0, aux_ph = 0;
      constexpr bool aux = EPI == EPI_BWD || EPI == EPI_UPD;
      for (int t = blockIdx.x; t < prm.ntiles; t += gridDim.x) {
        TileCoord tc = decode(t, prm);
        const int n0 = tc.nt * BN;
        int kb0;
        const int nkb = tile_kb(tc.split, &kb0);
        const int ckb = (prm.dbg & 8) ? nkb : kChunkKB;
        const int nchunks = (nkb + ckb - 1) / ckb;
        const int row0 = tc.m0 + q * 32;
        const bool live = row0 < prm.M;
        const int colw = n0 + h * C::CW;
        if (aux && live && lane == 0) {  // prefetch aprev / theta of the first groups while the MMAs run
          ptx::bulk_wait_read0();
#pragma unroll
          for (int g = 0; g < kAuxAhead && g < C::CW / 16; ++g) {
            ptx::mbar_arrive_expect_tx(&auxbar[e * NB + g], kHalfBox);
            ptx::tma_load_3d(ptx_ptr(ebuf_s + g * kHalfBox), &tAux, &auxbar[e * NB + g], colw + 16 * g, row0, tc.p);
          }
        }
        const float4 bias4 = load_bias4<C::CW, EPI>(prm, lane, colw, tc.p);
        float acc[C::CW];
#pragma unroll
        for (int j = 0; j < C::CW; ++j) acc[j] = 0.f;
        // fp32 promotion: every K-chunk's TMEM partial is added (round-to-nearest) into registers,
        // bounding the tensor-core accumulation chain to kChunkKB*BK*3/8 accumulates.
        for (int c = 0; c < nchunks; ++c, ++ch) {
          const int b = ch % C::NACC;
          ptx::mbar_wait(&tfull[b], (ch / C::NACC) & 1);
          ptx::tc_fence_after();
          // two TMEM loads in flight per wait (each load-wait round trip costs ~200 cycles with 8 warps)
#pragma unroll
          for (int c0 = 0; c0 < C::CW; c0 += 32) {
            uint32_t r0[16], r1[16];
            ptx::tmem_ld_32x32b_x16(lane_base + b * BN + h * C::CW + c0, r0);
            ptx::tmem_ld_32x32b_x16(lane_base + b * BN + h * C::CW + c0 + 16, r1);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              acc[c0 + j] += __uint_as_float(r0[j]);
              acc[c0 + 16 + j] += __uint_as_float(r1[j]);
            }
          }
          ptx::tc_fence_before();
          ptx::mbar_arrive(&tempty[b]);
        }
        if (!live || (prm.dbg & 2)) continue;
        const int pz = EPI == EPI_STORE ? tc.split * prm.batch + tc.p : tc.p;
        epi_tile_act<C::CW, EPI>(acc, prm, &tOut, &tAux, &auxbar[e * NB], aux_ph, ebuf_s, lane, row0, colw, tc.p, pz,
                                 bias4);
      }
      if (lane == 0) ptx::bulk_wait0();
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem_base, C::TMEM_COLS);
}


// ================================================================== v5: CTA-pair kernel (cta_group::2)
// Tiles of 256 x 256 per CTA pair (a 2-CTA cluster): CTA r stages rows [128r, 128r+128) of A (split
// into its own TMEM) and rows [128r, 128r+128) of the B tile; the leader (r = 0) issues
// tcgen05.mma.cta_group::2 (M = 256, N = 256), each CTA's TMEM receives its 128 x 256 slab of D.
// Per SM and k-block this halves the B bytes fetched from L2 and staged in smem relative to the
// 1-CTA kernel at the same MMA work, which is what bounds the 1-CTA kernel.
//   warpgroup 0: warp 0 lane 0 TMA producer; warp 1 lane 0 MMA issuer (leader only), warp 1 owns TMEM
//   warpgroup 1: transform (thread = row of A -> TMEM slot; B lo split in smem when B is plain fp32)
//   warpgroups 2-3: epilogue, 128 accumulator columns per thread (setmaxnreg moves registers there)
// Cross-CTA signalling: transform and epilogue warps of both CTAs arrive on the LEADER's ready /
// tempty barriers (mapa + release.cluster); the leader's commits multicast to both CTAs' empty,
// aempty and tfull barriers.
constexpr int k2Warps = 16, k2Threads = 32 * k2Warps;
constexpr int k2XfWarp0 = 4, k2EpiWarp0 = 8;
// PBN = pair tile width: 256 (one TMEM accumulator of 256 columns, 128 columns per epilogue thread)
// or 128 (two rotating accumulators of 128 columns, so the fused epilogue overlaps the next tile, and
// 32-KB stages, so 6 of them fit).
template <int PBN, int NB = 2>
struct Cfg2 {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = (PBN / 2) * BK * 4;
  static constexpr int STAGE_BYTES = A_BYTES + 2 * B_BYTES;
  static constexpr int EPI_BYTES = kEpiWarps * NB * kHalfBox;
  static constexpr int BAR_BYTES = 1024;
  static constexpr int STAGES_RAW = (kMaxSmem - 1024 - EPI_BYTES - BAR_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  static constexpr int NSLOT = 4;
  static constexpr int NACC = PBN == 256 ? 1 : 2;
  static constexpr int CW = PBN / 2;          // accumulator columns per epilogue thread
  static constexpr int ASLOT0 = NACC * PBN;   // accumulators: [0, 256); A slots: [256, 512)
  static constexpr int TMEM_COLS = 512;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + BAR_BYTES;
  static_assert(STAGES >= 2 && SMEM_BYTES <= kMaxSmem, "smem");
};

template <int PBN, bool AMN, bool BMN, bool BSPLIT, int EPI>
__global__ void __launch_bounds__(k2Threads, 1)
    gemm3xtf32_2sm_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tBhi,
                          const __grid_constant__ CUtensorMap tBlo, const __grid_constant__ CUtensorMap tOut,
                          const __grid_constant__ CUtensorMap tAux, const KParams prm) {
  constexpr int NB = EpiBoxes<EPI>::NB;
  using C = Cfg2<PBN, NB>;
  constexpr int k2BN = PBN, k2CW = C::CW;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ebuf_all = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(ebuf_all + C::EPI_BYTES);
  uint64_t* ready = full + C::STAGES;     // leader: both CTAs' transforms done with stage s
  uint64_t* empty = ready + C::STAGES;    // the pair's MMAs reading stage s have completed
  uint64_t* aempty = empty + C::STAGES;   // [NSLOT] the MMAs reading TMEM A slot j have completed
  uint64_t* tfull = aempty + C::NSLOT;    // [NACC] accumulator b holds a finished K-chunk
  uint64_t* tempty = tfull + C::NACC;     // [NACC] leader: both CTAs have drained accumulator b
  uint64_t* auxbar = tempty + C::NACC;    // [kEpiWarps][NB]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(auxbar + kEpiWarps * NB);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = ptx::cluster_ctarank();
  const int nkb_total = (prm.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&ready[s], 2 * 4);  // one arrival per transform warp of each CTA
      ptx::mbar_init(&empty[s], 1);
    }
    for (int j = 0; j < C::NSLOT; ++j) ptx::mbar_init(&aempty[j], 1);
    for (int b = 0; b < C::NACC; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 2 * kEpiWarps);  // one arrival per epilogue warp of each CTA
    }
    for (int e = 0; e < kEpiWarps * NB; ++e) ptx::mbar_init(&auxbar[e], 1);
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tA);
    ptx::prefetch_tmap(&tBhi);
    if (!BSPLIT) ptx::prefetch_tmap(&tBlo);
    if (prm.store) ptx::prefetch_tmap(&tOut);
    if (EPI == EPI_BWD || EPI == EPI_UPD) ptx::prefetch_tmap(&tAux);
  }
  if (warp == 1) {
    ptx::tmem_alloc2(tmem_slot, C::TMEM_COLS);
    ptx::tmem_relinquish2();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // the peer's barriers are initialised before any remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem_base = ptx::lds_u32(ptx::smem_u32(tmem_slot));
  PUSH_PDL_ENTRY();  // set-up above touched no global memory (common.cuh)

  const int cid = (int)ptx::cluster_id_x(), ncl = (int)ptx::ncluster_x();
  auto tile_kb = [&](int split, int* kb0) {
    *kb0 = split * prm.kb_per_split;
    return min(nkb_total, *kb0 + prm.kb_per_split) - *kb0;
  };
  // pair tile t -> (particle, split, 256-row block, 256-column block)
  auto decode2 = [&](int t, int* p, int* split, int* mp, int* nt) {
    *nt = t % prm.nt;
    t /= prm.nt;
    *mp = t % prm.mt;
    t /= prm.mt;
    *split = t % prm.splits;
    *p = t / prm.splits;
  };

  // setmaxnreg sits at the top of each role's branch so ptxas allocates that region to the new limit
  // (warpgroup 0: producer + MMA issuer + 2 idle warps -> 40; transform -> 104; epilogue -> 184).
  if (warp == 0) {
    ptx::setmaxnreg_dec<40>();
    if (lane == 0) {
      // ---------------- TMA producer (each CTA: its A rows and its half of the B tile)
      constexpr uint32_t kTx = C::A_BYTES + (BSPLIT ? C::B_BYTES : 2 * C::B_BYTES);
      uint32_t it = 0;
      for (int t = cid; t < prm.ntiles; t += ncl) {
        int p, split, mp, nt;
        decode2(t, &p, &split, &mp, &nt);
        const int m0 = mp * 256 + (int)crank * 128;
        const int nb0 = nt * k2BN + (int)crank * (k2BN / 2);
        int kb0;
        const int nkb = tile_kb(split, &kb0);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % C::STAGES;
          ptx::mbar_wait(&empty[s], ((it / C::STAGES) & 1) ^ 1);
          uint8_t* st = smem + s * C::STAGE_BYTES;
          ptx::mbar_arrive_expect_tx(&full[s], kTx);
          const int k = (kb0 + i) * BK;
          load_operand<AMN, BM>(&tA, st, &full[s], m0, k, p * prm.a_pz);
          load_operand<BMN, k2BN / 2>(&tBhi, st + C::A_BYTES, &full[s], nb0, k, p * prm.b_pz);
          if (!BSPLIT)
            load_operand<BMN, k2BN / 2>(&tBlo, st + C::A_BYTES + C::B_BYTES, &full[s], nb0, k, p * prm.b_pz);
        }
      }
    }
  } else if (warp == 1) {
    ptx::setmaxnreg_dec<40>();
    if (lane == 0 && crank == 0) {
      // ---------------- MMA issuer (leader): M = 256 across the pair, N = 256
      constexpr uint32_t idesc = ptx::idesc_tf32(256, k2BN, false, BMN);
      uint32_t it = 0, ch = 0;
      for (int t = cid; t < prm.ntiles; t += ncl) {
        int p, split, mp, nt;
        decode2(t, &p, &split, &mp, &nt);
        int kb0;
        const int nkb = tile_kb(split, &kb0);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int ckb = prm.chunk_kb;
          const bool first = (i % ckb) == 0;
          const bool last = (i % ckb) == ckb - 1 || i == nkb - 1;
          const int b = ch % C::NACC;
          if (first) ptx::mbar_wait(&tempty[b], ((ch / C::NACC) & 1) ^ 1);
          const int s = it % C::STAGES;
          const int slot = it % C::NSLOT;
          ptx::mbar_wait(&ready[s], (it / C::STAGES) & 1);
          ptx::tc_fence_after();
          const uint32_t b_hi = ptx::smem_u32(smem + s * C::STAGE_BYTES) + C::A_BYTES;
          const uint32_t b_lo = b_hi + C::B_BYTES;
          const uint32_t ta_hi = tmem_base + C::ASLOT0 + slot * 64, ta_lo = ta_hi + 32;
          const uint32_t d = tmem_base + b * PBN;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint64_t dbh = op_desc<BMN>(b_hi, ks), dbl = op_desc<BMN>(b_lo, ks);
            const uint32_t acc = (first && ks == 0) ? 0u : 1u;
            if (prm.dbg & 4) {
            } else if (prm.passes == 3) {
              ptx::mma2_tf32_ts(d, ta_lo + ks * 8, dbh, idesc, acc);
              ptx::mma2_tf32_ts(d, ta_hi + ks * 8, dbl, idesc, 1u);
              ptx::mma2_tf32_ts(d, ta_hi + ks * 8, dbh, idesc, 1u);
            } else {
              ptx::mma2_tf32_ts(d, ta_hi + ks * 8, dbh, idesc, acc);
            }
          }
          ptx::mma2_commit_mc(&empty[s], 3);
          ptx::mma2_commit_mc(&aempty[slot], 3);
          if (last) {
            ptx::mma2_commit_mc(&tfull[b], 3);
            ++ch;
          }
        }
      }
    }
  } else if (warp < k2XfWarp0) {
    ptx::setmaxnreg_dec<40>();  // idle warps of warpgroup 0
  } else if (warp < k2EpiWarp0) {
    // ---------------- transform warps (warpgroup 1: lane quarters 0..3)
    ptx::setmaxnreg_dec<104>();
    const int tx = threadIdx.x - 32 * k2XfWarp0;
    const int q = warp & 3;
    const int m = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    uint32_t it = 0;
    for (int t = cid; t < prm.ntiles; t += ncl) {
      int p, split, mp, nt;
      decode2(t, &p, &split, &mp, &nt);
      int kb0;
      const int nkb = tile_kb(split, &kb0);
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % C::STAGES;
        const int slot = it % C::NSLOT;
        ptx::mbar_wait(&full[s], (it / C::STAGES) & 1);
        ptx::mbar_wait(&aempty[slot], ((it / C::NSLOT) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t st = ptx::smem_u32(smem + s * C::STAGE_BYTES);
        uint32_t hi[32], lo[32];
        if constexpr (!AMN) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 v = ptx::lds_f4(st + m * 128 + ((c ^ (m & 7)) << 4));
            const float xv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float h = ptx::tf32_rna_fast(xv[u]);
              hi[4 * c + u] = __float_as_uint(h);
              lo[4 * c + u] = __float_as_uint(xv[u] - h);
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float x = ptx::lds_f32(st + q * 4096 + k * 128 + lane * 4);
            const float h = ptx::tf32_rna_fast(x);
            hi[k] = __float_as_uint(h);
            lo[k] = __float_as_uint(x - h);
          }
        }
        const uint32_t ta = tmem_base + lane_off + C::ASLOT0 + slot * 64;
        ptx::tmem_st_32x32b_x32(ta, hi);
        ptx::tmem_st_32x32b_x32(ta + 32, lo);
        if (BSPLIT) split_tile(st + C::A_BYTES, st + C::A_BYTES + C::B_BYTES, C::B_BYTES, tx);
        ptx::tmem_st_wait();
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&ready[s]), 0), 1);
      }
    }
  } else {
    // ---------------- epilogue warps (warpgroups 2-3): quarter q, column half h of the 256 columns
    ptx::setmaxnreg_inc<184>();  // the fp32 running sum (up to 128 columns) lives in registers
    const int e = warp - k2EpiWarp0;
    const int q = warp & 3;
    const int h = e >> 2;
    const uint32_t ebuf_s = ptx::smem_u32(ebuf_all + e * NB * kHalfBox);
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t tempty_leader = ptx::mapa(ptx::smem_u32(tempty), 0);  // + 8 * b for accumulator b
    uint32_t ch = 0, aux_ph = 0;
    constexpr bool bwd = EPI == EPI_BWD;
    for (int t = cid; t < prm.ntiles; t += ncl) {
      int p, split, mp, nt;
      decode2(t, &p, &split, &mp, &nt);
      int kb0;
      const int nkb = tile_kb(split, &kb0);
      const int nchunks = (nkb + prm.chunk_kb - 1) / prm.chunk_kb;
      const int row0 = mp * 256 + (int)crank * 128 + q * 32;
      const bool live = row0 < prm.M;
      const int colw = nt * k2BN + h * k2CW;
      if (bwd && live && lane == 0) {  // prefetch aprev of the first groups while the MMAs run
        ptx::bulk_wait_read0();
#pragma unroll
        for (int g = 0; g < kAuxAhead && g < k2CW / 16; ++g) {
          ptx::mbar_arrive_expect_tx(&auxbar[e * NB + g], kHalfBox);
          ptx::tma_load_3d(ptx_ptr(ebuf_s + g * kHalfBox), &tAux, &auxbar[e * NB + g], colw + 16 * g, row0, p);
        }
      }
      const float4 bias4 = load_bias4<k2CW, EPI>(prm, lane, colw, p);
      float acc[k2CW];
#pragma unroll
      for (int j = 0; j < k2CW; ++j) acc[j] = 0.f;
      for (int c = 0; c < nchunks; ++c, ++ch) {
        const int b = ch % C::NACC;
        ptx::mbar_wait(&tfull[b], (ch / C::NACC) & 1);
        ptx::tc_fence_after();
        // two TMEM loads in flight per wait (each load-wait round trip costs ~200 cycles with 8 warps)
#pragma unroll
        for (int c0 = 0; c0 < k2CW; c0 += 32) {
          uint32_t r0[16], r1[16];
          ptx::tmem_ld_32x32b_x16(lane_base + b * PBN + h * k2CW + c0, r0);
          ptx::tmem_ld_32x32b_x16(lane_base + b * PBN + h * k2CW + c0 + 16, r1);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            acc[c0 + j] += __uint_as_float(r0[j]);
            acc[c0 + 16 + j] += __uint_as_float(r1[j]);
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader + 8 * b, 1);
      }
      if (!live || (prm.dbg & 2)) continue;
      const int pz = EPI == EPI_STORE ? split * prm.batch + p : p;
      epi_tile_act<k2CW, EPI>(acc, prm, &tOut, &tAux, &auxbar[e * NB], aux_ph, ebuf_s, lane, row0, colw, p, pz,
                              bias4);
    }
    if (lane == 0) ptx::bulk_wait0();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // no CTA leaves while its peer may still signal it or read its TMEM
  if (warp == 1) ptx::tmem_dealloc2(tmem_base, C::TMEM_COLS);
}

// ------------------------------------------------------------------ host side
namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;
int g_sms = 0;
}  // namespace

int sm_count() { return g_sms; }

push_status get_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  });
  if (!g_encode) return fail(PUSH_E_CUDA, "cuTensorMapEncodeTiled not available from the driver");
  return PUSH_OK;
}

// 3-D fp32 tensor map {d0 (contiguous), d1, d2} with box {box0, box1, 1}, zero OOB fill.
push_status make_map(CUtensorMap* m, const float* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_el,
                     uint64_t stride2_el, uint32_t box1, CUtensorMapSwizzle swz, uint32_t box0) {
  if (d2 <= 1) {  // a shared operand: the stride of a unit dimension is never used
    d2 = 1;
    stride2_el = stride1_el * d1;
  }
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_el * 4, stride2_el * 4};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(PUSH_E_CUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string(int(r)) + ")");
  return PUSH_OK;
}

namespace {
// B operands are staged in UMMA-canonical swizzled layouts; the A operand only feeds the transform
// warps (which write it to TMEM), so an MN-major A is staged unswizzled for conflict-free column reads.
push_status make_operand_map(const float* ptr, const Operand& op, int mn_extent, int K, int batch, int box_rows,
                             CUtensorMap* m, bool is_a) {
  const int b = op.pstride == 0 ? 1 : batch;
  if (!op.mn_major)
    return make_map(m, ptr, K, mn_extent, b, op.ld, op.pstride, box_rows, CU_TENSOR_MAP_SWIZZLE_128B);
  return make_map(m, ptr, mn_extent, K, b, op.ld, op.pstride, 32,
                  is_a ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

template <int BN, bool AMN, bool BMN, bool BS, int EPI>
push_status launch_t(const CUtensorMap* maps, const KParams& kp, cudaStream_t stream) {
  using C = Cfg<BN, EpiBoxes<EPI>::NB>;
  static bool attr_set = false;
  if (!attr_set) {
    PUSH_CUDA_TRY(cudaFuncSetAttribute(gemm3xtf32_kernel<BN, AMN, BMN, BS, EPI>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES));
    attr_set = true;
  }
  const int grid = kp.ntiles < g_sms ? kp.ntiles : g_sms;
  launch_pdl(gemm3xtf32_kernel<BN, AMN, BMN, BS, EPI>, dim3(grid), dim3(kThreads), C::SMEM_BYTES, stream, maps[0],
             maps[1], maps[2], maps[3], maps[4], kp);
  PUSH_CUDA_TRY(cudaGetLastError());
  return PUSH_OK;
}

// Instantiated layouts: every (A, B) layout for the plain-store epilogue (debug GEMM entry, split-K
// weight gradients), the product's layouts for the fused ones (forward: K-major A and B; backward:
// K-major A, MN-major B).
template <int BN>
push_status launch_bn(bool amn, bool bmn, bool bs, int epi, const CUtensorMap* maps, const KParams& kp,
                      cudaStream_t s) {
  if (epi == EPI_FWD && !amn && !bmn)
    return bs ? launch_t<BN, false, false, true, EPI_FWD>(maps, kp, s)
              : launch_t<BN, false, false, false, EPI_FWD>(maps, kp, s);
  if (epi == EPI_BWD && !amn && bmn)
    return bs ? launch_t<BN, false, true, true, EPI_BWD>(maps, kp, s)
              : launch_t<BN, false, true, false, EPI_BWD>(maps, kp, s);
  if (epi == EPI_UPD && !amn && bmn && bs) return launch_t<BN, false, true, true, EPI_UPD>(maps, kp, s);
  if (epi != EPI_STORE) return fail(PUSH_E_INVALID, "gemm: fused epilogue with an unsupported operand layout");
  const int key = (amn ? 4 : 0) | (bmn ? 2 : 0) | (bs ? 1 : 0);
  switch (key) {
    case 0: return launch_t<BN, false, false, false, EPI_STORE>(maps, kp, s);
    case 1: return launch_t<BN, false, false, true, EPI_STORE>(maps, kp, s);
    case 2: return launch_t<BN, false, true, false, EPI_STORE>(maps, kp, s);
    case 3: return launch_t<BN, false, true, true, EPI_STORE>(maps, kp, s);
    case 4: return launch_t<BN, true, false, false, EPI_STORE>(maps, kp, s);
    case 5: return launch_t<BN, true, false, true, EPI_STORE>(maps, kp, s);
    case 6: return launch_t<BN, true, true, false, EPI_STORE>(maps, kp, s);
    default: return launch_t<BN, true, true, true, EPI_STORE>(maps, kp, s);
  }
}

template <int PBN, bool AMN, bool BMN, bool BS, int EPI>
push_status launch2_t(const CUtensorMap* maps, const KParams& kp, cudaStream_t stream) {
  static int max_pairs = 0;
  auto kern = gemm3xtf32_2sm_kernel<PBN, AMN, BMN, BS, EPI>;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (common.cuh)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.blockDim = dim3(k2Threads);
  cfg.dynamicSmemBytes = Cfg2<PBN, EpiBoxes<EPI>::NB>::SMEM_BYTES;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;  // the occupancy query sees the cluster shape only
  if (!max_pairs) {
    PUSH_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg2<PBN, EpiBoxes<EPI>::NB>::SMEM_BYTES));
    cfg.gridDim = dim3(g_sms);
    int n = 0;
    PUSH_CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
    max_pairs = n > 0 ? n : g_sms / 2;
  }
  const int pairs = kp.ntiles < max_pairs ? kp.ntiles : max_pairs;
  cfg.gridDim = dim3(2 * pairs);
  cfg.numAttrs = 2;
  PUSH_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], maps[4], kp));
  return PUSH_OK;
}

template <int PBN>
push_status launch2(bool amn, bool bmn, bool bs, int epi, const CUtensorMap* maps, const KParams& kp,
                    cudaStream_t s) {
  if (epi == EPI_FWD && !amn && !bmn)
    return bs ? launch2_t<PBN, false, false, true, EPI_FWD>(maps, kp, s)
              : launch2_t<PBN, false, false, false, EPI_FWD>(maps, kp, s);
  if (epi == EPI_BWD && !amn && bmn)
    return bs ? launch2_t<PBN, false, true, true, EPI_BWD>(maps, kp, s)
              : launch2_t<PBN, false, true, false, EPI_BWD>(maps, kp, s);
  if (epi != EPI_STORE) return fail(PUSH_E_INVALID, "gemm: fused epilogue with an unsupported operand layout");
  const int key = (amn ? 4 : 0) | (bmn ? 2 : 0) | (bs ? 1 : 0);
  switch (key) {
    case 0: return launch2_t<PBN, false, false, false, EPI_STORE>(maps, kp, s);
    case 1: return launch2_t<PBN, false, false, true, EPI_STORE>(maps, kp, s);
    case 2: return launch2_t<PBN, false, true, false, EPI_STORE>(maps, kp, s);
    case 3: return launch2_t<PBN, false, true, true, EPI_STORE>(maps, kp, s);
    case 4: return launch2_t<PBN, true, false, false, EPI_STORE>(maps, kp, s);
    case 5: return launch2_t<PBN, true, false, true, EPI_STORE>(maps, kp, s);
    case 6: return launch2_t<PBN, true, true, false, EPI_STORE>(maps, kp, s);
    default: return launch2_t<PBN, true, true, true, EPI_STORE>(maps, kp, s);
  }
}

}  // namespace

// Kernel choice (profiles/r01_gemm.md): 256-wide CTA-pair tiles for every GEMM with N % 256 == 0 whose
// K >= kFb256MinK (forward / backward) or with the plain-store epilogue (weight gradients, Gram);
// 128-wide pair tiles (two rotating TMEM accumulators) for the remaining forward / backward GEMMs with
// N % 128 == 0; the 1-CTA kernel for the rest.  The fp32 promotion chunk is fixed at kChunkKB k-blocks
// (longer chunks break the 1e-5 gradient bar).  These are compile-time constants: no environment
// variable reaches the product path.
constexpr int kFb256MinK = 256;

int choose_bn(int N) {
  if (N % 128 == 0) return 128;
  if (N % 64 == 0) return 64;
  return 32;
}

push_status run(const Problem& pb, cudaStream_t stream) {
  if (pb.M < 1 || pb.N < 1 || pb.K < 1 || pb.batch < 1) return fail(PUSH_E_SHAPE, "gemm: empty problem");
  if (pb.N % 32) return fail(PUSH_E_SHAPE, "gemm: N must be a multiple of 32");
  if (!pb.A.split) return fail(PUSH_E_INVALID, "gemm: A must be a plain fp32 operand (split in-kernel)");
  if (pb.A.mn_major && pb.M % 32) return fail(PUSH_E_SHAPE, "gemm: MN-major A needs M % 32 == 0");
  if ((pb.A.ld % 4) || (pb.B.ld % 4) || (pb.A.pstride % 4) || (pb.B.pstride % 4) || (pb.ldo % 4) ||
      (pb.out_pstride % 4))
    return fail(PUSH_E_SHAPE, "gemm: strides must be multiples of 4 elements");
  if ((pb.epi == EPI_BWD || pb.epi == EPI_UPD) && (!pb.aprev || (pb.ld_aprev % 4) || (pb.aprev_pstride % 4)))
    return fail(PUSH_E_SHAPE, "gemm: BWD / UPD need aprev with strides % 4 == 0");
  if (pb.epi == EPI_UPD && (!pb.srow || !pb.hptr || pb.batch != 1))
    return fail(PUSH_E_INVALID, "gemm: UPD needs srow, hptr and one batch");
  if (pb.epi != EPI_STORE && pb.splits != 1) return fail(PUSH_E_INVALID, "gemm: split-K only with EPI_STORE");
  if (pb.splits > 1 && pb.out_sstride != (int64_t)pb.batch * pb.out_pstride)
    return fail(PUSH_E_INVALID, "gemm: split partials must be [s][p] contiguous");
  push_status st;
  if ((st = get_encoder()) != PUSH_OK) return st;
  // CTA-pair kernel with 256-wide pair tiles for the weight-gradient GEMMs (C2 shape: 89 vs 113 us for
  // the 1-CTA kernel) and for forward/backward GEMMs with K >= 512 (C3: 19.5 -> 15.4 ms forward); at
  // K = 256 the 128-wide pair tiles (two rotating TMEM accumulators overlap the fused epilogue with
  // the next tile) are fastest; the 1-CTA kernel covers the remaining (narrow) shapes
  // (profiles/r01_gemm.md).
  const bool dbg_ok = !(pb.passes >> 8 & (1 | 8));
  // M <= 128 (a batch of 128 in the forward / backward GEMMs, C5b): a 256-row pair tile would spend half
  // its MMAs on rows past M, so the 1-CTA kernel (128-row tiles) takes those shapes
  const bool pair_ok = dbg_ok && !pb.no_pair && pb.M > BM && pb.epi != EPI_UPD;
  const bool pair256 = pair_ok && pb.N % 256 == 0 && (pb.epi == EPI_STORE || pb.K >= kFb256MinK);
  const bool pair128 = pair_ok && !pair256 && pb.N % 128 == 0;
  const bool pair = pair256 || pair128;
  const int BN = pair256 ? 256 : (pair128 ? 128 : choose_bn(pb.N));
  const int box_b = pair ? BN / 2 : BN;
  const int nkb = (pb.K + BK - 1) / BK;
  const int kbps = (nkb + pb.splits - 1) / pb.splits;
  if ((nkb + kbps - 1) / kbps != pb.splits) return fail(PUSH_E_SHAPE, "gemm: split count leaves an empty split");
  CUtensorMap maps[5];
  std::memset(maps, 0, sizeof(maps));
  if ((st = make_operand_map(pb.A.hi, pb.A, pb.M, pb.K, pb.batch, BM, &maps[0], true)) != PUSH_OK) return st;
  if ((st = make_operand_map(pb.B.hi, pb.B, pb.N, pb.K, pb.batch, box_b, &maps[1], false)) != PUSH_OK) return st;
  if (!pb.B.split) {
    if (!pb.B.lo) return fail(PUSH_E_INVALID, "gemm: pre-split B needs lo");
    if ((st = make_operand_map(pb.B.lo, pb.B, pb.N, pb.K, pb.batch, box_b, &maps[2], false)) != PUSH_OK) return st;
  }
  const int nout = pb.epi == EPI_STORE ? pb.splits * pb.batch : pb.batch;
  if (!pb.out && pb.epi != EPI_BWD) return fail(PUSH_E_INVALID, "gemm: only the BWD epilogue may skip its output");
  if (pb.out && (st = make_map(&maps[3], pb.out, pb.N, pb.M, nout, pb.ldo, pb.out_pstride, 32,
                               CU_TENSOR_MAP_SWIZZLE_64B, 16)) != PUSH_OK)
    return st;
  if ((pb.epi == EPI_BWD || pb.epi == EPI_UPD) &&
      (st = make_map(&maps[4], pb.aprev, pb.N, pb.M, pb.batch, pb.ld_aprev, pb.aprev_pstride, 32,
                     CU_TENSOR_MAP_SWIZZLE_64B, 16)) != PUSH_OK)
    return st;
  KParams kp;
  std::memset(&kp, 0, sizeof(kp));
  kp.M = pb.M; kp.N = pb.N; kp.K = pb.K; kp.batch = pb.batch; kp.splits = pb.splits; kp.kb_per_split = kbps;
  kp.passes = pb.passes & 0xff; kp.epi = pb.epi; kp.act = pb.act;
  kp.store = pb.out != nullptr;
  kp.chunk_kb = kChunkKB;
  kp.dbg = pb.passes >> 8;
  kp.mt = (pb.M + (pair ? 2 * BM : BM) - 1) / (pair ? 2 * BM : BM);
  kp.nt = pb.N / BN;
  kp.ntiles = kp.mt * kp.nt * pb.splits * pb.batch;
  kp.a_pz = pb.A.pstride == 0 ? 0 : 1;
  kp.b_pz = pb.B.pstride == 0 ? 0 : 1;
  kp.bias = pb.bias; kp.bias_pstride = pb.bias_pstride;
  kp.srow = pb.srow; kp.hptr = pb.hptr;
  kp.alpha = pb.alpha;
  kp.bpart = pb.bpart; kp.bp_sstride = pb.bp_sstride; kp.bp_pstride = pb.bp_pstride;
  kp.x = pb.x; kp.din = pb.xpart ? pb.din : 0; kp.xpart = pb.xpart;
  kp.xp_sstride = pb.xp_sstride; kp.xp_pstride = pb.xp_pstride;
  if (pair256) return launch2<256>(pb.A.mn_major, pb.B.mn_major, pb.B.split, pb.epi, maps, kp, stream);
  if (pair128) return launch2<128>(pb.A.mn_major, pb.B.mn_major, pb.B.split, pb.epi, maps, kp, stream);
  if (BN == 128) return launch_bn<128>(pb.A.mn_major, pb.B.mn_major, pb.B.split, pb.epi, maps, kp, stream);
  if (BN == 64) return launch_bn<64>(pb.A.mn_major, pb.B.mn_major, pb.B.split, pb.epi, maps, kp, stream);
  return launch_bn<32>(pb.A.mn_major, pb.B.mn_major, pb.B.split, pb.epi, maps, kp, stream);
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
