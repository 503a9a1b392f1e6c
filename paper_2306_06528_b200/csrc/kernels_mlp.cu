// kernels_mlp.cu — CUDA-core kernels of the per-particle gradient g_i (DESIGN.md a0-a5)
// for the layers that are too thin for the tensor cores (d_in <= 3 input layer,
// d_out = 1 output layer), the loss, and the write of g into G.
//
// g_i = -lambda * grad MSE_i + grad log p0(theta_i)   (Eq. eq:grad)
// Activations and deltas are plain fp32 arrays [particle][row][feature].  All
// reductions run in a fixed order that depends only on (B, layer shape), never on
// the number of ranks, so results are identical for every sharding.
#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace push {
namespace kern {

// ---------------------------------------------------------------- split (weights)
__global__ void split_hilo_kernel(const float* __restrict__ src, int64_t src_pstride, float* __restrict__ hi,
                                  float* __restrict__ lo, int64_t dst_pstride, int64_t count) {
  PUSH_PDL_ENTRY();
  const int p = blockIdx.y;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const float v = src[p * src_pstride + t];
    const float h = ptx::tf32_rna(v);
    hi[p * dst_pstride + t] = h;
    lo[p * dst_pstride + t] = v - h;
  }
}
void split_hilo(const float* src, int64_t src_pstride, float* hi, float* lo, int64_t dst_pstride, int64_t count,
                int batch, cudaStream_t s) {
  const int blocks = (int)std::min<int64_t>((count + 255) / 256, 4096);
  launch_pdl(split_hilo_kernel, dim3(dim3(blocks, batch)), dim3(256), 0, s, src, src_pstride, hi, lo, dst_pstride, count);
}

// ---------------------------------------------------------------- thin forward (narrow input)
// Narrow input (in <= kThinIn): thread = 4 consecutive output features (float4 store), W and b of
// those features held in registers, looping over the rows of a 32-row block (x[b][:] is a broadcast
// load; the stores of row b are coalesced).  Requires out % 4 == 0 (else VEC = 1: one feature).
constexpr int kThinIn = 8;
template <int NIN, int VEC>
__global__ void __launch_bounds__(256) thin_forward_narrow_kernel(const float* __restrict__ in, int64_t in_pstride,
                                                                  const float* __restrict__ theta, int64_t ld,
                                                                  int64_t off_w, int64_t off_b, int nin, int nout,
                                                                  int act, float* __restrict__ out,
                                                                  int64_t out_pstride, int B) {
  PUSH_PDL_ENTRY();
  constexpr int NI = NIN > 0 ? NIN : kThinIn;
  const int p = blockIdx.y;
  const int b0 = blockIdx.x * 32, b1 = min(B, b0 + 32);
  const float* x = in + p * in_pstride;
  const float* W = theta + p * ld + off_w;
  const float* bias = theta + p * ld + off_b;
  float* o_ = out + p * out_pstride;
  __shared__ float sx[32][NI];  // the block's x rows, loaded once (broadcast reads below)
  for (int c = threadIdx.x; c < 32 * NI; c += blockDim.x) {
    const int r = c / NI, i = c - r * NI;
    sx[r][i] = (b0 + r < b1 && i < nin) ? __ldg(x + (int64_t)(b0 + r) * nin + i) : 0.f;
  }
  __syncthreads();
  for (int o = threadIdx.x * VEC; o < nout; o += blockDim.x * VEC) {
    float w[VEC][NI], bo[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
#pragma unroll
      for (int i = 0; i < NI; ++i) w[v][i] = (NIN > 0 || i < nin) ? __ldg(W + (int64_t)(o + v) * nin + i) : 0.f;
      bo[v] = __ldg(bias + o + v);
    }
#pragma unroll 4
    for (int b = b0; b < b1; ++b) {
      float xv[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) xv[i] = sx[b - b0][i];
      float z[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < NI; ++i)
          if (NIN > 0 || i < nin) acc = fmaf(xv[i], w[v][i], acc);
        z[v] = act_fwd(acc + bo[v], act);
      }
      if constexpr (VEC == 4)
        *reinterpret_cast<float4*>(o_ + (int64_t)b * nout + o) = make_float4(z[0], z[1], z[2], z[3]);
      else
        o_[(int64_t)b * nout + o] = z[0];
    }
  }
}
// Generic thin layer (wide input): one thread per output element.
__global__ void thin_forward_kernel(const float* __restrict__ in, int64_t in_pstride, const float* __restrict__ theta,
                                    int64_t ld, int64_t off_w, int64_t off_b, int nin, int nout, int act,
                                    float* __restrict__ out, int64_t out_pstride, int B) {
  PUSH_PDL_ENTRY();
  const int p = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;  // B * nout < 2^31 (max_batch * width)
  if (t >= B * nout) return;
  const int b = t / nout, o = t - b * nout;
  const float* W = theta + p * ld + off_w + (int64_t)o * nin;
  const float* x = in + p * in_pstride + (int64_t)b * nin;
  float z = 0.f;
  for (int i = 0; i < nin; ++i) z = fmaf(__ldg(x + i), __ldg(W + i), z);
  out[p * out_pstride + t] = act_fwd(z + __ldg(theta + p * ld + off_b + o), act);
}
void thin_forward(const float* in, int64_t in_pstride, const float* theta, int64_t ld_theta, int64_t off_w,
                  int64_t off_b, int in_, int out, int act, float* dst, int64_t out_pstride, int B, int batch,
                  cudaStream_t s) {
  if (in_ <= kThinIn) {
    const dim3 grid((unsigned)((B + 31) / 32), batch);
    const bool v4 = out % 4 == 0 && out_pstride % 4 == 0;
    const int per = v4 ? 4 : 1;
    const int want = (out / per + 31) / 32 * 32;
    const int threads = want > 256 ? 256 : (want < 32 ? 32 : want);
#define PUSH_THIN_FWD(N, V)                                                                                     \
  launch_pdl(thin_forward_narrow_kernel<N, V>, dim3(grid), dim3(threads), 0, s, in, in_pstride, theta, ld_theta, off_w, off_b, in_, \
                                                            out, act, dst, out_pstride, B)
    if (v4) {
      if (in_ == 1) PUSH_THIN_FWD(1, 4);
      else if (in_ == 2) PUSH_THIN_FWD(2, 4);
      else if (in_ == 3) PUSH_THIN_FWD(3, 4);
      else PUSH_THIN_FWD(0, 4);
    } else {
      if (in_ == 1) PUSH_THIN_FWD(1, 1);
      else if (in_ == 2) PUSH_THIN_FWD(2, 1);
      else if (in_ == 3) PUSH_THIN_FWD(3, 1);
      else PUSH_THIN_FWD(0, 1);
    }
#undef PUSH_THIN_FWD
    return;
  }
  const int64_t tot = (int64_t)B * out;
  launch_pdl(thin_forward_kernel, dim3(dim3((unsigned)((tot + 255) / 256), batch)), dim3(256), 0, s, in, in_pstride, theta, ld_theta, off_w,
                                                                                 off_b, in_, out, act, dst,
                                                                                 out_pstride, B);
}

// ---------------------------------------------------------------- fused output layer (a3 + a4/a5 of the top)
// One 256-thread block per 32-row block rb of particle p:
//   phase 1 (warp w, rows 4w..4w+3): yhat_o = a_b . W_o + b_o (lanes split the features; fixed xor
//            tree), e = yhat - y, err2[b] = sum_o e^2, dL_o(b) = 2 e_o / (B d_out)   -> smem
//   phase 2 (thread t owns features i = t, t+256, ...; rows in ascending order):
//        wpart[rb][p][o][i]   = sum_b dL_o(b) a_b[i]                  (dW of the output layer)
//        dprev[b][i]          = (sum_o dL_o(b) W_o[i]) sigma'(a_b[i])  (delta of the layer below)
//        bprev[rb][p][i]      = sum_b dprev[b][i]                     (its bias-gradient partial)
//   and bpart[rb][p][o] = sum_b dL_o(b).
// SMEM: the block's 32 x H slab of A is staged once in shared memory (float4 loads), so phases 1
// and 2 read it on chip and A crosses HBM once (H <= kOutSmemH, H % 4 == 0); same arithmetic order.
constexpr int kOutSmemH = 1024;
template <int DOUT, bool SMEM>  // compile-time bound on d_out (loops below run to DOUT, masked by a.dout)
__global__ void __launch_bounds__(256) output_fused_kernel(const OutputArgs a) {
  PUSH_PDL_ENTRY();
  __shared__ float sdl[32][DOUT];
  __shared__ float serr[32][DOUT];
  extern __shared__ __align__(16) float sA[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.y;
  const int rb = blockIdx.x;
  const int rows = min(32, a.B - rb * 32);
  const float* __restrict__ Ag = a.A + p * a.a_pstride + (int64_t)rb * 32 * a.H;
  for (int c = threadIdx.x; c < 32 * DOUT; c += 256) (&sdl[0][0])[c] = 0.f;  // o >= dout stays 0 (times w = 0)
  if constexpr (!SMEM) __syncthreads();
  if constexpr (SMEM) {
    const int n4 = rows * a.H / 4;
    const float4* src = reinterpret_cast<const float4*>(Ag);
    float4* dst = reinterpret_cast<float4*>(sA);
#pragma unroll 4
    for (int k = threadIdx.x; k < n4; k += 256) dst[k] = __ldg(src + k);
    __syncthreads();
  }
  const float* __restrict__ A = SMEM ? sA : Ag;
  const float* __restrict__ W = a.theta + p * a.ld + a.off_w;
  const float* __restrict__ bias = a.theta + p * a.ld + a.off_b;
  const float scale = 2.0f / (float)((int64_t)a.B * a.dout);
  // phase 1: the warp's 4 rows advance together (4 independent chains, loads in flight together);
  // per row the order is lane-strided accumulation then the fixed xor tree
  for (int o = 0; o < a.dout; ++o) {
    const float* wrow = W + (int64_t)o * a.H;
    float part[4] = {0.f, 0.f, 0.f, 0.f};
    const int r0 = warp * 4;
#pragma unroll 2
    for (int i = lane; i < a.H; i += 32) {
      const float w = __ldg(wrow + i);
#pragma unroll
      for (int rr = 0; rr < 4; ++rr)
        if (r0 + rr < rows) part[rr] = fmaf(A[(int64_t)(r0 + rr) * a.H + i], w, part[rr]);
    }
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) part[rr] += __shfl_xor_sync(0xffffffffu, part[rr], m);
      const int r = r0 + rr, b = rb * 32 + r;
      float dl = 0.f;
      if (r < rows) {
        const float e = (part[rr] + __ldg(bias + o)) - __ldg(a.y + (int64_t)b * a.dout + o);
        dl = scale * e;
        if (lane == 0) serr[r][o] = e;
      }
      if (lane == 0) sdl[r][o] = dl;
    }
  }
  __syncwarp();
  if (lane < 4) {
    const int r = warp * 4 + lane;
    if (r < rows) {
      float e2 = 0.f;
      for (int o = 0; o < a.dout; ++o) e2 = fmaf(serr[r][o], serr[r][o], e2);
      a.err2[p * a.err_pstride + rb * 32 + r] = e2;
    }
  }
  __syncthreads();
  if (threadIdx.x < a.dout) {
    float sb = 0.f;
    for (int r = 0; r < 32; ++r) sb += sdl[r][threadIdx.x];
    a.bpart_out[(int64_t)rb * a.bo_sstride + p * a.bo_pstride + threadIdx.x] = sb;
  }
  // phase 2
  float* __restrict__ dprev = a.dprev ? a.dprev + p * a.dp_pstride + (int64_t)rb * 32 * a.H : nullptr;
  for (int i = threadIdx.x; i < a.H; i += 256) {
    float w[DOUT], wacc[DOUT];
#pragma unroll
    for (int o = 0; o < DOUT; ++o) {
      w[o] = o < a.dout ? __ldg(W + (int64_t)o * a.H + i) : 0.f;
      wacc[o] = 0.f;
    }
    float bacc = 0.f;
#pragma unroll 8
    for (int r = 0; r < rows; ++r) {
      const float av = A[(int64_t)r * a.H + i];
      float d = 0.f;
#pragma unroll
      for (int o = 0; o < DOUT; ++o) {
        const float dl = sdl[r][o];
        wacc[o] = fmaf(dl, av, wacc[o]);
        d = fmaf(dl, w[o], d);
      }
      if (dprev) {
        d *= act_deriv_from_a(av, a.act);
        dprev[(int64_t)r * a.H + i] = d;
        bacc += d;
      }
    }
    for (int o = 0; o < a.dout; ++o)
      a.wpart[(int64_t)rb * a.wo_sstride + p * a.wo_pstride + (int64_t)o * a.H + i] = wacc[o];
    if (dprev) a.bpart_prev[(int64_t)rb * a.bp_sstride + p * a.bp_pstride + i] = bacc;
  }
}
// Streaming form of the same block computation (same per-element arithmetic and order, so the same
// bits): the 32-row block is consumed in slabs of R rows staged by cp.async into an NST-deep ring,
// the copy of slab k + NST - 1 overlapping phases 1-2 of slab k, and W_L is staged once.  Thread t
// owns features i = t + 256 m (m < FPT) across all slabs, so the dW / bias partials stay in
// registers.  Keeps up to NST * R * H * 4 bytes of A in flight per CTA instead of loading the whole
// slab before any math (the one-shot kernel above stalled on long-scoreboard with one CTA per SM).
constexpr int kOutStreamSlabBytes = 32 * 1024;
// Phase 1 of NR consecutive slab rows (block rows r_base + lr0 ..): yhat_o = a_r . W_o + b_o with lanes
// splitting the features (ascending per lane, then a fixed xor tree), e = yhat - y, dL = scale e.
template <int DOUT, int NR>
__device__ __forceinline__ void out_phase1(const OutputArgs& a, const float* A, const float* sW, const float* bias,
                                           int H, int lr0, int r_base, int rows, int rb, int lane, float scale,
                                           float (*sdl)[DOUT], float (*serr)[DOUT]) {
  bool ok[NR];
#pragma unroll
  for (int rr = 0; rr < NR; ++rr) ok[rr] = r_base + lr0 + rr < rows;
  const float* a0 = A + lr0 * H;
  for (int o = 0; o < a.dout; ++o) {
    const float* wrow = sW + o * H;
    float part[NR];
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) part[rr] = 0.f;
#pragma unroll 4
    for (int i = lane; i < H; i += 32) {
      const float w = wrow[i];
#pragma unroll
      for (int rr = 0; rr < NR; ++rr)
        if (ok[rr]) part[rr] = fmaf(a0[rr * H + i], w, part[rr]);
    }
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) part[rr] += __shfl_xor_sync(0xffffffffu, part[rr], m);
      const int r = r_base + lr0 + rr, b = rb * 32 + r;
      float dl = 0.f;
      if (r < rows) {
        const float e = (part[rr] + __ldg(bias + o)) - __ldg(a.y + (int64_t)b * a.dout + o);
        dl = scale * e;
        if (lane == 0) serr[r][o] = e;
      }
      if (lane == 0 && r < 32) sdl[r][o] = dl;
    }
  }
}
// Phase 2 of one feature column over nr slab rows: ACT < 0 = no delta below (L = 1); 32-bit offsets.
template <int DOUT, int ACT>
__device__ __forceinline__ void out_phase2(const float* ai, int H, int nr, const float (*sd)[DOUT], const float (&wv)[DOUT],
                                           float (&wacc)[DOUT], float& bacc, float* dpb) {
  int off = 0;
#pragma unroll 8
  for (int r = 0; r < nr; ++r, off += H) {
    const float av = ai[off];
    float d = 0.f;
#pragma unroll
    for (int o = 0; o < DOUT; ++o) {
      const float dl = sd[r][o];
      wacc[o] = fmaf(dl, av, wacc[o]);
      d = fmaf(dl, wv[o], d);
    }
    if constexpr (ACT >= 0) {
      d *= act_deriv_from_a(av, ACT);
      dpb[off] = d;
      bacc += d;
    }
  }
}
template <int DOUT, int FPT>
__global__ void __launch_bounds__(256) output_stream_kernel(const OutputArgs a, int R, int NST) {
  PUSH_PDL_ENTRY();
  __shared__ float sdl[32][DOUT];
  __shared__ float serr[32][DOUT];
  extern __shared__ __align__(16) float sm[];  // [DOUT][H] W_L, then NST slabs of [R][H]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int p = blockIdx.y, rb = blockIdx.x, H = a.H;
  const int rows = min(32, a.B - rb * 32);
  const int nslab = (rows + R - 1) / R;
  float* sW = sm;
  float* sA = sm + DOUT * H;
  const float* __restrict__ Ag = a.A + p * a.a_pstride + (int64_t)rb * 32 * H;
  const float* __restrict__ Wg = a.theta + p * a.ld + a.off_w;
  const float* __restrict__ bias = a.theta + p * a.ld + a.off_b;
  const uint32_t sA_u = static_cast<uint32_t>(__cvta_generic_to_shared(sA));
  auto issue = [&](int k) {  // slab k -> ring slot k % NST (rows past `rows` are not loaded)
    if (k < nslab) {
      const int r0 = k * R, nr = min(R, rows - r0);
      const int n4 = nr * H / 4;
      const float4* src = reinterpret_cast<const float4*>(Ag + (int64_t)r0 * H);
      const uint32_t dst = sA_u + (uint32_t)((k % NST) * R * H) * 4u;
      for (int c = tid; c < n4; c += 256)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * c), "l"(src + c) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int k = 0; k < NST - 1; ++k) issue(k);
  for (int c = tid; c < a.dout * H; c += 256) sW[c] = __ldg(Wg + c);
  for (int c = tid; c < 32 * DOUT; c += 256) (&sdl[0][0])[c] = 0.f;  // o >= dout stays 0 (times w = 0)
  const float scale = 2.0f / (float)((int64_t)a.B * a.dout);
  float wacc[FPT][DOUT], bacc[FPT], wv[FPT][DOUT];
  float* __restrict__ dprev = a.dprev ? a.dprev + p * a.dp_pstride + (int64_t)rb * 32 * H : nullptr;
#pragma unroll
  for (int m = 0; m < FPT; ++m) {
    bacc[m] = 0.f;
#pragma unroll
    for (int o = 0; o < DOUT; ++o) wacc[m][o] = 0.f;
  }
  // phase-1 rows of this warp within a slab: RPW consecutive rows (R >= 8), or one row (R = 4)
  const int RPW = R >= 8 ? R / 8 : 1;
  for (int k = 0; k < nslab; ++k) {
    issue(k + NST - 1);  // one group per iteration (possibly empty): slab k has NST - 1 newer groups
    if (NST == 3) asm volatile("cp.async.wait_group 2;" ::: "memory");
    else if (NST == 2) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (k == 0) {
#pragma unroll
      for (int m = 0; m < FPT; ++m) {
        const int i = tid + 256 * m;
#pragma unroll
        for (int o = 0; o < DOUT; ++o) wv[m][o] = (i < H && o < a.dout) ? sW[o * H + i] : 0.f;
      }
    }
    const float* A = sA + (k % NST) * R * H;  // row r of the block at A[(r - k R) H]
    const int r_base = k * R;
    // phase 1: yhat, residual, dL for the slab's rows (per row: lane-strided sum, fixed xor tree);
    // the rows per warp are a compile-time count (a runtime-masked 4-row loop quadrupled the work at RPW 1)
    if (warp * RPW < R) {
      if (RPW == 4)
        out_phase1<DOUT, 4>(a, A, sW, bias, H, warp * 4, r_base, rows, rb, lane, scale, sdl, serr);
      else if (RPW == 2)
        out_phase1<DOUT, 2>(a, A, sW, bias, H, warp * 2, r_base, rows, rb, lane, scale, sdl, serr);
      else
        out_phase1<DOUT, 1>(a, A, sW, bias, H, warp, r_base, rows, rb, lane, scale, sdl, serr);
    }
    __syncthreads();
    // phase 2 over the slab's rows, ascending (activation and delta store resolved at compile time)
    const int nr = min(r_base + R, rows) - r_base;
    const int mode = dprev ? 1 + a.act : 0;
#pragma unroll
    for (int m = 0; m < FPT; ++m) {
      const int i = tid + 256 * m;
      if (i < H) {
        float* dpb = dprev ? dprev + (int64_t)r_base * H + i : nullptr;
        const float(*sd)[DOUT] = sdl + r_base;
        switch (mode) {
          case 0: out_phase2<DOUT, -1>(A + i, H, nr, sd, wv[m], wacc[m], bacc[m], dpb); break;
          case 1 + PUSH_ACT_TANH: out_phase2<DOUT, PUSH_ACT_TANH>(A + i, H, nr, sd, wv[m], wacc[m], bacc[m], dpb); break;
          case 1 + PUSH_ACT_RELU: out_phase2<DOUT, PUSH_ACT_RELU>(A + i, H, nr, sd, wv[m], wacc[m], bacc[m], dpb); break;
          default: out_phase2<DOUT, PUSH_ACT_IDENTITY>(A + i, H, nr, sd, wv[m], wacc[m], bacc[m], dpb); break;
        }
      }
    }
    __syncthreads();  // slot k % NST is refilled by the next iteration's issue
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  // rows past `rows` contribute dL = 0 to the output-bias partial (as in the one-shot kernel)
  for (int r = rows + tid; r < 32; r += 256)
    for (int o = 0; o < a.dout; ++o) sdl[r][o] = 0.f;
  if (lane < 4 && warp * 4 + lane < rows) {
    const int r = warp * 4 + lane;
    float e2 = 0.f;
    for (int o = 0; o < a.dout; ++o) e2 = fmaf(serr[r][o], serr[r][o], e2);
    a.err2[p * a.err_pstride + rb * 32 + r] = e2;
  }
  __syncthreads();
  if (tid < a.dout) {
    float sb = 0.f;
    for (int r = 0; r < 32; ++r) sb += sdl[r][tid];
    a.bpart_out[(int64_t)rb * a.bo_sstride + p * a.bo_pstride + tid] = sb;
  }
#pragma unroll
  for (int m = 0; m < FPT; ++m) {
    const int i = tid + 256 * m;
    if (i < H) {
      for (int o = 0; o < a.dout; ++o)
        a.wpart[(int64_t)rb * a.wo_sstride + p * a.wo_pstride + (int64_t)o * H + i] = wacc[m][o];
      if (dprev) a.bpart_prev[(int64_t)rb * a.bp_sstride + p * a.bp_pstride + i] = bacc[m];
    }
  }
}
template <int DOUT, int FPT>
static void output_stream_launch(const OutputArgs& a, int batch, cudaStream_t s) {
  int R = 32;
  while (R > 4 && (int64_t)R * a.H * 4 > kOutStreamSlabBytes) R >>= 1;
  const int nslab = (std::min(32, a.B) + R - 1) / R;
  const int NST = nslab >= 3 ? 3 : (nslab == 2 ? 2 : 1);
  const size_t smem = sizeof(float) * ((size_t)DOUT * a.H + (size_t)NST * R * a.H);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(output_stream_kernel<DOUT, FPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  launch_pdl(output_stream_kernel<DOUT, FPT>, dim3(dim3((a.B + 31) / 32, batch)), dim3(256), smem, s, a, R, NST);
}
template <int DOUT>
static void output_launch(const OutputArgs& a, int batch, cudaStream_t s) {
  const bool stream_ok = a.H % 4 == 0 && a.a_pstride % 4 == 0 && (reinterpret_cast<uintptr_t>(a.A) & 15) == 0 &&
                         a.H <= 2048 && DOUT * ((a.H + 255) / 256) <= 16;
  if (stream_ok) {
    const int fpt = (a.H + 255) / 256;
    if (fpt == 1) return output_stream_launch<DOUT, 1>(a, batch, s);
    if (fpt == 2) return output_stream_launch<DOUT, 2>(a, batch, s);
    if (fpt <= 4) return output_stream_launch<DOUT, 4>(a, batch, s);
    if constexpr (DOUT <= 2) return output_stream_launch<DOUT, 8>(a, batch, s);
  }
  const dim3 grid((a.B + 31) / 32, batch);
  const bool smem = a.H <= kOutSmemH && a.H % 4 == 0 && a.a_pstride % 4 == 0 &&
                    (reinterpret_cast<uintptr_t>(a.A) & 15) == 0;
  if (smem) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(output_fused_kernel<DOUT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           32 * kOutSmemH * 4);
      attr = true;
    }
    launch_pdl(output_fused_kernel<DOUT, true>, dim3(grid), dim3(256), (size_t)32 * a.H * 4, s, a);
  } else {
    launch_pdl(output_fused_kernel<DOUT, false>, dim3(grid), dim3(256), 0, s, a);
  }
}
void output_fused(const OutputArgs& a, int batch, cudaStream_t s) {
  if (a.dout == 1) output_launch<1>(a, batch, s);
  else if (a.dout == 2) output_launch<2>(a, batch, s);
  else if (a.dout <= 4) output_launch<4>(a, batch, s);
  else output_launch<kMaxDout>(a, batch, s);
}

// ---------------------------------------------------------------- predictive pushforward (NEXT-1)
// warp per (particle, row): lanes split the features, fixed xor tree (same order as output_fused)
__global__ void output_forward_kernel(const float* __restrict__ A, int64_t a_pstride, const float* __restrict__ theta,
                                      int64_t ld, int64_t off_w, int64_t off_b, int H, int dout,
                                      float* __restrict__ pred, int B) {
  PUSH_PDL_ENTRY();
  const int p = blockIdx.y, lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const float* arow = A + p * a_pstride + (int64_t)b * H;
  for (int o = 0; o < dout; ++o) {
    const float* wrow = theta + p * ld + off_w + (int64_t)o * H;
    float part = 0.f;
    for (int i = lane; i < H; i += 32) part = fmaf(__ldg(arow + i), __ldg(wrow + i), part);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) part += __shfl_xor_sync(0xffffffffu, part, m);
    if (lane == 0) pred[((int64_t)p * B + b) * dout + o] = part + __ldg(theta + p * ld + off_b + o);
  }
}
void output_forward(const float* A, int64_t a_pstride, const float* theta, int64_t ld, int64_t off_w, int64_t off_b,
                    int H, int dout, float* pred, int B, int batch, cudaStream_t s) {
  launch_pdl(output_forward_kernel, dim3(dim3((B + 7) / 8, batch)), dim3(256), 0, s, A, a_pstride, theta, ld, off_w, off_b, H, dout, pred, B);
}
__global__ void predict_stats_kernel(const float* __restrict__ pred, int n, int64_t m, float* __restrict__ mean,
                                     float* __restrict__ stdev) {
  PUSH_PDL_ENTRY();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= m) return;
  float s1 = 0.f;
  for (int p = 0; p < n; ++p) s1 += pred[(int64_t)p * m + t];
  const float mu = s1 / (float)n;
  float s2 = 0.f;
  for (int p = 0; p < n; ++p) {
    const float dv = pred[(int64_t)p * m + t] - mu;
    s2 = fmaf(dv, dv, s2);
  }
  if (mean) mean[t] = mu;
  if (stdev) stdev[t] = sqrtf(s2 / (float)n);
}
void predict_stats(const float* pred, int n, int64_t m, float* mean, float* stdev, cudaStream_t s) {
  launch_pdl(predict_stats_kernel, dim3((unsigned)((m + 255) / 256)), dim3(256), 0, s, pred, n, m, mean, stdev);
}

__global__ void loss_reduce_kernel(const float* __restrict__ err2, int64_t err_pstride, float* __restrict__ loss,
                                   int B, float denom) {
  PUSH_PDL_ENTRY();
  __shared__ float sh[256];
  const int p = blockIdx.x;
  float acc = 0.f;
  for (int b = threadIdx.x; b < B; b += 256) acc += err2[p * err_pstride + b];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w >= 1; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss[p] = sh[0] / denom;
}
void loss_reduce(const float* err2, int64_t err_pstride, float* loss, int B, int d_out, int batch, cudaStream_t s) {
  launch_pdl(loss_reduce_kernel, dim3(batch), dim3(256), 0, s, err2, err_pstride, loss, B, (float)((int64_t)B * d_out));
}

// ---------------------------------------------------------------- thin backward (generic)
__global__ void thin_backward_kernel(const float* __restrict__ dl, int64_t d_pstride, const float* __restrict__ theta,
                                     int64_t ld, int64_t off_w, int nin, int nout, const float* __restrict__ aprev,
                                     int64_t a_pstride, int act, float* __restrict__ o, int64_t o_pstride, int B) {
  PUSH_PDL_ENTRY();
  const int p = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B * nin) return;
  const int b = t / nin, i = t - b * nin;
  const float* W = theta + p * ld + off_w;
  const float* drow = dl + p * d_pstride + (int64_t)b * nout;
  float acc = 0.f;
  for (int k = 0; k < nout; ++k) acc = fmaf(__ldg(drow + k), __ldg(W + (int64_t)k * nin + i), acc);
  o[p * o_pstride + t] = acc * act_deriv_from_a(aprev[p * a_pstride + t], act);
}
void thin_backward(const float* dl, int64_t d_pstride, const float* theta, int64_t ld_theta, int64_t off_w, int in,
                   int out, const float* aprev, int64_t a_pstride, int act, float* o, int64_t o_pstride, int B,
                   int batch, cudaStream_t s) {
  const int64_t tot = (int64_t)B * in;
  launch_pdl(thin_backward_kernel, dim3(dim3((unsigned)((tot + 255) / 256), batch)), dim3(256), 0, s, 
      dl, d_pstride, theta, ld_theta, off_w, in, out, aprev, a_pstride, act, o, o_pstride, B);
}

// ---------------------------------------------------------------- thin weight-gradient partials (generic)
__global__ void thin_wgrad_kernel(const float* __restrict__ dl, int64_t d_pstride, const float* __restrict__ A,
                                  int64_t a_pstride, int nin, int nout, float* __restrict__ part, int B) {
  PUSH_PDL_ENTRY();
  const int p = blockIdx.z, s = blockIdx.y, P = gridDim.z;
  const int cols = nin + 1;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int tot = nout * cols;
  if (t >= tot) return;
  int o, i;
  if (cols >= nout) { o = t / cols; i = t - o * cols; }     // input index fastest: coalesced A
  else { i = t / nout; o = t - i * nout; }                 // output index fastest: coalesced delta
  const int b0 = s * THIN_CHUNK, b1 = min(B, b0 + THIN_CHUNK);
  const float* dcol = dl + p * d_pstride + o;
  float acc = 0.f;
  if (i == nin) {
    for (int b = b0; b < b1; ++b) acc += dcol[(int64_t)b * nout];
  } else {
    const float* acol = A + p * a_pstride + i;
    for (int b = b0; b < b1; ++b) acc = fmaf(dcol[(int64_t)b * nout], acol[(int64_t)b * nin], acc);
  }
  part[((int64_t)s * P + p) * tot + (int64_t)o * cols + i] = acc;
}
int thin_wgrad(const float* dl, int64_t d_pstride, const float* A, int64_t a_pstride, int in_eff, int out, float* part,
               int B, int batch, cudaStream_t s) {
  const int chunks = (B + THIN_CHUNK - 1) / THIN_CHUNK;
  const int64_t tot = (int64_t)out * (in_eff + 1);
  launch_pdl(thin_wgrad_kernel, dim3(dim3((unsigned)((tot + 255) / 256), chunks, batch)), dim3(256), 0, s, dl, d_pstride, A, a_pstride,
                                                                                       in_eff, out, part, B);
  return chunks;
}

// ---------------------------------------------------------------- finalize G rows of one layer
// G_p[off_w + t] = -lambda * sum_s part(s, p, t) + grad log p0(theta_p[off_w + t]) for t in [t0, t1)
// (t < in*out: weight (o, i) = (t / in, t % in) from W; else bias o = t - in*out from Bv).
// Few partials (<= kThreadSplits): one thread per element, ascending s.  Many partials over few
// elements: a CTA per 32 consecutive elements, warp w sums s = w, w+8, ... ascending (coalesced
// loads, 8 in flight), then the 8 warp sums in ascending w.  Either order depends only on the
// partial count, never on the sharding.
constexpr int kThreadSplits = 16;
__device__ __forceinline__ const float* part_ptr(const PartView& W, const PartView& Bv, int p, int64_t t, int nin,
                                                 int64_t nw, int* splits, int64_t* sstride) {
  if (t < nw) {
    *splits = W.splits;
    *sstride = W.sstride;
    const int o = (int)t / nin;  // t < in*out < 2^31
    return W.base + p * W.pstride + (int64_t)o * W.ostride + ((int)t - o * nin);
  }
  *splits = Bv.splits;
  *sstride = Bv.sstride;
  return Bv.base + p * Bv.pstride + (t - nw) * Bv.ostride;
}
__device__ __forceinline__ void finalize_store(const float* theta, float* grad, int64_t idx, float v, float lambda,
                                               int prior, float inv_sigma2) {
  const float pr = (prior == PUSH_PRIOR_GAUSSIAN) ? -theta[idx] * inv_sigma2 : 0.f;
  grad[idx] = fmaf(-lambda, v, pr);
}
// Sum of `splits` partials at stride ss in a fixed order that depends only on `splits`: ascending for
// splits <= 8, else 8 interleaved ascending chains (s = u mod 8) combined by a fixed tree (loads in flight).
template <typename V>
__device__ __forceinline__ V vadd(V a, V b);
template <>
__device__ __forceinline__ float vadd(float a, float b) { return a + b; }
template <>
__device__ __forceinline__ float4 vadd(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
template <typename V, bool MANY = true>  // MANY = false: splits <= 8 guaranteed (float4 path: registers)
__device__ __forceinline__ V sum_partials(const V* src, int splits, int64_t ss_v) {
  V zero;
  memset(&zero, 0, sizeof(V));
  if (!MANY || splits <= 8) {  // ascending; four loads issued before their adds (few registers: occupancy)
    V v = zero;
    for (int s0 = 0; s0 < splits; s0 += 4) {
      V t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] = s0 + u < splits ? __ldg(src + (s0 + u) * ss_v) : zero;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (s0 + u < splits) v = vadd(v, t[u]);
    }
    return v;
  }
  V a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = zero;
  int s = 0;
  for (; s + 8 <= splits; s += 8)
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = vadd(a[u], __ldg(src + (s + u) * ss_v));
  for (int u = 0; s + u < splits; ++u) a[u] = vadd(a[u], __ldg(src + (s + u) * ss_v));
  return vadd(vadd(vadd(a[0], a[1]), vadd(a[2], a[3])), vadd(vadd(a[4], a[5]), vadd(a[6], a[7])));
}
// mode 0: thread per element, 1: 32 consecutive elements per CTA with the partials split over its 8 warps
// (many partials), 2: thread per 4 consecutive elements (float4), 3: prior added in place
__device__ __forceinline__ void finalize_range(const PartView& W, const PartView& Bv, const float* theta,
                                               float* grad, int64_t ld, int64_t off_w, int nin, int nout,
                                               int64_t t0, int64_t t1, int mode, int64_t blk, float lambda,
                                               int prior, float inv_sigma2, int p) {
  const int64_t nw = (int64_t)nin * nout;
  const int lane = threadIdx.x & 31;
  if (mode == 2) {
    const int64_t t = t0 + 4 * (blk * blockDim.x + threadIdx.x);
    if (t >= t1) return;
    int splits;
    int64_t ss;
    const float* src = part_ptr(W, Bv, p, t, nin, nw, &splits, &ss);
    const float4 v = sum_partials<float4, false>(reinterpret_cast<const float4*>(src), splits, ss / 4);
    const int64_t idx = p * ld + off_w + t;
    float4 pr = make_float4(0.f, 0.f, 0.f, 0.f);
    if (prior == PUSH_PRIOR_GAUSSIAN) {
      const float4 th = *reinterpret_cast<const float4*>(theta + idx);
      pr = make_float4(-th.x * inv_sigma2, -th.y * inv_sigma2, -th.z * inv_sigma2, -th.w * inv_sigma2);
    }
    *reinterpret_cast<float4*>(grad + idx) = make_float4(fmaf(-lambda, v.x, pr.x), fmaf(-lambda, v.y, pr.y),
                                                         fmaf(-lambda, v.z, pr.z), fmaf(-lambda, v.w, pr.w));
    return;
  }
  if (mode == 1) {  // column group: 32 consecutive elements per CTA, warp w sums s = w, w + 8, ... ascending
    __shared__ float red[8][33];
    const int warp = threadIdx.x >> 5;  // blockDim.x == 256
    const int64_t t = t0 + blk * 32 + lane;
    float v = 0.f;
    if (t < t1) {
      int splits;
      int64_t ss;
      const float* src = part_ptr(W, Bv, p, t, nin, nw, &splits, &ss);
      for (int s0 = warp; s0 < splits; s0 += 64) {  // 8 coalesced loads in flight per lane
        float tt[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) tt[k] = s0 + 8 * k < splits ? __ldg(src + (int64_t)(s0 + 8 * k) * ss) : 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (s0 + 8 * k < splits) v += tt[k];
      }
    }
    red[warp][lane] = v;
    __syncthreads();
    if (warp == 0 && t < t1) {
      float r = red[0][lane];
#pragma unroll
      for (int w = 1; w < 8; ++w) r += red[w][lane];
      finalize_store(theta, grad, p * ld + off_w + t, r, lambda, prior, inv_sigma2);
    }
    return;
  }
  const int64_t t = t0 + blk * blockDim.x + threadIdx.x;
  if (t >= t1) return;
  if (mode == 3) {  // G already holds -lambda dW: add grad log p0 (Gaussian prior only; uniform launches none)
    const int64_t idx = p * ld + off_w + t;
    grad[idx] += -theta[idx] * inv_sigma2;
    return;
  }
  int splits;
  int64_t ss;
  const float* src = part_ptr(W, Bv, p, t, nin, nw, &splits, &ss);
  const float v = sum_partials(src, splits, ss);
  finalize_store(theta, grad, p * ld + off_w + t, v, lambda, prior, inv_sigma2);
}
// All layers in one launch: block b of the grid belongs to the job whose [blk0, blk0 + nb_w + nb_b)
// range contains it; within a job, blocks [0, nb_w) reduce the weight partials and the rest the bias
// partials, each part with the thread- or warp-per-element scheme its partial count calls for.
struct FinalizeTable {
  FinalizeJob j[kMaxFinalizeJobs];
  int n;
};
__global__ void finalize_all_kernel(const __grid_constant__ FinalizeTable t, const float* __restrict__ theta,
                                    float* __restrict__ grad,
                                    int64_t ld, float lambda, int prior, float inv_sigma2) {
  PUSH_PDL_ENTRY();
  const int p = blockIdx.y;
  int k = 0;
  while (k + 1 < t.n && (int)blockIdx.x >= t.j[k + 1].blk0) ++k;
  const FinalizeJob& J = t.j[k];
  const int b = blockIdx.x - J.blk0;
  const int64_t nw = (int64_t)J.in * J.out;
  if (b < J.nb_w)
    finalize_range(J.W, J.Bv, theta, grad, ld, J.off_w, J.in, J.out, 0, nw, J.w_warp, b, lambda, prior, inv_sigma2,
                   p);
  else
    finalize_range(J.W, J.Bv, theta, grad, ld, J.off_w, J.in, J.out, nw, nw + J.out, J.b_warp, b - J.nb_w, lambda,
                   prior, inv_sigma2, p);
}
FinalizeJob make_finalize_job(const PartView& W, const PartView& Bv, int64_t off_w, int in, int out) {
  // many partials over few elements: column groups (partials split over the CTA's warps); otherwise
  // thread-per-element reads one contiguous row of elements per partial, float4-wide when aligned
  auto warp_mode = [](int64_t elems, int splits) { return splits > kThreadSplits && elems < 32768; };
  FinalizeJob j{};
  j.W = W;
  j.Bv = Bv;
  j.off_w = off_w;
  j.in = in;
  j.out = out;
  const int64_t nw = (int64_t)in * out;
  const bool v4 = W.splits <= 8 && in % 4 == 0 && off_w % 4 == 0 && W.pstride % 4 == 0 && W.sstride % 4 == 0 &&
                  W.ostride % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(W.base) & 15) == 0;
  j.w_warp = warp_mode(nw, W.splits) ? 1 : (v4 ? 2 : 0);
  j.b_warp = warp_mode(out, Bv.splits) ? 1 : 0;
  auto blocks = [](int64_t elems, int mode) {
    return (int)(mode == 1 ? (elems + 31) / 32 : (mode == 2 ? (elems / 4 + 255) / 256 : (elems + 255) / 256));
  };
  j.nb_w = blocks(nw, j.w_warp);
  j.nb_b = blocks(out, j.b_warp);
  return j;
}
FinalizeJob make_finalize_job_wdirect(const PartView& Bv, int64_t off_w, int in, int out, int prior) {
  FinalizeJob j = make_finalize_job(PartView{nullptr, 0, 0, 0, 0}, Bv, off_w, in, out);
  j.w_warp = 3;
  j.nb_w = prior == PUSH_PRIOR_GAUSSIAN ? (int)(((int64_t)in * out + 255) / 256) : 0;
  return j;
}
void finalize_all(const FinalizeJob* jobs, int njobs, const float* theta, float* grad, int64_t ld, float lambda,
                  int prior, float inv_sigma2, int batch, cudaStream_t s) {
  FinalizeTable t{};
  t.n = njobs;
  int blk = 0;
  for (int k = 0; k < njobs; ++k) {
    t.j[k] = jobs[k];
    t.j[k].blk0 = blk;
    blk += jobs[k].nb_w + jobs[k].nb_b;
  }
  launch_pdl(finalize_all_kernel, dim3(dim3(blk, batch)), dim3(256), 0, s, t, theta, grad, ld, lambda, prior, inv_sigma2);
}

// ---------------------------------------------------------------- set_grads copy
__global__ void copy_rows_kernel(const float* __restrict__ src, int64_t d, float* __restrict__ dst, int64_t ld) {
  PUSH_PDL_ENTRY();
  const int p = blockIdx.y;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < d; t += (int64_t)gridDim.x * blockDim.x)
    dst[p * ld + t] = src[p * d + t];
}
void copy_rows(const float* src, int64_t d, float* dst, int64_t ld, int rows, cudaStream_t s) {
  const int blocks = (int)std::min<int64_t>((d + 255) / 256, 2048);
  launch_pdl(copy_rows_kernel, dim3(dim3(blocks, rows)), dim3(256), 0, s, src, d, dst, ld);
}

}  // namespace kern
}  // namespace push
