// kernels_mlp.cu — CUDA-core kernels of the per-particle gradient g_i (DESIGN.md a0-a5)
// for the layers that are too thin for the tensor cores (d_in <= 3 input layer,
// d_out = 1 output layer), the loss, the bias sums and the write of g into G.
//
// g_i = -lambda * grad MSE_i + grad log p0(theta_i)   (Eq. eq:grad)
// All reductions run in a fixed order that depends only on (B, layer shape),
// never on the number of ranks, so results are identical for every sharding.
#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace push {
namespace kern {

__device__ __forceinline__ void store_hilo(float* hi, float* lo, int64_t idx, float v) {
  const float h = ptx::tf32_rna(v);
  hi[idx] = h;
  lo[idx] = ptx::tf32_rna(v - h);
}
__device__ __forceinline__ float load_val(const float* hi, const float* lo, int64_t idx) {
  return lo ? hi[idx] + lo[idx] : hi[idx];
}

// ---------------------------------------------------------------- split
__global__ void split_hilo_kernel(const float* __restrict__ src, int64_t src_pstride, float* __restrict__ hi,
                                  float* __restrict__ lo, int64_t dst_pstride, int64_t count) {
  const int p = blockIdx.y;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    store_hilo(hi + p * dst_pstride, lo + p * dst_pstride, t, src[p * src_pstride + t]);
}
void split_hilo(const float* src, int64_t src_pstride, float* hi, float* lo, int64_t dst_pstride, int64_t count,
                int batch, cudaStream_t s) {
  const int blocks = (int)std::min<int64_t>((count + 255) / 256, 4096);
  split_hilo_kernel<<<dim3(blocks, batch), 256, 0, s>>>(src, src_pstride, hi, lo, dst_pstride, count);
}

// ---------------------------------------------------------------- thin forward (narrow input)
__global__ void thin_forward_kernel(const float* __restrict__ in_hi, const float* __restrict__ in_lo,
                                    int64_t in_pstride, const float* __restrict__ theta, int64_t ld, int64_t off_w,
                                    int64_t off_b, int nin, int nout, int act, float* __restrict__ out_hi,
                                    float* __restrict__ out_lo, int64_t out_pstride, int B) {
  const int p = blockIdx.y;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * nout) return;
  const int b = (int)(t / nout), o = (int)(t % nout);
  const float* W = theta + p * ld + off_w + (int64_t)o * nin;
  const int64_t ib = p * in_pstride + (int64_t)b * nin;
  float z = 0.f;
  for (int i = 0; i < nin; ++i) z = fmaf(load_val(in_hi, in_lo, ib + i), W[i], z);
  z += theta[p * ld + off_b + o];
  store_hilo(out_hi, out_lo, p * out_pstride + t, act_fwd(z, act));
}
void thin_forward(const float* in_hi, const float* in_lo, int64_t in_pstride, const float* theta, int64_t ld_theta,
                  int64_t off_w, int64_t off_b, int in, int out, int act, float* out_hi, float* out_lo,
                  int64_t out_pstride, int B, int batch, cudaStream_t s) {
  const int64_t tot = (int64_t)B * out;
  thin_forward_kernel<<<dim3((unsigned)((tot + 255) / 256), batch), 256, 0, s>>>(
      in_hi, in_lo, in_pstride, theta, ld_theta, off_w, off_b, in, out, act, out_hi, out_lo, out_pstride, B);
}

// ---------------------------------------------------------------- output layer + loss terms
// one warp per (particle, batch row); lanes split the input features; fixed xor-tree reduction.
__global__ void output_layer_kernel(const float* __restrict__ in_hi, const float* __restrict__ in_lo,
                                    int64_t in_pstride, const float* __restrict__ theta, int64_t ld, int64_t off_w,
                                    int64_t off_b, int nin, int nout, const float* __restrict__ y,
                                    float* __restrict__ err2, int64_t err_pstride, float* __restrict__ d_hi,
                                    float* __restrict__ d_lo, int64_t d_pstride, int B) {
  const int p = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const int64_t ib = p * in_pstride + (int64_t)b * nin;
  const float scale = 2.0f / (float)((int64_t)B * nout);
  float e2 = 0.f;
  for (int o = 0; o < nout; ++o) {
    const float* W = theta + p * ld + off_w + (int64_t)o * nin;
    float part = 0.f;
    for (int i = lane; i < nin; i += 32) part = fmaf(load_val(in_hi, in_lo, ib + i), W[i], part);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) part += __shfl_xor_sync(0xffffffffu, part, m);
    const float yhat = part + theta[p * ld + off_b + o];
    const float e = yhat - y[(int64_t)b * nout + o];
    e2 = fmaf(e, e, e2);
    if (lane == 0) store_hilo(d_hi, d_lo, p * d_pstride + (int64_t)b * nout + o, scale * e);
  }
  if (lane == 0) err2[p * err_pstride + b] = e2;
}
void output_layer(const float* in_hi, const float* in_lo, int64_t in_pstride, const float* theta, int64_t ld_theta,
                  int64_t off_w, int64_t off_b, int in, int out, const float* y, float* err2, int64_t err_pstride,
                  float* d_hi, float* d_lo, int64_t d_pstride, int B, int batch, cudaStream_t s) {
  output_layer_kernel<<<dim3((B + 7) / 8, batch), 256, 0, s>>>(in_hi, in_lo, in_pstride, theta, ld_theta, off_w,
                                                                off_b, in, out, y, err2, err_pstride, d_hi, d_lo,
                                                                d_pstride, B);
}

__global__ void loss_reduce_kernel(const float* __restrict__ err2, int64_t err_pstride, float* __restrict__ loss,
                                   int B, float denom) {
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
  loss_reduce_kernel<<<batch, 256, 0, s>>>(err2, err_pstride, loss, B, (float)((int64_t)B * d_out));
}

// ---------------------------------------------------------------- thin backward
__global__ void thin_backward_kernel(const float* __restrict__ d_hi, const float* __restrict__ d_lo,
                                     int64_t d_pstride, const float* __restrict__ theta, int64_t ld, int64_t off_w,
                                     int nin, int nout, const float* __restrict__ a_hi,
                                     const float* __restrict__ a_lo, int64_t a_pstride, int act,
                                     float* __restrict__ o_hi, float* __restrict__ o_lo, int64_t o_pstride, int B) {
  const int p = blockIdx.y;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * nin) return;
  const int b = (int)(t / nin), i = (int)(t % nin);
  const float* W = theta + p * ld + off_w;
  const int64_t db = p * d_pstride + (int64_t)b * nout;
  float acc = 0.f;
  for (int o = 0; o < nout; ++o) acc = fmaf(load_val(d_hi, d_lo, db + o), W[(int64_t)o * nin + i], acc);
  const float a = load_val(a_hi, a_lo, p * a_pstride + t);
  store_hilo(o_hi, o_lo, p * o_pstride + t, acc * act_deriv_from_a(a, act));
}
void thin_backward(const float* d_hi, const float* d_lo, int64_t d_pstride, const float* theta, int64_t ld_theta,
                   int64_t off_w, int in, int out, const float* a_hi, const float* a_lo, int64_t a_pstride, int act,
                   float* o_hi, float* o_lo, int64_t o_pstride, int B, int batch, cudaStream_t s) {
  const int64_t tot = (int64_t)B * in;
  thin_backward_kernel<<<dim3((unsigned)((tot + 255) / 256), batch), 256, 0, s>>>(
      d_hi, d_lo, d_pstride, theta, ld_theta, off_w, in, out, a_hi, a_lo, a_pstride, act, o_hi, o_lo, o_pstride, B);
}

// ---------------------------------------------------------------- thin weight-gradient partials
__global__ void thin_wgrad_kernel(const float* __restrict__ d_hi, const float* __restrict__ d_lo,
                                  int64_t d_pstride, const float* __restrict__ a_hi,
                                  const float* __restrict__ a_lo, int64_t a_pstride, int nin, int nout,
                                  float* __restrict__ part, int B) {
  const int p = blockIdx.z, s = blockIdx.y, P = gridDim.z;
  const int cols = nin + 1;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)nout * cols;
  if (t >= tot) return;
  int o, i;
  if (cols >= nout) { o = (int)(t / cols); i = (int)(t % cols); }     // input index fastest: coalesced A
  else { i = (int)(t / nout); o = (int)(t % nout); }                 // output index fastest: coalesced delta
  const int b0 = s * THIN_CHUNK, b1 = min(B, b0 + THIN_CHUNK);
  const int64_t dbase = p * d_pstride + o, abase = p * a_pstride + i;
  float acc = 0.f;
  if (i == nin) {
    for (int b = b0; b < b1; ++b) acc += load_val(d_hi, d_lo, dbase + (int64_t)b * nout);
  } else {
    for (int b = b0; b < b1; ++b)
      acc = fmaf(load_val(d_hi, d_lo, dbase + (int64_t)b * nout), load_val(a_hi, a_lo, abase + (int64_t)b * nin), acc);
  }
  part[((int64_t)s * P + p) * tot + (int64_t)o * cols + i] = acc;
}
int thin_wgrad(const float* d_hi, const float* d_lo, int64_t d_pstride, const float* a_hi, const float* a_lo,
               int64_t a_pstride, int in_eff, int out, float* part, int B, int batch, cudaStream_t s) {
  const int chunks = (B + THIN_CHUNK - 1) / THIN_CHUNK;
  const int64_t tot = (int64_t)out * (in_eff + 1);
  thin_wgrad_kernel<<<dim3((unsigned)((tot + 255) / 256), chunks, batch), 256, 0, s>>>(
      d_hi, d_lo, d_pstride, a_hi, a_lo, a_pstride, in_eff, out, part, B);
  return chunks;
}

// ---------------------------------------------------------------- finalize G rows of one layer
__global__ void finalize_kernel(PartView W, PartView Bv, const float* __restrict__ theta, float* __restrict__ grad,
                                int64_t ld, int64_t off_w, int nin, int nout, float lambda, int prior,
                                float inv_sigma2) {
  const int p = blockIdx.y;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nw = (int64_t)nin * nout;
  if (t >= nw + nout) return;
  float v = 0.f;
  if (t < nw) {
    const int o = (int)(t / nin), i = (int)(t % nin);
    const float* src = W.base + p * W.pstride + (int64_t)o * W.ostride + i;
    for (int s = 0; s < W.splits; ++s) v += src[s * W.sstride];
  } else {
    const int o = (int)(t - nw);
    const float* src = Bv.base + p * Bv.pstride + (int64_t)o * Bv.ostride;
    for (int s = 0; s < Bv.splits; ++s) v += src[s * Bv.sstride];
  }
  const int64_t idx = p * ld + off_w + t;
  const float pr = (prior == PUSH_PRIOR_GAUSSIAN) ? -theta[idx] * inv_sigma2 : 0.f;
  grad[idx] = fmaf(-lambda, v, pr);
}
void finalize_layer(PartView W, PartView Bv, const float* theta, float* grad, int64_t ld, int64_t off_w, int in,
                    int out, float lambda, int prior, float inv_sigma2, int batch, cudaStream_t s) {
  const int64_t tot = (int64_t)in * out + out;
  finalize_kernel<<<dim3((unsigned)((tot + 255) / 256), batch), 256, 0, s>>>(W, Bv, theta, grad, ld, off_w, in, out,
                                                                             lambda, prior, inv_sigma2);
}

// ---------------------------------------------------------------- set_grads copy
__global__ void copy_rows_kernel(const float* __restrict__ src, int64_t d, float* __restrict__ dst, int64_t ld) {
  const int p = blockIdx.y;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < d; t += (int64_t)gridDim.x * blockDim.x)
    dst[p * ld + t] = src[p * d + t];
}
void copy_rows(const float* src, int64_t d, float* dst, int64_t ld, int rows, cudaStream_t s) {
  const int blocks = (int)std::min<int64_t>((d + 255) / 256, 2048);
  copy_rows_kernel<<<dim3(blocks, rows), 256, 0, s>>>(src, d, dst, ld);
}

}  // namespace kern
}  // namespace push
