// kernels.h — launchers for the CUDA-core kernels of the SVGD step (non-GEMM parts).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/push.h"

namespace push {
namespace kern {

constexpr int THIN_CHUNK = 256;  // batch rows per thin weight-gradient partial (fixed: P-invariant order)

// ---------------------------------------------------------------- a0 helpers
// Weights only: hi = tf32_rn(x), lo = x - hi for x = src[p*src_pstride + t], t < count, p < batch.
void split_hilo(const float* src, int64_t src_pstride, float* hi, float* lo, int64_t dst_pstride, int64_t count,
                int batch, cudaStream_t s);

// ---------------------------------------------------------------- a1 / a2 thin forward
// out[p][b][o] = sigma( sum_i in[p*in_pstride + b*in + i] W_p[o][i] + bias_p[o] )   (plain fp32)
//   W_p = theta + p*ld_theta + off_w  ([out][in] row-major), bias_p = theta + p*ld_theta + off_b
void thin_forward(const float* in, int64_t in_pstride, const float* theta, int64_t ld_theta, int64_t off_w,
                  int64_t off_b, int in_, int out, int act, float* dst, int64_t out_pstride, int B, int batch,
                  cudaStream_t s);

// ---------------------------------------------------------------- a3 fused output layer (+ top of a4/a5)
constexpr int kMaxDout = 8;  // output width handled by output_fused
struct OutputArgs {
  const float* A;            // input of the output layer [p][B][H] (a_pstride; 0 = shared x)
  int64_t a_pstride;
  int H, dout, B, act;       // act: hidden activation (for sigma' of A when dprev != nullptr)
  const float* theta;        // W_L at theta + p*ld + off_w ([dout][H]), b_L at off_b
  int64_t ld, off_w, off_b;
  const float* y;            // [B][dout]
  float* err2;               // [p][B] sum_o e^2 (err_pstride)
  int64_t err_pstride;
  float* wpart;              // (rb, p, o, i) at rb*wo_sstride + p*wo_pstride + o*H + i
  int64_t wo_sstride, wo_pstride;
  float* bpart_out;          // (rb, p, o) at rb*bo_sstride + p*bo_pstride + o
  int64_t bo_sstride, bo_pstride;
  float* dprev;              // nullptr, or delta of the layer below [p][B][H] (dp_pstride)
  int64_t dp_pstride;
  float* bpart_prev;         // (rb, p, i) at rb*bp_sstride + p*bp_pstride + i
  int64_t bp_sstride, bp_pstride;
};
void output_fused(const OutputArgs& a, int batch, cudaStream_t s);
// Predictive forward of the output layer: yhat[p][b][o] = A_b . W_o + b_o  (pred laid out [p][B][d_out])
void output_forward(const float* A, int64_t a_pstride, const float* theta, int64_t ld, int64_t off_w, int64_t off_b,
                    int H, int dout, float* pred, int B, int batch, cudaStream_t s);
// Cross-particle mean and population std of pred [n][m] (ascending particle order); mean/std may be NULL.
void predict_stats(const float* pred, int n, int64_t m, float* mean, float* stdev, cudaStream_t s);
// loss[p] = sum_b err2[p][b] / (B d_out)   (fixed-order tree reduction)
void loss_reduce(const float* err2, int64_t err_pstride, float* loss, int B, int d_out, int batch, cudaStream_t s);

// ---------------------------------------------------------------- a4 thin backprop (generic)
// o[p][b][i] = (sum_k delta[p][b][k] W_p[k][i]) * sigma'(aprev[p][b][i])
void thin_backward(const float* dl, int64_t d_pstride, const float* theta, int64_t ld_theta, int64_t off_w, int in,
                   int out, const float* aprev, int64_t a_pstride, int act, float* o, int64_t o_pstride, int B,
                   int batch, cudaStream_t s);

// ---------------------------------------------------------------- a5 thin weight gradient partials (generic)
// part[s][p][o][i'] = sum_{b in chunk s} delta[p][b][o] * A(p,b,i'),  i' < in_eff + 1, A(.,.,in_eff) = 1
// (in_eff = 0 gives the bias-only column sums).  chunks of THIN_CHUNK rows; returns #chunks.
int thin_wgrad(const float* dl, int64_t d_pstride, const float* A, int64_t a_pstride, int in_eff, int out, float* part,
               int B, int batch, cudaStream_t s);

// ---------------------------------------------------------------- a5 finalize into G
struct PartView {
  const float* base;
  int splits;
  int64_t sstride, pstride, ostride;  // element (s, p, o, i) at base + s*sstride + p*pstride + o*ostride + i
};
// G_p[off_w + o*in + i] = -lambda * sum_s W(s,p,o,i) + prior(theta)   (o < out, i < in)
// G_p[off_b + o]        = -lambda * sum_s Bv(s,p,o,0) + prior(theta)
// G_p[off_w + o*in + i] = -lambda * sum_s W(s,p,o,i) + prior(theta), G_p[off_b + o] likewise from Bv, for every
// layer job in ONE launch (issued after the backward pass; the partial buffers are per layer).
struct FinalizeJob {
  PartView W, Bv;
  int64_t off_w;
  int in, out;
  int nb_w, nb_b;        // blocks for the weight / bias parts
  int w_warp, b_warp;    // 0 thread per element, 1 column group (many partials), 2 thread per 4 elements,
                         // 3 weights already in G (-lambda dW stored by the GEMM): add the prior in place
  int blk0;              // first block of this job (set by finalize_all)
};
constexpr int kMaxFinalizeJobs = 16;
FinalizeJob make_finalize_job(const PartView& W, const PartView& Bv, int64_t off_w, int in, int out);
// Same, for a layer whose weight gradient the GEMM already wrote into G as -lambda dW (split-K 1):
// only the bias partials are reduced, plus the Gaussian prior added to the weights in place.
FinalizeJob make_finalize_job_wdirect(const PartView& Bv, int64_t off_w, int in, int out, int prior);
void finalize_all(const FinalizeJob* jobs, int njobs, const float* theta, float* grad, int64_t ld, float lambda,
                  int prior, float inv_sigma2, int batch, cudaStream_t s);

// ---------------------------------------------------------------- K0 init (R14)
struct InitTable {
  int n_layers;
  int64_t off[17];   // start of layer l in the canonical row (off[L] = d)
  float bound[16];   // fp32(1/sqrt(in_l)), rounded once on the host
};
void init_theta(float* theta, int64_t ld, int row0, int rows, int64_t d, uint64_t seed, const InitTable& t,
                cudaStream_t s);

// ---------------------------------------------------------------- a7 distances
// Column ranges ("tensors") over which separate distance matrices are summed: one range [0, ld) for
// the canonical kernel over the whole theta, or W_l / b_l of every layer for PUSH_VAR_PER_TENSOR.
constexpr int kMaxTensors = 2 * 15;
struct TSplit { int s[kMaxTensors + 1]; };  // splits of tensor t are [s[t], s[t+1])
struct DistPlan {
  int T;        // tile side (8, 16, 32 or 64)
  int ntile;    // ceil(n / T)
  int npairs;   // ntile*(ntile+1)/2 upper tile pairs
  int splits;   // S_d (all tensors)
  int64_t cols; // columns per split (multiple of the staged sub-chunk width)
  int tensors;  // T_k
  TSplit tsplit;
  std::vector<int64_t> ranges;  // [begin, end) column range of every split (uploaded to the device)
};
// toff/tsize: the tensors' column ranges; `total` = the column count the split width is sized from.
// The plan depends only on (n, tensor ranges), never on the number of ranks.
DistPlan dist_plan(int n, int tensors, const int64_t* toff, const int64_t* tsize, int64_t total);
// part[s][i][j] = sum_{c in range s} (theta_ic - theta_jc)^2; ranges_dev = pl.ranges on the device
void dist_partial(const float* theta, int64_t ld, int n, const DistPlan& pl, const int64_t* ranges_dev, float* part,
                  cudaStream_t s);
// Where split s's partial lives: rank q = the owner of s (s0[q] <= s < s0[q+1]) at slot q*smax + s - s0[q]
// (NEXT-4: each rank's partials all-gathered in rank blocks of smax).  Identity: P = 1, s0 = {0, splits}.
constexpr int kMaxRanks = 64;
struct RankSlots {
  int P, smax;
  int s0[kMaxRanks + 1];
};
// D[t][i][j] = sum_{s in tensor t} part[slot(s)][i][j] (ascending s), D_ii = +0
void dist_reduce(const float* part, int n, const DistPlan& pl, const RankSlots& rs, float* D, cudaStream_t s);

// Centred symmetric Gram form of a7 (gram.cu; canonical kernel, 2 <= n <= kGramMaxN, both exchange modes).
// Plan: splits x ceil(n/64) i-blocks ~ one wave, ranges whole 128-column units of [0, ld) (T = 0 marks it).
constexpr int kGramMaxN = 256;
DistPlan gram_plan(int n, int64_t ld);
int gram_np(int n);                 // MMA N: n rounded up to a power of two >= 16
int64_t gram_part_floats(int n);    // floats of one split's partial block: ceil(n/64) x 128 x gram_np(n)
// part[s] (s < splits, block of gram_part_floats(n)) = [X; Y] of split s's columns of theta (rows 0..n-1,
// pitch ld, centred on row 0); ranges_dev: the splits' [begin, end) column pairs relative to theta
push_status gram_partial(const float* theta, int64_t ld, int n, int splits, const int64_t* ranges_dev, float* part,
                         cudaStream_t s);
// sums = the S split blocks summed in ascending order (split s's block at slot rs(s), as dist_reduce;
// gram_part_floats(n) floats), then (n > kGramDInBandwidth) D_ij = D_ji = max(G_ii + G_jj - 2 G_ij, 0), D_ii = +0;
// for smaller n the bandwidth kernel evaluates D from the sums (bandwidth_kernel's gsums argument)
constexpr int kGramDInBandwidth = 128;
bool gram_d_in_bandwidth(int n);
void gram_dist(const float* part, int n, int S, const RankSlots& rs, float* sums, float* D, cudaStream_t s);

// ---------------------------------------------------------------- a8 + a9 bandwidth and kernel matrix
// Per tensor t (one CTA each): h_t from D_t (rule, c = fp32 1/ln n or 1/ln(n+1), or fixed bw_h);
// K[t][i][j] = exp(-D_t[row0+i][j]/h_t), srow[t][i] = sum_j K[t][i][j]
// gsums != nullptr (Gram form, one tensor, n <= kGramDInBandwidth): D is first evaluated from the summed Gram
// blocks (gram_np(n) columns) and written to D, then used as above.
void bandwidth_kernel(const float* D, int n, int row0, int nl, int rule, float c_ln, float bw_h, float* h, float* K,
                      float* srow, int tensors, cudaStream_t s, const float* gsums = nullptr);

// ---------------------------------------------------------------- a10 fused update
// theta_next[row0+i][c] = theta_i[c] + (eps/n)[ sum_j K_ij (g_j[c] - r theta_j[c]) + r s_i theta_i[c] ], r = 2/h
// Returns the number of kernels launched (1).
int svgd_update(const float* theta, const float* grad, int64_t ld, int n, int row0, int nl, const float* K,
                const float* srow, const float* h, float eps_over_n, float* theta_next, cudaStream_t s);
int update_row_block(int n, int nl, int64_t ld);
// Tensor-core update (push_api update_tc): lhs [nl][2n] = [K, -rK] (g_first) or [-rK, K], r = 2/h, rows at
// `pitch` (>= 2n, a multiple of 4), npad >= nl rows (the padding is zeroed); the GEMM (EPI_UPD) contracts
// U = lhs [G; Theta] and writes theta_next[i][c] = theta[i][c] + eps_n (U[i][c] + r s_i theta[i][c])
void update_lhs(const float* K, int nl, int npad, int n, int pitch, const float* h, bool g_first, float* lhs,
                cudaStream_t s);
// a10 as one streaming tensor-core contraction (upd.cu, R28), n <= 64, rows <= 64:
// out[i][c] = sum_q L[i][q] B[q][c], B = the 2n x w operand at b ([G; Theta] when g_first), L the folded
// coefficients (eps_n K_ij on G rows; -eps_n r K_ij on Theta rows plus 1 + eps_n r (s_i - K_ii) on the own
// particle own_row + i), split into tf32 hi / lo (lhs_hi, lhs_lo: scratch of update_tc_npad(rows) x
// round_up(2n, 4) floats each); = th_i + eps_n (sum_j K_ij (g_j - r th_j) + r s_i th_i); w % 128 == 0
constexpr int kUpdTcMaxRows = 64;
int update_tc_npad(int rows);
push_status update_tc_stream(const float* b, bool g_first, int n, int64_t w, int rows, int own_row, const float* K,
                             const float* h, float* lhs_hi, float* lhs_lo, float* out, const float* srow, float eps_n,
                             cudaStream_t s);
// NEXT-2 variants: column segments of <= kVarSegCols columns inside one tensor (x = begin, y = end, z = tensor)
constexpr int kVarSegCols = 128;
std::vector<int4> var_segments(int tensors, const int64_t* toff, const int64_t* tsize);
// element c of tensor t (segment table segs_dev, nseg entries):
//   theta_next_ic = theta_ic + eps_d [ sum_j K^t_ij (g_jc - r_t theta_jc) + r_t s^t_i theta_ic + pcoef sum_j theta_jc ]
//   r_t = (2/h_t) alpha   (canonical weights: eps_d = eps/n, alpha = 1; paper: eps_d = eps, alpha = 1/n)
int svgd_update_var(const float* theta, const float* grad, int64_t ld, int n, int row0, int nl, const float* K,
                    const float* srow, const float* h, const int4* segs_dev, int nseg, float alpha, float eps_d,
                    float pcoef, float* theta_next, cudaStream_t s);

// ---------------------------------------------------------------- NEXT-3: deep ensembles and diagonal SWAG
// theta[p][k] += eps * g[p][k] for the own rows (in place)
void ensemble_step(float* theta, const float* grad, int64_t ld, int rows, float eps, cudaStream_t s);
// mean <- (mean k + x)/(k+1), sq <- (sq k + x^2)/(k+1) elementwise over count elements (k = snapshots so far)
void swag_collect(const float* x, float* mean, float* sq, int64_t count, int64_t k, cudaStream_t s);
// out[r][c] = mean + sqrt(max(sq - mean^2, 0)) * z(seed, row0 + r, c)   (counter-based Box-Muller, see push.h)
void swag_sample(const float* mean, const float* sq, int64_t ld, int64_t d, int row0, int rows, uint64_t seed,
                 float* out, cudaStream_t s);

// copy rows (device, pitched) for set_grads: dst[p*ld + k] = src[p*d + k]
void copy_rows(const float* src, int64_t d, float* dst, int64_t ld, int rows, cudaStream_t s);

}  // namespace kern
}  // namespace push
