// push_api.cu — the C-ABI of include/push.h: context, workspace carving, state machine,
// the orchestration of one SVGD particle step, row exchange (NCCL or loopback), profiling.
//
// Step structure (PAPER.md:655-660 Fig. supp:svgd):
//   push_particle_grads  a0-a5   (pstep on every local particle; all-gather Theta)
//   push_svgd_step       a6-a10  (all-gather G; distances; median h; K; fused update)
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/push.h"
#include "../../include/push_debug.h"
#include "common.cuh"
#include "gemm.h"
#include "kernels.h"
#include "nccl_dl.h"

namespace push {

// ------------------------------------------------------------------ error state
namespace {
thread_local std::string t_err;
}
void set_error(const std::string& msg) { t_err = msg; }
push_status fail(push_status st, const std::string& msg) {
  t_err = msg;
  return st;
}

// ------------------------------------------------------------------ plan
constexpr int kMaxN = 2048;  // a10 keeps 16 kernel rows x n in shared memory

struct LayerPlan {
  int in = 0, out = 0;
  int64_t off_w = 0, off_b = 0;  // canonical offsets in a particle row
  bool gemm = false;             // tensor-core path (hidden layer with in, out % 32 == 0)
  bool wraw = false;             // GEMM reads W straight from Theta (16-B aligned) and splits it in smem
  int64_t woff = 0;              // offset of this layer's hi/lo weight copy (per-particle block), !wraw only
  int wsplit_max = 1;            // weight-gradient split count at max_batch (partial buffer size)
};

constexpr int kGramMinN = 32;       // a7 in the Gram form from this many particles (measured crossover)
constexpr int kNcclMaxCtas = 16;    // SMs the NCCL collectives may take while the GEMMs run (ncclConfig maxCTAs)
constexpr int kTcUpdateMinN = 128;
constexpr int kTcStreamMinN = 32;  // a10 as the streaming tensor-core contraction for 32 <= n <= 64  // a10 on the tensor cores from this many particles (measured crossover)
constexpr int kMaxX0 = 4;  // thin first layer whose weight grads are fused into layer 1's BWD epilogue

struct Plan {
  int n = 0, world = 1, nl = 0, L = 0, Bmax = 0, Hmax = 0, RB = 0;
  int64_t d = 0, ld = 0;
  std::vector<LayerPlan> layers;
  int64_t wsplit_total = 0;                 // per particle elements of the hi/lo weight copies
  std::vector<int64_t> act_pst;             // per layer 0..L-2 activation particle stride
  int64_t dlt_pst = 0;                      // delta buffer particle stride
  int64_t wpart_elems = 0, tpart_elems = 0;  // (unused totals kept for reference)
  bool fuse_x0 = false;                     // layer 0 thin + layer 1 GEMM: dW_0 from layer 1's BWD epilogue
  kern::DistPlan dist{};
  int tensors = 1;                          // distance / kernel matrices (2L under PUSH_VAR_PER_TENSOR)
  std::vector<int64_t> toff, tsize;         // their column ranges
  std::vector<int4> useg;                   // variant update segments (variant != 0)
  // NEXT-4 d-sharded kernel phase: rank q owns the distance splits [ds_s0[q], ds_s0[q+1]) = the columns
  // [ds_c0[q], ds_c0[q+1]) (whole splits, so every sum keeps the order of the all-gather path)
  bool ds = false;
  std::vector<int> ds_s0;
  std::vector<int64_t> ds_c0;
  int64_t ds_wmax = 0;  // widest column panel
  int ds_smax = 0;      // most splits on one rank (the all-gathered partial slots per rank)
  bool gram = false;    // a7 as the centred symmetric Gram product (gram.cu); dist holds its split plan
  bool tc_update = false;  // a10 as the contraction [K, -rK] x [G; Theta] on the tensor cores
  bool tc_stream = false;  // a10 as the streaming transposed contraction with the fused update (upd.cu)
  // byte offsets into the workspace
  size_t o_ulhs = 0, o_gsum = 0;
  size_t o_theta0, o_theta1, o_grad, o_whi, o_wlo, o_dlt0, o_dlt1, o_err2, o_loss, o_loss_all, o_opw, o_opb,
      o_xpart, o_dpart, o_D, o_K, o_s, o_h, o_xbuf, o_ybuf, o_pred, o_swag_mean, o_swag_sq, o_dranges, o_useg,
      o_pth, o_pg, o_pth2, o_pack_th, o_pack_g;
  std::vector<size_t> o_act;
  // per-layer partial buffers, all alive until the single finalize launch at the end of a5
  std::vector<size_t> o_wpart, o_tpart, o_bpart;
  size_t total = 0;
};

static int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

static push_status validate(const push_config* c, int world) {
  if (!c) return fail(PUSH_E_INVALID, "cfg is NULL");
  if (world < 1) return fail(PUSH_E_INVALID, "world_size must be >= 1");
  if (c->n_particles < 1 || c->n_particles > kMaxN)
    return fail(PUSH_E_SHAPE, "n_particles must be in [1, " + std::to_string(kMaxN) + "]");
  if (c->n_particles % world) return fail(PUSH_E_INVALID, "n_particles % world_size != 0 (R18)");
  if (c->n_layers < 1 || c->n_layers > PUSH_MAX_LAYERS) return fail(PUSH_E_SHAPE, "n_layers must be in [1, 15]");
  for (int l = 0; l <= c->n_layers; ++l)
    if (c->dims[l] < 1) return fail(PUSH_E_SHAPE, "dims must be >= 1");
  if (c->dims[c->n_layers] > kern::kMaxDout)
    return fail(PUSH_E_SHAPE, "output width d_out must be <= " + std::to_string(kern::kMaxDout));
  if (c->activation < PUSH_ACT_TANH || c->activation > PUSH_ACT_IDENTITY)
    return fail(PUSH_E_INVALID, "bad activation");
  if (c->prior != PUSH_PRIOR_UNIFORM && c->prior != PUSH_PRIOR_GAUSSIAN) return fail(PUSH_E_INVALID, "bad prior");
  if (c->prior == PUSH_PRIOR_GAUSSIAN && !(c->prior_sigma > 0.f)) return fail(PUSH_E_INVALID, "prior_sigma <= 0");
  if (!(c->lik_scale > 0.f)) return fail(PUSH_E_INVALID, "lik_scale must be > 0");
  if (c->bw_rule < PUSH_BW_MEDIAN_LN_N || c->bw_rule > PUSH_BW_FIXED) return fail(PUSH_E_INVALID, "bad bw_rule");
  if (c->bw_rule == PUSH_BW_FIXED && !(c->bw_h > 0.f)) return fail(PUSH_E_INVALID, "bw_h <= 0 (SPEC.md:100)");
  if (!(c->step_size > 0.f)) return fail(PUSH_E_INVALID, "step_size must be > 0");
  if (c->max_batch < 1) return fail(PUSH_E_SHAPE, "max_batch must be >= 1");
  if (c->swag != 0 && c->swag != 1) return fail(PUSH_E_INVALID, "swag must be 0 or 1");
  if (c->variant < 0 || c->variant > PUSH_VARIANT_PAPER) return fail(PUSH_E_INVALID, "bad variant");
  if (c->exchange != PUSH_XCHG_ALLGATHER && c->exchange != PUSH_XCHG_DSHARD) return fail(PUSH_E_INVALID, "bad exchange");
  if (c->exchange == PUSH_XCHG_DSHARD && c->variant != 0)
    return fail(PUSH_E_INVALID, "exchange DSHARD needs variant 0");
  if (world > kern::kMaxRanks) return fail(PUSH_E_INVALID, "world_size > 64");
  if (c->reserved != 0) return fail(PUSH_E_INVALID, "reserved must be 0");
  return PUSH_OK;
}

// Split-K count of a weight-gradient GEMM (K = B): enough splits that one particle's layer has >= 32
// 128x128 output tiles, at most 8 and at most one per 1024 rows.  It depends only on (B, layer shape),
// never on the number of particles per rank, so the dW summation order is the same for every P.
// Weight-gradient GEMMs whose N = in is a multiple of 256 run on 256 x 256 CTA-pair tiles: there the
// count is the one (<= 8, >= 1024 rows per split) that minimises waves x k-blocks per tile over the
// n particles' tiles on B200's 74 SM pairs; a larger count must cut that by >= 10% (every split adds
// a partial round trip through HBM and the finalize pass).  This
// depends on (B, layer shape, n), never on the sharding, so the summation order is P-invariant.
constexpr int kPlanSmPairs = 148 / 2;
static int wgrad_splits(int B, int out, int in, int n) {
  const int cap = std::min(8, std::max(1, B / 1024));
  if (in % 256 == 0) {
    const int64_t tiles = (int64_t)((out + 255) / 256) * (in / 256) * n;
    const int64_t nkb = (B + 31) / 32;
    int best = 1;
    int64_t best_cost = INT64_MAX / 16;
    for (int want = 1; want <= cap; ++want) {
      const int S = gemm::effective_splits(B, want);
      const int64_t cost = ((tiles * S + kPlanSmPairs - 1) / kPlanSmPairs) * ((nkb + S - 1) / S);
      if (10 * cost < 9 * best_cost) {  // a split must buy >= 10%: each one adds a partial round trip
        best_cost = cost;
        best = S;
      }
    }
    return best;
  }
  const int tiles = ((out + 127) / 128) * ((in + 127) / 128);
  const int want = std::min({cap, std::max(1, (32 + tiles - 1) / tiles)});
  return gemm::effective_splits(B, want);
}

// A weight-gradient GEMM with one split writes -lambda dW straight into G (TMA-legal when the layer's
// weights start on a 16-B boundary and rows are whole 16-B units).  Run-time splits are capped at the
// max_batch count, so one split at max_batch means one split for every batch and no partial buffer.
static bool wgrad_in_g(int off_w_mod4, int in, int S) { return S == 1 && off_w_mod4 == 0 && in % 4 == 0; }

static push_status make_plan(const push_config* c, int world, Plan* p) {
  push_status st = validate(c, world);
  if (st != PUSH_OK) return st;
  Plan& P = *p;
  P.n = c->n_particles;
  P.world = world;
  P.nl = P.n / world;
  P.L = c->n_layers;
  P.Bmax = c->max_batch;
  P.RB = (P.Bmax + gemm::kRowBlock - 1) / gemm::kRowBlock;
  P.layers.resize(P.L);
  int64_t off = 0;
  P.Hmax = 1;
  for (int l = 0; l < P.L; ++l) {
    LayerPlan& lp = P.layers[l];
    lp.in = c->dims[l];
    lp.out = c->dims[l + 1];
    lp.off_w = off;
    off += (int64_t)lp.in * lp.out;
    lp.off_b = off;
    off += lp.out;
    lp.gemm = (l < P.L - 1) && (lp.in % 32 == 0) && (lp.out % 32 == 0);
    if (l < P.L - 1) P.Hmax = std::max(P.Hmax, lp.out);
  }
  P.d = off;
  // 512-B rows: whole 128-column tiles for the tensor-core update (a10) and the TMA boxes
  P.ld = round_up(P.d, 128);
  P.fuse_x0 = P.L >= 3 && !P.layers[0].gemm && P.layers[1].gemm && P.layers[0].in <= kMaxX0;
  P.wsplit_total = 0;
  int64_t max_w = 0, max_t = 0;
  for (int l = 0; l < P.L; ++l) {
    LayerPlan& lp = P.layers[l];
    lp.wraw = lp.gemm && (lp.off_w % 4 == 0);
    if (lp.gemm && !lp.wraw) {
      lp.woff = P.wsplit_total;
      P.wsplit_total += round_up((int64_t)lp.in * lp.out, 32);
    }
    if (lp.gemm) {
      max_w = std::max<int64_t>(max_w, (int64_t)lp.in * lp.out);
      max_t = std::max<int64_t>(max_t, lp.out);  // bias-only column sums
    } else if (l < P.L - 1) {
      max_t = std::max<int64_t>(max_t, (int64_t)lp.out * (lp.in + 1));
    }
  }
  P.act_pst.assign(std::max(P.L - 1, 0), 0);
  for (int l = 0; l + 1 < P.L; ++l) P.act_pst[l] = round_up((int64_t)P.Bmax * P.layers[l].out, 32);
  P.dlt_pst = round_up((int64_t)P.Bmax * P.Hmax, 32);
  const int chunks_max = (P.Bmax + kern::THIN_CHUNK - 1) / kern::THIN_CHUNK;
  P.wpart_elems = 8 * (int64_t)P.nl * max_w;
  P.tpart_elems = (int64_t)chunks_max * P.nl * max_t;
  // distance tensors: the whole row [0, ld) (canonical), [0, d) (other variants) or every W_l / b_l
  if (c->variant & PUSH_VAR_PER_TENSOR) {
    for (const LayerPlan& lp : P.layers) {
      P.toff.push_back(lp.off_w);
      P.tsize.push_back((int64_t)lp.in * lp.out);
      P.toff.push_back(lp.off_b);
      P.tsize.push_back(lp.out);
    }
  } else {
    P.toff.push_back(0);
    P.tsize.push_back(c->variant ? P.d : P.ld);
  }
  P.tensors = (int)P.toff.size();
  P.dist = kern::dist_plan(P.n, P.tensors, P.toff.data(), P.tsize.data(), c->variant ? P.d : P.ld);
  if (c->variant) P.useg = kern::var_segments(P.tensors, P.toff.data(), P.tsize.data());
  P.ds = c->exchange == PUSH_XCHG_DSHARD;
  // Canonical kernel, 32 <= n <= 256 (both exchange modes): a7 as the centred symmetric Gram product on
  // the tensor cores (gram.cu; R27) — one HBM stream of Theta, no CUDA-core pair loop.  Its
  // split plan replaces the direct-form plan; it depends only on (n, ld), so every sharding (and the
  // d-sharded mode, which owns whole splits) sums the same partials in the same order.  Below 32
  // particles the direct form is HBM-bound already (n <= 8: 0.84 of HBM at C5) and a Gram stage carries
  // too few bytes (C5: 1.09 ms Gram vs 0.12 ms direct; C2: 29 vs 25 us).
  if (c->variant == 0 && P.n >= kGramMinN && P.n <= kern::kGramMaxN) {
    P.dist = kern::gram_plan(P.n, P.ld);
    P.gram = true;
  }
  // Many particles (n >= kTcUpdateMinN, e.g. C4 at n = 256): a10 is FP32-issue bound on the CUDA cores
  // (2 n_local flops per streamed element); as the contraction U = [K, -rK] [G; Theta] on the tensor
  // cores (3xTF32, K = 2n) plus an elementwise pass it is memory-bound (C4 a10 0.060 -> 0.033 ms).  At
  // n = 64 (C3, S1) the staged CUDA-core kernel measured faster (1.19 vs 1.32 ms at C3; fusing the fix-up
  // into a transposed GEMM epilogue measured slower still, 2.3 ms), so it keeps those.  The choice
  // depends on n only (never on n_local or the exchange mode), so every sharding and the d-sharded
  // panels take the same arithmetic (P-invariance).
  P.tc_update = c->variant == 0 && P.n >= kTcUpdateMinN && P.ld % 128 == 0;
  // 32 <= n <= 64 (C3, S1): theta' as one streaming contraction with the folded coefficients (upd.cu,
  // DESIGN.md R28): B read once from HBM, no U round trip (the staged CUDA-core kernel was FP32-issue /
  // latency bound at ~0.3 of HBM there; this one measured 0.77-0.81 of HBM).  n only, as above.
  P.tc_stream = c->variant == 0 && P.n >= kTcStreamMinN && P.n <= kern::kUpdTcMaxRows && P.ld % 128 == 0;
  if (P.ds) {
    const int S = P.dist.splits;
    for (int q = 0; q <= world; ++q) P.ds_s0.push_back((int)((int64_t)q * S / world));
    for (int q = 0; q <= world; ++q) P.ds_c0.push_back(P.ds_s0[q] < S ? P.dist.ranges[2 * P.ds_s0[q]] : P.ld);
    for (int q = 0; q < world; ++q) {
      P.ds_wmax = std::max(P.ds_wmax, P.ds_c0[q + 1] - P.ds_c0[q]);
      P.ds_smax = std::max(P.ds_smax, P.ds_s0[q + 1] - P.ds_s0[q]);
    }
  }

  size_t cur = 0;
  auto take = [&](int64_t elems) {
    size_t o = cur;
    cur += (size_t)round_up(std::max<int64_t>(elems, 1) * 4, 256);
    return o;
  };
  const int64_t nld = (int64_t)P.n * P.ld;
  const LayerPlan& top = P.layers[P.L - 1];
  // Theta[0], G, Theta[1] adjacent (n*ld*4 is a multiple of 256): [Theta_cur; G] or [G; Theta_cur] is
  // one 2n x ld operand for the tensor-core update
  P.o_theta0 = take(nld);
  P.o_grad = take(nld);
  P.o_theta1 = take(nld);
  P.o_whi = take(P.nl * P.wsplit_total);
  P.o_wlo = take(P.nl * P.wsplit_total);
  P.o_act.resize(P.act_pst.size());
  for (size_t l = 0; l < P.act_pst.size(); ++l) P.o_act[l] = take(P.nl * P.act_pst[l]);
  P.o_dlt0 = take(P.nl * P.dlt_pst);
  P.o_dlt1 = take(P.nl * P.dlt_pst);
  P.o_err2 = take((int64_t)P.nl * P.Bmax);
  P.o_loss = take(P.nl);
  P.o_loss_all = take(P.n);
  P.o_wpart.assign(P.L, SIZE_MAX);  // SIZE_MAX: no partial buffer (thin layer or dW straight into G)
  P.o_tpart.assign(P.L, 0);
  P.o_bpart.assign(P.L, 0);
  for (int l = 0; l < P.L; ++l) {
    const LayerPlan& lp = P.layers[l];
    const int smax = wgrad_splits(P.Bmax, lp.out, lp.in, P.n);
    P.layers[l].wsplit_max = smax;
    if (lp.gemm && !wgrad_in_g((int)(lp.off_w % 4), lp.in, smax))
      P.o_wpart[l] = take((int64_t)smax * P.nl * lp.in * lp.out);
    // thin weight partials (thin hidden layers) or bias-only column sums (GEMM layers under a thin one)
    if (l < P.L - 1) P.o_tpart[l] = take((int64_t)chunks_max * P.nl * lp.out * (lp.gemm ? 1 : lp.in + 1));
    if (l < P.L - 1) P.o_bpart[l] = take((int64_t)P.RB * P.nl * lp.out);
  }
  P.o_opw = take((int64_t)P.RB * P.nl * top.out * top.in);
  P.o_opb = take((int64_t)P.RB * P.nl * top.out);
  P.o_xpart = take(P.fuse_x0 ? (int64_t)P.RB * P.nl * P.layers[0].out * P.layers[0].in : 1);
  P.o_dpart = take((int64_t)(P.ds ? world * P.ds_smax : P.dist.splits) *
                   (P.gram ? kern::gram_part_floats(P.n) : (int64_t)P.n * P.n));
  P.o_ulhs = take(P.tc_update ? (int64_t)(P.ds ? P.n : P.nl) * round_up(2 * P.n, 4)
                               : (P.tc_stream ? 2 * (int64_t)kern::kUpdTcMaxRows * round_up(2 * P.n, 4) : 1));
  P.o_gsum = take(P.gram ? kern::gram_part_floats(P.n) : 1);
  P.o_D = take((int64_t)P.tensors * P.n * P.n);
  P.o_K = take((int64_t)P.tensors * (P.ds ? P.n : P.nl) * P.n);  // d-sharded: K of all n rows
  P.o_s = take((int64_t)P.tensors * (P.ds ? P.n : P.nl));
  const int64_t pan = P.ds ? (int64_t)P.n * P.ds_wmax : 1;  // column panels (n x w) and send/recv staging
  // [Theta panel (even steps); G panel; Theta panel (odd steps)] at the own pitch: the tensor-core update's
  // 2n x w operand in the same row order as the all-gather path's Theta[0], G, Theta[1] (bit-identity)
  P.o_pth = take(3 * pan);
  P.o_pg = take(1);
  P.o_pth2 = take(pan);
  P.o_pack_th = take(pan);
  P.o_pack_g = take(pan);
  P.o_h = take(32);
  P.o_dranges = take(2 * (int64_t)P.dist.ranges.size());  // int64 pairs (2 floats' room each)
  P.o_useg = take(4 * (int64_t)P.useg.size());
  P.o_xbuf = take((int64_t)P.Bmax * P.layers[0].in);
  P.o_ybuf = take((int64_t)P.Bmax * top.out);
  P.o_pred = take((int64_t)P.n * P.Bmax * top.out);
  P.o_swag_mean = take(c->swag ? (int64_t)P.nl * P.ld : 1);
  P.o_swag_sq = take(c->swag ? (int64_t)P.nl * P.ld : 1);
  P.total = cur;
  return PUSH_OK;
}

// floats of one split's distance partial (the direct form's n x n, or the Gram form's [X; Y] blocks)
static int64_t part_block(const Plan& P) {
  return P.gram ? kern::gram_part_floats(P.n) : (int64_t)P.n * P.n;
}

// ------------------------------------------------------------------ profiling classes
enum PClass {
  PC_INIT = 0, PC_SPLIT, PC_FWD_THIN, PC_FWD_GEMM, PC_OUTPUT, PC_LOSS, PC_BWD_THIN, PC_BWD_GEMM, PC_WGRAD_GEMM,
  PC_WGRAD_THIN, PC_FINALIZE, PC_EXCHANGE, PC_DIST, PC_BANDWIDTH, PC_UPDATE, PC_COPY, PC_N
};
static const char* kClassNames[PC_N] = {"init",        "split_hilo",  "fwd_thin",   "fwd_gemm",
                                        "output_loss", "loss_reduce", "bwd_thin",   "bwd_gemm",
                                        "wgrad_gemm",  "wgrad_thin",  "finalize_g", "exchange",
                                        "distances",   "bandwidth_k", "svgd_update", "copy"};

struct ProfRec {
  int cls;
  cudaEvent_t e0, e1;
  double bytes, flops;
  int launches;
};

struct LocalGroup;

}  // namespace push

// ------------------------------------------------------------------ context
struct push_ctx {
  push_config cfg{};
  push::Plan P;
  int rank = 0, world = 1;
  int row0 = 0;
  int device = 0;
  uint8_t* ws = nullptr;
  float* theta[2] = {nullptr, nullptr};
  int cur = 0;
  float* grad = nullptr;
  float *whi = nullptr, *wlo = nullptr;
  std::vector<float*> act;             // activations A_0 .. A_{L-2}
  float* dlt[2] = {nullptr, nullptr};  // delta ping-pong
  float *err2 = nullptr, *loss = nullptr, *loss_all = nullptr;
  std::vector<float*> wpart, tpart, bpart;  // per layer
  float *opw = nullptr, *opb = nullptr, *xpart = nullptr;
  float *dpart = nullptr, *D = nullptr, *K = nullptr, *srow = nullptr, *h = nullptr;
  float* gsum = nullptr;  // Gram form: the split partials summed
  float* ulhs = nullptr;  // tensor-core update: [K, -rK] or [-rK, K] (n_local x 2n)
  int64_t* dranges = nullptr;  // distance split ranges (device copy of P.dist.ranges)
  int4* useg = nullptr;        // variant update segments (device copy of P.useg)
  // NEXT-4 (d-sharded kernel phase): this rank's panel width, its splits (ranges relative to the panel),
  // where every rank's partials live, and the panels / staging buffers
  int64_t ds_w = 0, ds_c = 0;
  push::kern::DistPlan dist_own;
  push::kern::RankSlots slots{};
  float *pbase = nullptr, *pg = nullptr, *pth2 = nullptr, *pack_th = nullptr, *pack_g = nullptr;  // pg = pbase + n w
  bool ds_deferred = false;  // local group: this rank's step runs in the last rank's call
  float *xbuf = nullptr, *ybuf = nullptr;
  float* pred = nullptr;  // predictive pushforward: n x B x d_out (own rows, then all-gathered)
  float *swag_mean = nullptr, *swag_sq = nullptr;  // SWAG moments of the own rows (n_local x ld)
  int64_t swag_count = 0;
  int pred_B = 0;
  int state = 0;  // 0 READY, 1 GRADS_READY
  bool broken = false;
  bool has_grads = false, has_step = false;
  float c_ln = 1.f;
  // exchange
  push::nccl::Comm comm = nullptr;
  std::shared_ptr<push::LocalGroup> group;
  // comm stream: the Theta all-gather (a6/C1) runs beside the gradient kernels (P > 1)
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_theta = nullptr, ev_fork2 = nullptr, ev_grad = nullptr;
  // captured whole steps: a7-a9 (they read Theta only) forked onto k_stream at the start of the gradient
  // phase and joined before a10 (kphase_ready: D / h / K of the current Theta are in flight there)
  cudaStream_t k_stream = nullptr, w_stream = nullptr;  // w_stream: side work of the gradient phase
  cudaEvent_t ev_kfork = nullptr, ev_kdone = nullptr;
  bool kphase_ready = false;
  bool theta_pending = false;
  // CUDA-graph replay of a whole step (push_step_graph): one executable per Theta buffer parity
  struct GraphEntry {
    int B = 0;
    float* loss = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0;
  };
  GraphEntry graphs[2];
  cudaStream_t cap_stream = nullptr;
  bool graph_warm = false;
  // profiling
  bool prof_on = false;
  std::vector<push::ProfRec> recs;
  std::vector<int32_t> trace;  // kernel class of every launch while profiling, in launch order
  std::vector<cudaEvent_t> ev_pool;
  int64_t launches = 0;
};

namespace push {

struct LocalGroup {
  std::vector<push_ctx*> members;
};

static push_status sticky(push_ctx* c, push_status st) {
  if (st == PUSH_E_CUDA || st == PUSH_E_NCCL) c->broken = true;
  return st;
}

// Join a Theta all-gather that an eager push_particle_grads left on the comm stream: every
// entry that reads or exchanges Theta, or issues collectives on `s`, orders itself after it first.
static push_status join_theta(push_ctx* c, cudaStream_t s) {
  if (!c->theta_pending) return PUSH_OK;
  PUSH_CUDA_TRY(cudaStreamWaitEvent(s, c->ev_theta, 0));
  c->theta_pending = false;
  return PUSH_OK;
}

static cudaEvent_t get_event(push_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Run `f` (which launches `nlaunch` kernels of class `cls`), bracketing it with events when profiling.
static push_status run_k(push_ctx* c, int cls, int nlaunch, double bytes, double flops, cudaStream_t s,
                         const std::function<push_status()>& f) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->prof_on) {
    e0 = get_event(c);
    e1 = get_event(c);
    cudaEventRecord(e0, s);
  }
  push_status st = f();
  if (st == PUSH_OK) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) st = fail(PUSH_E_CUDA, std::string("kernel launch (") + kClassNames[cls] + "): " +
                                                     cudaGetErrorString(e));
  }
  c->launches += nlaunch;
  if (c->prof_on) {
    for (int k = 0; k < nlaunch; ++k) c->trace.push_back(cls);
    cudaEventRecord(e1, s);
    c->recs.push_back(ProfRec{cls, e0, e1, bytes, flops, nlaunch});
  }
  return st;
}

// ------------------------------------------------------------------ exchange
enum BufKind { BUF_THETA = 0, BUF_GRAD = 1, BUF_LOSS = 2, BUF_PRED = 3 };

static float* buf_of(push_ctx* c, int kind, size_t* per_rank) {
  if (kind == BUF_THETA) {
    *per_rank = (size_t)c->P.nl * c->P.ld;
    return c->theta[c->cur];
  }
  if (kind == BUF_GRAD) {
    *per_rank = (size_t)c->P.nl * c->P.ld;
    return c->grad;
  }
  if (kind == BUF_PRED) {
    *per_rank = (size_t)c->P.nl * c->pred_B * c->P.layers[c->P.L - 1].out;
    return c->pred;
  }
  *per_rank = (size_t)c->P.nl;
  return c->loss_all;
}

// In-place all-gather of the row blocks of `kind` (rank r's block at r*per_rank).
static push_status exchange(push_ctx* c, int kind, cudaStream_t s) {
  size_t cnt = 0;
  float* buf = buf_of(c, kind, &cnt);
  if (kind == BUF_LOSS)
    PUSH_CUDA_TRY(cudaMemcpyAsync(buf + c->rank * cnt, c->loss, cnt * 4, cudaMemcpyDeviceToDevice, s));
  if (c->world == 1 && !c->comm) return PUSH_OK;
  const double bytes = 4.0 * cnt * (c->world - 1);
  if (c->group) {
    return run_k(c, PC_EXCHANGE, 0, bytes, 0, s, [&]() -> push_status {
      for (int q = 0; q < c->world; ++q) {
        if (q == c->rank) continue;
        push_ctx* pc = c->group->members[q];
        size_t cq = 0;
        const float* src = kind == BUF_LOSS ? pc->loss : buf_of(pc, kind, &cq) + q * cnt;
        PUSH_CUDA_TRY(cudaMemcpyAsync(buf + q * cnt, src, cnt * 4, cudaMemcpyDeviceToDevice, s));
      }
      return PUSH_OK;
    });
  }
  return run_k(c, PC_EXCHANGE, 0, bytes, 0, s,
               [&]() { return nccl::allgather_f32(buf + c->rank * cnt, buf, cnt, c->comm, s); });
}

// ------------------------------------------------------------------ grads (a0-a5)
struct ActView {
  const float* p;
  int64_t pst;  // particle stride (0: shared x)
};

// Input of layer l: x for l == 0, else the activation A_{l-1}.
static ActView layer_input(push_ctx* c, int l, const float* x) {
  if (l == 0) return ActView{x, 0};
  return ActView{c->act[l - 1], c->P.act_pst[l - 1]};
}

static push_status run_kphase(push_ctx* c, cudaStream_t s);

// fork_kphase (captured whole steps): a7-a9 start on k_stream as soon as Theta_all is complete, beside the
// gradient kernels, and do_step joins them before a10
static push_status do_grads(push_ctx* c, const float* x, const float* y, int B, cudaStream_t s,
                            bool fork_kphase = false) {
  const Plan& P = c->P;
  const int nl = P.nl, L = P.L, act = c->cfg.activation;
  const int64_t ld = P.ld;
  const int RB = (B + gemm::kRowBlock - 1) / gemm::kRowBlock;
  float* th = c->theta[c->cur] + (int64_t)c->row0 * ld;  // own rows
  float* g = c->grad + (int64_t)c->row0 * ld;
  const float lambda = c->cfg.lik_scale;
  const float inv_s2 = c->cfg.prior == PUSH_PRIOR_GAUSSIAN ? 1.0f / (c->cfg.prior_sigma * c->cfg.prior_sigma) : 0.f;
  push_status st;
  // side stream (captured steps only, fork_kphase): work off the backward critical path — the loss
  // reduction and each layer's weight gradient — forked from s and joined in order.  side_ev holds the
  // completion events not yet joined (oldest first); side_join_prev joins all but the newest.
  cudaStream_t ws = fork_kphase ? c->w_stream : s;
  std::vector<cudaEvent_t> side_ev;
  auto side_fork = [&]() -> push_status {
    if (ws == s) return PUSH_OK;
    cudaEvent_t e = get_event(c);
    PUSH_CUDA_TRY(cudaEventRecord(e, s));
    PUSH_CUDA_TRY(cudaStreamWaitEvent(ws, e, 0));
    c->ev_pool.push_back(e);
    return PUSH_OK;
  };
  auto side_done = [&]() -> push_status {
    if (ws == s) return PUSH_OK;
    cudaEvent_t e = get_event(c);
    PUSH_CUDA_TRY(cudaEventRecord(e, ws));
    side_ev.push_back(e);
    return PUSH_OK;
  };
  auto side_join = [&]() -> push_status {
    if (side_ev.empty()) return PUSH_OK;
    PUSH_CUDA_TRY(cudaStreamWaitEvent(s, side_ev.front(), 0));
    c->ev_pool.push_back(side_ev.front());
    side_ev.erase(side_ev.begin());
    return PUSH_OK;
  };
  auto side_join_prev = [&]() -> push_status {
    while (side_ev.size() > 1)
      if (side_join() != PUSH_OK) return PUSH_E_CUDA;
    return PUSH_OK;
  };
  // a5 epilogue: every layer's partials are reduced into G by ONE launch after the backward pass
  std::vector<kern::FinalizeJob> jobs;
  // PUSH_VAR_PRIOR_SUM: G keeps the likelihood term only; a10 adds the unweighted prior sum
  const int prior_g = (c->cfg.variant & PUSH_VAR_PRIOR_SUM) ? PUSH_PRIOR_UNIFORM : c->cfg.prior;
  auto finalize = [&](int l, const kern::PartView& W, const kern::PartView& Bv, bool w_in_g = false) {
    const LayerPlan& lp = P.layers[l];
    jobs.push_back(w_in_g ? kern::make_finalize_job_wdirect(Bv, lp.off_w, lp.in, lp.out, prior_g)
                          : kern::make_finalize_job(W, Bv, lp.off_w, lp.in, lp.out));
    return PUSH_OK;
  };

  // C1: Theta rows of every rank (needed by a7/a10; unchanged during the gradient phase, whose kernels
  // only read the own rows, which the in-place all-gather only reads): on the comm stream, joined in
  // push_svgd_step
  if ((c->world > 1 || c->comm) && !P.ds) {
    PUSH_CUDA_TRY(cudaEventRecord(c->ev_fork, s));
    PUSH_CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, c->ev_fork, 0));
    if ((st = exchange(c, BUF_THETA, c->comm_stream)) != PUSH_OK) return st;
    PUSH_CUDA_TRY(cudaEventRecord(c->ev_theta, c->comm_stream));
    c->theta_pending = true;
  }
  // single process only: with an exchange, a7-a9 stay in the step where they hide the G all-gather (C2)
  if (fork_kphase && !P.ds && c->world == 1 && !c->comm) {
    PUSH_CUDA_TRY(cudaEventRecord(c->ev_kfork, s));
    PUSH_CUDA_TRY(cudaStreamWaitEvent(c->k_stream, c->ev_kfork, 0));
    if (c->theta_pending) PUSH_CUDA_TRY(cudaStreamWaitEvent(c->k_stream, c->ev_theta, 0));
    if ((st = run_kphase(c, c->k_stream)) != PUSH_OK) return st;
    PUSH_CUDA_TRY(cudaEventRecord(c->ev_kdone, c->k_stream));
    c->kphase_ready = true;
  }

  // a0: tf32 hi/lo copies of tensor-core weights that are not 16-B aligned in Theta (the others, and all
  // activations, are split on the staged tile inside the GEMM)
  for (int l = 0; l < L; ++l) {
    const LayerPlan& lp = P.layers[l];
    if (!lp.gemm || lp.wraw) continue;
    const int64_t cnt = (int64_t)lp.in * lp.out;
    st = run_k(c, PC_SPLIT, 1, 12.0 * cnt * nl, 0, s, [&] {
      kern::split_hilo(th + lp.off_w, ld, c->whi + lp.woff, c->wlo + lp.woff, P.wsplit_total, cnt, nl, s);
      return PUSH_OK;
    });
    if (st != PUSH_OK) return st;
  }

  // a1/a2: hidden layers forward
  for (int l = 0; l + 1 < L; ++l) {
    const LayerPlan& lp = P.layers[l];
    const ActView in = layer_input(c, l, x);
    const double fl = 2.0 * B * lp.out * (double)lp.in * nl;
    if (lp.gemm) {
      gemm::Problem pb;
      pb.M = B; pb.N = lp.out; pb.K = lp.in; pb.batch = nl; pb.splits = 1; pb.passes = 3;
      pb.A = gemm::Operand{in.p, nullptr, true, false, lp.in, in.pst};
      pb.B = lp.wraw ? gemm::Operand{th + lp.off_w, nullptr, true, false, lp.in, ld}
                     : gemm::Operand{c->whi + lp.woff, c->wlo + lp.woff, false, false, lp.in, P.wsplit_total};
      pb.epi = gemm::EPI_FWD; pb.act = act;
      pb.out = c->act[l]; pb.ldo = lp.out; pb.out_pstride = P.act_pst[l];
      pb.bias = th + lp.off_b; pb.bias_pstride = ld;
      st = run_k(c, PC_FWD_GEMM, 1, 0, fl, s, [&] { return gemm::run(pb, s); });
    } else {
      st = run_k(c, PC_FWD_THIN, 1, 4.0 * B * lp.out * nl, fl, s, [&] {
        kern::thin_forward(in.p, in.pst, th, ld, lp.off_w, lp.off_b, lp.in, lp.out, act, c->act[l], P.act_pst[l], B,
                           nl, s);
        return PUSH_OK;
      });
    }
    if (st != PUSH_OK) return st;
  }

  // a3 (+ the top of a4/a5): output layer, residuals, per-particle loss, dW_L / db_L partials,
  // delta of the layer below and its bias partials, in one pass over A_{L-2}
  std::vector<char> bias_ready(L, 0);  // bias partials of layer l sit in bpart[l & 1]
  bool x0_ready = false;               // dW_0 partials sit in xpart
  {
    const LayerPlan& lp = P.layers[L - 1];
    const ActView in = layer_input(c, L - 1, x);
    kern::OutputArgs oa{};
    oa.A = in.p; oa.a_pstride = in.pst; oa.H = lp.in; oa.dout = lp.out; oa.B = B; oa.act = act;
    oa.theta = th; oa.ld = ld; oa.off_w = lp.off_w; oa.off_b = lp.off_b; oa.y = y;
    oa.err2 = c->err2; oa.err_pstride = P.Bmax;
    oa.wpart = c->opw; oa.wo_sstride = (int64_t)nl * lp.out * lp.in; oa.wo_pstride = (int64_t)lp.out * lp.in;
    oa.bpart_out = c->opb; oa.bo_sstride = (int64_t)nl * lp.out; oa.bo_pstride = lp.out;
    if (L >= 2) {
      oa.dprev = c->dlt[0]; oa.dp_pstride = P.dlt_pst;
      oa.bpart_prev = c->bpart[L - 2]; oa.bp_sstride = (int64_t)nl * lp.in; oa.bp_pstride = lp.in;
      bias_ready[L - 2] = 1;
    }
    const double bytes = 4.0 * B * lp.in * nl * (L >= 2 ? 2 : 1);
    st = run_k(c, PC_OUTPUT, 1, bytes, 2.0 * B * lp.out * (double)lp.in * nl * 3, s, [&] {
      kern::output_fused(oa, nl, s);
      return PUSH_OK;
    });
    if (st != PUSH_OK) return st;
    if ((st = side_fork()) != PUSH_OK) return st;  // the loss reduction is off the critical path
    st = run_k(c, PC_LOSS, 1, 0, 0, ws, [&] {
      kern::loss_reduce(c->err2, P.Bmax, c->loss, B, lp.out, nl, ws);
      return PUSH_OK;
    });
    if (st != PUSH_OK) return st;
    if ((st = side_done()) != PUSH_OK) return st;
    kern::PartView W{c->opw, RB, oa.wo_sstride, oa.wo_pstride, lp.in};
    kern::PartView Bv{c->opb, RB, oa.bo_sstride, oa.bo_pstride, 1};
    if ((st = finalize(L - 1, W, Bv)) != PUSH_OK) return st;
  }

  // a4/a5: backprop and weight gradients, layer by layer (delta_l in dlt[xb])
  int xb = 0;
  for (int l = L - 2; l >= 0; --l) {
    const LayerPlan& lp = P.layers[l];
    const float* dl = c->dlt[xb];
    const ActView ap = layer_input(c, l, x);
    if (lp.gemm) {
      // never more splits than the partial buffer was sized for at max_batch
      const int S = std::min(wgrad_splits(B, lp.out, lp.in, P.n), lp.wsplit_max);
      gemm::Problem pb;
      pb.M = lp.out; pb.N = lp.in; pb.K = B; pb.batch = nl; pb.splits = S; pb.passes = 3;
      pb.A = gemm::Operand{dl, nullptr, true, true, lp.out, P.dlt_pst};
      pb.B = gemm::Operand{ap.p, nullptr, true, true, lp.in, ap.pst};
      pb.epi = gemm::EPI_STORE;
      // one split: the epilogue writes -lambda dW straight into G's rows (no partial round trip)
      const bool w_in_g = wgrad_in_g((int)(lp.off_w % 4), lp.in, S);
      if (w_in_g) {
        pb.out = g + lp.off_w; pb.ldo = lp.in; pb.out_pstride = ld; pb.alpha = -lambda;
      } else {
        pb.out = c->wpart[l]; pb.ldo = lp.in; pb.out_pstride = (int64_t)lp.out * lp.in;
        pb.out_sstride = (int64_t)nl * lp.out * lp.in;
      }
      const double fl = 2.0 * B * lp.out * (double)lp.in * nl;
      // captured steps: the weight gradient of layer l (reads delta_l and A_{l-1}) beside the backward GEMM
      // of layer l (reads delta_l too); joined before delta_l's buffer is overwritten (layer l - 1)
      if ((st = side_join()) != PUSH_OK) return st;
      if ((st = side_fork()) != PUSH_OK) return st;
      st = run_k(c, PC_WGRAD_GEMM, 1, 0, fl, ws, [&] { return gemm::run(pb, ws); });
      if (st != PUSH_OK) return st;
      kern::PartView W{c->wpart[l], S, (int64_t)nl * lp.out * lp.in, (int64_t)lp.out * lp.in, lp.in};
      kern::PartView Bv{c->bpart[l], RB, (int64_t)nl * lp.out, lp.out, 1};
      if (!bias_ready[l]) {  // delta_l came from a generic thin backward: column sums here
        int chunks = 0;
        st = run_k(c, PC_WGRAD_THIN, 1, 4.0 * B * lp.out * nl, 0, ws, [&] {
          chunks = kern::thin_wgrad(dl, P.dlt_pst, nullptr, 0, 0, lp.out, c->tpart[l], B, nl, ws);
          return PUSH_OK;
        });
        if (st != PUSH_OK) return st;
        Bv = kern::PartView{c->tpart[l], chunks, (int64_t)nl * lp.out, lp.out, 1};
      }
      if ((st = side_done()) != PUSH_OK) return st;
      if ((st = finalize(l, W, Bv, w_in_g)) != PUSH_OK) return st;
    } else if (l == 0 && x0_ready) {
      kern::PartView W{c->xpart, RB, (int64_t)nl * lp.out * lp.in, (int64_t)lp.out * lp.in, lp.in};
      kern::PartView Bv{c->bpart[0], RB, (int64_t)nl * lp.out, lp.out, 1};
      if ((st = finalize(l, W, Bv)) != PUSH_OK) return st;
    } else {
      int chunks = 0;
      st = run_k(c, PC_WGRAD_THIN, 1, 4.0 * B * (lp.in + lp.out) * nl, 2.0 * B * lp.out * (double)(lp.in + 1) * nl,
                 s, [&] {
                   chunks = kern::thin_wgrad(dl, P.dlt_pst, ap.p, ap.pst, lp.in, lp.out, c->tpart[l], B, nl, s);
                   return PUSH_OK;
                 });
      if (st != PUSH_OK) return st;
      const int64_t cols = lp.in + 1;
      kern::PartView W{c->tpart[l], chunks, (int64_t)nl * lp.out * cols, (int64_t)lp.out * cols, cols};
      kern::PartView Bv{c->tpart[l] + lp.in, chunks, (int64_t)nl * lp.out * cols, (int64_t)lp.out * cols, cols};
      if ((st = finalize(l, W, Bv)) != PUSH_OK) return st;
    }
    if (l == 0) break;
    // delta_{l-1} = (delta_l W_l) * sigma'(a_{l-1}) overwrites delta_{l+1}: the side work reading it is done
    if ((st = side_join_prev()) != PUSH_OK) return st;
    const ActView aprev = layer_input(c, l, x);  // = A_{l-1}
    float* o = c->dlt[xb ^ 1];
    const double fl = 2.0 * B * lp.out * (double)lp.in * nl;
    if (lp.gemm) {
      gemm::Problem pb;
      pb.M = B; pb.N = lp.in; pb.K = lp.out; pb.batch = nl; pb.splits = 1; pb.passes = 3;
      pb.A = gemm::Operand{dl, nullptr, true, false, lp.out, P.dlt_pst};
      pb.B = lp.wraw ? gemm::Operand{th + lp.off_w, nullptr, true, true, lp.in, ld}
                     : gemm::Operand{c->whi + lp.woff, c->wlo + lp.woff, false, true, lp.in, P.wsplit_total};
      pb.epi = gemm::EPI_BWD; pb.act = act;
      pb.out = o; pb.ldo = lp.in; pb.out_pstride = P.dlt_pst;
      pb.aprev = aprev.p; pb.ld_aprev = lp.in; pb.aprev_pstride = aprev.pst;
      pb.bpart = c->bpart[l - 1]; pb.bp_sstride = (int64_t)nl * lp.in; pb.bp_pstride = lp.in;
      if (l == 1 && P.fuse_x0) {
        pb.x = x; pb.din = P.layers[0].in; pb.xpart = c->xpart;
        pb.out = nullptr;  // delta_0 only feeds the fused first-layer partials: never stored
        pb.xp_sstride = (int64_t)nl * lp.in * P.layers[0].in; pb.xp_pstride = (int64_t)lp.in * P.layers[0].in;
        x0_ready = true;
      }
      st = run_k(c, PC_BWD_GEMM, 1, 0, fl, s, [&] { return gemm::run(pb, s); });
      bias_ready[l - 1] = 1;
    } else {
      st = run_k(c, PC_BWD_THIN, 1, 8.0 * B * lp.in * nl, fl, s, [&] {
        kern::thin_backward(dl, P.dlt_pst, th, ld, lp.off_w, lp.in, lp.out, aprev.p, aprev.pst, act, o, P.dlt_pst, B,
                            nl, s);
        return PUSH_OK;
      });
      bias_ready[l - 1] = 0;
    }
    if (st != PUSH_OK) return st;
    xb ^= 1;
  }
  while (!side_ev.empty())
    if ((st = side_join()) != PUSH_OK) return st;
  return run_k(c, PC_FINALIZE, 1, 0, 0, s, [&] {
    kern::finalize_all(jobs.data(), (int)jobs.size(), th, g, ld, lambda, prior_g, inv_s2, nl, s);
    return PUSH_OK;
  });
}

// ------------------------------------------------------------------ step (a6-a10)
// ------------------------------------------------------------------ NEXT-4: d-sharded kernel phase
// (include/push.h PUSH_XCHG_DSHARD).  Rank q owns the columns [c_q, c_q + w_q)
// of every particle for a7-a10: three phases, each a collective step of the group.
//   1  transpose: own rows' Theta / G columns of rank q -> rows [r n_l, (r+1) n_l) of q's panels
//      (n x w_q, pitch w_q); the distance partials of q's whole splits over its panel
//   2  all-gather of the partials (rank blocks of smax n^2), the fixed-order reduction into D, h and K
//      of all n rows, the update of all n rows of the panel into pth2
//   3  transpose back: panel rows of rank r -> r's next Theta buffer, columns of q
// Every element sees the same splits, sums and update arithmetic as the all-gather path: results are
// bit-identical for every P.
// a10 on the tensor cores (P.tc_update): U = lhs B with lhs = [K, -rK] (g_first) or [-rK, K] (`rows` rows
// of K) and B = the 2n x w operand at `b` (pitch w, MN-major: [G; Theta] when g_first, else [Theta; G]),
// and out[i] = own[i] + eps_n (U_i + r s_i own[i]) written by the GEMM's EPI_UPD epilogue (pitch w).
static push_status update_tc(push_ctx* c, const float* b, bool g_first, int64_t w, int rows, const float* K,
                             const float* srow, const float* own, float* out, float eps_n, cudaStream_t s) {
  const Plan& P = c->P;
  if (w == 0) return PUSH_OK;
  const int pitch = (int)round_up(2 * P.n, 4);
  kern::update_lhs(K, rows, rows, P.n, pitch, c->h, g_first, c->ulhs, s);
  // U = [K, -rK] [G; Theta] with theta_i + (eps/n)(U_i + r s_i theta_i) in the GEMM epilogue (EPI_UPD: the
  // own theta tile is loaded beside the accumulator; the former fix-up pass's arithmetic, no U round trip)
  gemm::Problem pb;
  pb.M = rows; pb.N = (int)w; pb.K = 2 * P.n; pb.batch = 1; pb.splits = 1; pb.passes = 3;
  pb.A = gemm::Operand{c->ulhs, nullptr, true, false, pitch, 0};
  pb.B = gemm::Operand{b, nullptr, true, true, w, 0};
  pb.epi = gemm::EPI_UPD; pb.no_pair = true; pb.alpha = eps_n;
  pb.aprev = own; pb.ld_aprev = w; pb.aprev_pstride = (int64_t)rows * w;
  pb.srow = srow; pb.hptr = c->h;
  pb.out = out; pb.ldo = w; pb.out_pstride = (int64_t)rows * w;
  return gemm::run(pb, s);
}

// the d-sharded Theta panel of the current step (n x w at the own pitch; see Plan.o_pth)
static float* pan_theta(push_ctx* c) { return c->pbase + (c->cur ? 2 : 0) * (int64_t)c->P.n * c->ds_w; }

static push_status ds_phase1(push_ctx* c, cudaStream_t s) {
  const Plan& P = c->P;
  const int W = c->world, nl = P.nl;
  const int64_t ld = P.ld, wo = c->ds_w;
  push_status st = run_k(c, PC_EXCHANGE, 0, 8.0 * P.n * wo, 0, s, [&]() -> push_status {
    if (c->group || !c->comm) {  // loopback (or a single rank): pull the own columns from every row owner
      for (int q = 0; q < W && wo > 0; ++q) {
        push_ctx* pc = c->group ? c->group->members[q] : c;
        const int64_t src = (int64_t)q * nl * ld + c->ds_c;
        PUSH_CUDA_TRY(cudaMemcpy2DAsync(pan_theta(c) + (int64_t)q * nl * wo, wo * 4, pc->theta[c->cur] + src, ld * 4,
                                        wo * 4, nl, cudaMemcpyDeviceToDevice, s));
        PUSH_CUDA_TRY(cudaMemcpy2DAsync(c->pg + (int64_t)q * nl * wo, wo * 4, pc->grad + src, ld * 4, wo * 4, nl,
                                        cudaMemcpyDeviceToDevice, s));
      }
      return PUSH_OK;
    }
    const float* th = c->theta[c->cur] + (int64_t)c->row0 * ld;
    const float* g = c->grad + (int64_t)c->row0 * ld;
    for (int q = 0; q < W; ++q) {  // pack the own rows' columns of rank q (contiguous n_l x w_q blocks)
      const int64_t wq = P.ds_c0[q + 1] - P.ds_c0[q];
      if (wq == 0) continue;
      const int64_t dst = (int64_t)q * nl * P.ds_wmax;
      PUSH_CUDA_TRY(cudaMemcpy2DAsync(c->pack_th + dst, wq * 4, th + P.ds_c0[q], ld * 4, wq * 4, nl,
                                      cudaMemcpyDeviceToDevice, s));
      PUSH_CUDA_TRY(cudaMemcpy2DAsync(c->pack_g + dst, wq * 4, g + P.ds_c0[q], ld * 4, wq * 4, nl,
                                      cudaMemcpyDeviceToDevice, s));
    }
    push_status e = nccl::group_start();
    for (int q = 0; q < W && e == PUSH_OK; ++q) {
      const int64_t wq = P.ds_c0[q + 1] - P.ds_c0[q];
      const int64_t dst = (int64_t)q * nl * P.ds_wmax;
      if (wq > 0 && e == PUSH_OK) e = nccl::send_f32(c->pack_th + dst, nl * wq, q, c->comm, s);
      if (wq > 0 && e == PUSH_OK) e = nccl::send_f32(c->pack_g + dst, nl * wq, q, c->comm, s);
      if (wo > 0 && e == PUSH_OK) e = nccl::recv_f32(pan_theta(c) + (int64_t)q * nl * wo, nl * wo, q, c->comm, s);
      if (wo > 0 && e == PUSH_OK) e = nccl::recv_f32(c->pg + (int64_t)q * nl * wo, nl * wo, q, c->comm, s);
    }
    const push_status e2 = nccl::group_end();
    return e != PUSH_OK ? e : e2;
  });
  if (st != PUSH_OK || c->dist_own.splits == 0) return st;
  float* part = c->dpart + (int64_t)c->rank * P.ds_smax * part_block(P);
  if (P.gram)
    return run_k(c, PC_DIST, 1, 4.0 * P.n * wo, 2.0 * P.n * (double)P.n * wo, s, [&] {
      return kern::gram_partial(pan_theta(c), wo, P.n, c->dist_own.splits, c->dranges, part, s);
    });
  return run_k(c, PC_DIST, 1, 4.0 * P.n * wo, 3.0 * P.n * (double)P.n * wo / 2, s, [&] {
    kern::dist_partial(pan_theta(c), wo, P.n, c->dist_own, c->dranges, part, s);
    return PUSH_OK;
  });
}

static push_status ds_phase2(push_ctx* c, cudaStream_t s) {
  const Plan& P = c->P;
  const int W = c->world;
  const int64_t blk = (int64_t)P.ds_smax * part_block(P), wo = c->ds_w;
  push_status st = PUSH_OK;
  if (W > 1 || c->comm) {
    st = run_k(c, PC_EXCHANGE, 0, 4.0 * blk * (W - 1), 0, s, [&]() -> push_status {
      if (c->group) {
        for (int q = 0; q < W; ++q)
          if (q != c->rank)
            PUSH_CUDA_TRY(cudaMemcpyAsync(c->dpart + q * blk, c->group->members[q]->dpart + q * blk, blk * 4,
                                          cudaMemcpyDeviceToDevice, s));
        return PUSH_OK;
      }
      return nccl::allgather_f32(c->dpart + c->rank * blk, c->dpart, blk, c->comm, s);
    });
    if (st != PUSH_OK) return st;
  }
  st = run_k(c, PC_DIST, P.gram ? (kern::gram_d_in_bandwidth(P.n) ? 1 : 2) : 1, 4.0 * P.n * P.n * (double)P.dist.splits, 0, s, [&] {
    if (P.gram)
      kern::gram_dist(c->dpart, P.n, P.dist.splits, c->slots, c->gsum, c->D, s);
    else
      kern::dist_reduce(c->dpart, P.n, P.dist, c->slots, c->D, s);
    return PUSH_OK;
  });
  if (st != PUSH_OK) return st;
  st = run_k(c, PC_BANDWIDTH, (int64_t)P.n * P.n >= 16384 ? 2 : 1, 4.0 * P.n * P.n, 0, s, [&] {
    kern::bandwidth_kernel(c->D, P.n, 0, P.n, c->cfg.bw_rule, c->c_ln, c->cfg.bw_h, c->h, c->K, c->srow, 1, s,
                           P.gram && kern::gram_d_in_bandwidth(P.n) ? c->gsum : nullptr);
    return PUSH_OK;
  });
  if (st != PUSH_OK || wo == 0) return st;
  const float eps_n = c->cfg.step_size / (float)P.n;
  return run_k(c, PC_UPDATE, P.tc_update ? 2 : (P.tc_stream ? 2 : 1), 12.0 * P.n * (double)wo, 2.0 * P.n * (double)P.n * wo, s,
               [&]() -> push_status {
    float* pth = pan_theta(c);
    if (P.tc_stream) {  // every row of the panel; operand order as the all-gather path at this parity
      const int64_t half = (int64_t)kern::kUpdTcMaxRows * round_up(2 * P.n, 4);
      return kern::update_tc_stream(c->cur ? c->pg : pth, c->cur == 1, P.n, wo, P.n, 0, c->K, c->h, c->ulhs,
                                    c->ulhs + half, c->pth2, c->srow, eps_n, s);
    }
    if (P.tc_update)  // every row of the panel; [Theta; G] or [G; Theta] as the all-gather path at this parity
      return update_tc(c, c->cur ? c->pg : pth, c->cur == 1, wo, P.n, c->K, c->srow, pth, c->pth2, eps_n, s);
    kern::svgd_update(pth, c->pg, wo, P.n, 0, P.n, c->K, c->srow, c->h, eps_n, c->pth2, s);
    return PUSH_OK;
  });
}

static push_status ds_phase3(push_ctx* c, cudaStream_t s) {
  const Plan& P = c->P;
  const int W = c->world, nl = P.nl;
  const int64_t ld = P.ld, wo = c->ds_w;
  return run_k(c, PC_EXCHANGE, 0, 4.0 * P.n * wo, 0, s, [&]() -> push_status {
    if (c->group || !c->comm) {  // loopback: push the updated columns into every row owner's next buffer
      for (int q = 0; q < W && wo > 0; ++q) {
        push_ctx* pc = c->group ? c->group->members[q] : c;
        PUSH_CUDA_TRY(cudaMemcpy2DAsync(pc->theta[c->cur ^ 1] + (int64_t)q * nl * ld + c->ds_c, ld * 4,
                                        c->pth2 + (int64_t)q * nl * wo, wo * 4, wo * 4, nl, cudaMemcpyDeviceToDevice,
                                        s));
      }
      return PUSH_OK;
    }
    push_status e = nccl::group_start();
    for (int q = 0; q < W && e == PUSH_OK; ++q) {
      const int64_t wq = P.ds_c0[q + 1] - P.ds_c0[q];
      if (wo > 0 && e == PUSH_OK) e = nccl::send_f32(c->pth2 + (int64_t)q * nl * wo, nl * wo, q, c->comm, s);
      if (wq > 0 && e == PUSH_OK) e = nccl::recv_f32(c->pack_th + (int64_t)q * nl * P.ds_wmax, nl * wq, q, c->comm, s);
    }
    const push_status e2 = nccl::group_end();
    if (e != PUSH_OK || e2 != PUSH_OK) return e != PUSH_OK ? e : e2;
    float* nxt = c->theta[c->cur ^ 1] + (int64_t)c->row0 * ld;
    for (int q = 0; q < W; ++q) {  // unpack rank q's columns into the own rows
      const int64_t wq = P.ds_c0[q + 1] - P.ds_c0[q];
      if (wq == 0) continue;
      PUSH_CUDA_TRY(cudaMemcpy2DAsync(nxt + P.ds_c0[q], ld * 4, c->pack_th + (int64_t)q * nl * P.ds_wmax, wq * 4,
                                      wq * 4, nl, cudaMemcpyDeviceToDevice, s));
    }
    return PUSH_OK;
  });
}

// The whole group's d-sharded step on one stream (loopback groups: called by the last rank).
static push_status ds_group_step(const std::vector<push_ctx*>& m, cudaStream_t s) {
  push_status st;
  for (push_ctx* c : m)
    if ((st = ds_phase1(c, s)) != PUSH_OK) return st;
  for (push_ctx* c : m)
    if ((st = ds_phase2(c, s)) != PUSH_OK) return st;
  for (push_ctx* c : m)
    if ((st = ds_phase3(c, s)) != PUSH_OK) return st;
  for (push_ctx* c : m) c->cur ^= 1;
  return PUSH_OK;
}

// a7 (distances) + a8/a9 (bandwidth, K, s) of the current Theta on stream s (all-gather mode: Theta_all must
// be complete on s).  They read Theta only, so a captured whole step runs them beside the gradient phase.
static push_status run_kphase(push_ctx* c, cudaStream_t s) {
  const Plan& P = c->P;
  push_status st;
  const float* th = c->theta[c->cur];
  const double nd4 = 4.0 * P.n * (double)P.d;
  if (P.gram) {
    st = run_k(c, PC_DIST, kern::gram_d_in_bandwidth(P.n) ? 2 : 3, nd4, 2.0 * P.n * (double)P.n * P.ld, s, [&]() -> push_status {
      push_status g = kern::gram_partial(th, P.ld, P.n, P.dist.splits, c->dranges, c->dpart, s);
      if (g != PUSH_OK) return g;
      kern::gram_dist(c->dpart, P.n, P.dist.splits, c->slots, c->gsum, c->D, s);
      return PUSH_OK;
    });
  } else {
    st = run_k(c, PC_DIST, 2, nd4, 3.0 * P.n * (double)P.n * P.d / 2, s, [&] {
      kern::dist_partial(th, P.ld, P.n, P.dist, c->dranges, c->dpart, s);
      kern::dist_reduce(c->dpart, P.n, P.dist, c->slots, c->D, s);
      return PUSH_OK;
    });
  }
  if (st != PUSH_OK) return st;
  return run_k(c, PC_BANDWIDTH, (int64_t)P.nl * P.n >= 16384 ? 2 : 1, 4.0 * P.tensors * P.n * P.n, 0, s, [&] {
    kern::bandwidth_kernel(c->D, P.n, c->row0, P.nl, c->cfg.bw_rule, c->c_ln, c->cfg.bw_h, c->h, c->K, c->srow,
                           P.tensors, s, P.gram && kern::gram_d_in_bandwidth(P.n) ? c->gsum : nullptr);
    return PUSH_OK;
  });
}

static push_status do_step(push_ctx* c, cudaStream_t s) {
  const Plan& P = c->P;
  push_status st;
  if (P.ds) return ds_group_step({c}, s);  // NCCL ranks (or one rank): three collective phases
  if ((st = join_theta(c, s)) != PUSH_OK) return st;  // the Theta all-gather started by the gradient call
  // C2: g rows of every rank, on the comm stream while a7-a9 (which read Theta only) run; joined before a10
  const bool xg = c->world > 1 || c->comm;
  if (xg) {
    PUSH_CUDA_TRY(cudaEventRecord(c->ev_fork2, s));
    PUSH_CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, c->ev_fork2, 0));
    if ((st = exchange(c, BUF_GRAD, c->comm_stream)) != PUSH_OK) return st;
    PUSH_CUDA_TRY(cudaEventRecord(c->ev_grad, c->comm_stream));
  }
  const float* th = c->theta[c->cur];
  const double nd4 = 4.0 * P.n * (double)P.d;
  if (c->kphase_ready) {  // a7-a9 ran on k_stream beside the gradient phase (captured whole step)
    PUSH_CUDA_TRY(cudaStreamWaitEvent(s, c->ev_kdone, 0));
    c->kphase_ready = false;
  } else if ((st = run_kphase(c, s)) != PUSH_OK) {
    return st;
  }
  if (xg) PUSH_CUDA_TRY(cudaStreamWaitEvent(s, c->ev_grad, 0));  // G rows of every rank have landed
  const float eps_n = c->cfg.step_size / (float)P.n;
  float* next = c->theta[c->cur ^ 1];
  const int var = c->cfg.variant;
  st = run_k(c, PC_UPDATE, (var == 0 && P.tc_update) ? 2 : ((var == 0 && P.tc_stream) ? 2 : 1), 2.0 * nd4 + 4.0 * P.nl * (double)P.d,
             2.0 * P.nl * (double)P.n * P.d, s, [&] {
    if (var == 0 && P.tc_stream) {
      const bool g_first = c->grad < th;  // layout Theta[0], G, Theta[1]
      const int64_t half = (int64_t)kern::kUpdTcMaxRows * round_up(2 * P.n, 4);
      return kern::update_tc_stream(g_first ? c->grad : th, g_first, P.n, P.ld, P.nl, c->row0, c->K, c->h, c->ulhs,
                                    c->ulhs + half, next + (int64_t)c->row0 * P.ld, c->srow, eps_n, s);
    } else if (var == 0 && P.tc_update) {
      // layout Theta[0], G, Theta[1]: [G; Theta_cur] or [Theta_cur; G] is one 2n x ld operand
      const bool g_first = c->grad < th;
      return update_tc(c, g_first ? c->grad : th, g_first, P.ld, P.nl, c->K, c->srow,
                       th + (int64_t)c->row0 * P.ld, next + (int64_t)c->row0 * P.ld, eps_n, s);
    } else if (var == 0) {
      kern::svgd_update(th, c->grad, P.ld, P.n, c->row0, P.nl, c->K, c->srow, c->h, eps_n, next, s);
    } else {  // NEXT-2 (include/push.h PUSH_VAR_*): weights w_d = eps or eps/n, repulsion eps/n
      const bool pn = var & PUSH_VAR_PAPER_NORM;
      const float eps_d = pn ? c->cfg.step_size : eps_n;
      const float alpha = pn ? (float)(1.0 / P.n) : 1.0f;
      const float pcoef = (var & PUSH_VAR_PRIOR_SUM) && c->cfg.prior == PUSH_PRIOR_GAUSSIAN
                              ? (float)(-1.0 / ((double)c->cfg.prior_sigma * c->cfg.prior_sigma))
                              : 0.f;
      kern::svgd_update_var(th, c->grad, P.ld, P.n, c->row0, P.nl, c->K, c->srow, c->h, c->useg, (int)P.useg.size(),
                            alpha, eps_d, pcoef, next, s);
    }
    return PUSH_OK;
  });
  if (st != PUSH_OK) return st;
  c->cur ^= 1;
  return PUSH_OK;
}

// ------------------------------------------------------------------ predictive pushforward (NEXT-1)
// ppush(mu)(g(x; .)) = {g(x; theta_i)}: every particle's forward on x, all-gathered
// to every rank, then the cross-particle mean and population standard deviation per output.
static push_status do_predict(push_ctx* c, const float* x, int B, cudaStream_t s) {
  const Plan& P = c->P;
  const int nl = P.nl, L = P.L, act = c->cfg.activation;
  const int64_t ld = P.ld;
  const float* th = c->theta[c->cur] + (int64_t)c->row0 * ld;
  push_status st;
  for (int l = 0; l + 1 < L; ++l) {
    const LayerPlan& lp = P.layers[l];
    const ActView in = layer_input(c, l, x);
    const double fl = 2.0 * B * lp.out * (double)lp.in * nl;
    if (lp.gemm) {
      gemm::Problem pb;
      pb.M = B; pb.N = lp.out; pb.K = lp.in; pb.batch = nl; pb.splits = 1; pb.passes = 3;
      pb.A = gemm::Operand{in.p, nullptr, true, false, lp.in, in.pst};
      pb.B = lp.wraw ? gemm::Operand{th + lp.off_w, nullptr, true, false, lp.in, ld}
                     : gemm::Operand{c->whi + lp.woff, c->wlo + lp.woff, false, false, lp.in, P.wsplit_total};
      if (!lp.wraw) {
        const int64_t cnt = (int64_t)lp.in * lp.out;
        st = run_k(c, PC_SPLIT, 1, 12.0 * cnt * nl, 0, s, [&] {
          kern::split_hilo(th + lp.off_w, ld, c->whi + lp.woff, c->wlo + lp.woff, P.wsplit_total, cnt, nl, s);
          return PUSH_OK;
        });
        if (st != PUSH_OK) return st;
      }
      pb.epi = gemm::EPI_FWD; pb.act = act;
      pb.out = c->act[l]; pb.ldo = lp.out; pb.out_pstride = P.act_pst[l];
      pb.bias = th + lp.off_b; pb.bias_pstride = ld;
      st = run_k(c, PC_FWD_GEMM, 1, 0, fl, s, [&] { return gemm::run(pb, s); });
    } else {
      st = run_k(c, PC_FWD_THIN, 1, 4.0 * B * lp.out * nl, fl, s, [&] {
        kern::thin_forward(in.p, in.pst, th, ld, lp.off_w, lp.off_b, lp.in, lp.out, act, c->act[l], P.act_pst[l], B,
                           nl, s);
        return PUSH_OK;
      });
    }
    if (st != PUSH_OK) return st;
  }
  const LayerPlan& top = P.layers[L - 1];
  const ActView in = layer_input(c, L - 1, x);
  c->pred_B = B;
  float* own = c->pred + (size_t)c->row0 * B * top.out;
  st = run_k(c, PC_OUTPUT, 1, 4.0 * B * top.in * nl, 2.0 * B * top.out * (double)top.in * nl, s, [&] {
    kern::output_forward(in.p, in.pst, th, ld, top.off_w, top.off_b, top.in, top.out, own, B, nl, s);
    return PUSH_OK;
  });
  if (st != PUSH_OK) return st;
  return exchange(c, BUF_PRED, s);
}

static push_status check_ctx(push_ctx* c) {
  if (!c) return fail(PUSH_E_INVALID, "ctx is NULL");
  if (c->broken) return fail(PUSH_E_STATE, "context is in a failed state after an earlier CUDA/NCCL error");
  cudaSetDevice(c->device);
  if (c->comm) {  // a failed or aborted peer surfaces here (re-raised at the next call)
    push_status st = nccl::async_error(c->comm);
    if (st != PUSH_OK) {
      c->broken = true;
      return st;
    }
  }
  return PUSH_OK;
}

// Host wait on `s` that polls the NCCL communicator while it waits: a dead or failed peer would otherwise
// block cudaStreamSynchronize forever.  On an asynchronous NCCL error, or after kSyncTimeoutS without
// progress, the communicator is aborted (its kernels are released) and the context turns broken.
constexpr double kSyncTimeoutS = 600.0;
static push_status wait_stream(push_ctx* c, cudaStream_t s) {
  if (!c->comm) {
    PUSH_CUDA_TRY(cudaStreamSynchronize(s));
    return PUSH_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return PUSH_OK;
    if (q != cudaErrorNotReady) return fail(PUSH_E_CUDA, std::string("stream: ") + cudaGetErrorString(q));
    push_status st = nccl::async_error(c->comm);
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (st == PUSH_OK && dt > kSyncTimeoutS)
      st = fail(PUSH_E_NCCL, "no progress for " + std::to_string((int)kSyncTimeoutS) + " s (peer lost?)");
    if (st != PUSH_OK) {
      c->broken = true;
      nccl::comm_release(c->comm, true);  // ncclCommAbort: unblocks the pending collectives
      c->comm = nullptr;
      return st;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

static push_status init_one(push_ctx* c, const push_config* cfg, int rank, int world, void* ws, size_t ws_bytes,
                            const float* theta0_host) {
  push_status st = make_plan(cfg, world, &c->P);
  if (st != PUSH_OK) return st;
  if (rank < 0 || rank >= world) return fail(PUSH_E_INVALID, "rank out of range");
  if (!ws) return fail(PUSH_E_INVALID, "dev_workspace is NULL");
  if (reinterpret_cast<uintptr_t>(ws) % 256) return fail(PUSH_E_INVALID, "dev_workspace must be 256-byte aligned");
  if (ws_bytes < c->P.total) return fail(PUSH_E_SHAPE, "workspace too small: need " + std::to_string(c->P.total));
  int dev = 0;
  PUSH_CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  PUSH_CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) return fail(PUSH_E_UNSUPPORTED, "libpush_b200 needs an sm_100 (B200) device");
  c->cfg = *cfg;
  c->rank = rank;
  c->world = world;
  c->row0 = rank * c->P.nl;
  c->device = dev;
  c->ws = static_cast<uint8_t*>(ws);
  const Plan& P = c->P;
  auto F = [&](size_t o) { return reinterpret_cast<float*>(c->ws + o); };
  c->ulhs = F(P.o_ulhs);
  c->theta[0] = F(P.o_theta0);
  c->theta[1] = F(P.o_theta1);
  c->grad = F(P.o_grad);
  c->whi = F(P.o_whi);
  c->wlo = F(P.o_wlo);
  for (size_t l = 0; l < P.o_act.size(); ++l) c->act.push_back(F(P.o_act[l]));
  c->dlt[0] = F(P.o_dlt0);
  c->dlt[1] = F(P.o_dlt1);
  for (int l = 0; l < P.L; ++l) {
    c->wpart.push_back(P.o_wpart[l] == SIZE_MAX ? nullptr : F(P.o_wpart[l]));
    c->tpart.push_back(F(P.o_tpart[l]));
    c->bpart.push_back(F(P.o_bpart[l]));
  }
  c->opw = F(P.o_opw);
  c->opb = F(P.o_opb);
  c->xpart = F(P.o_xpart);
  c->err2 = F(P.o_err2);
  c->loss = F(P.o_loss);
  c->loss_all = F(P.o_loss_all);
  c->dpart = F(P.o_dpart);
  c->D = F(P.o_D);
  c->gsum = F(P.o_gsum);
  c->K = F(P.o_K);
  c->srow = F(P.o_s);
  c->h = F(P.o_h);
  c->dranges = reinterpret_cast<int64_t*>(c->ws + P.o_dranges);
  c->useg = reinterpret_cast<int4*>(c->ws + P.o_useg);
  c->pbase = F(P.o_pth);
  c->pth2 = F(P.o_pth2);
  c->pack_th = F(P.o_pack_th);
  c->pack_g = F(P.o_pack_g);
  c->dist_own = P.dist;
  c->slots.P = 1;
  c->slots.smax = P.dist.splits;
  c->slots.s0[0] = 0;
  c->slots.s0[1] = P.dist.splits;
  if (P.ds) {  // own splits, column ranges relative to the panel start
    const int s0 = P.ds_s0[rank], s1 = P.ds_s0[rank + 1];
    c->ds_c = P.ds_c0[rank];
    c->ds_w = P.ds_c0[rank + 1] - P.ds_c0[rank];
    c->pg = c->pbase + (int64_t)P.n * c->ds_w;
    c->dist_own.splits = s1 - s0;
    c->dist_own.ranges.clear();
    for (int k = 2 * s0; k < 2 * s1; ++k) c->dist_own.ranges.push_back(P.dist.ranges[k] - c->ds_c);
    c->slots.P = world;
    c->slots.smax = P.ds_smax;
    for (int q = 0; q <= world; ++q) c->slots.s0[q] = P.ds_s0[q];
  }
  c->xbuf = F(P.o_xbuf);
  c->ybuf = F(P.o_ybuf);
  c->pred = F(P.o_pred);
  if (cfg->swag) {
    c->swag_mean = F(P.o_swag_mean);
    c->swag_sq = F(P.o_swag_sq);
  }
  // bandwidth constant c_n = fp32(1/ln n) or fp32(1/ln(n+1)), computed once in double (R4)
  if (cfg->bw_rule == PUSH_BW_MEDIAN_LN_N)
    c->c_ln = P.n > 1 ? (float)(1.0 / std::log((double)P.n)) : 1.f;
  else if (cfg->bw_rule == PUSH_BW_MEDIAN_LN_N1)
    c->c_ln = (float)(1.0 / std::log((double)P.n + 1.0));

  PUSH_CUDA_TRY(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
  PUSH_CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  PUSH_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  PUSH_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_theta, cudaEventDisableTiming));
  PUSH_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork2, cudaEventDisableTiming));
  PUSH_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_grad, cudaEventDisableTiming));
  PUSH_CUDA_TRY(cudaStreamCreateWithFlags(&c->k_stream, cudaStreamNonBlocking));
  PUSH_CUDA_TRY(cudaStreamCreateWithFlags(&c->w_stream, cudaStreamNonBlocking));
  PUSH_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_kfork, cudaEventDisableTiming));
  PUSH_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_kdone, cudaEventDisableTiming));
  cudaStream_t s = nullptr;
  const size_t nld = (size_t)P.n * P.ld;
  PUSH_CUDA_TRY(cudaMemsetAsync(c->theta[0], 0, nld * 4, s));
  PUSH_CUDA_TRY(cudaMemsetAsync(c->theta[1], 0, nld * 4, s));
  PUSH_CUDA_TRY(cudaMemsetAsync(c->grad, 0, nld * 4, s));
  if (!c->dist_own.ranges.empty())
    PUSH_CUDA_TRY(cudaMemcpyAsync(c->dranges, c->dist_own.ranges.data(), c->dist_own.ranges.size() * 8,
                                  cudaMemcpyHostToDevice, s));
  if (!P.useg.empty())
    PUSH_CUDA_TRY(cudaMemcpyAsync(c->useg, P.useg.data(), P.useg.size() * sizeof(int4), cudaMemcpyHostToDevice, s));
  if (theta0_host) {
    PUSH_CUDA_TRY(cudaMemcpy2DAsync(c->theta[0], P.ld * 4, theta0_host, P.d * 4, P.d * 4, P.n,
                                    cudaMemcpyHostToDevice, s));
  } else {
    kern::InitTable t{};
    t.n_layers = P.L;
    for (int l = 0; l < P.L; ++l) {
      t.off[l] = P.layers[l].off_w;
      t.bound[l] = (float)(1.0 / std::sqrt((double)P.layers[l].in));
    }
    t.off[P.L] = P.d;
    st = run_k(c, PC_INIT, 1, 4.0 * nld, 0, s, [&] {
      kern::init_theta(c->theta[0], P.ld, 0, P.n, P.d, cfg->seed, t, s);
      return PUSH_OK;
    });
    if (st != PUSH_OK) return st;
  }
  PUSH_CUDA_TRY(cudaStreamSynchronize(s));
  return PUSH_OK;
}

}  // namespace push

static bool force_nccl() {
  static const int v = [] {
    const char* e = getenv("PUSH_FORCE_NCCL");
    return e && *e && *e != '0' ? 1 : 0;
  }();
  return v != 0;
}

using namespace push;

// ================================================================== C ABI
extern "C" {

const char* push_version(void) {
  return "libpush_b200 abi=1 sm_100a (tcgen05 3xTF32 GEMM, radix-select median, fused SVGD update)";
}

const char* push_last_error(void) { return push::t_err.c_str(); }

push_status push_get_unique_id(uint8_t id[128]) {
  if (!id) return fail(PUSH_E_INVALID, "id is NULL");
  nccl::UniqueId u;
  push_status st = nccl::get_unique_id(&u);
  if (st != PUSH_OK) return st;
  std::memcpy(id, u.internal, 128);
  return PUSH_OK;
}

push_status push_workspace_size(const push_config* cfg, int32_t world_size, size_t* bytes) {
  if (!bytes) return fail(PUSH_E_INVALID, "bytes is NULL");
  Plan P;
  push_status st = make_plan(cfg, world_size, &P);
  if (st != PUSH_OK) return st;
  *bytes = P.total;
  return PUSH_OK;
}

push_status push_init(const push_config* cfg, int32_t rank, int32_t world_size, const uint8_t* nccl_id,
                      void* dev_workspace, size_t ws_bytes, const float* theta0_host, push_ctx** out) {
  if (!out) return fail(PUSH_E_INVALID, "out is NULL");
  *out = nullptr;
  if (world_size > 1 && !nccl_id) return fail(PUSH_E_INVALID, "nccl_id required when world_size > 1");
  push_ctx* c = new (std::nothrow) push_ctx();
  if (!c) return fail(PUSH_E_NOMEM, "out of host memory");
  push_status st = init_one(c, cfg, rank, world_size, dev_workspace, ws_bytes, theta0_host);
  if (st == PUSH_OK && world_size > 1) {
    nccl::UniqueId u;
    std::memcpy(u.internal, nccl_id, 128);
    st = nccl::comm_init_rank(&c->comm, world_size, u, rank, kNcclMaxCtas);
    int cnt = 0;
    if (st == PUSH_OK) st = nccl::comm_count(c->comm, &cnt);
    if (st == PUSH_OK && cnt != world_size)
      st = fail(PUSH_E_NCCL, "NCCL communicator has " + std::to_string(cnt) + " ranks, expected " +
                                 std::to_string(world_size));
    if (st == PUSH_OK)
      fprintf(stderr, "libpush_b200: NCCL communicator rank %d of %d (nranks %d, maxCTAs %d, device %d)\n", rank,
              world_size, cnt, kNcclMaxCtas, c->device);
    if (st != PUSH_OK && c->comm) nccl::comm_release(c->comm, true), c->comm = nullptr;
  } else if (st == PUSH_OK && force_nccl()) {
    // test hook (PUSH_FORCE_NCCL=1): a single-rank NCCL communicator, so that one GPU exercises the
    // NCCL exchange path (comm stream, in-place all-gathers, graph capture of NCCL calls)
    nccl::UniqueId u;
    st = nccl::get_unique_id(&u);
    if (st == PUSH_OK) st = nccl::comm_init_rank(&c->comm, 1, u, 0);
  }
  if (st != PUSH_OK) {
    delete c;
    return st;
  }
  *out = c;
  return PUSH_OK;
}

push_status push_init_local_group(const push_config* cfg, int32_t world_size, void* const* dev_workspaces,
                                  size_t ws_bytes, const float* theta0_host, push_ctx** out_ctxs) {
  if (!out_ctxs || !dev_workspaces) return fail(PUSH_E_INVALID, "NULL argument");
  if (world_size < 1) return fail(PUSH_E_INVALID, "world_size must be >= 1");
  auto grp = std::make_shared<LocalGroup>();
  for (int r = 0; r < world_size; ++r) out_ctxs[r] = nullptr;
  for (int r = 0; r < world_size; ++r) {
    push_ctx* c = new (std::nothrow) push_ctx();
    if (!c) return fail(PUSH_E_NOMEM, "out of host memory");
    push_status st = init_one(c, cfg, r, world_size, dev_workspaces[r], ws_bytes, theta0_host);
    if (st != PUSH_OK) {
      delete c;
      for (int q = 0; q < r; ++q) {
        delete out_ctxs[q];
        out_ctxs[q] = nullptr;
      }
      return st;
    }
    c->group = grp;
    grp->members.push_back(c);
    out_ctxs[r] = c;
  }
  return PUSH_OK;
}

push_status push_particle_grads(push_ctx* c, const float* x_dev, const float* y_dev, int32_t B, float* loss_dev,
                                void* stream) {
  push_status st = check_ctx(c);
  if (st != PUSH_OK) return st;
  if (!x_dev || !y_dev) return fail(PUSH_E_INVALID, "x_dev / y_dev is NULL");
  if (B < 1 || B > c->P.Bmax) return fail(PUSH_E_SHAPE, "B must be in [1, max_batch] (SPEC.md:55)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  st = do_grads(c, x_dev, y_dev, B, s);
  if (st == PUSH_OK && loss_dev) {
    st = run_k(c, PC_COPY, 0, 8.0 * c->P.nl, 0, s, [&]() -> push_status {
      PUSH_CUDA_TRY(cudaMemcpyAsync(loss_dev, c->loss, 4 * c->P.nl, cudaMemcpyDeviceToDevice, s));
      return PUSH_OK;
    });
  }
  if (st != PUSH_OK) return sticky(c, st);
  c->state = 1;
  c->has_grads = true;
  return PUSH_OK;
}

push_status push_set_grads(push_ctx* c, const float* g_dev, void* stream) {
  push_status st = check_ctx(c);
  if (st != PUSH_OK) return st;
  if (!g_dev) return fail(PUSH_E_INVALID, "g_dev is NULL");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  st = join_theta(c, s);
  if (st == PUSH_OK) st = exchange(c, BUF_THETA, s);
  if (st == PUSH_OK)
    st = run_k(c, PC_COPY, 1, 8.0 * c->P.nl * c->P.d, 0, s, [&] {
      kern::copy_rows(g_dev, c->P.d, c->grad + (int64_t)c->row0 * c->P.ld, c->P.ld, c->P.nl, s);
      return PUSH_OK;
    });
  if (st != PUSH_OK) return sticky(c, st);
  c->state = 1;
  c->has_grads = true;
  return PUSH_OK;
}

push_status push_svgd_step(push_ctx* c, void* stream) {
  push_status st = check_ctx(c);
  if (st != PUSH_OK) return st;
  if (c->state != 1) return fail(PUSH_E_STATE, "svgd_step needs fresh gradients (SPEC.md:350)");
  if (c->P.ds && c->group) {  // loopback d-sharding: the last rank's call runs every member's phases
    const auto& m = c->group->members;
    if (c->rank + 1 < c->world) {
      c->ds_deferred = true;
    } else {
      for (push_ctx* pc : m)
        if (pc != c && (!pc->ds_deferred || pc->state != 1))
          return fail(PUSH_E_STATE, "loopback d-sharded step: ranks 0..P-2 must call svgd_step first");
      st = ds_group_step(m, static_cast<cudaStream_t>(stream));
      if (st != PUSH_OK) return sticky(c, st);
      for (push_ctx* pc : m) {
        pc->ds_deferred = false;
        pc->state = 0;
        pc->has_step = true;
      }
    }
    return PUSH_OK;
  }
  st = do_step(c, static_cast<cudaStream_t>(stream));
  if (st != PUSH_OK) return sticky(c, st);
  c->state = 0;
  c->has_step = true;
  return PUSH_OK;
}

static bool graphs_disabled() {
  static const int v = [] {
    const char* e = getenv("PUSH_NO_GRAPH");
    return e && *e && *e != '0' ? 1 : 0;
  }();
  return v != 0;
}

push_status push_step_graph(push_ctx* c, const float* x_dev, const float* y_dev, int32_t B, float* loss_dev,
                            void* stream) {
  push_status st = check_ctx(c);
  if (st != PUSH_OK) return st;
  if (!x_dev || !y_dev) return fail(PUSH_E_INVALID, "x_dev / y_dev is NULL");
  if (B < 1 || B > c->P.Bmax) return fail(PUSH_E_SHAPE, "B must be in [1, max_batch] (SPEC.md:55)");
  if (c->group && c->world > 1)
    return fail(PUSH_E_STATE, "whole-step calls need every rank's gradients first: use the lockstep calls in a local group");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = join_theta(c, s)) != PUSH_OK) return sticky(c, st);
  const int din = c->P.layers[0].in, dout = c->P.layers[c->P.L - 1].out;
  // the captured step always reads the context's fixed batch buffers
  auto stage = [&]() -> push_status {
    if (x_dev != c->xbuf) PUSH_CUDA_TRY(cudaMemcpyAsync(c->xbuf, x_dev, (size_t)B * din * 4, cudaMemcpyDeviceToDevice, s));
    if (y_dev != c->ybuf) PUSH_CUDA_TRY(cudaMemcpyAsync(c->ybuf, y_dev, (size_t)B * dout * 4, cudaMemcpyDeviceToDevice, s));
    return PUSH_OK;
  };
  if ((st = stage()) != PUSH_OK) return sticky(c, st);
  if (c->prof_on || graphs_disabled() || !c->graph_warm) {
    // eager path (profiling, PUSH_NO_GRAPH=1, or the first call, which also initialises every
    // kernel's one-time attributes so that the capture below records stream work only)
    if ((st = push_particle_grads(c, c->xbuf, c->ybuf, B, loss_dev, stream)) != PUSH_OK) return st;
    if ((st = push_svgd_step(c, stream)) != PUSH_OK) return st;
    c->graph_warm = true;
    return PUSH_OK;
  }
  push_ctx::GraphEntry& g = c->graphs[c->cur];
  if (!g.exec || g.B != B || g.loss != loss_dev) {
    if (g.exec) {
      cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
    }
    const int cur0 = c->cur;
    const int64_t l0 = c->launches;
    cudaGraph_t graph = nullptr;
    PUSH_CUDA_TRY(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    st = do_grads(c, c->xbuf, c->ybuf, B, c->cap_stream, /*fork_kphase=*/true);
    if (st == PUSH_OK && loss_dev) {
      cudaError_t e = cudaMemcpyAsync(loss_dev, c->loss, 4 * c->P.nl, cudaMemcpyDeviceToDevice, c->cap_stream);
      if (e != cudaSuccess) st = fail(PUSH_E_CUDA, cudaGetErrorString(e));
    }
    if (st == PUSH_OK) st = do_step(c, c->cap_stream);
    cudaError_t e = cudaStreamEndCapture(c->cap_stream, &graph);
    c->cur = cur0;  // capturing executed nothing
    c->theta_pending = false;
    c->kphase_ready = false;
    if (st != PUSH_OK || e != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      return sticky(c, st != PUSH_OK ? st : fail(PUSH_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e)));
    }
    e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return sticky(c, fail(PUSH_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e)));
    g.kernels = c->launches - l0;
    c->launches = l0;
    g.B = B;
    g.loss = loss_dev;
  }
  cudaError_t e = cudaGraphLaunch(g.exec, s);
  if (e != cudaSuccess) return sticky(c, fail(PUSH_E_CUDA, std::string("graph launch: ") + cudaGetErrorString(e)));
  c->launches += g.kernels;
  c->cur ^= 1;
  c->state = 0;
  c->has_grads = c->has_step = true;
  return PUSH_OK;
}

push_status push_step_host(push_ctx* c, const float* x_host, const float* y_host, int32_t B, float* loss_host,
                           void* stream) {
  push_status st = check_ctx(c);
  if (st != PUSH_OK) return st;
  if (!x_host || !y_host) return fail(PUSH_E_INVALID, "x_host / y_host is NULL");
  if (B < 1 || B > c->P.Bmax) return fail(PUSH_E_SHAPE, "B must be in [1, max_batch]");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int din = c->P.layers[0].in, dout = c->P.layers[c->P.L - 1].out;
  auto copy_in = [&]() -> push_status {
    PUSH_CUDA_TRY(cudaMemcpyAsync(c->xbuf, x_host, (size_t)B * din * 4, cudaMemcpyHostToDevice, s));
    PUSH_CUDA_TRY(cudaMemcpyAsync(c->ybuf, y_host, (size_t)B * dout * 4, cudaMemcpyHostToDevice, s));
    return PUSH_OK;
  };
  if ((st = copy_in()) != PUSH_OK) return sticky(c, st);
  if ((st = push_step_graph(c, c->xbuf, c->ybuf, B, nullptr, stream)) != PUSH_OK) return st;
  if (loss_host) {
    cudaError_t e = cudaMemcpyAsync(loss_host, c->loss, 4 * c->P.nl, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return sticky(c, fail(PUSH_E_CUDA, cudaGetErrorString(e)));
  }
  return sticky(c, wait_stream(c, s));
}

push_status push_predict(push_ctx* c, const float* x_dev, int32_t B, float* pred_dev, float* mean_dev, float* std_dev,
                         void* stream) {
  push_status st = check_ctx(c);
  if (st != PUSH_OK) return st;
  if (!x_dev) return fail(PUSH_E_INVALID, "x_dev is NULL");
  if (B < 1 || B > c->P.Bmax) return fail(PUSH_E_SHAPE, "B must be in [1, max_batch] (SPEC.md:55)");
  if (c->group && c->world > 1)
    return fail(PUSH_E_STATE, "push_predict gathers every rank's predictions: not available in a loopback group");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = join_theta(c, s)) != PUSH_OK) return sticky(c, st);
  if ((st = do_predict(c, x_dev, B, s)) != PUSH_OK) return sticky(c, st);
  const int dout = c->P.layers[c->P.L - 1].out;
  const size_t per = (size_t)B * dout;
  if (mean_dev || std_dev) {
    st = run_k(c, PC_OUTPUT, 1, 4.0 * c->P.n * per, 0, s, [&] {
      kern::predict_stats(c->pred, c->P.n, (int64_t)per, mean_dev, std_dev, s);
      return PUSH_OK;
    });
    if (st != PUSH_OK) return sticky(c, st);
  }
  if (pred_dev) {
    cudaError_t e = cudaMemcpyAsync(pred_dev, c->pred, 4 * per * c->P.n, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return sticky(c, fail(PUSH_E_CUDA, cudaGetErrorString(e)));
  }
  return PUSH_OK;
}

push_status push_ensemble_step(push_ctx* c, void* stream) {
  push_status st = check_ctx(c);
  if (st != PUSH_OK) return st;
  if (c->state != 1) return fail(PUSH_E_STATE, "ensemble_step needs fresh gradients");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = join_theta(c, s)) != PUSH_OK) return sticky(c, st);  // the gradient call's Theta all-gather
  const Plan& P = c->P;
  float* th = c->theta[c->cur] + (int64_t)c->row0 * P.ld;
  const float* g = c->grad + (int64_t)c->row0 * P.ld;
  st = run_k(c, PC_UPDATE, 1, 12.0 * P.nl * (double)P.d, 2.0 * P.nl * (double)P.d, s, [&] {
    kern::ensemble_step(th, g, P.ld, P.nl, c->cfg.step_size, s);
    return PUSH_OK;
  });
  if (st != PUSH_OK) return sticky(c, st);
  c->state = 0;
  return PUSH_OK;
}

push_status push_swag_collect(push_ctx* c, void* stream) {
  push_status st = check_ctx(c);
  if (st != PUSH_OK) return st;
  if (!c->swag_mean) return fail(PUSH_E_STATE, "SWAG buffers not allocated (cfg.swag = 0)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Plan& P = c->P;
  const float* th = c->theta[c->cur] + (int64_t)c->row0 * P.ld;
  const int64_t k = c->swag_count;
  st = run_k(c, PC_UPDATE, 1, 20.0 * P.nl * (double)P.ld, 0, s, [&] {
    kern::swag_collect(th, c->swag_mean, c->swag_sq, (int64_t)P.nl * P.ld, k, s);
    return PUSH_OK;
  });
  if (st != PUSH_OK) return sticky(c, st);
  c->swag_count = k + 1;
  return PUSH_OK;
}

push_status push_swag_sample(push_ctx* c, uint64_t seed, float* out_dev, void* stream) {
  push_status st = check_ctx(c);
  if (st != PUSH_OK) return st;
  if (!out_dev) return fail(PUSH_E_INVALID, "out_dev is NULL");
  if (!c->swag_mean) return fail(PUSH_E_STATE, "SWAG buffers not allocated (cfg.swag = 0)");
  if (c->swag_count < 1) return fail(PUSH_E_STATE, "no SWAG moments collected yet");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Plan& P = c->P;
  st = run_k(c, PC_UPDATE, 1, 12.0 * P.nl * (double)P.d, 0, s, [&] {
    kern::swag_sample(c->swag_mean, c->swag_sq, P.ld, P.d, c->row0, P.nl, seed, out_dev, s);
    return PUSH_OK;
  });
  return st == PUSH_OK ? PUSH_OK : sticky(c, st);
}

push_status push_gather(push_ctx* c, int32_t what, float* out_host, void* stream) {
  push_status st = check_ctx(c);
  if (st != PUSH_OK) return st;
  if (!out_host) return fail(PUSH_E_INVALID, "out_host is NULL");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = join_theta(c, s)) != PUSH_OK) return sticky(c, st);
  const Plan& P = c->P;
  auto sync = [&]() -> push_status { return wait_stream(c, s); };
  switch (what) {
    case PUSH_WHAT_THETA:
    case PUSH_WHAT_GRAD: {
      if (what == PUSH_WHAT_GRAD && !c->has_grads) return fail(PUSH_E_STATE, "no gradients yet");
      st = exchange(c, what == PUSH_WHAT_THETA ? BUF_THETA : BUF_GRAD, s);
      if (st != PUSH_OK) return sticky(c, st);
      const float* src = what == PUSH_WHAT_THETA ? c->theta[c->cur] : c->grad;
      cudaError_t e = cudaMemcpy2DAsync(out_host, P.d * 4, src, P.ld * 4, P.d * 4, P.n, cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) return sticky(c, fail(PUSH_E_CUDA, cudaGetErrorString(e)));
      break;
    }
    case PUSH_WHAT_DIST:
    case PUSH_WHAT_H:
    case PUSH_WHAT_KERNEL: {
      if (!c->has_step) return fail(PUSH_E_STATE, "no SVGD step yet");
      const float* src =
          what == PUSH_WHAT_DIST ? c->D : (what == PUSH_WHAT_H ? c->h : c->K + (P.ds ? (int64_t)c->row0 * P.n : 0));
      const size_t T = P.tensors;
      const size_t cnt = what == PUSH_WHAT_DIST ? T * P.n * P.n : (what == PUSH_WHAT_H ? T : T * P.nl * P.n);
      cudaError_t e = cudaMemcpyAsync(out_host, src, cnt * 4, cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) return sticky(c, fail(PUSH_E_CUDA, cudaGetErrorString(e)));
      break;
    }
    case PUSH_WHAT_LOSS: {
      if (!c->has_grads) return fail(PUSH_E_STATE, "no loss yet");
      st = exchange(c, BUF_LOSS, s);
      if (st != PUSH_OK) return sticky(c, st);
      cudaError_t e = cudaMemcpyAsync(out_host, c->loss_all, (size_t)P.n * 4, cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) return sticky(c, fail(PUSH_E_CUDA, cudaGetErrorString(e)));
      break;
    }
    default:
      return fail(PUSH_E_INVALID, "unknown PUSH_WHAT");
  }
  st = sync();
  return st == PUSH_OK ? PUSH_OK : sticky(c, st);
}

push_status push_profile_enable(push_ctx* c, int32_t enable) {
  if (!c) return fail(PUSH_E_INVALID, "ctx is NULL");
  for (auto& r : c->recs) {
    c->ev_pool.push_back(r.e0);
    c->ev_pool.push_back(r.e1);
  }
  c->recs.clear();
  c->trace.clear();
  c->prof_on = enable != 0;
  return PUSH_OK;
}

push_status push_profile_trace(push_ctx* c, int32_t* classes, int32_t max_n, int32_t* n) {
  if (!c || !n || (max_n > 0 && !classes)) return fail(PUSH_E_INVALID, "NULL argument");
  *n = (int32_t)c->trace.size();
  for (int32_t i = 0; i < max_n && i < *n; ++i) classes[i] = c->trace[i];
  return PUSH_OK;
}

push_status push_profile_read(push_ctx* c, push_profile_row* rows, int32_t max_rows, int32_t* n_rows) {
  if (!c || !rows || !n_rows) return fail(PUSH_E_INVALID, "NULL argument");
  PUSH_CUDA_TRY(cudaDeviceSynchronize());
  const int n = std::min<int>(max_rows, PC_N);
  for (int i = 0; i < n; ++i) {
    std::memset(&rows[i], 0, sizeof(push_profile_row));
    std::strncpy(rows[i].name, kClassNames[i], sizeof(rows[i].name) - 1);
  }
  for (auto& r : c->recs) {
    if (r.cls >= n) continue;
    float ms = 0.f;
    PUSH_CUDA_TRY(cudaEventElapsedTime(&ms, r.e0, r.e1));
    rows[r.cls].ms += ms;
    rows[r.cls].launches += r.launches;
    rows[r.cls].alg_bytes += r.bytes;
    rows[r.cls].alg_flops += r.flops;
  }
  *n_rows = n;
  return PUSH_OK;
}

push_status push_launch_count(push_ctx* c, int64_t* count) {
  if (!c || !count) return fail(PUSH_E_INVALID, "NULL argument");
  *count = c->launches;
  return PUSH_OK;
}

push_status push_destroy(push_ctx* c) {
  if (!c) return PUSH_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (c->comm) nccl::comm_release(c->comm, c->broken);
  for (auto& r : c->recs) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (auto& gph : c->graphs)
    if (gph.exec) cudaGraphExecDestroy(gph.exec);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_theta) cudaEventDestroy(c->ev_theta);
  if (c->ev_fork2) cudaEventDestroy(c->ev_fork2);
  if (c->ev_grad) cudaEventDestroy(c->ev_grad);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->ev_kfork) cudaEventDestroy(c->ev_kfork);
  if (c->ev_kdone) cudaEventDestroy(c->ev_kdone);
  if (c->k_stream) cudaStreamDestroy(c->k_stream);
  if (c->w_stream) cudaStreamDestroy(c->w_stream);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  delete c;
  return PUSH_OK;
}

// ------------------------------------------------------------------ debug: isolated GEMM
static push_status dbg_gemm(int passes, int32_t a_mn, int32_t b_mn, int32_t b_split, int32_t M, int32_t N, int32_t K,
                            int32_t batch, const float* A, const float* Bm, float* C, void* stream) {
  if (M < 1 || N < 1 || K < 1 || batch < 1) return fail(PUSH_E_SHAPE, "empty GEMM");
  if (N % 32) return fail(PUSH_E_SHAPE, "N % 32 != 0");
  if (a_mn && M % 32) return fail(PUSH_E_SHAPE, "MN-major A needs M % 32 == 0");
  if ((!a_mn || !b_mn) && K % 4) return fail(PUSH_E_SHAPE, "K-major operands need K % 4 == 0");
  if (a_mn && (int64_t)M * K % 4) return fail(PUSH_E_SHAPE, "batch stride must be a multiple of 4");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t na = (int64_t)M * K, nb = (int64_t)N * K;
  if (na % 4 || nb % 4) return fail(PUSH_E_SHAPE, "batch strides must be multiples of 4");
  float* buf = nullptr;
  if (!b_split) {
    PUSH_CUDA_TRY(cudaMallocAsync(&buf, sizeof(float) * 2 * batch * nb, s));
    kern::split_hilo(Bm, nb, buf, buf + batch * nb, nb, nb, batch, s);
  }
  gemm::Problem pb;
  pb.M = M; pb.N = N; pb.K = K; pb.batch = batch; pb.splits = 1; pb.passes = passes;
  pb.A = gemm::Operand{A, nullptr, true, a_mn != 0, a_mn ? M : K, na};
  if (b_split)
    pb.B = gemm::Operand{Bm, nullptr, true, b_mn != 0, b_mn ? N : K, nb};
  else
    pb.B = gemm::Operand{buf, buf + batch * nb, false, b_mn != 0, b_mn ? N : K, nb};
  pb.epi = gemm::EPI_STORE;
  pb.out = C; pb.ldo = N; pb.out_pstride = (int64_t)M * N; pb.out_sstride = 0;
  float* zb = nullptr;
  if ((passes >> 8) & 32) {  // experiment: the forward epilogue (bias 0, tanh) instead of a plain store
    PUSH_CUDA_TRY(cudaMallocAsync(&zb, sizeof(float) * N, s));
    PUSH_CUDA_TRY(cudaMemsetAsync(zb, 0, sizeof(float) * N, s));
    pb.epi = gemm::EPI_FWD; pb.act = ((passes >> 8) & 64) ? PUSH_ACT_IDENTITY : PUSH_ACT_TANH;
    pb.bias = zb; pb.bias_pstride = 0;
    pb.passes = passes & ~(96 << 8);
  }
  push_status st = gemm::run(pb, s);
  if (buf) cudaFreeAsync(buf, s);
  if (zb) cudaFreeAsync(zb, s);
  return st;
}

push_status pushdbg_gemm3xtf32(int32_t a_mn, int32_t b_mn, int32_t M, int32_t N, int32_t K, int32_t batch,
                               const float* A_dev, const float* B_dev, float* C_dev, void* stream) {
  return dbg_gemm(3, a_mn, b_mn, 0, M, N, K, batch, A_dev, B_dev, C_dev, stream);
}
push_status pushdbg_gemm1xtf32(int32_t a_mn, int32_t b_mn, int32_t M, int32_t N, int32_t K, int32_t batch,
                               const float* A_dev, const float* B_dev, float* C_dev, void* stream) {
  return dbg_gemm(1, a_mn, b_mn, 0, M, N, K, batch, A_dev, B_dev, C_dev, stream);
}
push_status pushdbg_gemm(int32_t passes, int32_t a_mn, int32_t b_mn, int32_t b_split, int32_t M, int32_t N, int32_t K,
                         int32_t batch, const float* A_dev, const float* B_dev, float* C_dev, void* stream) {
  // low byte: 1 or 3 passes; bits 8+: kernel experiment flags (bit 8: skip the in-smem hi/lo split)
  if ((passes & 0xff) != 1 && (passes & 0xff) != 3) return fail(PUSH_E_INVALID, "passes must be 1 or 3");
  return dbg_gemm(passes, a_mn, b_mn, b_split, M, N, K, batch, A_dev, B_dev, C_dev, stream);
}

}  // extern "C"
