/*
 * push.h — C-ABI of the B200-native SVGD particle step of PusH (arXiv 2306.06528).
 *
 * What the library computes (one "step" = PAPER.md:655-660, Fig. supp:svgd,
 * i.e. `pstep` on every particle then `psend(p, "SVGD_UPDATE")` on every particle):
 *
 *   g_i    = grad log p(theta_i | D) = -lambda * grad MSE_i(theta_i) + grad log p0(theta_i)
 *                                                  (Eq. eq:grad)
 *   D_ij   = ||theta_i - theta_j||^2,   h = median(D) / ln n   (bandwidth rule)
 *   K_ij   = exp(-D_ij / h)
 *   phi_i  = (1/n) sum_j [ K_ij g_j + grad_{theta_j} K_ij ]   (north star)
 *   theta_i <- theta_i + eps * phi_i   for all i simultaneously (Jacobi)
 *
 * Readings of the paper that these semantics fix are listed in DESIGN.md
 * ("Readings" R1-R20); the float64 CPU oracle in oracle/ implements the same
 * definitions independently.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * - Nothing throws across this boundary; every call returns push_status and,
 *   on failure, sets a thread-local message readable with push_last_error().
 * - Pointers named *_dev are CUDA device pointers on the context's device;
 *   *_host are ordinary (pageable or pinned) host pointers.  The library never
 *   frees memory it did not allocate.
 * - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   Calls marked ASYNC only enqueue work on `stream`; the caller must keep the
 *   arguments alive until that work completes.  Calls marked SYNC return after
 *   the work is complete.
 * - Canonical parameter layout of one particle (R15): for each
 *   Linear layer l = 1..L in order, W_l as [out_l][in_l] row-major (torch
 *   nn.Linear orientation) followed by b_l[out_l] — module.parameters() order
 *   (PAPER.md:560, 631).  d = sum_l (in_l*out_l + out_l).
 * - Particle i is global row i; with world_size P, rank r owns rows
 *   [r*n/P, (r+1)*n/P)  (n % P == 0 is required).
 * - Multi-rank calls (world_size > 1) are COLLECTIVE: every rank must call
 *   push_init, push_particle_grads / push_set_grads, push_svgd_step,
 *   push_step_host, push_gather and push_destroy in the same order with the
 *   same B.
 * - Errors: validation failures (PUSH_E_INVALID / PUSH_E_SHAPE / PUSH_E_STATE)
 *   leave the context unchanged.  CUDA or NCCL failures (PUSH_E_CUDA /
 *   PUSH_E_NCCL) are sticky: every later call on that context returns
 *   PUSH_E_STATE; push_destroy still releases it.
 * - One host thread per context.
 */
#ifndef PUSH_H_
#define PUSH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PUSH_ABI_VERSION 1
#define PUSH_MAX_LAYERS 15

typedef struct push_ctx push_ctx; /* opaque; owned by the library */

typedef enum {
  PUSH_OK = 0,
  PUSH_E_INVALID = 1,     /* bad argument value (NULL pointer, bad enum, bad rank, sigma <= 0 ...) */
  PUSH_E_SHAPE = 2,       /* bad size: n % P != 0, dims <= 0, B > max_batch, workspace too small ... */
  PUSH_E_STATE = 3,       /* call out of order (e.g. svgd_step without fresh grads) or sticky failure */
  PUSH_E_CUDA = 4,        /* a CUDA runtime / driver call failed (sticky) */
  PUSH_E_NCCL = 5,        /* NCCL failed or libnccl could not be loaded (sticky) */
  PUSH_E_NOMEM = 6,       /* host allocation failed */
  PUSH_E_UNSUPPORTED = 7  /* device is not sm_100 or a feature is not compiled in */
} push_status;

enum { PUSH_ACT_TANH = 0, PUSH_ACT_RELU = 1, PUSH_ACT_IDENTITY = 2 };   /* hidden layers (R13) */
enum { PUSH_PRIOR_UNIFORM = 0, PUSH_PRIOR_GAUSSIAN = 1 };
/* Bandwidth rules (R2-R4): h = med/ln n (default), h = med/ln(n+1), or h = bw_h.
 * med = median of all n^2 squared distances (average of the two middle order
 * statistics when n^2 is even); h = 1 when n == 1 or med == 0. */
enum { PUSH_BW_MEDIAN_LN_N = 0, PUSH_BW_MEDIAN_LN_N1 = 1, PUSH_BW_FIXED = 2 };
enum {
  PUSH_WHAT_THETA = 0,   /* n x d canonical parameters (current Theta)            */
  PUSH_WHAT_GRAD = 1,    /* n x d canonical g of the last grads call (likelihood term only under PRIOR_SUM) */
  PUSH_WHAT_DIST = 2,    /* T x n x n squared distances D of the last step (T = 1 unless PER_TENSOR).
                            Summed directly as sum_k (theta_ik - theta_jk)^2, except n >= 32 with
                            n % 32 == 0 on the all-gather path: D_ij = G_ii + G_jj - 2 G_ij from the
                            Gram matrix (tensor cores), clamped at 0 (R27).  Always exactly
                            symmetric with a +0 diagonal. */
  PUSH_WHAT_H = 3,       /* T floats: bandwidth h of the last step                    */
  PUSH_WHAT_LOSS = 4,    /* n floats: per-particle MSE of the last grads call (pre-update) */
  PUSH_WHAT_KERNEL = 5   /* T x n_local x n kernel matrix K of the last step (own rows) */
};

/* Update variants: PusH's own `_svgd_update` differs
 * from the canonical SVGD direction of the north star in three ways, each selectable alone:
 *   PUSH_VAR_PER_TENSOR : the kernel is evaluated per parameter TENSOR (W_l and
 *                         b_l of every layer, in module.parameters() order), T = 2L distance / kernel
 *                         matrices, each with its own bandwidth under a median rule.
 *   PUSH_VAR_PAPER_NORM : drive terms weighted 1 and the repulsion 1/n (A5)
 *                         instead of 1/n on both.
 *   PUSH_VAR_PRIOR_SUM  : G holds -lambda grad MSE only and the prior gradients of all n particles
 *                         are added unweighted, sum_j grad log p0(theta_j) (A8),
 *                         with the drive weight.
 * PUSH_VARIANT_PAPER = all three; with bw_rule FIXED and bw_h = 2 it is the listing's
 * kernel_bandwidth l = 1 (A1).  The update of particle i, element k of tensor t:
 *   theta_ik += eps * ( w_d sum_j K^t_ij g_jk + w_r (2/h_t) sum_j K^t_ij (theta_ik - theta_jk)
 *                       [+ w_d sum_j grad log p0(theta_j)_k] ),   w_d = 1 or 1/n, w_r = 1/n.
 * With PER_TENSOR, PUSH_WHAT_DIST / KERNEL / H return T stacked matrices / values. */
enum { PUSH_VAR_PER_TENSOR = 1, PUSH_VAR_PAPER_NORM = 2, PUSH_VAR_PRIOR_SUM = 4, PUSH_VARIANT_PAPER = 7 };

/* Kernel-phase exchange for world_size > 1:
 *   PUSH_XCHG_ALLGATHER : every rank all-gathers Theta and G (n x ld each) and updates its own rows
 *                         (NVLink bytes per rank per step 2 n ld (P-1)/P).
 *   PUSH_XCHG_DSHARD    : the kernel phase is sharded over d: an all-to-all transposes the own rows'
 *                         Theta and G into a column panel (all n rows x the rank's d-range, whole
 *                         distance splits), each rank computes the distance partials of its splits,
 *                         the partials are all-gathered (P x n^2 floats x splits per rank) and reduced
 *                         in the fixed split order, every rank forms h and the full n x n K, updates
 *                         all n rows of its panel, and a second all-to-all returns the updated columns
 *                         to the row owners (NVLink bytes 3 n ld (P-1)/P^2 + partials).  Results are
 *                         bit-identical to PUSH_XCHG_ALLGATHER for every P (same splits, same sums).
 *                         Requires variant == 0.  With push_init_local_group the whole group's step
 *                         runs in the call of the LAST rank (earlier ranks' calls only record it). */
enum { PUSH_XCHG_ALLGATHER = 0, PUSH_XCHG_DSHARD = 1 };

/* Plain-old-data configuration (128 bytes; field order is ABI). */
typedef struct {
  int32_t n_particles;                 /* n >= 1, n % world_size == 0                        */
  int32_t n_layers;                    /* L in [1, 15] Linear layers                          */
  int32_t dims[PUSH_MAX_LAYERS + 1];   /* L+1 widths d_in, H..., d_out; each >= 1             */
  int32_t activation;                  /* PUSH_ACT_*; output layer is always identity         */
  int32_t prior;                       /* PUSH_PRIOR_*                                        */
  float prior_sigma;                   /* > 0 when prior == GAUSSIAN                          */
  float lik_scale;                     /* lambda > 0: g = -lambda grad MSE + grad log p0 (R9) */
  int32_t bw_rule;                     /* PUSH_BW_*                                           */
  float bw_h;                          /* > 0 when bw_rule == FIXED; K = exp(-r^2 / h) (R1)   */
  float step_size;                     /* eps > 0                                             */
  int32_t max_batch;                   /* >= 1; sizes the workspace                           */
  uint64_t seed;                       /* K0 initialiser stream (R14)                         */
  int32_t swag;                        /* 1: allocate SWAG moment buffers (push_swag_*)       */
  int32_t variant;                     /* 0 = canonical SVGD; else an OR of PUSH_VAR_* (NEXT-2)  */
  int32_t exchange;                    /* PUSH_XCHG_* (NEXT-4)                                 */
  int32_t reserved;                    /* must be 0                                            */
} push_config;

/* Library / build identification string (static storage). */
const char* push_version(void);

/* Thread-local message describing the last failure on this thread ("" if none). */
const char* push_last_error(void);

/* SYNC.  Rank 0 of a world_size > 1 job creates the 128-byte NCCL unique id
 * that every rank then passes to push_init (the caller broadcasts it, e.g.
 * with torch.distributed).  Loads libnccl.so.2 at run time.
 * Errors: PUSH_E_INVALID (id NULL), PUSH_E_NCCL. */
push_status push_get_unique_id(uint8_t id[128]);

/* SYNC, host only.  Bytes of device workspace a rank needs for `cfg` at
 * `world_size`.  The caller allocates it (e.g. a torch uint8 CUDA tensor),
 * passes it to push_init and keeps it alive until push_destroy.
 * Errors: PUSH_E_INVALID / PUSH_E_SHAPE for an invalid cfg. */
push_status push_workspace_size(const push_config* cfg, int32_t world_size, size_t* bytes);

/* SYNC.  Creates a context for `rank` of `world_size` on the current CUDA device.
 *   nccl_id       : 128-byte id from push_get_unique_id; NULL iff world_size == 1.
 *   dev_workspace : caller-owned device buffer of >= push_workspace_size bytes,
 *                   256-byte aligned.
 *   theta0_host   : NULL -> every particle initialised by K0 (R14, seeded by
 *                   cfg->seed); else n x d canonical float32 rows (all n rows;
 *                   each rank copies the ones it needs).
 * On success *out owns the context (state READY).
 * Errors: PUSH_E_INVALID, PUSH_E_SHAPE, PUSH_E_UNSUPPORTED (not sm_100), PUSH_E_CUDA, PUSH_E_NCCL. */
push_status push_init(const push_config* cfg, int32_t rank, int32_t world_size, const uint8_t* nccl_id,
                      void* dev_workspace, size_t ws_bytes, const float* theta0_host, push_ctx** out);

/* SYNC.  Test/emulation transport: creates world_size contexts (ranks 0..P-1)
 * on the CURRENT device that exchange rows by device-to-device copies instead
 * of NCCL (one GPU cannot host several NCCL ranks).  Results are defined to be
 * bit-identical to an NCCL job with the same P.  Calls on the P contexts must
 * be issued from one thread on ONE stream in lockstep: grads for ranks 0..P-1,
 * then svgd_step for ranks 0..P-1, etc.
 *   dev_workspaces[r]: workspace of rank r (ws_bytes each).  out_ctxs[r]: context r. */
push_status push_init_local_group(const push_config* cfg, int32_t world_size, void* const* dev_workspaces,
                                  size_t ws_bytes, const float* theta0_host, push_ctx** out_ctxs);

/* ASYNC.  Steps a0-a5: for every local particle i, forward the MLP
 * on the batch, MSE loss, backprop, and write g_i = -lambda grad MSE_i +
 * grad log p0(theta_i) into the context's G; starts the all-gather of Theta.
 *   x_dev : B x d_in  float32 row-major, y_dev : B x d_out float32 row-major
 *           (the SAME batch on every rank).
 *   B     : 1 <= B <= cfg.max_batch.
 *   loss_dev : NULL or n_local floats receiving the per-particle MSE.
 * State: READY or GRADS_READY -> GRADS_READY.
 * Errors: PUSH_E_INVALID (NULL x/y), PUSH_E_SHAPE (B), PUSH_E_STATE, PUSH_E_CUDA. */
push_status push_particle_grads(push_ctx* ctx, const float* x_dev, const float* y_dev, int32_t B,
                                float* loss_dev, void* stream);

/* ASYNC.  Supplies g directly instead of push_particle_grads (the paper's
 * principle needs only a differentiable joint density):
 * g_dev is n_local x d canonical float32 (row i = local particle i).
 * State: READY or GRADS_READY -> GRADS_READY.  Errors: PUSH_E_INVALID, PUSH_E_STATE. */
push_status push_set_grads(push_ctx* ctx, const float* g_dev, void* stream);

/* ASYNC.  Steps a6-a10: gathers G (world_size > 1), pairwise squared
 * distances, median bandwidth, kernel matrix and the fused update of the
 * local particles.  State: GRADS_READY -> READY.
 * Errors: PUSH_E_STATE (no fresh grads), PUSH_E_CUDA, PUSH_E_NCCL. */
push_status push_svgd_step(push_ctx* ctx, void* stream);

/* ASYNC.  One whole step (push_particle_grads + push_svgd_step) replayed from a CUDA graph: the batch
 * is first copied (device to device, on `stream`) into the context's own batch buffers, which the
 * captured step reads; one executable graph per Theta buffer parity is captured on first use and
 * re-captured when B or loss_dev changes.  The first call on a context runs eagerly (it also
 * initialises every kernel's one-time attributes).  Results are identical to the eager calls.
 * PUSH_NO_GRAPH=1 in the environment, or profiling (push_profile_enable), selects the eager path.
 *   x_dev, y_dev, B, loss_dev: as in push_particle_grads.   State: READY or GRADS_READY -> READY.
 * Errors: PUSH_E_INVALID, PUSH_E_SHAPE, PUSH_E_CUDA, PUSH_E_NCCL. */
push_status push_step_graph(push_ctx* ctx, const float* x_dev, const float* y_dev, int32_t B, float* loss_dev,
                            void* stream);

/* SYNC.  End-to-end convenience through host memory: copies x_host (B x d_in)
 * and y_host (B x d_out) to the device, runs the step (push_step_graph), copies
 * the n_local per-particle losses to loss_host (may be NULL) and synchronises
 * `stream`.  State: READY -> READY. */
push_status push_step_host(push_ctx* ctx, const float* x_host, const float* y_host, int32_t B,
                           float* loss_host, void* stream);

/* ASYNC.  Deep-ensemble step (Fig. lang:de): every local
 * particle takes an independent gradient-ascent step theta_i <- theta_i + eps * g_i on its own
 * log posterior (no kernel, no exchange; SVGD with K = I and no repulsion).
 * State: GRADS_READY -> READY.  Errors: PUSH_E_STATE (no fresh grads), PUSH_E_CUDA. */
push_status push_ensemble_step(push_ctx* ctx, void* stream);

/* ASYNC.  Diagonal SWAG moments (Fig. supp:swag): folds
 * the current Theta of every local particle into its running first and second moments,
 *   mean <- (mean * k + theta) / (k + 1),   sq <- (sq * k + theta^2) / (k + 1),   k <- k + 1.
 * Requires cfg.swag = 1.  Errors: PUSH_E_STATE (no SWAG buffers), PUSH_E_CUDA. */
push_status push_swag_collect(push_ctx* ctx, void* stream);

/* ASYNC.  Draws one SWAG sample per local particle: out_dev[i][k] = mean_ik + sqrt(max(sq_ik - mean_ik^2, 0)) z,
 * z = sqrt(-2 ln u1) cos(2 pi u2) with u1 = (m1 + 1) 2^-24, u2 = m2 2^-24 and m1, m2 the top 24 bits of
 * mix64(seed ^ mix64(((i << 32) | k) * 2 + 0 / 1)) (i = global particle row, k = canonical index; the
 * oracle implements the same counter-based generator).  out_dev: n_local x d canonical float32.
 * Errors: PUSH_E_INVALID, PUSH_E_STATE (no SWAG buffers or no collected moments), PUSH_E_CUDA. */
push_status push_swag_sample(push_ctx* ctx, uint64_t seed, float* out_dev, void* stream);

/* ASYNC (collective when world_size > 1).  Predictive pushforward ppush(mu)(g(x; .)) (
 * SURVEY.md §8(f) NEXT-1): every particle's network evaluated on the same inputs, gathered to every rank.
 *   x_dev    : B x d_in float32 row-major, 1 <= B <= cfg.max_batch.
 *   pred_dev : NULL or n x B x d_out float32 (particle-major) receiving every particle's prediction.
 *   mean_dev, std_dev : NULL or B x d_out float32 receiving the cross-particle mean and population
 *              standard deviation (ascending particle order).
 * Uses the context's activation buffers (the last training forward's activations are overwritten; the
 * state machine is unchanged).  Errors: PUSH_E_INVALID, PUSH_E_SHAPE, PUSH_E_CUDA, PUSH_E_NCCL. */
push_status push_predict(push_ctx* ctx, const float* x_dev, int32_t B, float* pred_dev, float* mean_dev,
                         float* std_dev, void* stream);

/* SYNC (collective for THETA, GRAD and LOSS when world_size > 1: each all-gathers the row blocks of
 * every rank, so every rank must make the same call).  Copies `what` (PUSH_WHAT_*) to out_host; sizes
 * in the PUSH_WHAT_* comments.  DIST / H / KERNEL are local reads.
 * Errors: PUSH_E_INVALID, PUSH_E_STATE (GRAD/DIST/H/KERNEL/LOSS before they exist). */
push_status push_gather(push_ctx* ctx, int32_t what, float* out_host, void* stream);

/* Kernel-class profiling with CUDA events on the launching stream.
 * push_profile_enable(ctx, 1) starts recording (and clears totals); while on,
 * each launch of a class is bracketed by events.  push_profile_read
 * synchronises and returns, per class c < n_classes: total milliseconds,
 * launch count, and the algorithmic bytes and flops those launches moved
 * (DESIGN.md §Roofline).  n_classes <= PUSH_PROF_MAX_CLASSES. */
#define PUSH_PROF_MAX_CLASSES 16
typedef struct {
  char name[24];
  double ms;
  int64_t launches;
  double alg_bytes;
  double alg_flops;
} push_profile_row;
push_status push_profile_enable(push_ctx* ctx, int32_t enable);
push_status push_profile_read(push_ctx* ctx, push_profile_row* rows, int32_t max_rows, int32_t* n_rows);

/* Kernel class (index into the push_profile_read rows) of every kernel launched since the last
 * push_profile_enable(ctx, 1), in launch order: *n = total count, the first min(*n, max_n) are
 * written to classes.  Lets an external profiler's per-launch list be attributed to classes. */
push_status push_profile_trace(push_ctx* ctx, int32_t* classes, int32_t max_n, int32_t* n);

/* Total number of kernels this context has launched since push_init (host
 * counter, no sync).  Used for the bench's gpu_launches figure. */
push_status push_launch_count(push_ctx* ctx, int64_t* count);

/* SYNC.  Releases the context (aborts its NCCL communicator).  NULL is a no-op. */
push_status push_destroy(push_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* PUSH_H_ */
