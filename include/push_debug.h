/*
 * push_debug.h — test-only entry points of libpush_b200.so (not part of the
 * stable ABI).  They expose single kernels of the product path so tests can
 * check them in isolation; they run exactly the kernels push_particle_grads
 * uses.
 */
#ifndef PUSH_DEBUG_H_
#define PUSH_DEBUG_H_

#include <stdint.h>

#include "push.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ASYNC (allocates and frees its scratch with cudaMallocAsync on `stream`).
 * Batched fp32 GEMM computed by the product's tcgen05 3xTF32 kernel
 * (operands split into tf32 hi + lo, three tensor-core products per k-step):
 *
 *   C[p][m][n] = sum_k A(p, m, k) * B(p, k, n),   p < batch
 *
 *   a_mn = 0: A is [batch][M][K] (K contiguous)   a_mn = 1: A is [batch][K][M]
 *   b_mn = 0: B is [batch][N][K] (K contiguous)   b_mn = 1: B is [batch][K][N]
 *   C is [batch][M][N] row-major float32.
 * Constraints: M, N, K >= 1; N % 32 == 0; K % 4 == 0 when a_mn == 0 or b_mn == 0;
 * M % 32 == 0 when a_mn == 1.  Errors: PUSH_E_SHAPE, PUSH_E_CUDA. */
push_status pushdbg_gemm3xtf32(int32_t a_mn, int32_t b_mn, int32_t M, int32_t N, int32_t K, int32_t batch,
                               const float* A_dev, const float* B_dev, float* C_dev, void* stream);

/* ASYNC.  Single-pass (1xTF32) variant of the same kernel: only hi*hi, for
 * the precision test that shows why the product uses three passes. */
push_status pushdbg_gemm1xtf32(int32_t a_mn, int32_t b_mn, int32_t M, int32_t N, int32_t K, int32_t batch,
                               const float* A_dev, const float* B_dev, float* C_dev, void* stream);

/* ASYNC.  General form of the two entries above: passes = 1 or 3; b_split = 1 feeds B as
 * plain fp32 split into hi/lo on the staged tile inside the kernel (the path the weight-gradient
 * GEMM uses for its activation operand); b_split = 0 pre-splits B into a hi/lo pair in global
 * memory (the path the forward/backward GEMMs use for the weights).  A is always split in-kernel.
 * Same layouts, constraints and errors as pushdbg_gemm3xtf32 (PUSH_E_INVALID for bad passes). */
push_status pushdbg_gemm(int32_t passes, int32_t a_mn, int32_t b_mn, int32_t b_split, int32_t M, int32_t N, int32_t K,
                         int32_t batch, const float* A_dev, const float* B_dev, float* C_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PUSH_DEBUG_H_ */
