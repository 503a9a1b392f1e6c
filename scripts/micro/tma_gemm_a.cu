// Microbenchmark: the GEMM A-operand stream (K-major activations [rows][K], K = 512) through a TMA ring,
// 128-row boxes of 32 fp32 (SWIZZLE_128B, the GEMM's k-block) vs 128 fp32 (SWIZZLE_NONE), one CTA per SM
// walking 128-row blocks and all of K; consumer only releases stages.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2306_06528_b200/csrc -o tma_gemm_a tma_gemm_a.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"

using namespace push;

__global__ void __launch_bounds__(64, 1) ring(const __grid_constant__ CUtensorMap map, int mblocks, int K, int bw,
                                              int stage_bytes, int stages, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int kst = K / bw;
  int n = 0;
  for (int mb = blockIdx.x; mb < mblocks; mb += gridDim.x) n += kst;
  if (threadIdx.x == 0) {
    int i = 0;
    for (int mb = blockIdx.x; mb < mblocks; mb += gridDim.x)
      for (int k = 0; k < kst; ++k, ++i) {
        const int s = i % stages;
        ptx::mbar_wait(&empty[s], ((i / stages) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&full[s], stage_bytes);
        ptx::tma_load_3d(smem + s * stage_bytes, &map, &full[s], k * bw, mb * 128, 0);
      }
  } else if (threadIdx.x == 32) {
    float acc = 0.f;
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      ptx::mbar_wait(&full[s], (i / stages) & 1);
      acc += ptx::lds_f32(ptx::smem_u32(smem + s * stage_bytes + 4 * (i & 31)));
      ptx::mbar_arrive(&empty[s]);
    }
    if (acc == 1234.5f) sink[0] = acc;
  }
}

int main() {
  const int rows = 64 * 8192, K = 512;
  float *d, *sink;
  cudaMalloc(&d, sizeof(float) * (size_t)rows * K);
  cudaMalloc(&sink, 4);
  cudaMemset(d, 0, sizeof(float) * (size_t)rows * K);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int bw : {32, 64, 128}) {
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, 1};
    cuuint64_t strides[2] = {(cuuint64_t)K * 4, (cuuint64_t)K * rows * 4};
    cuuint32_t box[3] = {(cuuint32_t)bw, 128, 1};
    cuuint32_t es[3] = {1, 1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        bw == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int sb = bw * 128 * 4;
    for (int stages : {2, 4, 6, 8, 12}) {
      if (stages * sb > 200 * 1024) continue;
      auto run = [&] { ring<<<148, 64, stages * sb + 2048>>>(m, rows / 128, K, bw, sb, stages, sink); };
      run();
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("box %3d x 128 rows, %2d stages (%3d KB): %8.1f us  %7.1f GB/s %s\n", bw, stages, stages * sb / 1024,
             ms * 200, 4.0 * rows * K / (ms / 5 * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
