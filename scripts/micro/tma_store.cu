// Microbenchmark: TMA tensor STORE and LOAD rates of the GEMM epilogue's box shapes (32 rows x 16 fp32 =
// 64-B rows, SWIZZLE_64B) against 32 rows x 32 fp32 (128-B rows, SWIZZLE_128B), 8 warps per CTA each
// streaming boxes of its own 32-row slab, one CTA per SM, a 134 MB [rows][256] fp32 matrix (C2's delta).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2306_06528_b200/csrc -o tma_store tma_store.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"

using namespace push;

// mode 0: stores, mode 1: loads.  Warp w of CTA b walks row slabs (b * 8 + w) + k * gridDim.x * 8, all
// 256 columns in boxes of BW columns; 2 boxes in flight per warp.
template <int BW>
__global__ void __launch_bounds__(256, 1) box_kernel(const __grid_constant__ CUtensorMap map, int rows, int mode) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* base = dsm + ((1024u - (ptx::smem_u32(dsm) & 1023u)) & 1023u);
  auto buf = reinterpret_cast<uint8_t(*)[2][32 * BW * 4]>(base);
  __shared__ uint64_t bar[8][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    ptx::mbar_init(&bar[warp][0], 1);
    ptx::mbar_init(&bar[warp][1], 1);
    ptx::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 8 * 2 * 32 * BW; i += blockDim.x) reinterpret_cast<float*>(buf)[i] = 1.f;
  ptx::fence_proxy_async_smem();
  __syncthreads();
  if (lane != 0) return;
  uint32_t ph[2] = {0, 0};
  int k = 0;
  for (int slab = blockIdx.x * 8 + warp; slab * 32 < rows; slab += gridDim.x * 8) {
    for (int c = 0; c < 256; c += BW, ++k) {
      const int b = k & 1;
      if (mode == 0) {
        ptx::bulk_wait_read1();
        ptx::tma_store_3d(&map, buf[warp][b], c, slab * 32, 0);
        ptx::bulk_commit();
      } else {
        if (k >= 2) {
          ptx::mbar_wait(&bar[warp][b], ph[b]);
          ph[b] ^= 1;
        }
        ptx::mbar_arrive_expect_tx(&bar[warp][b], 32 * BW * 4);
        ptx::tma_load_3d(buf[warp][b], &map, &bar[warp][b], c, slab * 32, 0);
      }
    }
  }
  if (mode == 0) ptx::bulk_wait0();
  else
    for (int b = 0; b < 2; ++b)
      if (k > b) ptx::mbar_wait(&bar[warp][b], ph[b]);
}

int main() {
  const int rows = 131072;  // 16 particles x 8192
  float* d;
  cudaMalloc(&d, sizeof(float) * rows * 256);
  cudaMemset(d, 0, sizeof(float) * rows * 256);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  auto mk = [&](CUtensorMap* m, int bw, CUtensorMapSwizzle swz) {
    cuuint64_t dims[3] = {256, (cuuint64_t)rows, 1};
    cuuint64_t strides[2] = {256 * 4, (cuuint64_t)rows * 256 * 4};
    cuuint32_t box[3] = {(cuuint32_t)bw, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = 4.0 * rows * 256;
  for (int mode : {0, 1})
    for (int grid : {148, 296}) {
      CUtensorMap m16, m32;
      mk(&m16, 16, CU_TENSOR_MAP_SWIZZLE_64B);
      mk(&m32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
      for (int w = 0; w < 2; ++w) {
        cudaFuncSetAttribute(box_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
        cudaFuncSetAttribute(box_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
        auto run = [&](int which) {
          if (which == 0) box_kernel<16><<<grid, 256, 8 * 2 * 32 * 16 * 4 + 1024>>>(m16, rows, mode);
          else box_kernel<32><<<grid, 256, 8 * 2 * 32 * 32 * 4 + 1024>>>(m32, rows, mode);
        };
        for (int which : {0, 1}) {
          run(which);
          cudaEventRecord(a);
          for (int r = 0; r < 10; ++r) run(which);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (w == 1)
            printf("%s grid %d box 32x%d: %7.2f us  %7.1f GB/s %s\n", mode ? "load " : "store", grid,
                   which ? 32 : 16, ms * 100, bytes / (ms / 10 * 1e-3) / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        }
      }
    }
  return 0;
}
