// Microbenchmark: issue rate of tcgen05.mma kind::tf32 (M = 128, K = 8) on one SM as a function of N and
// of where A lives (TMEM vs shared memory), and the cost of a commit after every g MMAs.  One thread
// issues R MMAs back to back into one accumulator; cycles from the first issue to the commit's arrival.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2306_06528_b200/csrc -o mma_rate mma_rate.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"

using namespace push;

template <int N, bool A_TMEM>
__global__ void __launch_bounds__(128, 1) mma_kernel(int R, int group, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  // A tile: 128 rows x 128 B (SW128 K-major); B tile: N rows x 128 B
  uint8_t* atile = smem;
  uint8_t* btile = smem + 128 * 128;
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (128 + N) * 32; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::fence_mbar_init();
  }
  if (threadIdx.x < 32) {
    ptx::tmem_alloc(&slot, 512);
    ptx::tmem_relinquish();
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tb = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = ptx::idesc_tf32(128, N, false, false);
    const uint32_t ab = ptx::smem_u32(atile), bb = ptx::smem_u32(btile);
    int ph = 0;
    // warm-up
    for (int r = 0; r < 16; ++r) {
      if (A_TMEM)
        ptx::mma_tf32_ts(tb, tb + 256 + (r & 3) * 8, ptx::umma_desc(bb + (r & 3) * 32, 16, 1024, 2), idesc, 1u);
      else
        ptx::mma_tf32(tb, ptx::umma_desc(ab + (r & 3) * 32, 16, 1024, 2),
                      ptx::umma_desc(bb + (r & 3) * 32, 16, 1024, 2), idesc, 1u);
    }
    ptx::mma_commit(&bar[0]);
    ptx::mbar_wait(&bar[0], ph);
    ph ^= 1;
    const long long t0 = clock64();
    if (group < 0) {  // loop-invariant operands: the hardware floor without per-MMA descriptor math
      const uint64_t bd = ptx::umma_desc(bb, 16, 1024, 2);
      for (int r = 0; r < R; r += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) ptx::mma_tf32_ts(tb, tb + 256, bd, idesc, 1u);
      }
    } else
    for (int r = 0; r < R; ++r) {
      if (A_TMEM)
        ptx::mma_tf32_ts(tb, tb + 256 + (r & 3) * 8, ptx::umma_desc(bb + (r & 3) * 32, 16, 1024, 2), idesc, 1u);
      else
        ptx::mma_tf32(tb, ptx::umma_desc(ab + (r & 3) * 32, 16, 1024, 2),
                      ptx::umma_desc(bb + (r & 3) * 32, 16, 1024, 2), idesc, 1u);
      if (group > 0 && (r + 1) % group == 0) ptx::mma_commit(&bar[1]);
    }
    ptx::mma_commit(&bar[0]);
    ptx::mbar_wait(&bar[0], ph);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tb, 512);
}

template <int N, bool AT>
void run(int grid, int group) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * grid);
  const int smem = 1024 + (128 + 256) * 128;
  cudaFuncSetAttribute(mma_kernel<N, AT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int R = 4096;
  mma_kernel<N, AT><<<grid, 128, smem>>>(R, group, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += h[i];
  avg /= grid;
  const double cyc = avg / R;
  printf("N=%3d A=%s grid=%3d commit/%d: %7.1f cycles per MMA  (%6.0f MAC/clk)  %s\n", N, AT ? "tmem" : "smem", grid,
         group, cyc, 128.0 * N * 8 / cyc, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int grid : {1, 148}) {
    run<32, true>(grid, 0);
    run<64, true>(grid, 0);
    run<128, true>(grid, 0);
    run<256, true>(grid, 0);
    run<64, false>(grid, 0);
    run<128, false>(grid, 0);
    run<256, false>(grid, 0);
  }
  run<32, true>(1, -1);
  run<64, true>(1, -1);
  run<128, true>(1, -1);
  run<256, true>(1, -1);
  return 0;
}
