// Microbenchmark: HBM read rate of a row-strided stream (n rows of ld floats, each CTA owning a column
// range of every row), as a function of the contiguous bytes fetched per row per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_rows stream_rows.cu && /tmp/stream_rows
#include <cstdio>
#include <cuda_runtime.h>

template <int CW>  // columns per row per step (float4 per thread along columns)
__global__ void __launch_bounds__(256) stream_kernel(const float* __restrict__ th, long long ld, int n, long long cols,
                                                     float* out) {
  const long long c0 = blockIdx.x * cols, c1 = c0 + cols;
  constexpr int T4 = CW / 4;             // threads per row
  constexpr int RPP = 256 / T4;          // rows per pass
  const int tr = threadIdx.x / T4, tc = threadIdx.x % T4;
  float acc = 0.f;
  for (long long c = c0; c < c1; c += CW) {
#pragma unroll
    for (int r = tr; r < 64; r += RPP) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(th + (long long)r * ld + c + 4 * tc));
      acc += v.x + v.y + v.z + v.w;
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const int n = 64;
  const long long ld = 1053312;  // S1
  float* th;
  float* out;
  cudaMalloc(&th, sizeof(float) * n * ld);
  cudaMalloc(&out, 4);
  cudaMemset(th, 0, sizeof(float) * n * ld);
  for (int grid : {148, 296, 592, 1184}) {
  printf("grid %d\n", grid);
  const long long cols = (ld / grid) / 256 * 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto kern, const char* name) {
    for (int w = 0; w < 3; ++w) kern<<<grid, 256>>>(th, ld, n, cols, out);
    cudaEventRecord(a);
    for (int w = 0; w < 10; ++w) kern<<<grid, 256>>>(th, ld, n, cols, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 4.0 * n * cols * grid;
    printf("%-8s %8.2f us  %7.1f GB/s\n", name, ms * 100, bytes / (ms / 10 * 1e-3) / 1e9);
  };
  run(stream_kernel<32>, "128B");
  run(stream_kernel<64>, "256B");
  run(stream_kernel<128>, "512B");
  run(stream_kernel<256>, "1KB");
  run(stream_kernel<512>, "2KB");
  }
  return 0;
}
