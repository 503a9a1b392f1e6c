// Microbenchmark: HBM read rate of the a7 / a10 streaming pattern (64 rows of ld fp32, each CTA owning a
// column range of every row) through a TMA ring, vs box shape, bytes per stage, ring depth and CTAs per
// SM.  The consumer only releases stages (no compute): the pipeline's own ceiling.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2306_06528_b200/csrc -o /tmp/tma_stream \
//        tma_stream.cu -lcuda && /tmp/tma_stream
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace push;

// mode 0: tensor boxes {32 fp32, R rows} (SWIZZLE_128B), nbox per stage along the columns
// mode 1: tensor boxes {128 fp32, R rows} (SWIZZLE_NONE), nbox per stage along the rows
// mode 2: 1-D bulk copies of seg bytes per row, R rows per stage (lanes of warp 0 issue)
__global__ void __launch_bounds__(64, 1) ring_kernel(const __grid_constant__ CUtensorMap map, const float* base,
                                                   long long ld, int mode, int R, int nbox, int stage_bytes,
                                                   int stages, long long cols_per_cta, int cols_per_stage,
                                                   int nrows, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const long long c0 = blockIdx.x * cols_per_cta;
  // steps: column blocks x row groups
  const int rgroups = (mode == 0 || mode == 3) ? 1 : nrows / (R * (mode == 1 ? nbox : 1));
  const int csteps = (int)(cols_per_cta / cols_per_stage);
  const int nst = csteps * rgroups;
  if (warp == 0) {
    for (int i = 0; i < nst; ++i) {
      const int s = i % stages;
      const int cs = i / rgroups, rg = i % rgroups;
      const long long col = c0 + (long long)cs * cols_per_stage;
      if (lane == 0) ptx::mbar_wait(&empty[s], ((i / stages) & 1) ^ 1);
      __syncwarp();
      if (mode == 0) {
        if (lane == 0) {
          ptx::mbar_arrive_expect_tx(&full[s], stage_bytes);
          for (int j = 0; j < nbox; ++j)
            ptx::tma_load_3d(smem + s * stage_bytes + j * (R * 128), &map, &full[s], (int)(col + 32 * j), 0, 0);
        }
      } else if (mode == 1) {
        if (lane == 0) {
          ptx::mbar_arrive_expect_tx(&full[s], stage_bytes);
          for (int j = 0; j < nbox; ++j)
            ptx::tma_load_3d(smem + s * stage_bytes + j * (R * 512), &map, &full[s], (int)col,
                             (rg * nbox + j) * R, 0);
        }
      } else if (mode == 3) {
        if (lane == 0) {
          ptx::mbar_arrive_expect_tx(&full[s], stage_bytes);
          ptx::tma_load_3d(smem + s * stage_bytes, &map, &full[s], (int)col, 0, 0);
        }
      } else {
        const int seg = cols_per_stage * 4;
        if (lane == 0) ptx::mbar_arrive_expect_tx(&full[s], stage_bytes);
        __syncwarp();
        for (int r = lane; r < R; r += 32) {
          const float* src = base + (long long)(rg * R + r) * ld + col;
          const uint32_t dst = ptx::smem_u32(smem + s * stage_bytes + r * seg);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
              "l"(src), "r"(seg), "r"(ptx::smem_u32(&full[s]))
              : "memory");
        }
      }
    }
  } else if (threadIdx.x == 32) {
    float acc = 0.f;
    for (int i = 0; i < nst; ++i) {
      const int s = i % stages;
      ptx::mbar_wait(&full[s], (i / stages) & 1);
      acc += ptx::lds_f32(ptx::smem_u32(smem + s * stage_bytes + 4 * (i & 31)));
      ptx::mbar_arrive(&empty[s]);
    }
    if (acc == 1234.5f) sink[0] = acc;
  }
}

// LDG reference: each thread UNR float4 loads in flight
template <int UNR>
__global__ void __launch_bounds__(512) ldg_kernel(const float* th, long long ld, int nrows, long long cols_per_cta,
                                                  float* sink) {
  const long long c0 = blockIdx.x * cols_per_cta;
  const int per_row4 = (int)(cols_per_cta / 4);
  float acc = 0.f;
  const long long total = (long long)nrows * per_row4;
  for (long long b = threadIdx.x; b < total; b += 512LL * UNR) {
    float4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const long long e = b + 512LL * u;
      if (e < total) {
        const int r = (int)(e / per_row4), c4 = (int)(e % per_row4);
        v[u] = __ldg(reinterpret_cast<const float4*>(th + (long long)r * ld + c0 + 4 * c4));
      } else
        v[u] = make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) sink[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;

int main() {
  const int n = 64;
  const long long ld = 1053312;
  float *th, *sink;
  cudaMalloc(&th, sizeof(float) * n * ld);
  cudaMalloc(&sink, 4);
  cudaMemset(th, 0, sizeof(float) * n * ld);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch, double bytes, const char* name) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(a);
    for (int w = 0; w < 10; ++w) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("%-48s %8.2f us  %7.1f GB/s %s\n", name, ms * 100, bytes / (ms / 10 * 1e-3) / 1e9,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  auto mkmap = [&](CUtensorMap* m, int box0, int box1, CUtensorMapSwizzle swz) {
    cuuint64_t dims[3] = {(cuuint64_t)ld, (cuuint64_t)n, 1};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)ld * n * 4};
    cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)box1, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, th, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  };
  cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  char name[128];
  for (int bw : {128, 132, 136, 144}) {
    for (int R : {32, 64}) {
      for (int stages : {3, 4, 6}) {
        const int sb = bw * R * 4;
        if (stages * sb > 224 * 1024) continue;
        CUtensorMap m;
        mkmap(&m, bw, R, CU_TENSOR_MAP_SWIZZLE_NONE);
        const int grid = 148, cps = 128;
        const long long cpc = (ld / grid) / cps * cps;
        const double bytes = 4.0 * R * cpc * grid;
        snprintf(name, sizeof name, "padded box %dx%d stages %d (%d KB)", bw, R, stages, stages * sb / 1024);
        timeit([&] {
          ring_kernel<<<grid, 64, stages * sb + 2048>>>(m, th, ld, 3, R, 1, sb, stages, cpc, cps, R, sink);
        }, bytes, name);
      }
    }
  }
  for (int per_sm : {1, 2}) {
    const int grid = 148 * per_sm;
    const int budget = (224 / per_sm) * 1024;  // ring bytes per CTA
    // mode 0: gram pattern
    for (int nbox : {1, 2, 4, 8}) {
      const int sb = nbox * 64 * 128;
      for (int stages : {2, 4, 6, 8, 12, 16, 24}) {
        if (stages * sb > budget) continue;
        CUtensorMap m;
        mkmap(&m, 32, 64, CU_TENSOR_MAP_SWIZZLE_128B);
        const int cps = 32 * nbox;
        const long long cpc = (ld / grid) / cps * cps;
        const double bytes = 4.0 * n * cpc * grid;
        snprintf(name, sizeof name, "%d/SM box32x64 x%d stages %d (%d KB)", per_sm, nbox, stages, stages * sb / 1024);
        timeit([&] {
          ring_kernel<<<grid, 64, stages * sb + 2048>>>(m, th, ld, 0, 64, nbox, sb, stages, cpc, cps, n, sink);
        }, bytes, name);
      }
    }
    // mode 1: upd pattern (128 columns x R rows boxes)
    for (int R : {32, 64}) {
      for (int nbox : {1, 2}) {
        if (R * nbox > 64) continue;
        const int sb = nbox * R * 512;
        for (int stages : {2, 4, 6, 8, 12}) {
          if (stages * sb > budget) continue;
          CUtensorMap m;
          mkmap(&m, 128, R, CU_TENSOR_MAP_SWIZZLE_NONE);
          const int cps = 128;
          const long long cpc = (ld / grid) / cps * cps;
          const double bytes = 4.0 * n * cpc * grid;
          snprintf(name, sizeof name, "%d/SM box128x%d x%d stages %d (%d KB)", per_sm, R, nbox, stages,
                   stages * sb / 1024);
          timeit([&] {
            ring_kernel<<<grid, 64, stages * sb + 2048>>>(m, th, ld, 1, R, nbox, sb, stages, cpc, cps, n, sink);
          }, bytes, name);
        }
      }
    }
    // mode 2: 1-D bulk, 64 rows x seg
    for (int seg : {256, 512, 1024}) {
      const int sb = 64 * seg;
      for (int stages : {2, 3, 4, 6, 8}) {
        if (stages * sb > budget) continue;
        CUtensorMap m;
        mkmap(&m, 32, 64, CU_TENSOR_MAP_SWIZZLE_128B);
        const int cps = seg / 4;
        const long long cpc = (ld / grid) / cps * cps;
        const double bytes = 4.0 * n * cpc * grid;
        snprintf(name, sizeof name, "%d/SM bulk 64x%dB stages %d (%d KB)", per_sm, seg, stages, stages * sb / 1024);
        timeit([&] {
          ring_kernel<<<grid, 64, stages * sb + 2048>>>(m, th, ld, 2, 64, 1, sb, stages, cpc, cps, n, sink);
        }, bytes, name);
      }
    }
    {
      const long long cpc = (ld / grid) / 4 * 4;
      const double bytes = 4.0 * n * cpc * grid;
      snprintf(name, sizeof name, "%d/SM ldg 512 thr x8 float4", per_sm);
      timeit([&] { ldg_kernel<8><<<grid, 512>>>(th, ld, n, cpc, sink); }, bytes, name);
    }
  }
  return 0;
}
