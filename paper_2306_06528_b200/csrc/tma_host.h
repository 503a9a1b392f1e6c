// tma_host.h — host-side TMA tensor-map helpers shared by the tcgen05 kernels (gemm.cu, gram.cu).
#pragma once
#include <cuda.h>

#include <cstdint>

#include "../../include/push.h"

namespace push {
namespace gemm {
// Resolve cuTensorMapEncodeTiled from the driver (once); also records the SM count.
push_status get_encoder();
// SMs of the current device (valid after get_encoder()).
int sm_count();
// 3-D fp32 tensor map {d0 (contiguous), d1, d2}, element strides stride1 / stride2, box {box0, box1, 1},
// zero out-of-bounds fill.
push_status make_map(CUtensorMap* m, const float* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_el,
                     uint64_t stride2_el, uint32_t box1, CUtensorMapSwizzle swz, uint32_t box0 = 32);
}  // namespace gemm
}  // namespace push
