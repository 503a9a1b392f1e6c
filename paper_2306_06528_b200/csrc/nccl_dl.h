// nccl_dl.h — minimal run-time binding to NCCL (only the calls the SVGD exchange needs).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

#include "../../include/push.h"

namespace push {
namespace nccl {
struct UniqueId {
  char internal[128];
};
using Comm = void*;

push_status load();
push_status get_unique_id(UniqueId* id);
push_status comm_init_rank(Comm* comm, int nranks, const UniqueId& id, int rank);
// in-place when send == recv + rank*count
push_status allgather_f32(const float* send, float* recv, size_t count, Comm comm, cudaStream_t s);
void comm_release(Comm comm, bool abort);
}  // namespace nccl
}  // namespace push
