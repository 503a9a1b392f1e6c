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
// ncclCommInitRankConfig with maxCTAs = max_ctas (NCCL 2.28 config struct): caps the SMs the collectives
// take from the concurrently running GEMMs (the Theta all-gather overlaps the gradient phase)
push_status comm_init_rank(Comm* comm, int nranks, const UniqueId& id, int rank, int max_ctas = 0);
// ncclCommCount (the communicator's rank count, checked against world_size after init)
push_status comm_count(Comm comm, int* count);
// ncclCommGetAsyncError: PUSH_OK, or PUSH_E_NCCL with the error text (a failed or aborted peer)
push_status async_error(Comm comm);
// in-place when send == recv + rank*count
push_status allgather_f32(const float* send, float* recv, size_t count, Comm comm, cudaStream_t s);
// grouped point-to-point (the NEXT-4 all-to-all transposes): group_start; send/recv ...; group_end
push_status group_start();
push_status group_end();
push_status send_f32(const float* buf, size_t count, int peer, Comm comm, cudaStream_t s);
push_status recv_f32(float* buf, size_t count, int peer, Comm comm, cudaStream_t s);
void comm_release(Comm comm, bool abort);
}  // namespace nccl
}  // namespace push
