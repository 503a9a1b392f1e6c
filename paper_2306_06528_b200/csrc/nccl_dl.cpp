// nccl_dl.cpp — NCCL loaded at run time (dlopen "libnccl.so.2"), so single-GPU use of
// the library has no NCCL dependency and multi-rank use binds to whichever libnccl
// the process already has loaded (torch's bundled one when torch is imported first).
#include "nccl_dl.h"

#include <dlfcn.h>
#include <nccl.h>  // types only (ncclConfig_t, NCCL_CONFIG_INITIALIZER); every call goes through dlsym

#include <mutex>
#include <string>

#include "common.cuh"

namespace push {
namespace nccl {
namespace {
using Result = int;  // ncclResult_t; 0 = ncclSuccess
using FnGetUniqueId = Result (*)(UniqueId*);
using FnCommInitRank = Result (*)(Comm*, int, UniqueId, int);
using FnAllGather = Result (*)(const void*, void*, size_t, int, Comm, cudaStream_t);
using FnCommDestroy = Result (*)(Comm);
using FnSend = Result (*)(const void*, size_t, int, int, Comm, cudaStream_t);
using FnRecv = Result (*)(void*, size_t, int, int, Comm, cudaStream_t);
using FnGroup = Result (*)();
using FnGetErrorString = const char* (*)(Result);
using FnCommInitRankConfig = Result (*)(Comm*, int, UniqueId, int, ncclConfig_t*);
using FnCommCount = Result (*)(Comm, int*);
using FnGetAsyncError = Result (*)(Comm, Result*);

struct Api {
  void* h = nullptr;
  FnGetUniqueId get_unique_id = nullptr;
  FnCommInitRank comm_init_rank = nullptr;
  FnAllGather all_gather = nullptr;
  FnCommDestroy comm_destroy = nullptr;
  FnCommDestroy comm_abort = nullptr;
  FnSend send = nullptr;
  FnRecv recv = nullptr;
  FnGroup group_start = nullptr, group_end = nullptr;
  FnGetErrorString err = nullptr;
  FnCommInitRankConfig init_config = nullptr;
  FnCommCount count = nullptr;
  FnGetAsyncError async_err = nullptr;
  std::string why;
};
Api g_api;
std::once_flag g_once;

constexpr int kNcclFloat32 = 7;  // ncclDataType_t ncclFloat32

push_status nfail(const char* what, Result r) {
  std::string m = std::string(what) + " failed: ";
  m += g_api.err ? g_api.err(r) : std::to_string(r);
  return fail(PUSH_E_NCCL, m);
}
}  // namespace

push_status load() {
  std::call_once(g_once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      g_api.why = e ? e : "dlopen(libnccl.so.2) failed";
      return;
    }
    g_api.h = h;
    g_api.get_unique_id = reinterpret_cast<FnGetUniqueId>(dlsym(h, "ncclGetUniqueId"));
    g_api.comm_init_rank = reinterpret_cast<FnCommInitRank>(dlsym(h, "ncclCommInitRank"));
    g_api.all_gather = reinterpret_cast<FnAllGather>(dlsym(h, "ncclAllGather"));
    g_api.comm_destroy = reinterpret_cast<FnCommDestroy>(dlsym(h, "ncclCommDestroy"));
    g_api.comm_abort = reinterpret_cast<FnCommDestroy>(dlsym(h, "ncclCommAbort"));
    g_api.err = reinterpret_cast<FnGetErrorString>(dlsym(h, "ncclGetErrorString"));
    g_api.send = reinterpret_cast<FnSend>(dlsym(h, "ncclSend"));
    g_api.recv = reinterpret_cast<FnRecv>(dlsym(h, "ncclRecv"));
    g_api.group_start = reinterpret_cast<FnGroup>(dlsym(h, "ncclGroupStart"));
    g_api.group_end = reinterpret_cast<FnGroup>(dlsym(h, "ncclGroupEnd"));
    g_api.init_config = reinterpret_cast<FnCommInitRankConfig>(dlsym(h, "ncclCommInitRankConfig"));
    g_api.count = reinterpret_cast<FnCommCount>(dlsym(h, "ncclCommCount"));
    g_api.async_err = reinterpret_cast<FnGetAsyncError>(dlsym(h, "ncclCommGetAsyncError"));
    if (!g_api.get_unique_id || !g_api.comm_init_rank || !g_api.all_gather || !g_api.comm_destroy || !g_api.send ||
        !g_api.recv || !g_api.group_start || !g_api.group_end)
      g_api.why = "libnccl.so.2 lacks required symbols";
  });
  if (!g_api.why.empty()) return fail(PUSH_E_NCCL, g_api.why);
  return PUSH_OK;
}

push_status get_unique_id(UniqueId* id) {
  push_status st = load();
  if (st != PUSH_OK) return st;
  Result r = g_api.get_unique_id(id);
  return r ? nfail("ncclGetUniqueId", r) : PUSH_OK;
}

push_status comm_init_rank(Comm* comm, int nranks, const UniqueId& id, int rank, int max_ctas) {
  push_status st = load();
  if (st != PUSH_OK) return st;
  if (max_ctas > 0 && g_api.init_config) {
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.maxCTAs = max_ctas;
    Result r = g_api.init_config(comm, nranks, id, rank, &cfg);
    return r ? nfail("ncclCommInitRankConfig", r) : PUSH_OK;
  }
  Result r = g_api.comm_init_rank(comm, nranks, id, rank);
  return r ? nfail("ncclCommInitRank", r) : PUSH_OK;
}

push_status comm_count(Comm comm, int* count) {
  if (!g_api.count) return fail(PUSH_E_NCCL, "ncclCommCount not available");
  Result r = g_api.count(comm, count);
  return r ? nfail("ncclCommCount", r) : PUSH_OK;
}

push_status async_error(Comm comm) {
  if (!comm || !g_api.async_err) return PUSH_OK;
  Result e = 0;
  Result r = g_api.async_err(comm, &e);
  if (r) return nfail("ncclCommGetAsyncError", r);
  return e ? nfail("NCCL asynchronous error", e) : PUSH_OK;
}

push_status allgather_f32(const float* send, float* recv, size_t count, Comm comm, cudaStream_t s) {
  Result r = g_api.all_gather(send, recv, count, kNcclFloat32, comm, s);
  return r ? nfail("ncclAllGather", r) : PUSH_OK;
}

push_status group_start() {
  Result r = g_api.group_start();
  return r ? nfail("ncclGroupStart", r) : PUSH_OK;
}
push_status group_end() {
  Result r = g_api.group_end();
  return r ? nfail("ncclGroupEnd", r) : PUSH_OK;
}
push_status send_f32(const float* buf, size_t count, int peer, Comm comm, cudaStream_t s) {
  Result r = g_api.send(buf, count, kNcclFloat32, peer, comm, s);
  return r ? nfail("ncclSend", r) : PUSH_OK;
}
push_status recv_f32(float* buf, size_t count, int peer, Comm comm, cudaStream_t s) {
  Result r = g_api.recv(buf, count, kNcclFloat32, peer, comm, s);
  return r ? nfail("ncclRecv", r) : PUSH_OK;
}

void comm_release(Comm comm, bool abort) {
  if (!comm || !g_api.h) return;
  if (abort && g_api.comm_abort)
    g_api.comm_abort(comm);
  else
    g_api.comm_destroy(comm);
}

}  // namespace nccl
}  // namespace push
