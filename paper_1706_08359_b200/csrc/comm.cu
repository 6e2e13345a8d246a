// comm.cu — NCCL implementation of the row-sharded allreduce hook.
//
// One process per GPU; ranks exchange a 128-byte ncclUniqueId out of band
// (bench.py uses torch.distributed for that plumbing) and build a
// communicator. hbg_comm_allreduce matches hbg_allreduce_fn: an in-place fp64
// SUM on the caller's stream over NVLink/NVSwitch. The leaf histogram is SoA
// fp64 with counts as exact integers, so one collective covers all three
// statistics. NCCL is loaded with dlopen so libhbg.so itself has no hard
// dependency on it (single-GPU users never need it).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "hbg_internal.h"

namespace hbg {
namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.handle) break;
    }
    if (!api.handle) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(api.handle, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(api.handle, "ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(api.handle, "ncclAllReduce"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(api.handle, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(api.handle, "ncclGetErrorString"));
  });
  if (!api.handle || !api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy)
    throw Error(HBG_ERR_NCCL, "NCCL (libnccl.so.2) is not available");
  return api;
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const auto& api = nccl();
  throw Error(HBG_ERR_NCCL, std::string(what) + ": " + (api.error_string ? api.error_string(r) : "nccl error"));
}

}  // namespace
}  // namespace hbg

struct hbg_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, device = 0;
};

using namespace hbg;

extern "C" {

int hbg_comm_get_unique_id(uint8_t* out) {
  return guarded_call([&] {
    require(out != nullptr, "null output");
    static_assert(sizeof(ncclUniqueId) == HBG_COMM_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    check_nccl(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof id);
  });
}

int hbg_comm_init(hbg_comm** out, int32_t nranks, int32_t rank, const uint8_t* unique_id, int32_t device) {
  return guarded_call([&] {
    require(out != nullptr && unique_id != nullptr, "null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank/nranks");
    *out = nullptr;
    int prev = 0;
    HBG_CUDA(cudaGetDevice(&prev));
    HBG_CUDA(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof id);
    auto* c = new hbg_comm;
    c->rank = rank;
    c->nranks = nranks;
    c->device = device;
    ncclResult_t r = nccl().comm_init_rank(&c->comm, nranks, id, rank);
    cudaSetDevice(prev);
    if (r != ncclSuccess) {
      delete c;
      check_nccl(r, "ncclCommInitRank");
    }
    *out = c;
  });
}

int hbg_comm_destroy(hbg_comm* comm) {
  return guarded_call([&] {
    if (!comm) return;
    if (comm->comm) nccl().comm_destroy(comm->comm);
    delete comm;
  });
}

int hbg_comm_allreduce(double* d_buf, int64_t n_values, void* stream, void* ctx) {
  return guarded_call([&] {
    auto* c = static_cast<hbg_comm*>(ctx);
    require(c != nullptr && c->comm != nullptr, "null communicator");
    if (n_values == 0) return;
    check_nccl(nccl().all_reduce(d_buf, d_buf, static_cast<size_t>(n_values), ncclFloat64, ncclSum,
                                 c->comm, static_cast<cudaStream_t>(stream)),
               "ncclAllReduce");
  });
}

}  // extern "C"
