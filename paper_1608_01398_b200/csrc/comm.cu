// Communicators of the sharded native loop (gi_fit_sharded).
//
// Two backends behind one interface:
//   * NCCL -- production multi-GPU (one process per GPU).  libnccl.so.2 is
//     opened with dlopen at first use (the copy torch already loaded, else the
//     system one), so the library has no link-time NCCL dependency.  n-length
//     partial products are all-reduced in place on the fit's stream.
//   * host callbacks -- the caller supplies all-reduce / all-gather on host
//     buffers (e.g. torch.distributed with gloo); device buffers are staged
//     through the host.  Lets the same sharded loop run and be tested where
//     several ranks share one GPU.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <vector>

#include "../../include/genoiht_cuda.h"
#include "comm.cuh"
#include "handle.cuh"

namespace {

struct NcclApi {
  bool ready = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank =
        reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ready = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.all_gather &&
                api.comm_destroy;
  });
  return api;
}

#define NCCL_TRY(expr)                                                                    \
  do {                                                                                    \
    ncclResult_t _r = (expr);                                                             \
    if (_r != ncclSuccess) {                                                              \
      gi_set_error("%s failed: %s", #expr,                                                \
                   nccl().error_string ? nccl().error_string(_r) : "NCCL error");         \
      return -1;                                                                          \
    }                                                                                     \
  } while (0)

}  // namespace

// ------------------------------------------------------------------ collectives
int gi_comm::allreduce_device(double* dbuf, int64_t count, int op, cudaStream_t s) {
  if (count <= 0) return 0;
  if (kind == kNccl) {  // also at world 1: a real (local) NCCL collective
    NCCL_TRY(nccl().all_reduce(dbuf, dbuf, (size_t)count, ncclFloat64, op ? ncclMax : ncclSum,
                               static_cast<ncclComm_t>(nccl_comm), s));
    return 0;
  }
  if (world <= 1) return 0;
  std::vector<double> host((size_t)count);
  GI_CUDA_TRY(cudaMemcpyAsync(host.data(), dbuf, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
  GI_CUDA_TRY(cudaStreamSynchronize(s));
  if (allreduce(ctx, host.data(), count, op) != 0) {
    gi_set_error("host all-reduce callback failed");
    return -1;
  }
  GI_CUDA_TRY(cudaMemcpyAsync(dbuf, host.data(), sizeof(double) * count, cudaMemcpyHostToDevice, s));
  GI_CUDA_TRY(cudaStreamSynchronize(s));
  return 0;
}

int gi_comm::allgather_device(const double* dsend, int64_t count, double* drecv,
                              cudaStream_t s) {
  if (count <= 0) return 0;
  if (kind == kNccl) {  // also at world 1: a real (local) NCCL collective
    NCCL_TRY(nccl().all_gather(dsend, drecv, (size_t)count, ncclFloat64,
                               static_cast<ncclComm_t>(nccl_comm), s));
    return 0;
  }
  if (world <= 1) {
    GI_CUDA_TRY(cudaMemcpyAsync(drecv, dsend, sizeof(double) * count, cudaMemcpyDeviceToDevice,
                                s));
    return 0;
  }
  std::vector<double> mine((size_t)count), all((size_t)(count * world));
  GI_CUDA_TRY(cudaMemcpyAsync(mine.data(), dsend, sizeof(double) * count, cudaMemcpyDeviceToHost,
                              s));
  GI_CUDA_TRY(cudaStreamSynchronize(s));
  if (allgather(ctx, mine.data(), count, all.data()) != 0) {
    gi_set_error("host all-gather callback failed");
    return -1;
  }
  GI_CUDA_TRY(cudaMemcpyAsync(drecv, all.data(), sizeof(double) * count * world,
                              cudaMemcpyHostToDevice, s));
  GI_CUDA_TRY(cudaStreamSynchronize(s));
  return 0;
}

gi_comm::~gi_comm() {
  if (kind == kNccl && nccl_comm && nccl().ready)
    nccl().comm_destroy(static_cast<ncclComm_t>(nccl_comm));
}

// ------------------------------------------------------------------ C ABI
extern "C" {

int gi_comm_nccl_available(void) { return nccl().ready ? 1 : 0; }

int gi_comm_nccl_unique_id(uint8_t* out) {
  CHECK_ARG(out != nullptr, "NULL argument");
  CHECK_ARG(nccl().ready, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  NCCL_TRY(nccl().get_unique_id(&id));
  memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}

int gi_comm_create_nccl(const uint8_t* id, int world, int rank, int device, gi_comm** out) {
  CHECK_ARG(id && out, "NULL argument");
  CHECK_ARG(world >= 1 && rank >= 0 && rank < world, "invalid world size / rank");
  CHECK_ARG(nccl().ready, "libnccl.so.2 could not be loaded");
  DeviceGuard g(device);
  ncclUniqueId uid;
  memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  NCCL_TRY(nccl().comm_init_rank(&c, world, uid, rank));
  gi_comm* comm = new gi_comm();
  comm->kind = gi_comm::kNccl;
  comm->world = world;
  comm->rank = rank;
  comm->device = device;
  comm->nccl_comm = c;
  *out = comm;
  return 0;
}

int gi_comm_create_callbacks(int world, int rank, void* ctx, gi_comm_allreduce_fn allreduce,
                             gi_comm_allgather_fn allgather, gi_comm** out) {
  CHECK_ARG(out && allreduce && allgather, "NULL argument");
  CHECK_ARG(world >= 1 && rank >= 0 && rank < world, "invalid world size / rank");
  gi_comm* comm = new gi_comm();
  comm->kind = gi_comm::kCallbacks;
  comm->world = world;
  comm->rank = rank;
  comm->ctx = ctx;
  comm->allreduce = allreduce;
  comm->allgather = allgather;
  *out = comm;
  return 0;
}

int gi_comm_free(gi_comm* comm) {
  delete comm;
  return 0;
}

}  // extern "C"
