// Internal definition of gi_comm (see comm.cu).  Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/genoiht_cuda.h"

struct gi_comm {
  enum Kind { kNccl = 0, kCallbacks = 1 };
  int kind = kCallbacks;
  int world = 1, rank = 0, device = 0;
  void* nccl_comm = nullptr;  // ncclComm_t
  void* ctx = nullptr;
  gi_comm_allreduce_fn allreduce = nullptr;
  gi_comm_allgather_fn allgather = nullptr;

  // in-place all-reduce of a device buffer on stream s (op 0 = sum, 1 = max)
  int allreduce_device(double* dbuf, int64_t count, int op, cudaStream_t s);
  // all-gather of device buffers on stream s, recv = world x count rank-major
  // (NCCL: in the stream, no host sync; callbacks: staged through the host)
  int allgather_device(const double* dsend, int64_t count, double* drecv, cudaStream_t s);
  ~gi_comm();
};
