// Internal: device-memory handles and the gi_matrix struct shared by capi.cu
// and fit.cu.  Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"

#define CHECK_ARG(cond, msg)   \
  do {                         \
    if (!(cond)) {             \
      gi_set_error("%s", msg); \
      return -1;               \
    }                          \
  } while (0)

#define TRY(expr)                 \
  do {                            \
    if ((expr) != 0) return -1;   \
  } while (0)

namespace gi_internal {

struct DevMem {
  void* ptr = nullptr;
  int device = 0;
  ~DevMem() {
    if (ptr) {
      int prev = 0;
      cudaGetDevice(&prev);
      cudaSetDevice(device);
      cudaFree(ptr);
      cudaSetDevice(prev);
    }
  }
};

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

inline int alloc(std::shared_ptr<DevMem>& out, size_t bytes, int device, bool zero) {
  out = std::make_shared<DevMem>();
  out->device = device;
  if (bytes == 0) bytes = 16;
  GI_CUDA_TRY(cudaMalloc(&out->ptr, bytes));
  if (zero) GI_CUDA_TRY(cudaMemset(out->ptr, 0, bytes));
  return 0;
}

// grow-only scratch buffer
struct Scratch {
  std::shared_ptr<DevMem> mem;
  size_t bytes = 0;
  int ensure(size_t want, int device) {
    if (want <= bytes && mem) return 0;
    TRY(alloc(mem, want, device, false));
    bytes = want;
    return 0;
  }
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(mem->ptr);
  }
};

inline int sm_count_of(int device) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return sms;
}

}  // namespace gi_internal
using namespace gi_internal;

struct gi_matrix {
  int device = 0;
  int sms = 148;
  int64_t n = 0, p = 0, nb = 0, T = 0, G = 0;
  std::shared_ptr<DevMem> x;         // swizzled tiles (shared by with_stats copies)
  std::shared_ptr<DevMem> miss_cnt;  // int32[p]
  std::shared_ptr<DevMem> gmiss;     // uint8[G]
  std::shared_ptr<DevMem> s1cnt;     // int32[2p]: sum of dosages, observed count (all rows)
  std::shared_ptr<DevMem> u, v;      // fp64[p], owned per handle
  cudaStream_t stream = nullptr;
  std::mutex mu;
  Scratch s_a, s_b, s_c, s_d;
  // workspaces of the native fit loop (fit.cu): a pool, so independent fits on
  // one matrix run concurrently, each on its own stream.  Shared with the
  // with_stats copies (a workspace depends on the shape, not on the stats).
  struct FitPool {
    std::mutex mu;
    std::vector<std::shared_ptr<void>> items;
  };
  std::shared_ptr<FitPool> fit_pool = std::make_shared<FitPool>();

  gi::MatrixDesc desc() const {
    gi::MatrixDesc d;
    d.x = x ? static_cast<const uint8_t*>(x->ptr) : nullptr;
    d.n = n;
    d.p = p;
    d.nb = nb;
    d.T = T;
    d.G = G;
    return d;
  }
  double* du() const { return static_cast<double*>(u->ptr); }
  double* dv() const { return static_cast<double*>(v->ptr); }
  ~gi_matrix() {
    if (stream) {
      DeviceGuard g(device);
      cudaStreamDestroy(stream);
    }
  }
};

