// Internal: device-memory handles and the gi_matrix struct shared by capi.cu
// and fit.cu.  Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <atomic>
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
      // like cudaFree: no stream may still be using the buffer; the bytes then
      // go back to the device pool (kept mapped, see device_pool) for reuse
      cudaDeviceSynchronize();
      cudaFreeAsync(ptr, 0);
      cudaSetDevice(prev);
    }
  }
};

// The device's default stream-ordered pool, set to keep up to a quarter of the
// device memory mapped after frees: CV fold copies and fit workspaces are
// allocated and dropped repeatedly, and re-mapping gigabytes through
// cudaMalloc/cudaFree costs milliseconds each.  Beyond that the driver returns
// freed memory at synchronisation points, so other allocators (torch) and
// processes get it back.
inline cudaMemPool_t device_pool(int device) {
  static std::mutex mu;
  static bool configured[64] = {};
  cudaMemPool_t pool = nullptr;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (device >= 0 && device < 64 && !configured[device]) {
    size_t free_b = 0, total_b = 0;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaMemGetInfo(&free_b, &total_b);
    cudaSetDevice(prev);
    uint64_t keep = (uint64_t)total_b / 4;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    configured[device] = true;
  }
  return pool;
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// Device buffer from the pool, usable from any stream on return.
inline int alloc(std::shared_ptr<DevMem>& out, size_t bytes, int device, bool zero) {
  out = std::make_shared<DevMem>();
  out->device = device;
  if (bytes == 0) bytes = 16;
  cudaMemPool_t pool = device_pool(device);
  cudaError_t e = cudaMallocAsync(&out->ptr, bytes, 0);
  if (e == cudaErrorMemoryAllocation && pool) {  // give back cached bytes, retry once
    cudaGetLastError();
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(&out->ptr, bytes, 0);
  }
  if (e != cudaSuccess) {
    out->ptr = nullptr;
    GI_CUDA_TRY(e);
  }
  if (zero) GI_CUDA_TRY(cudaMemsetAsync(out->ptr, 0, bytes, 0));
  GI_CUDA_TRY(cudaStreamSynchronize(0));
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
  std::shared_ptr<DevMem> x3;        // optional base-3 copy for X^T r (shared likewise)
  int64_t T3 = 0;
  std::shared_ptr<DevMem> mlist, mofs;  // missing-genotype lists beside x3 (missing.cu)
  int64_t mtotal = 0;                   // their entries
  std::shared_ptr<DevMem> miss_cnt;  // int32[p]
  std::shared_ptr<DevMem> gmiss;     // uint8[G]
  std::shared_ptr<DevMem> s1cnt;     // int32[2p]: sum of dosages, observed count (all rows)
  // a fold handle (gi_matrix_with_masked_stats): its rows (0/1 per sample) and
  // the (sum of dosages, observed count) pairs over them
  std::vector<uint8_t> fold_keep;
  std::shared_ptr<DevMem> fold_s1cnt;
  std::shared_ptr<DevMem> u, v;      // fp64[p], owned per handle
  cudaStream_t stream = nullptr;
  std::mutex mu;
  Scratch s_a, s_b, s_c, s_d, s_e;
  int any_missing = -1;              // cached: any genotype code 01 (-1: not known yet)
  // Identity of this handle.  The native fit loop's workspaces (fit.cu) live
  // in a process-wide pool per device keyed by shape, so fits on any matrix of
  // that shape (CV fold copies, with_stats copies) reuse them; the uid tells
  // the resident-input path which handle primed a workspace.
  uint64_t uid = next_uid();
  static uint64_t next_uid() {
    static std::atomic<uint64_t> counter{0};
    return ++counter;
  }

  gi::MatrixDesc desc() const {
    gi::MatrixDesc d;
    d.x = x ? static_cast<const uint8_t*>(x->ptr) : nullptr;
    d.n = n;
    d.p = p;
    d.nb = nb;
    d.T = T;
    d.G = G;
    d.x3 = x3 ? static_cast<const uint8_t*>(x3->ptr) : nullptr;
    d.T3 = x3 ? T3 : 0;
    d.mlist = x3 && mlist ? static_cast<const uint16_t*>(mlist->ptr) : nullptr;
    d.mofs = x3 && mofs ? static_cast<const int64_t*>(mofs->ptr) : nullptr;
    d.mtotal = d.mlist ? mtotal : 0;
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

