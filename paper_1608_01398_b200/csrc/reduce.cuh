// Deterministic block / grid reductions shared by the solver kernels
// (solver.cu) and the fused image norm of ax.cu: fixed grids write per-block
// partials and the last block to finish (threadfence + atomic ticket) folds
// them in block order, so repeated runs and any stream interleaving give
// identical bits.
#pragma once

#include "common.cuh"

namespace gi {

constexpr int kRedBlocks = 296;
constexpr int kRedThreads = 256;

struct RedWs {
  double* partials;        // kRedBlocks * 8
  unsigned int* ticket;    // 1 counter, zero-initialised
};

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ double warp_max(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// block-wide sum of NV values per thread; result valid in thread 0
template <int NV>
__device__ __forceinline__ void block_sum(double (&x)[NV], double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    x[q] = warp_sum(x[q]);
    if (lane == 0) sh[q * 32 + warp] = x[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += sh[q * 32 + w];
      x[q] = s;
    }
  }
  __syncthreads();
}

// Deterministic fold of per-block partials by the first warp of the last
// block: lane l sums partials l, l+32, ... in order, then a fixed xor tree.
// The loop is unrolled over the grids the kernels launch (<= 2 kRedBlocks
// blocks) with predicated loads, so a lane's loads all issue before its adds
// instead of one L2 round trip per partial; the additions keep their order
// (b = lane, lane + 32, ...), so the sums are the same bits as a plain loop.
constexpr int kFoldUnroll = (2 * kRedBlocks + 31) / 32;

__device__ __forceinline__ double fold_sum(const double* partials, int stride, int slot,
                                           unsigned nblocks) {
  const unsigned lane = threadIdx.x & 31;
  double v[kFoldUnroll];
#pragma unroll
  for (int q = 0; q < kFoldUnroll; ++q) {
    const unsigned b = lane + 32u * q;
    v[q] = b < nblocks ? partials[b * stride + slot] : 0.0;
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < kFoldUnroll; ++q)
    if (lane + 32u * q < nblocks) s += v[q];
  for (unsigned b = lane + 32u * kFoldUnroll; b < nblocks; b += 32) s += partials[b * stride + slot];
  return warp_sum(s);
}

__device__ __forceinline__ double fold_max(const double* partials, unsigned nblocks) {
  const unsigned lane = threadIdx.x & 31;
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < kFoldUnroll; ++q) {
    const unsigned b = lane + 32u * q;
    if (b < nblocks) s = fmax(s, partials[b]);
  }
  for (unsigned b = lane + 32u * kFoldUnroll; b < nblocks; b += 32) s = fmax(s, partials[b]);
  return warp_max(s);
}

// returns true in every thread of the last block to arrive
__device__ __forceinline__ bool last_block(unsigned int* ticket) {
  __shared__ bool is_last;
  __threadfence();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(ticket, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  return is_last;
}

}  // namespace gi
