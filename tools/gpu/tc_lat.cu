// tcgen05 i8 MMA timing from one issuing thread (M=128, N=8, K=32, A in TMEM):
//  (a) issue cost per MMA + commit (no wait),  (b) MMA -> commit -> mbarrier
//  completion latency seen by a waiter.
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n@!P1 bra W%=;\n}\n" ::"r"(bar), "r"(ph), "r"(0x989680u) : "memory");
}
__global__ void lat(int iters, int mode, long long* out) {
  __shared__ __align__(1024) uint8_t sB[8 * 32 * 4];
  __shared__ uint32_t th;
  __shared__ __align__(8) uint64_t bar[8];
  for (int i = threadIdx.x; i < (int)sizeof(sB); i += blockDim.x) sB[i] = 1;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&th)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[i])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = th;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 10) | (1u << 17) | (8u << 24);
    const uint32_t sa = su32(sB);
    const uint64_t bd = (uint64_t)((sa >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
    long long t0 = clock64();
    uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < iters; ++i) {
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n}\n" ::"r"(t + 256), "r"(t), "l"(bd), "r"(idesc), "r"(1u), "r"(0u), "r"(0u), "r"(0u), "r"(0u) : "memory");
      if (mode >= 1) {
        const int b = i & 7;
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[b])) : "memory");
        if (mode == 2) { wait_bar(su32(&bar[b]), ph[b]); ph[b] ^= 1u; }
        if (mode == 1 && i >= 7) { const int b2 = (i + 1) & 7; wait_bar(su32(&bar[b2]), ph[b2]); ph[b2] ^= 1u; }
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "n"(512));
}
int main() {
  long long* d; cudaMalloc(&d, 8 * 148);
  const char* names[3] = {"mma only", "mma+commit, wait 7 behind", "mma+commit+wait (latency)"};
  for (int mode = 0; mode < 3; ++mode) {
    const int iters = 4096;
    lat<<<148, 128>>>(iters, mode, d); cudaDeviceSynchronize();
    lat<<<148, 128>>>(iters, mode, d); cudaError_t e = cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%-28s: %.1f cycles per iteration (%s)\n", names[mode], mx / iters, cudaGetErrorString(e));
  }
  return 0;
}
