// tcgen05.mma kind::i8 issue rate vs N (M=128, K=32, A from TMEM, B from smem):
// one CTA per SM issues `iters` MMAs back to back into one accumulator.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_rate tc_rate.cu && ./tc_rate
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int N, int NACC, bool SS, int ISSUERS = 1>
__global__ void rate(int iters, long long* cycles) {
  __shared__ __align__(1024) uint8_t sB[256 * 128];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 256 * 128; i += blockDim.x) sB[i] = (uint8_t)(i * 7);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(ISSUERS));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base;
  if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < ISSUERS) {
    const int who = threadIdx.x >> 5;
    constexpr uint32_t LBO = (N / 8) * 128, SBO = 128;
    const uint32_t idesc = (2u << 4) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint32_t saddr = smem_u32(sB);
    const uint64_t bdesc = (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(LBO >> 4) << 16) |
                           ((uint64_t)(SBO >> 4) << 32) | (1ull << 46);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = i > 0;
      const uint32_t dcol = tbase + 256 + (uint32_t)(((i % NACC) * (N < 32 ? 32 : N) + who * 128) % 256);
      if (SS) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n}\n" ::"r"(
                dcol),
            "l"(bdesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
            : "memory");
      } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n}\n" ::"r"(
                dcol),
            "r"(tbase + 8 * (i & 15)), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u),
            "r"(0u)
            : "memory");
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar))
        : "memory");
    if (who == 0) asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::
            "r"(smem_u32(&bar)), "r"(0u)
        : "memory");
    if (who == 0) cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(512));
}

template <int N, int NACC, bool SS, int ISSUERS = 1>
void run(long long* d) {
  const int iters = 20000;
  rate<N, NACC, SS, ISSUERS><<<148, 128>>>(iters, d);
  cudaDeviceSynchronize();
  rate<N, NACC, SS, ISSUERS><<<148, 128>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("N=%3d acc=%d %s issuers=%d: %.2f cycles per MMA, %.0f MAC/clk/SM (%s)\n", N, NACC,
         SS ? "A smem" : "A tmem", ISSUERS, mx / iters / ISSUERS,
         128.0 * N * 32 * iters * ISSUERS / mx, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  run<8, 1, false>(d);
  run<8, 1, false, 2>(d);
  run<8, 1, false, 4>(d);
  run<32, 1, false, 2>(d);
  run<64, 1, false, 2>(d);
  run<8, 1, true, 2>(d);
  return 0;
}
