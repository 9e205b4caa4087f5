// Probe of the tcgen05 int8 MMA conventions the X^T R kernel relies on
// (sm_100a): A (u8 doses) written to TMEM by tcgen05.st.32x32b (lane = row m,
// 4 K-bytes per 32-bit column), B (s8 residual digits) in shared memory in the
// canonical K-major no-swizzle layout, D (s32) in TMEM read back by
// tcgen05.ld.32x32b.  Compares D with a host GEMM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe tc_probe.cu && ./tc_probe
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int N, int K>
__global__ void probe(const uint8_t* A, const int8_t* B, int32_t* D) {
  __shared__ __align__(1024) uint8_t sB[N * K];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr uint32_t LBO = (N / 8) * 128, SBO = 128;
  for (int idx = threadIdx.x; idx < N * K; idx += blockDim.x) {
    const int n = idx / K, k = idx % K;
    sB[(k / 16) * LBO + (n / 8) * SBO + (n % 8) * 16 + (k % 16)] = (uint8_t)B[idx];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base;
  const int m = threadIdx.x;  // row of A = TMEM lane
  for (int c = 0; c < K / 4; c += 4) {
    uint32_t v[4];
    for (int q = 0; q < 4; ++q) {
      const uint8_t* src = A + m * K + 4 * (c + q);
      v[q] = src[0] | (src[1] << 8) | (src[2] << 16) | ((uint32_t)src[3] << 24);
    }
    const uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16) + c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
                 : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  constexpr uint32_t DCOL = 64;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint32_t a_t = tbase + 8 * ks;
      const uint32_t saddr = smem_u32(sB) + ks * 2 * LBO;
      const uint64_t bdesc = (uint64_t)((saddr >> 4) & 0x3FFF) |
                             ((uint64_t)((LBO >> 4) & 0x3FFF) << 16) |
                             ((uint64_t)((SBO >> 4) & 0x3FFF) << 32) | (1ull << 46);
      const uint32_t acc = ks > 0 ? 1u : 0u;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n}\n" ::"r"(
              tbase + DCOL),
          "r"(a_t), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
          : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar))
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::
          "r"(smem_u32(&bar)),
      "r"(0u)
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "r"(tbase + ((uint32_t)(32 * warp) << 16) + DCOL + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int q = 0; q < 8; ++q) D[m * N + c + q] = (int32_t)r[q];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(128));
  (void)lane;
}

template <int N, int K>
int run() {
  std::vector<uint8_t> A(128 * K);
  std::vector<int8_t> B(N * K);
  srand(N * 1000 + K);
  for (auto& x : A) x = rand() % 3;
  for (auto& x : B) x = (int8_t)(rand() % 128 - 64);
  uint8_t* dA;
  int8_t* dB;
  int32_t* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xFF, 128 * N * 4);
  probe<N, K><<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<int32_t> D(128 * N);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      int32_t want = 0;
      for (int k = 0; k < K; ++k) want += (int32_t)A[m * K + k] * (int32_t)B[n * K + k];
      if (want != D[m * N + n]) {
        if (bad < 5) printf("  m=%d n=%d got %d want %d\n", m, n, D[m * N + n], want);
        ++bad;
      }
    }
  printf("N=%d K=%d: %s, %d mismatches (%s)\n", N, K, bad ? "FAIL" : "ok", bad,
         cudaGetErrorString(e));
  return bad;
}

int main() {
  int bad = 0;
  bad += run<8, 32>();
  bad += run<8, 64>();
  bad += run<16, 128>();
  bad += run<32, 64>();
  return bad != 0;
}
