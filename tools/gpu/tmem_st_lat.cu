// tcgen05.st.32x32b.x16 cost: store + wait::st per iteration, and 4 stores per wait.
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(int iters, int per_wait, int warps_active, long long* out) {
  __shared__ uint32_t th;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&th)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = th;
  const int warp = threadIdx.x / 32;
  uint32_t v[16];
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 16 + i;
  long long t0 = clock64();
  if (warp < warps_active) {
    const uint32_t base = t + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
    for (int i = 0; i < iters; ++i) {
      for (int q = 0; q < per_wait; ++q) {
        const uint32_t a = base + (uint32_t)(q * 16 % 128);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(a),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      v[0] += 1;
    }
  }
  long long dt = clock64() - t0;
  if (threadIdx.x == 0) out[blockIdx.x] = dt;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "n"(512));
}
int main() {
  long long* d; cudaMalloc(&d, 8 * 148);
  int cfg[][2] = {{1, 1}, {4, 1}, {1, 4}, {4, 4}, {8, 4}, {1, 8}, {8, 8}};
  for (auto& c : cfg) {
    const int iters = 2000;
    k<<<148, 256>>>(iters, c[1], c[0], d); cudaDeviceSynchronize();
    k<<<148, 256>>>(iters, c[1], c[0], d); cudaError_t e = cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("warps=%d stores/wait=%d: %.1f cycles per iteration, %.1f per store (%s)\n", c[0], c[1], mx / iters, mx / iters / c[1], cudaGetErrorString(e));
  }
  return 0;
}
