// Missing-genotype lists: X^T r over the base-3 copy for matrices WITH missing
// genotypes (BASELINE config 5).
//
// Reference: _aty_kernel geno_matrix.py:142-165 accumulates, per SNP j,
//   t_j = sum_i dose_ij r_i   and   m_j = sum_{i missing in j} r_i,
// and returns v_j (t_j - u_j (sum_r - m_j)).  The lookup-table kernel over the
// 2-bit tiles pays a second table lookup per packed byte for m_j (9 instead of
// 5 B of shared-memory traffic per byte; aty.cu), which bounds config 5 at
// ~0.53 of HBM.  Here m_j comes from a compact list of the missing positions
// instead, and t_j from the base-3 copy (layout.cu pack3_kernel maps the
// missing code to dose 0, so the base-3 sweep is exactly t_j):
//
//   list    per 4 KiB block (tile t of 512 samples, group g of 32 SNPs), one
//           uint16 per missing genotype: (SNP lane << 9) | sample offset,
//           round-robin over the lanes within windows of 32 samples; ofs[t G + g] = first entry of the
//           block (int64, T G + 1 entries).  At 2% missing that is 0.04 B per
//           genotype next to the base-3 stream's 0.2 (2-bit tiles: 0.25).
//   missum  one CTA per chunk of groups walks every tile in order: the tile's
//           fp32 centred residuals rt (the same rt the table kernels read) are
//           converted to fixed point in shared memory at a per-tile
//           power-of-two scale (|q| <= 2^21, so a block column's sum stays
//           below 2^31), each warp adds its block's entries with integer
//           shared-memory atomics (exact, so the result does not depend on
//           the order the atomics land in), and the per-tile sums are added to
//           an fp64 accumulator per SNP in tile order (deterministic).  m_j is
//           written to out[j]; the base-3 kernel's epilogue then adds u_j m_j
//           and overwrites out[j] with the gradient (aty.cu,
//           FastArgs::miss_in_out).  Block offsets, residual slice and entries
//           of the next tile are staged by bulk async copies (two stages).
//
// The fixed-point step rounds each rt to 2^-22 of its tile's max|rt|: over the
// ~n/50 missing genotypes of a column at 2% that is ~3e-5 rms(r), below the
// fp32-table error of the dose sums t_j themselves (~8e-5 rms(r) at n = 500k)
// and far inside the fast kernel's 2e-6 rms(g) bar.  (Exact 42-bit fixed
// point as two 21-bit halves cost a second atomic and an 8-byte read per
// entry: 10.1 ms for config 5's 5.1e9 entries, 14 shared-memory wavefronts
// per 32 entries.)
#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace gi {

namespace {

// missing codes (01) of a 2-bit word -> bit 2s of field s
__device__ __forceinline__ uint32_t missing_bits(uint32_t w) {
  return w & ~(w >> 1) & 0x55555555u;
}

// entries per block, one warp per block
__global__ void miss_count_kernel(MatrixDesc m, int64_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nblk = m.T * m.G;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t b = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); b < nblk;
       b += warps) {
    const uint32_t* blk = reinterpret_cast<const uint32_t*>(m.x + b * GI_BLOCK_BYTES);
    int c = 0;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) c += __popc(missing_bits(blk[q * 32 + lane]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[b] = c;
  }
}

// the 16 missing flags of a 2-bit word (bit s = sample s)
__device__ __forceinline__ uint32_t missing_mask16(uint32_t w) {
  uint32_t x = missing_bits(w);
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0F0F0F0Fu;
  x = (x | (x >> 4)) & 0x00FF00FFu;
  return (x | (x >> 8)) & 0x0000FFFFu;
}

// the entries, one warp per block, in windows of kWin words (16 kWin
// samples): lane L gathers the missing flags of SNP L over the window (word w
// at byte ((L ^ w) << 7) + 4 L of the swizzled block) and the window's entries
// are written round by round -- every lane's first missing sample, then every
// lane's second, ... -- so consecutive entries tend to name different SNPs
// (fewer colliding shared-memory atomics in missum_kernel) and nearby samples
// (fewer bank conflicts on the residual reads)
template <int kWin>
__global__ void miss_fill_kernel(MatrixDesc m, const int64_t* __restrict__ ofs,
                                 uint16_t* __restrict__ ent) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const int64_t nblk = m.T * m.G;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t b = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); b < nblk;
       b += warps) {
    const uint8_t* blk = m.x + b * GI_BLOCK_BYTES;
    int64_t pos = ofs[b];
    for (int w0 = 0; w0 < 32; w0 += kWin) {
      uint64_t mk = 0;
#pragma unroll
      for (int k = 0; k < kWin; ++k) {
        const int w = w0 + k;
        mk |= (uint64_t)missing_mask16(
                  *reinterpret_cast<const uint32_t*>(blk + ((lane ^ w) << 7) + (lane << 2)))
              << (16 * k);
      }
      while (true) {
        const uint32_t act = __ballot_sync(0xffffffffu, mk != 0);
        if (!act) break;
        if (mk) {
          const int bit = __ffsll((long long)mk) - 1;
          mk &= mk - 1;
          ent[pos + __popc(act & lt)] = (uint16_t)((lane << 9) | (16 * w0 + bit));
        }
        pos += __popc(act);
      }
    }
  }
}

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void bar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void bar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

constexpr int kMsWarps = 16;
constexpr int kMsThreads = kMsWarps * 32;
constexpr int kMsMaxGroups = 128;         // fp64 accumulators per CTA (32 KiB)
constexpr int kMsEntCap = 88 * 1024;      // entry bytes staged per tile and stage
constexpr int kMsOfsCap = kMsMaxGroups + 3;  // block offsets per stage (+ alignment slack)

struct MissArgs {
  MatrixDesc m;
  const float* rt;  // centred fp32 residual, T x 512 (zero-padded)
  double* out;      // m_j (read back by the base-3 kernel's epilogue)
  int64_t chunks;
};

struct MsStage {
  uint8_t ent[kMsEntCap];
  int64_t ofs[kMsOfsCap + 1];
  float rt[GI_TILE_SAMPLES];
};

struct MsSmem {
  double acc[kMsMaxGroups * 32];
  int rq[GI_TILE_SAMPLES];  // fixed-point rt of the tile
  MsStage st[2];
  int bsum[kMsWarps][32];
  float wmax[kMsWarps];
  uint64_t bar[2];
  // what each stage holds: entry index at ent[0] (aligned down), first/last
  // block offset index (aligned down), whether the entries fit (else global)
  int64_t ent0[2];
  int ofs_shift[2];
  int ent_ok[2];
};

// One CTA per chunk of <= kMsMaxGroups SNP groups walks every sample tile.
// Thread 0 keeps the next tile's block offsets, residual slice and entries in
// flight (bulk async copies into the other stage) while the CTA works on this
// one; it reads the next-but-one tile's entry range (two offsets) from global
// memory a tile ahead, so no load of the pipeline waits on another.
__global__ void __launch_bounds__(kMsThreads, 1) missum_kernel(MissArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  MsSmem& S = *reinterpret_cast<MsSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const MatrixDesc& m = a.m;
  int* bh = S.bsum[warp];
  bh[lane] = 0;
  if (tid == 0) {
    bar_init(su32(&S.bar[0]));
    bar_init(su32(&S.bar[1]));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase[2] = {0u, 0u};

  for (int64_t chunk = blockIdx.x; chunk < a.chunks; chunk += gridDim.x) {
    const int64_t g0 = chunk * m.G / a.chunks, g1 = (chunk + 1) * m.G / a.chunks;
    const int ng = (int)(g1 - g0);
    GI_ASSERT(ng <= kMsMaxGroups);
    for (int e = tid; e < ng * 32; e += kMsThreads) S.acc[e] = 0.0;

    // thread 0: stage tile t into stage st, given its entry range [e_lo, e_hi)
    auto issue = [&](int64_t t, int st, int64_t e_lo, int64_t e_hi) {
      const uint32_t bar = su32(&S.bar[st]);
      const int64_t o_lo = (t * m.G + g0) & ~int64_t(1);  // 16-byte aligned int64 index
      const int64_t o_n = ((t * m.G + g1 + 2) & ~int64_t(1)) - o_lo;  // covers g1, even count
      const int64_t x_lo = e_lo & ~int64_t(7);  // 16-byte aligned uint16 index
      const int64_t x_n = ((e_hi + 7) & ~int64_t(7)) - x_lo;
      const bool fits = x_n * 2 <= kMsEntCap;
      S.ent0[st] = x_lo;
      S.ofs_shift[st] = (int)(t * m.G + g0 - o_lo);
      S.ent_ok[st] = fits ? 1 : 0;
      const uint32_t bytes = (uint32_t)(o_n * 8) + GI_TILE_SAMPLES * 4 +
                             (fits ? (uint32_t)(x_n * 2) : 0u);
      bar_expect(bar, bytes);
      bulk_copy(su32(S.st[st].ofs), m.mofs + o_lo, (uint32_t)(o_n * 8), bar);
      bulk_copy(su32(S.st[st].rt), a.rt + t * GI_TILE_SAMPLES, GI_TILE_SAMPLES * 4, bar);
      if (fits && x_n > 0) bulk_copy(su32(S.st[st].ent), m.mlist + x_lo, (uint32_t)(x_n * 2), bar);
    };
    int64_t nx_lo = 0, nx_hi = 0;  // thread 0: entry range of the tile after the next issue
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the previous chunk's reads
      issue(0, 0, m.mofs[g0], m.mofs[g1]);
      if (m.T > 1) {
        nx_lo = m.mofs[m.G + g0];
        nx_hi = m.mofs[m.G + g1];
      }
    }
    int st = 0;
    for (int64_t t = 0; t < m.T; ++t) {
      if (tid == 0 && t + 1 < m.T) {
        // the other stage was released by the __syncthreads ending tile t - 1;
        // order those generic reads before the async-proxy writes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(t + 1, st ^ 1, nx_lo, nx_hi);
        if (t + 2 < m.T) {
          nx_lo = m.mofs[(t + 2) * m.G + g0];
          nx_hi = m.mofs[(t + 2) * m.G + g1];
        }
      }
      bar_wait(su32(&S.bar[st]), phase[st]);
      phase[st] ^= 1u;
      const MsStage& B = S.st[st];
      const float r0 = B.rt[tid];
      float mx = fabsf(r0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) S.wmax[warp] = mx;
      __syncthreads();  // wmax; also: the previous tile's rq readers are done
      mx = S.wmax[0];
#pragma unroll
      for (int w = 1; w < kMsWarps; ++w) mx = fmaxf(mx, S.wmax[w]);
      int ex = 0;
      if (mx > 0.f) frexpf(mx, &ex);  // max|rt| < 2^ex
      const int sc = 21 - ex;         // |q| <= 2^21: 512 of them sum below 2^31
      S.rq[tid] = __float2int_rn(ldexpf(r0, sc));
      const double inv = ldexp(1.0, -sc);
      __syncthreads();  // rq
      const int shift = S.ofs_shift[st];
      const int64_t x0 = S.ent0[st];
      const bool staged = S.ent_ok[st] != 0;
      const uint16_t* ent_s = reinterpret_cast<const uint16_t*>(B.ent);
      for (int gl = warp; gl < ng; gl += kMsWarps) {
        const int64_t s = B.ofs[shift + gl], e = B.ofs[shift + gl + 1];
        if (staged) {
          // four entries per lane in flight: their reads, then their atomics
          const uint16_t* p = ent_s + (s - x0);
          const int cnt = (int)(e - s);
          for (int i = lane; i < cnt; i += 128) {
            uint32_t v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = i + 32 * k < cnt ? p[i + 32 * k] : 0xFFFFu;
            int q[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) q[k] = v[k] != 0xFFFFu ? S.rq[v[k] & 511u] : 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (v[k] != 0xFFFFu) atomicAdd(bh + (v[k] >> 9), q[k]);
          }
        } else {
          for (int64_t i = s + lane; i < e; i += 32) {
            const uint32_t v = __ldg(m.mlist + i);
            atomicAdd(bh + (v >> 9), S.rq[v & 511u]);
          }
        }
        __syncwarp();
        const int tot = bh[lane];
        bh[lane] = 0;
        S.acc[gl * 32 + lane] += (double)tot * inv;  // exact product, tile order
        __syncwarp();
      }
      __syncthreads();  // this stage's buffers are free for tile t + 2
      st ^= 1;
    }
    for (int e = tid; e < ng * 32; e += kMsThreads) {
      const int64_t j = g0 * 32 + e;
      if (j < m.p) a.out[j] = S.acc[e];
    }
    __syncthreads();
  }
}

constexpr int kMsSmem = (int)sizeof(MsSmem);

}  // namespace

int missing_list_count(const MatrixDesc& m, int64_t* d_cnt, cudaStream_t s) {
  const int64_t nblk = m.T * m.G;
  if (nblk == 0) return 0;
  int64_t grid = (nblk + 7) / 8;
  if (grid > 148 * 16) grid = 148 * 16;
  miss_count_kernel<<<(unsigned)grid, 256, 0, s>>>(m, d_cnt);
  GI_LAUNCH_CHECK();
  return 0;
}

int missing_list_scan(const int64_t* d_cnt, int64_t* d_ofs, int64_t nblk, void* tmp,
                      size_t& tmp_bytes, cudaStream_t s) {
  // exclusive scan over nblk + 1 counts (the last count is zero) -> ofs
  GI_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, d_cnt, d_ofs, (int)(nblk + 1), s));
  return 0;
}

int missing_list_fill(const MatrixDesc& m, const int64_t* d_ofs, uint16_t* d_ent, cudaStream_t s) {
  const int64_t nblk = m.T * m.G;
  if (nblk == 0) return 0;
  int64_t grid = (nblk + 7) / 8;
  if (grid > 148 * 16) grid = 148 * 16;
  static const int win = [] {
    const char* e = getenv("GI_MISS_WIN");
    const int w = e ? atoi(e) : 2;
    return w == 1 || w == 2 || w == 4 ? w : 2;
  }();
  if (win == 1)
    miss_fill_kernel<1><<<(unsigned)grid, 256, 0, s>>>(m, d_ofs, d_ent);
  else if (win == 4)
    miss_fill_kernel<4><<<(unsigned)grid, 256, 0, s>>>(m, d_ofs, d_ent);
  else
    miss_fill_kernel<2><<<(unsigned)grid, 256, 0, s>>>(m, d_ofs, d_ent);
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_missum(const MatrixDesc& m, const float* rt, double* out, int num_sms, cudaStream_t s) {
  if (m.p == 0 || m.G == 0 || m.T == 0) return 0;
  static std::once_flag once;
  static cudaError_t cfg_err = cudaSuccess;
  std::call_once(once, [] {
    cfg_err = cudaFuncSetAttribute(missum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kMsSmem);
  });
  GI_CUDA_TRY(cfg_err);
  MissArgs a;
  a.m = m;
  a.rt = rt;
  a.out = out;
  // groups per chunk: the expected entry bytes of a (tile, chunk) at most 80%
  // of a stage (a tile that overflows reads its entries from global memory),
  // then chunks in whole waves over the SMs
  const double per_block = m.T * m.G > 0 ? 2.0 * (double)m.mtotal / (double)(m.T * m.G) : 0.0;
  int64_t gmax = kMsMaxGroups;
  if (per_block > 0.0 && per_block * gmax > 0.8 * kMsEntCap)
    gmax = std::max<int64_t>(1, (int64_t)(0.8 * kMsEntCap / per_block));
  int64_t chunks = (m.G + gmax - 1) / gmax;
  chunks = (int64_t)num_sms * ((chunks + num_sms - 1) / num_sms);
  if (chunks > m.G) chunks = m.G;
  a.chunks = chunks;
  const int grid = (int)(chunks < num_sms ? chunks : num_sms);
  missum_kernel<<<grid, kMsThreads, kMsSmem, s>>>(a);
  GI_LAUNCH_CHECK();
  return 0;
}

}  // namespace gi
