// Matrix construction kernels: BED bytes <-> swizzled sample tiles, the
// counter-based synthetic generator, and per-SNP standardisation statistics.
//
// Reference behaviour replaced:
//   PackedGenotypeMatrix.from_bed_buffer  geno_matrix.py:281-292 (bytes kept verbatim)
//   _stats_kernel / _packed_stats         geno_matrix.py:106-139, :239-246
//   random_packed_matrix                  simulate.py:56-65 (same law, hash-based stream)
#include <climits>

#include "common.cuh"

namespace gi {

// ---------------------------------------------------------------- upload
// d_bed: `count` SNPs x nb bytes (variant-major, as read from a BED file),
// first SNP = j0.  One thread per 32-bit word of the tiled layout.
__global__ void upload_tiles_kernel(MatrixDesc m, uint8_t* __restrict__ x,
                                    const uint8_t* __restrict__ bed, int64_t j0,
                                    int64_t count) {
  const int64_t words = m.T * GI_TILE_WORDS;
  const int64_t total = count * words;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jj = e / words;
    const int64_t wg = e - jj * words;  // global word index along samples
    const int64_t j = j0 + jj;
    const uint8_t* row = bed + jj * m.nb;
    uint32_t word = 0;
    const int64_t b0 = wg * 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t b = b0 + k;
      if (b < m.nb) word |= (uint32_t)row[b] << (8 * k);
    }
    const int64_t t = wg >> 5;
    const int w = (int)(wg & 31);
    *reinterpret_cast<uint32_t*>(x + word_offset_chk(m, t, j, w)) = word;
  }
}

__global__ void download_tiles_kernel(MatrixDesc m, const uint8_t* __restrict__ x,
                                      uint8_t* __restrict__ bed, int64_t j0, int64_t count) {
  const int64_t total = count * m.nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jj = e / m.nb;
    const int64_t b = e - jj * m.nb;
    bed[e] = x[byte_offset(j0 + jj, b, m.G)];
  }
}

static int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return (int)g;
}

int launch_upload_tiles(const MatrixDesc& m, uint8_t* x, const uint8_t* d_bed, int64_t j0,
                        int64_t count, cudaStream_t s) {
  if (count <= 0) return 0;
  upload_tiles_kernel<<<grid_for(count * m.T * 32, 256), 256, 0, s>>>(m, x, d_bed, j0, count);
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_download_tiles(const MatrixDesc& m, uint8_t* d_bed, int64_t j0, int64_t count,
                          cudaStream_t s) {
  if (count <= 0 || m.nb == 0) return 0;
  download_tiles_kernel<<<grid_for(count * m.nb, 256), 256, 0, s>>>(m, m.x, d_bed, j0, count);
  GI_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------- synth
// Must stay bit-identical to oracle/genoiht_oracle.c (ora_key, ora_synth).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

__device__ __forceinline__ uint64_t synth_key(uint64_t seed, uint64_t j, uint64_t i) {
  return mix64(seed * 0x9E3779B97F4A7C15ULL + j * 0xD1B54A32D192ED03ULL +
               i * 0x8CB92BA72F3D8DD7ULL + 0x632BE59BD9B4E019ULL);
}

__device__ __forceinline__ uint32_t thr_from(double prob) {
  const double scale = 4294967296.0;
  const double t = floor(__dmul_rn(prob, scale));
  return t >= scale ? 0xFFFFFFFFu : (uint32_t)t;
}

// One thread per (SNP, word); j_base is the global index of local SNP 0 so
// that a SNP-sharded matrix holds exactly the bytes of the unsharded one.
__global__ void synth_kernel(MatrixDesc m, uint8_t* __restrict__ x, uint64_t seed,
                             int64_t j_base, double maf_lo, double maf_hi, double missing) {
  const int64_t words = m.T * GI_TILE_WORDS;
  const int64_t total = m.p * words;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / words;
    const int64_t wg = e - j * words;
    const uint64_t jg = (uint64_t)(j + j_base);
    const uint64_t hf = synth_key(seed, jg, 0xFFFFFFFFFFFFULL);
    const double unit = __dmul_rn((double)(hf >> 11), 1.0 / 9007199254740992.0);
    const double f = __dadd_rn(maf_lo, __dmul_rn(__dsub_rn(maf_hi, maf_lo), unit));
    const double q = __dsub_rn(1.0, f);
    const double p0 = __dmul_rn(q, q);
    const double p1 = __dadd_rn(p0, __dmul_rn(__dmul_rn(2.0, f), q));
    const uint32_t t0 = thr_from(p0), t1 = thr_from(p1), tm = thr_from(missing);
    uint32_t word = 0;
    const int64_t i0 = wg * 16;
    for (int s = 0; s < 16; ++s) {
      const int64_t i = i0 + s;
      if (i >= m.n) break;
      const uint64_t h = synth_key(seed, jg, (uint64_t)i);
      const uint32_t ud = (uint32_t)h, um = (uint32_t)(h >> 32);
      uint32_t code = ud < t0 ? 0u : (ud < t1 ? 2u : 3u);
      if (um < tm) code = 1u;
      word |= code << (2 * s);
    }
    *reinterpret_cast<uint32_t*>(x + word_offset_chk(m, wg >> 5, j, (int)(wg & 31))) = word;
  }
}

int launch_synth(const MatrixDesc& m, uint8_t* x, uint64_t seed, int64_t j_base,
                 double maf_lo, double maf_hi, double missing, cudaStream_t s) {
  if (m.p == 0) return 0;
  synth_kernel<<<grid_for(m.p * m.T * 32, 256), 256, 0, s>>>(m, x, seed, j_base, maf_lo,
                                                              maf_hi, missing);
  GI_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------- stats
// One warp per SNP group, lane L = SNP 32g + L; at row q the warp reads one
// 128-byte line (word L ^ q of each SNP).  Counts are integers, so u and v
// come out bit-identical to the reference's fp64 sums (geno_matrix.py:134-139).
// d_rowmask (optional): one uint32 per (tile, word), bit 2s set when sample
// 16w + s of the tile is included (cross-validation training rows).
__global__ void stats_kernel(MatrixDesc m, const uint32_t* __restrict__ rowmask,
                             double* __restrict__ u, double* __restrict__ v,
                             int32_t* __restrict__ missing_cnt, int32_t* __restrict__ s1cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= m.G) return;
  const int64_t j = g * 32 + lane;
  int cnt = 0, s1 = 0, s2 = 0, miss = 0;
  for (int64_t t = 0; t < m.T; ++t) {
    GI_ASSERT(g < m.G);
  const uint8_t* blk = m.x + block_offset(t, g, m.G);
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
      const uint32_t word = *reinterpret_cast<const uint32_t*>(blk + (q << 7) + (lane << 2));
      const int w = lane ^ q;
      const int64_t first = t * GI_TILE_SAMPLES + 16 * w;
      const int64_t nvalid64 = m.n - first;
      const int nvalid = nvalid64 >= 16 ? 16 : (nvalid64 <= 0 ? 0 : (int)nvalid64);
      uint32_t valid = nvalid >= 16 ? 0x55555555u : ((1u << (2 * nvalid)) - 1u) & 0x55555555u;
      if (rowmask) valid &= rowmask[t * 32 + w];
      const uint32_t lo = word & 0x55555555u;
      const uint32_t hi = (word >> 1) & 0x55555555u;
      const int c_miss = __popc(lo & ~hi & valid);
      const int c_het = __popc(hi & ~lo & valid);
      const int c_hom = __popc(hi & lo & valid);
      cnt += __popc(valid) - c_miss;
      s1 += c_het + 2 * c_hom;
      s2 += c_het + 4 * c_hom;
      miss += c_miss;
    }
  }
  if (j >= m.p) return;
  const double dc = (double)cnt, d1 = (double)s1, d2 = (double)s2;
  u[j] = cnt > 0 ? __ddiv_rn(d1, dc) : 0.0;
  double vj = 0.0;
  if (cnt >= 2) {
    const double var = __ddiv_rn(__dsub_rn(d2, __ddiv_rn(__dmul_rn(d1, d1), dc)),
                                 __dsub_rn(dc, 1.0));
    vj = var > 0.0 ? __ddiv_rn(1.0, __dsqrt_rn(var)) : 0.0;
  }
  v[j] = vj;
  if (missing_cnt) missing_cnt[j] = miss;
  if (s1cnt) {
    s1cnt[2 * j] = s1;
    s1cnt[2 * j + 1] = cnt;
  }
}

int launch_stats(const MatrixDesc& m, const uint32_t* d_rowmask, double* u, double* v,
                 int32_t* d_missing_cnt, int32_t* d_s1cnt, cudaStream_t s) {
  if (m.p == 0) return 0;
  const int threads = 256;
  const int64_t blocks = (m.G * 32 + threads - 1) / threads;
  stats_kernel<<<(unsigned)blocks, threads, 0, s>>>(m, d_rowmask, u, v, d_missing_cnt,
                                                     d_s1cnt);
  GI_LAUNCH_CHECK();
  return 0;
}

// flags[g] = 1 when any SNP of group g has a missing genotype (lets the X^T r
// kernel skip the missing-sum lookups for whole groups).
__global__ void group_flags_kernel(int64_t p, int64_t G, const int32_t* __restrict__ miss,
                                   uint8_t* __restrict__ flags) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= G) return;
  int any = 0;
  for (int l = 0; l < 32; ++l) {
    const int64_t j = g * 32 + l;
    if (j < p && miss[j] > 0) any = 1;
  }
  flags[g] = (uint8_t)any;
}

int launch_group_flags(const MatrixDesc& m, const int32_t* d_missing_cnt, uint8_t* flags,
                       cudaStream_t s) {
  if (m.G == 0) return 0;
  group_flags_kernel<<<(unsigned)((m.G + 255) / 256), 256, 0, s>>>(m.p, m.G, d_missing_cnt,
                                                                    flags);
  GI_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------- base-3 copy
// x3 block (t3, g) holds samples 640 t3 .. +639 of SNPs 32 g .. +31 with the
// 2-bit blocks' swizzle (word w of SNP L at byte (L ^ w) * 128 + 4 L); byte b
// of word w packs samples i = 640 t3 + 20 w + 5 b + s, s < 5, as
// sum_s dose_s 3^s (<= 242), dose 0/1/2 for codes 00/10/11.  Built only when
// no SNP has a missing genotype (code 01); samples >= n and SNPs >= p are 0.
// One CTA per output block at a time: the 2-3 source blocks holding its 640
// samples are staged in shared memory with coalesced 16-byte loads, then lane
// L of each warp assembles word L ^ q of SNP L from its own SNP's source words
// (bank = L, conflict-free) and the warp stores row q of the output block.
// The 20 codes of an output word are one 40-bit window of the source words;
// a 1024-entry table maps each 10-bit run of 5 codes to its base-3 byte.
constexpr int kPack3Threads = 256;

__global__ void __launch_bounds__(kPack3Threads) pack3_kernel(MatrixDesc m,
                                                              uint8_t* __restrict__ x3) {
  __shared__ __align__(16) uint32_t src[3][1024];
  __shared__ uint8_t lut[1024];
  for (int v = threadIdx.x; v < 1024; v += kPack3Threads) {
    uint32_t val = 0u, mul = 1u;
    for (int s2 = 0; s2 < 5; ++s2) {
      const uint32_t code = (v >> (2 * s2)) & 3u;
      val += (code == 2u ? 1u : (code == 3u ? 2u : 0u)) * mul;
      mul *= 3u;
    }
    lut[v] = (uint8_t)val;
  }
  const int64_t nblk = m.T3 * m.G;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t t3 = blk / m.G, g = blk - t3 * m.G;
    const int64_t s0 = t3 * GI_TILE3_SAMPLES;  // first sample of the block
    const int64_t ta = s0 / GI_TILE_SAMPLES;   // first source tile
    int64_t tb = (s0 + GI_TILE3_SAMPLES - 1) / GI_TILE_SAMPLES;
    if (tb > m.T - 1) tb = m.T - 1;
    __syncthreads();  // the lut, or the previous block's reads, are done
    for (int c = 0; c <= (int)(tb - ta); ++c)
      reinterpret_cast<uint4*>(src[c])[threadIdx.x] =
          reinterpret_cast<const uint4*>(m.x + block_offset(ta + c, g, m.G))[threadIdx.x];
    __syncthreads();
    for (int e = threadIdx.x; e < 1024; e += kPack3Threads) {
      const int q = e >> 5, L = e & 31, w = L ^ q;
      const int64_t i0 = s0 + 20 * w;  // first sample of the word
      uint32_t out = 0u;
      if (g * 32 + L < m.p && i0 < m.n) {
        const int rel0 = (int)(i0 - ta * GI_TILE_SAMPLES);
        const int rw0 = rel0 >> 4, o2 = 2 * (rel0 & 15);
        uint32_t sw[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int rw = rw0 + c, tc = rw >> 5, wi = rw & 31;
          sw[c] = tc <= (int)(tb - ta) ? src[tc][((L ^ wi) << 5) + L] : 0u;
        }
        const uint64_t lo = (uint64_t)sw[0] | ((uint64_t)sw[1] << 32);
        uint64_t win = lo >> o2;
        if (o2 > 24) win |= (uint64_t)sw[2] << (64 - o2);
        const int64_t valid = m.n - i0 < 20 ? m.n - i0 : 20;  // samples >= n are 0
        win &= (1ull << (2 * valid)) - 1ull;
#pragma unroll
        for (int b = 0; b < 4; ++b) out |= (uint32_t)lut[(win >> (10 * b)) & 1023u] << (8 * b);
      }
      reinterpret_cast<uint32_t*>(x3 + blk * GI_BLOCK_BYTES)[e] = out;
    }
  }
}

int launch_pack3(const MatrixDesc& m, uint8_t* x3, cudaStream_t s) {
  if (m.T3 == 0 || m.G == 0) return 0;
  int64_t blocks = m.T3 * m.G;
  if (blocks > 148 * 16) blocks = 148 * 16;
  pack3_kernel<<<(unsigned)blocks, kPack3Threads, 0, s>>>(m, x3);
  GI_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------- subset rows
// dst holds m samples: sample i of dst = sample rows[i] of src.  One CTA per
// (dst tile, SNP group), 8 warps.  Warp w builds rows q = w, w + 8, ... of the
// dst block; lane L assembles word q ^ L of SNP 32 g + L, so every store is
// one coalesced 128-B row.  When the tile's source samples lie in at most
// kSubStage consecutive source tiles (sorted rows, as for CV folds) those
// blocks are staged in shared memory with 16-B loads; the gather of a code
// then reads byte (L ^ sw) * 128 + 4 L + .. of a staged block -- bank L, so
// conflict-free.  Other row sets read the source blocks from global memory.
// The source index of dst sample 16 w' + s is kept at srow[s * 32 + w'], so
// the 32 lanes (w' = q ^ L) read 32 distinct banks.  Padding codes stay zero.
constexpr int kSubStage = 8;

__global__ void __launch_bounds__(256) subset_rows_kernel(MatrixDesc src, MatrixDesc dst,
                                                          uint8_t* __restrict__ x,
                                                          const int64_t* __restrict__ rows) {
  __shared__ __align__(16) uint8_t stage[kSubStage * GI_BLOCK_BYTES];
  __shared__ int32_t srow[GI_TILE_SAMPLES];
  __shared__ int s_lo, s_hi;
  const int64_t tp = blockIdx.x / dst.G;
  const int64_t g = blockIdx.x - tp * dst.G;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_lo = INT_MAX;
    s_hi = -1;
  }
  __syncthreads();
  for (int e = tid; e < GI_TILE_SAMPLES; e += blockDim.x) {
    const int64_t i = tp * GI_TILE_SAMPLES + e;
    int32_t si = -1;
    if (i < dst.n) {
      si = (int32_t)rows[i];
      GI_ASSERT(si >= 0 && si < src.n);
      atomicMin(&s_lo, si >> 9);
      atomicMax(&s_hi, si >> 9);
    }
    srow[(e & 15) * 32 + (e >> 4)] = si;
  }
  __syncthreads();
  const int lo = s_lo;
  const bool staged = s_hi >= 0 && s_hi - lo < kSubStage;
  if (staged) {
    const int nblk = s_hi - lo + 1;
    for (int e = tid; e < nblk * (GI_BLOCK_BYTES / 16); e += blockDim.x) {
      const int b = e / (GI_BLOCK_BYTES / 16), o = e - b * (GI_BLOCK_BYTES / 16);
      reinterpret_cast<uint4*>(stage)[e] = __ldg(
          reinterpret_cast<const uint4*>(src.x + block_offset(lo + b, g, src.G)) + o);
    }
  }
  __syncthreads();
  const int warp = tid >> 5, L = tid & 31;
  uint8_t* out = x + block_offset(tp, g, dst.G);
  for (int q = warp; q < 32; q += 8) {
    const int wq = q ^ L;
    uint32_t word = 0;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int32_t si = srow[s * 32 + wq];
      if (si >= 0) {
        const int off = (((L ^ ((si >> 4) & 31))) << 7) + (L << 2) + ((si >> 2) & 3);
        const uint32_t b = staged ? stage[((si >> 9) - lo) * GI_BLOCK_BYTES + off]
                                  : __ldg(src.x + block_offset(si >> 9, g, src.G) + off);
        word |= ((b >> (2 * (si & 3))) & 3u) << (2 * s);
      }
    }
    *reinterpret_cast<uint32_t*>(out + (q << 7) + (L << 2)) = word;
  }
}

int launch_subset_rows(const MatrixDesc& src, const MatrixDesc& dst, uint8_t* x,
                       const int64_t* d_rows, cudaStream_t s) {
  if (dst.p == 0 || dst.n == 0) return 0;
  const int64_t blocks = dst.T * dst.G;
  subset_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(src, dst, x, d_rows);
  GI_LAUNCH_CHECK();
  return 0;
}

}  // namespace gi
