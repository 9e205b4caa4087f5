// Shared definitions for the sm_100a genoiht kernels.
//
// Device layout of a packed genotype matrix ("swizzled sample tiles"):
//   * samples are cut into tiles of 512 (128 packed bytes per SNP, 32 words);
//   * SNPs are cut into groups of 32 (one per lane of the X^T r warp);
//   * block (tile t, group g) is 4 KiB at offset ((t * G) + g) * 4096;
//   * inside a block, 32-bit word w (samples 512t + 16w .. +15, LSB-first
//     2-bit codes exactly as in the BED file) of SNP 32g + L is stored at byte
//     offset ((L ^ w) * 128 + 4 * L).
// A warp reading row q of a block therefore gets lane L = word (L ^ q) of SNP
// L: one coalesced 128-byte line, and each lane at a distinct sample position,
// which is what makes the X^T r lookup tables bank-conflict free (aty.cu).
// Bytes past ceil(n/4) and SNPs past p are zero (dose 0, never read as data).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

// Device-side bounds checks, compiled in with -DGI_DEBUG (make DEBUG=1 builds
// libgenoiht_cuda_debug.so; tests run against it with GI_LIB_PATH).  A failed
// check prints the condition and traps, which surfaces as a CUDA error.
#ifdef GI_DEBUG
#define GI_ASSERT(cond)                                                         \
  do {                                                                          \
    if (!(cond)) {                                                              \
      printf("GI_ASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      __trap();                                                                 \
    }                                                                           \
  } while (0)
#else
#define GI_ASSERT(cond) \
  do {                  \
  } while (0)
#endif

#define GI_TILE_SAMPLES 512
#define GI_TILE_BYTES 128
#define GI_TILE_WORDS 32
#define GI_GROUP 32
#define GI_BLOCK_BYTES 4096
// base-3 copy for X^T r (missing-free matrices): 5 genotypes per byte, so a
// 128-byte tile row holds 640 samples; same 4 KiB block swizzle
#define GI_TILE3_SAMPLES 640

namespace gi {

struct MatrixDesc {
  const uint8_t* x;   // swizzled tiles
  int64_t n;          // samples
  int64_t p;          // SNPs
  int64_t nb;         // ceil(n/4) bytes per SNP in the BED layout
  int64_t T;          // sample tiles = ceil(nb / 128)
  int64_t G;          // SNP groups = ceil(p / 32)
  const uint8_t* x3 = nullptr;  // optional base-3 tiles (read only by X^T r)
  int64_t T3 = 0;               // base-3 sample tiles = ceil(n / 640)
  // with x3 on a matrix with missing genotypes: the missing positions per
  // 4 KiB block, (lane << 9) | sample offset, and each block's first entry
  // (T G + 1 offsets; missing.cu)
  const uint16_t* mlist = nullptr;
  const int64_t* mofs = nullptr;
  int64_t mtotal = 0;  // entries
};

__host__ __device__ inline int64_t tiles3_of(int64_t n) {
  return (n + GI_TILE3_SAMPLES - 1) / GI_TILE3_SAMPLES;
}

__host__ __device__ inline int64_t block_offset(int64_t t, int64_t g, int64_t G) {
  return (t * G + g) * (int64_t)GI_BLOCK_BYTES;
}

// byte offset of word w of SNP j in tile t, bounds-checked in debug builds
__device__ inline int64_t word_offset_chk(const MatrixDesc& m, int64_t t, int64_t j, int w) {
  GI_ASSERT(t >= 0 && t < m.T && j >= 0 && j < m.G * 32 && w >= 0 && w < 32);
  const int L = (int)(j & 31);
  return ((t * m.G + (j >> 5)) * (int64_t)GI_BLOCK_BYTES) + (int64_t)(((L ^ w) << 7) + (L << 2));
}

// byte offset of word w of SNP j in tile t
__host__ __device__ inline int64_t word_offset(int64_t t, int64_t j, int w, int64_t G) {
  const int L = (int)(j & 31);
  return block_offset(t, j >> 5, G) + (int64_t)(((L ^ w) << 7) + (L << 2));
}

// byte offset of packed byte b (BED column index) of SNP j
__host__ __device__ inline int64_t byte_offset(int64_t j, int64_t b, int64_t G) {
  const int64_t t = b >> 7;
  const int w = (int)((b >> 2) & 31);
  return word_offset(t, j, w, G) + (b & 3);
}

int launch_residual(int64_t n, const double* y, const double* fit, const double* C, int c,
                    const double* bcov, const uint8_t* keep, double n_eff, double* r,
                    double* scal, double* partials, unsigned int* ticket, cudaStream_t s);
// residual + optional beta writes + (gcov != NULL) covariate gradient, fused
int launch_refresh_residual(int64_t n, const double* y, const double* fit, const double* C,
                            int c, const double* bcov, const uint8_t* keep, double n_eff,
                            double* r, double* scal, double* gcov, int64_t sk,
                            const int64_t* sidx, const double* sval, double* beta,
                            double* partials, unsigned int* ticket, cudaStream_t s);
int launch_center(int64_t n, int64_t n_pad, const double* r, const uint8_t* keep, double* scal,
                  float* rt, double* partials, unsigned int* ticket, cudaStream_t s);
int launch_covgrad(int64_t n, const double* C, int c, const double* r, double* gcov,
                   double* partials, unsigned int* ticket, cudaStream_t s);
int launch_maxabs(int64_t m, const double* x, double* scal, int slot, double* partials,
                  unsigned int* ticket, cudaStream_t s);
int launch_sumsq(int64_t m, const double* x, double* scal, int slot, double* partials,
                 unsigned int* ticket, cudaStream_t s);
int launch_add_cov(int64_t n, const double* C, int c, const double* w, double* x,
                   cudaStream_t s);
int launch_image_sumsq(int64_t m, const double* x, const double* C, int c, const double* w,
                       const uint8_t* keep, double* scal, int slot, int ratio_out,
                       double ratio_num, double* host_out, double* partials,
                       unsigned int* ticket, cudaStream_t s);
// segments of 8-byte words copied (or gathered through idx) to out[dst ...]
constexpr int kMaxPub = 6;
struct PubSeg {
  const void* src;
  const int64_t* idx;  // NULL: plain copy
  int64_t count;
  int64_t dst;
};
struct PubArgs {
  PubSeg seg[kMaxPub];
  int nseg = 0;
  void add(const void* src, int64_t count, int64_t dst, const int64_t* idx = nullptr) {
    if (count > 0) seg[nseg++] = PubSeg{src, idx, count, dst};
  }
};
int launch_publish(const PubArgs& a, void* out, cudaStream_t s);
int64_t topk_blocks(int64_t p);
int launch_topk(int64_t p, int64_t k, int mode, const double* beta, const double* g, double mu,
                int64_t idx_base, uint64_t* cand_key, int64_t* cand_idx, double* cand_val,
                int64_t* out_idx, double* out_val, uint64_t* out_key, int64_t* out_count,
                cudaStream_t s, const double* mu_dev = nullptr,
                unsigned int* ticket = nullptr);
// sharded loop exchanges (solver.cu): gather this shard's (max|g|, g on the
// global support), fold the all-gathered rows, merge all-gathered top-k lists
int launch_shard_gather(int64_t kg, const int64_t* gsel, const double* g, const double* scal3,
                        double* mine, cudaStream_t s);
int launch_shard_fold(int world, int64_t kg, const double* all, double* out, cudaStream_t s);
int launch_shard_merge(int world, int64_t ke, const double* all, uint64_t* ckey, int64_t* cidx,
                       double* cval, int64_t* out_idx, double* out_val, uint64_t* out_key,
                       int64_t* out_count, cudaStream_t s);
int launch_scatter(int64_t k, const int64_t* idx, const double* val, double* beta,
                   cudaStream_t s);
int launch_gather(int64_t k, const int64_t* idx, const double* src, double* dst,
                  cudaStream_t s);
}  // namespace gi

// error plumbing shared with capi.cu
void gi_set_error(const char* fmt, ...);

#define GI_CUDA_TRY(expr)                                                        \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      gi_set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),       \
                   __FILE__, __LINE__);                                          \
      return -1;                                                                 \
    }                                                                            \
  } while (0)

#define GI_LAUNCH_CHECK()                                                        \
  do {                                                                           \
    cudaError_t _e = cudaGetLastError();                                         \
    if (_e != cudaSuccess) {                                                     \
      gi_set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e),   \
                   __FILE__, __LINE__);                                          \
      return -1;                                                                 \
    }                                                                            \
  } while (0)

// Kernel-layer entry points (host side), all stream-ordered; return 0 or -1.
namespace gi {
int launch_upload_tiles(const MatrixDesc& m, uint8_t* x, const uint8_t* d_bed_chunk,
                        int64_t j0, int64_t count, cudaStream_t s);
int launch_download_tiles(const MatrixDesc& m, uint8_t* d_bed_chunk, int64_t j0,
                          int64_t count, cudaStream_t s);
int launch_synth(const MatrixDesc& m, uint8_t* x, uint64_t seed, int64_t j_base,
                 double maf_lo, double maf_hi, double missing, cudaStream_t s);
int launch_subset_rows(const MatrixDesc& src, const MatrixDesc& dst, uint8_t* x,
                       const int64_t* d_rows, cudaStream_t s);
int launch_stats(const MatrixDesc& m, const uint32_t* d_rowmask, double* u, double* v,
                 int32_t* d_missing_cnt, int32_t* d_s1cnt, cudaStream_t s);
int launch_pack3(const MatrixDesc& m, uint8_t* x3, cudaStream_t s);
// missing-genotype lists (missing.cu): per-block counts (T G + 1 slots, the
// last left zero), their exclusive scan (tmp == nullptr: size query), the
// entries; and the per-SNP missing sums m_j = sum rt over the missing samples
int missing_list_count(const MatrixDesc& m, int64_t* d_cnt, cudaStream_t s);
int missing_list_scan(const int64_t* d_cnt, int64_t* d_ofs, int64_t nblk, void* tmp,
                      size_t& tmp_bytes, cudaStream_t s);
int missing_list_fill(const MatrixDesc& m, const int64_t* d_ofs, uint16_t* d_ent, cudaStream_t s);
int launch_missum(const MatrixDesc& m, const float* rt, double* out, int num_sms, cudaStream_t s);
int launch_group_flags(const MatrixDesc& m, const int32_t* d_missing_cnt, uint8_t* flags,
                       cudaStream_t s);
int launch_aty_fast(const MatrixDesc& m, const uint8_t* group_missing, const float* rt,
                    const double* u, const double* v, const int32_t* s1cnt,
                    const double* d_scal, double scale, double* out, int num_sms,
                    cudaStream_t s, double* d_gmax = nullptr, const PubArgs* pub = nullptr,
                    unsigned int* pub_ticket = nullptr, void* pub_out = nullptr,
                    double* part = nullptr, unsigned int* cticket = nullptr);
// X^T r work decomposition (aty.cu) and the partial-sum buffer it needs when
// tiles are sliced (0: single-slice plan); chunk tickets: at most 2 * num_sms
void aty_fast_plan(const MatrixDesc& m, int num_sms, bool sliced, int64_t& chunks,
                   int64_t& slices);
int64_t aty_fast_part_doubles(const MatrixDesc& m, int num_sms);
int launch_aty_exact(const MatrixDesc& m, const double* r_pad, const double* u,
                     const double* v, const double* d_sum_r, double scale, double* out,
                     cudaStream_t s, double* d_gmax = nullptr, const PubArgs* pub = nullptr,
                     unsigned int* pub_ticket = nullptr, void* pub_out = nullptr);
// exact gradient on k listed columns, after a fast sweep (aty.cu); part holds
// support_grad_part_doubles(kcap, T) doubles, tickets kcap zeroed counters
int64_t support_grad_part_doubles(int64_t kcap, int64_t T);
int launch_support_grad(const MatrixDesc& m, const double* r_pad, const double* u,
                        const double* v, const double* d_sum_r, double scale, const int64_t* idx,
                        int64_t k, double* out, double* pub_out, double* part,
                        unsigned int* tickets, cudaStream_t s);
int launch_ax(const MatrixDesc& m, const double* u, const double* v, const int64_t* idx,
              const double* w, int64_t k, double* out, int accumulate, cudaStream_t s);
// X_S w fused with its image norm (see ax.cu, AxNorm); returns -2 when k is
// too large for one launch (the caller then runs launch_ax + image_sumsq)
int launch_ax_norm(const MatrixDesc& m, const double* u, const double* v, const int64_t* idx,
                   const double* w, int64_t k, const double* C, int c, const double* wc,
                   const uint8_t* keep, double* scal, int slot, int ratio_out, double ratio_num,
                   double* host_out, double* partials, unsigned int* ticket, cudaStream_t s);
// X_S w fused with the refresh's residual, loss, sum r, g_cov (c <= 8) and the
// pending beta writes; -2 when k or c is too large (two-kernel path instead)
int launch_ax_residual(const MatrixDesc& m, const double* u, const double* v,
                       const int64_t* idx, const double* w, int64_t k, const double* y,
                       const double* C, int c, const double* bcov, const uint8_t* keep,
                       double n_eff, double* r, double* scal, double* gcov, int64_t sk,
                       const int64_t* sidx, const double* sval, double* beta, double* partials,
                       unsigned int* ticket, cudaStream_t s);
int launch_decompress(const MatrixDesc& m, const double* u, const double* v,
                      const int64_t* idx, int64_t k, double* out_t, cudaStream_t s);
// X^T R on the tensor cores (xtr_mma.cu): the digit image of up to 32
// residuals (16 with missing genotypes), then one sweep of the 2-bit tiles.
// One descriptor per right-hand side (a device array of them).
struct XtrRhs {
  const double* r;          // residual, n entries
  const uint8_t* keep;      // optional row mask (rows with 0 count as r = 0)
  const double* u;          // standardisation of this right-hand side (p each)
  const double* v;
  const int32_t* s1cnt;     // (sum of doses, observed count) over its rows
  double* out;              // p outputs: scale_out * v_j (...) as _aty_kernel
  unsigned long long* gmax; // optional: atomicMax of |out_j / scale_out| (double bits)
};
constexpr int kXtrMaxRhs = 32;
int xtr_mma_cols(int nrhs);
int xtr_mma_max_rhs(bool any_missing);
int64_t xtr_mma_qimg_bytes(const MatrixDesc& m, int nrhs);
int launch_xtr_quant(int64_t n, int64_t T, int nrhs, const XtrRhs* d_rhs, double* qscal,
                     long long* qsum, int8_t* qimg, double* partials, int64_t partial_cap,
                     unsigned int* tickets, cudaStream_t s);
int launch_xtr_mma(const MatrixDesc& m, const uint8_t* gmiss, bool any_missing, int nrhs,
                   const int8_t* qimg, const double* qscal, const long long* qsum,
                   const XtrRhs* d_rhs, double scale_out, int num_sms, cudaStream_t s,
                   const PubArgs* pub = nullptr, unsigned int* pub_ticket = nullptr,
                   void* pub_out = nullptr);
}  // namespace gi
