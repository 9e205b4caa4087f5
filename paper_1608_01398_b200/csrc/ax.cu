// Sparse standardized forward product and active-column decode.
//
// Reference: _ax_cols_kernel geno_matrix.py:168-194 (via ax_columns :328-349,
// ax_parts :553-562) and _decompress_kernel :216-236 (via decompress :366-373).
//
// ax: out_i (+)= sum_t [dose_ij * scale_t - obs_ij * shift_t], scale_t = w_t v_j,
// shift_t = u_j scale_t, columns visited in the caller's order for every sample
// and columns with scale_t == 0 skipped -- the reference's exact per-sample
// operation sequence, so the result is bit-identical to _ax_cols_kernel.  The
// four possible per-code terms of column t are formed once per CTA in shared
// memory (dose * scale is exact for dose in {0, 1, 2}; one rounding in the
// subtraction, as in the reference), then each genotype costs one table read
// and one fp64 add.
#include "common.cuh"
#include "reduce.cuh"

namespace gi {

constexpr int kAxMaxCols = 1024;

// kNorm: instead of storing X_S w, reduce its image norm in the same pass --
// sum over the kept rows of (x_i + C_i wc)^2 with the per-element operations of
// image_sumsq_kernel (add_cov, mask, square) -- and let the last block write
// scal[slot], optionally scal[ratio_out] = ratio_num / scal[slot] and the
// mapped pair host_out = {scal[slot], ratio} (the native loop's image phase).
struct AxNorm {
  const double* C;
  int c;
  const double* wc;
  const uint8_t* keep;
  double* scal;
  int slot;
  int ratio_out;
  double ratio_num;
  double* host_out;
  RedWs ws;
};

// kRes (the native loop's refresh, unsharded): with f = X_S w, write the
// residual r_i = keep_i ? y_i - (f_i + C_i b_cov) : 0 and reduce loss, sum r
// and (c <= 8) g_cov = -C^T r -- refresh_residual_kernel's per-element
// operations -- plus the pending beta writes (block 0).
struct AxRes {
  const double* y;
  const double* C;
  int c;
  const double* bcov;
  const uint8_t* keep;
  double n_eff;
  double* r;
  double* scal;
  double* gcov;  // NULL: no covariate gradient here
  int64_t sk;
  const int64_t* sidx;
  const double* sval;
  double* beta;
  RedWs ws;
};

enum AxMode { kAxStore = 0, kAxNorm = 1, kAxRes = 2 };

template <int kMode>
__global__ void ax_kernel(MatrixDesc m, const double* __restrict__ u,
                          const double* __restrict__ v, const int64_t* __restrict__ idx,
                          const double* __restrict__ w, int k, double* __restrict__ out,
                          int accumulate, AxNorm nm, AxRes rs) {
  constexpr bool kNorm = kMode == kAxNorm;
  constexpr bool kRes = kMode == kAxRes;
  if (kRes && blockIdx.x == 0)
    for (int64_t t = threadIdx.x; t < rs.sk; t += blockDim.x) rs.beta[rs.sidx[t]] = rs.sval[t];
  __shared__ double terms[kAxMaxCols][4];
  __shared__ int64_t cols[kAxMaxCols];
  __shared__ int live[kAxMaxCols];
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    const int64_t j = idx[t];
    GI_ASSERT(j >= 0 && j < m.p);
    const double scale = __dmul_rn(w[t], v[j]);
    const double shift = __dmul_rn(u[j], scale);
    cols[t] = j;
    live[t] = scale != 0.0;
    terms[t][0] = __dsub_rn(0.0 * scale, shift);      // code 00: dose 0, observed
    terms[t][1] = __dsub_rn(0.0 * scale, 0.0 * shift);  // code 01: missing
    terms[t][2] = __dsub_rn(scale, shift);              // code 10: dose 1
    terms[t][3] = __dsub_rn(__dmul_rn(2.0, scale), shift);  // code 11: dose 2
  }
  __syncthreads();
  // one thread per packed byte (4 samples): at the small n of path and CV fits
  // a thread per 16-sample word left most SMs idle.  Each sample still adds the
  // columns' terms in the caller's order (same bits as _ax_cols_kernel).
  const int64_t nbytes = (m.n + 3) / 4;
  double nacc[1] = {0.0};
  constexpr int kRv = 10;  // kRes reductions: r^2, r, 8 covariate columns
  double racc[kRes ? kRv : 1];
#pragma unroll
  for (int q = 0; q < (kRes ? kRv : 1); ++q) racc[q] = 0.0;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbytes;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = b * 4;
    const int cnt = (int)((m.n - i0) < 4 ? (m.n - i0) : 4);
    double acc[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) acc[s] = (accumulate && s < cnt) ? out[i0 + s] : 0.0;
    const int64_t tile = b >> 7;
    const int wp = (int)((b >> 2) & 31);
    const int bo = (int)(b & 3);
    // columns in batches of 8: issue the 8 independent byte loads first, then
    // accumulate in the caller's column order
    for (int t0 = 0; t0 < k; t0 += 8) {
      uint32_t bytes[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int t = t0 + q;
        bytes[q] = (t < k && live[t])
                       ? (uint32_t)__ldg(m.x + word_offset_chk(m, tile, cols[t], wp) + bo)
                       : 0u;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int t = t0 + q;
        if (t < k && live[t]) {
#pragma unroll
          for (int s = 0; s < 4; ++s)
            acc[s] = __dadd_rn(acc[s], terms[t][(bytes[q] >> (2 * s)) & 3u]);
        }
      }
    }
    if (kMode == kAxStore) {
#pragma unroll
      for (int s = 0; s < 4; ++s)
        if (s < cnt) out[i0 + s] = acc[s];
    } else if constexpr (kRes) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        if (s >= cnt) continue;
        const int64_t i = i0 + s;
        double ri = 0.0;
        if (!rs.keep || rs.keep[i]) {
          double f = acc[s];
          if (rs.c > 0) {
            double cb = 0.0;
            for (int l = 0; l < rs.c; ++l) cb = __dadd_rn(cb, __dmul_rn(rs.C[i * rs.c + l], rs.bcov[l]));
            f = k > 0 ? __dadd_rn(f, cb) : cb;
          }
          ri = __dsub_rn(rs.y[i], f);
        }
        rs.r[i] = ri;
        racc[0] += ri * ri;
        racc[1] += ri;
        if (rs.gcov) {
#pragma unroll
          for (int l = 0; l < 8; ++l)
            if (l < rs.c) racc[2 + l] += rs.C[i * rs.c + l] * ri;
        }
      }
    } else {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        if (s >= cnt) continue;
        double xi = acc[s];
        if (nm.c > 0) {
          double cb = 0.0;
          for (int l = 0; l < nm.c; ++l)
            cb = __dadd_rn(cb, __dmul_rn(nm.C[(i0 + s) * nm.c + l], nm.wc[l]));
          xi = __dadd_rn(xi, cb);
        }
        if (nm.keep && !nm.keep[i0 + s]) xi = 0.0;
        nacc[0] += xi * xi;
      }
    }
  }
  if constexpr (kRes) {
    __shared__ double shr[kRv * 32];
    block_sum<kRv>(racc, shr);
    if (threadIdx.x == 0)
      for (int q = 0; q < kRv; ++q) rs.ws.partials[blockIdx.x * kRv + q] = racc[q];
    if (last_block(rs.ws.ticket) && threadIdx.x < 32) {
      const double s2 = fold_sum(rs.ws.partials, kRv, 0, gridDim.x);
      const double s1 = fold_sum(rs.ws.partials, kRv, 1, gridDim.x);
      double gl[8];
      if (rs.gcov)
        for (int l = 0; l < rs.c; ++l) gl[l] = fold_sum(rs.ws.partials, kRv, 2 + l, gridDim.x);
      if (threadIdx.x == 0) {
        rs.scal[0] = 0.5 * s2;
        rs.scal[1] = rs.n_eff > 0.0 ? s1 / rs.n_eff : 0.0;
        rs.scal[6] = s1;
        if (rs.gcov)
          for (int l = 0; l < rs.c; ++l) rs.gcov[l] = -gl[l];
        *rs.ws.ticket = 0u;
      }
    }
  }
  if (kNorm) {
    __shared__ double sh[32];
    block_sum<1>(nacc, sh);
    if (threadIdx.x == 0) nm.ws.partials[blockIdx.x] = nacc[0];
    if (last_block(nm.ws.ticket) && threadIdx.x < 32) {
      const double sum = fold_sum(nm.ws.partials, 1, 0, gridDim.x);
      if (threadIdx.x == 0) {
        nm.scal[nm.slot] = sum;
        double ratio = 0.0;
        if (nm.ratio_out >= 0) {
          ratio = nm.ratio_num / sum;
          nm.scal[nm.ratio_out] = ratio;
        }
        if (nm.host_out) {
          nm.host_out[0] = sum;
          nm.host_out[1] = ratio;
        }
        *nm.ws.ticket = 0u;
      }
    }
  }
}

int launch_ax(const MatrixDesc& m, const double* u, const double* v, const int64_t* idx,
              const double* w, int64_t k, double* out, int accumulate, cudaStream_t s) {
  if (m.n == 0) return 0;
  const int64_t nbytes = (m.n + 3) / 4;
  const int threads = 128;
  int64_t blocks = (nbytes + threads - 1) / threads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (k <= 0) {
    if (!accumulate) GI_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * m.n, s));
    return 0;
  }
  for (int64_t c0 = 0; c0 < k; c0 += kAxMaxCols) {
    const int kc = (int)((k - c0) < kAxMaxCols ? (k - c0) : kAxMaxCols);
    ax_kernel<kAxStore><<<(unsigned)blocks, threads, 0, s>>>(m, u, v, idx + c0, w + c0, kc, out,
                                                              (accumulate || c0 > 0) ? 1 : 0,
                                                              AxNorm{}, AxRes{});
    GI_LAUNCH_CHECK();
  }
  return 0;
}

int launch_ax_norm(const MatrixDesc& m, const double* u, const double* v, const int64_t* idx,
                   const double* w, int64_t k, const double* C, int c, const double* wc,
                   const uint8_t* keep, double* scal, int slot, int ratio_out, double ratio_num,
                   double* host_out, double* partials, unsigned int* ticket, cudaStream_t s) {
  if (k > kAxMaxCols || m.n == 0) return -2;  // caller falls back to ax + image_sumsq
  const int64_t nbytes = (m.n + 3) / 4;
  const int threads = 128;
  int64_t blocks = (nbytes + threads - 1) / threads;
  if (blocks > 2 * kRedBlocks) blocks = 2 * kRedBlocks;  // partials: <= 16 * kRedBlocks
  const AxNorm nm{C, c, wc, keep, scal, slot, ratio_out, ratio_num, host_out,
                  RedWs{partials, ticket}};
  ax_kernel<kAxNorm><<<(unsigned)blocks, threads, 0, s>>>(m, u, v, idx, w, (int)k, nullptr, 0, nm,
                                                          AxRes{});
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_ax_residual(const MatrixDesc& m, const double* u, const double* v,
                       const int64_t* idx, const double* w, int64_t k, const double* y,
                       const double* C, int c, const double* bcov, const uint8_t* keep,
                       double n_eff, double* r, double* scal, double* gcov, int64_t sk,
                       const int64_t* sidx, const double* sval, double* beta, double* partials,
                       unsigned int* ticket, cudaStream_t s) {
  if (k > kAxMaxCols || c > 8 || m.n == 0) return -2;  // caller uses the two-kernel path
  const int64_t nbytes = (m.n + 3) / 4;
  const int threads = 128;
  int64_t blocks = (nbytes + threads - 1) / threads;
  if (blocks > kRedBlocks) blocks = kRedBlocks;  // partials: 10 per block
  const AxRes rs{y, C, c, bcov, keep, n_eff, r, scal, c > 0 ? gcov : nullptr, sk, sidx, sval,
                 beta, RedWs{partials, ticket}};
  ax_kernel<kAxRes><<<(unsigned)blocks, threads, 0, s>>>(m, u, v, idx, w, (int)k, nullptr, 0,
                                                         AxNorm{}, rs);
  GI_LAUNCH_CHECK();
  return 0;
}

// out_t is (k, n) row-major: out_t[t, i] = ((dose - u) * v) * obs.
__global__ void decompress_kernel(MatrixDesc m, const double* __restrict__ u,
                                  const double* __restrict__ v, const int64_t* __restrict__ idx,
                                  int64_t k, double* __restrict__ out_t) {
  const int64_t words = (m.n + 15) / 16;
  const int64_t total = words * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / words;
    const int64_t wg = e - t * words;
    const int64_t j = idx[t];
    GI_ASSERT(j >= 0 && j < m.p);
    const double uj = u[j], vj = v[j];
    const uint32_t word =
        *reinterpret_cast<const uint32_t*>(m.x + word_offset_chk(m, wg >> 5, j, (int)(wg & 31)));
    const int64_t i0 = wg * 16;
    double* row = out_t + t * m.n;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      if (i0 + s < m.n) {
        const uint32_t code = (word >> (2 * s)) & 3u;
        const double d = code == 2u ? 1.0 : (code == 3u ? 2.0 : 0.0);
        const double o = code == 1u ? 0.0 : 1.0;
        row[i0 + s] = __dmul_rn(__dmul_rn(__dsub_rn(d, uj), vj), o);
      }
    }
  }
}

int launch_decompress(const MatrixDesc& m, const double* u, const double* v, const int64_t* idx,
                      int64_t k, double* out_t, cudaStream_t s) {
  if (k <= 0 || m.n == 0) return 0;
  const int64_t total = ((m.n + 15) / 16) * k;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  decompress_kernel<<<(unsigned)blocks, 256, 0, s>>>(m, u, v, idx, k, out_t);
  GI_LAUNCH_CHECK();
  return 0;
}

}  // namespace gi
