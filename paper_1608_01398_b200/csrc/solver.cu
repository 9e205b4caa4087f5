// Device-side pieces of the IHT iteration other than X^T r and X_S w:
// residual refresh, centring, covariate gradient, sup-norm reductions and the
// hard-threshold top-k select.
//
// Reference: _refresh_state iht.py:183-191, iht_step iht.py:253-323,
// top_k_indices iht.py:36-49 / hard_threshold :52-58.
//
// All reductions are deterministic: fixed grids write per-block partials and
// the last block to finish (threadfence + atomic ticket) folds them in block
// order, so repeated runs and any stream interleaving give identical bits.
#include "common.cuh"
#include "reduce.cuh"

namespace gi {

// ---------------------------------------------------------------- residual
// r_i = keep_i ? y_i - (fit_i + sum_l C[i, l] bcov[l]) : 0;
// scal[0] = 0.5 * sum r^2 (loss), scal[1] = sum r / n_eff (centring mean).
__global__ void residual_kernel(int64_t n, const double* __restrict__ y,
                                const double* __restrict__ fit, const double* __restrict__ C,
                                int c, const double* __restrict__ bcov,
                                const uint8_t* __restrict__ keep, double n_eff,
                                double* __restrict__ r, double* __restrict__ scal, RedWs ws) {
  __shared__ double sh[64];
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double ri = 0.0;
    if (!keep || keep[i]) {
      double f = fit ? fit[i] : 0.0;
      if (c > 0) {
        double cb = 0.0;
        for (int l = 0; l < c; ++l) cb = __dadd_rn(cb, __dmul_rn(C[i * c + l], bcov[l]));
        f = fit ? __dadd_rn(f, cb) : cb;
      }
      ri = __dsub_rn(y[i], f);
    }
    r[i] = ri;
    acc[0] += ri * ri;
    acc[1] += ri;
  }
  block_sum<2>(acc, sh);
  if (threadIdx.x == 0) {
    ws.partials[blockIdx.x * 2] = acc[0];
    ws.partials[blockIdx.x * 2 + 1] = acc[1];
  }
  if (last_block(ws.ticket) && threadIdx.x < 32) {
    const double s2 = fold_sum(ws.partials, 2, 0, gridDim.x);
    const double s1 = fold_sum(ws.partials, 2, 1, gridDim.x);
    if (threadIdx.x == 0) {
      scal[0] = 0.5 * s2;
      scal[1] = n_eff > 0.0 ? s1 / n_eff : 0.0;
      *ws.ticket = 0u;
    }
  }
}
// Refresh prologue of the native loop: optional beta writes (block 0:
// beta[sidx[t]] = sval[t]), the residual as residual_kernel, and with kCov the
// covariate gradient gcov[l] = -sum_i C[i, l] r_i of covgrad_kernel in the
// same pass -- same grid, per-thread order and block-order fold, so the same
// bits as the two separate kernels.  Partials: 10 per block.
template <bool kCov>
__global__ void refresh_residual_kernel(int64_t n, const double* __restrict__ y,
                                        const double* __restrict__ fit,
                                        const double* __restrict__ C, int c,
                                        const double* __restrict__ bcov,
                                        const uint8_t* __restrict__ keep, double n_eff,
                                        double* __restrict__ r, double* __restrict__ scal,
                                        double* __restrict__ gcov, int64_t sk,
                                        const int64_t* __restrict__ sidx,
                                        const double* __restrict__ sval,
                                        double* __restrict__ beta, RedWs ws) {
  constexpr int NV = kCov ? 10 : 2;
  __shared__ double sh[NV * 32];
  if (blockIdx.x == 0)
    for (int64_t t = threadIdx.x; t < sk; t += blockDim.x) beta[sidx[t]] = sval[t];
  double acc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double ri = 0.0;
    if (!keep || keep[i]) {
      double f = fit ? fit[i] : 0.0;
      if (c > 0) {
        double cb = 0.0;
        for (int l = 0; l < c; ++l) cb = __dadd_rn(cb, __dmul_rn(C[i * c + l], bcov[l]));
        f = fit ? __dadd_rn(f, cb) : cb;
      }
      ri = __dsub_rn(y[i], f);
    }
    r[i] = ri;
    acc[0] += ri * ri;
    acc[1] += ri;
    if (kCov) {
#pragma unroll
      for (int l = 0; l < 8; ++l)
        if (l < c) acc[2 + l] += C[i * c + l] * ri;
    }
  }
  block_sum<NV>(acc, sh);
  if (threadIdx.x == 0)
    for (int q = 0; q < NV; ++q) ws.partials[blockIdx.x * NV + q] = acc[q];
  if (last_block(ws.ticket) && threadIdx.x < 32) {
    const double s2 = fold_sum(ws.partials, NV, 0, gridDim.x);
    const double s1 = fold_sum(ws.partials, NV, 1, gridDim.x);
    double gl[8];
    if (kCov)
      for (int l = 0; l < c; ++l) gl[l] = fold_sum(ws.partials, NV, 2 + l, gridDim.x);
    if (threadIdx.x == 0) {
      scal[0] = 0.5 * s2;
      scal[1] = n_eff > 0.0 ? s1 / n_eff : 0.0;
      scal[6] = s1;  // sum of r, for the exact X^T r kernel
      if (kCov)
        for (int l = 0; l < c; ++l) gcov[l] = -gl[l];
      *ws.ticket = 0u;
    }
  }
}


// rt_i = keep_i ? fp32(r_i - mean) : 0 over the padded length; scal[2] = sum rt.
__global__ void center_kernel(int64_t n, int64_t n_pad, const double* __restrict__ r,
                              const uint8_t* __restrict__ keep, double* __restrict__ scal,
                              float* __restrict__ rt, RedWs ws) {
  __shared__ double sh[32];
  const double mean = scal[1];
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pad;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.0f;
    if (i < n && (!keep || keep[i])) v = (float)(r[i] - mean);
    rt[i] = v;
    acc[0] += (double)v;
  }
  block_sum<1>(acc, sh);
  if (threadIdx.x == 0) ws.partials[blockIdx.x] = acc[0];
  if (last_block(ws.ticket) && threadIdx.x < 32) {
    const double s = fold_sum(ws.partials, 1, 0, gridDim.x);
    if (threadIdx.x == 0) {
      scal[2] = s;
      scal[3] = 0.0;  // max|g| accumulator of the X^T r epilogue that follows
      *ws.ticket = 0u;
    }
  }
}

// gcov[l] = -sum_i C[i, l] r_i  (covariate block of the gradient)
__global__ void covgrad_kernel(int64_t n, const double* __restrict__ C, int stride, int c,
                               const double* __restrict__ r, double* __restrict__ gcov,
                               RedWs ws) {
  __shared__ double sh[8 * 32];
  double acc[8];
#pragma unroll
  for (int l = 0; l < 8; ++l) acc[l] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = r[i];
#pragma unroll
    for (int l = 0; l < 8; ++l)
      if (l < c) acc[l] += C[i * stride + l] * ri;
  }
  block_sum<8>(acc, sh);
  if (threadIdx.x == 0)
    for (int l = 0; l < 8; ++l) ws.partials[blockIdx.x * 8 + l] = acc[l];
  if (last_block(ws.ticket) && threadIdx.x < 32) {
    for (int l = 0; l < c; ++l) {
      const double s = fold_sum(ws.partials, 8, l, gridDim.x);
      if (threadIdx.x == 0) gcov[l] = -s;
    }
    if (threadIdx.x == 0) *ws.ticket = 0u;
  }
}

// scal[slot] = max_j |x_j|
__global__ void maxabs_kernel(int64_t m, const double* __restrict__ x, double* __restrict__ scal,
                              int slot, RedWs ws) {
  __shared__ double sh[32];
  double mx = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    mx = fmax(mx, fabs(x[i]));
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, sh[w]);
    ws.partials[blockIdx.x] = mx;
  }
  if (last_block(ws.ticket) && threadIdx.x < 32) {
    const double s = fold_max(ws.partials, gridDim.x);
    if (threadIdx.x == 0) {
      scal[slot] = s;
      *ws.ticket = 0u;
    }
  }
}

// scal[slot] = sum_i x_i^2
__global__ void sumsq_kernel(int64_t m, const double* __restrict__ x, double* __restrict__ scal,
                             int slot, RedWs ws) {
  __shared__ double sh[32];
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    acc[0] += x[i] * x[i];
  block_sum<1>(acc, sh);
  if (threadIdx.x == 0) ws.partials[blockIdx.x] = acc[0];
  if (last_block(ws.ticket) && threadIdx.x < 32) {
    const double s = fold_sum(ws.partials, 1, 0, gridDim.x);
    if (threadIdx.x == 0) {
      scal[slot] = s;
      *ws.ticket = 0u;
    }
  }
}

// Fused image norm of the native loop: scal[slot] = sum_i keep_i (x_i + C_i w)^2
// -- add_cov, mask and sumsq in one pass, with the same per-element operations
// (so the same bits).  When ratio_out >= 0 the last block also writes the
// normalised step scal[ratio_out] = ratio_num / scal[slot] (iht.py:244), and
// host_out (mapped host memory, may be NULL) receives {scal[slot], ratio}.
__global__ void image_sumsq_kernel(int64_t m, const double* __restrict__ x,
                                   const double* __restrict__ C, int c,
                                   const double* __restrict__ w, const uint8_t* __restrict__ keep,
                                   double* __restrict__ scal, int slot, int ratio_out,
                                   double ratio_num, double* __restrict__ host_out, RedWs ws) {
  __shared__ double sh[32];
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    double xi = x[i];
    if (c > 0) {
      double cb = 0.0;
      for (int l = 0; l < c; ++l) cb = __dadd_rn(cb, __dmul_rn(C[i * c + l], w[l]));
      xi = __dadd_rn(xi, cb);
    }
    if (keep && !keep[i]) xi = 0.0;
    acc[0] += xi * xi;
  }
  block_sum<1>(acc, sh);
  if (threadIdx.x == 0) ws.partials[blockIdx.x] = acc[0];
  if (last_block(ws.ticket) && threadIdx.x < 32) {
    const double s = fold_sum(ws.partials, 1, 0, gridDim.x);
    if (threadIdx.x == 0) {
      scal[slot] = s;
      double ratio = 0.0;
      if (ratio_out >= 0) {
        ratio = ratio_num / s;
        scal[ratio_out] = ratio;
      }
      if (host_out) {
        host_out[0] = s;
        host_out[1] = ratio;
      }
      *ws.ticket = 0u;
    }
  }
}

// Copy (or gather, when idx != NULL) up to kMaxPub segments of 8-byte words
// into `out` -- mapped host memory -- so a phase's results reach the host with
// one small launch instead of one copy-engine transfer per array.
__global__ void publish_kernel(PubArgs a, unsigned long long* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int q = 0; q < a.nseg; ++q) {
    const PubSeg sg = a.seg[q];
    const unsigned long long* src = static_cast<const unsigned long long*>(sg.src);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < sg.count; t += stride)
      out[sg.dst + t] = sg.idx ? src[sg.idx[t]] : src[t];
  }
}

// out = x + C @ w (length n; C row-major (n, c)); used for X_S w + C w_cov
__global__ void add_cov_kernel(int64_t n, const double* __restrict__ C, int c,
                               const double* __restrict__ w, double* __restrict__ x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double cb = 0.0;
    for (int l = 0; l < c; ++l) cb = __dadd_rn(cb, __dmul_rn(C[i * c + l], w[l]));
    x[i] = __dadd_rn(x[i], cb);
  }
}

static int red_grid(int64_t m) {
  int64_t g = (m + kRedThreads - 1) / kRedThreads;
  if (g > kRedBlocks) g = kRedBlocks;
  if (g < 1) g = 1;
  return (int)g;
}

int launch_refresh_residual(int64_t n, const double* y, const double* fit, const double* C,
                            int c, const double* bcov, const uint8_t* keep, double n_eff,
                            double* r, double* scal, double* gcov, int64_t sk,
                            const int64_t* sidx, const double* sval, double* beta,
                            double* partials, unsigned int* ticket, cudaStream_t s) {
  RedWs ws{partials, ticket};
  if (gcov && c > 0 && c <= 8)
    refresh_residual_kernel<true><<<red_grid(n), kRedThreads, 0, s>>>(
        n, y, fit, C, c, bcov, keep, n_eff, r, scal, gcov, sk, sidx, sval, beta, ws);
  else
    refresh_residual_kernel<false><<<red_grid(n), kRedThreads, 0, s>>>(
        n, y, fit, C, c, bcov, keep, n_eff, r, scal, nullptr, sk, sidx, sval, beta, ws);
  GI_LAUNCH_CHECK();
  if (gcov && c > 8) return launch_covgrad(n, C, c, r, gcov, partials, ticket, s);
  return 0;
}

int launch_residual(int64_t n, const double* y, const double* fit, const double* C, int c,
                    const double* bcov, const uint8_t* keep, double n_eff, double* r,
                    double* scal, double* partials, unsigned int* ticket, cudaStream_t s) {
  RedWs ws{partials, ticket};
  residual_kernel<<<red_grid(n), kRedThreads, 0, s>>>(n, y, fit, C, c, bcov, keep, n_eff, r,
                                                     scal, ws);
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_center(int64_t n, int64_t n_pad, const double* r, const uint8_t* keep, double* scal,
                  float* rt, double* partials, unsigned int* ticket, cudaStream_t s) {
  RedWs ws{partials, ticket};
  center_kernel<<<red_grid(n_pad), kRedThreads, 0, s>>>(n, n_pad, r, keep, scal, rt, ws);
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_covgrad(int64_t n, const double* C, int c, const double* r, double* gcov,
                   double* partials, unsigned int* ticket, cudaStream_t s) {
  if (c <= 0) return 0;
  RedWs ws{partials, ticket};
  // 8 columns per launch; column block l0 reads C[i * c + l0 + l] through a
  // row stride of c
  for (int l0 = 0; l0 < c; l0 += 8) {
    const int cc = c - l0 < 8 ? c - l0 : 8;
    covgrad_kernel<<<red_grid(n), kRedThreads, 0, s>>>(n, C + l0, c, cc, r, gcov + l0, ws);
    GI_LAUNCH_CHECK();
  }
  return 0;
}

int launch_maxabs(int64_t m, const double* x, double* scal, int slot, double* partials,
                  unsigned int* ticket, cudaStream_t s) {
  RedWs ws{partials, ticket};
  maxabs_kernel<<<red_grid(m), kRedThreads, 0, s>>>(m, x, scal, slot, ws);
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_sumsq(int64_t m, const double* x, double* scal, int slot, double* partials,
                 unsigned int* ticket, cudaStream_t s) {
  RedWs ws{partials, ticket};
  sumsq_kernel<<<red_grid(m), kRedThreads, 0, s>>>(m, x, scal, slot, ws);
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_image_sumsq(int64_t m, const double* x, const double* C, int c, const double* w,
                       const uint8_t* keep, double* scal, int slot, int ratio_out,
                       double ratio_num, double* host_out, double* partials,
                       unsigned int* ticket, cudaStream_t s) {
  RedWs ws{partials, ticket};
  image_sumsq_kernel<<<red_grid(m), kRedThreads, 0, s>>>(m, x, C, c, w, keep, scal, slot,
                                                         ratio_out, ratio_num, host_out, ws);
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_publish(const PubArgs& a, void* out, cudaStream_t s) {
  int64_t most = 0;
  for (int q = 0; q < a.nseg; ++q) most = a.seg[q].count > most ? a.seg[q].count : most;
  if (most == 0) return 0;
  int64_t blocks = (most + 255) / 256;
  if (blocks > 64) blocks = 64;
  publish_kernel<<<(unsigned)blocks, 256, 0, s>>>(a, static_cast<unsigned long long*>(out));
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_add_cov(int64_t n, const double* C, int c, const double* w, double* x,
                   cudaStream_t s) {
  if (c <= 0 || n == 0) return 0;
  add_cov_kernel<<<red_grid(n), kRedThreads, 0, s>>>(n, C, c, w, x);
  GI_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------- top-k
// Exact k largest under the total order (key desc, index asc) -- the
// reference's "ties go to the lower index" rule (iht.py:44-49).  Keys are the
// bit patterns of |value| (non-negative doubles order like uint64), stored +1
// so that 0 marks an empty slot.  Radix select over 8 key digits and 4 digits
// of ~index (MSB first), stopping as soon as the boundary bin is taken whole.
constexpr int kTopkChunk = 4096;
constexpr int kTopkThreads = 512;

// Shared-memory state of one block-wide select, declared once per kernel
// (static __shared__ inside the templates would be duplicated per Get type).
struct SelShared {
  unsigned int hist[256];
  uint64_t s_key, s_kmask;
  uint32_t s_sec, s_smask;
  int64_t s_kk;
  int s_done;
};

template <typename Get>
__device__ void block_select(int64_t m, int64_t k, Get get, uint64_t& thr_key,
                             uint32_t& thr_sec, SelShared& sh) {
  unsigned int* hist = sh.hist;
  uint64_t &s_key = sh.s_key, &s_kmask = sh.s_kmask;
  uint32_t &s_sec = sh.s_sec, &s_smask = sh.s_smask;
  int64_t& s_kk = sh.s_kk;
  int& s_done = sh.s_done;
  if (threadIdx.x == 0) {
    s_key = 0;
    s_kmask = 0;
    s_sec = 0;
    s_smask = 0;
    s_kk = k;
    s_done = 0;
  }
  __syncthreads();
  for (int d = 0; d < 12; ++d) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0u;
    __syncthreads();
    const uint64_t pk = s_key, mk = s_kmask;
    const uint32_t ps = s_sec, ms = s_smask;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
      uint64_t key;
      uint32_t sec;
      get(i, key, sec);
      if ((key & mk) == pk && (sec & ms) == ps) {
        const unsigned digit = d < 8 ? (unsigned)((key >> (56 - 8 * d)) & 255u)
                                     : (unsigned)((sec >> (24 - 8 * (d - 8))) & 255u);
        atomicAdd(&hist[digit], 1u);
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // warp-parallel search for the boundary bin: lane l owns bins 8l..8l+7;
      // `above` = number of candidates in bins higher than the lane's range
      const int lane = threadIdx.x;
      unsigned c[8];
      unsigned tot = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        c[q] = hist[8 * lane + q];
        tot += c[q];
      }
      unsigned incl = tot;  // inclusive suffix sum over lanes >= lane
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_down_sync(0xffffffffu, incl, o);
        if (lane + o < 32) incl += t;
      }
      const unsigned above = incl - tot;
      const int64_t need0 = s_kk;
      // the boundary lane: above < need0 <= above + tot (or lane 0 if total < need0)
      const bool mine = ((int64_t)above < need0 && need0 <= (int64_t)(above + tot)) ||
                        (lane == 0 && (int64_t)incl < need0);
      if (mine) {
        int64_t need = need0 - (int64_t)above;
        int bin = 8 * lane + 7;
        for (int q = 7; q >= 0; --q) {
          bin = 8 * lane + q;
          if ((int64_t)c[q] >= need) break;
          need -= c[q];
        }
        if (d < 8) {
          s_key |= (uint64_t)bin << (56 - 8 * d);
          s_kmask |= (uint64_t)255u << (56 - 8 * d);
        } else {
          s_sec |= (uint32_t)bin << (24 - 8 * (d - 8));
          s_smask |= 255u << (24 - 8 * (d - 8));
        }
        s_kk = need;
        if ((int64_t)hist[bin] == need) s_done = 1;
      }
    }
    __syncthreads();
    if (s_done) break;
  }
  thr_key = s_key;
  thr_sec = s_sec;
  __syncthreads();
}

__device__ __forceinline__ bool ge_thr(uint64_t key, uint32_t sec, uint64_t tk, uint32_t ts) {
  return key > tk || (key == tk && sec >= ts);
}


// mode 0: value = g_j; mode 1: value = beta_j - mu * g_j.  key = |value|.
__device__ __forceinline__ double topk_value(int mode, const double* beta, const double* g,
                                             double mu, int64_t j) {
  if (mode == 0) return g[j];
  return __dsub_rn(beta[j], __dmul_rn(mu, g[j]));
}

__device__ __forceinline__ uint64_t key_of(double val) {
  return (uint64_t)__double_as_longlong(fabs(val)) + 1ull;
}

// Exact top-k over `mc` candidates -> out (unordered) + count, by one block.
// kL2: read the candidates through L2 only (ld.global.cg) -- they were written
// by other blocks of the same launch (the fused form below).
template <bool kL2>
__device__ void topk_merge_body(int64_t mc, int64_t k, const uint64_t* cand_key,
                                const int64_t* cand_idx, const double* cand_val,
                                int64_t* out_idx, double* out_val, uint64_t* out_key,
                                int64_t* out_count, SelShared& sh) {
  __shared__ unsigned int s_pos;
  if (threadIdx.x == 0) s_pos = 0u;
  __syncthreads();
  auto key_at = [&](int64_t i) -> uint64_t {
    return kL2 ? (uint64_t)__ldcg(reinterpret_cast<const unsigned long long*>(cand_key) + i)
               : cand_key[i];
  };
  auto idx_at = [&](int64_t i) -> int64_t {
    return kL2 ? (int64_t)__ldcg(reinterpret_cast<const long long*>(cand_idx) + i)
               : cand_idx[i];
  };
  auto get = [&](int64_t i, uint64_t& key, uint32_t& sec) {
    key = key_at(i);
    sec = ~(uint32_t)idx_at(i);
  };
  uint64_t tk;
  uint32_t ts;
  block_select(mc, k, get, tk, ts, sh);
  if (tk == 0) tk = 1;  // never take empty slots
  for (int64_t i = threadIdx.x; i < mc; i += blockDim.x) {
    uint64_t key;
    uint32_t sec;
    get(i, key, sec);
    if (ge_thr(key, sec, tk, ts)) {
      const unsigned pos = atomicAdd(&s_pos, 1u);
      if (pos < k) {
        out_idx[pos] = idx_at(i);
        out_val[pos] = kL2 ? __ldcg(cand_val + i) : cand_val[i];
        if (out_key) out_key[pos] = key;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *out_count = s_pos < k ? (int64_t)s_pos : k;
}

struct MergeOut {
  unsigned int* ticket;  // NULL: the merge runs as its own kernel
  int64_t* idx;
  double* val;
  uint64_t* key;
  int64_t* count;
};

// One block per chunk of kTopkChunk elements; writes k candidate slots
// (cand_key = 0 marks an unused slot).
__global__ void __launch_bounds__(kTopkThreads) topk_local_kernel(
    int64_t p, int64_t k, int mode, const double* __restrict__ beta,
    const double* __restrict__ g, double mu_host, const double* __restrict__ mu_dev,
    int64_t idx_base, uint64_t* __restrict__ cand_key,
    int64_t* __restrict__ cand_idx, double* __restrict__ cand_val, MergeOut mo) {
  __shared__ uint64_t keys[kTopkChunk];
  __shared__ unsigned int s_pos;
  __shared__ SelShared sel;
  const double mu = mu_dev ? *mu_dev : mu_host;
  const int64_t lo = (int64_t)blockIdx.x * kTopkChunk;
  const int64_t hi = lo + kTopkChunk < p ? lo + kTopkChunk : p;
  const int64_t m = hi - lo;
  {
    // all of a thread's loads first, then the keys (the same operations as
    // topk_value): a strided loop issued them one round trip at a time
    constexpr int kPer = kTopkChunk / kTopkThreads;
    double gv[kPer], bv[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int64_t i = threadIdx.x + (int64_t)q * kTopkThreads;
      gv[q] = i < m ? __ldg(g + lo + i) : 0.0;
      bv[q] = (mode != 0 && i < m) ? __ldg(beta + lo + i) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int64_t i = threadIdx.x + (int64_t)q * kTopkThreads;
      if (i < m) keys[i] = key_of(mode == 0 ? gv[q] : __dsub_rn(bv[q], __dmul_rn(mu, gv[q])));
    }
  }
  if (threadIdx.x == 0) s_pos = 0u;
  __syncthreads();
  uint64_t tk;
  uint32_t ts;
  auto get = [&](int64_t i, uint64_t& key, uint32_t& sec) {
    key = keys[i];
    sec = ~(uint32_t)(idx_base + lo + i);
  };
  const int64_t kk = k < m ? k : m;
  if (kk < m) {
    block_select(m, kk, get, tk, ts, sel);
  } else {
    tk = 1;
    ts = 0;  // take everything
  }
  uint64_t* ok = cand_key + (int64_t)blockIdx.x * k;
  int64_t* oi = cand_idx + (int64_t)blockIdx.x * k;
  double* ov = cand_val + (int64_t)blockIdx.x * k;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    uint64_t key;
    uint32_t sec;
    get(i, key, sec);
    if (ge_thr(key, sec, tk, ts)) {
      const unsigned pos = atomicAdd(&s_pos, 1u);
      GI_ASSERT(pos < kk);
      ok[pos] = key;
      oi[pos] = idx_base + lo + i;
      ov[pos] = topk_value(mode, beta, g, mu, lo + i);
    }
  }
  __syncthreads();
  for (int64_t s = s_pos + threadIdx.x; s < k; s += blockDim.x) {
    ok[s] = 0;
    oi[s] = -1;
    ov[s] = 0.0;
  }
  // fused merge: the last block to finish selects over all blocks' candidates
  if (mo.ticket) {
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = atomicAdd(mo.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (is_last) {
      __threadfence();
      topk_merge_body<true>((int64_t)gridDim.x * k, k, cand_key, cand_idx, cand_val, mo.idx,
                            mo.val, mo.key, mo.count, sel);
      if (threadIdx.x == 0) *mo.ticket = 0u;
    }
  }
}

__global__ void __launch_bounds__(kTopkThreads) topk_merge_kernel(
    int64_t mc, int64_t k, const uint64_t* __restrict__ cand_key,
    const int64_t* __restrict__ cand_idx, const double* __restrict__ cand_val,
    int64_t* __restrict__ out_idx, double* __restrict__ out_val, uint64_t* __restrict__ out_key,
    int64_t* __restrict__ out_count) {
  __shared__ SelShared sel;
  topk_merge_body<false>(mc, k, cand_key, cand_idx, cand_val, out_idx, out_val, out_key,
                         out_count, sel);
}

int64_t topk_blocks(int64_t p) { return (p + kTopkChunk - 1) / kTopkChunk; }

int launch_topk(int64_t p, int64_t k, int mode, const double* beta, const double* g, double mu,
                int64_t idx_base, uint64_t* cand_key, int64_t* cand_idx, double* cand_val,
                int64_t* out_idx, double* out_val, uint64_t* out_key, int64_t* out_count,
                cudaStream_t s, const double* mu_dev, unsigned int* ticket) {
  if (k <= 0 || p <= 0) {
    GI_CUDA_TRY(cudaMemsetAsync(out_count, 0, sizeof(int64_t), s));
    return 0;
  }
  const int64_t nb = topk_blocks(p);
  // with a ticket (zero on entry, zero again on exit) the merge runs in the
  // last local block: one launch instead of two
  const MergeOut mo{ticket, out_idx, out_val, out_key, out_count};
  topk_local_kernel<<<(unsigned)nb, kTopkThreads, 0, s>>>(p, k, mode, beta, g, mu, mu_dev,
                                                          idx_base, cand_key, cand_idx, cand_val,
                                                          mo);
  GI_LAUNCH_CHECK();
  if (!ticket) {
    topk_merge_kernel<<<1, kTopkThreads, 0, s>>>(nb * k, k, cand_key, cand_idx, cand_val, out_idx,
                                         out_val, out_key, out_count);
    GI_LAUNCH_CHECK();
  }
  return 0;
}

// ---------------------------------------------------------------- shard exchange
// Device side of the sharded loop's exchanges (fit.cu, gi_fit_sharded).
// mine = [max|g| (scal[3]), g[gsel[t]] or 0 for each global support entry t]
__global__ void shard_gather_kernel(int64_t kg, const int64_t* __restrict__ gsel,
                                    const double* __restrict__ g,
                                    const double* __restrict__ scal3,
                                    double* __restrict__ mine) {
  if (threadIdx.x == 0) mine[0] = *scal3;
  for (int64_t t = threadIdx.x; t < kg; t += blockDim.x)
    mine[1 + t] = gsel[t] >= 0 ? g[gsel[t]] : 0.0;
}

// out = [max over ranks of all[r][0], sum over ranks of all[r][1 + t]], ranks in
// order (the same operations as the host fold it replaces)
__global__ void shard_fold_kernel(int world, int64_t kg, const double* __restrict__ all,
                                  double* __restrict__ out) {
  const int64_t row = 1 + kg;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int r = 0; r < world; ++r) m = fmax(m, all[r * row]);
    out[0] = m;
  }
  for (int64_t t = threadIdx.x; t < kg; t += blockDim.x) {
    double acc = 0.0;
    for (int r = 0; r < world; ++r) acc += all[r * row + 1 + t];
    out[1 + t] = acc;
  }
}

// rank-major [key | idx | val] x world -> contiguous candidate arrays
__global__ void shard_cands_kernel(int world, int64_t ke, const double* __restrict__ all,
                                   uint64_t* __restrict__ ckey, int64_t* __restrict__ cidx,
                                   double* __restrict__ cval) {
  const int64_t total = (int64_t)world * ke;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / ke, s2 = e - r * ke;
    const double* base = all + r * 3 * ke;
    ckey[e] = (uint64_t)__double_as_longlong(base[s2]);
    cidx[e] = (int64_t)__double_as_longlong(base[ke + s2]);
    cval[e] = base[2 * ke + s2];
  }
}

int launch_shard_gather(int64_t kg, const int64_t* gsel, const double* g, const double* scal3,
                        double* mine, cudaStream_t s) {
  shard_gather_kernel<<<1, 256, 0, s>>>(kg, gsel, g, scal3, mine);
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_shard_fold(int world, int64_t kg, const double* all, double* out, cudaStream_t s) {
  shard_fold_kernel<<<1, 256, 0, s>>>(world, kg, all, out);
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_shard_merge(int world, int64_t ke, const double* all, uint64_t* ckey, int64_t* cidx,
                       double* cval, int64_t* out_idx, double* out_val, uint64_t* out_key,
                       int64_t* out_count, cudaStream_t s) {
  const int64_t total = (int64_t)world * ke;
  shard_cands_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(world, ke, all, ckey, cidx,
                                                                     cval);
  GI_LAUNCH_CHECK();
  topk_merge_kernel<<<1, kTopkThreads, 0, s>>>(total, ke, ckey, cidx, cval, out_idx, out_val,
                                               out_key, out_count);
  GI_LAUNCH_CHECK();
  return 0;
}

// dense beta update: beta[idx[t]] = val[t]
__global__ void scatter_kernel(int64_t k, const int64_t* __restrict__ idx,
                               const double* __restrict__ val, double* __restrict__ beta) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < k) beta[idx[t]] = val[t];
}

__global__ void gather_kernel(int64_t k, const int64_t* __restrict__ idx,
                              const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < k) dst[t] = src[idx[t]];
}

int launch_scatter(int64_t k, const int64_t* idx, const double* val, double* beta,
                   cudaStream_t s) {
  if (k <= 0) return 0;
  scatter_kernel<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(k, idx, val, beta);
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_gather(int64_t k, const int64_t* idx, const double* src, double* dst,
                  cudaStream_t s) {
  if (k <= 0) return 0;
  gather_kernel<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(k, idx, src, dst);
  GI_LAUNCH_CHECK();
  return 0;
}

}  // namespace gi
