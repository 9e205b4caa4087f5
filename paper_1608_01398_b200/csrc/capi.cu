// C ABI of libgenoiht_cuda.so (include/genoiht_cuda.h): handle management,
// host-buffer operators and the stateless device primitives of the IHT loop.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <memory>
#include <mutex>
#include <vector>

#include "../../include/genoiht_cuda.h"
#include "handle.cuh"

// ------------------------------------------------------------------ errors
static thread_local char g_err[1024] = "";

void gi_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static int matrix_shell(int64_t n, int64_t p, int device, gi_matrix** out,
                        std::unique_ptr<gi_matrix>& h, bool zero_tiles = true) {
  CHECK_ARG(out != nullptr, "output handle pointer is NULL");
  CHECK_ARG(n >= 0 && p >= 0, "matrix dimensions must be non-negative");
  int count = 0;
  GI_CUDA_TRY(cudaGetDeviceCount(&count));
  CHECK_ARG(device >= 0 && device < count, "CUDA device index out of range");
  h.reset(new gi_matrix());
  h->device = device;
  h->sms = sm_count_of(device);
  h->n = n;
  h->p = p;
  h->nb = (n + 3) / 4;
  h->T = (h->nb + GI_TILE_BYTES - 1) / GI_TILE_BYTES;
  h->G = (p + GI_GROUP - 1) / GI_GROUP;
  GI_CUDA_TRY(cudaSetDevice(device));
  GI_CUDA_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  TRY(alloc(h->x, (size_t)(h->T * h->G) * GI_BLOCK_BYTES, device, zero_tiles));
  TRY(alloc(h->u, sizeof(double) * p, device, true));
  TRY(alloc(h->v, sizeof(double) * p, device, true));
  TRY(alloc(h->miss_cnt, sizeof(int32_t) * p, device, true));
  TRY(alloc(h->gmiss, (size_t)h->G, device, true));
  TRY(alloc(h->s1cnt, sizeof(int32_t) * 2 * p, device, true));
  return 0;
}

// The base-3 copy X^T r streams instead of the 2-bit tiles: 1.6 instead of 2
// bits per genotype, so 20% fewer HBM bytes and table lookups per sweep.  A
// matrix with missing genotypes gets it too when they are at most 5% of the
// genotypes: the base-3 copy holds them as dose 0 and a list of their
// positions (missing.cu, 2 B each) supplies the missing sums m_j, which the
// 2-bit kernel gets from a second table lookup per byte.  Built only when it
// leaves 1/8 of the device memory free; GI_BASE3=0 disables it, GI_MISSLIST=0
// keeps matrices with missing genotypes on the 2-bit tiles.
// want: 0 drop the copy, 1 build it if possible.
static int set_base3(gi_matrix* h, int want) {
  if (!want) {
    if (h->x3) GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
    h->x3.reset();
    h->mlist.reset();
    h->mofs.reset();
    h->T3 = 0;
    return 0;
  }
  if (h->x3 || h->n == 0 || h->p == 0) return 0;
  std::vector<int32_t> miss((size_t)h->p);
  GI_CUDA_TRY(cudaMemcpy(miss.data(), h->miss_cnt->ptr, sizeof(int32_t) * h->p,
                         cudaMemcpyDeviceToHost));
  int64_t total = 0;
  for (int32_t c : miss) total += c;
  if (total > 0) {
    const char* env = getenv("GI_MISSLIST");
    if ((env && env[0] == '0') || (double)total > 0.05 * (double)h->n * (double)h->p) return 0;
  }
  const int64_t T3 = gi::tiles3_of(h->n);
  const int64_t nblk = h->T * h->G;
  const size_t bytes3 = (size_t)(T3 * h->G) * GI_BLOCK_BYTES;
  const size_t list_bytes = total > 0 ? (size_t)total * 2 + (size_t)(nblk + 1) * 8 : 0;
  size_t free_b = 0, total_b = 0;
  GI_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  // the list build also needs nblk + 1 counts and the scan's scratch
  if (bytes3 + 2 * list_bytes + total_b / 8 > free_b) return 0;
  std::shared_ptr<DevMem> x3, mlist, mofs;
  if (total > 0) {
    gi::MatrixDesc d = h->desc();
    std::shared_ptr<DevMem> cnt, tmp;
    TRY(alloc(cnt, (size_t)(nblk + 1) * 8, h->device, true));
    // + 16 B: staged offset ranges end on a 16-byte boundary
    TRY(alloc(mofs, (size_t)(nblk + 1) * 8 + 16, h->device, false));
    // + 16 B: the staged copies round the entry range up to 16-byte units
    TRY(alloc(mlist, (size_t)total * 2 + 16, h->device, false));
    TRY(gi::missing_list_count(d, static_cast<int64_t*>(cnt->ptr), h->stream));
    size_t tmp_bytes = 0;
    TRY(gi::missing_list_scan(static_cast<int64_t*>(cnt->ptr), static_cast<int64_t*>(mofs->ptr),
                              nblk, nullptr, tmp_bytes, h->stream));
    TRY(alloc(tmp, tmp_bytes + 16, h->device, false));
    TRY(gi::missing_list_scan(static_cast<int64_t*>(cnt->ptr), static_cast<int64_t*>(mofs->ptr),
                              nblk, tmp->ptr, tmp_bytes, h->stream));
    int64_t got = 0;
    GI_CUDA_TRY(cudaMemcpyAsync(&got, static_cast<int64_t*>(mofs->ptr) + nblk, 8,
                                cudaMemcpyDeviceToHost, h->stream));
    GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (got != total) {
      gi_set_error("internal: missing-genotype list holds %lld entries, counts say %lld",
                   (long long)got, (long long)total);
      return -1;
    }
    TRY(gi::missing_list_fill(d, static_cast<int64_t*>(mofs->ptr),
                              static_cast<uint16_t*>(mlist->ptr), h->stream));
    GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  TRY(alloc(x3, bytes3, h->device, false));
  h->x3 = x3;
  h->T3 = T3;
  h->mlist = mlist;
  h->mofs = mofs;
  h->mtotal = total;
  TRY(gi::launch_pack3(h->desc(), static_cast<uint8_t*>(x3->ptr), h->stream));
  GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

static int finish_stats(gi_matrix* h) {
  gi::MatrixDesc d = h->desc();
  TRY(gi::launch_stats(d, nullptr, h->du(), h->dv(), static_cast<int32_t*>(h->miss_cnt->ptr),
                       static_cast<int32_t*>(h->s1cnt->ptr), h->stream));
  TRY(gi::launch_group_flags(d, static_cast<int32_t*>(h->miss_cnt->ptr),
                             static_cast<uint8_t*>(h->gmiss->ptr), h->stream));
  GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
  const char* env = getenv("GI_BASE3");
  TRY(set_base3(h, !(env && env[0] == '0')));
  return 0;
}

extern "C" {

int gi_version(void) { return 100; }

const char* gi_last_error(void) { return g_err; }

int gi_device_count(int* count) {
  CHECK_ARG(count != nullptr, "count is NULL");
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *count = c;
  return 0;
}

int gi_device_info(int device, int* sm_count, int64_t* mem_bytes, int64_t* l2_bytes) {
  cudaDeviceProp prop;
  GI_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (mem_bytes) *mem_bytes = (int64_t)prop.totalGlobalMem;
  if (l2_bytes) *l2_bytes = (int64_t)prop.l2CacheSize;
  return 0;
}

int gi_device_sync(int device) {
  DeviceGuard g(device);
  GI_CUDA_TRY(cudaDeviceSynchronize());
  return 0;
}

int gi_matrix_create(int64_t n, int64_t p, int device, gi_matrix** out) {
  std::unique_ptr<gi_matrix> h;
  TRY(matrix_shell(n, p, device, out, h));
  *out = h.release();
  return 0;
}

int gi_matrix_upload_bed(gi_matrix* h, int64_t j0, int64_t count, const uint8_t* data) {
  CHECK_ARG(h != nullptr, "NULL handle");
  CHECK_ARG(j0 >= 0 && count >= 0 && j0 + count <= h->p, "SNP range out of bounds");
  if (count == 0 || h->nb == 0) return 0;
  CHECK_ARG(data != nullptr, "BED buffer is NULL");
  std::lock_guard<std::mutex> lock(h->mu);
  DeviceGuard g(h->device);
  // stream through a pinned staging buffer in chunks of ~256 MiB
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>((int64_t)(256ll << 20) / h->nb,
                                                               count));
  TRY(h->s_a.ensure((size_t)(chunk * h->nb), h->device));
  void* pinned = nullptr;
  GI_CUDA_TRY(cudaMallocHost(&pinned, (size_t)(chunk * h->nb)));
  int rc = 0;
  const gi::MatrixDesc d = h->desc();
  for (int64_t c0 = 0; c0 < count && rc == 0; c0 += chunk) {
    const int64_t cnt = std::min(chunk, count - c0);
    memcpy(pinned, data + c0 * h->nb, (size_t)(cnt * h->nb));
    if (cudaMemcpyAsync(h->s_a.mem->ptr, pinned, (size_t)(cnt * h->nb), cudaMemcpyHostToDevice,
                        h->stream) != cudaSuccess) {
      gi_set_error("H2D copy of the BED buffer failed");
      rc = -1;
      break;
    }
    rc = gi::launch_upload_tiles(d, static_cast<uint8_t*>(h->x->ptr), h->s_a.as<uint8_t>(),
                                 j0 + c0, cnt, h->stream);
    if (rc == 0 && cudaStreamSynchronize(h->stream) != cudaSuccess) {
      gi_set_error("BED upload failed");
      rc = -1;
    }
  }
  cudaFreeHost(pinned);
  return rc;
}

int gi_matrix_finalize(gi_matrix* h) {
  CHECK_ARG(h != nullptr, "NULL handle");
  std::lock_guard<std::mutex> lock(h->mu);
  DeviceGuard g(h->device);
  return finish_stats(h);
}

int gi_matrix_from_bed(const uint8_t* data, int64_t n, int64_t p, int device, gi_matrix** out) {
  gi_matrix* h = nullptr;
  TRY(gi_matrix_create(n, p, device, &h));
  std::unique_ptr<gi_matrix> guard(h);
  TRY(gi_matrix_upload_bed(h, 0, p, data));
  TRY(gi_matrix_finalize(h));
  *out = guard.release();
  return 0;
}

int gi_matrix_synth(uint64_t seed, int64_t n, int64_t p, int64_t j_base, double maf_lo,
                    double maf_hi, double missing, int device, gi_matrix** out) {
  std::unique_ptr<gi_matrix> h;
  TRY(matrix_shell(n, p, device, out, h));
  DeviceGuard g(device);
  TRY(gi::launch_synth(h->desc(), static_cast<uint8_t*>(h->x->ptr), seed, j_base, maf_lo, maf_hi,
                       missing, h->stream));
  TRY(finish_stats(h.get()));
  *out = h.release();
  return 0;
}

int gi_matrix_with_stats(const gi_matrix* src, const double* u, const double* v, gi_matrix** out) {
  CHECK_ARG(src && u && v && out, "NULL argument");
  std::unique_ptr<gi_matrix> h(new gi_matrix());
  h->device = src->device;
  h->sms = src->sms;
  h->n = src->n;
  h->p = src->p;
  h->nb = src->nb;
  h->T = src->T;
  h->G = src->G;
  h->x = src->x;
  h->x3 = src->x3;
  h->T3 = src->T3;
  h->mlist = src->mlist;
  h->mofs = src->mofs;
  h->mtotal = src->mtotal;
  h->miss_cnt = src->miss_cnt;
  h->gmiss = src->gmiss;
  h->s1cnt = src->s1cnt;
  DeviceGuard g(h->device);
  GI_CUDA_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  TRY(alloc(h->u, sizeof(double) * h->p, h->device, false));
  TRY(alloc(h->v, sizeof(double) * h->p, h->device, false));
  GI_CUDA_TRY(cudaMemcpy(h->u->ptr, u, sizeof(double) * h->p, cudaMemcpyHostToDevice));
  GI_CUDA_TRY(cudaMemcpy(h->v->ptr, v, sizeof(double) * h->p, cudaMemcpyHostToDevice));
  *out = h.release();
  return 0;
}

int gi_matrix_subset_rows(const gi_matrix* src, const int64_t* rows, int64_t m, gi_matrix** out) {
  CHECK_ARG(src != nullptr, "NULL handle");
  for (int64_t i = 0; i < m; ++i)
    CHECK_ARG(rows[i] >= 0 && rows[i] < src->n, "row index out of range");
  std::unique_ptr<gi_matrix> h;
  // the gather kernel writes every word of every block (padding codes as 0)
  TRY(matrix_shell(m, src->p, src->device, out, h, m == 0 || src->p == 0));
  DeviceGuard g(src->device);
  if (m > 0 && src->p > 0) {
    std::shared_ptr<DevMem> drows;
    TRY(alloc(drows, sizeof(int64_t) * m, src->device, false));
    GI_CUDA_TRY(cudaMemcpy(drows->ptr, rows, sizeof(int64_t) * m, cudaMemcpyHostToDevice));
    TRY(gi::launch_subset_rows(src->desc(), h->desc(), static_cast<uint8_t*>(h->x->ptr),
                               static_cast<const int64_t*>(drows->ptr), h->stream));
    GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  TRY(finish_stats(h.get()));
  *out = h.release();
  return 0;
}

int gi_matrix_free(gi_matrix* h) {
  if (h) {
    DeviceGuard g(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    delete h;
  }
  return 0;
}

int gi_matrix_xtr_format(gi_matrix* h, int set, int* base3) {
  CHECK_ARG(h != nullptr, "NULL handle");
  CHECK_ARG(set >= -1 && set <= 1, "set must be -1 (query), 0 or 1");
  if (set >= 0) {
    std::lock_guard<std::mutex> lock(h->mu);
    DeviceGuard g(h->device);
    TRY(set_base3(h, set));
  }
  if (base3) *base3 = h->x3 ? (h->mlist ? 2 : 1) : 0;
  return 0;
}

int gi_matrix_shape(const gi_matrix* h, int64_t* n, int64_t* p, int* device) {
  CHECK_ARG(h != nullptr, "NULL handle");
  if (n) *n = h->n;
  if (p) *p = h->p;
  if (device) *device = h->device;
  return 0;
}

int gi_matrix_stats(const gi_matrix* h, double* u, double* v) {
  CHECK_ARG(h != nullptr, "NULL handle");
  DeviceGuard g(h->device);
  if (h->p == 0) return 0;
  if (u) GI_CUDA_TRY(cudaMemcpy(u, h->u->ptr, sizeof(double) * h->p, cudaMemcpyDeviceToHost));
  if (v) GI_CUDA_TRY(cudaMemcpy(v, h->v->ptr, sizeof(double) * h->p, cudaMemcpyDeviceToHost));
  return 0;
}

int gi_matrix_read_bed(const gi_matrix* hc, int64_t j0, int64_t count, uint8_t* out) {
  gi_matrix* h = const_cast<gi_matrix*>(hc);
  CHECK_ARG(h != nullptr, "NULL handle");
  CHECK_ARG(j0 >= 0 && count >= 0 && j0 + count <= h->p, "SNP range out of bounds");
  if (count == 0 || h->nb == 0) return 0;
  std::lock_guard<std::mutex> lock(h->mu);
  DeviceGuard g(h->device);
  const int64_t chunk = std::max<int64_t>(1, (int64_t)(256ll << 20) / h->nb);
  TRY(h->s_a.ensure((size_t)(std::min(chunk, count) * h->nb), h->device));
  for (int64_t c0 = 0; c0 < count; c0 += chunk) {
    const int64_t cnt = std::min(chunk, count - c0);
    TRY(gi::launch_download_tiles(h->desc(), h->s_a.as<uint8_t>(), j0 + c0, cnt, h->stream));
    GI_CUDA_TRY(cudaMemcpyAsync(out + c0 * h->nb, h->s_a.mem->ptr, (size_t)(cnt * h->nb),
                                cudaMemcpyDeviceToHost, h->stream));
    GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  return 0;
}

int gi_matrix_missing_counts(const gi_matrix* h, int32_t* out) {
  CHECK_ARG(h && out, "NULL argument");
  DeviceGuard g(h->device);
  if (h->p) GI_CUDA_TRY(cudaMemcpy(out, h->miss_cnt->ptr, sizeof(int32_t) * h->p,
                                   cudaMemcpyDeviceToHost));
  return 0;
}

int gi_matrix_device_stats(const gi_matrix* h, const double** d_u, const double** d_v) {
  CHECK_ARG(h != nullptr, "NULL handle");
  if (d_u) *d_u = h->du();
  if (d_v) *d_v = h->dv();
  return 0;
}

int64_t gi_padded_samples(const gi_matrix* h) { return h ? h->T * GI_TILE_SAMPLES : 0; }

static void build_rowmask(const gi_matrix* h, const uint8_t* keep, std::vector<uint32_t>& mask) {
  mask.assign((size_t)(h->T * GI_TILE_WORDS), 0u);
  for (int64_t i = 0; i < h->n; ++i)
    if (keep[i]) mask[(size_t)(i >> 4)] |= 1u << (2 * (i & 15));
}

int gi_matrix_masked_stats(const gi_matrix* hc, const uint8_t* keep, double* u, double* v) {
  gi_matrix* h = const_cast<gi_matrix*>(hc);
  CHECK_ARG(h && keep && u && v, "NULL argument");
  if (h->p == 0) return 0;
  std::vector<uint32_t> mask;
  build_rowmask(h, keep, mask);
  std::lock_guard<std::mutex> lock(h->mu);
  DeviceGuard g(h->device);
  TRY(h->s_a.ensure(mask.size() * 4, h->device));
  TRY(h->s_b.ensure(sizeof(double) * 2 * h->p, h->device));
  GI_CUDA_TRY(cudaMemcpyAsync(h->s_a.mem->ptr, mask.data(), mask.size() * 4,
                              cudaMemcpyHostToDevice, h->stream));
  double* du = h->s_b.as<double>();
  TRY(gi::launch_stats(h->desc(), h->s_a.as<uint32_t>(), du, du + h->p, nullptr, nullptr,
                       h->stream));
  GI_CUDA_TRY(cudaMemcpyAsync(u, du, sizeof(double) * h->p, cudaMemcpyDeviceToHost, h->stream));
  GI_CUDA_TRY(cudaMemcpyAsync(v, du + h->p, sizeof(double) * h->p, cudaMemcpyDeviceToHost,
                              h->stream));
  GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

// A copy of src (same tiles) standardised with the statistics of the rows
// with keep != 0, computed on the device -- subset_rows(rows).u / .v without
// the host round trip of gi_matrix_masked_stats + gi_matrix_with_stats (CV
// folds in train mode, model_select.py:87-93).
int gi_matrix_with_masked_stats(const gi_matrix* srcc, const uint8_t* keep, gi_matrix** out) {
  gi_matrix* src = const_cast<gi_matrix*>(srcc);
  CHECK_ARG(src && keep && out, "NULL argument");
  std::vector<uint32_t> mask;
  build_rowmask(src, keep, mask);
  std::unique_ptr<gi_matrix> h(new gi_matrix());
  h->device = src->device;
  h->sms = src->sms;
  h->n = src->n;
  h->p = src->p;
  h->nb = src->nb;
  h->T = src->T;
  h->G = src->G;
  h->x = src->x;
  h->x3 = src->x3;
  h->T3 = src->T3;
  h->mlist = src->mlist;
  h->mofs = src->mofs;
  h->mtotal = src->mtotal;
  h->miss_cnt = src->miss_cnt;
  h->gmiss = src->gmiss;
  h->s1cnt = src->s1cnt;
  h->any_missing = src->any_missing;
  DeviceGuard g(h->device);
  GI_CUDA_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  TRY(alloc(h->u, sizeof(double) * std::max<int64_t>(h->p, 1), h->device, true));
  TRY(alloc(h->v, sizeof(double) * std::max<int64_t>(h->p, 1), h->device, true));
  h->fold_keep.resize((size_t)h->n);
  for (int64_t i = 0; i < h->n; ++i) h->fold_keep[(size_t)i] = keep[i] != 0;
  if (h->p > 0) {
    TRY(alloc(h->fold_s1cnt, sizeof(int32_t) * 2 * h->p, h->device, false));
    TRY(h->s_a.ensure(mask.size() * 4, h->device));
    GI_CUDA_TRY(cudaMemcpyAsync(h->s_a.mem->ptr, mask.data(), mask.size() * 4,
                                cudaMemcpyHostToDevice, h->stream));
    TRY(gi::launch_stats(h->desc(), h->s_a.as<uint32_t>(), h->du(), h->dv(), nullptr,
                         static_cast<int32_t*>(h->fold_s1cnt->ptr), h->stream));
    GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  *out = h.release();
  return 0;
}

// ------------------------------------------------------- host-buffer operators
// One aty_genetic sweep on h's stream (caller holds h->mu and the device):
// r, out on the host; u, v device pointers (the handle's or caller stats).
static int aty_enqueue(gi_matrix* h, const double* r, double sum_r, const double* du,
                       const double* dv, double* out, int mode) {
  const int64_t npad = h->T * GI_TILE_SAMPLES;
  // scratch layout: s_a = r (fp64 padded) | rt (fp32 padded); s_b = out; s_c = scalars/partials
  TRY(h->s_a.ensure(sizeof(double) * npad + sizeof(float) * npad + 64, h->device));
  TRY(h->s_b.ensure(sizeof(double) * h->p, h->device));
  TRY(h->s_c.ensure(sizeof(double) * (16 + 8 * 296) + 64, h->device));
  double* dr = h->s_a.as<double>();
  float* drt = reinterpret_cast<float*>(dr + npad);
  double* scal = h->s_c.as<double>();
  double* partials = scal + 16;
  unsigned int* ticket = reinterpret_cast<unsigned int*>(partials + 8 * 296);
  GI_CUDA_TRY(cudaMemsetAsync(dr, 0, sizeof(double) * npad, h->stream));
  GI_CUDA_TRY(cudaMemcpyAsync(dr, r, sizeof(double) * h->n, cudaMemcpyHostToDevice, h->stream));
  if (mode == 0) {
    GI_CUDA_TRY(cudaMemcpyAsync(scal, &sum_r, sizeof(double), cudaMemcpyHostToDevice, h->stream));
    TRY(gi::launch_aty_exact(h->desc(), dr, du, dv, scal, 1.0, h->s_b.as<double>(), h->stream));
  } else {
    GI_CUDA_TRY(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), h->stream));
    // mean over the n real samples, then centred fp32 copy and its sum
    TRY(gi::launch_residual(h->n, dr, nullptr, nullptr, 0, nullptr, nullptr, (double)h->n,
                            dr, scal, partials, ticket, h->stream));
    TRY(gi::launch_center(h->n, npad, dr, nullptr, scal, drt, partials, ticket, h->stream));
    TRY(gi::launch_aty_fast(h->desc(), static_cast<const uint8_t*>(h->gmiss->ptr), drt, du, dv,
                            static_cast<const int32_t*>(h->s1cnt->ptr), scal, 1.0,
                            h->s_b.as<double>(), h->sms, h->stream));
  }
  GI_CUDA_TRY(cudaMemcpyAsync(out, h->s_b.mem->ptr, sizeof(double) * h->p,
                              cudaMemcpyDeviceToHost, h->stream));
  return 0;
}

// Whether the matrix holds any missing genotype (cached on the handle).
static int has_missing(gi_matrix* h, bool& out) {
  if (h->any_missing < 0) {
    std::vector<uint8_t> flags((size_t)h->G);
    if (h->G)
      GI_CUDA_TRY(cudaMemcpy(flags.data(), h->gmiss->ptr, (size_t)h->G, cudaMemcpyDeviceToHost));
    int any = 0;
    for (uint8_t f : flags) any |= f ? 1 : 0;
    h->any_missing = any;
  }
  out = h->any_missing != 0;
  return 0;
}

// Tensor-core X^T R (xtr_mma.cu) for B residuals (rows of R, host), optional
// per-RHS stats U, V (rows, host): batches of up to 32 residuals (16 when the
// matrix has missing genotypes) per sweep of the tiles.
static int aty_mma_enqueue(gi_matrix* h, const double* R, const double* U, const double* V,
                           int64_t B, double* G) {
  bool miss = false;
  TRY(has_missing(h, miss));
  const int64_t maxb = gi::xtr_mma_max_rhs(miss), n = h->n, p = h->p;
  const gi::MatrixDesc d = h->desc();
  const int64_t bsz = std::min<int64_t>(maxb, B);
  const int64_t qbytes = gi::xtr_mma_qimg_bytes(d, (int)bsz);
  const int64_t pcap = 4 * 148 * bsz;
  // s_e: R (bsz x n) | qscal (2 bsz) | qsum (bsz) | partials | tickets | descriptors | image
  const size_t off_desc = ((sizeof(double) * (size_t)(bsz * n + 3 * bsz + pcap) +
                            sizeof(unsigned int) * (size_t)bsz) + 255) & ~(size_t)255;
  const size_t off_q = (off_desc + sizeof(gi::XtrRhs) * (size_t)bsz + 1023) & ~(size_t)1023;
  TRY(h->s_e.ensure(off_q + (size_t)qbytes, h->device));
  TRY(h->s_b.ensure(sizeof(double) * (size_t)(bsz * p), h->device));
  double* dR = h->s_e.as<double>();
  double* qscal = dR + bsz * n;
  long long* qsum = reinterpret_cast<long long*>(qscal + 2 * bsz);
  double* partials = reinterpret_cast<double*>(qsum + bsz);
  unsigned int* tickets = reinterpret_cast<unsigned int*>(partials + pcap);
  gi::XtrRhs* ddesc = reinterpret_cast<gi::XtrRhs*>(h->s_e.as<char>() + off_desc);
  int8_t* qimg = reinterpret_cast<int8_t*>(h->s_e.as<char>() + off_q);
  double *du = h->du(), *dv = h->dv();
  if (U) {
    TRY(h->s_d.ensure(sizeof(double) * 2 * (size_t)(bsz * p), h->device));
    du = h->s_d.as<double>();
    dv = du + bsz * p;
  }
  std::vector<gi::XtrRhs> desc((size_t)bsz);
  for (int64_t b = 0; b < bsz; ++b) {
    gi::XtrRhs& x = desc[(size_t)b];
    x.r = dR + b * n;
    x.keep = nullptr;
    x.u = U ? du + b * p : du;
    x.v = U ? dv + b * p : dv;
    x.s1cnt = static_cast<const int32_t*>(h->s1cnt->ptr);
    x.out = h->s_b.as<double>() + b * p;
    x.gmax = nullptr;
  }
  GI_CUDA_TRY(cudaMemcpyAsync(ddesc, desc.data(), sizeof(gi::XtrRhs) * desc.size(),
                              cudaMemcpyHostToDevice, h->stream));
  GI_CUDA_TRY(cudaMemsetAsync(tickets, 0, sizeof(unsigned int) * bsz, h->stream));
  for (int64_t b0 = 0; b0 < B; b0 += bsz) {
    const int64_t nb = std::min<int64_t>(bsz, B - b0);
    GI_CUDA_TRY(cudaMemcpyAsync(dR, R + b0 * n, sizeof(double) * nb * n, cudaMemcpyHostToDevice,
                                h->stream));
    if (U) {
      GI_CUDA_TRY(cudaMemcpyAsync(du, U + b0 * p, sizeof(double) * nb * p,
                                  cudaMemcpyHostToDevice, h->stream));
      GI_CUDA_TRY(cudaMemcpyAsync(dv, V + b0 * p, sizeof(double) * nb * p,
                                  cudaMemcpyHostToDevice, h->stream));
    }
    TRY(gi::launch_xtr_quant(n, h->T, (int)nb, ddesc, qscal, qsum, qimg, partials, pcap, tickets,
                             h->stream));
    TRY(gi::launch_xtr_mma(d, static_cast<const uint8_t*>(h->gmiss->ptr), miss, (int)nb, qimg,
                           qscal, qsum, ddesc, 1.0, h->sms, h->stream));
    GI_CUDA_TRY(cudaMemcpyAsync(G + b0 * p, h->s_b.mem->ptr, sizeof(double) * nb * p,
                                cudaMemcpyDeviceToHost, h->stream));
  }
  return 0;
}

int gi_aty(gi_matrix* h, const double* r, double sum_r, double* out, int mode) {
  CHECK_ARG(h && r && out, "NULL argument");
  if (h->p == 0) return 0;
  std::lock_guard<std::mutex> lock(h->mu);
  DeviceGuard g(h->device);
  if (mode == 2)
    TRY(aty_mma_enqueue(h, r, nullptr, nullptr, 1, out));
  else
    TRY(aty_enqueue(h, r, sum_r, h->du(), h->dv(), out, mode));
  GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int gi_aty_batched(gi_matrix* h, const double* R, const double* sum_R, const double* U,
                   const double* V, int64_t B, double* G, int mode) {
  CHECK_ARG(h && (B == 0 || (R && G)), "NULL argument");
  CHECK_ARG(B >= 0, "negative batch size");
  CHECK_ARG((U == nullptr) == (V == nullptr), "U and V must both be given or both be NULL");
  CHECK_ARG(mode != 0 || B == 0 || sum_R != nullptr, "mode 0 needs the residual sums");
  if (h->p == 0 || B == 0) return 0;
  std::lock_guard<std::mutex> lock(h->mu);
  DeviceGuard g(h->device);
  const int64_t p = h->p;
  if (mode == 2) {
    TRY(aty_mma_enqueue(h, R, U, V, B, G));
    GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
    return 0;
  }
  double *du = h->du(), *dv = h->dv();
  if (U) {
    TRY(h->s_d.ensure(sizeof(double) * 2 * p, h->device));
    du = h->s_d.as<double>();
    dv = du + p;
  }
  for (int64_t b = 0; b < B; ++b) {
    if (U) {  // stream-ordered: the previous sweep has read the previous stats
      GI_CUDA_TRY(cudaMemcpyAsync(du, U + b * p, sizeof(double) * p, cudaMemcpyHostToDevice,
                                  h->stream));
      GI_CUDA_TRY(cudaMemcpyAsync(dv, V + b * p, sizeof(double) * p, cudaMemcpyHostToDevice,
                                  h->stream));
    }
    TRY(aty_enqueue(h, R + b * h->n, sum_R ? sum_R[b] : 0.0, du, dv, G + b * p, mode));
  }
  GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int gi_ax_cols(gi_matrix* h, const int64_t* idx, const double* w, int64_t k, double* out) {
  CHECK_ARG(h && out, "NULL argument");
  for (int64_t t = 0; t < k; ++t)
    CHECK_ARG(idx[t] >= 0 && idx[t] < h->p, "variant index out of range");
  if (h->n == 0) return 0;
  std::lock_guard<std::mutex> lock(h->mu);
  DeviceGuard g(h->device);
  TRY(h->s_a.ensure(sizeof(int64_t) * (k + 1) + sizeof(double) * (k + 1), h->device));
  TRY(h->s_b.ensure(sizeof(double) * h->n, h->device));
  int64_t* didx = h->s_a.as<int64_t>();
  double* dw = reinterpret_cast<double*>(didx + k + 1);
  if (k > 0) {
    GI_CUDA_TRY(cudaMemcpyAsync(didx, idx, sizeof(int64_t) * k, cudaMemcpyHostToDevice, h->stream));
    GI_CUDA_TRY(cudaMemcpyAsync(dw, w, sizeof(double) * k, cudaMemcpyHostToDevice, h->stream));
  }
  TRY(gi::launch_ax(h->desc(), h->du(), h->dv(), didx, dw, k, h->s_b.as<double>(), 0, h->stream));
  GI_CUDA_TRY(cudaMemcpyAsync(out, h->s_b.mem->ptr, sizeof(double) * h->n,
                              cudaMemcpyDeviceToHost, h->stream));
  GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

int gi_decompress(gi_matrix* h, const int64_t* idx, int64_t k, double* out_t) {
  CHECK_ARG(h && out_t, "NULL argument");
  for (int64_t t = 0; t < k; ++t)
    CHECK_ARG(idx[t] >= 0 && idx[t] < h->p, "variant index out of range");
  if (k == 0 || h->n == 0) return 0;
  std::lock_guard<std::mutex> lock(h->mu);
  DeviceGuard g(h->device);
  TRY(h->s_a.ensure(sizeof(int64_t) * k, h->device));
  TRY(h->s_b.ensure(sizeof(double) * h->n * k, h->device));
  GI_CUDA_TRY(cudaMemcpyAsync(h->s_a.mem->ptr, idx, sizeof(int64_t) * k, cudaMemcpyHostToDevice,
                              h->stream));
  TRY(gi::launch_decompress(h->desc(), h->du(), h->dv(), h->s_a.as<int64_t>(), k,
                            h->s_b.as<double>(), h->stream));
  GI_CUDA_TRY(cudaMemcpyAsync(out_t, h->s_b.mem->ptr, sizeof(double) * h->n * k,
                              cudaMemcpyDeviceToHost, h->stream));
  GI_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

// ------------------------------------------------------------ device primitives
#define STREAM(s) static_cast<cudaStream_t>(s)

int gi_dev_ax(gi_matrix* h, const double* u, const double* v, const int64_t* d_idx,
              const double* d_w, int64_t k, double* d_out, int accumulate, void* stream) {
  CHECK_ARG(h && d_out, "NULL argument");
  return gi::launch_ax(h->desc(), u ? u : h->du(), v ? v : h->dv(), d_idx, d_w, k, d_out,
                       accumulate, STREAM(stream));
}

int gi_dev_aty_fast(gi_matrix* h, const double* u, const double* v, const int32_t* d_s1cnt,
                    const float* d_rt, const double* d_scal, double scale, double* d_out,
                    void* stream) {
  CHECK_ARG(h && d_rt && d_scal && d_out, "NULL argument");
  return gi::launch_aty_fast(h->desc(), static_cast<const uint8_t*>(h->gmiss->ptr), d_rt,
                             u ? u : h->du(), v ? v : h->dv(),
                             d_s1cnt ? d_s1cnt : static_cast<const int32_t*>(h->s1cnt->ptr),
                             d_scal, scale, d_out, h->sms, STREAM(stream));
}

int gi_dev_aty_exact(gi_matrix* h, const double* u, const double* v, const double* d_rpad,
                     const double* d_sum_r, double scale, double* d_out, void* stream) {
  CHECK_ARG(h && d_rpad && d_sum_r && d_out, "NULL argument");
  return gi::launch_aty_exact(h->desc(), d_rpad, u ? u : h->du(), v ? v : h->dv(), d_sum_r, scale,
                              d_out, STREAM(stream));
}

int gi_dev_stats(gi_matrix* h, const uint32_t* d_rowmask, double* d_u, double* d_v,
                 int32_t* d_s1cnt, void* stream) {
  CHECK_ARG(h && d_u && d_v, "NULL argument");
  return gi::launch_stats(h->desc(), d_rowmask, d_u, d_v, nullptr, d_s1cnt, STREAM(stream));
}

int64_t gi_red_partials(void) { return 8 * 296; }

int gi_dev_residual(int64_t n, const double* d_y, const double* d_fit, const double* d_C,
                    int64_t c, const double* d_bcov, const uint8_t* d_keep, double n_eff,
                    double* d_r, double* d_scal, double* d_partials, uint32_t* d_ticket,
                    void* stream) {
  return gi::launch_residual(n, d_y, d_fit, d_C, (int)c, d_bcov, d_keep, n_eff, d_r, d_scal,
                             d_partials, d_ticket, STREAM(stream));
}

int gi_dev_center(int64_t n, int64_t n_pad, const double* d_r, const uint8_t* d_keep,
                  double* d_scal, float* d_rt, double* d_partials, uint32_t* d_ticket,
                  void* stream) {
  return gi::launch_center(n, n_pad, d_r, d_keep, d_scal, d_rt, d_partials, d_ticket,
                           STREAM(stream));
}

int gi_dev_covgrad(int64_t n, const double* d_C, int64_t c, const double* d_r, double* d_gcov,
                   double* d_partials, uint32_t* d_ticket, void* stream) {
  return gi::launch_covgrad(n, d_C, (int)c, d_r, d_gcov, d_partials, d_ticket, STREAM(stream));
}

int gi_dev_maxabs(int64_t m, const double* d_x, double* d_scal, int slot, double* d_partials,
                  uint32_t* d_ticket, void* stream) {
  return gi::launch_maxabs(m, d_x, d_scal, slot, d_partials, d_ticket, STREAM(stream));
}

int gi_dev_sumsq(int64_t m, const double* d_x, double* d_scal, int slot, double* d_partials,
                 uint32_t* d_ticket, void* stream) {
  return gi::launch_sumsq(m, d_x, d_scal, slot, d_partials, d_ticket, STREAM(stream));
}

int gi_dev_add_cov(int64_t n, const double* d_C, int64_t c, const double* d_w, double* d_x,
                   void* stream) {
  return gi::launch_add_cov(n, d_C, (int)c, d_w, d_x, STREAM(stream));
}

int64_t gi_topk_slots(int64_t p, int64_t k) { return gi::topk_blocks(p) * (k > 0 ? k : 1); }

int gi_dev_topk(int64_t p, int64_t k, int mode, const double* d_beta, const double* d_g,
                double mu, int64_t idx_base, uint64_t* d_ckey, int64_t* d_cidx, double* d_cval,
                int64_t* d_out_idx, double* d_out_val, uint64_t* d_out_key, int64_t* d_count,
                void* stream) {
  return gi::launch_topk(p, k, mode, d_beta, d_g, mu, idx_base, d_ckey, d_cidx, d_cval,
                         d_out_idx, d_out_val, d_out_key, d_count, STREAM(stream));
}

int gi_dev_scatter(int64_t k, const int64_t* d_idx, const double* d_val, double* d_beta,
                   void* stream) {
  return gi::launch_scatter(k, d_idx, d_val, d_beta, STREAM(stream));
}

int gi_dev_gather(int64_t k, const int64_t* d_idx, const double* d_src, double* d_dst,
                  void* stream) {
  return gi::launch_gather(k, d_idx, d_src, d_dst, STREAM(stream));
}

}  // extern "C"
