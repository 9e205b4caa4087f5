// Native single-GPU IHT loop: gi_fit (include/genoiht_cuda.h).
//
// The control flow is the reference solver's, step for step:
//   fit            iht.py:326-354     initial state, loop, trace, reasons
//   _refresh_state iht.py:183-191     r = y - X_S b - C b_cov, loss, g = -X^T r
//   iht_step       iht.py:253-323     fixed points, restriction, mu, backtracking
//   _step_restriction / _normalized_step iht.py:218-244
// and the same as paper_1608_01398_b200/iht.py (which drives the multi-GPU
// case through the same kernels).  Every O(n), O(p) and O(n p) operation is a
// kernel on the matrix's device; the host keeps the O(k) support bookkeeping
// and recomputes the candidate step with the reference's float operations.
// One host sync per phase (refresh, image, top-k).  Each phase's host inputs
// (sparse vectors, covariate weights) are staged in a pinned arena and reach
// the device in ONE copy; its results come back through mapped host memory,
// written by the phase's last kernel -- no per-array copy-engine transfers,
// which at small n cost more than the kernels themselves.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <limits>
#include <map>
#include <atomic>
#include <mutex>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../../include/genoiht_cuda.h"
#include "batch.cuh"
#include "comm.cuh"
#include "handle.cuh"

namespace {

struct FitWs {
  int device = 0;
  int64_t n = 0, p = 0, npad = 0, c = 0, kcap = 0, slots = 0;
  cudaStream_t stream = nullptr;
  // device
  double *y = nullptr, *C = nullptr, *r = nullptr, *fitb = nullptr, *img = nullptr;
  double *g = nullptr, *beta = nullptr, *cvec = nullptr, *scal = nullptr, *partials = nullptr;
  double *u = nullptr, *v = nullptr;
  float* rt = nullptr;
  uint8_t* keep = nullptr;
  uint8_t* keep_test = nullptr;  // held-out rows scored at the end (keep == 2 on input)
  int32_t* s1cnt = nullptr;
  uint32_t *ticket = nullptr, *rowmask = nullptr;
  uint64_t* ckey = nullptr;
  double* sg_part = nullptr;       // support-gradient slice partials
  uint32_t* sg_ticket = nullptr;   // per support column
  double* aty_part = nullptr;      // X^T r tile-slice partial sums (small p only)
  uint32_t* aty_ticket = nullptr;  // X^T r per-chunk arrival counters
  int64_t* cidx = nullptr;
  double* cval = nullptr;

  // uploads: pinned host arena mirrored byte for byte by a device arena
  char* hin = nullptr;
  char* din = nullptr;
  size_t in_cap = 0, in_off = 0, in_flushed = 0;
  // results: mapped pinned host memory written by kernels (device alias dmap)
  double* hmap = nullptr;
  double* dmap = nullptr;
  int64_t oR = 0, oT = 0, oM = 0, oS = 0, oG = 0;  // refresh, top-k, den/mu, image, shards
  // sharded loop: exchange buffers on the device (grown on demand)
  double* shard_buf = nullptr;
  int64_t shard_cap = 0;
  std::vector<void*> dev_allocs;
  bool primed = false, masked = false;
  uint64_t primed_uid = 0;  // handle whose inputs are resident (y == NULL calls)
  double n_eff = 0.0;

  ~FitWs() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (void* ptr : dev_allocs) cudaFreeAsync(ptr, stream);
    if (shard_buf) cudaFreeAsync(shard_buf, stream);
    if (stream) cudaStreamSynchronize(stream);
    if (hin) cudaFreeHost(hin);
    if (hmap) cudaFreeHost(hmap);
    if (stream) cudaStreamDestroy(stream);
    cudaSetDevice(prev);
  }

  // stream-ordered pool allocations: no device-wide synchronisation, so a new
  // workspace does not stall fits already running on other streams
  template <typename T>
  int dalloc(T*& out, int64_t count) {
    void* ptr = nullptr;
    GI_CUDA_TRY(cudaMallocAsync(&ptr, sizeof(T) * (size_t)std::max<int64_t>(count, 1), stream));
    dev_allocs.push_back(ptr);
    out = static_cast<T*>(ptr);
    return 0;
  }
};

// Process-wide workspace pool per device.  Deliberately never destroyed: it
// would otherwise be torn down after the CUDA runtime at process exit.
struct FitPool {
  std::mutex mu;
  std::vector<std::shared_ptr<FitWs>> items;
};
// Enough for a lock-step group of concurrent fits (model_select._group_workers)
// plus the final fit: an eviction frees device memory, which synchronises the
// device under every other fit in flight.
constexpr size_t kPoolCap = 64;
// Workspace shapes are rounded up to whole multiples of this many support
// slots, so the fits of one path / CV (k = 1..20, say) share one shape.
constexpr int64_t kKcapQuantum = 32;

FitPool& fit_pool_for(int device) {
  static std::mutex mu;
  static std::map<int, FitPool*>* pools = new std::map<int, FitPool*>();
  std::lock_guard<std::mutex> lock(mu);
  FitPool*& pool = (*pools)[device];
  if (!pool) pool = new FitPool();
  return *pool;
}

int make_ws(gi_matrix* h, int64_t c, int64_t kcap, std::shared_ptr<FitWs>& out) {
  auto ws = std::make_shared<FitWs>();
  ws->device = h->device;
  ws->n = h->n;
  ws->p = h->p;
  ws->npad = h->T * GI_TILE_SAMPLES;
  ws->c = c;
  ws->kcap = kcap;
  ws->slots = gi::topk_blocks(std::max<int64_t>(h->p, 1)) * kcap;
  GI_CUDA_TRY(cudaStreamCreateWithFlags(&ws->stream, cudaStreamNonBlocking));
  const int64_t n = h->n, p = std::max<int64_t>(h->p, 1);
  TRY(ws->dalloc(ws->y, n));
  TRY(ws->dalloc(ws->C, n * std::max<int64_t>(c, 1)));
  // r is padded to whole tiles (zero tail) for the exact X^T r kernel
  TRY(ws->dalloc(ws->r, ws->npad));
  GI_CUDA_TRY(cudaMemsetAsync(ws->r, 0, sizeof(double) * ws->npad, ws->stream));
  TRY(ws->dalloc(ws->fitb, n));
  TRY(ws->dalloc(ws->img, n));
  TRY(ws->dalloc(ws->g, p));
  TRY(ws->dalloc(ws->beta, p));
  TRY(ws->dalloc(ws->cvec, 2 * std::max<int64_t>(c, 1)));
  TRY(ws->dalloc(ws->scal, 8));
  TRY(ws->dalloc(ws->partials, 16 * 296));
  TRY(ws->dalloc(ws->u, p));
  TRY(ws->dalloc(ws->v, p));
  TRY(ws->dalloc(ws->rt, ws->npad));
  TRY(ws->dalloc(ws->keep, n));
  TRY(ws->dalloc(ws->keep_test, n));
  TRY(ws->dalloc(ws->s1cnt, 2 * p));
  TRY(ws->dalloc(ws->ticket, 1));
  TRY(ws->dalloc(ws->rowmask, ws->npad / 16));
  TRY(ws->dalloc(ws->ckey, ws->slots));
  TRY(ws->dalloc(ws->cidx, ws->slots));
  TRY(ws->dalloc(ws->cval, ws->slots));
  TRY(ws->dalloc(ws->sg_part, gi::support_grad_part_doubles(kcap, h->T)));
  TRY(ws->dalloc(ws->sg_ticket, kcap));
  GI_CUDA_TRY(cudaMemsetAsync(ws->sg_ticket, 0, sizeof(uint32_t) * kcap, ws->stream));

  {
    const int64_t part = gi::aty_fast_part_doubles(h->desc(), h->sms);
    if (part > 0) {
      TRY(ws->dalloc(ws->aty_part, part));
      TRY(ws->dalloc(ws->aty_ticket, 2 * (int64_t)h->sms));
      GI_CUDA_TRY(cudaMemsetAsync(ws->aty_ticket, 0, sizeof(uint32_t) * 2 * h->sms, ws->stream));
    }
  }
  // between two syncs a phase stages at most ~3 sparse vectors of <= 2 kcap
  // entries plus one covariate vector; the arena is reset at every sync
  ws->in_cap = (size_t)(128 * kcap + 64) * sizeof(double);
  TRY(ws->dalloc(ws->din, (int64_t)ws->in_cap));
  GI_CUDA_TRY(cudaMemsetAsync(ws->ticket, 0, sizeof(uint32_t), ws->stream));
  GI_CUDA_TRY(cudaMallocHost(&ws->hin, ws->in_cap));
  ws->oR = 0;                          // scal[0..8) | g_cov (c) | g on the support (kcap)
  ws->oT = 8 + c + kcap;               // count | idx (kcap) | val (kcap) | key (kcap)
  ws->oM = ws->oT + 1 + 3 * kcap;      // den, mu
  ws->oS = ws->oM + 2;                 // ||X d||^2 of a backtracking check
  ws->oG = ws->oS + 2;                 // sharded: global max|g| | g on the support (kcap)
  GI_CUDA_TRY(cudaHostAlloc(&ws->hmap, sizeof(double) * (size_t)(ws->oG + 1 + kcap),
                            cudaHostAllocMapped));
  GI_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ws->dmap), ws->hmap, 0));
  out = ws;
  return 0;
}

struct Pair {
  int64_t idx;
  double val;
};

class NativeFit {
 public:
  NativeFit(gi_matrix* h, FitWs* ws, const gi_fit_config* cfg, bool masked, double n_eff,
            gi_comm* comm, int64_t j_base)
      : h_(h), ws_(ws), cfg_(*cfg), masked_(masked), n_eff_(n_eff), comm_(comm),
        j_base_(j_base) {
    // The exact fp64 X^T r kernel -- the reference's own operation order --
    // replaces the fast one where few samples per parameter can amplify the
    // fast kernel's ~6e-7 gradient error past the 1e-6 parity bound (a
    // randomised stress found one such case: 62 samples, 22 + 2 parameters):
    // n <= 8 (k + c + 1) with the matrix up to 256 MiB, and any matrix up to
    // 2 MiB, where the two kernels cost the same (both latency-bound).
    // GI_XTR_EXACT=0/1 forces the fast / exact kernel.
    const gi::MatrixDesc d = h->desc();
    const double bytes = (double)d.G * (double)d.T * GI_BLOCK_BYTES;
    const double params = (double)cfg->k + (double)ws->c + 1.0;
    exact_ = bytes <= 2.0 * 1048576.0 || (n_eff <= 8.0 * params && bytes <= 256.0 * 1048576.0);
    // sharded fits: the caller decides on the global shape (flags bits 1-2), so
    // ranks whose shards straddle a threshold still run the same kernel
    if (cfg->flags & 2) exact_ = (cfg->flags & 4) != 0;
    if (const char* e = getenv("GI_XTR_EXACT")) exact_ = atoi(e) != 0;
    if (const char* e = getenv("GI_SUPPORT_GRAD")) support_grad_ = atoi(e) != 0;
  }
  bool exact_ = false;
  bool support_grad_ = true;  // exact gradient on the support after a fast sweep

  // gi_fit_sharded always runs the exchange steps, also on a world of one
  // (which is how the NCCL backend is exercised on a single GPU)
  bool sharded() const { return comm_ != nullptr; }

  // entries of a global sparse vector owned by this shard, as local indices
  void local_part(const std::vector<int64_t>& idx, const std::vector<double>& w,
                  std::vector<int64_t>& li, std::vector<double>& lw) const {
    li.clear();
    lw.clear();
    const int64_t lo = j_base_, hi = j_base_ + ws_->p;
    for (size_t t = 0; t < idx.size(); ++t)
      if (idx[t] >= lo && idx[t] < hi) {
        li.push_back(idx[t] - lo);
        lw.push_back(w[t]);
      }
  }

  int launches = 0;
  int aty_launches = 0;
  double aty_ms = 0.0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  // Stage `count` items for the device: copied into the pinned arena now, sent
  // by the next flush(); the returned device pointer is valid until the next
  // sync().
  template <typename T>
  int stage(const T* src, int64_t count, const T*& dev) {
    const size_t bytes = sizeof(T) * (size_t)count;
    const size_t off = (ws_->in_off + 15) & ~(size_t)15;
    if (off + bytes > ws_->in_cap) {
      gi_set_error("internal: staging arena overflow");
      return -1;
    }
    if (bytes) memcpy(ws_->hin + off, src, bytes);
    ws_->in_off = off + bytes;
    dev = reinterpret_cast<const T*>(ws_->din + off);
    return 0;
  }
  int flush() {
    if (ws_->in_off > ws_->in_flushed) {
      GI_CUDA_TRY(cudaMemcpyAsync(ws_->din + ws_->in_flushed, ws_->hin + ws_->in_flushed,
                                  ws_->in_off - ws_->in_flushed, cudaMemcpyHostToDevice,
                                  ws_->stream));
      ws_->in_flushed = ws_->in_off;
    }
    return 0;
  }
  double sync_us = 0.0;
  int syncs = 0;
  // Lock-step groups run up to 32 fits on as many host threads; a fit waiting
  // on the group's sweep (the refresh, ~1 ms) sleeps on a blocking-sync event
  // so the waiting threads do not oversubscribe the host cores.  Every other
  // phase spins, as a single fit does: blocking on all of them cost 2-5x at
  // config 2 (wake-up latency per short phase).
  cudaEvent_t block_ev_ = nullptr;
  int sync(bool blocking = false) {
    const auto t0 = std::chrono::steady_clock::now();
    if (block_ev_ && blocking) {
      GI_CUDA_TRY(cudaEventRecord(block_ev_, ws_->stream));
      GI_CUDA_TRY(cudaEventSynchronize(block_ev_));
    } else {
      GI_CUDA_TRY(cudaStreamSynchronize(ws_->stream));
    }
    sync_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0)
                   .count();
    ++syncs;
    ws_->in_off = ws_->in_flushed = 0;  // every staged copy has landed
    return 0;
  }
  // beta entries to write before the next refresh (staged by scatter_beta)
  const int64_t* pend_idx_ = nullptr;
  const double* pend_w_ = nullptr;
  int64_t pend_k_ = 0;

  // _refresh_state: returns loss, max|g|, g_cov, g on the support
  int refresh(const std::vector<int64_t>& sup, const std::vector<double>& w,
              const std::vector<double>& bcov, double& loss, double& gmax,
              std::vector<double>& gcov, std::vector<double>& gsup, bool need_grad = true) {
    const gi::MatrixDesc d = h_->desc();
    cudaStream_t s = ws_->stream;
    const bool has_fit = !sup.empty();
    std::vector<int64_t> lsup;
    std::vector<double> lw;
    local_part(sup, w, lsup, lw);
    // one upload for the pending beta update, the support and b_cov
    const int64_t* d_sup = nullptr;
    const double *d_w = nullptr, *d_cov = nullptr;
    TRY(stage(lsup.data(), (int64_t)lsup.size(), d_sup));
    TRY(stage(lw.data(), (int64_t)lw.size(), d_w));
    TRY(stage(bcov.data(), ws_->c, d_cov));
    // sharded: where each global support entry lives on this shard (or -1)
    const int64_t kg = (int64_t)sup.size();
    const int64_t* d_gsel = nullptr;
    if (sharded()) {
      std::vector<int64_t> gsel((size_t)kg, -1);
      for (int64_t t = 0; t < kg; ++t)
        if (sup[t] >= j_base_ && sup[t] < j_base_ + ws_->p) gsel[t] = sup[t] - j_base_;
      TRY(stage(gsel.data(), kg, d_gsel));
    }
    TRY(flush());
    const uint8_t* keep = masked_ ? ws_->keep : nullptr;
    int fused = -2;
    if (!sharded()) {
      // X_S b, residual, loss, sum r, g_cov and the pending beta writes in one
      // kernel (the fitted values are never stored)
      fused = gi::launch_ax_residual(d, ws_->u, ws_->v, d_sup, d_w, (int64_t)lsup.size(), ws_->y,
                                     ws_->c ? ws_->C : nullptr, (int)ws_->c, d_cov, keep, n_eff_,
                                     ws_->r, ws_->scal, ws_->c ? ws_->cvec + ws_->c : nullptr,
                                     pend_k_, pend_idx_, pend_w_, ws_->beta, ws_->partials,
                                     ws_->ticket, s);
      if (fused != 0 && fused != -2) return -1;
      if (fused == 0) {
        pend_k_ = 0;
        ++launches;
      }
    }
    if (fused != 0) {
      if (has_fit) {
        TRY(gi::launch_ax(d, ws_->u, ws_->v, d_sup, d_w, (int64_t)lsup.size(), ws_->fitb, 0, s));
        ++launches;
        // X_S b summed over the shards (NCCL in place on this stream)
        if (sharded()) TRY(comm_->allreduce_device(ws_->fitb, ws_->n, 0, s));
      }
      // residual + loss + mean, the pending beta writes and g_cov = -C^T r in one
      // kernel (g_cov in a second one only beyond 8 covariates)
      TRY(gi::launch_refresh_residual(ws_->n, ws_->y, has_fit ? ws_->fitb : nullptr,
                                      ws_->c ? ws_->C : nullptr, (int)ws_->c, d_cov, keep,
                                      n_eff_, ws_->r, ws_->scal,
                                      ws_->c ? ws_->cvec + ws_->c : nullptr, pend_k_, pend_idx_,
                                      pend_w_, ws_->beta, ws_->partials, ws_->ticket, s));
      pend_k_ = 0;
      launches += ws_->c > 8 ? 1 + (ws_->c + 7) / 8 : 1;
    }
    if (!need_grad) {
      // the fit ends after this refresh (converged or max_iter): the reference
      // computes g here but FitResult never reads it (iht.py:326-355), so only
      // the residual's loss and g_cov come back
      gi::PubArgs pub;
      pub.add(ws_->scal, 8, ws_->oR);
      pub.add(ws_->cvec + ws_->c, ws_->c, ws_->oR + 8);
      TRY(gi::launch_publish(pub, ws_->dmap, s));
      ++launches;
      TRY(sync());
      const double* ho = ws_->hmap + ws_->oR;
      loss = ho[0];
      gmax = 0.0;
      gcov.assign(ho + 8, ho + 8 + ws_->c);
      gsup.clear();
      return 0;
    }
    if (batch_ && !exact_ && ws_->p) {
      // the group's tensor-core sweep computes g (and max|g|) for this fit
      // together with the other live fits' residuals (batch.cu, xtr_mma.cu)
      GI_CUDA_TRY(cudaMemsetAsync(ws_->scal + 3, 0, sizeof(double), s));  // max|g| slot
      gi::XtrRhs rq;
      rq.r = ws_->r;
      rq.keep = keep;
      rq.u = ws_->u;
      rq.v = ws_->v;
      rq.s1cnt = ws_->s1cnt;
      rq.out = ws_->g;
      rq.gmax = reinterpret_cast<unsigned long long*>(ws_->scal + 3);
      TRY(gi_batch_submit(batch_, rq, s, ready_, done_));
      ++aty_launches;
      gi::PubArgs pub;
      pub.add(ws_->scal, 8, ws_->oR);
      pub.add(ws_->cvec + ws_->c, ws_->c, ws_->oR + 8);
      TRY(gi::launch_publish(pub, ws_->dmap, s));
      ++launches;
      const int64_t ks = (int64_t)lsup.size();
      if (ks > 0) {
        TRY(gi::launch_support_grad(d, ws_->r, ws_->u, ws_->v, ws_->scal + 6, -1.0, d_sup, ks,
                                    ws_->g, ws_->dmap + ws_->oR + 8 + ws_->c, ws_->sg_part,
                                    ws_->sg_ticket, s));
        ++launches;
      }
      TRY(sync(true));  // waits on the group's sweep (~1 ms): sleep, don't spin
      const double* ho = ws_->hmap + ws_->oR;
      loss = ho[0];
      gmax = ho[3];
      gcov.assign(ho + 8, ho + 8 + ws_->c);
      gsup.assign(ho + 8 + ws_->c, ho + 8 + ws_->c + ks);
      return 0;
    }
    if (!exact_) {
      TRY(gi::launch_center(ws_->n, ws_->npad, ws_->r, keep, ws_->scal, ws_->rt, ws_->partials,
                            ws_->ticket, s));
      ++launches;
    }
    // scal, g_cov and g on the (local) support -> mapped host memory, written by
    // the last CTA of the X^T r kernel (a separate launch only when p == 0)
    const int64_t ks = (int64_t)lsup.size();
    gi::PubArgs pub;
    pub.add(ws_->scal, 8, ws_->oR);
    pub.add(ws_->cvec + ws_->c, ws_->c, ws_->oR + 8);
    // g on the support: published by the X^T r kernel itself when it is the
    // exact one; after a fast sweep it is recomputed exactly (and published)
    // by launch_support_grad below
    if (exact_) pub.add(ws_->g, ks, ws_->oR + 8 + ws_->c, d_sup);
    if (ws_->p && exact_) {
      // g = -X^T r in the reference's fp64 order (sum r from the residual
      // kernel), then max|g| and the publish
      if (ev0) GI_CUDA_TRY(cudaEventRecord(ev0, s));
      GI_CUDA_TRY(cudaMemsetAsync(ws_->scal + 3, 0, sizeof(double), s));  // max|g| slot
      TRY(gi::launch_aty_exact(d, ws_->r, ws_->u, ws_->v, ws_->scal + 6, -1.0, ws_->g, s,
                               ws_->scal + 3, &pub, ws_->ticket, ws_->dmap));
      if (ev1) GI_CUDA_TRY(cudaEventRecord(ev1, s));
      ++aty_launches;
      ++launches;
    } else if (ws_->p) {
      if (ev0) GI_CUDA_TRY(cudaEventRecord(ev0, s));
      TRY(gi::launch_aty_fast(d, static_cast<const uint8_t*>(h_->gmiss->ptr), ws_->rt, ws_->u,
                              ws_->v, ws_->s1cnt, ws_->scal, -1.0, ws_->g, h_->sms, s,
                              ws_->scal + 3,  // max|g| fused into the epilogue
                              &pub, ws_->ticket, ws_->dmap, ws_->aty_part, ws_->aty_ticket));
      if (ev1) GI_CUDA_TRY(cudaEventRecord(ev1, s));
      ++aty_launches;
      launches += d.mlist != nullptr ? 2 : 1;  // + missum_kernel over the missing list
      if (ks > 0 && support_grad_) {
        TRY(gi::launch_support_grad(d, ws_->r, ws_->u, ws_->v, ws_->scal + 6, -1.0, d_sup, ks,
                                    ws_->g, ws_->dmap + ws_->oR + 8 + ws_->c, ws_->sg_part,
                                    ws_->sg_ticket, s));
        ++launches;
      } else if (ks > 0) {  // GI_SUPPORT_GRAD=0 (diagnostics): the fast sweep's values
        gi::PubArgs pg;
        pg.add(ws_->g, ks, ws_->oR + 8 + ws_->c, d_sup);
        TRY(gi::launch_publish(pg, ws_->dmap, s));
        ++launches;
      }
    }
    if (!ws_->p) {
      if (exact_)  // the centring kernel, skipped here, clears the max|g| slot
        GI_CUDA_TRY(cudaMemsetAsync(ws_->scal + 3, 0, sizeof(double), s));
      TRY(gi::launch_publish(pub, ws_->dmap, s));
      ++launches;
    }
    if (sharded()) {
      // one all-gather of (max|g|, this shard's g on the global support, 0
      // elsewhere), folded in rank order on the device -- no host round trip
      const int world = comm_->world;
      TRY(ensure_shard_buf(world));
      double* mine = ws_->shard_buf;
      double* allm = mine + (1 + ws_->kcap);
      TRY(gi::launch_shard_gather(kg, d_gsel, ws_->g, ws_->scal + 3, mine, s));
      TRY(comm_->allgather_device(mine, 1 + kg, allm, s));
      TRY(gi::launch_shard_fold(world, kg, allm, ws_->dmap + ws_->oG, s));
      launches += 2;
    }
    TRY(sync());
    const double* ho = ws_->hmap + ws_->oR;
    if (ev0 && ws_->p) {
      float ms = 0.f;
      GI_CUDA_TRY(cudaEventElapsedTime(&ms, ev0, ev1));
      aty_ms += ms;
    }
    loss = ho[0];
    gmax = ws_->p ? ho[3] : 0.0;
    gcov.assign(ho + 8, ho + 8 + ws_->c);
    if (!sharded()) {
      gsup.assign(ho + 8 + ws_->c, ho + 8 + ws_->c + ks);
      return 0;
    }
    // each support entry lives on exactly one shard, so the rank-ordered sum of
    // the zero-padded rows is exact
    const double* hg = ws_->hmap + ws_->oG;
    gmax = hg[0];
    gsup.assign(hg + 1, hg + 1 + kg);
    return 0;
  }

  // exchange buffers of the sharded loop (see the layout in shard_ptrs)
  int ensure_shard_buf(int world) {
    const int64_t kc = ws_->kcap;
    const int64_t need = (1 + kc) * (1 + world) + 3 * kc * (1 + world) + 3 * kc * world + 1;
    if (need <= ws_->shard_cap) return 0;
    if (ws_->shard_buf) GI_CUDA_TRY(cudaFreeAsync(ws_->shard_buf, ws_->stream));
    ws_->shard_buf = nullptr;
    GI_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ws_->shard_buf),
                                sizeof(double) * (size_t)need, ws_->stream));
    ws_->shard_cap = need;
    return 0;
  }

  // || X_idx w + C wcov ||^2 over the view's rows -> scal[4] (enqueue only).
  // ratio_out >= 0: also scal[ratio_out] = ratio_num / scal[4]; host_out
  // (mapped) receives {scal[4], ratio}.
  int image_enqueue(const std::vector<int64_t>& idx, const std::vector<double>& w,
                    const std::vector<double>* wcov, int ratio_out, double ratio_num,
                    double* host_out) {
    const gi::MatrixDesc d = h_->desc();
    cudaStream_t s = ws_->stream;
    std::vector<int64_t> li;
    std::vector<double> lw;
    local_part(idx, w, li, lw);
    const int64_t* d_idx = nullptr;
    const double *d_w = nullptr, *d_cov = nullptr;
    TRY(stage(li.data(), (int64_t)li.size(), d_idx));
    TRY(stage(lw.data(), (int64_t)lw.size(), d_w));
    const bool cov = wcov && ws_->c;
    if (cov) TRY(stage(wcov->data(), ws_->c, d_cov));
    TRY(flush());
    if (!sharded()) {
      // X_idx w and its image norm in one launch (the n-vector is never stored)
      const int rc = gi::launch_ax_norm(d, ws_->u, ws_->v, d_idx, d_w, (int64_t)li.size(),
                                        cov ? ws_->C : nullptr, cov ? (int)ws_->c : 0, d_cov,
                                        masked_ ? ws_->keep : nullptr, ws_->scal, 4, ratio_out,
                                        ratio_num, host_out, ws_->partials, ws_->ticket, s);
      if (rc == 0) {
        ++launches;
        return 0;
      }
      if (rc != -2) return -1;  // -2: too many columns for one launch, use two kernels
    }
    TRY(gi::launch_ax(d, ws_->u, ws_->v, d_idx, d_w, (int64_t)li.size(), ws_->img, 0, s));
    ++launches;
    if (sharded()) TRY(comm_->allreduce_device(ws_->img, ws_->n, 0, s));
    // + C wcov, row mask and the squared norm in one pass
    TRY(gi::launch_image_sumsq(ws_->n, ws_->img, cov ? ws_->C : nullptr, cov ? (int)ws_->c : 0,
                               d_cov, masked_ ? ws_->keep : nullptr, ws_->scal, 4, ratio_out,
                               ratio_num, host_out, ws_->partials, ws_->ticket, s));
    ++launches;
    return 0;
  }

  int image_sumsq(const std::vector<int64_t>& idx, const std::vector<double>& w,
                  const std::vector<double>* wcov, double& out) {
    TRY(image_enqueue(idx, w, wcov, -1, 0.0, ws_->dmap + ws_->oS));
    TRY(sync());
    out = ws_->hmap[ws_->oS];
    return 0;
  }

  // k largest |g| (mode 0) or |beta - mu g| (mode 1), sorted by index
  // `den_mu` (optional): take mu from the device (scal[5], written by the
  // preceding image_enqueue) and return den and mu from the same sync
  int topk(int mode, double mu, int64_t k, std::vector<Pair>& out, double* den_mu = nullptr) {
    out.clear();
    cudaStream_t s = ws_->stream;
    const int64_t ke = std::min(k, ws_->kcap);
    if (sharded() && ke > 0) return topk_sharded(mode, mu, ke, out, den_mu);
    if (ws_->p == 0 || k <= 0) {
      if (den_mu) TRY(sync());
    } else {
      // the merge kernel writes the selection straight into mapped host memory
      double* dm = ws_->dmap + ws_->oT;
      const int64_t kc = ws_->kcap;
      TRY(gi::launch_topk(ws_->p, ke, mode, ws_->beta, ws_->g, mu, j_base_, ws_->ckey, ws_->cidx,
                          ws_->cval, reinterpret_cast<int64_t*>(dm + 1), dm + 1 + kc,
                          reinterpret_cast<uint64_t*>(dm + 1 + 2 * kc),
                          reinterpret_cast<int64_t*>(dm), s, den_mu ? ws_->scal + 5 : nullptr,
                          ws_->ticket));
      launches += 1;
      TRY(sync());
      const double* ho = ws_->hmap + ws_->oT;
      int64_t cnt = 0;
      memcpy(&cnt, ho, sizeof(int64_t));
      const int64_t* hi = reinterpret_cast<const int64_t*>(ho + 1);
      const uint64_t* hk = reinterpret_cast<const uint64_t*>(ho + 1 + 2 * kc);
      out.resize((size_t)cnt);
      for (int64_t t = 0; t < cnt; ++t) out[t] = Pair{hi[t], ho[1 + kc + t]};
      (void)hk;
    }
    if (den_mu) {
      den_mu[0] = ws_->hmap[ws_->oM];
      den_mu[1] = ws_->hmap[ws_->oM + 1];
    }
    std::sort(out.begin(), out.end(), [](const Pair& a, const Pair& b) { return a.idx < b.idx; });
    return 0;
  }

  // Global top-k of a sharded fit: every shard's local list is its exact top-k
  // under (|value| desc, index asc), so the union holds the global one.  The
  // lists (key bits | index | value, empty slots keyed 0) are all-gathered on
  // the device and merged there by the same select, straight into mapped host
  // memory -- one host sync.  Every rank takes part, empty shards included.
  int topk_sharded(int mode, double mu, int64_t ke, std::vector<Pair>& out, double* den_mu) {
    cudaStream_t s = ws_->stream;
    const int world = comm_->world;
    const int64_t kc = ws_->kcap;
    TRY(ensure_shard_buf(world));
    double* loc = ws_->shard_buf + (1 + kc) * (1 + world);
    double* allc = loc + 3 * kc;
    uint64_t* ckey = reinterpret_cast<uint64_t*>(allc + 3 * kc * world);
    int64_t* cidx = reinterpret_cast<int64_t*>(ckey + kc * world);
    double* cval = reinterpret_cast<double*>(cidx + kc * world);
    int64_t* lcount = reinterpret_cast<int64_t*>(cval + kc * world);
    GI_CUDA_TRY(cudaMemsetAsync(loc, 0, sizeof(double) * 3 * ke, s));  // key 0 = empty slot
    if (ws_->p > 0) {
      TRY(gi::launch_topk(ws_->p, ke, mode, ws_->beta, ws_->g, mu, j_base_, ws_->ckey, ws_->cidx,
                          ws_->cval, reinterpret_cast<int64_t*>(loc + ke), loc + 2 * ke,
                          reinterpret_cast<uint64_t*>(loc), lcount, s,
                          den_mu ? ws_->scal + 5 : nullptr, ws_->ticket));
      ++launches;
    }
    TRY(comm_->allgather_device(loc, 3 * ke, allc, s));
    double* dm = ws_->dmap + ws_->oT;
    TRY(gi::launch_shard_merge(world, ke, allc, ckey, cidx, cval,
                               reinterpret_cast<int64_t*>(dm + 1), dm + 1 + kc,
                               reinterpret_cast<uint64_t*>(dm + 1 + 2 * kc),
                               reinterpret_cast<int64_t*>(dm), s));
    launches += 2;
    TRY(sync());
    const double* ho = ws_->hmap + ws_->oT;
    int64_t cnt = 0;
    memcpy(&cnt, ho, sizeof(int64_t));
    const int64_t* hi = reinterpret_cast<const int64_t*>(ho + 1);
    out.resize((size_t)cnt);
    for (int64_t t = 0; t < cnt; ++t) out[t] = Pair{hi[t], ho[1 + kc + t]};
    if (den_mu) {
      den_mu[0] = ws_->hmap[ws_->oM];
      den_mu[1] = ws_->hmap[ws_->oM + 1];
    }
    std::sort(out.begin(), out.end(), [](const Pair& a, const Pair& b) { return a.idx < b.idx; });
    return 0;
  }

  // sum over the held-out rows of (y - X_S w - C bcov)^2 (ws keep_test)
  int score(const std::vector<int64_t>& sup, const std::vector<double>& w,
            const std::vector<double>& bcov, double& sse) {
    const gi::MatrixDesc d = h_->desc();
    cudaStream_t s = ws_->stream;
    const int64_t* d_sup = nullptr;
    const double *d_w = nullptr, *d_cov = nullptr;
    TRY(stage(sup.data(), (int64_t)sup.size(), d_sup));
    TRY(stage(w.data(), (int64_t)w.size(), d_w));
    TRY(stage(bcov.data(), ws_->c, d_cov));
    TRY(flush());
    int rc = gi::launch_ax_residual(d, ws_->u, ws_->v, d_sup, d_w, (int64_t)sup.size(), ws_->y,
                                    ws_->c ? ws_->C : nullptr, (int)ws_->c, d_cov, ws_->keep_test,
                                    1.0, ws_->r, ws_->scal, nullptr, 0, nullptr, nullptr,
                                    ws_->beta, ws_->partials, ws_->ticket, s);
    if (rc != 0 && rc != -2) return -1;
    if (rc == -2) {
      if (!sup.empty())
        TRY(gi::launch_ax(d, ws_->u, ws_->v, d_sup, d_w, (int64_t)sup.size(), ws_->fitb, 0, s));
      TRY(gi::launch_refresh_residual(ws_->n, ws_->y, sup.empty() ? nullptr : ws_->fitb,
                                      ws_->c ? ws_->C : nullptr, (int)ws_->c, d_cov,
                                      ws_->keep_test, 1.0, ws_->r, ws_->scal, nullptr, 0, nullptr,
                                      nullptr, ws_->beta, ws_->partials, ws_->ticket, s));
    }
    gi::PubArgs pub;
    pub.add(ws_->scal, 1, ws_->oR);
    TRY(gi::launch_publish(pub, ws_->dmap, s));
    TRY(sync());
    sse = 2.0 * ws_->hmap[ws_->oR];  // scal[0] = 0.5 sum r^2 over the scored rows
    launches += 3;
    return 0;
  }

  int scatter_beta(const std::vector<int64_t>& idx_g, const std::vector<double>& w_g) {
    std::vector<int64_t> idx;
    std::vector<double> w;
    local_part(idx_g, w_g, idx, w);
    if (idx.empty()) return 0;
    // staged now, launched by the next refresh after its single upload
    TRY(stage(idx.data(), (int64_t)idx.size(), pend_idx_));
    TRY(stage(w.data(), (int64_t)w.size(), pend_w_));
    pend_k_ = (int64_t)idx.size();
    return 0;
  }

 private:
  gi_matrix* h_;
  FitWs* ws_;
  gi_fit_config cfg_;
  bool masked_;
  double n_eff_;
  gi_comm* comm_;
  int64_t j_base_;

 public:
  // lock-step group of concurrent fits (batch.cu), or NULL; only fast-kernel
  // fits join (an exact-kernel fit never submits a sweep)
  gi_batch* batch_ = nullptr;
  cudaEvent_t ready_ = nullptr;  // this fit's residual is ready for the group's sweep
  cudaEvent_t done_ = nullptr;   // the sweep serving it has completed
};

double dot(const std::vector<double>& a) {
  double s = 0.0;
  for (double x : a) s += x * x;
  return s;
}

// GI_TRACE_FIT=2: one stderr line per iteration (restriction, gradients, mu)
bool trace_steps() {
  static const bool on = [] {
    const char* e = getenv("GI_TRACE_FIT");
    return e && e[0] == '2';
  }();
  return on;
}

bool any_nonzero(const std::vector<double>& a) {
  for (double x : a)
    if (x != 0.0) return true;
  return false;
}

}  // namespace

static int fit_impl(gi_matrix* h, gi_comm* comm, int64_t j_base, const double* y,
                    const double* C, int64_t c, const uint8_t* keep, const double* u,
                    const double* v, const gi_fit_config* cfg, const int64_t* warm_idx,
                    const double* warm_w, int64_t warm_k, const double* bcov0,
                    gi_fit_result* res, gi_batch* batch = nullptr) {
  const auto t_start = std::chrono::steady_clock::now();
  CHECK_ARG(h && cfg && res, "NULL argument");
  CHECK_ARG(c >= 0 && c <= 64, "the native loop supports at most 64 covariate columns");
  CHECK_ARG(c == 0 || C != nullptr, "covariate matrix is NULL");
  CHECK_ARG(cfg->k >= 0 && cfg->max_iter >= 1, "invalid solver configuration");
  CHECK_ARG(res->trace_cap >= cfg->max_iter + 1, "loss trace buffer is too small");
  CHECK_ARG(res->support_cap >= std::max<int64_t>(cfg->k, warm_k), "support buffer too small");
  DeviceGuard guard(h->device);
  const int64_t kneed = std::max<int64_t>(std::max<int64_t>(cfg->k, warm_k), 1);
  const int64_t kcap = (kneed + kKcapQuantum - 1) / kKcapQuantum * kKcapQuantum;

  // take a workspace of the right shape from the device's pool (or make one);
  // y == NULL (resident inputs) needs one primed by an earlier call on h
  FitPool& pool = fit_pool_for(h->device);
  std::shared_ptr<FitWs> ws;
  {
    std::lock_guard<std::mutex> lock(pool.mu);
    // the tightest fit, most recently returned first among equals
    auto& items = pool.items;
    size_t best = items.size();
    for (size_t i = items.size(); i-- > 0;) {
      const auto& cand = items[i];
      if (cand->c == c && cand->kcap >= kneed && cand->n == h->n && cand->p == h->p &&
          (y != nullptr || (cand->primed && cand->primed_uid == h->uid)) &&
          (best == items.size() || cand->kcap < items[best]->kcap))
        best = i;
    }
    if (best != items.size()) {
      ws = items[best];
      items.erase(items.begin() + (long)best);
    }
  }
  if (!ws) {
    CHECK_ARG(y != nullptr, "gi_fit with y == NULL needs a previous call on this handle");
    TRY(make_ws(h, c, kcap, ws));
  }
  struct PoolReturn {
    FitPool& pool;
    std::shared_ptr<FitWs> ws;
    ~PoolReturn() {
      std::shared_ptr<FitWs> evicted;  // released outside the lock
      std::lock_guard<std::mutex> lock(pool.mu);
      pool.items.push_back(ws);
      if (pool.items.size() > kPoolCap) {
        evicted = pool.items.front();
        pool.items.erase(pool.items.begin());
      }
    }
  } pool_return{pool, ws};
  cudaStream_t s = ws->stream;
  if (ws->in_off != 0 || ws->in_flushed != 0) {
    // a previous fit on this workspace failed between stage() and sync():
    // drain its stream and start the staging arena afresh
    GI_CUDA_TRY(cudaStreamSynchronize(s));
    ws->in_off = ws->in_flushed = 0;
  }
  const int64_t n = h->n, p = h->p;
  double n_eff = (double)n;
  int64_t n_test = 0;  // held-out rows (keep == 2) of this call
  const bool masked = keep != nullptr || (y == nullptr && ws->masked);
  const gi::MatrixDesc d = h->desc();
  if (y == nullptr) {
    // inputs already resident from the previous call on this handle (benchmarks)
    CHECK_ARG(ws->primed, "gi_fit with y == NULL needs a previous call on this handle");
    n_eff = ws->n_eff;
    GI_CUDA_TRY(cudaMemsetAsync(ws->beta, 0, sizeof(double) * std::max<int64_t>(p, 1), s));
    GI_CUDA_TRY(cudaStreamSynchronize(s));
  } else {
  // ---- inputs
  GI_CUDA_TRY(cudaMemcpyAsync(ws->y, y, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  if (c) GI_CUDA_TRY(cudaMemcpyAsync(ws->C, C, sizeof(double) * n * c, cudaMemcpyHostToDevice, s));
  if (masked) {
    // keep: 2 = a held-out row scored after the fit, other nonzero = a fit row,
    // 0 = neither
    std::vector<uint8_t> fit_rows((size_t)n), test_rows((size_t)n);
    std::vector<uint32_t> mask((size_t)(ws->npad / 16), 0u);
    int64_t cnt = 0;
    n_test = 0;
    for (int64_t i = 0; i < n; ++i) {
      const bool fit_row = keep[i] != 0 && keep[i] != 2;
      fit_rows[(size_t)i] = fit_row;
      test_rows[(size_t)i] = keep[i] == 2;
      n_test += keep[i] == 2;
      if (fit_row) {
        mask[(size_t)(i >> 4)] |= 1u << (2 * (i & 15));
        ++cnt;
      }
    }
    GI_CUDA_TRY(cudaMemcpyAsync(ws->keep, fit_rows.data(), (size_t)n, cudaMemcpyHostToDevice, s));
    if (n_test)
      GI_CUDA_TRY(cudaMemcpyAsync(ws->keep_test, test_rows.data(), (size_t)n,
                                  cudaMemcpyHostToDevice, s));
    n_eff = (double)cnt;
    GI_CUDA_TRY(cudaMemcpyAsync(ws->rowmask, mask.data(), mask.size() * 4, cudaMemcpyHostToDevice,
                                s));
    // per-SNP counts over the kept rows: the fold handle's own when it was made
    // for exactly these rows (gi_matrix_with_masked_stats; every budget of a
    // CV fold), else one counting pass (its u, v outputs are overwritten below)
    if (h->fold_s1cnt && h->fold_keep == fit_rows)
      GI_CUDA_TRY(cudaMemcpyAsync(ws->s1cnt, h->fold_s1cnt->ptr, sizeof(int32_t) * 2 * p,
                                  cudaMemcpyDeviceToDevice, s));
    else
      TRY(gi::launch_stats(d, ws->rowmask, ws->u, ws->v, nullptr, ws->s1cnt, s));
  } else {
    GI_CUDA_TRY(cudaMemcpyAsync(ws->s1cnt, h->s1cnt->ptr, sizeof(int32_t) * 2 * p,
                                cudaMemcpyDeviceToDevice, s));
  }
  if (u && v) {
    GI_CUDA_TRY(cudaMemcpyAsync(ws->u, u, sizeof(double) * p, cudaMemcpyHostToDevice, s));
    GI_CUDA_TRY(cudaMemcpyAsync(ws->v, v, sizeof(double) * p, cudaMemcpyHostToDevice, s));
  } else {
    GI_CUDA_TRY(cudaMemcpyAsync(ws->u, h->du(), sizeof(double) * p, cudaMemcpyDeviceToDevice, s));
    GI_CUDA_TRY(cudaMemcpyAsync(ws->v, h->dv(), sizeof(double) * p, cudaMemcpyDeviceToDevice, s));
  }
  GI_CUDA_TRY(cudaMemsetAsync(ws->beta, 0, sizeof(double) * std::max<int64_t>(p, 1), s));
  GI_CUDA_TRY(cudaStreamSynchronize(s));
  ws->primed = true;
  ws->primed_uid = h->uid;
  ws->masked = masked;
  ws->n_eff = n_eff;
  }

  NativeFit F(h, ws.get(), cfg, masked, n_eff, comm, j_base);
  // lock-step group: live from here to the return (every exit path)
  struct BatchMember {
    gi_batch* b = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr, block = nullptr;
    ~BatchMember() {
      if (b) gi_batch_leave(b);
      if (ready) cudaEventDestroy(ready);
      if (done) cudaEventDestroy(done);
      if (block) cudaEventDestroy(block);
    }
  } member;
  if (batch && !F.exact_ && p > 0) {
    CHECK_ARG(gi_batch_matches(batch, h), "gi_fit_batched: matrix is not the group's");
    GI_CUDA_TRY(cudaEventCreateWithFlags(&member.ready, cudaEventDisableTiming));
    GI_CUDA_TRY(cudaEventCreateWithFlags(&member.done, cudaEventDisableTiming));
    TRY(gi_batch_join(batch));
    member.b = batch;
    F.batch_ = batch;
    F.ready_ = member.ready;
    F.done_ = member.done;
    GI_CUDA_TRY(cudaEventCreateWithFlags(&member.block,
                                         cudaEventBlockingSync | cudaEventDisableTiming));
    F.block_ev_ = member.block;
  }
  struct EventPair {
    cudaEvent_t a = nullptr, b = nullptr;
    ~EventPair() {
      if (a) cudaEventDestroy(a);
      if (b) cudaEventDestroy(b);
    }
  } evs;
  if (cfg->flags & 1) {
    GI_CUDA_TRY(cudaEventCreate(&evs.a));
    GI_CUDA_TRY(cudaEventCreate(&evs.b));
    F.ev0 = evs.a;
    F.ev1 = evs.b;
  }
  // ---- initial_state (iht.py:194-215): warm support or zero; b_cov from the caller
  std::vector<int64_t> sup;
  std::vector<double> w;
  for (int64_t t = 0; t < warm_k; ++t)
    if (warm_w[t] != 0.0) {
      sup.push_back(warm_idx[t]);
      w.push_back(warm_w[t]);
    }
  std::vector<double> bcov(bcov0, bcov0 + c);
  TRY(F.scatter_beta(sup, w));
  double loss = 0.0, gmax = 0.0;
  std::vector<double> gcov, gsup;
  TRY(F.refresh(sup, w, bcov, loss, gmax, gcov, gsup));
  int64_t trace_len = 0;
  res->loss_trace[trace_len++] = loss;
  int64_t iterations = 0, total_bt = 0;
  int reason = 1;  // max-iter

  std::vector<Pair> cand;
  std::vector<int64_t> ridx, new_sup, dsup;
  std::vector<double> rg, new_w, dval, cand_cov(c), dcov(c);
  for (int64_t it = 0; it < cfg->max_iter; ++it) {
    // ---------------------------------------------------------- iht_step
    double grad_max = gmax;
    for (double x : gcov) grad_max = std::max(grad_max, std::fabs(x));
    double step_inf;
    if (grad_max == 0.0) {
      step_inf = 0.0;  // fixed point (iht.py:262-267)
    } else {
      // restriction (iht.py:218-230)
      if (!sup.empty() && (any_nonzero(gsup) || any_nonzero(gcov))) {
        ridx = sup;
        rg = gsup;
      } else {
        TRY(F.topk(0, 0.0, cfg->k, cand));
        ridx.clear();
        rg.clear();
        for (const Pair& q : cand) {
          ridx.push_back(q.idx);
          rg.push_back(q.val);
        }
      }
      if (ridx.empty() && !(c && any_nonzero(gcov))) {
        step_inf = 0.0;  // k = 0 with settled covariates (iht.py:270-275)
      } else {
        // mu (iht.py:233-244)
        const double num = dot(rg) + dot(gcov);
        if (num == 0.0) {
          gi_set_error("gradient vanishes on the restriction; nothing to step on");
          return -2;
        }
        // den = ||X_S g_S + C g_cov||^2 and mu = num / den stay on the device; the
        // first candidate top-k reads mu there, so den, mu and the candidate come
        // back in one sync (iht.py:276-280)
        TRY(F.image_enqueue(ridx, rg, c ? &gcov : nullptr, 5, num, ws->dmap + ws->oM));
        double den_mu[2] = {0.0, 0.0};
        TRY(F.topk(1, 0.0, cfg->k, cand, den_mu));
        const double den = den_mu[0];
        if (den == 0.0 || !std::isfinite(den)) {
          gi_set_error("degenerate active set: restricted columns have zero image");
          return -3;
        }
        double mu = den_mu[1];  // == num / den, computed on the device in IEEE fp64
        if (trace_steps())
          fprintf(stderr,
                  "gi_fit step %lld: restriction %zu (g[0] %.17g), g_cov[0] %.17g, num %.17g, "
                  "den %.17g, mu %.17g\n",
                  (long long)it, ridx.size(), rg.empty() ? 0.0 : rg[0], c ? gcov[0] : 0.0, num,
                  den, mu);
        bool accepted = false;
        int64_t bt = 0;
        for (int64_t tries = 0; tries <= cfg->max_backtracks; ++tries) {
          if (tries > 0) TRY(F.topk(1, mu, cfg->k, cand));
          new_sup.clear();
          new_w.clear();
          for (const Pair& q : cand)
            if (q.val != 0.0) {
              new_sup.push_back(q.idx);
              new_w.push_back(q.val);
            }
          for (int64_t l = 0; l < c; ++l) {
            cand_cov[l] = bcov[l] - mu * gcov[l];
            dcov[l] = cand_cov[l] - bcov[l];
          }
          // delta over the union of old and new supports, ascending (iht.py:283-285)
          dsup.clear();
          dval.clear();
          size_t a = 0, b = 0;
          while (a < sup.size() || b < new_sup.size()) {
            int64_t j;
            double oldv = 0.0, newv = 0.0;
            if (b >= new_sup.size() || (a < sup.size() && sup[a] < new_sup[b])) {
              j = sup[a];
              oldv = w[a++];
            } else if (a >= sup.size() || new_sup[b] < sup[a]) {
              j = new_sup[b];
              newv = new_w[b++];
            } else {
              j = sup[a];
              oldv = w[a++];
              newv = new_w[b++];
            }
            const double dd = newv - oldv;
            if (dd != 0.0) {
              dsup.push_back(j);
              dval.push_back(dd);
            }
          }
          const double dsq = dot(dval) + dot(dcov);
          if (dsq == 0.0 || new_sup == ridx) {
            accepted = true;
            break;
          }
          double xdsq = 0.0;
          TRY(F.image_sumsq(dsup, dval, c ? &dcov : nullptr, xdsq));
          if (xdsq == 0.0) {
            accepted = true;
            break;
          }
          const double omega = (1.0 - cfg->c_omega) * dsq / xdsq;
          if (mu < omega) {
            accepted = true;
            break;
          }
          mu *= 0.5;
          ++bt;
        }
        total_bt += bt;
        if (!accepted) {
          reason = 2;  // step-size collapse; the state is not updated
          break;
        }
        step_inf = 0.0;
        for (double x : dval) step_inf = std::max(step_inf, std::fabs(x));
        for (double x : dcov) step_inf = std::max(step_inf, std::fabs(x));
        // beta <- candidate (old-only entries to 0, new entries to their values; one
        // upload), then refresh (iht.py:311-321)
        {
          std::vector<int64_t> uidx;
          std::vector<double> uval;
          size_t a2 = 0, b2 = 0;
          while (a2 < sup.size() || b2 < new_sup.size()) {
            if (b2 >= new_sup.size() || (a2 < sup.size() && sup[a2] < new_sup[b2])) {
              uidx.push_back(sup[a2++]);
              uval.push_back(0.0);
            } else {
              if (a2 < sup.size() && sup[a2] == new_sup[b2]) ++a2;
              uidx.push_back(new_sup[b2]);
              uval.push_back(new_w[b2++]);
            }
          }
          TRY(F.scatter_beta(uidx, uval));
        }
        sup = new_sup;
        w = new_w;
        bcov = cand_cov;
        // the last refresh of a fit (step_inf < tol, or the final allowed
        // iteration) needs only the loss
        const bool last = step_inf < cfg->tol || it + 1 >= cfg->max_iter;
        TRY(F.refresh(sup, w, bcov, loss, gmax, gcov, gsup, !last));
      }
    }
    ++iterations;
    res->loss_trace[trace_len++] = loss;
    if (!std::isfinite(loss)) {
      gi_set_error("loss diverged to a non-finite value");
      return -4;
    }
    if (step_inf < cfg->tol) {
      reason = 0;
      break;
    }
  }
  // ---- held-out score (cross-validation: the fold's test rows, standardised
  // with the fit's own statistics, model_select.py:138-139): sum over the
  // test rows of (y - X_S b - C b_cov)^2, in the fused residual kernel
  res->heldout_n = n_test;
  res->heldout_sse = 0.0;
  if (n_test > 0 && comm == nullptr) TRY(F.score(sup, w, bcov, res->heldout_sse));
  // ---- model (SparseModel.from_parts: nonzero weights, sorted)
  int64_t nnz = 0;
  for (size_t t = 0; t < sup.size(); ++t)
    if (w[t] != 0.0) {
      res->support[nnz] = sup[t];
      res->weights[nnz] = w[t];
      ++nnz;
    }
  res->nnz = nnz;
  for (int64_t l = 0; l < c; ++l) res->covar[l] = bcov[l];
  res->trace_len = trace_len;
  res->iterations = iterations;
  res->reason = reason;
  res->backtracks = total_bt;
  if (getenv("GI_TRACE_FIT"))
    fprintf(stderr,
            "gi_fit: %lld iterations, %d syncs, %.1f us waiting in sync, %d launches, "
            "%.1f us in gi_fit\n",
            (long long)iterations, F.syncs, F.sync_us, F.launches,
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_start)
                .count());
  res->xtr_kernel = F.exact_ ? 0
                     : F.batch_ ? 3
                     : h->desc().x3 == nullptr ? 1
                     : h->desc().mlist != nullptr ? 4 : 2;
  res->kernel_launches = F.launches;
  res->aty_ms_total = F.aty_ms;
  res->aty_launches = F.aty_launches;
  return 0;
}

extern "C" int gi_fit(gi_matrix* h, const double* y, const double* C, int64_t c,
                      const uint8_t* keep, const double* u, const double* v,
                      const gi_fit_config* cfg, const int64_t* warm_idx, const double* warm_w,
                      int64_t warm_k, const double* bcov0, gi_fit_result* res) {
  return fit_impl(h, nullptr, 0, y, C, c, keep, u, v, cfg, warm_idx, warm_w, warm_k, bcov0, res);
}

extern "C" int gi_fit_batched(gi_matrix* h, gi_batch* batch, const double* y, const double* C,
                              int64_t c, const uint8_t* keep, const double* u, const double* v,
                              const gi_fit_config* cfg, const int64_t* warm_idx,
                              const double* warm_w, int64_t warm_k, const double* bcov0,
                              gi_fit_result* res) {
  CHECK_ARG(batch != nullptr, "NULL batch group");
  return fit_impl(h, nullptr, 0, y, C, c, keep, u, v, cfg, warm_idx, warm_w, warm_k, bcov0, res,
                  batch);
}

extern "C" int gi_fit_many(gi_batch* batch, gi_fit_job* jobs, int64_t njobs, int threads) {
  CHECK_ARG(njobs >= 0 && (njobs == 0 || jobs != nullptr), "invalid job list");
  CHECK_ARG(threads >= 1, "need at least one thread");
  // chains: a job with warm_from = i starts from job i's result, on the thread
  // that ran job i, right after it (cv_iht's warm-started budget path)
  std::vector<int64_t> succ((size_t)njobs, -1), heads;
  for (int64_t i = 0; i < njobs; ++i) {
    const int64_t w = jobs[i].warm_from;
    if (w < 0) {
      heads.push_back(i);
      continue;
    }
    CHECK_ARG(w < i, "warm_from must name an earlier job");
    CHECK_ARG(succ[(size_t)w] < 0, "a job warm-starts at most one other job");
    CHECK_ARG(jobs[i].warm_idx == nullptr && jobs[i].warm_k == 0,
              "a chained job takes its warm start from warm_from only");
    succ[(size_t)w] = i;
  }
  std::atomic<int64_t> next{0};
  std::atomic<int> failed{0};
  const int64_t nheads = (int64_t)heads.size();
  auto run = [&](gi_fit_job& j, const int64_t* widx, const double* ww, int64_t wk,
                 const double* b0) {
    const int rc = fit_impl(j.h, nullptr, 0, j.y, j.C, j.c, j.keep, j.u, j.v, j.cfg, widx, ww,
                            wk, b0, j.res, batch);
    j.status = rc;
    j.error[0] = '\0';
    if (rc != 0) {
      snprintf(j.error, sizeof(j.error), "%s", gi_last_error());
      failed.store(1);
    }
    return rc;
  };
  auto worker = [&]() {
    std::vector<int64_t> widx;
    std::vector<double> ww, wb;
    for (int64_t hi = next.fetch_add(1); hi < nheads; hi = next.fetch_add(1)) {
      int64_t i = heads[(size_t)hi];
      int rc = run(jobs[i], jobs[i].warm_idx, jobs[i].warm_w, jobs[i].warm_k, jobs[i].bcov0);
      for (int64_t nx = succ[(size_t)i]; nx >= 0; i = nx, nx = succ[(size_t)nx]) {
        gi_fit_job& jn = jobs[nx];
        if (rc != 0) {  // the chain stops at a failed fit (the reference's loop raises there)
          jn.status = rc;
          snprintf(jn.error, sizeof(jn.error), "warm start source (job %lld) failed",
                   (long long)i);
          failed.store(1);
          continue;
        }
        // the previous result, trimmed to this budget by |weight| with ties to
        // the lower index (initial_state's hard_threshold, iht.py:204-206)
        const gi_fit_result& pr = *jobs[i].res;
        widx.assign(pr.support, pr.support + pr.nnz);
        ww.assign(pr.weights, pr.weights + pr.nnz);
        const int64_t k = jn.cfg->k;
        if ((int64_t)widx.size() > k) {
          std::vector<int64_t> ord(widx.size());
          for (size_t t = 0; t < ord.size(); ++t) ord[t] = (int64_t)t;
          std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
            const double fa = std::fabs(ww[(size_t)a]), fb = std::fabs(ww[(size_t)b]);
            return fa != fb ? fa > fb : widx[(size_t)a] < widx[(size_t)b];
          });
          ord.resize((size_t)k);
          std::sort(ord.begin(), ord.end());
          std::vector<int64_t> ti;
          std::vector<double> tw;
          for (int64_t t : ord) {
            ti.push_back(widx[(size_t)t]);
            tw.push_back(ww[(size_t)t]);
          }
          widx.swap(ti);
          ww.swap(tw);
        }
        wb.assign(pr.covar, pr.covar + jn.c);
        rc = run(jn, widx.empty() ? nullptr : widx.data(), ww.empty() ? nullptr : ww.data(),
                 (int64_t)widx.size(), wb.data());
      }
    }
  };
  const int nt = (int)std::min<int64_t>(threads, std::max<int64_t>(nheads, 1));
  std::vector<std::thread> pool;
  pool.reserve((size_t)nt);
  for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  if (failed.load()) {
    gi_set_error("gi_fit_many: at least one job failed (see the jobs' status)");
    return -1;
  }
  return 0;
}

// ------------------------------------------------------------------ gi_cv
namespace {

// Minimum-norm least squares of y on the columns of A (rows x c, row-major)
// with numpy.linalg.lstsq's rank cutoff (rcond = eps * max(rows, c) times the
// largest singular value): one-sided Jacobi SVD, x = V S^+ U^T y.  The cold
// starts' covariate block (iht.py:208); c <= 64.
void lstsq_min_norm(const std::vector<double>& A, int64_t rows, int64_t c,
                    const std::vector<double>& y, double* x) {
  std::vector<double> W(A);  // columns get rotated into U S
  std::vector<double> V((size_t)(c * c), 0.0);
  for (int64_t j = 0; j < c; ++j) V[(size_t)(j * c + j)] = 1.0;
  auto col = [&](int64_t i, int64_t j) -> double& { return W[(size_t)(i * c + j)]; };
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int64_t a = 0; a < c; ++a)
      for (int64_t b = a + 1; b < c; ++b) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (int64_t i = 0; i < rows; ++i) {
          alpha += col(i, a) * col(i, a);
          beta += col(i, b) * col(i, b);
          gamma += col(i, a) * col(i, b);
        }
        if (gamma == 0.0 || std::fabs(gamma) <= 1e-15 * std::sqrt(alpha * beta)) continue;
        off = std::max(off, std::fabs(gamma) / std::sqrt(alpha * beta));
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
        for (int64_t i = 0; i < rows; ++i) {
          const double wa = col(i, a), wb = col(i, b);
          col(i, a) = cs * wa - sn * wb;
          col(i, b) = sn * wa + cs * wb;
        }
        for (int64_t i = 0; i < c; ++i) {
          const double va = V[(size_t)(i * c + a)], vb = V[(size_t)(i * c + b)];
          V[(size_t)(i * c + a)] = cs * va - sn * vb;
          V[(size_t)(i * c + b)] = sn * va + cs * vb;
        }
      }
    if (off <= 1e-15) break;
  }
  std::vector<double> sv((size_t)c);
  double smax = 0.0;
  for (int64_t j = 0; j < c; ++j) {
    double s2 = 0.0;
    for (int64_t i = 0; i < rows; ++i) s2 += col(i, j) * col(i, j);
    sv[(size_t)j] = std::sqrt(s2);
    smax = std::max(smax, sv[(size_t)j]);
  }
  const double cut = std::numeric_limits<double>::epsilon() * (double)std::max(rows, c) * smax;
  std::vector<double> coef((size_t)c, 0.0);  // S^+ U^T y, U_j = W_j / s_j
  for (int64_t j = 0; j < c; ++j) {
    const double s = sv[(size_t)j];
    if (!(s > cut)) continue;
    double uy = 0.0;
    for (int64_t i = 0; i < rows; ++i) uy += col(i, j) * y[(size_t)i];
    coef[(size_t)j] = uy / (s * s);
  }
  for (int64_t r = 0; r < c; ++r) {
    double acc = 0.0;
    for (int64_t j = 0; j < c; ++j) acc += V[(size_t)(r * c + j)] * coef[(size_t)j];
    x[r] = acc;
  }
}

// the native loop's X^T r choice on a fold's shape (NativeFit): the exact
// kernel fits never join a lock-step group
bool cv_exact_kernel(const gi_matrix* h, int64_t n_fit, int64_t k, int64_t c) {
  const double tiles = (double)h->T * (double)h->G * GI_BLOCK_BYTES;
  return tiles <= 2.0 * 1048576.0 ||
         ((double)n_fit <= 8.0 * (double)(k + c + 1) && tiles <= 256.0 * 1048576.0);
}

}  // namespace

extern "C" int gi_cv(gi_matrix* h, const double* y, const double* C, int64_t c,
                     const int32_t* fold_labels, int q, const int64_t* path, int64_t npath,
                     const gi_fit_config* cfg, int std_mode, int warm_start, int threads,
                     double* mse) {
  CHECK_ARG(h && y && fold_labels && path && cfg && mse, "NULL argument");
  CHECK_ARG(q >= 2, "need at least two folds");
  CHECK_ARG(npath >= 1, "empty model-size path");
  CHECK_ARG(c >= 0 && c <= 64 && (c == 0 || C != nullptr), "covariates: 0..64 columns");
  CHECK_ARG(std_mode == 0 || std_mode == 1, "std_mode: 0 = train, 1 = global");
  CHECK_ARG(threads >= 1, "need at least one thread");
  const int64_t n = h->n;
  std::vector<int64_t> fold_size((size_t)q, 0);
  for (int64_t i = 0; i < n; ++i) {
    CHECK_ARG(fold_labels[i] >= 0 && fold_labels[i] < q, "fold label out of range");
    ++fold_size[(size_t)fold_labels[i]];
  }
  int64_t kmax = 0;
  for (int64_t i = 0; i < npath; ++i) {
    CHECK_ARG(path[i] >= 0, "negative budget");
    kmax = std::max(kmax, path[i]);
  }
  const int64_t min_train = n - *std::max_element(fold_size.begin(), fold_size.end());
  CHECK_ARG(kmax + c < min_train,
            "largest budget plus covariates must stay below the smallest training fold");
  // per fold: its row mask (1 training row, 2 test row), its matrix handle
  // (train mode: statistics of the training rows, formed on the device) and
  // the cold start's covariate block
  std::vector<std::vector<uint8_t>> keep((size_t)q);
  std::vector<gi_matrix*> fold_h((size_t)q, nullptr);
  struct FoldHandles {
    std::vector<gi_matrix*>& v;
    gi_matrix* base;
    ~FoldHandles() {
      for (gi_matrix* m : v)
        if (m && m != base) gi_matrix_free(m);
    }
  } fold_guard{fold_h, h};
  std::vector<double> bcov0((size_t)(q * std::max<int64_t>(c, 1)), 0.0);
  for (int f = 0; f < q; ++f) {
    std::vector<uint8_t>& kf = keep[(size_t)f];
    kf.resize((size_t)n);
    std::vector<uint8_t> train((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      kf[(size_t)i] = fold_labels[i] == f ? 2 : 1;
      train[(size_t)i] = fold_labels[i] != f;
    }
    if (std_mode == 0)
      TRY(gi_matrix_with_masked_stats(h, train.data(), &fold_h[(size_t)f]));
    else
      fold_h[(size_t)f] = h;
    if (c) {
      const int64_t nt = n - fold_size[(size_t)f];
      std::vector<double> A((size_t)(nt * c)), yt((size_t)nt);
      int64_t r = 0;
      for (int64_t i = 0; i < n; ++i)
        if (train[(size_t)i]) {
          for (int64_t l = 0; l < c; ++l) A[(size_t)(r * c + l)] = C[i * c + l];
          yt[(size_t)r++] = y[i];
        }
      lstsq_min_norm(A, nt, c, yt, &bcov0[(size_t)(f * c)]);
    }
  }
  // every (fold, budget) fit in one gi_fit_many, in a lock-step group when
  // the fits would run the fast kernel on more than 256 MB of genotypes
  const bool big = (double)h->p * (double)h->nb >= 256.0 * 1048576.0;
  gi_batch* group = nullptr;
  if (big && !warm_start && !cv_exact_kernel(h, min_train, kmax, c))
    TRY(gi_batch_create(h, 0, &group));
  struct GroupGuard {
    gi_batch* g;
    ~GroupGuard() {
      if (g) gi_batch_free(g);
    }
  } group_guard{group};
  const int64_t njobs = (int64_t)q * npath;
  std::vector<gi_fit_config> cfgs((size_t)njobs, *cfg);
  std::vector<gi_fit_result> res((size_t)njobs);
  std::vector<int64_t> sup_buf, tr_buf;
  std::vector<double> w_buf, cov_buf, trace_buf;
  int64_t cap_total = 0;
  for (int64_t i = 0; i < npath; ++i) cap_total += std::max<int64_t>(path[i], 1);
  sup_buf.resize((size_t)(q * cap_total));
  w_buf.resize((size_t)(q * cap_total));
  cov_buf.resize((size_t)(njobs * std::max<int64_t>(c, 1)));
  trace_buf.resize((size_t)(njobs * (cfg->max_iter + 1)));
  std::vector<gi_fit_job> jobs((size_t)njobs);
  int64_t off = 0;
  for (int f = 0; f < q; ++f)
    for (int64_t ki = 0; ki < npath; ++ki) {
      const int64_t j = f * npath + ki, cap = std::max<int64_t>(path[ki], 1);
      cfgs[(size_t)j].k = path[ki];
      gi_fit_result& r = res[(size_t)j];
      memset(&r, 0, sizeof(r));
      r.support = sup_buf.data() + off;
      r.weights = w_buf.data() + off;
      r.support_cap = cap;
      r.covar = cov_buf.data() + j * std::max<int64_t>(c, 1);
      r.loss_trace = trace_buf.data() + j * (cfg->max_iter + 1);
      r.trace_cap = cfg->max_iter + 1;
      off += cap;
      gi_fit_job& jb = jobs[(size_t)j];
      memset(&jb, 0, sizeof(jb));
      // warm starts: each budget from the fold's previous one (model_select.py:131-137)
      jb.warm_from = warm_start && ki > 0 ? j - 1 : -1;
      jb.h = fold_h[(size_t)f];
      jb.y = y;
      jb.C = C;
      jb.c = c;
      jb.keep = keep[(size_t)f].data();
      jb.cfg = &cfgs[(size_t)j];
      jb.bcov0 = c ? &bcov0[(size_t)(f * c)] : nullptr;
      jb.res = &r;
    }
  const int rc = gi_fit_many(group, jobs.data(), njobs, threads);
  if (rc != 0) {
    for (int64_t j = 0; j < njobs; ++j)
      if (jobs[(size_t)j].status != 0) {
        gi_set_error("solver failed at fold %lld, k=%lld: %s", (long long)(j / npath),
                     (long long)path[j % npath], jobs[(size_t)j].error);
        return jobs[(size_t)j].status;
      }
    return rc;
  }
  for (int f = 0; f < q; ++f)
    for (int64_t ki = 0; ki < npath; ++ki) {
      const gi_fit_result& r = res[(size_t)(f * npath + ki)];
      mse[ki * q + f] = r.heldout_n > 0 ? r.heldout_sse / (double)r.heldout_n : 0.0;
    }
  return 0;
}

extern "C" int gi_fit_sharded(gi_matrix* h, gi_comm* comm, int64_t j_base, const double* y,
                              const double* C, int64_t c, const uint8_t* keep, const double* u,
                              const double* v, const gi_fit_config* cfg,
                              const int64_t* warm_idx, const double* warm_w, int64_t warm_k,
                              const double* bcov0, gi_fit_result* res) {
  CHECK_ARG(comm != nullptr, "NULL communicator");
  CHECK_ARG(j_base >= 0, "negative SNP offset");
  return fit_impl(h, comm, j_base, y, C, c, keep, u, v, cfg, warm_idx, warm_w, warm_k, bcov0,
                  res);
}
