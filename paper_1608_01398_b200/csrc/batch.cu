// Lock-step batching of the X^T r sweeps of concurrent fits: the multi-RHS
// X^T R of cross-validation (north-star item 6; reference model_select.py:124-139,
// which runs one _aty_kernel sweep per fold fit and iteration).
//
// Fits that share one genotype matrix -- the q x |path| cold-start fold fits of
// cv_iht over row masks, or the budgets of a model-size path -- run on their
// own threads and streams (gi_fit_batched).  At each refresh a fit hands its
// residual, row mask, fold statistics and gradient buffer to the group and
// blocks; when every live fit of the group is waiting (or 32 have gathered,
// 16 with missing genotypes) the last to arrive launches ONE tensor-core sweep
// (xtr_mma.cu) for all of them on the group's stream, after each fit's
// residual is ready (events), and every fit's stream then waits on that
// sweep.  Fits join on entry and leave on exit, so a fit that finishes (or is
// in a backtracking phase, which needs no sweep) never holds the others for
// longer than its own phase.  Results equal the single-RHS tensor-core sweep
// of each fit: per-RHS integer sums do not interact.
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <deque>
#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/genoiht_cuda.h"
#include "batch.cuh"

namespace {
constexpr int kEvents = 64;  // ring of per-sweep completion events
}

struct gi_batch {
  int device = 0;
  int sms = 148;
  gi::MatrixDesc desc;                 // the shared tiles (checked per fit)
  std::shared_ptr<DevMem> tiles_ref;   // keeps the tiles alive
  std::shared_ptr<DevMem> gmiss_ref;
  bool any_missing = false;
  int max_rhs = 32;
  int wait_us = 0;  // optional straggler bound (GI_BATCH_WAIT_US), 0 = none
  cudaStream_t stream = nullptr;
  // device scratch, reused by consecutive sweeps in stream order
  gi::XtrRhs* d_desc = nullptr;
  double* qscal = nullptr;
  long long* qsum = nullptr;
  double* partials = nullptr;
  int64_t pcap = 0;
  unsigned int* tickets = nullptr;
  int8_t* qimg = nullptr;
  // from the device's stream-ordered pool (kept mapped): a CV creates and
  // drops a group, and cudaMalloc / cudaFree of the ~0.3 GB digit image cost
  // ~15 / ~40 ms at config 4
  std::vector<std::shared_ptr<DevMem>> allocs;
  cudaEvent_t events[kEvents] = {};
  uint64_t sweeps = 0;
  // group state
  std::mutex mu;
  std::condition_variable cv;
  int live = 0;
  struct Req {
    gi::XtrRhs rhs;
    cudaEvent_t ready;   // the fit's residual is ready (recorded on the fit's stream)
    cudaEvent_t done;    // recorded on the group's stream after the sweep that serves it
    int64_t sweep = -1;  // index of that sweep (-2: it failed)
  };
  std::deque<Req*> pending;
  // statistics
  uint64_t rhs_total = 0;

  ~gi_batch() {
    DeviceGuard g(device);
    if (stream) cudaStreamSynchronize(stream);
    allocs.clear();
    for (cudaEvent_t e : events)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }

  // Launch one sweep for the first (up to max_rhs) pending requests; caller
  // holds mu.  On a CUDA error every pending request fails (sweep = -2).
  int launch_locked() {
    const int rc = launch_sweep();
    if (rc != 0) {
      for (Req* r : pending) r->sweep = -2;
      pending.clear();
      cv.notify_all();
    }
    return rc;
  }

  int launch_sweep() {
    const int nb = (int)std::min<size_t>(pending.size(), (size_t)max_rhs);
    if (nb == 0) return 0;
    std::vector<gi::XtrRhs> rhs((size_t)nb);
    const int64_t sweep = (int64_t)sweeps;
    cudaEvent_t done = events[sweep % kEvents];
    for (int b = 0; b < nb; ++b) {
      Req* r = pending[(size_t)b];
      rhs[(size_t)b] = r->rhs;
      GI_CUDA_TRY(cudaStreamWaitEvent(stream, r->ready, 0));
    }
    // pageable source: staged by the driver at the call, so `rhs` may go
    GI_CUDA_TRY(cudaMemcpyAsync(d_desc, rhs.data(), sizeof(gi::XtrRhs) * (size_t)nb,
                                cudaMemcpyHostToDevice, stream));
    TRY(gi::launch_xtr_quant(desc.n, desc.T, nb, d_desc, qscal, qsum, qimg, partials, pcap,
                             tickets, stream));
    TRY(gi::launch_xtr_mma(desc, static_cast<const uint8_t*>(gmiss_ref->ptr), any_missing, nb,
                           qimg, qscal, qsum, d_desc, -1.0, sms, stream));
    GI_CUDA_TRY(cudaEventRecord(done, stream));
    for (int b = 0; b < nb; ++b) {
      // each fit waits on its own event: no aliasing however many sweeps pass
      // before its thread wakes
      GI_CUDA_TRY(cudaEventRecord(pending[(size_t)b]->done, stream));
      pending[(size_t)b]->sweep = sweep;
    }
    pending.erase(pending.begin(), pending.begin() + nb);
    ++sweeps;
    rhs_total += (uint64_t)nb;
    cv.notify_all();
    return 0;
  }
};

int gi_batch_submit(gi_batch* b, const gi::XtrRhs& rhs, cudaStream_t s, cudaEvent_t ready,
                    cudaEvent_t done) {
  GI_CUDA_TRY(cudaEventRecord(ready, s));
  gi_batch::Req req;
  req.rhs = rhs;
  req.ready = ready;
  req.done = done;
  std::unique_lock<std::mutex> lock(b->mu);
  b->pending.push_back(&req);
  if ((int)b->pending.size() >= b->live || (int)b->pending.size() >= b->max_rhs)
    b->launch_locked();  // failure is reported through req.sweep
  // Optional straggler bound (GI_BATCH_WAIT_US): a waiter that has waited
  // that long without a sweep launches what has gathered.  Off by default:
  // at config 4, 100 / 300 / 1000 us gave 0.60-0.65 / 0.42-0.47 / 0.39-0.54 s
  // (240 / 180 / 140 sweeps for 713 residuals) against ~0.27-0.48 s with ~40
  // sweeps when every live fit is waited for.
  while (req.sweep == -1) {
    if (b->wait_us <= 0) {
      b->cv.wait(lock);
    } else if (b->cv.wait_for(lock, std::chrono::microseconds(b->wait_us)) ==
                   std::cv_status::timeout &&
               req.sweep == -1 && !b->pending.empty()) {
      b->launch_locked();
    }
  }
  if (req.sweep < 0) {
    gi_set_error("batched X^T r sweep failed: %s", gi_last_error());
    return -1;
  }
  GI_CUDA_TRY(cudaStreamWaitEvent(s, req.done, 0));
  return 0;
}

int gi_batch_join(gi_batch* b) {
  std::lock_guard<std::mutex> lock(b->mu);
  ++b->live;
  return 0;
}

int gi_batch_leave(gi_batch* b) {
  std::lock_guard<std::mutex> lock(b->mu);
  --b->live;
  // the fits still waiting may now all be waiting
  if (!b->pending.empty() && (int)b->pending.size() >= b->live) return b->launch_locked();
  return 0;
}

bool gi_batch_matches(const gi_batch* b, const gi_matrix* h) {
  return b->desc.x == h->desc().x && b->desc.n == h->n && b->desc.p == h->p;
}

extern "C" {

int gi_batch_create(gi_matrix* h, int max_rhs, gi_batch** out) {
  CHECK_ARG(h && out, "NULL argument");
  DeviceGuard g(h->device);
  auto* b = new gi_batch();
  b->device = h->device;
  b->sms = h->sms;
  b->desc = h->desc();
  b->desc.x3 = nullptr;  // the tensor-core sweep reads the 2-bit tiles
  b->desc.T3 = 0;
  b->tiles_ref = h->x;
  b->gmiss_ref = h->gmiss;
  {
    std::vector<uint8_t> flags((size_t)h->G);
    if (h->G && cudaMemcpy(flags.data(), h->gmiss->ptr, (size_t)h->G, cudaMemcpyDeviceToHost) !=
                    cudaSuccess) {
      delete b;
      gi_set_error("gi_batch_create: reading the missing-genotype flags failed");
      return -1;
    }
    for (uint8_t f : flags) b->any_missing |= f != 0;
  }
  if (const char* w = getenv("GI_BATCH_WAIT_US")) b->wait_us = atoi(w);
  const int cap = gi::xtr_mma_max_rhs(b->any_missing);
  b->max_rhs = max_rhs > 0 && max_rhs < cap ? max_rhs : cap;
  auto fail = [&](cudaError_t e) {
    gi_set_error("gi_batch_create: %s", cudaGetErrorString(e));
    delete b;
    return -1;
  };
  cudaError_t e = cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return fail(e);
  for (auto& ev : b->events)
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return fail(e);
  auto dev = [&](size_t bytes, bool zero, auto** p) {
    std::shared_ptr<DevMem> m;
    if (alloc(m, bytes, b->device, zero) != 0) return false;
    b->allocs.push_back(m);
    *p = static_cast<std::remove_reference_t<decltype(*p)>>(m->ptr);
    return true;
  };
  const int mr = b->max_rhs;
  b->pcap = 4 * 148 * (int64_t)mr;
  // the digit image is written in full by each sweep's quantiser before use
  if (!dev(sizeof(gi::XtrRhs) * mr, true, &b->d_desc) ||
      !dev(sizeof(double) * 2 * mr, true, &b->qscal) ||
      !dev(sizeof(long long) * mr, true, &b->qsum) ||
      !dev(sizeof(double) * b->pcap, true, &b->partials) ||
      !dev(sizeof(unsigned int) * mr, true, &b->tickets) ||
      !dev((size_t)gi::xtr_mma_qimg_bytes(b->desc, mr), false, &b->qimg)) {
    delete b;
    return -1;
  }
  *out = b;
  return 0;
}

int gi_batch_stats(const gi_batch* b, int64_t* sweeps, int64_t* rhs) {
  CHECK_ARG(b != nullptr, "NULL batch");
  if (sweeps) *sweeps = (int64_t)b->sweeps;
  if (rhs) *rhs = (int64_t)b->rhs_total;
  return 0;
}

int gi_batch_free(gi_batch* b) {
  if (b) {
    CHECK_ARG(b->live == 0, "gi_batch_free: fits are still running in this group");
    delete b;
  }
  return 0;
}

}  // extern "C"
