/*
 * genoiht_cuda.h -- C ABI of libgenoiht_cuda.so, the sm_100a (B200) drop-in for
 * the IHT hot path of the reference package genoiht 0.1.0
 * (/root/reference/pkg/src/genoiht; arXiv 1608.01398 re-implementation).
 *
 * Conventions
 *   - Every function returns 0 on success and -1 on failure; gi_last_error()
 *     returns a thread-local message for the failing call.
 *   - Plain pointers and sizes only.  "Host" arguments are borrowed for the
 *     duration of the call; outputs are caller-allocated, as with the
 *     reference's numba kernels (geno_matrix.py:334, :361, :369).
 *   - gi_matrix handles own device memory.  A handle may be shared by several
 *     host threads: host-buffer calls serialise on a per-handle mutex, like the
 *     reference's _KERNEL_LOCK (geno_matrix.py:58-61); results never depend on
 *     which thread calls.
 *   - gi_dev_* functions take DEVICE pointers (on the handle's device) and a
 *     CUDA stream (cudaStream_t passed as void*, NULL = legacy default stream);
 *     they only enqueue work.  They are the building blocks of the device IHT
 *     loop (paper_1608_01398_b200/iht.py) and hold no hidden state, so any
 *     number of fits may run concurrently on one matrix.
 *   - Genotype bytes use the reference's BED layout on the host side:
 *     variant-major uint8[p, ceil(n/4)], four samples per byte from the least
 *     significant bit pair, codes 00 -> 0, 01 -> missing, 10 -> 1, 11 -> 2
 *     (plink_io.py:3-15).  On the device they live in the swizzled sample-tile
 *     layout described in paper_1608_01398_b200/csrc/common.cuh.
 */
#ifndef GENOIHT_CUDA_H
#define GENOIHT_CUDA_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gi_matrix gi_matrix;

/* ---------------------------------------------------------------- runtime */
int gi_version(void);
const char *gi_last_error(void);
/* number of visible CUDA devices (0 when none) */
int gi_device_count(int *count);
/* SM count, total HBM bytes and L2 bytes of a device */
int gi_device_info(int device, int *sm_count, int64_t *mem_bytes, int64_t *l2_bytes);
/* cudaDeviceSynchronize on `device` (used by timing code) */
int gi_device_sync(int device);

/* ---------------------------------------------------------- construction */
/* Replaces PackedGenotypeMatrix.from_bed_buffer (geno_matrix.py:281-292) and
 * _packed_stats (:239-246): uploads `data` (host, variant-major p x ceil(n/4),
 * kept verbatim) to `device` and computes u, v bit-identically. */
int gi_matrix_from_bed(const uint8_t *data, int64_t n, int64_t p, int device, gi_matrix **out);
/* Streaming construction (a BED file larger than host RAM, or one SNP shard of
 * it): create an empty n x p matrix, upload variant-major rows [j0, j0+count)
 * in any number of calls (host buffer count x ceil(n/4), staged through pinned
 * memory), then compute the statistics once.  read_bed (plink_io.py:82-100). */
int gi_matrix_create(int64_t n, int64_t p, int device, gi_matrix **out);
int gi_matrix_upload_bed(gi_matrix *h, int64_t j0, int64_t count, const uint8_t *data);
int gi_matrix_finalize(gi_matrix *h);
/* Device-side synthetic genotypes with the law of random_packed_matrix
 * (simulate.py:56-65) from a counter-based stream; SNP j_base + j of the
 * unsharded matrix gets identical bytes in any shard.  CPU twin: oracle/. */
int gi_matrix_synth(uint64_t seed, int64_t n, int64_t p, int64_t j_base, double maf_lo,
                    double maf_hi, double missing, int device, gi_matrix **out);
/* Replaces PackedGenotypeMatrix.with_stats (geno_matrix.py:310-316): new handle
 * sharing the packed bytes, with caller stats (host arrays of length p). */
int gi_matrix_with_stats(const gi_matrix *h, const double *u, const double *v, gi_matrix **out);
/* Replaces PackedGenotypeMatrix.subset_rows (geno_matrix.py:305-308): rows are
 * gathered on the device into a new matrix whose u, v are recomputed. */
int gi_matrix_subset_rows(const gi_matrix *h, const int64_t *rows, int64_t m, gi_matrix **out);
int gi_matrix_free(gi_matrix *h);

/* ------------------------------------------------------------ inspection */
int gi_matrix_shape(const gi_matrix *h, int64_t *n, int64_t *p, int *device);
/* No reference counterpart (device layout): X^T r streams a base-3 copy (5
 * genotypes per byte, 1.6 bits) built at finalize -- for a matrix with missing
 * genotypes (at most 5% of them) together with a list of their positions
 * (2 B each) that supplies the missing sums.  set = -1 queries, 0 drops the
 * copy, 1 builds it when possible; *base3 (may be NULL) receives 0 (2-bit
 * tiles), 1 (base-3 copy) or 2 (base-3 copy + missing-genotype list).  Changing the format
 * must not overlap a fit or X^T r on the same handle (it frees or replaces
 * the copy); with_stats copies made earlier keep the copy they share. */
int gi_matrix_xtr_format(gi_matrix *h, int set, int *base3);
/* u, v (host out, length p): PackedGenotypeMatrix.u / .v */
int gi_matrix_stats(const gi_matrix *h, double *u, double *v);
/* BED bytes of SNPs [j0, j0 + count) (host out, count x ceil(n/4)); backs
 * PackedGenotypeMatrix.data, to_codes (:294-296) and write_bed (plink_io.py:103-112) */
int gi_matrix_read_bed(const gi_matrix *h, int64_t j0, int64_t count, uint8_t *out);
/* per-SNP count of missing genotypes (host out, length p) */
int gi_matrix_missing_counts(const gi_matrix *h, int32_t *out);
/* device pointers of the handle's u and v (length p) */
int gi_matrix_device_stats(const gi_matrix *h, const double **d_u, const double **d_v);
/* column statistics over the rows with keep[i] != 0 (host in, length n):
 * the u, v that subset_rows(rows) would compute, without re-packing */
int gi_matrix_masked_stats(const gi_matrix *h, const uint8_t *keep, double *u, double *v);
/* a copy of h (same tiles) standardised with those statistics, computed on the
 * device (no host round trip): a CV fold's matrix in train mode
 * (model_select.py:87-93) */
int gi_matrix_with_masked_stats(const gi_matrix *h, const uint8_t *keep, gi_matrix **out);

/* ------------------------------------------------ operator protocol (host) */
/* aty_genetic (geno_matrix.py:351-364).  mode 0: exact -- bit-identical to
 * _aty_kernel (:142-165) when sum_r is numpy's r.sum(); mode 1: fast lookup-
 * table kernel (fp32 tables, fp64 accumulation; sum_r ignored); mode 2:
 * tensor-core kernel (tcgen05.mma kind::i8 over the 2-bit tiles: exact
 * integer sums of the residual quantised to 2^-26 of its range; sum_r
 * ignored). */
int gi_aty(gi_matrix *h, const double *r, double sum_r, double *out, int mode);
/* Batched aty_genetic for B right-hand sides, e.g. the residuals of q CV folds
 * (zero outside each fold) with each fold's own statistics (reference
 * model_select.py:87-93, :131-137; SURVEY.md section 8(b) gi_aty_batched).
 * R is (B, n) row-major; U, V are (B, p) row-major per-RHS stats, or NULL for
 * the handle's; sum_R[b] plays sum_r of gi_aty (mode 0; may be NULL in mode 1);
 * G is (B, p).  G[b] equals gi_aty of R[b] under stats (U[b], V[b]) -- bit for
 * bit in mode 0.  Modes 0 and 1: one X^T r sweep per RHS, queued back to back
 * on the matrix's stream with one host sync.  Mode 2 (the multi-RHS X^T R):
 * ONE tensor-core sweep of the tiles per batch of up to 32 right-hand sides
 * (16 when the matrix has missing genotypes); each decoded genotype tile feeds
 * every right-hand side of the batch (xtr_mma.cu). */
int gi_aty_batched(gi_matrix *h, const double *R, const double *sum_R, const double *U,
                   const double *V, int64_t B, double *G, int mode);
/* ax_columns (geno_matrix.py:328-349), bit-identical to _ax_cols_kernel (:168-194) */
int gi_ax_cols(gi_matrix *h, const int64_t *idx, const double *w, int64_t k, double *out);
/* decompress (geno_matrix.py:366-373): out_t is (k, n) row-major, i.e. the
 * reference's out_t before its final transpose; bit-identical to :216-236 */
int gi_decompress(gi_matrix *h, const int64_t *idx, int64_t k, double *out_t);

/* ------------------------------------------- device primitives (IHT loop) */
/* u, v may be NULL to use the handle's own statistics. */
int gi_dev_ax(gi_matrix *h, const double *u, const double *v, const int64_t *d_idx,
              const double *d_w, int64_t k, double *d_out, int accumulate, void *stream);
/* g = scale * X^T r with the lookup-table kernel.  d_rt = fp32(r - mean) on the
 * view's rows (zero elsewhere), padded to gi_padded_samples(h) entries, as
 * written by gi_dev_center; d_scal[1] = mean, d_scal[2] = sum(d_rt).
 * d_s1cnt: per-SNP (sum of dosages, observed count) over the view's rows
 * (gi_dev_stats), NULL = all rows of the handle. */
int gi_dev_aty_fast(gi_matrix *h, const double *u, const double *v, const int32_t *d_s1cnt,
                    const float *d_rt, const double *d_scal, double scale, double *d_out,
                    void *stream);
/* exact kernel: d_rpad fp64 padded to gi_padded_samples(h), d_sum_r device scalar */
int gi_dev_aty_exact(gi_matrix *h, const double *u, const double *v, const double *d_rpad,
                     const double *d_sum_r, double scale, double *d_out, void *stream);
int64_t gi_padded_samples(const gi_matrix *h);
/* masked column statistics into device arrays; d_rowmask has one uint32 per
 * (tile, word) = gi_padded_samples/16 entries, bit 2s set for included sample s
 * (NULL = all rows); d_s1cnt (optional) receives int32 (sum, count) pairs */
int gi_dev_stats(gi_matrix *h, const uint32_t *d_rowmask, double *d_u, double *d_v,
                 int32_t *d_s1cnt, void *stream);

/* Reduction workspace: d_partials >= gi_red_partials() doubles, d_ticket one
 * zero-initialised uint32 (the kernels leave it zero again). */
int64_t gi_red_partials(void);
/* r = keep ? y - (fit + C bcov) : 0; d_scal[0] = 0.5 r.r, d_scal[1] = sum(r)/n_eff.
 * d_fit, d_C, d_keep may be NULL; C is row-major (n, c). */
int gi_dev_residual(int64_t n, const double *d_y, const double *d_fit, const double *d_C,
                    int64_t c, const double *d_bcov, const uint8_t *d_keep, double n_eff,
                    double *d_r, double *d_scal, double *d_partials, uint32_t *d_ticket,
                    void *stream);
/* rt = keep ? fp32(r - d_scal[1]) : 0 over n_pad entries; d_scal[2] = sum(rt) */
int gi_dev_center(int64_t n, int64_t n_pad, const double *d_r, const uint8_t *d_keep,
                  double *d_scal, float *d_rt, double *d_partials, uint32_t *d_ticket,
                  void *stream);
/* d_gcov[l] = -sum_i C[i, l] r_i, l < c */
int gi_dev_covgrad(int64_t n, const double *d_C, int64_t c, const double *d_r, double *d_gcov,
                   double *d_partials, uint32_t *d_ticket, void *stream);
/* d_scal[slot] = max |x| */
int gi_dev_maxabs(int64_t m, const double *d_x, double *d_scal, int slot, double *d_partials,
                  uint32_t *d_ticket, void *stream);
/* d_scal[slot] = x . x */
int gi_dev_sumsq(int64_t m, const double *d_x, double *d_scal, int slot, double *d_partials,
                 uint32_t *d_ticket, void *stream);
/* x += C w (C row-major (n, c)) */
int gi_dev_add_cov(int64_t n, const double *d_C, int64_t c, const double *d_w, double *d_x,
                   void *stream);

/* Hard-threshold select (top_k_indices iht.py:36-49, hard_threshold :52-58):
 * the k largest |value| under (|value| desc, index asc), value = g_j (mode 0)
 * or beta_j - mu * g_j (mode 1, computed with the reference's two roundings).
 * Candidate scratch: gi_topk_slots(p, k) entries each of d_ckey/d_cidx/d_cval.
 * Outputs (unordered, *d_count <= k): global index (idx_base + local j),
 * value, key (|value| bits + 1). */
int64_t gi_topk_slots(int64_t p, int64_t k);
int gi_dev_topk(int64_t p, int64_t k, int mode, const double *d_beta, const double *d_g,
                double mu, int64_t idx_base, uint64_t *d_ckey, int64_t *d_cidx, double *d_cval,
                int64_t *d_out_idx, double *d_out_val, uint64_t *d_out_key, int64_t *d_count,
                void *stream);
/* beta[idx[t]] = val[t];  dst[t] = src[idx[t]] */
int gi_dev_scatter(int64_t k, const int64_t *d_idx, const double *d_val, double *d_beta,
                   void *stream);
int gi_dev_gather(int64_t k, const int64_t *d_idx, const double *d_src, double *d_dst,
                  void *stream);

/* ------------------------------------------------------ native solver loop */
/* IhtConfig (iht.py:120-140) */
typedef struct {
  int64_t k;
  int64_t max_iter;
  double tol;
  double c_omega;
  int64_t max_backtracks;
  int64_t flags;  /* bit 0: time every X^T r launch with CUDA events (aty_ms_total);
                     bit 1: the caller chooses the X^T r kernel (bit 2 set = the exact
                     fp64 kernel) -- gi_fit_sharded callers pass the choice made on
                     the GLOBAL shape so every rank and the unsharded fit agree */
} gi_fit_config;

/* FitResult (iht.py:172-180); caller-allocated arrays, capacities in *_cap */
typedef struct {
  int64_t *support;      /* out: sorted support (nonzero weights only) */
  double *weights;       /* out: matching weights */
  int64_t support_cap;   /* in: >= max(k, warm_k) */
  int64_t nnz;           /* out */
  double *covar;         /* out: c covariate coefficients */
  double *loss_trace;    /* out: loss after initial state and each accepted step */
  int64_t trace_cap;     /* in: >= max_iter + 1 */
  int64_t trace_len;     /* out */
  int64_t iterations;    /* out */
  int64_t backtracks;    /* out: total step halvings */
  int64_t kernel_launches; /* out */
  double aty_ms_total;   /* out: summed X^T r kernel time (flags bit 0) */
  int64_t aty_launches;  /* out: X^T r launches */
  int reason;            /* out: 0 converged, 1 max-iter, 2 step-size collapse */
  double heldout_sse;    /* out: sum over the rows with keep == 2 of (y - X_S b - C b_cov)^2 */
  int64_t heldout_n;     /* out: their count */
  int xtr_kernel;        /* out: X^T r kernel the loop ran: 0 exact fp64, 1 fast over the
                            2-bit tiles, 2 fast over the base-3 copy, 3 the lock-step
                            group's tensor-core sweeps (gi_fit_batched), 4 fast over
                            the base-3 copy plus the missing-genotype list */
} gi_fit_result;

/* Replaces genoiht.fit (iht.py:326-354) on one GPU: the complete IHT loop with
 * device kernels, one host sync per phase.  y (n) and C (row-major n x c,
 * c <= 64) are host arrays over the handle's n samples; keep (n, optional)
 * restricts the fit to rows with keep != 0, 2 (cross-validation training rows:
 * other rows' residuals are pinned to 0); rows with keep == 2 are held out and
 * scored after the fit (heldout_sse / heldout_n: the fold's test rows,
 * model_select.py:138-139); u, v (p, optional) override the
 * handle's stats; warm_idx/warm_w (warm_k, sorted, may be NULL) seed the
 * support; bcov0 (c) is the initial covariate block (least squares on the
 * caller side, as in initial_state iht.py:207-208).  y == NULL reuses the y, C,
 * keep and stats left resident on the device by the previous gi_fit call on
 * this handle (benchmarks).  Returns 0, -1 (CUDA /
 * argument error), -2 "gradient vanishes ..." (ValueError, iht.py:237),
 * -3 "degenerate active set ..." (ValueError, iht.py:243) or -4 "loss diverged
 * ..." (FloatingPointError, iht.py:348). */
int gi_fit(gi_matrix *h, const double *y, const double *C, int64_t c, const uint8_t *keep,
           const double *u, const double *v, const gi_fit_config *cfg, const int64_t *warm_idx,
           const double *warm_w, int64_t warm_k, const double *bcov0, gi_fit_result *res);

/* ------------------------------------------- lock-step groups (multi-RHS) */
/* Concurrent fits over one matrix (cross-validation folds as row masks, the
 * budgets of a model-size path) share their X^T r sweeps: gi_fit_batched is
 * gi_fit whose refresh hands the residual to the group; when every live fit
 * of the group waits, ONE tensor-core sweep (gi_aty_batched mode 2) serves
 * all of them (<= 32 residuals, 16 with missing genotypes).  The reference
 * runs one _aty_kernel sweep per fold fit and iteration (model_select.py:124-139).
 * A group is tied to the tiles of h (with_stats copies share them).  Fits of a
 * group must run on separate host threads; results equal each fit's own
 * tensor-core sweep. */
typedef struct gi_batch gi_batch;
int gi_batch_create(gi_matrix *h, int max_rhs, gi_batch **out);
int gi_batch_stats(const gi_batch *b, int64_t *sweeps, int64_t *rhs);
int gi_batch_free(gi_batch *b);
int gi_fit_batched(gi_matrix *h, gi_batch *batch, const double *y, const double *C, int64_t c,
                   const uint8_t *keep, const double *u, const double *v,
                   const gi_fit_config *cfg, const int64_t *warm_idx, const double *warm_w,
                   int64_t warm_k, const double *bcov0, gi_fit_result *res);

/* Many fits in one call (no reference counterpart: cv_iht's fold x budget
 * loop, model_select.py:124-139, and a model-size path, cli.py:326-331, run
 * their fits one after another): job i is gi_fit (batch == NULL) or
 * gi_fit_batched (batch != NULL) with job i's arguments, run on `threads`
 * native worker threads that take the jobs in index order.  Each job's
 * status (0 or a gi_fit error code) and error message land in the job; the
 * call returns 0 when every job succeeded, -1 otherwise.  Chains of jobs
 * (warm_from) give the warm-started budget path of cv_iht (model_select.py:131-137).  Host threads of
 * the caller's language (and its interpreter lock) stay out of the fits'
 * start-up: a Python thread pool needed ~1 ms per job to hand 32 fits their
 * threads. */
typedef struct gi_fit_job {
  gi_matrix *h;
  const double *y;
  const double *C;
  int64_t c;
  const uint8_t *keep;
  const double *u;
  const double *v;
  const gi_fit_config *cfg;
  const int64_t *warm_idx;
  const double *warm_w;
  int64_t warm_k;
  const double *bcov0;
  gi_fit_result *res;
  int64_t warm_from; /* -1, or an earlier job whose result warm-starts this one
                        (trimmed to cfg->k as initial_state does); the job then
                        runs on that job's thread right after it, and
                        warm_idx / warm_w / warm_k / bcov0 are ignored */
  int status;       /* out */
  char error[256];  /* out: gi_last_error() of a failed job */
} gi_fit_job;
int gi_fit_many(gi_batch *batch, gi_fit_job *jobs, int64_t njobs, int threads);

/* Replaces the fold x budget loop of genoiht.cv_iht (model_select.py:101-139):
 * q folds (fold_labels[i] in 0..q-1 over the handle's n samples) x the npath
 * budgets of path, each fit cold-started (covariate block by minimum-norm
 * least squares on the fold's training rows, as numpy.linalg.lstsq,
 * iht.py:208) or, with warm_start, from the fold's previous budget
 * (model_select.py:131-137), on the fold's training rows -- std_mode 0:
 * standardised with the training rows' statistics (model_select.py:87-93), 1:
 * with the handle's -- and scored on the fold's test rows: mse[ki * q + f] =
 * mean squared prediction error of budget path[ki] on fold f
 * (model_select.py:138-139).  The fits run through gi_fit_many on `threads`
 * native threads, cold starts in a lock-step group (shared tensor-core X^T R
 * sweeps) when the fast kernel runs on more than 256 MB of genotypes, warm
 * starts as one chain per fold.  select_k, the final
 * fit and refit_least_squares stay with the caller (model_select.py:141-146).
 * A failed fit returns its status with "solver failed at fold f, k=k: ...". */
int gi_cv(gi_matrix *h, const double *y, const double *C, int64_t c, const int32_t *fold_labels,
          int q, const int64_t *path, int64_t npath, const gi_fit_config *cfg, int std_mode,
          int warm_start, int threads, double *mse);

/* ------------------------------------------------ SNP-sharded native loop */
/* One process per GPU, each holding a contiguous SNP block [j_base, j_base +
 * p_local) of the matrix.  The shards exchange only the
 * n-length partial products X_S w (all-reduce, in place on the device), max|g|
 * with the support's gradient entries, and the k top-k candidates per shard
 * (all-gathers); every rank takes identical decisions. */
typedef struct gi_comm gi_comm;
/* host collectives supplied by the caller (e.g. torch.distributed / gloo):
 * in-place all-reduce (op 0 sum, 1 max) and rank-major all-gather */
typedef int (*gi_comm_allreduce_fn)(void *ctx, double *buf, int64_t count, int op);
typedef int (*gi_comm_allgather_fn)(void *ctx, const double *send, int64_t count, double *recv);
int gi_comm_nccl_available(void);
/* 128-byte ncclUniqueId from rank 0, to be broadcast to the other ranks */
int gi_comm_nccl_unique_id(uint8_t *out);
int gi_comm_create_nccl(const uint8_t *id, int world, int rank, int device, gi_comm **out);
int gi_comm_create_callbacks(int world, int rank, void *ctx, gi_comm_allreduce_fn allreduce,
                             gi_comm_allgather_fn allgather, gi_comm **out);
int gi_comm_free(gi_comm *comm);
/* gi_fit over the local shard h (global SNP indices in warm_idx and in the
 * result), joined through comm; y, C, keep, bcov0 are replicated. */
int gi_fit_sharded(gi_matrix *h, gi_comm *comm, int64_t j_base, const double *y, const double *C,
                   int64_t c, const uint8_t *keep, const double *u, const double *v,
                   const gi_fit_config *cfg, const int64_t *warm_idx, const double *warm_w,
                   int64_t warm_k, const double *bcov0, gi_fit_result *res);

#ifdef __cplusplus
}
#endif
#endif /* GENOIHT_CUDA_H */
