/*
 * genoiht_oracle.c -- CPU restatement of the reference's packed-genotype kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package
 * (paper_1608_01398_b200/) links, loads or calls this file.  It is built into
 * oracle/_build/libgenoiht_oracle.so and used by tests/, __graft_entry__.smoke()
 * (as the checker) and bench.py's cpu_baseline / --impl reference leg (as the
 * timed CPU path of the reference algorithm).
 *
 * Every function restates one numba kernel of the reference package
 * `genoiht` 0.1.0 (/root/reference/pkg/src/genoiht/geno_matrix.py) with the
 * same arithmetic, the same per-element operation order and the same work
 * partition (column chunks of 256, sample chunks of 1024), so that results are
 * bit-identical to the reference for any thread count.  Compile with
 * -ffp-contract=off: numba (fastmath=False) never contracts a*b+c into an FMA.
 *
 * Layout: `data` is the reference's variant-major buffer uint8[p, nb],
 * nb = ceil(n/4), four samples per byte starting at the least significant bit
 * pair, codes 00 -> dose 0, 01 -> missing, 10 -> dose 1, 11 -> dose 2
 * (geno_matrix.py:28-34, plink_io.py:3-15).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORA_COL_CHUNK 256   /* geno_matrix.py:55 */
#define ORA_ROW_CHUNK 1024  /* geno_matrix.py:56 */

/* Per-byte expansion tables, geno_matrix.py:37-53. */
static double k_dose[256][4];
static double k_miss[256][4];
static double k_obs[256][4];
static int k_tables_ready = 0;

static void ora_build_tables(void) {
    static const double code_dose[4] = {0.0, 0.0, 1.0, 2.0};
    if (k_tables_ready) return;
    for (int byte = 0; byte < 256; ++byte) {
        for (int slot = 0; slot < 4; ++slot) {
            int code = (byte >> (2 * slot)) & 3;
            int missing = (code == 1);
            k_miss[byte][slot] = missing ? 1.0 : 0.0;
            k_obs[byte][slot] = missing ? 0.0 : 1.0;
            k_dose[byte][slot] = missing ? 0.0 : code_dose[code];
        }
    }
    k_tables_ready = 1;
}

int ora_set_threads(int count) {
#ifdef _OPENMP
    if (count > 0) omp_set_num_threads(count);
    return omp_get_max_threads();
#else
    (void)count;
    return 1;
#endif
}

/* _stats_kernel, geno_matrix.py:106-139: integer-valued fp64 sums over the
 * observed entries, then u = s1/cnt and v = 1/sqrt(var) with ddof = 1. */
void ora_stats(const uint8_t *data, int64_t p, int64_t nb, int64_t n,
               double *u, double *v) {
    static const double code_dose[4] = {0.0, 0.0, 1.0, 2.0};
    const int64_t nfull = n / 4;
    const int64_t rem = n - 4 * nfull;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < p; ++j) {
        const uint8_t *col = data + j * nb;
        double cnt = 0.0, s1 = 0.0, s2 = 0.0;
        for (int64_t b = 0; b < nfull; ++b) {
            const int byte = col[b];
            for (int s = 0; s < 4; ++s) {
                const int code = (byte >> (2 * s)) & 3;
                if (code != 1) {
                    const double d = code_dose[code];
                    cnt += 1.0;
                    s1 += d;
                    s2 += d * d;
                }
            }
        }
        if (rem > 0) {
            const int byte = col[nfull];
            for (int s = 0; s < rem; ++s) {
                const int code = (byte >> (2 * s)) & 3;
                if (code != 1) {
                    const double d = code_dose[code];
                    cnt += 1.0;
                    s1 += d;
                    s2 += d * d;
                }
            }
        }
        u[j] = cnt > 0.0 ? s1 / cnt : 0.0;
        if (cnt >= 2.0) {
            const double var = (s2 - s1 * s1 / cnt) / (cnt - 1.0);
            v[j] = var > 0.0 ? 1.0 / sqrt(var) : 0.0;
        } else {
            v[j] = 0.0;
        }
    }
}

/* _aty_kernel, geno_matrix.py:142-165.  r_pad has 4*nb entries, zero past n;
 * sum_r is the caller's numpy r.sum() (geno_matrix.py:363). */
void ora_aty(const uint8_t *data, int64_t p, int64_t nb, const double *u,
             const double *v, const double *r_pad, double sum_r, double *out) {
    ora_build_tables();
    const int64_t nchunk = (p + ORA_COL_CHUNK - 1) / ORA_COL_CHUNK;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nchunk; ++c) {
        const int64_t lo = c * ORA_COL_CHUNK;
        const int64_t hi = lo + ORA_COL_CHUNK < p ? lo + ORA_COL_CHUNK : p;
        for (int64_t j = lo; j < hi; ++j) {
            const uint8_t *col = data + j * nb;
            double t = 0.0, m = 0.0;
            for (int64_t b = 0; b < nb; ++b) {
                const int byte = col[b];
                const double *rr = r_pad + 4 * b;
                const double *dz = k_dose[byte];
                const double *ms = k_miss[byte];
                t += dz[0] * rr[0] + dz[1] * rr[1] + dz[2] * rr[2] + dz[3] * rr[3];
                m += ms[0] * rr[0] + ms[1] * rr[1] + ms[2] * rr[2] + ms[3] * rr[3];
            }
            out[j] = v[j] * (t - u[j] * (sum_r - m));
        }
    }
}

/* _ax_cols_kernel, geno_matrix.py:168-194: out[i] += sum_t dose*scale - obs*shift
 * with the column order of idx fixed inside each 1024-sample chunk. */
void ora_ax_cols(const uint8_t *data, int64_t p, int64_t nb, int64_t n,
                 const double *u, const double *v, const int64_t *idx,
                 int64_t k, const double *w, double *out) {
    (void)p;
    ora_build_tables();
    const int64_t nchunk = (n + ORA_ROW_CHUNK - 1) / ORA_ROW_CHUNK;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nchunk; ++c) {
        const int64_t s_lo = c * ORA_ROW_CHUNK;
        const int64_t s_hi = s_lo + ORA_ROW_CHUNK < n ? s_lo + ORA_ROW_CHUNK : n;
        const int64_t b_lo = s_lo / 4, b_last = (s_hi - 1) / 4;
        for (int64_t t = 0; t < k; ++t) {
            const int64_t j = idx[t];
            const double scale = w[t] * v[j];
            if (scale == 0.0) continue;
            const double shift = u[j] * scale;
            const uint8_t *col = data + j * nb;
            for (int64_t b = b_lo; b < b_last; ++b) {
                const int byte = col[b];
                double *o = out + 4 * b;
                for (int s = 0; s < 4; ++s)
                    o[s] += k_dose[byte][s] * scale - k_obs[byte][s] * shift;
            }
            const int byte = col[b_last];
            const int64_t base = 4 * b_last;
            for (int64_t s = 0; s < s_hi - base; ++s)
                out[base + s] += k_dose[byte][s] * scale - k_obs[byte][s] * shift;
        }
    }
}

/* _decompress_kernel, geno_matrix.py:216-236: out_t[t, i] = (dose - u) * v * obs. */
void ora_decompress(const uint8_t *data, int64_t p, int64_t nb, int64_t n,
                    const double *u, const double *v, const int64_t *idx,
                    int64_t k, double *out_t) {
    (void)p;
    ora_build_tables();
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < k; ++t) {
        const int64_t j = idx[t];
        const double uj = u[j], vj = v[j];
        const uint8_t *col = data + j * nb;
        double *row = out_t + t * n;
        for (int64_t i = 0; i < n; ++i) {
            const int byte = col[i >> 2];
            const int s = (int)(i & 3);
            row[i] = (k_dose[byte][s] - uj) * vj * k_obs[byte][s];
        }
    }
}

/* ------------------------------------------------------------------------
 * CPU twin of the product's counter-based synthetic genotype generator
 * (paper_1608_01398_b200/csrc/synth.cu).  Same distribution as the
 * reference's random_packed_matrix (simulate.py:56-65: per-SNP frequency
 * f ~ U(lo, hi), dosage ~ Binomial(2, f), code = [0, 2, 3][dosage], missing
 * -> code 1 with probability `missing`), drawn from a stateless hash so that
 * any slice can be generated independently and the CPU and GPU emit the same
 * bytes.  Writes the reference's variant-major layout uint8[p_count, nb] for
 * SNPs [j0, j0 + p_count).
 * ------------------------------------------------------------------------ */
static inline uint64_t ora_mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ULL;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBULL;
    x ^= x >> 31;
    return x;
}

static inline uint64_t ora_key(uint64_t seed, uint64_t j, uint64_t i) {
    return ora_mix64(seed * 0x9E3779B97F4A7C15ULL + j * 0xD1B54A32D192ED03ULL +
                     i * 0x8CB92BA72F3D8DD7ULL + 0x632BE59BD9B4E019ULL);
}

void ora_synth_thresholds(uint64_t seed, int64_t j, double maf_lo, double maf_hi,
                          double missing, uint32_t thr[3]) {
    const uint64_t h = ora_key(seed, (uint64_t)j, 0xFFFFFFFFFFFFULL);
    const double unit = (double)(h >> 11) * (1.0 / 9007199254740992.0);
    const double f = maf_lo + (maf_hi - maf_lo) * unit;
    const double q = 1.0 - f;
    const double p0 = q * q;
    const double p1 = p0 + 2.0 * f * q;
    const double scale = 4294967296.0;
    double t0 = floor(p0 * scale), t1 = floor(p1 * scale), tm = floor(missing * scale);
    thr[0] = t0 >= scale ? 0xFFFFFFFFu : (uint32_t)t0;
    thr[1] = t1 >= scale ? 0xFFFFFFFFu : (uint32_t)t1;
    thr[2] = tm >= scale ? 0xFFFFFFFFu : (uint32_t)tm;
}

void ora_synth(uint64_t seed, int64_t n, int64_t j0, int64_t p_count, double maf_lo,
               double maf_hi, double missing, uint8_t *out) {
    const int64_t nb = (n + 3) / 4;
#pragma omp parallel for schedule(static)
    for (int64_t jj = 0; jj < p_count; ++jj) {
        const int64_t j = j0 + jj;
        uint32_t thr[3];
        ora_synth_thresholds(seed, j, maf_lo, maf_hi, missing, thr);
        uint8_t *col = out + jj * nb;
        for (int64_t b = 0; b < nb; ++b) {
            int byte = 0;
            for (int s = 0; s < 4; ++s) {
                const int64_t i = 4 * b + s;
                if (i >= n) break;
                const uint64_t h = ora_key(seed, (uint64_t)j, (uint64_t)i);
                const uint32_t ud = (uint32_t)h, um = (uint32_t)(h >> 32);
                int code = ud < thr[0] ? 0 : (ud < thr[1] ? 2 : 3);
                if (um < thr[2]) code = 1;
                byte |= code << (2 * s);
            }
            col[b] = (uint8_t)byte;
        }
    }
}
