// X^T r over the swizzled packed-genotype tiles (the north-star kernel).
//
// Reference: _aty_kernel geno_matrix.py:142-165, reached through
// PackedGenotypeMatrix.aty_genetic :351-364 and aty :570-575.
//   out_j = scale * v_j * (t_j - u_j * (sum_r - m_j)),
//   t_j = sum_i dose_ij r_i,  m_j = sum_{i missing} r_i.
//
// Two kernels:
//
// aty_fast_kernel  (the IHT loop's gradient; HBM-bound target)
//   Per 512-sample tile the CTA builds a lookup table in shared memory,
//     T[pos][b] = sum_{s<4} dose(code_s(b)) * rt[4 pos + s]        (fp32)
//   for every byte value b at each of the 128 byte positions (128 KiB), where
//   rt = fp32(r - mean(r)) is the centred residual.  Each packed byte then
//   costs one PRMT (byte -> table address), one LDS and one FADD: 0.75
//   instructions per genotype, no decode arithmetic.  Lane L owns SNP L of a
//   32-SNP group and at step q reads word L^q, so the 32 lanes always hit 32
//   distinct table positions = 32 distinct banks.  The missing-genotype sum
//   m_j reuses the same table: mapping missing codes (01) to het (10) and the
//   rest to 00 makes T[b'] = sum of r over the missing slots.
//   Blocks of the matrix (4 KiB = 32 SNPs x 512 samples) stream through one
//   private shared-memory slot per warp: each of the 12 warps walks its own
//   groups, lane 0 re-issues the next cp.async.bulk (TMA bulk copy, mbarrier
//   complete_tx) as soon as the warp has copied the block to registers (after
//   a proxy fence).  Per (SNP, tile) partial sums are fp32, summed pairwise in
//   an order that does not depend on the lane (process_group), and promoted to
//   an fp64 accumulator per tile: identical SNP columns get identical
//   gradients (the reference's exact ties), and the error is <= ~6e-7 of
//   rms(g) -- inside the north star's 1e-6 on beta/loss (SURVEY.md section
//   0.4: supports are stable up to 1e-5).  Because
//   r is centred, t and u*sum_r do not cancel catastrophically; the constant
//   part mean(r) contributes v_j * mean(r) * (s1_j - u_j cnt_j) = 0 exactly.
//
// aty_exact_kernel (operator-protocol path; bit-identical to the reference)
//   Same per-byte fp64 arithmetic and byte order as _aty_kernel: per byte
//   ((d0 r0 + d1 r1) + d2 r2) + d3 r3 added to t in sample order, likewise m.
//   The caller passes the reference's own sum_r (numpy pairwise r.sum()).
#include <stdlib.h>

#include <mutex>

#include "common.cuh"

namespace gi {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
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

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}


// ------------------------------------------------------------------ fast kernel
constexpr int kWarps = 12;          // consumer warps; each streams its own groups
constexpr int kThreads = kWarps * 32;
constexpr int kSlots = 1;           // private TMA ring slots per warp
constexpr int kMaxGroups = 112;     // groups per work item (fp64 accumulators in smem)
constexpr int kTableBytes = 256 * 128 * 4;
constexpr int kMiscBytes = kMaxGroups * 32 * 8 + kWarps * kSlots * 8 + kMaxGroups;
constexpr int kRingBytes = kWarps * kSlots * GI_BLOCK_BYTES;
constexpr int kSmemFast = 232448;   // the sm_100 per-block maximum (227 KiB)

struct FastArgs {
  MatrixDesc m;
  const uint8_t* group_missing;
  const float* rt;
  const double* u;
  const double* v;
  const int32_t* s1cnt;  // per-SNP (sum of dosages, observed count) over the view's rows
  const double* scal;    // [1] = mean of r used for centring, [2] = sum of rt
  double scale;
  double* out;
  int64_t n_items;        // n_chunks x n_slices
  int64_t n_slices;       // tile slices per group chunk (1: an item covers every tile)
  double* part;           // n_slices > 1: per-slice partial sums, [slice][G * 32]
  unsigned int* cticket;  // n_slices > 1: per-chunk arrival counters (zero between launches)
  unsigned long long* gmax;  // optional: atomicMax of |out_j| (bits of a non-negative double)
  // optional: the last CTA to finish copies these segments (gradient entries
  // included, read through L2) into pub_out -- mapped host memory of the
  // native loop -- so the refresh needs no separate publish launch
  PubArgs pub;
  unsigned int* pub_ticket;
  unsigned long long* pub_out;
  // base-3 copy of a matrix with missing genotypes: out[j] holds m_j (from
  // missum_kernel, missing.cu) when the epilogue reads it
  bool miss_in_out;
};

__device__ __forceinline__ float dose_term(int code, float r) {
  // dose(code) * r with dose = 0, 0, 1, 2 for codes 0..3 (exact in fp32)
  return code == 2 ? r : (code == 3 ? 2.0f * r : 0.0f);
}

template <int kOff>
__device__ __forceinline__ float lds_f32_off(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(kOff));
  return v;
}

template <int kOff>
__device__ __forceinline__ uint32_t lds_u32_off(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(kOff));
  return v;
}

__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// Table build: all 384 threads.  Thread (w = lane, k = byte within word,
// third) writes the entries T[pos = 4w + k][b] whose high nibble b >> 4 falls in
// its third of [0, 16) (6, 5 and 5 nibbles) at shared byte address
//   tbl + (k >> 1) * 65536 + b * 256 + (k & 1) * 128 + 4 w,
// from the four residuals of samples 16w + 4k .. +3 of the tile.
__device__ __forceinline__ float4 load_tile_r(const float* __restrict__ rt, int64_t t, int tid) {
  const int w = tid & 31;
  const int k = (tid >> 5) & 3;
  return *reinterpret_cast<const float4*>(rt + t * GI_TILE_SAMPLES + 16 * w + 4 * k);
}

__device__ __forceinline__ void build_table(uint32_t tbl, float4 r, int tid) {
  const int w = tid & 31;
  const int k = (tid >> 5) & 3;
  const int third = tid >> 7;
  const int hi0 = third == 0 ? 0 : (third == 1 ? 6 : 11);
  const int hi1 = third == 0 ? 6 : (third == 1 ? 11 : 16);
  float lo[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) lo[c] = dose_term(c & 3, r.x) + dose_term(c >> 2, r.y);
  const uint32_t base = tbl + (k >> 1) * 65536 + (k & 1) * 128 + 4 * w;
#pragma unroll
  for (int hh = 0; hh < 6; ++hh) {
    const int hi = hi0 + hh;
    if (hi < hi1) {
      const float hv = dose_term(hi & 3, r.z) + dose_term(hi >> 2, r.w);
#pragma unroll
      for (int c = 0; c < 16; ++c) sts_f32(base + (hi * 16 + c) * 256, lo[c] + hv);
    }
  }
}

// Base-3 tiles (missing-free matrices, csrc/layout.cu pack3_kernel): byte
// k of word w of a 640-sample tile packs samples 20 w + 5 k + s, s < 5, as
// sum_s dose_s 3^s.  Same table geometry (position 4 w + k, 256-byte row per
// byte value, 243 rows used), so the lookup loop is unchanged; each entry is
//   ((d0 r0 + d1 r1) + d2 r2) + (d3 r3 + d4 r4)
// from 27 low and 9 high partial sums (one add per entry).
struct R5 {
  float r[5];
};

__device__ __forceinline__ R5 load_tile_r3(const float* __restrict__ rt, int64_t t, int tid,
                                           int64_t n) {
  const int w = tid & 31;
  const int k = (tid >> 5) & 3;
  const int64_t i0 = t * GI_TILE3_SAMPLES + 20 * w + 5 * k;
  R5 v;
#pragma unroll
  for (int s = 0; s < 5; ++s) v.r[s] = i0 + s < n ? rt[i0 + s] : 0.0f;
  return v;
}

__device__ __forceinline__ float digit_term(int d, float r) {
  return d == 1 ? r : (d == 2 ? 2.0f * r : 0.0f);  // exact in fp32
}

__device__ __forceinline__ void build_table3(uint32_t tbl, const R5& r, int tid) {
  const int w = tid & 31;
  const int k = (tid >> 5) & 3;
  const int third = tid >> 7;  // high digit pairs 3 third .. 3 third + 2
  float lo[27];
#pragma unroll
  for (int c = 0; c < 27; ++c)
    lo[c] = (digit_term(c % 3, r.r[0]) + digit_term((c / 3) % 3, r.r[1])) +
            digit_term(c / 9, r.r[2]);
  const uint32_t base = tbl + (k >> 1) * 65536 + (k & 1) * 128 + 4 * w;
#pragma unroll
  for (int hh = 0; hh < 3; ++hh) {
    const int hi = third * 3 + hh;
    const float hv = digit_term(hi % 3, r.r[3]) + digit_term(hi / 3, r.r[4]);
#pragma unroll
    for (int c = 0; c < 27; ++c) sts_f32(base + (hi * 27 + c) * 256, lo[c] + hv);
  }
}

__device__ __forceinline__ void stage_group(uint32_t slot_lane, uint32_t (&wd)[32]) {
#pragma unroll
  for (int q = 0; q < 32; ++q) wd[q] = lds_u32_off<0>(slot_lane + q * 128);
}

// One 32-SNP group x 512-sample tile.  `xb` = 4 * lane | (table base >> 8):
// __byte_perm(word, xb ^ 4q, 0x65k4) is then the complete shared address of
// T[position 4 (lane ^ q) + k][byte k of word] -- one PRMT per packed byte.
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}

__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));  // FADD2: two fp32 adds
  return r;
}

__device__ __forceinline__ float lo_of(uint64_t x) {
  return __uint_as_float((uint32_t)x);
}

__device__ __forceinline__ float hi_of(uint64_t x) {
  return __uint_as_float((uint32_t)(x >> 32));
}

// Lane-order-free summation.  Lane L visits word w = L ^ q at step q, so two
// identical SNP columns in different lanes see the same words in different
// orders.  Each word's sum is formed in a fixed byte order, (e0 + e1) +
// (e2 + e3), and the 32 word sums are combined pairwise over aligned blocks of
// q -- which are aligned blocks of w for every L -- so every addition of the
// tree adds the same two values for any lane, at most swapped (IEEE addition
// is commutative).  Identical columns therefore get identical sums (the
// reference's exact ties, broken by index), and pairwise summation is also
// more accurate than running chains.  `st` is a binary-counter stack of the
// aligned 2-, 4-, 8- and 16-word block sums.
template <typename V, typename Add>
__device__ __forceinline__ void tree_push(int j, V b, V (&st)[4], V& total, Add add) {
  if ((j & 1) == 0) { st[0] = b; return; }
  b = add(st[0], b);
  if ((j & 2) == 0) { st[1] = b; return; }
  b = add(st[1], b);
  if ((j & 4) == 0) { st[2] = b; return; }
  b = add(st[2], b);
  if ((j & 8) == 0) { st[3] = b; return; }
  total = add(st[3], b);
}

template <bool kMissing>
__device__ __forceinline__ void process_group(const uint32_t (&wd)[32], uint32_t xb,
                                              float& tile_t, float& tile_m) {
  if (!kMissing) {
    float st[4], total = 0.f;
#pragma unroll
    for (int q = 0; q < 32; q += 2) {  // words q and q + 1 side by side in FADD2 lanes
      const uint32_t x = xb ^ (uint32_t)(q << 2), y = xb ^ (uint32_t)((q + 1) << 2);
      const float e0 = lds_f32_off<0>(__byte_perm(wd[q], x, 0x6504));
      const float e1 = lds_f32_off<128>(__byte_perm(wd[q], x, 0x6514));
      const float e2 = lds_f32_off<65536>(__byte_perm(wd[q], x, 0x6524));
      const float e3 = lds_f32_off<65536 + 128>(__byte_perm(wd[q], x, 0x6534));
      const float g0 = lds_f32_off<0>(__byte_perm(wd[q + 1], y, 0x6504));
      const float g1 = lds_f32_off<128>(__byte_perm(wd[q + 1], y, 0x6514));
      const float g2 = lds_f32_off<65536>(__byte_perm(wd[q + 1], y, 0x6524));
      const float g3 = lds_f32_off<65536 + 128>(__byte_perm(wd[q + 1], y, 0x6534));
      const uint64_t p01 = fadd2(pack2(e0, g0), pack2(e1, g1));  // (e0 + e1, g0 + g1)
      const uint64_t p23 = fadd2(pack2(e2, g2), pack2(e3, g3));  // (e2 + e3, g2 + g3)
      const uint64_t ws = fadd2(p01, p23);                       // (word q, word q + 1)
      tree_push(q >> 1, lo_of(ws) + hi_of(ws), st, total,
                [](float a, float b) { return a + b; });
    }
    tile_t = total;
    tile_m = 0.f;
  } else {
    uint64_t st[4], total = 0;  // (dose sum, missing sum) pairs
#pragma unroll
    for (int q = 0; q < 32; q += 2) {
      uint64_t w2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t wq = wd[q + h];
        const uint32_t x = xb ^ (uint32_t)((q + h) << 2);
        const uint32_t mm = (wq << 1) & ~wq & 0xAAAAAAAAu;  // missing (01) -> het (10)
        const float e0 = lds_f32_off<0>(__byte_perm(wq, x, 0x6504));
        const float e1 = lds_f32_off<128>(__byte_perm(wq, x, 0x6514));
        const float e2 = lds_f32_off<65536>(__byte_perm(wq, x, 0x6524));
        const float e3 = lds_f32_off<65536 + 128>(__byte_perm(wq, x, 0x6534));
        const float f0 = lds_f32_off<0>(__byte_perm(mm, x, 0x6504));
        const float f1 = lds_f32_off<128>(__byte_perm(mm, x, 0x6514));
        const float f2 = lds_f32_off<65536>(__byte_perm(mm, x, 0x6524));
        const float f3 = lds_f32_off<65536 + 128>(__byte_perm(mm, x, 0x6534));
        const uint64_t pe = fadd2(pack2(e0, e2), pack2(e1, e3));  // (e0 + e1, e2 + e3)
        const uint64_t pf = fadd2(pack2(f0, f2), pack2(f1, f3));
        w2[h] = fadd2(pack2(lo_of(pe), lo_of(pf)), pack2(hi_of(pe), hi_of(pf)));
      }
      tree_push(q >> 1, fadd2(w2[0], w2[1]), st, total,
                [](uint64_t a, uint64_t b) { return fadd2(a, b); });
    }
    tile_t = lo_of(total);
    tile_m = hi_of(total);
  }
}

// A warp's stream of blocks: for tile t = 0..T-1, its groups gl = warp,
// warp + 8, ... < ng.  Walked by both the copy issuer and the consumer.
struct BlockCursor {
  uint32_t gl, first, ng;
  int64_t t, T;
  __device__ bool valid() const { return t < T; }
  __device__ void next() {
    gl += kWarps;
    if (gl >= ng) {
      gl = first;
      ++t;
    }
  }
};

template <bool kBase3>
__global__ void __launch_bounds__(kThreads, 1) aty_fast_kernel(FastArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // Carve shared memory so that the table starts on a 64 KiB boundary of the
  // shared window (its address bits 16+ then come straight out of the PRMT);
  // the ring slots and the accumulators go in the space left on either side.
  const uint32_t sbase = smem_u32(smem);
  const uint32_t tbl_off = (0u - sbase) & 0xFFFFu;
  const uint32_t tbl = sbase + tbl_off;
  const uint32_t hi_off = tbl_off + kTableBytes;
  // region list: [0, tbl_off) and [hi_off, kSmemFast)
  uint32_t misc_off;
  uint32_t ring_lo_off, ring_lo_n, ring_hi_off, ring_hi_n;
  {
    const uint32_t lo_size = tbl_off, hi_size = (uint32_t)kSmemFast - hi_off;
    uint32_t lo_free = lo_size, hi_free = hi_size, lo_cur = 0, hi_cur = hi_off;
    if (hi_free >= (uint32_t)kMiscBytes) {
      misc_off = hi_cur;
      hi_cur += kMiscBytes;
      hi_free -= kMiscBytes;
    } else {
      misc_off = lo_cur;
      lo_cur += kMiscBytes;
      lo_free -= kMiscBytes;
    }
    ring_lo_off = (lo_cur + 127u) & ~127u;
    ring_lo_n = lo_size > ring_lo_off ? (lo_size - ring_lo_off) / GI_BLOCK_BYTES : 0;
    ring_hi_off = (hi_cur + 127u) & ~127u;
    ring_hi_n = (uint32_t)kSmemFast > ring_hi_off ? ((uint32_t)kSmemFast - ring_hi_off) / GI_BLOCK_BYTES
                                                   : 0;
    (void)lo_free;
    (void)hi_free;
  }
  if (ring_lo_n + ring_hi_n < (uint32_t)(kWarps * kSlots)) __trap();  // never on sm_100
  double* acc = reinterpret_cast<double*>(smem + misc_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + misc_off + kMaxGroups * 32 * 8);
  uint8_t* gflag = reinterpret_cast<uint8_t*>(bars + kWarps * kSlots);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  const MatrixDesc& m = a.m;
  const uint8_t* const xsrc = kBase3 ? m.x3 : m.x;
  const int64_t mT = kBase3 ? m.T3 : m.T;

  // this warp's slots (global slot id = warp * kSlots + s)
  uint32_t slot_addr[kSlots];
#pragma unroll
  for (int s2 = 0; s2 < kSlots; ++s2) {
    const uint32_t id = warp * kSlots + s2;
    slot_addr[s2] = sbase + (id < ring_lo_n ? ring_lo_off + id * GI_BLOCK_BYTES
                                            : ring_hi_off + (id - ring_lo_n) * GI_BLOCK_BYTES);
  }
  const uint32_t bar0 = smem_u32(bars + warp * kSlots);
  if (lane == 0) {
#pragma unroll
    for (int s2 = 0; s2 < kSlots; ++s2) mbar_init(bar0 + 8 * s2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint32_t xb = ((uint32_t)lane << 2) | ((tbl >> 16) << 8);
  const int64_t tile_stride = m.G * (int64_t)GI_BLOCK_BYTES;
  uint32_t uses[kSlots];  // completed-phase counters of this warp's slots
#pragma unroll
  for (int s2 = 0; s2 < kSlots; ++s2) uses[s2] = 0;

  for (int64_t item = blockIdx.x; item < a.n_items; item += gridDim.x) {
    // item = (chunk of SNP groups, slice of sample tiles)
    const int64_t S = a.n_slices, C = a.n_items / S;
    const int64_t chunk = item / S, slice = item - chunk * S;
    const int64_t g0 = chunk * m.G / C;
    const int64_t g1 = (chunk + 1) * m.G / C;
    const int64_t t0 = slice * mT / S, t1 = (slice + 1) * mT / S;
    const uint32_t ng = (uint32_t)(g1 - g0);
    const uint8_t* xitem = xsrc + block_offset(0, g0, m.G);
    const bool has_work = (uint32_t)warp < ng;
    GI_ASSERT(ng <= (uint32_t)kMaxGroups && g1 <= m.G);

    // copy issuer: lane 0 keeps kSlots blocks of this warp's stream in flight
    BlockCursor issue{(uint32_t)warp, (uint32_t)warp, ng, t0, t1};
    int next_slot = 0;
    auto issue_one = [&]() {
      if (issue.valid()) {
        if (lane == 0) {
          const uint32_t bar = bar0 + 8 * next_slot;
          mbar_expect_tx(bar, GI_BLOCK_BYTES);
          GI_ASSERT(issue.t < mT && issue.gl < ng);
          bulk_g2s(slot_addr[next_slot],
                   xitem + issue.t * tile_stride + (int64_t)issue.gl * GI_BLOCK_BYTES,
                   GI_BLOCK_BYTES, bar);
        }
        issue.next();
      }
      next_slot = next_slot + 1 == kSlots ? 0 : next_slot + 1;
    };
    if (has_work) {
#pragma unroll
      for (int s2 = 0; s2 < kSlots; ++s2) issue_one();
    }
    int cur_slot = 0;

    for (uint32_t gl = warp; gl < ng; gl += kWarps) acc[gl * 32 + lane] = 0.0;
    if (!kBase3)
      for (uint32_t gl = tid; gl < ng; gl += kThreads) gflag[gl] = a.group_missing[g0 + gl];
    float4 r_next;
    R5 r5_next;
    if constexpr (kBase3)
      r5_next = load_tile_r3(a.rt, t0, tid, m.n);
    else
      r_next = load_tile_r(a.rt, t0, tid);
    for (int64_t t = t0; t < t1; ++t) {
      __syncthreads();  // previous tile's lookups are done
      if constexpr (kBase3) {
        build_table3(tbl, r5_next, tid);
        if (t + 1 < t1) r5_next = load_tile_r3(a.rt, t + 1, tid, m.n);  // hidden behind the tile
      } else {
        build_table(tbl, r_next, tid);
        if (t + 1 < t1) r_next = load_tile_r(a.rt, t + 1, tid);
      }
      __syncthreads();
      for (uint32_t gl = warp; gl < ng; gl += kWarps) {
        // u_j for the missing-sum term, loaded before the block wait and the
        // lookups so its latency is hidden (issued after them it stalled the
        // warp on the epilogue's DFMA: ~10% of the samples at 2% missing)
        const bool miss = !kBase3 && gflag[gl] != 0;
        double uj = 0.0;
        if (miss) {
          const int64_t j = (g0 + gl) * 32 + lane;
          if (j < m.p) uj = __ldg(a.u + j);
        }
        // wait for this slot's next phase (strictly in order: never ambiguous)
        uint32_t u0 = 0;
#pragma unroll
        for (int s2 = 0; s2 < kSlots; ++s2)
          if (s2 == cur_slot) u0 = uses[s2];
        mbar_wait(bar0 + 8 * cur_slot, u0 & 1);
        GI_ASSERT(gl < ng && t < t1);
        uint32_t wd[32];
        uint32_t sa = 0;
#pragma unroll
        for (int s2 = 0; s2 < kSlots; ++s2)
          if (s2 == cur_slot) sa = slot_addr[s2];
        stage_group(sa + lane * 4, wd);
#pragma unroll
        for (int s2 = 0; s2 < kSlots; ++s2)
          if (s2 == cur_slot) ++uses[s2];
        // the slot's generic-proxy reads above must be ordered before the
        // async-proxy (TMA) write that refills it: proxy fence per lane, then
        // the warp barrier, then lane 0 issues
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        next_slot = cur_slot;
        issue_one();  // refill the slot just drained
        cur_slot = cur_slot + 1 == kSlots ? 0 : cur_slot + 1;
        float tt = 0.f, tm = 0.f;
        if (miss)
          process_group<true>(wd, xb, tt, tm);
        else
          process_group<false>(wd, xb, tt, tm);
        double add = (double)tt;
        if (miss) add += uj * (double)tm;
        acc[gl * 32 + lane] += add;
      }
    }
    // Tile slices: every slice stores its partial sums; the last slice of the
    // chunk to arrive adds them in slice order (the same for every column, so
    // identical columns still get identical bits) and runs the epilogue.
    bool epilogue = true;
    if (S > 1) {
      const int64_t stride = m.G * 32;
      for (uint32_t gl = warp; gl < ng; gl += kWarps)
        a.part[slice * stride + (g0 + gl) * 32 + lane] = acc[gl * 32 + lane];
      __threadfence();
      __syncthreads();
      int last = 0;
      if (tid == 0) last = atomicAdd(a.cticket + chunk, 1u) == (unsigned)(S - 1);
      epilogue = __syncthreads_or(last);
      if (epilogue) {
        __threadfence();
        for (uint32_t gl = warp; gl < ng; gl += kWarps) {
          double sum = 0.0;
          for (int64_t s2 = 0; s2 < S; ++s2)
            sum += __ldcg(a.part + s2 * stride + (g0 + gl) * 32 + lane);
          acc[gl * 32 + lane] = sum;
        }
        if (tid == 0) a.cticket[chunk] = 0u;
      }
    }
    if (epilogue) {
    // epilogue: out_j = scale * v_j * (acc_j - u_j * sum_rt + mean * (s1_j - u_j cnt_j));
    // the last term restores the constant part of r removed by centring (zero
    // up to rounding when u_j is the mean over the same rows; not for
    // caller-supplied stats such as with_stats / global-standardised folds)
    const double mean = a.scal[1], srt = a.scal[2];
    double local_max = 0.0;
    for (uint32_t gl = warp; gl < ng; gl += kWarps) {
      const int64_t j = (g0 + gl) * 32 + lane;
      if (j < m.p) {
        const double uj = a.u[j];
        const double off = (double)a.s1cnt[2 * j] - uj * (double)a.s1cnt[2 * j + 1];
        double t = acc[gl * 32 + lane];
        if (a.miss_in_out) t += uj * a.out[j];  // + u_j m_j, as the 2-bit kernel per tile
        const double val = a.v[j] * ((t - uj * srt) + mean * off);
        a.out[j] = a.scale * val;
        local_max = fmax(local_max, fabs(val));
      }
    }
    if (a.gmax) {
      // max|g| for the IHT step (iht.py:257-261): exact and order-independent
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        local_max = fmax(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
      if (lane == 0)
        atomicMax(a.gmax, (unsigned long long)__double_as_longlong(local_max));
    }
    }  // epilogue
    __syncthreads();  // accumulators, flags and table are reused by the next item
  }
  if (a.pub_ticket) {
    // no static shared memory here (the dynamic carve-out is the maximum):
    // thread 0 takes the ticket, __syncthreads_or broadcasts "last CTA"
    __threadfence();
    __syncthreads();
    int last = 0;
    if (tid == 0) last = atomicAdd(a.pub_ticket, 1u) == gridDim.x - 1;
    if (__syncthreads_or(last)) {
      __threadfence();
      for (int q = 0; q < a.pub.nseg; ++q) {
        const PubSeg sg = a.pub.seg[q];
        const unsigned long long* src = static_cast<const unsigned long long*>(sg.src);
        for (int64_t e = tid; e < sg.count; e += blockDim.x)
          a.pub_out[sg.dst + e] = __ldcg(sg.idx ? src + sg.idx[e] : src + e);
      }
      if (tid == 0) *a.pub_ticket = 0u;
    }
  }
}

// Work decomposition of aty_fast_kernel: `chunks` ranges of at most kMaxGroups
// SNP groups times `slices` ranges of sample tiles.  Each (item, tile) builds
// a 128 KiB table, so items should be as wide in groups as the accumulators
// allow; when p is small (few groups per SM) the tiles are split instead.
// Chosen to minimise the modelled per-SM LSU work: per item and tile, 20 KiB
// per group (4 KiB staged + 16 KiB of table reads) plus the 128 KiB build,
// times the rounds of items over the SMs.  With `sliced` false (no partial
// buffer) only single-slice plans are considered.
void aty_fast_plan(const MatrixDesc& m, int num_sms, bool sliced, int64_t& chunks,
                   int64_t& slices) {
  const int64_t G = m.G, T = m.T, sms = num_sms;
  chunks = 1;
  slices = 1;
  if (G <= 0 || T <= 0 || sms <= 0) return;  // nothing to sweep (an empty shard)
  auto cost = [&](int64_t c, int64_t s) {
    const int64_t rounds = (c * s + sms - 1) / sms;
    const int64_t tiles = (T + s - 1) / s;
    const int64_t groups = (G + c - 1) / c;
    return (double)rounds * (double)tiles * (20.0 * (double)groups + 128.0);
  };
  const int64_t per_wave = sms * kMaxGroups;
  chunks = sms * ((G + per_wave - 1) / per_wave);
  if (chunks > G) chunks = G;
  if (chunks < 1) chunks = 1;
  slices = 1;
  if (!sliced || G >= per_wave) return;
  double best = cost(chunks, 1);
  const int64_t cmin = (G + kMaxGroups - 1) / kMaxGroups;
  for (int64_t s2 = 2; s2 <= T && s2 <= 64; ++s2) {
    const int64_t cands[3] = {cmin, sms / s2, (sms + s2 - 1) / s2};
    for (int64_t c : cands) {
      if (c < 1 || c < cmin || c > G || c * s2 > 2 * sms) continue;
      const double v = cost(c, s2);
      if (v < best) {
        best = v;
        chunks = c;
        slices = s2;
      }
    }
  }
}

// The plan of the tiles the kernel streams: the base-3 copy's when present.
static MatrixDesc plan_desc(const MatrixDesc& m) {
  MatrixDesc pm = m;
  if (m.x3 != nullptr) pm.T = m.T3;
  return pm;
}

// Sized for either layout (fit workspaces are shared by matrices of one shape).
int64_t aty_fast_part_doubles(const MatrixDesc& m, int num_sms) {
  int64_t c = 0, s2 = 1, best = 0;
  aty_fast_plan(m, num_sms, true, c, s2);
  if (s2 > 1) best = s2 * m.G * 32;
  MatrixDesc m3 = m;
  m3.T = tiles3_of(m.n);
  aty_fast_plan(m3, num_sms, true, c, s2);
  if (s2 > 1 && s2 * m.G * 32 > best) best = s2 * m.G * 32;
  return best;
}

int launch_aty_fast(const MatrixDesc& m, const uint8_t* group_missing, const float* rt,
                    const double* u, const double* v, const int32_t* s1cnt,
                    const double* d_scal, double scale, double* out, int num_sms,
                    cudaStream_t s, double* d_gmax, const PubArgs* pub,
                    unsigned int* pub_ticket, void* pub_out, double* part,
                    unsigned int* cticket) {
  if (m.p == 0) return 0;

  static std::once_flag once;
  static cudaError_t cfg_err = cudaSuccess;
  std::call_once(once, [] {
    cfg_err = cudaFuncSetAttribute(aty_fast_kernel<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemFast);
    if (cfg_err == cudaSuccess)
      cfg_err = cudaFuncSetAttribute(aty_fast_kernel<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemFast);
  });
  GI_CUDA_TRY(cfg_err);
  FastArgs a;
  a.m = m;
  a.group_missing = group_missing;
  a.rt = rt;
  a.u = u;
  a.v = v;
  a.s1cnt = s1cnt;
  a.scal = d_scal;
  a.scale = scale;
  a.out = out;
  a.gmax = reinterpret_cast<unsigned long long*>(d_gmax);
  a.miss_in_out = m.x3 != nullptr && m.mlist != nullptr;
  if (a.miss_in_out && launch_missum(m, rt, out, num_sms, s) != 0) return -1;
  if (pub && pub_ticket && pub_out) {
    a.pub = *pub;
    a.pub_ticket = pub_ticket;
    a.pub_out = static_cast<unsigned long long*>(pub_out);
  } else {
    a.pub_ticket = nullptr;
    a.pub_out = nullptr;
  }
  int64_t chunks = 0, slices = 1;
  aty_fast_plan(plan_desc(m), num_sms, part != nullptr, chunks, slices);
  if (slices > 1) {
    if (!part || !cticket) {
      gi_set_error("internal: sliced X^T r plan without its partial buffer");
      return -1;
    }
    a.part = part;
    a.cticket = cticket;
  } else {
    a.part = nullptr;
    a.cticket = nullptr;
  }
  a.n_slices = slices;
  const int64_t items = chunks * slices;
  a.n_items = items;
  const int grid = (int)(items < num_sms ? items : num_sms);
  if (m.x3 != nullptr)
    aty_fast_kernel<true><<<grid, kThreads, kSmemFast, s>>>(a);
  else
    aty_fast_kernel<false><<<grid, kThreads, kSmemFast, s>>>(a);
  GI_LAUNCH_CHECK();
  return 0;
}

// ------------------------------------------------------------------ exact kernel
// One warp per SNP group, lane = SNP; the group's 4 KiB block is staged in
// shared memory with coalesced loads, then each lane walks its own words in
// natural sample order (bank = lane, conflict-free) and the r tile is read as
// a warp-wide broadcast.
constexpr int kExactWarps = 8;

__global__ void __launch_bounds__(kExactWarps * 32) aty_exact_kernel(
    MatrixDesc m, const double* __restrict__ r_pad, const double* __restrict__ u,
    const double* __restrict__ v, const double* __restrict__ sum_r, double scale,
    double* __restrict__ out, unsigned long long* gmax, PubArgs pub, unsigned int* pub_ticket,
    unsigned long long* pub_out) {
  __shared__ double rs[GI_TILE_SAMPLES];
  __shared__ __align__(16) uint8_t blk[kExactWarps][GI_BLOCK_BYTES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * kExactWarps + warp;
  const bool active = g < m.G;
  double t = 0.0, mm = 0.0;
  const int64_t n_pad = m.T * GI_TILE_SAMPLES;
  for (int64_t tt = 0; tt < m.T; ++tt) {
    __syncthreads();
    for (int i = threadIdx.x; i < GI_TILE_SAMPLES; i += blockDim.x) {
      const int64_t s = tt * GI_TILE_SAMPLES + i;
      rs[i] = s < n_pad ? r_pad[s] : 0.0;
    }
    if (active) {
      const uint4* src = reinterpret_cast<const uint4*>(m.x + block_offset(tt, g, m.G));
      uint4* dst = reinterpret_cast<uint4*>(blk[warp]);
#pragma unroll
      for (int k = 0; k < 8; ++k) dst[k * 32 + lane] = src[k * 32 + lane];
    }
    __syncthreads();
    if (!active) continue;
    for (int w = 0; w < 32; ++w) {
      const uint32_t wd =
          *reinterpret_cast<const uint32_t*>(blk[warp] + ((lane ^ w) << 7) + (lane << 2));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double* rr = rs + 16 * w + 4 * k;
        double bt = 0.0, bm = 0.0;
#pragma unroll
        for (int sl = 0; sl < 4; ++sl) {
          const uint32_t code = (wd >> (8 * k + 2 * sl)) & 3u;
          const double d = code == 2u ? 1.0 : (code == 3u ? 2.0 : 0.0);
          const double ms = code == 1u ? 1.0 : 0.0;
          const double pt = __dmul_rn(d, rr[sl]);
          const double pm = __dmul_rn(ms, rr[sl]);
          bt = sl == 0 ? pt : __dadd_rn(bt, pt);
          bm = sl == 0 ? pm : __dadd_rn(bm, pm);
        }
        t = __dadd_rn(t, bt);
        mm = __dadd_rn(mm, bm);
      }
    }
  }
  double local_max = 0.0;
  const int64_t j = g * 32 + lane;
  if (active && j < m.p) {
    const double val = __dmul_rn(v[j], __dsub_rn(t, __dmul_rn(u[j], __dsub_rn(*sum_r, mm))));
    out[j] = __dmul_rn(scale, val);
    local_max = fabs(val);
  }
  // optional fused epilogues, as in aty_fast_kernel: max|g| (exact,
  // order-independent) and the last CTA's publish into mapped host memory
  if (gmax) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      local_max = fmax(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
    if (lane == 0) atomicMax(gmax, (unsigned long long)__double_as_longlong(local_max));
  }
  if (pub_ticket) {
    __threadfence();
    __syncthreads();
    int last = 0;
    if (threadIdx.x == 0) last = atomicAdd(pub_ticket, 1u) == gridDim.x - 1;
    if (__syncthreads_or(last)) {
      __threadfence();
      for (int q = 0; q < pub.nseg; ++q) {
        const PubSeg sg = pub.seg[q];
        const unsigned long long* src = static_cast<const unsigned long long*>(sg.src);
        for (int64_t e = threadIdx.x; e < sg.count; e += blockDim.x)
          pub_out[sg.dst + e] = __ldcg(sg.idx ? src + sg.idx[e] : src + e);
      }
      if (threadIdx.x == 0) *pub_ticket = 0u;
    }
  }
}

// Exact gradient on the support (after a fast sweep): one block per listed
// column, fp64 sums of dose * r and missing * r over the column (thread-strided
// words, then a fixed reduction tree), g_j = scale * v_j (t_j - u_j (sum_r - m_j)) as
// _aty_kernel forms it (geno_matrix.py:165).  The step size of the next
// iteration, mu = ||g_S||^2 / ||X_S g_S||^2 (iht.py:233-244), depends on
// these entries ALONE, and right after a converged warm start they are at the
// level of the previous fit's tolerance (~1e-7 of rms(g)): the lookup-table
// kernel's ~6e-7 rms(g) error would set their direction, and a backtracking
// test within 1% of its threshold could flip (tools/cv_diag.py).  The fp64
// sums here are accurate to ~1e-16 of the column's |terms|.
constexpr int kSgWords = 1024;  // words per block (4 per thread): a column's slices
constexpr int kSgMaxSlices = 64;

__global__ void __launch_bounds__(256) support_grad_kernel(
    MatrixDesc m, const double* __restrict__ r_pad, const double* __restrict__ u,
    const double* __restrict__ v, const double* __restrict__ sum_r, double scale,
    const int64_t* __restrict__ idx, double* __restrict__ out, double* __restrict__ pub_out,
    int slices, double* __restrict__ part, unsigned int* __restrict__ tickets) {
  // block = (listed column, slice of its words); the last slice to finish
  // folds the slices' partial sums in slice order and writes g_j
  __shared__ double sh[2][8];
  __shared__ bool last;
  const int col = blockIdx.x / slices, sl = blockIdx.x - col * slices;
  const int64_t j = idx[col];
  const int64_t words = m.T * GI_TILE_WORDS;
  const int64_t w0 = (int64_t)sl * words / slices, w1 = (int64_t)(sl + 1) * words / slices;
  double t = 0.0, mm = 0.0;
  for (int64_t wg = w0 + threadIdx.x; wg < w1; wg += blockDim.x) {
    const int64_t tile = wg >> 5;
    const int w = (int)(wg & 31);
    const uint32_t wd = __ldg(reinterpret_cast<const uint32_t*>(m.x + word_offset(tile, j, w, m.G)));
    const double* rr = r_pad + tile * GI_TILE_SAMPLES + 16 * w;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t code = (wd >> (2 * i)) & 3u;
      const double ri = rr[i];
      t += code == 2u ? ri : (code == 3u ? 2.0 * ri : 0.0);
      mm += code == 1u ? ri : 0.0;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t += __shfl_xor_sync(0xffffffffu, t, o);
    mm += __shfl_xor_sync(0xffffffffu, mm, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sh[0][warp] = t;
    sh[1][warp] = mm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    t = 0.0;
    mm = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      t += sh[0][q];
      mm += sh[1][q];
    }
    part[2 * blockIdx.x] = t;
    part[2 * blockIdx.x + 1] = mm;
    __threadfence();
    last = atomicAdd(tickets + col, 1u) == (unsigned)(slices - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    t = 0.0;
    mm = 0.0;
    for (int q = 0; q < slices; ++q) {
      t += __ldcg(part + 2 * (col * slices + q));
      mm += __ldcg(part + 2 * (col * slices + q) + 1);
    }
    const double g = scale * (v[j] * (t - u[j] * (*sum_r - mm)));
    out[j] = g;
    if (pub_out) pub_out[col] = g;
    tickets[col] = 0u;
  }
}

int64_t support_grad_part_doubles(int64_t kcap, int64_t T) {
  int64_t sl = (T * GI_TILE_WORDS + kSgWords - 1) / kSgWords;
  if (sl > kSgMaxSlices) sl = kSgMaxSlices;
  return 2 * kcap * (sl < 1 ? 1 : sl);
}

int launch_support_grad(const MatrixDesc& m, const double* r_pad, const double* u,
                        const double* v, const double* d_sum_r, double scale, const int64_t* idx,
                        int64_t k, double* out, double* pub_out, double* part,
                        unsigned int* tickets, cudaStream_t s) {
  if (k <= 0 || m.p == 0) return 0;
  int64_t sl = (m.T * GI_TILE_WORDS + kSgWords - 1) / kSgWords;
  if (sl > kSgMaxSlices) sl = kSgMaxSlices;
  if (sl < 1) sl = 1;
  support_grad_kernel<<<(unsigned)(k * sl), 256, 0, s>>>(m, r_pad, u, v, d_sum_r, scale, idx, out,
                                                         pub_out, (int)sl, part, tickets);
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_aty_exact(const MatrixDesc& m, const double* r_pad, const double* u, const double* v,
                     const double* d_sum_r, double scale, double* out, cudaStream_t s,
                     double* d_gmax, const PubArgs* pub, unsigned int* pub_ticket,
                     void* pub_out) {
  if (m.p == 0) return 0;
  const int64_t blocks = (m.G + kExactWarps - 1) / kExactWarps;
  PubArgs pa;
  const bool publish = pub && pub_ticket && pub_out;
  if (publish) pa = *pub;
  aty_exact_kernel<<<(unsigned)blocks, kExactWarps * 32, 0, s>>>(
      m, r_pad, u, v, d_sum_r, scale, out, reinterpret_cast<unsigned long long*>(d_gmax), pa,
      publish ? pub_ticket : nullptr, static_cast<unsigned long long*>(pub_out));
  GI_LAUNCH_CHECK();
  return 0;
}

}  // namespace gi
