// X^T R on the 5th-generation tensor cores: exact integer sums over the 2-bit
// genotype tiles for 1..32 right-hand sides in ONE sweep of the matrix.
//
// Reference: _aty_kernel geno_matrix.py:142-165 (one residual per call; the
// CV loop model_select.py:124-139 calls it once per fold fit):
//   out_j = scale * v_j * (t_j - u_j * (sum_r - m_j)),
//   t_j = sum_i dose_ij r_i,  m_j = sum_{i missing} r_i.
//
// Formulation.  Each residual is centred and quantised to an integer,
// R_i = round((r_i - mean) / s) with |R_i| <= 2^26 (s = max|r - mean| / 2^26,
// resolution 1.5e-8 of the largest centred residual), and split into four
// balanced base-128 digits q_0..q_3 in [-64, 63], R = sum_d 128^d q_d.  Then
//   T_j = sum_i dose_ij R_i = sum_d 128^d (A_dose B_d)_j,
//   M_j = sum_{i missing} R_i = sum_d 128^d (A_miss B_d)_j
// are int8 x int8 -> int32 products on the tensor cores (tcgen05.mma
// kind::i8): A = u8 doses (0/1/2) or missing flags (0/1) of 128 SNPs, one
// TMEM lane per SNP; B = the s8 digit columns (4 per right-hand side) of a
// 128-sample chunk in shared memory.  Every partial sum is an exact integer
// (|T_j| <= 2 * 64 * n * 128^3 < 2^53), so the result is independent of the
// summation order (identical SNP columns get identical bits -- the
// reference's exact ties), and
//   out_j = scale * v_j * (s (T_j + u_j (M_j - sum_i R_i)) + mean (s1_j - u_j cnt_j))
// differs from the reference's fp64 sum only by the quantisation of r:
// ~1e-8 of rms(g), 30-60x below the lookup-table kernel (aty.cu).
//
// Data path per CTA (one per SM, persistent, two M-tile slots):
//   * 8 decode warps, 4 per slot; warp (slot, g) owns SNP group g of the
//     slot's current 128-SNP M-tile = TMEM lane quarter g.  Each streams its
//     group's 4 KiB blocks (one 512-sample tile) through two private TMA
//     slots, reads its 32 words (lane L reads word w of SNP L at row L ^ w,
//     bank L: conflict-free), and per 128-sample chunk decodes 8 words into 32
//     TMEM columns of u8 doses with one PRMT per 4 genotypes (the 2-bit codes,
//     spread into nibbles, index a 4-byte dose table in a register: code ->
//     dose 0/0/1/2, or -> missing flag 0/1/0/0), stored by tcgen05.st.
//     The K order inside a chunk is a fixed permutation of the samples; the
//     digit image B is written in the same order.
//   * ISS issuer warps per slot: issuer e issues the chunk's k-steps e,
//     e + ISS, ... (M=128, N, K=32 each) into its own accumulator, so ISS
//     MMA streams overlap (one thread issues one MMA per ~55 cycles; four
//     streams reach one per ~16, measured on the B200: tools/gpu/tc_rate.cu).
//     tcgen05.commit frees the chunk's A/B buffers and, after an M-tile's
//     last chunk, hands the accumulators to the epilogue.
//   * The decode warps run the epilogue of their M-tile: tcgen05.ld of the
//     accumulators (summed over issuers, exact), digits recombined in int64,
//     one fp64 formula per (SNP, right-hand side).
// HBM traffic per sweep: the 2-bit tiles once, plus the digit image (4 B per
// sample per RHS, L2-resident) -- for every right-hand side at once.
#include <stdlib.h>

#include <mutex>

#include "common.cuh"
#include "reduce.cuh"

namespace gi {
namespace {

constexpr int kDecWarps = 8;       // 2 slots x 4 SNP groups
constexpr int kChunkSamples = 128;  // one MMA chunk: 8 words, 32 TMEM columns, 4 k-steps
// blocks (<= 128 KiB) + digit rings (<= 128 KiB, 192 KiB together) + barriers;
// > half the SM, so one CTA per SM owns all of TMEM
constexpr int kSmemMma = 200 * 1024;
constexpr uint32_t kDoseLut = 0x02010000u;  // code 0, 1, 2, 3 -> dose 0, 0, 1, 2
// per-warp phase timers of CTA 0 (GI_MMA_PROF=1 at run time), compiled in
// only with -DGI_MMA_PROFILE: they cost issue slots in the decode loop
#ifdef GI_MMA_PROFILE
constexpr bool kMmaProfile = true;
#else
constexpr bool kMmaProfile = false;
#endif
constexpr uint32_t kMissLut = 0x00000100u;  // code 1 (missing) -> 1

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void bar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void bar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void bar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity), "r"(0x989680u)  // suspend until the phase completes (not a spin)
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

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
}

__device__ __forceinline__ void mma_i8(uint32_t d_t, uint32_t a_t, uint64_t bdesc, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n}\n" ::"r"(d_t),
      "r"(a_t), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}

// Decoding: column 4 w + s of a chunk holds, in byte b, the value for sample
//   16 w + (2b, 8 + 2b, 2b + 1, 9 + 2b)[s]        (digit_k_of_sample below).
// The four PRMT selector words of a code word: nibble b of sel[s] holds the
// code of sample (2b, 8 + 2b, 2b + 1, 9 + 2b)[s] in its low two bits and
// zeros above (five ALU ops per word).
__device__ __forceinline__ void selectors(uint32_t w, uint32_t (&sel)[4]) {
  const uint32_t E = w & 0x33333333u, O = (w >> 2) & 0x33333333u;
  sel[0] = E;
  sel[1] = E >> 16;
  sel[2] = O;
  sel[3] = O >> 16;
}

// PTX prmt (default mode): selector nibble bits 0-2 pick a byte, bit 3 would
// replicate its sign -- always 0 here.  Written in asm because __byte_perm
// ignores bit 3, so the compiler would re-mask every selector it cannot
// prove clean (an extra LOP3 per PRMT).
__device__ __forceinline__ uint32_t prmt(uint32_t lut, uint32_t hi, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(lut), "r"(hi), "r"(sel));
  return d;
}

// Four words' selectors -> 16 TMEM columns of u8 values through `lut`
// (held in a register with `hi`, an opaque zero: the table operands then stay
// shared registers instead of a copy per PRMT).
__device__ __forceinline__ void lut16(const uint32_t (&sel)[4][4], uint32_t lut, uint32_t hi,
                                      uint32_t (&o)[16]) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) o[4 * q + s2] = prmt(lut, hi, sel[q][s2]);
}

// Position k (0..127) of sample o (0..127) of a chunk in the decoded K order.
__host__ __device__ __forceinline__ int digit_k_of_sample(int o) {
  const int w = o >> 4, r = o & 15;
  int s, b;
  if ((r & 1) == 0) {
    s = r < 8 ? 0 : 1;
    b = (r & 7) >> 1;
  } else {
    s = r < 8 ? 2 : 3;
    b = ((r - 1) & 7) >> 1;
  }
  return 16 * w + 4 * s + b;
}

struct MmaArgs {
  MatrixDesc m;
  const uint8_t* gmiss;      // per group: any missing genotype
  const int8_t* qimg;        // digit image: 4T chunks x 128 N bytes
  int nrhs;
  const double* qscal;       // per RHS: scale, mean
  const long long* qsum;     // per RHS: sum of the quantised residual
  const XtrRhs* rhs;         // per RHS: stats, output, max|g|
  double scale_out;
  int64_t n_mtiles;
  long long* prof;           // optional (debug): per-warp phase cycles of CTA 0, 8 per warp
  PubArgs pub;               // optional publish by the last CTA (native IHT loop)
  unsigned int* pub_ticket;
  unsigned long long* pub_out;
};

__device__ __forceinline__ bool mtile_missing(const uint8_t* gmiss, int64_t mt, int64_t G) {
  bool any = false;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t g = 4 * mt + q;
    if (g < G && gmiss[g]) any = true;
  }
  return any;
}

template <int N, int ISS, bool MISS>
struct Cfg {
  static constexpr int kAcols = MISS ? 64 : 32;         // per A buffer: dose (+ missing)
  static constexpr int kDcols = MISS ? 2 * N : N;       // per accumulator: dose (+ missing)
  static constexpr int kDtot = 2 * ISS * kDcols;        // 2 slots x ISS accumulators
  // A buffers per slot: as many as TMEM holds (2..4), so the decode warps run
  // that many chunks ahead of the MMA completions
  static constexpr uint32_t kQBytes = 128u * N;         // digit image per chunk
  static constexpr int kRingFit = 65536 / (int)kQBytes;
  static constexpr int kRing = kRingFit < 8 ? kRingFit : 8;
  static constexpr int kNbufFit = (512 - kDtot) / (2 * kAcols);
  static constexpr int kNbufMax = kNbufFit < kRing - 2 ? kNbufFit : kRing - 2;
  static constexpr int kNbuf = (kNbufMax > 4 ? 4 : kNbufMax) & ~1;  // whole commit groups
  static_assert(kNbuf >= 2, "TMEM columns");
  static constexpr int kAtot = 2 * kNbuf * kAcols;
  static_assert(kAtot + kDtot <= 512, "TMEM columns");
  static_assert(N == 8 || (N % 16 == 0 && N <= 128), "MMA N");
  static constexpr int kThreads = (kDecWarps + 2 * ISS) * 32;
  static constexpr uint32_t kLBO = (N / 8) * 128;       // next 16 samples of K
  static constexpr uint32_t kSBO = 128;                 // next 8 digit columns
  // digit-image ring per slot (kRing <= 8 chunks, <= 64 KiB): the copy for
  // chunk i + kLead is issued when chunk i starts (its slot was freed by chunk
  // i - kNbuf), so its L2 latency hides behind kLead chunks
  static constexpr int kLead = kRing - kNbuf;
  static_assert(kLead >= 1, "digit ring");
  // an issuer commits once per kCB chunks (a commit costs ~250 cycles of the
  // issuing thread, more than an N = 8 MMA: tools/gpu/tc_lat.cu)
  // (with two A buffers a chunk's afull is published only during the next
  // chunk, after which the decode warps wait for chunk - 2: commit groups of
  // two would wait on a chunk not yet published)
  static constexpr int kCB = kNbuf >= 4 ? 2 : 1;
  // publish a chunk's A buffer one chunk late (its stores land behind the
  // next decode) only with >= 4 buffers; with 2 the delay would hold back the
  // MMAs the next buffer reuse waits for
  static constexpr bool kDefer = kNbuf >= 4;
  static_assert(kNbuf % kCB == 0 && kRing % kCB == 0, "commit groups");
  // TMA block slots per decode warp: 4 (16 KiB of prefetch per warp) when the
  // digit rings leave room, else 2
  static constexpr int kBlkSlots = (2 * kRing * (int)kQBytes) <= 65536 ? 4 : 2;
  static constexpr int kBlkBytes = kDecWarps * kBlkSlots * GI_BLOCK_BYTES;
  // kind::i8: D s32, A u8 (doses), B s8 (digits), K-major, M = 128
  static constexpr uint32_t kIdesc = (2u << 4) | (0u << 7) | (1u << 10) |
                                     ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
};

// Barriers (per slot): afull[kNbuf] (A buffer written: 4 decode warps),
// bfull[kRing] (digit chunk landed: tx), done[kRing] (chunk's MMAs complete:
// one commit per issuer; frees A buffer i % kNbuf and digit slot i % kRing),
// dfull (accumulators final), dempty (epilogue has read them).  Chunk
// counters are 32-bit: a slot runs < 2^31 chunks (4 T per M-tile).
template <int N, int ISS, bool MISS>
__global__ void __launch_bounds__(Cfg<N, ISS, MISS>::kThreads, 1) xtr_mma_kernel(MmaArgs a) {
  using C = Cfg<N, ISS, MISS>;
  constexpr int R = C::kRing, NB = C::kNbuf;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int kBlkSlots = C::kBlkSlots;
  uint8_t* blk = smem;                          // [warp][slot] 4 KiB blocks
  uint8_t* bbuf = smem + C::kBlkBytes;             // [slot][ring] digit chunks
  uint64_t* bars = reinterpret_cast<uint64_t*>(bbuf + 2 * R * C::kQBytes);
  const uint32_t b_blk = su32(bars);                    // [8 warps][kBlkSlots]
  const uint32_t b_afull = b_blk + 8 * 8 * kBlkSlots;   // [2 slots][NB]
  const uint32_t b_bfull = b_afull + 8 * 2 * NB;        // [2 slots][R]
  const uint32_t b_done = b_bfull + 8 * 2 * R;          // [2 slots][R]
  const uint32_t b_dfull = b_done + 8 * 2 * R;          // [2]
  const uint32_t b_dempty = b_dfull + 8 * 2;            // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 8 * kBlkSlots + 2 * NB + 4 * R + 4);
  // the right-hand sides' descriptors and quantiser scalars, read by every
  // epilogue: cached here instead of a dependent global load per use
  XtrRhs* s_rhs = reinterpret_cast<XtrRhs*>(
      reinterpret_cast<uint8_t*>(tmem_holder) + 16);
  double* s_q = reinterpret_cast<double*>(s_rhs + kXtrMaxRhs);  // [rhs]: scale, mean, sum
  static_assert(C::kBlkBytes + 2 * R * C::kQBytes + 8 * (8 * kBlkSlots + 2 * NB + 4 * R + 4) +
                        16 + kXtrMaxRhs * (sizeof(XtrRhs) + 3 * sizeof(double)) <=
                    kSmemMma,
                "shared memory");
  for (int q = threadIdx.x; q < a.nrhs; q += blockDim.x) {
    s_rhs[q] = a.rhs[q];
    s_q[3 * q] = a.qscal[2 * q];
    s_q[3 * q + 1] = a.qscal[2 * q + 1];
    s_q[3 * q + 2] = (double)a.qsum[q];
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_holder)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < 8 * kBlkSlots; ++i) bar_init(b_blk + 8 * i, 1);
    for (int i = 0; i < 2 * NB; ++i) bar_init(b_afull + 8 * i, 4);
    for (int i = 0; i < 2 * R; ++i) bar_init(b_bfull + 8 * i, 1);
    for (int i = 0; i < 2 * R; ++i) bar_init(b_done + 8 * i, ISS);
    for (int i = 0; i < 2; ++i) bar_init(b_dfull + 8 * i, ISS);
    for (int i = 0; i < 2; ++i) bar_init(b_dempty + 8 * i, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const MatrixDesc& m = a.m;
  const int64_t T = m.T, G = m.G;
  const uint32_t nchunks = (uint32_t)(4 * T);
  const int64_t mt_stride = 2 * (int64_t)gridDim.x;
  const int64_t tile_stride = G * (int64_t)GI_BLOCK_BYTES;

  if (warp < kDecWarps) {
    // ------------------------------------------------------------ decode warps
    const int sl = warp >> 2, gq = warp & 3;
    const uint32_t lane_base = (uint32_t)(gq * 32) << 16;
    uint32_t zero, dose_lut, miss_lut;  // opaque registers (see lut16)
    asm volatile("mov.b32 %0, 0;" : "=r"(zero));
    asm volatile("mov.b32 %0, %1;" : "=r"(dose_lut) : "n"(kDoseLut));
    asm volatile("mov.b32 %0, %1;" : "=r"(miss_lut) : "n"(kMissLut));
    const uint32_t slot0 = su32(blk + (warp * kBlkSlots) * GI_BLOCK_BYTES);
    const uint32_t myb = b_blk + 8 * (warp * kBlkSlots);
    const uint32_t ring0 = su32(bbuf + sl * R * C::kQBytes);
    // the slot's chunk sequence over all its M-tiles; the digit image repeats
    // every nchunks.  Warp gq = 0, lane 0 keeps the digit copies kLead ahead.
    const int64_t first_mt = 2 * (int64_t)blockIdx.x + sl;
    const uint32_t my_mts =
        first_mt < a.n_mtiles ? (uint32_t)((a.n_mtiles - first_mt + mt_stride - 1) / mt_stride) : 0u;
    const uint32_t total = my_mts * nchunks;
    const bool digit_lane = gq == 0 && lane == 0;
    uint32_t dk = 0, dq = 0, dr = 0;  // next digit copy: sequence position, image chunk, ring slot
    auto issue_digits = [&]() {
      if (dk < total) {
        const uint32_t bf = b_bfull + 8 * (sl * R + dr);
        bar_arrive_tx(bf, C::kQBytes);
        bulk_g2s(ring0 + dr * C::kQBytes, a.qimg + (int64_t)dq * C::kQBytes, C::kQBytes, bf);
        ++dk;
        dq = dq + 1 == nchunks ? 0u : dq + 1;
        dr = dr + 1 == (uint32_t)R ? 0u : dr + 1;
      }
    };
    if (digit_lane)
      for (int k = 0; k < C::kLead; ++k) issue_digits();
    uint32_t bt = 0;       // blocks this warp has consumed: slot bt % S, phase (bt / S) & 1
    uint32_t ci = 0;       // position in the chunk sequence
    uint32_t wb = 0;       // A buffer of chunk ci (ci % NB)
    uint32_t wr = 0;       // done-barrier slot of chunk ci - NB ((ci - NB) % R)
    uint32_t wph = 0;      // its phase parity
    uint32_t mt_done = 0;  // M-tiles this slot has finished
    int pend = -1;         // A buffer stored but not yet published (afull)
    const bool prof = kMmaProfile && a.prof != nullptr && blockIdx.x == 0 && lane == 0;
    // block wait, done wait, block loads + refill, decode, stores + publish, other, epilogue
    long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tp = prof ? clock64() : 0;
    auto tick = [&](int q) {
      if (prof) {
        const long long t2 = clock64();
        pc[q] += t2 - tp;
        tp = t2;
      }
    };
    for (int64_t mt = first_mt; mt < a.n_mtiles; mt += mt_stride) {
      const int64_t g = 4 * mt + gq;
      const bool valid = g < G;
      const bool miss = MISS && mtile_missing(a.gmiss, mt, G);
      const uint8_t* src = m.x + g * (int64_t)GI_BLOCK_BYTES;
      if (valid && lane == 0) {
        for (int q = 0; q < kBlkSlots && q < T; ++q) {
          const uint32_t s = (bt + q) % kBlkSlots;
          bar_arrive_tx(myb + 8 * s, GI_BLOCK_BYTES);
          bulk_g2s(slot0 + s * GI_BLOCK_BYTES, src + q * tile_stride, GI_BLOCK_BYTES, myb + 8 * s);
        }
      }
      for (int64_t t = 0; t < T; ++t) {
        const uint32_t s = bt % kBlkSlots;
        uint32_t wd[32];
        if (valid) {
          tick(5);
          bar_wait(myb + 8 * s, (bt / kBlkSlots) & 1u);
          tick(0);
          ++bt;
          const uint32_t base = slot0 + s * GI_BLOCK_BYTES + 4u * lane;
#pragma unroll
          for (int w = 0; w < 32; ++w) {
            uint32_t x;
            asm volatile("ld.shared.u32 %0, [%1];"
                         : "=r"(x)
                         : "r"(base + (uint32_t)((lane ^ w) << 7)));
            wd[w] = x;
          }
          tick(2);
        }
#pragma unroll
        for (int hq = 0; hq < 4; ++hq) {
          if (ci >= (uint32_t)NB && (ci % C::kCB) == 0) {
            // chunks ci - NB .. ci - NB + kCB - 1 consumed (one commit group):
            // their A buffers and digit slots are free
            tick(5);
            bar_wait(b_done + 8 * (sl * R + wr + C::kCB - 1), wph);
            tick(1);
            wr += C::kCB;
            if (wr == (uint32_t)R) {
              wr = 0;
              wph ^= 1u;
            }
          }
          tc_fence_after();
          if (digit_lane) issue_digits();
          tick(5);
          if (valid) {
            // decode the chunk into registers, then publish the PREVIOUS chunk
            // (its stores have had this decode to land: the ~130-cycle
            // store -> wait::st latency stays off the critical path), then
            // issue this chunk's stores
            uint32_t sel[4][4], o1[16], o2[16], m1[16], m2[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) selectors(wd[8 * hq + q], sel[q]);
            lut16(sel, dose_lut, zero, o1);
            if (MISS && miss) lut16(sel, miss_lut, zero, m1);
#pragma unroll
            for (int q = 0; q < 4; ++q) selectors(wd[8 * hq + 4 + q], sel[q]);
            lut16(sel, dose_lut, zero, o2);
            if (MISS && miss) lut16(sel, miss_lut, zero, m2);
            tick(3);
            if (C::kDefer && pend >= 0) {
              asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
              tc_fence_before();
              __syncwarp();
              if (lane == 0) bar_arrive(b_afull + 8 * (sl * NB + pend));
            }
            const uint32_t acol = tmem + lane_base + (uint32_t)((sl * NB + wb) * C::kAcols);
            tmem_st16(acol, o1);
            tmem_st16(acol + 16, o2);
            if (MISS && miss) {
              tmem_st16(acol + 32, m1);
              tmem_st16(acol + 48, m2);
            }
            pend = (int)wb;
            if (!C::kDefer) {
              asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
              tc_fence_before();
              __syncwarp();
              if (lane == 0) bar_arrive(b_afull + 8 * (sl * NB + pend));
              pend = -1;
            }
          } else {
            __syncwarp();
            if (lane == 0) bar_arrive(b_afull + 8 * (sl * NB + wb));
          }
          tick(4);
          ++ci;
          wb = wb + 1 == (uint32_t)NB ? 0u : wb + 1;
        }
        // refill the tile's slot only now: every loaded word has been consumed
        // by the decode (a register dependency), so the generic reads are
        // complete before the async-proxy write -- no proxy fence needed, and
        // kBlkSlots - 1 tiles stay in flight
        if (valid) {
          __syncwarp();
          if (lane == 0 && t + kBlkSlots < T) {
            const uint32_t s2 = (bt - 1) % kBlkSlots;
            bar_arrive_tx(myb + 8 * s2, GI_BLOCK_BYTES);
            bulk_g2s(slot0 + s2 * GI_BLOCK_BYTES, src + (t + kBlkSlots) * tile_stride,
                     GI_BLOCK_BYTES, myb + 8 * s2);
          }
        }
      }
      if (pend >= 0) {  // publish the M-tile's last chunk
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) bar_arrive(b_afull + 8 * (sl * NB + pend));
        pend = -1;
      }
      // ---------------------------------------------------------- epilogue
      tick(5);
      bar_wait(b_dfull + 8 * sl, mt_done & 1u);
      tc_fence_after();
      const int64_t j = g * 32 + lane;
      const bool live_j = valid && j < m.p;
      // per-SNP statistics of the two right-hand sides of an 8-column step,
      // loaded one step ahead so their global latency overlaps the TMEM reads
      // and arithmetic of the current step (the epilogue took 18% of a decode
      // warp's cycles at config 4 with a dependent descriptor load per use)
      double nu[2] = {0.0, 0.0}, nv[2] = {0.0, 0.0};
      int ns1[2] = {0, 0}, ncn[2] = {0, 0};
      auto fetch = [&](int c0n) {
#pragma unroll
        for (int rb = 0; rb < 2; ++rb) {
          const int rhs = c0n / 4 + rb;
          if (rhs < a.nrhs && live_j) {
            const XtrRhs& rd = s_rhs[rhs];
            nu[rb] = __ldg(rd.u + j);
            nv[rb] = __ldg(rd.v + j);
            ns1[rb] = __ldg(rd.s1cnt + 2 * j);
            ncn[rb] = __ldg(rd.s1cnt + 2 * j + 1);
          }
        }
      };
      fetch(0);
#pragma unroll 1
      for (int c0 = 0; c0 < N; c0 += 8) {
        const double cu[2] = {nu[0], nu[1]}, cv[2] = {nv[0], nv[1]};
        const int cs1[2] = {ns1[0], ns1[1]}, ccn[2] = {ncn[0], ncn[1]};
        if (c0 + 8 < N) fetch(c0 + 8);
        int32_t dd[8] = {0, 0, 0, 0, 0, 0, 0, 0}, mm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int e = 0; e < ISS; ++e) {
          const uint32_t dcol =
              tmem + lane_base + (uint32_t)(C::kAtot + (sl * ISS + e) * C::kDcols + c0);
          uint32_t v8[8];
          tmem_ld8(dcol, v8);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int q = 0; q < 8; ++q) dd[q] += (int32_t)v8[q];
          if (MISS && miss) {
            tmem_ld8(dcol + N, v8);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int q = 0; q < 8; ++q) mm[q] += (int32_t)v8[q];
          }
        }
        if (c0 + 8 >= N) {  // accumulators drained: the next M-tile may start
          tc_fence_before();
          __syncwarp();
          if (lane == 0) bar_arrive(b_dempty + 8 * sl);
        }
#pragma unroll
        for (int rb = 0; rb < 2; ++rb) {
          const int rhs = c0 / 4 + rb;
          if (rhs < a.nrhs) {  // warp-uniform
            const XtrRhs& rd = s_rhs[rhs];
            double val = 0.0;
            if (live_j) {
              const long long Tq = (long long)dd[4 * rb] + 128ll * dd[4 * rb + 1] +
                                   16384ll * dd[4 * rb + 2] + 2097152ll * dd[4 * rb + 3];
              const long long Mq = (long long)mm[4 * rb] + 128ll * mm[4 * rb + 1] +
                                   16384ll * mm[4 * rb + 2] + 2097152ll * mm[4 * rb + 3];
              const double sc = s_q[3 * rhs], mean = s_q[3 * rhs + 1], sr = s_q[3 * rhs + 2];
              const double uj = cu[rb], vj = cv[rb];
              const double off = (double)cs1[rb] - uj * (double)ccn[rb];
              const double inner = (double)Tq + uj * ((double)Mq - sr);
              val = vj * (inner * sc + mean * off);
              rd.out[j] = a.scale_out * val;
            }
            if (rd.gmax) {  // max|g| for the IHT step (iht.py:257-261), order-free
              double mx = fabs(val);
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
              if (lane == 0 && mx > 0.0)
                atomicMax(rd.gmax, (unsigned long long)__double_as_longlong(mx));
            }
          }
        }
      }
      ++mt_done;
      tick(6);
    }
    if (prof)
      for (int q = 0; q < 8; ++q) a.prof[warp * 8 + q] = pc[q];
  } else {
    // ------------------------------------------------------------ MMA issuers
    const int iw = warp - kDecWarps, sl = iw / ISS, e = iw % ISS;
    if (lane == 0) {
      const bool prof = kMmaProfile && a.prof != nullptr && blockIdx.x == 0;
      long long pc[4] = {0, 0, 0, 0};  // afull wait, bfull wait, MMA + commit, dempty wait
      long long tp = prof ? clock64() : 0;
      auto tick = [&](int q) {
        if (prof) {
          const long long t2 = clock64();
          pc[q] += t2 - tp;
          tp = t2;
        }
      };
      const uint32_t ring0 = su32(bbuf + sl * R * C::kQBytes);
      uint32_t b = 0, bph = 0;  // A buffer of the chunk and its afull phase
      uint32_t r = 0, rph = 0;  // digit slot and its bfull phase
      uint32_t mt_done = 0;
      for (int64_t mt = 2 * (int64_t)blockIdx.x + sl; mt < a.n_mtiles; mt += mt_stride) {
        const bool miss = MISS && mtile_missing(a.gmiss, mt, G);
        if (mt_done >= 1) {
          tick(2);
          bar_wait(b_dempty + 8 * sl, (mt_done - 1) & 1u);
          tick(3);
          tc_fence_after();
        }
        const uint32_t dcol = tmem + (uint32_t)(C::kAtot + (sl * ISS + e) * C::kDcols);
        for (uint32_t c = 0; c < nchunks; ++c) {
          tick(2);
          bar_wait(b_afull + 8 * (sl * NB + b), bph);
          tick(0);
          bar_wait(b_bfull + 8 * (sl * R + r), rph);
          tick(1);
          tc_fence_after();
          const uint32_t acol = tmem + (uint32_t)((sl * NB + b) * C::kAcols);
          const uint32_t bsm = ring0 + r * C::kQBytes;
#pragma unroll
          for (int ks = e; ks < 4; ks += ISS) {
            const uint32_t sa = bsm + (uint32_t)ks * 2u * C::kLBO;
            const uint64_t bdesc = (uint64_t)((sa >> 4) & 0x3FFF) |
                                   ((uint64_t)((C::kLBO >> 4) & 0x3FFF) << 16) |
                                   ((uint64_t)((C::kSBO >> 4) & 0x3FFF) << 32) | (1ull << 46);
            const uint32_t acc = (c > 0 || ks != e) ? 1u : 0u;
            mma_i8(dcol, acol + 8u * ks, bdesc, C::kIdesc, acc);
            if (MISS && miss) mma_i8(dcol + N, acol + 32u + 8u * ks, bdesc, C::kIdesc, acc);
          }
          if ((c % C::kCB) == C::kCB - 1) mma_commit(b_done + 8 * (sl * R + r));
          if (++b == (uint32_t)NB) {
            b = 0;
            bph ^= 1u;
          }
          if (++r == (uint32_t)R) {
            r = 0;
            rph ^= 1u;
          }
        }
        mma_commit(b_dfull + 8 * sl);
        ++mt_done;
      }
      tick(2);
      if (prof)
        for (int q = 0; q < 4; ++q) a.prof[warp * 8 + q] = pc[q];
    }
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  if (a.pub_ticket) {
    __threadfence();
    __syncthreads();
    int last = 0;
    if (threadIdx.x == 0) last = atomicAdd(a.pub_ticket, 1u) == gridDim.x - 1;
    if (__syncthreads_or(last)) {
      __threadfence();
      for (int q = 0; q < a.pub.nseg; ++q) {
        const PubSeg sg = a.pub.seg[q];
        const unsigned long long* srcp = static_cast<const unsigned long long*>(sg.src);
        for (int64_t e2 = threadIdx.x; e2 < sg.count; e2 += blockDim.x)
          a.pub_out[sg.dst + e2] = __ldcg(sg.idx ? srcp + sg.idx[e2] : srcp + e2);
      }
      if (threadIdx.x == 0) *a.pub_ticket = 0u;
    }
  }
}

// ------------------------------------------------------------------ quantiser
// Per right-hand side b (blockIdx.y): over the rows with keep != 0, sum r,
// count, max r and min r; the last block folds them (block order, fixed tree)
// into qscal[b] = {s, mean} with s = max|r - mean| / 2^26, and zeroes qsum[b].
__global__ void xtr_qstats_kernel(int64_t n, const XtrRhs* __restrict__ rhs,
                                  double* __restrict__ qscal, long long* __restrict__ qsum,
                                  double* __restrict__ partials, unsigned int* __restrict__ ticket) {
  __shared__ double sh[4 * 32];
  __shared__ bool is_last;
  const int b = blockIdx.y;
  const double* rb = rhs[b].r;
  const uint8_t* kb = rhs[b].keep;
  double acc[2] = {0.0, 0.0};
  double mx = -INFINITY, mn = INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!kb || kb[i]) {
      const double x = rb[i];
      acc[0] += x;
      acc[1] += 1.0;
      mx = fmax(mx, x);
      mn = fmin(mn, x);
    }
  }
  block_sum<2>(acc, sh);
  mx = warp_max(mx);
  mn = -warp_max(-mn);
  if ((threadIdx.x & 31) == 0) {
    sh[64 + (threadIdx.x >> 5)] = mx;
    sh[96 + (threadIdx.x >> 5)] = mn;
  }
  __syncthreads();
  double* pb = partials + (int64_t)b * gridDim.x * 4;
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mx = fmax(mx, sh[64 + w]);
      mn = fmin(mn, sh[96 + w]);
    }
    pb[blockIdx.x * 4 + 0] = acc[0];
    pb[blockIdx.x * 4 + 1] = acc[1];
    pb[blockIdx.x * 4 + 2] = mx;
    pb[blockIdx.x * 4 + 3] = mn;
    __threadfence();
    is_last = atomicAdd(ticket + b, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (is_last && threadIdx.x < 32) {
    __threadfence();
    const double s = fold_sum(pb, 4, 0, gridDim.x);
    const double cnt = fold_sum(pb, 4, 1, gridDim.x);
    double hi = -INFINITY, lo = INFINITY;
    for (unsigned q = threadIdx.x; q < gridDim.x; q += 32) {
      hi = fmax(hi, __ldcg(pb + q * 4 + 2));
      lo = fmin(lo, __ldcg(pb + q * 4 + 3));
    }
    hi = warp_max(hi);
    lo = -warp_max(-lo);
    if (threadIdx.x == 0) {
      const double mean = cnt > 0.0 ? s / cnt : 0.0;
      const double big = cnt > 0.0 ? fmax(hi - mean, mean - lo) : 0.0;
      // |R| = |round((r - mean) / s)| <= 2^26: the four balanced base-128
      // digits reach 63 * (1 + 128 + 128^2 + 128^3) > 2^26
      qscal[2 * b] = big > 0.0 ? big * (1.0 + 0x1p-40) * 0x1p-26 : 1.0;
      qscal[2 * b + 1] = mean;
      qsum[b] = 0;
      ticket[b] = 0u;
    }
  }
}

// R_i -> four s8 digits in the chunk image (K order of `selectors`); sum of R_i.
// Columns of right-hand sides past nrhs are written as zeros.
template <int N>
__global__ void xtr_quant_kernel(int64_t n, int64_t n_pad, int nrhs,
                                 const XtrRhs* __restrict__ rhs, const double* __restrict__ qscal,
                                 long long* __restrict__ qsum, int8_t* __restrict__ qimg) {
  const int b = blockIdx.y;  // right-hand side slot (N / 4 of them)
  const double* rb = b < nrhs ? rhs[b].r : nullptr;
  const uint8_t* kb = b < nrhs ? rhs[b].keep : nullptr;
  long long part = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pad;
       i += (int64_t)gridDim.x * blockDim.x) {
    long long R = 0;
    if (b < nrhs && i < n && (!kb || kb[i])) {
      const double s = qscal[2 * b], mean = qscal[2 * b + 1];
      R = __double2ll_rn((rb[i] - mean) / s);
    }
    part += R;
    const int64_t c = i >> 7;
    const int k = digit_k_of_sample((int)(i & 127));
    int8_t* base = qimg + c * (128 * N) + (k >> 4) * (N / 8) * 128 + (k & 15);
    long long x = R;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const int q = (int)(((x + 64) & 127) - 64);
      x = (x - q) >> 7;
      const int col = 4 * b + d;
      base[(col >> 3) * 128 + (col & 7) * 16] = (int8_t)q;
    }
  }
  if (b < nrhs) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0 && part != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(qsum + b), (unsigned long long)part);
  }
}

template <int N, int ISS, bool MISS>
int launch_mma_t(const MmaArgs& a, int num_sms, cudaStream_t s) {
  using C = Cfg<N, ISS, MISS>;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(xtr_mma_kernel<N, ISS, MISS>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMma);
  });
  GI_CUDA_TRY(err);
  const int64_t slots = (a.n_mtiles + 1) / 2;
  const int grid = (int)(slots < num_sms ? slots : num_sms);
  xtr_mma_kernel<N, ISS, MISS><<<grid, C::kThreads, kSmemMma, s>>>(a);
  GI_LAUNCH_CHECK();
  return 0;
}

}  // namespace

int xtr_mma_cols(int nrhs) {
  return nrhs <= 2 ? 8 : (nrhs <= 4 ? 16 : (nrhs <= 8 ? 32 : (nrhs <= 16 ? 64 : 128)));
}

int64_t xtr_mma_qimg_bytes(const MatrixDesc& m, int nrhs) {
  return m.T * 4 * 128 * (int64_t)xtr_mma_cols(nrhs);
}

int xtr_mma_max_rhs(bool any_missing) { return any_missing ? 16 : kXtrMaxRhs; }

int launch_xtr_quant(int64_t n, int64_t T, int nrhs, const XtrRhs* d_rhs, double* qscal,
                     long long* qsum, int8_t* qimg, double* partials, int64_t partial_cap,
                     unsigned int* tickets, cudaStream_t s) {
  if (nrhs < 1 || nrhs > kXtrMaxRhs) {
    gi_set_error("X^T R on the tensor cores takes 1..32 right-hand sides (got %d)", nrhs);
    return -1;
  }
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148) blocks = 148;
  if (blocks < 1) blocks = 1;
  while (blocks > 1 && (int64_t)blocks * 4 * nrhs > partial_cap) blocks /= 2;
  if ((int64_t)blocks * 4 * nrhs > partial_cap) {
    gi_set_error("internal: quantiser partial buffer too small");
    return -1;
  }
  xtr_qstats_kernel<<<dim3(blocks, nrhs), 256, 0, s>>>(n, d_rhs, qscal, qsum, partials, tickets);
  GI_LAUNCH_CHECK();
  const int N = xtr_mma_cols(nrhs);
  const int64_t n_pad = T * GI_TILE_SAMPLES;
  int qblocks = (int)((n_pad + 255) / 256);
  if (qblocks > 4 * 148) qblocks = 4 * 148;
  const dim3 grid(qblocks, N / 4);
  switch (N) {
    case 8: xtr_quant_kernel<8><<<grid, 256, 0, s>>>(n, n_pad, nrhs, d_rhs, qscal, qsum, qimg); break;
    case 16: xtr_quant_kernel<16><<<grid, 256, 0, s>>>(n, n_pad, nrhs, d_rhs, qscal, qsum, qimg); break;
    case 32: xtr_quant_kernel<32><<<grid, 256, 0, s>>>(n, n_pad, nrhs, d_rhs, qscal, qsum, qimg); break;
    case 64: xtr_quant_kernel<64><<<grid, 256, 0, s>>>(n, n_pad, nrhs, d_rhs, qscal, qsum, qimg); break;
    default: xtr_quant_kernel<128><<<grid, 256, 0, s>>>(n, n_pad, nrhs, d_rhs, qscal, qsum, qimg); break;
  }
  GI_LAUNCH_CHECK();
  return 0;
}

int launch_xtr_mma(const MatrixDesc& m, const uint8_t* gmiss, bool any_missing, int nrhs,
                   const int8_t* qimg, const double* qscal, const long long* qsum,
                   const XtrRhs* d_rhs, double scale_out, int num_sms, cudaStream_t s,
                   const PubArgs* pub, unsigned int* pub_ticket, void* pub_out) {
  if (m.p == 0) return 0;
  static long long* prof_buf = nullptr;
  const bool prof = getenv("GI_MMA_PROF") != nullptr;
  if (prof && !prof_buf) GI_CUDA_TRY(cudaMallocManaged(&prof_buf, 8 * 32 * sizeof(long long)));
  if (nrhs < 1 || nrhs > xtr_mma_max_rhs(any_missing)) {
    gi_set_error("X^T R on the tensor cores: %d right-hand sides (1..32, <= 16 with missing "
                 "genotypes)", nrhs);
    return -1;
  }
  MmaArgs a;
  a.m = m;
  a.gmiss = gmiss;
  a.qimg = qimg;
  a.nrhs = nrhs;
  a.qscal = qscal;
  a.qsum = qsum;
  a.rhs = d_rhs;
  a.scale_out = scale_out;
  a.n_mtiles = (m.G + 3) / 4;
  a.prof = prof ? prof_buf : nullptr;
  if (pub && pub_ticket && pub_out) {
    a.pub = *pub;
    a.pub_ticket = pub_ticket;
    a.pub_out = static_cast<unsigned long long*>(pub_out);
  } else {
    a.pub_ticket = nullptr;
    a.pub_out = nullptr;
  }
  const int N = xtr_mma_cols(nrhs);
  int rc;
  if (any_missing) {
    switch (N) {
      case 8: rc = launch_mma_t<8, 2, true>(a, num_sms, s); break;
      case 16: rc = launch_mma_t<16, 2, true>(a, num_sms, s); break;
      case 32: rc = launch_mma_t<32, 2, true>(a, num_sms, s); break;
      default: rc = launch_mma_t<64, 1, true>(a, num_sms, s); break;
    }
  } else {
    switch (N) {
      case 8: rc = launch_mma_t<8, 4, false>(a, num_sms, s); break;
      case 16: rc = launch_mma_t<16, 4, false>(a, num_sms, s); break;
      case 32: rc = launch_mma_t<32, 2, false>(a, num_sms, s); break;
      case 64: rc = launch_mma_t<64, 2, false>(a, num_sms, s); break;
      default: rc = launch_mma_t<128, 1, false>(a, num_sms, s); break;
    }
  }
  if (prof && rc == 0) {
    GI_CUDA_TRY(cudaStreamSynchronize(s));
    for (int w = 0; w < 16; ++w)
      fprintf(stderr, "mma prof warp %2d: %11lld %11lld %11lld %11lld %11lld %11lld %11lld\n", w,
              prof_buf[w * 8], prof_buf[w * 8 + 1], prof_buf[w * 8 + 2], prof_buf[w * 8 + 3],
              prof_buf[w * 8 + 4], prof_buf[w * 8 + 5], prof_buf[w * 8 + 6]);
  }
  return rc;
}

}  // namespace gi
