// ozaki.cu — stage (4), S_b = A_b^H A_b (Eq. 3; north_star (4)), on the tcgen05
// integer tensor cores by exact digit splitting (the Ozaki scheme).
//
// FP64 has no tcgen05 kind; B200's FP64 tensor path is the legacy DMMA.8x8x4 (37 TFLOP/s
// measured, gram.cuh).  tcgen05.mma kind::i8 runs at 4.5 POPS nominal, so the Gram is
// evaluated as a short sum of EXACT int8 x int8 -> int32 products:
//
//   1. column scaling: every column j of A (a parameter) gets an exponent E_j with
//      max_k max(|Re A_kj|, |Im A_kj|) < 2^E_j, and X_kj = rint(A_kj 2^(54 - E_j)) is an
//      integer with |X| < 2^54 (rounding error <= 2^-55 of the column maximum);
//   2. digits: X = sum_{p=0..6} d_p 256^(6-p), d_p in [-128, 127], |d_0| <= 64 — seven int8
//      slices (the bytes of X + 128 sum 256^p, shifted by 128: digit_bytes / digits8);
//   3. real embedding: Re S = C^T C and Im S = C^T D over K' = 2 N_s, with
//      C = [Re A; Im A] and D = [Im A; -Re A] (so S = A^H A exactly);
//   4. products: G_t = sum_{p+q=t} C_p^T Y_q (Y = C or D) for t = 0..6, each an exact int32
//      accumulation in TMEM (|G_t| <= 7 * 128^2 * 16384 < 2^31 per K' chunk of 16384);
//      the dropped terms p+q >= 7 weigh <= 2^-51 of the leading one, i.e. the result carries
//      FP64-level error relative to max|A_.i| max|A_.j| (about what a K-long FP64 dot
//      product of the same columns commits);
//   5. recombination in FP64: S_ij = 2^(E_i + E_j - 60) sum_t 256^(6-t) G_t (Horner).
//
// Kernels: oz_colmax (column maxima), oz_split (digits, transposed to K-major int8 rows
// [slice][column][Re A | Im A | -Re A]), gram_i8 (persistent, warp-specialised: one TMA
// producer lane, one MMA-issuing lane, eight epilogue warps; 128 x 64 tiles of the lower
// triangle, the 28 digit-slice products of a 32-byte K step as 10 tcgen05.mma of N = 64 k into
// 7 TMEM accumulators), launched once per K' <= 16384 range (launch_herm: the launches add
// their FP64 partials to S in a fixed order, which keeps the concurrently running tiles'
// operand streams inside L2).
#include <cuda.h>

#include <algorithm>
#include <vector>

#include "ozaki.cuh"

namespace sr {
namespace oz {
namespace {

constexpr int BM = 128;                   // tile rows (i, A-operand rows, TMEM lanes)
constexpr int BN = 64;                    // tile cols (j, B-operand rows, TMEM columns per accumulator)
#ifndef SR_OZ_BKB
#define SR_OZ_BKB 64
#endif
// K bytes per pipeline stage = one swizzle row: 64 (64-byte swizzle, 2 stages of 86 KB) or
// 32 (32-byte swizzle, one MMA K step per stage, 5 stages of 43 KB)
constexpr int BKB = SR_OZ_BKB;
constexpr int kStages = BKB == 64 ? 2 : 5;
constexpr uint32_t kSwzLayout = BKB == 64 ? 4u : 6u;    // UMMA descriptor layout type: SWIZZLE_64B / _32B
constexpr uint32_t kSwzSBO = 8u * BKB;                 // bytes between 8-row core-matrix groups
constexpr int kASlice = BM * BKB;         // 8 KB
constexpr int kBSlice = BN * BKB;         // 4 KB
constexpr int kAStage = kSlices * kASlice;
constexpr int kStageBytes = kSlices * (kASlice + kBSlice);   // 86016
constexpr int kChunkK = 16384;            // K' per exact int32 accumulation
#ifndef SR_OZ_A_TMEM
#define SR_OZ_A_TMEM 0   // measured slower: 23.4 vs 20.2 ms at configs[1] (profiles/r01_tcgen05_rate.txt)
#endif
constexpr bool kATmem = SR_OZ_A_TMEM;     // operand A staged into TMEM by tcgen05.cp
constexpr uint32_t kACol = kSlices * BN;  // TMEM columns [448, 504): the A digits of one K step
#ifndef SR_OZ_EXP
#define SR_OZ_EXP 0   // energy experiments (tools only): 1 no S stores, 2 no epilogue, 3 L2-resident operands,
                      // 4 CRT-like MMA mix (16 N=64 MMAs per K step), 5 = 4 + doubled TMA bytes,
                      // 6 = doubled TMA bytes with the normal mix (results of 4-6 are wrong by design)
#endif
#ifndef SR_OZ_BAND
#define SR_OZ_BAND 8
#endif
#ifndef SR_OZ_PF
#define SR_OZ_PF 0   // > 0: the producer prefetches the boxes of stage kk + SR_OZ_PF into L2
#endif
#ifndef SR_OZ_SPLITBAR
#define SR_OZ_SPLITBAR 0   // 1: per-slice TMA boxes completing on three barriers per stage, so the
                           // first MMAs of a stage start once A0 and B0-3 have arrived
#endif
constexpr bool kSplitBar = SR_OZ_SPLITBAR;
constexpr int kBand = SR_OZ_BAND;         // row panels per rasterisation band
constexpr int kNonFinite = 1 << 20;       // column exponent marking a column with Inf / NaN
constexpr int kMaxBlk = 24;
constexpr int kEpiWarps = 8;              // two per TMEM lane quarter, 32 columns each
constexpr int kThreads = 64 + 32 * kEpiWarps;   // warp 0 TMA, warp 1 MMA + TMEM owner, warps 2.. epilogue
constexpr size_t kSmem = (size_t)kStages * kStageBytes + 1024 + 256;
// tcgen05 instruction descriptor: D s32 (bits 4-5 = 2), A/B signed int8 (bits 7-9, 10-12 = 1),
// both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
constexpr uint32_t idesc_n(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}
constexpr uint32_t kIdesc = idesc_n(BN);

struct Blk {
  long long col0;        // first row of this block in the slice matrix (column of A within the group)
  double2* C;            // output: S_b (MODE_HERM, ld n) or the matrix updated in place (MODE_SUB)
  long long ldc;
  long long tile_begin;  // first global tile index (tiles come in Re/Im pairs)
  int n, RT, CT;
  int jlim;              // > 0: only column tiles J < jlim (a lower trapezoid, row-major); 0: all
  int rect;              // 1: a full m x n rectangle C = X^H Y (rows of X from row0), no mirror
  int m;                 // rect: rows of C
  long long row0;        // rect: first A-operand row (slice-matrix row) relative to col0
};
// Epilogues: MODE_HERM writes S = G with its conjugate mirror (stage 4); MODE_SUB applies
// C -= G to the lower triangle i >= j (Cholesky trailing update, chol.cu).
enum { MODE_HERM = 0, MODE_SUB = 1 };
struct Params {
  int nblk;
  int kstages;           // K' / BKB of this launch
  int spc;               // stages per exact accumulation chunk
  long long kbase;       // first K stage of this launch (K-split launches, see launch_herm)
  int acc_in;            // 1: add to the partial S a previous K-split launch wrote (MODE_HERM)
  int defer;             // 1: a later K-split launch continues the sum (no mirror / final diagonal yet)
  long long Kp;          // padded sample count (bytes per slice-row segment)
  long long total_tiles;
  const int* expo;
  Blk b[kMaxBlk];
};

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// Bounded wait: a lost arrival traps (kernel error) after ~20 s instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  long long t0 = 0;
  for (int it = 0;; it++) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (it == 0) t0 = clock64();
    else if ((it & 1023) == 0 && clock64() - t0 > 40000000000LL) __trap();
  }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
// L2 prefetch of a future stage's box (no shared-memory write, no barrier).
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(map), "r"(c0), "r"(c1),
               "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc_) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(taddr), "l"(sdesc_));
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t acc,
                                       uint32_t idesc = kIdesc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// K-major operand, 64-byte swizzle: 8-row core groups 512 bytes apart (SBO), LBO unused (1),
// descriptor version 1 (sm_100), layout type 4 = SWIZZLE_64B (6 = SWIZZLE_32B).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(kSwzSBO >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)kSwzLayout << 61);
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// v * 2^k: one multiply when 2^k is a normal double, scalbn otherwise.
__device__ __forceinline__ double pow2_scale(double v, int k) {
  if (k >= -1022 && k <= 1023) return v * __longlong_as_double((long long)(k + 1023) << 52);
  return scalbn(v, k);
}

// Global tile t -> (block, row panel I, column panel J, pass).  Within a block the lower
// triangle tiles (J <= 2I + 1, i.e. some i >= j) are rasterised in bands of kBand row
// panels, column-major inside a band, and come in (Re, Im) pairs sharing the A panel.
template <int R = 2>
__device__ __forceinline__ void decode(const Params& P, long long t, int& b, int& I, int& J, int& pass) {
  b = 0;
  while (b + 1 < P.nblk && t >= P.b[b + 1].tile_begin) b++;
  long long u = t - P.b[b].tile_begin;
  pass = (int)(u & 1);
  u >>= 1;
  const int RT = P.b[b].RT, CT = P.b[b].CT;
  if (P.b[b].rect) {   // rectangle: column-major (the tiles of one column panel share its B operand)
    I = (int)(u % RT);
    J = (int)(u / RT);
    return;
  }
  if (P.b[b].jlim > 0) {   // trapezoid: row I holds min(CT, 2I + 2, jlim) tiles
    const int jl = min(CT, P.b[b].jlim);
    for (int i = 0; i < RT; i++) {
      const int c = min(jl, R * i + R);
      if (u < c) {
        I = i;
        J = (int)u;
        return;
      }
      u -= c;
    }
    I = J = 0;
    return;
  }
  // a band spans the same number of A rows for 128-row (R = 2) and 256-row (R = 4) tiles
  constexpr int band = kBand * 2 / R > 0 ? kBand * 2 / R : 1;
  for (int I0 = 0; I0 < RT; I0 += band) {
    const int I1 = min(RT, I0 + band), h = I1 - I0;
    long long cnt = 0;
    for (int i = I0; i < I1; i++) cnt += min(CT, R * i + R);
    if (u >= cnt) {
      u -= cnt;
      continue;
    }
    const int full = min(CT, R * I0);
    if (u < (long long)full * h) {
      J = (int)(u / h);
      I = I0 + (int)(u % h);
      return;
    }
    u -= (long long)full * h;
    for (int j = full; j < CT; j++) {
      const int lo = max(I0, j / R);
      const int c = I1 - lo;
      if (u < c) {
        J = j;
        I = lo + (int)u;
        return;
      }
      u -= c;
    }
  }
  I = J = 0;   // unreachable for t < total_tiles
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    gram_i8(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b, const Params P) {
  TraceScope trace_(MODE == MODE_HERM ? TR_GRAM : TR_TRAIL, P.b[0].n);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kStages);
  const uint32_t tfull = smem_u32(bars + 2 * kStages), tempty = smem_u32(bars + 2 * kStages + 1);
  // split barriers (kSplitBar): fullB = B slices 4-6, fullC = A slices 1-6 (full0 = A0 + B0-3)
  const uint32_t fullB0 = smem_u32(bars + 2 * kStages + 4), fullC0 = smem_u32(bars + 3 * kStages + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
      if (kSplitBar) {
        mbar_init(fullB0 + 8 * s, 1);
        mbar_init(fullC0 + 8 * s, 1);
      }
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, kEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm_a) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm_b) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t smem_base = smem_u32(smem);

  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (long long t = blockIdx.x; t < P.total_tiles; t += gridDim.x) {
        int b, I, J, pass;
        decode(P, t, b, I, J, pass);
        const int rowA = SR_OZ_EXP == 3 ? (int)P.b[b].col0
                                         : (int)(P.b[b].col0 + (P.b[b].rect ? P.b[b].row0 : 0) + (long long)I * BM);
        const int rowB = SR_OZ_EXP == 3 ? (int)P.b[b].col0 : (int)(P.b[b].col0 + (long long)J * BN);
        const int kB = pass ? (int)P.Kp : 0;
        for (int kk = 0; kk < P.kstages; kk++) {
          mbar_wait(empty0 + 8 * s, ph ^ 1);
          if (kSplitBar) {   // per-slice boxes (maps of one slice per box), three barriers
            const uint32_t sa = smem_base + s * kStageBytes, sbq = sa + kAStage;
            const int kc = (int)(P.kbase + kk) * BKB;
            mbar_expect_tx(full0 + 8 * s, kASlice + 4 * kBSlice);
            mbar_expect_tx(fullB0 + 8 * s, 3 * kBSlice);
            mbar_expect_tx(fullC0 + 8 * s, (kSlices - 1) * kASlice);
            tma_load_3d(sa, &tm_a, kc, rowA, 0, full0 + 8 * s);
#pragma unroll
            for (int q = 0; q < 4; q++) tma_load_3d(sbq + q * kBSlice, &tm_b, kB + kc, rowB, q, full0 + 8 * s);
#pragma unroll
            for (int q = 4; q < kSlices; q++) tma_load_3d(sbq + q * kBSlice, &tm_b, kB + kc, rowB, q, fullB0 + 8 * s);
#pragma unroll
            for (int p = 1; p < kSlices; p++) tma_load_3d(sa + p * kASlice, &tm_a, kc, rowA, p, fullC0 + 8 * s);
            if (++s == kStages) {
              s = 0;
              ph ^= 1;
            }
            continue;
          }
          constexpr int kRep = (SR_OZ_EXP == 5 || SR_OZ_EXP == 6) ? 2 : 1;
          mbar_expect_tx(full0 + 8 * s, kRep * kStageBytes);
          const uint32_t sa = smem_base + s * kStageBytes;
#pragma unroll
          for (int rep = 0; rep < kRep; rep++) {
            const int kc = (int)(P.kbase + kk) * BKB;
            tma_load_3d(sa, &tm_a, kc, rowA, 0, full0 + 8 * s);
            tma_load_3d(sa + kAStage, &tm_b, kB + kc, rowB, 0, full0 + 8 * s);
          }
          if (SR_OZ_PF > 0 && kk + SR_OZ_PF < P.kstages) {
            const int kp = (int)(P.kbase + kk + SR_OZ_PF) * BKB;
            tma_prefetch_3d(&tm_a, kp, rowA, 0);
            tma_prefetch_3d(&tm_b, kB + kp, rowB, 0);
          }
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ---------------- MMA issuer (one thread for the CTA)
      int s = 0;
      uint32_t ph = 0, acc_ph = 0;
      for (long long t = blockIdx.x; t < P.total_tiles; t += gridDim.x) {
        for (int kk = 0; kk < P.kstages; kk++) {
          const int kin = kk % P.spc;
          if (kin == 0) {   // accumulators drained by the epilogue?
            mbar_wait(tempty, acc_ph ^ 1);
            acc_ph ^= 1;
            tc_fence_after();
          }
          if (kSplitBar && MODE >= 0) {
            const uint32_t sa = smem_base + s * kStageBytes, sb = sa + kAStage;
            mbar_wait(full0 + 8 * s, ph);   // A0, B0-3: (p = 0, q = 0..3)
            tc_fence_after();
#pragma unroll
            for (int ks = 0; ks < BKB / 32; ks++)
              mma_i8(tmem, sdesc(sa + ks * 32), sdesc(sb + ks * 32), (kin > 0 || ks > 0) ? 1u : 0u, idesc_n(4 * BN));
            mbar_wait(fullB0 + 8 * s, ph);  // B4-6: (p = 0, q = 4..6)
            tc_fence_after();
#pragma unroll
            for (int ks = 0; ks < BKB / 32; ks++)
              mma_i8(tmem + (uint32_t)(4 * BN), sdesc(sa + ks * 32), sdesc(sb + 4 * kBSlice + ks * 32),
                     (kin > 0 || ks > 0) ? 1u : 0u, idesc_n(3 * BN));
            mbar_wait(fullC0 + 8 * s, ph);  // A1-6: p >= 1
            tc_fence_after();
#pragma unroll
            for (int ks = 0; ks < BKB / 32; ks++)
#pragma unroll
              for (int p = 1; p < kSlices; p++) {
                const uint64_t ad = sdesc(sa + p * kASlice + ks * 32);
#pragma unroll
                for (int q = 0; q + p < kSlices; q += 4) {
                  const int nq = (kSlices - p - q) < 4 ? (kSlices - p - q) : 4;
                  mma_i8(tmem + (uint32_t)((p + q) * BN), ad, sdesc(sb + q * kBSlice + ks * 32), 1u, idesc_n(BN * nq));
                }
              }
            tc_commit(empty0 + 8 * s);
            if (kin == P.spc - 1 || kk == P.kstages - 1) tc_commit(tfull);
            if (++s == kStages) {
              s = 0;
              ph ^= 1;
            }
            continue;
          }
          mbar_wait(full0 + 8 * s, ph);
          tc_fence_after();
          const uint32_t sa = smem_base + s * kStageBytes, sb = sa + kAStage;
#pragma unroll
          for (int ks = 0; ks < BKB / 32; ks++) {
            if (kATmem) {
              // A digits of this K step -> TMEM (7 x 128 lanes x 32 bytes = 56 columns), so the
              // MMAs read only B through the shared-memory port.  tcgen05.cp and tcgen05.mma
              // from this thread execute in issue order: the copy of step ks+1 cannot
              // overtake the MMAs of step ks that read the same columns.
#pragma unroll
              for (int p = 0; p < kSlices; p++) tmem_cp_128x256b(tmem + kACol + 8 * p, sdesc(sa + p * kASlice + ks * 32));
            }
            if (SR_OZ_EXP == 4 || SR_OZ_EXP == 5) {   // CRT-like mix: 16 independent N = 64 products
#pragma unroll
              for (int m = 0; m < 16; m++)
                mma_i8(tmem + (uint32_t)((m & 7) * BN), sdesc(sa + (m % kSlices) * kASlice + ks * 32),
                       sdesc(sb + (m % kSlices) * kBSlice + ks * 32), (kin > 0 || ks > 0 || m > 7) ? 1u : 0u,
                       idesc_n(BN));
              continue;
            }
#pragma unroll
            for (int p = 0; p < kSlices; p++) {
              const uint64_t ad = sdesc(sa + p * kASlice + ks * 32);
              const uint32_t acc = (kin > 0 || ks > 0 || p > 0) ? 1u : 0u;
              if (kATmem) {
#pragma unroll
                for (int q = 0; q + p < kSlices; q++)
                  mma_i8_ts(tmem + (uint32_t)((p + q) * BN), tmem + kACol + 8 * p,
                            sdesc(sb + q * kBSlice + ks * 32), acc);
              } else {
                // Slice pairs (p, q..q+k-1) in ONE MMA of N = 64 k <= 256: the B slices are
                // adjacent 64-row groups in shared memory and the accumulators of the digit
                // diagonals p+q..p+q+k-1 are adjacent 64-column groups in TMEM.  10 MMAs per
                // K step instead of 28, reading each A slice once.
#pragma unroll
                for (int q = 0; q + p < kSlices; q += 4) {
                  const int nq = (kSlices - p - q) < 4 ? (kSlices - p - q) : 4;
                  mma_i8(tmem + (uint32_t)((p + q) * BN), ad, sdesc(sb + q * kBSlice + ks * 32), acc,
                         idesc_n(BN * nq));
                }
              }
            }
          }
          tc_commit(empty0 + 8 * s);   // frees the smem stage when these MMAs complete
          if (kin == P.spc - 1 || kk == P.kstages - 1) tc_commit(tfull);
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else {   // ---------------- epilogue: TMEM -> FP64 recombination -> S
    const int q4 = warp & 3;             // TMEM lane quarter this warp may access
    const int rl = q4 * 32 + lane;       // tile row of this thread
    const int c0 = ((warp - 2) >> 2) * (BN / 2);   // first of this warp's 32 tile columns
    const int nchunks = (P.kstages + P.spc - 1) / P.spc;
    uint32_t c = 0;
    for (long long t = blockIdx.x; t < P.total_tiles; t += gridDim.x) {
      int b, I, J, pass;
      decode(P, t, b, I, J, pass);
      const Blk& B = P.b[b];
      const int n = B.n;
      const int i = I * BM + rl;
      const bool row_ok = i < (B.rect ? B.m : n);
      const int ei = row_ok ? P.expo[B.col0 + (B.rect ? B.row0 : 0) + i] : 0;
      double* Cb = reinterpret_cast<double*>(B.C);
      const long long ldc = B.ldc;
      for (int ch = 0; ch < nchunks; ch++, c++) {
        mbar_wait(tfull, c & 1);
        tc_fence_after();
        if (SR_OZ_EXP == 2) {   // energy experiment: no epilogue work at all
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty);
          continue;
        }
        // Phase 1: TMEM -> registers, the seven digit-diagonal sums combined by Horner
        // (exact int32 -> FP64), then TMEM is released so the next tile's MMAs overlap
        // phase 2 (scaling and the global writes).
        double vals[BN / 2];
#pragma unroll
        for (int cc = 0; cc < BN / 16; cc++) {
          uint32_t g[kSlices][8];
#pragma unroll
          for (int tt = 0; tt < kSlices; tt++)
            tmem_ld8(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(tt * BN + c0 + cc * 8), g[tt]);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 8; e++) {
            double v = (double)(int)g[0][e];
#pragma unroll
            for (int tt = 1; tt < kSlices; tt++) v = fma(v, 256.0, (double)(int)g[tt][e]);
            vals[cc * 8 + e] = v;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
        if (SR_OZ_EXP == 1 && vals[0] != 12345.0) continue;   // energy experiment: no stores
        // Phase 2 (column exponents fetched once per lane, broadcast by shuffles)
        const int jl = J * BN + c0 + lane;
        const int ej_lane = jl < n ? P.expo[B.col0 + jl] : 0;
        const int jb = J * BN + c0;
        double* dp = Cb + 2 * ((long long)i * ldc + jb) + pass;   // C[i][j], j = jb + e
        double* mp = Cb + 2 * ((long long)jb * ldc + i) + pass;   // C[j][i]
        const long long mstep = 2 * ldc;
#pragma unroll
        for (int e = 0; e < BN / 2; e++, mp += mstep) {
          const int ej = __shfl_sync(0xffffffffu, ej_lane, e);
          const int j = jb + e;
          if (!row_ok || j >= n || (!B.rect && j > i)) continue;
          // a non-finite input column poisons its row and column of the result, as in FP64
          const double val = (ei == kNonFinite || ej == kNonFinite) ? __longlong_as_double(0x7FF8000000000000LL)
                                                                     : pow2_scale(vals[e], ei + ej - 60);
          if (MODE == MODE_SUB) {
            // C -= G on the lower triangle by a fire-and-forget reduction in L2
            // (red.global.add.f64): each element receives exactly one addend per launch
            // (Re pass -> .x, Im pass -> .y), so the result is deterministic.
            atomicAdd(dp + 2 * e, -val);
            continue;
          }
          if (B.rect) {   // rectangle: store or accumulate, no mirror, no diagonal special case
            double acc = val;
            if (ch > 0 || P.acc_in) acc += dp[2 * e];
            dp[2 * e] = acc;
            continue;
          }
          if (nchunks == 1 && !P.acc_in && !P.defer) {
            if (i == j) {
              dp[2 * e] = pass ? 0.0 : val;
            } else {
              dp[2 * e] = val;
              *mp = pass ? -val : val;
            }
            continue;
          }
          double acc = val;
          if (ch > 0 || P.acc_in) acc += dp[2 * e];
          if (ch + 1 < nchunks || P.defer) {
            dp[2 * e] = acc;
          } else if (i == j) {
            dp[2 * e] = pass ? 0.0 : acc;
          } else {
            dp[2 * e] = acc;
            *mp = pass ? -acc : acc;
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}


// ---------------------------------------------------------------- CTA-pair variant
// gram_i8_2sm: the same product on CTA pairs (cluster of 2, tcgen05 cta_group::2): a pair
// computes a 256 x 64 tile, each CTA holding its own 128 rows of A (and of the result in
// its TMEM), and the B operand of every MMA split between the two CTAs by N (the first N/2
// rows of B from the leader's shared memory, the rest from the peer's).  B reaches each SM
// once instead of twice, so the shared-memory traffic per K step and SM drops from 138 KB
// (TMA writes 42 + MMA reads 96) to 116 KB (40 + 48 + 28), below the tensor time of the
// step.  Slice pairs per K step (12 MMAs, N = 64 k, k in {1, 2, 4} so that every N/2
// boundary falls on a slice or half-slice boundary):
//   region  rows  leader holds        peer holds           used by (p, q..)
//   R0      128   slices 0,1          slices 2,3           (p, 0..3) for p <= 3
//   R1       64   slice 4             slice 5              (p, 4..5) for p <= 1
//   R2       64   slice 0             slice 1              (p, 0..1) for p = 4, 5
//   H0..H3   32   rows 0-31 of 0,2,4,6  rows 32-63 of 0,2,4,6  (p, q) single: (6,0) (4,2) (2,4) (0,6)
constexpr int kR0 = 128, kR1 = 64, kR2 = 64, kH = 32;
constexpr int kB2Rows = kR0 + kR1 + kR2 + 4 * kH;                    // 384
constexpr int kStage2 = kSlices * kASlice + kB2Rows * BKB;          // 81920
constexpr size_t kSmem2 = (size_t)kStages * kStage2 + 1024 + 256;
constexpr uint32_t idesc2_n(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(bar_cluster) : "memory");
}
// TMA into this CTA's shared memory, completing on the (leader's) barrier at a shared::cluster address.
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.cta_group::2 [%0], [%1, {%2, "
      "%3, %4}], [%5];\n" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t acc,
                                            uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {   // arrives on `bar` in both CTAs of the pair
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(bar),
      "h"((unsigned short)3)
      : "memory");
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gram_i8_2sm(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b2,
                const __grid_constant__ CUtensorMap tm_b1, const __grid_constant__ CUtensorMap tm_h,
                const Params P) {
  TraceScope trace_(MODE == MODE_HERM ? TR_GRAM : TR_TRAIL, P.b[0].n);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStage2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kStages);
  const uint32_t tfull = smem_u32(bars + 2 * kStages), tempty = smem_u32(bars + 2 * kStages + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const long long cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const uint32_t full0_lead = mapa_shared(full0, 0), tempty_lead = mapa_shared(tempty, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * kEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm_a) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm_b2) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm_b1) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm_h) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();   // both CTAs' barriers initialised and TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t smem_base = smem_u32(smem);

  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer (both CTAs; completion on the leader's barrier)
      int s = 0;
      uint32_t ph = 0;
      for (long long t = cid; t < P.total_tiles; t += ncl) {
        int b, I, J, pass;
        decode<4>(P, t, b, I, J, pass);
        const int rowA = (int)(P.b[b].col0 + (long long)(2 * I + (int)rank) * BM);
        const int rowB = (int)(P.b[b].col0 + (long long)J * BN);
        const int kB = pass ? (int)P.Kp : 0;
        for (int kk = 0; kk < P.kstages; kk++) {
          mbar_wait(empty0 + 8 * s, ph ^ 1);
          if (rank == 0) mbar_expect_tx(full0 + 8 * s, 2 * kStage2);
          const uint32_t sa = smem_base + s * kStage2, sb = sa + kSlices * kASlice;
          const uint32_t fb = full0_lead + 8 * s;
          const int kc = (int)(P.kbase + kk) * BKB;
          tma_load_3d_pair(sa, &tm_a, kc, rowA, 0, fb);
          tma_load_3d_pair(sb, &tm_b2, kB + kc, rowB, rank ? 2 : 0, fb);                       // R0
          tma_load_3d_pair(sb + kR0 * BKB, &tm_b1, kB + kc, rowB, rank ? 5 : 4, fb);          // R1
          tma_load_3d_pair(sb + (kR0 + kR1) * BKB, &tm_b1, kB + kc, rowB, rank ? 1 : 0, fb);  // R2
#pragma unroll
          for (int h = 0; h < 4; h++)                                                            // H0..H3
            tma_load_3d_pair(sb + (kR0 + kR1 + kR2 + h * kH) * BKB, &tm_h, kB + kc, rowB + (int)rank * kH, 2 * h, fb);
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {   // ---------------- MMA issuer (leader CTA only)
      int s = 0;
      uint32_t ph = 0, acc_ph = 0;
      for (long long t = cid; t < P.total_tiles; t += ncl) {
        for (int kk = 0; kk < P.kstages; kk++) {
          const int kin = kk % P.spc;
          if (kin == 0) {   // accumulators drained by both CTAs' epilogues?
            mbar_wait(tempty, acc_ph ^ 1);
            acc_ph ^= 1;
            tc_fence_after();
          }
          mbar_wait(full0 + 8 * s, ph);
          tc_fence_after();
          const uint32_t sa = smem_base + s * kStage2, sb = sa + kSlices * kASlice;
          const uint32_t r0 = sb, r1 = sb + kR0 * BKB, r2 = r1 + kR1 * BKB, h0 = r2 + kR2 * BKB;
#pragma unroll
          for (int ks = 0; ks < BKB / 32; ks++) {
            const uint32_t ko = ks * 32;
            const uint32_t first = (kin > 0 || ks > 0) ? 1u : 0u;
            // D column of digit diagonal d: 64 d.  A slice p: sa + p * kASlice.
#pragma unroll
            for (int p = 0; p < kSlices; p++) {
              const uint64_t ad = sdesc(sa + p * kASlice + ko);
              const uint32_t acc = (first || p > 0) ? 1u : 0u;
              if (p <= 3) mma_i8_pair(tmem + 64 * p, ad, sdesc(r0 + ko), acc, idesc2_n(256));         // q 0..3
              if (p <= 1) mma_i8_pair(tmem + 64 * (p + 4), ad, sdesc(r1 + ko), acc, idesc2_n(128));   // q 4..5
              if (p == 4 || p == 5) mma_i8_pair(tmem + 64 * p, ad, sdesc(r2 + ko), acc, idesc2_n(128));   // q 0..1
              if (p == 4) mma_i8_pair(tmem + 64 * 6, ad, sdesc(h0 + 1 * kH * BKB + ko), acc, idesc2_n(64));   // q 2
              if (p == 2) mma_i8_pair(tmem + 64 * 6, ad, sdesc(h0 + 2 * kH * BKB + ko), acc, idesc2_n(64));   // q 4
              if (p == 0) mma_i8_pair(tmem + 64 * 6, ad, sdesc(h0 + 3 * kH * BKB + ko), acc, idesc2_n(64));   // q 6
              if (p == 6) mma_i8_pair(tmem + 64 * 6, ad, sdesc(h0 + ko), acc, idesc2_n(64));                  // q 0
            }
          }
          tc_commit_pair(empty0 + 8 * s);   // frees the stage in both CTAs when these MMAs complete
          if (kin == P.spc - 1 || kk == P.kstages - 1) tc_commit_pair(tfull);
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else {   // ---------------- epilogue (both CTAs, own 128 rows): TMEM -> FP64 recombination -> S
    const int q4 = warp & 3;             // TMEM lane quarter this warp may access
    const int rl = q4 * 32 + lane;       // tile row of this thread
    const int c0 = ((warp - 2) >> 2) * (BN / 2);   // first of this warp's 32 tile columns
    const int nchunks = (P.kstages + P.spc - 1) / P.spc;
    uint32_t c = 0;
    for (long long t = cid; t < P.total_tiles; t += ncl) {
      int b, I, J, pass;
      decode<4>(P, t, b, I, J, pass);
      I = 2 * I + rank;   // this CTA's 128-row half of the 256-row tile
      const Blk& B = P.b[b];
      const int n = B.n;
      const int i = I * BM + rl;
      const bool row_ok = i < n;
      const int ei = row_ok ? P.expo[B.col0 + i] : 0;
      double* Cb = reinterpret_cast<double*>(B.C);
      const long long ldc = B.ldc;
      for (int ch = 0; ch < nchunks; ch++, c++) {
        mbar_wait(tfull, c & 1);
        tc_fence_after();
        // Phase 1: TMEM -> registers, the seven digit-diagonal sums combined by Horner
        // (exact int32 -> FP64), then TMEM is released so the next tile's MMAs overlap
        // phase 2 (scaling and the global writes).
        double vals[BN / 2];
#pragma unroll
        for (int cc = 0; cc < BN / 16; cc++) {
          uint32_t g[kSlices][8];
#pragma unroll
          for (int tt = 0; tt < kSlices; tt++)
            tmem_ld8(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(tt * BN + c0 + cc * 8), g[tt]);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 8; e++) {
            double v = (double)(int)g[0][e];
#pragma unroll
            for (int tt = 1; tt < kSlices; tt++) v = fma(v, 256.0, (double)(int)g[tt][e]);
            vals[cc * 8 + e] = v;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_lead);   // the leader's MMA issuer waits for both CTAs
        // Phase 2 (column exponents fetched once per lane, broadcast by shuffles)
        const int jl = J * BN + c0 + lane;
        const int ej_lane = jl < n ? P.expo[B.col0 + jl] : 0;
        const int jb = J * BN + c0;
        double* dp = Cb + 2 * ((long long)i * ldc + jb) + pass;   // C[i][j], j = jb + e
        double* mp = Cb + 2 * ((long long)jb * ldc + i) + pass;   // C[j][i]
        const long long mstep = 2 * ldc;
#pragma unroll
        for (int e = 0; e < BN / 2; e++, mp += mstep) {
          const int ej = __shfl_sync(0xffffffffu, ej_lane, e);
          const int j = jb + e;
          if (!row_ok || j >= n || j > i) continue;
          // a non-finite input column poisons its row and column of the result, as in FP64
          const double val = (ei == kNonFinite || ej == kNonFinite) ? __longlong_as_double(0x7FF8000000000000LL)
                                                                     : pow2_scale(vals[e], ei + ej - 60);
          if (MODE == MODE_SUB) {
            // C -= G on the lower triangle by a fire-and-forget reduction in L2
            // (red.global.add.f64): each element receives exactly one addend per launch
            // (Re pass -> .x, Im pass -> .y), so the result is deterministic.
            atomicAdd(dp + 2 * e, -val);
            continue;
          }
          if (nchunks == 1 && !P.acc_in && !P.defer) {
            if (i == j) {
              dp[2 * e] = pass ? 0.0 : val;
            } else {
              dp[2 * e] = val;
              *mp = pass ? -val : val;
            }
            continue;
          }
          double acc = val;
          if (ch > 0 || P.acc_in) acc += dp[2 * e];
          if (ch + 1 < nchunks || P.defer) {
            dp[2 * e] = acc;
          } else if (i == j) {
            dp[2 * e] = pass ? 0.0 : acc;
          } else {
            dp[2 * e] = acc;
            *mp = pass ? -acc : acc;
          }
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

// Column maxima of max(|Re|, |Im|) over samples, as the bit patterns of |x|: for
// non-negative doubles the order of the patterns is the order of the values, and Inf / NaN
// patterns exceed every finite one, so a non-finite entry marks its column (kNonFinite).
__device__ __forceinline__ unsigned long long abs_bits(double x) {
  return (unsigned long long)__double_as_longlong(x) & 0x7FFFFFFFFFFFFFFFULL;
}
constexpr unsigned long long kInfBits = 0x7FF0000000000000ULL;
__global__ void oz_colmax(const double2* __restrict__ A, long long lda, long long c0, int n, long long K,
                          int rows_per, unsigned long long* __restrict__ mx) {
  TraceScope trace_(TR_COLMAX, 0);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const long long k0 = (long long)blockIdx.y * rows_per, k1 = min(K, k0 + rows_per);
  unsigned long long m = 0;
  for (long long k = k0; k < k1; k++) {
    const double2 v = A[k * lda + c0 + j];
    m = max(m, max(abs_bits(v.x), abs_bits(v.y)));
  }
  atomicMax(mx + j, m);
}

// Column exponent E with max < 2^E (0 for an all-zero column, kNonFinite if Inf / NaN).
__device__ __forceinline__ int column_exponent(unsigned long long mbits) {
  if (mbits >= kInfBits) return kNonFinite;
  int e = 0;
  const double m = __longlong_as_double((long long)mbits);
  if (m > 0.0) frexp(m, &e);
  return e;
}

// Signed base-256 digits from bytes: with C = 128 sum_{p<7} 256^p (> 2^54 > |X|),
// U = X + C lies in [0, 2^56) and X = sum_p (u_p - 128) 256^(6-p) for the bytes u_p of U, so
// the int8 digits are the bytes of U xor 0x80...80 — d_p in [-128, 127], |d_0| <= 64 as
// for balanced digits.  digits8 takes eight values and returns pk[p] = digit p of value r in
// byte r: an 8x8 byte transpose (32 byte permutes) instead of per-digit integer arithmetic.
constexpr unsigned long long kDigitBias = 0x0080808080808080ULL;   // C
__device__ __forceinline__ uint64_t digit_bytes(long long x) {
  return ((unsigned long long)x + kDigitBias) ^ kDigitBias;   // bytes 0..6 = digits 6..0
}
__device__ __forceinline__ void transpose4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t& o0,
                                           uint32_t& o1, uint32_t& o2, uint32_t& o3) {
  const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
  const uint32_t t2 = __byte_perm(c, d, 0x5140), t3 = __byte_perm(c, d, 0x7362);
  o0 = __byte_perm(t0, t2, 0x5410);
  o1 = __byte_perm(t0, t2, 0x7632);
  o2 = __byte_perm(t1, t3, 0x5410);
  o3 = __byte_perm(t1, t3, 0x7632);
}
__device__ __forceinline__ void digits8(const uint64_t (&u)[8], uint64_t (&pk)[kSlices]) {
  uint32_t lo[8], hi[8];   // transposed rows: byte j of every value, values 0-3 | 4-7
  uint32_t T[8][2];
#pragma unroll
  for (int r = 0; r < 8; r++) {
    lo[r] = (uint32_t)u[r];
    hi[r] = (uint32_t)(u[r] >> 32);
  }
  transpose4(lo[0], lo[1], lo[2], lo[3], T[0][0], T[1][0], T[2][0], T[3][0]);   // bytes 0-3, values 0-3
  transpose4(lo[4], lo[5], lo[6], lo[7], T[0][1], T[1][1], T[2][1], T[3][1]);   // bytes 0-3, values 4-7
  transpose4(hi[0], hi[1], hi[2], hi[3], T[4][0], T[5][0], T[6][0], T[7][0]);   // bytes 4-7, values 0-3
  transpose4(hi[4], hi[5], hi[6], hi[7], T[4][1], T[5][1], T[6][1], T[7][1]);   // bytes 4-7, values 4-7
#pragma unroll
  for (int p = 0; p < kSlices; p++) pk[p] = (uint64_t)T[6 - p][0] | ((uint64_t)T[6 - p][1] << 32);
}

// Digits of 32 columns x 64 samples, written as K-major int8 rows
// E[p][j][part * Kp + k], part 0 = Re A, 1 = Im A, 2 = -Re A.
constexpr int kSplitRow = 80;   // smem bytes per staged 64-byte row (conflict-light, 16-B aligned)
constexpr size_t kSplitSmem = (size_t)3 * kSlices * 32 * kSplitRow;
__global__ void __launch_bounds__(256) oz_split(const double2* __restrict__ A, long long lda, long long c0, int n,
                                                long long K, long long Kp, const unsigned long long* __restrict__ mx,
                                                int8_t* __restrict__ E, int* __restrict__ expo) {
  TraceScope trace_(TR_SPLIT, 0);
  extern __shared__ uint8_t ssm[];
  const int t = threadIdx.x, jl = t & 31, kg = t >> 5;
  const int j = blockIdx.x * 32 + jl;
  const long long k0 = (long long)blockIdx.y * 64;
  int e = 0;
  if (j < n) {
    e = column_exponent(mx[j]);
    if (blockIdx.y == 0 && kg == 0) expo[j] = e;
    if (e == kNonFinite) e = 0;   // digits of a marked column are never used
  }
  uint64_t pk[3][kSlices];
  {
    const int ks = 54 - e;   // scaling by 2^ks: one exact multiply unless 2^ks is not a normal double
    const bool fast = ks >= -1022 && ks <= 1023;
    const double sc = fast ? __longlong_as_double((long long)(ks + 1023) << 52) : 0.0;
    uint64_t ur[8], ui[8], un[8];
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const long long k = k0 + kg * 8 + r;
      double2 v = make_double2(0.0, 0.0);
      if (j < n && k < K) v = A[k * lda + c0 + j];
      const long long xr = llrint(fast ? v.x * sc : scalbn(v.x, ks)), xi = llrint(fast ? v.y * sc : scalbn(v.y, ks));
      ur[r] = digit_bytes(xr);
      ui[r] = digit_bytes(xi);
      un[r] = digit_bytes(-xr);
    }
    digits8(ur, pk[0]);
    digits8(ui, pk[1]);
    digits8(un, pk[2]);
  }
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int p = 0; p < kSlices; p++)
      *reinterpret_cast<uint64_t*>(ssm + ((a * kSlices + p) * 32 + jl) * kSplitRow + kg * 8) = pk[a][p];
  __syncthreads();
  for (int c = t; c < 3 * kSlices * 32 * 4; c += 256) {
    const int row = c >> 2, q = c & 3;
    const int a = row / (kSlices * 32), rem = row % (kSlices * 32), p = rem / 32, jj = blockIdx.x * 32 + rem % 32;
    if (jj >= n) continue;
    const uint4 v = *reinterpret_cast<const uint4*>(ssm + row * kSplitRow + q * 16);
    *reinterpret_cast<uint4*>(E + ((long long)p * n + jj) * (3 * Kp) + a * Kp + k0 + q * 16) = v;
  }
}

// Digits of the rows of L (row-major along K, ld ldl) for C -= L L^H: row i plays the role
// of a column of A = L^H (A_ki = conj(L_ik)), so the parts are [Re L | -Im L | -Re L].
// One warp per row: row maximum by shuffles, then 8 consecutive k per lane per pass.
__global__ void __launch_bounds__(256) oz_split_rows(const double2* __restrict__ L, long long ldl, int m, int K,
                                                     int Kp, int8_t* __restrict__ E, int* __restrict__ expo) {
  TraceScope trace_(TR_SPLIT_ROWS, 0);
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= m) return;
  const double2* row = L + (long long)i * ldl;
  unsigned long long mx = 0;
  for (int k = lane; k < K; k += 32) mx = max(mx, max(abs_bits(row[k].x), abs_bits(row[k].y)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = column_exponent(mx);
  if (lane == 0) expo[i] = e;
  if (e == kNonFinite) e = 0;
  const int ks = 54 - e;   // scaling by 2^ks as in oz_split
  const bool fast = ks >= -1022 && ks <= 1023;
  const double sc = fast ? __longlong_as_double((long long)(ks + 1023) << 52) : 0.0;
  for (int k0 = lane * 8; k0 < Kp; k0 += 256) {
    uint64_t pk[3][kSlices];
    {
      uint64_t ur[8], ui[8], un[8];
#pragma unroll
      for (int r = 0; r < 8; r++) {
        const int k = k0 + r;
        const double2 v = k < K ? row[k] : make_double2(0.0, 0.0);
        const long long xr = llrint(fast ? v.x * sc : scalbn(v.x, ks)), xi = llrint(fast ? -v.y * sc : scalbn(-v.y, ks));
        ur[r] = digit_bytes(xr);
        ui[r] = digit_bytes(xi);
        un[r] = digit_bytes(-xr);
      }
      digits8(ur, pk[0]);
      digits8(ui, pk[1]);
      digits8(un, pk[2]);
    }
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int p = 0; p < kSlices; p++)
        *reinterpret_cast<uint64_t*>(E + ((long long)p * m + i) * (3LL * Kp) + (long long)a * Kp + k0) = pk[a][p];
  }
}

// ---------------------------------------------------------------- host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

sr_status get_encode(EncodeFn& fn) {
  static EncodeFn cached = nullptr;
  if (!cached) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    SR_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return SR_ERR_CUDA;
    }
    cached = reinterpret_cast<EncodeFn>(p);
  }
  fn = cached;
  return SR_OK;
}

sr_status make_map(CUtensorMap& m, void* base, long long Kp, long long ncols, int rows, int box_slices = kSlices) {
  EncodeFn enc;
  SR_TRY(get_encode(enc));
  const cuuint64_t dims[3] = {(cuuint64_t)(3 * Kp), (cuuint64_t)ncols, (cuuint64_t)kSlices};
  const cuuint64_t strides[2] = {(cuuint64_t)(3 * Kp), (cuuint64_t)(3 * Kp * ncols)};
  const cuuint32_t box[3] = {(cuuint32_t)BKB, (cuuint32_t)rows, (cuuint32_t)box_slices};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, BKB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return SR_ERR_CUDA;
  }
  return SR_OK;
}

long long pad_k(long long ns) { return std::max<long long>(64, (ns + 63) / 64 * 64); }

sr_status set_attrs() {
  static unsigned long long attr = 0;
  if (first_on_device(attr)) {
    SR_CUDA(cudaFuncSetAttribute(gram_i8<MODE_HERM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    SR_CUDA(cudaFuncSetAttribute(gram_i8<MODE_SUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    SR_CUDA(cudaFuncSetAttribute(gram_i8_2sm<MODE_HERM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem2));
    SR_CUDA(cudaFuncSetAttribute(gram_i8_2sm<MODE_SUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem2));
    SR_CUDA(cudaFuncSetAttribute(oz_split, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSplitSmem));
  }
  return SR_OK;
}

long long lower_tiles(int n, int jlim = 0, int R = 2) {
  const int RT = (n + R * BN - 1) / (R * BN), CT = (n + BN - 1) / BN;
  const int jl = jlim > 0 ? std::min(CT, jlim) : CT;
  long long cnt = 0;
  for (int i = 0; i < RT; i++) cnt += std::min(jl, R * i + R);
  return cnt;
}

// Blocks are processed in groups whose digit slices fit a fixed budget (all blocks at once
// when they fit; the buffer is reused group by group otherwise).
constexpr size_t kSliceBudget = (size_t)6 << 30;
size_t slice_bytes(long long Kp, long long ncols) { return (size_t)kSlices * 3 * Kp * ncols; }

struct Group {
  int b0, b1;
  long long ncols;
};
std::vector<Group> plan(long long Kp, int nblk, const int64_t* offs, size_t& max_bytes) {
  std::vector<Group> g;
  max_bytes = 0;
  int b = 0;
  while (b < nblk) {
    int e = b + 1;
    while (e < nblk && slice_bytes(Kp, offs[e + 1] - offs[b]) <= kSliceBudget && e - b < kMaxBlk) e++;
    g.push_back({b, e, offs[e] - offs[b]});
    max_bytes = std::max(max_bytes, slice_bytes(Kp, offs[e] - offs[b]));
    b = e;
  }
  return g;
}

}  // namespace

size_t workspace_bytes(long long ns, int nblk, const int64_t* offs) {
  const long long Kp = pad_k(ns);
  size_t mb = 0;
  std::vector<Group> g = plan(Kp, nblk, offs, mb);
  long long mc = 0;
  for (auto& x : g) mc = std::max(mc, x.ncols);
  return round256(mb) + round256((size_t)mc * 8) + round256((size_t)mc * 4);
}

// Grid of the block-QGT launch: one persistent CTA per SM by default; SR_GRAM_CTAS=n sets
// n CTAs (more than the SMs makes the kernel non-persistent, so that concurrent work on
// other streams -- the pipelined step's block solves -- gets SMs as CTAs retire).
// CTA-pair Gram kernel (gram_i8_2sm) for the block QGT: SR_GRAM_2SM=1 (experimental).
bool gram_pairs() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SR_GRAM_2SM");
    v = e ? atoi(e) != 0 : 0;
  }
  return v != 0;
}

long long gram_ctas() {
  static long long v = -1;
  if (v < 0) {
    const char* e = getenv("SR_GRAM_CTAS");
    v = e && atoll(e) > 0 ? atoll(e) : kNumSMs;
  }
  return v;
}

// K' per launch of the block-QGT / NTK Gram (SR_OZ_KSPLIT, default 16384).  A tile's K
// stream is K' x 7 slices x 192 rows; the concurrently running tiles share panels only while
// they stay within an L2-sized window of one another, and over a long K they drift apart:
// at K' = 65536 (configs[3]) ncu measured 2.47 TB of DRAM reads for one 16512-column block
// (216x the slice bytes, L2 hit rate 41%), at K' = 16384 64.6 GB (85% hits), and the
// sustained rate 1793 vs 2645 int8 TOPS (0.547 vs 0.374 pJ/op; profiles/README.md).  So a
// long K is cut into launches of K' <= SR_OZ_KSPLIT, each adding its FP64 partial to S in a
// fixed order (the first writes, later ones read-add-write, the last writes the mirror): the
// results stay deterministic and differ from one launch only in FP64 summation order.
long long ksplit_stages() {
  static long long v = -1;
  if (v < 0) {
    const char* e = getenv("SR_OZ_KSPLIT");
    const long long k = e && atoll(e) > 0 ? atoll(e) : 16384;
    v = std::max<long long>(1, k / BKB);
  }
  return v;
}

sr_status launch_herm(const CUtensorMap& ma, const CUtensorMap& mb, Params P, long long total_stages,
                      cudaStream_t st, bool accumulate = false) {
  const long long split = ksplit_stages();
  const unsigned grid = (unsigned)std::min<long long>(P.total_tiles, gram_ctas());
  for (long long s0 = 0; s0 < total_stages; s0 += split) {
    P.kbase = s0;
    P.kstages = (int)std::min(split, total_stages - s0);
    P.acc_in = s0 > 0 || accumulate;
    P.defer = s0 + split < total_stages;
    timer_begin("gram_i8", st);
    gram_i8<MODE_HERM><<<grid, kThreads, kSmem, st>>>(ma, mb, P);
    timer_end(st);
    SR_LAUNCHED();
  }
  return SR_OK;
}

sr_status block_qgt_i8(long long ns, int nblk, const int64_t* offs, const double2* A, long long lda, double2* S,
                       void* ws, size_t ws_bytes, cudaStream_t st, long long ldc, bool accumulate) {
  long long s_total = 0;
  for (int b = 0; b < nblk; b++) s_total += (offs[b + 1] - offs[b]) * (offs[b + 1] - offs[b]);
  if (ns == 0 && accumulate) return SR_OK;
  if (ns == 0) {   // empty batch: S = 0, nothing read
    SR_CUDA(cudaMemsetAsync(S, 0, (size_t)s_total * sizeof(double2), st));
    return SR_OK;
  }
  if (ws_bytes < workspace_bytes(ns, nblk, offs) || !ws) {
    set_error("sr_block_qgt_i8: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  const long long Kp = pad_k(ns);
  size_t mb = 0;
  std::vector<Group> groups = plan(Kp, nblk, offs, mb);
  long long mc = 0;
  for (auto& x : groups) mc = std::max(mc, x.ncols);
  Arena a(ws, ws_bytes);
  int8_t* E = a.take<int8_t>(mb);
  unsigned long long* mx = a.take<unsigned long long>(mc);
  int* expo = a.take<int>(mc);

  SR_TRY(set_attrs());
  long long soff = 0;
  for (const Group& G : groups) {
    const long long c0 = offs[G.b0], nc = G.ncols;
    SR_CUDA(cudaMemsetAsync(mx, 0, (size_t)nc * 8, st));
    {
      const int rows_per = 256;
      dim3 g((unsigned)((nc + 255) / 256), (unsigned)((ns + rows_per - 1) / rows_per));
      oz_colmax<<<g, 256, 0, st>>>(A, lda, c0, (int)nc, ns, rows_per, mx);
      SR_LAUNCHED();
    }
    {
      dim3 g((unsigned)((nc + 31) / 32), (unsigned)(Kp / 64));
      oz_split<<<g, 256, kSplitSmem, st>>>(A, lda, c0, (int)nc, ns, Kp, mx, E, expo);
      SR_LAUNCHED();
    }
    Params P{};
    P.nblk = G.b1 - G.b0;
    P.Kp = Kp;
    P.kstages = (int)(2 * Kp / BKB);
    P.spc = kChunkK / BKB;
    P.expo = expo;
    const bool pair = gram_pairs();
    const int R = pair ? 4 : 2;   // 64-column tiles per row tile (256- or 128-row tiles)
    long long tiles = 0;
    for (int k = 0; k < P.nblk; k++) {
      const int b = G.b0 + k;
      Blk& B = P.b[k];
      B.n = (int)(offs[b + 1] - offs[b]);
      B.col0 = offs[b] - c0;
      B.C = S + soff;
      B.ldc = ldc > 0 ? ldc : B.n;   // ldc > 0: one block written with that leading dimension
      soff += (long long)B.n * B.n;
      B.RT = (B.n + R * BN - 1) / (R * BN);
      B.CT = (B.n + BN - 1) / BN;
      B.tile_begin = tiles;
      tiles += 2 * lower_tiles(B.n, 0, R);
    }
    P.total_tiles = tiles;
    CUtensorMap ma, mb2;
    SR_TRY(make_map(ma, E, Kp, nc, BM, kSplitBar && !gram_pairs() ? 1 : kSlices));
    if (pair) {
      CUtensorMap mbb2, mbb1, mbh;
      SR_TRY(make_map(mbb2, E, Kp, nc, BN, 2));
      SR_TRY(make_map(mbb1, E, Kp, nc, BN, 1));
      SR_TRY(make_map(mbh, E, Kp, nc, BN / 2, 1));
      const unsigned grid = 2 * (unsigned)std::min<long long>(tiles, kNumSMs / 2);
      const long long total = 2 * Kp / BKB, split = ksplit_stages();
      for (long long s0 = 0; s0 < total; s0 += split) {   // K-split launches as launch_herm
        P.kbase = s0;
        P.kstages = (int)std::min(split, total - s0);
        P.acc_in = s0 > 0 || accumulate;
        P.defer = s0 + split < total;
        timer_begin("gram_i8", st);
        gram_i8_2sm<MODE_HERM><<<grid, kThreads, kSmem2, st>>>(ma, mbb2, mbb1, mbh, P);
        timer_end(st);
        SR_LAUNCHED();
      }
    } else {
      SR_TRY(make_map(mb2, E, Kp, nc, BN, kSplitBar ? 1 : kSlices));
      SR_TRY(launch_herm(ma, mb2, P, 2 * Kp / BKB, st, accumulate));
    }
  }
  return SR_OK;
}

size_t trail_workspace_bytes(long long m, long long K) {
  const long long Kp = pad_k(K);
  return round256((size_t)kSlices * 3 * Kp * m) + round256((size_t)m * 4);
}

sr_status trail_split_i8(const double2* L, long long ldl, long long m, long long K, void* ws, size_t ws_bytes,
                         cudaStream_t st) {
  if (m <= 0 || K <= 0) return SR_OK;
  const long long Kp = pad_k(K);
  if (2 * Kp > kChunkK || m >= (1LL << 31) / kSlices) {
    set_error("trail_update_i8: K or m too large");
    return SR_ERR_INVALID;
  }
  if (ws_bytes < trail_workspace_bytes(m, K)) {
    set_error("trail_update_i8: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  Arena a(ws, ws_bytes);
  int8_t* E = a.take<int8_t>((size_t)kSlices * 3 * Kp * m);
  int* expo = a.take<int>(m);
  oz_split_rows<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(L, ldl, (int)m, (int)K, (int)Kp, E, expo);
  SR_LAUNCHED();
  return SR_OK;
}

sr_status trail_apply_i8(long long m, long long K, double2* C, long long ldc, void* ws, long long r0, int jlim,
                         long long ctas, cudaStream_t st) {
  if (m <= r0 || K <= 0) return SR_OK;
  SR_TRY(set_attrs());
  const long long Kp = pad_k(K);
  Arena a(ws, trail_workspace_bytes(m, K));
  int8_t* E = a.take<int8_t>((size_t)kSlices * 3 * Kp * m);
  int* expo = a.take<int>(m);
  Params P{};
  P.nblk = 1;
  P.Kp = Kp;
  P.kstages = (int)(2 * Kp / BKB);
  P.spc = kChunkK / BKB;
  P.expo = expo;
  Blk& B = P.b[0];
  B.col0 = r0;
  B.C = C + r0 * ldc + r0;
  B.ldc = ldc;
  B.n = (int)(m - r0);
  B.RT = (B.n + BM - 1) / BM;
  B.CT = (B.n + BN - 1) / BN;
  B.jlim = jlim;
  B.tile_begin = 0;
  P.total_tiles = 2 * lower_tiles(B.n, jlim);
  CUtensorMap ma, mb;
  SR_TRY(make_map(ma, E, Kp, m, BM, kSplitBar ? 1 : kSlices));
  SR_TRY(make_map(mb, E, Kp, m, BN, kSplitBar ? 1 : kSlices));
  const long long want = ctas > 0 ? ctas : ctas < 0 ? (P.total_tiles + (-ctas) - 1) / (-ctas) : kNumSMs;
  const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(P.total_tiles, want));
  timer_begin("trail_i8", st);
  gram_i8<MODE_SUB><<<grid, kThreads, kSmem, st>>>(ma, mb, P);
  timer_end(st);
  SR_LAUNCHED();
  return SR_OK;
}

sr_status trail_update_i8(const double2* L, long long ldl, long long m, long long K, double2* C, long long ldc,
                          void* ws, size_t ws_bytes, int max_ctas, cudaStream_t st) {
  if (m <= 0 || K <= 0) return SR_OK;
  SR_TRY(trail_split_i8(L, ldl, m, K, ws, ws_bytes, st));
  return trail_apply_i8(m, K, C, ldc, ws, 0, 0, max_ctas, st);
}

size_t rows_workspace_bytes(long long m, long long K) { return trail_workspace_bytes(m, K); }

sr_status gram_rows_i8(const double2* L, long long ldl, long long m, long long K, double2* C, long long ldc, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
  if (m <= 0) return SR_OK;
  if (K <= 0 || m >= (1LL << 31) / kSlices) {
    set_error("gram_rows_i8: bad sizes");
    return SR_ERR_INVALID;
  }
  if (ws_bytes < rows_workspace_bytes(m, K) || !ws) {
    set_error("gram_rows_i8: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  SR_TRY(set_attrs());
  const long long Kp = pad_k(K);
  Arena a(ws, ws_bytes);
  int8_t* E = a.take<int8_t>((size_t)kSlices * 3 * Kp * m);
  int* expo = a.take<int>(m);
  // rows scaled and split with the imaginary part negated (as for the trailing updates), so
  // the column-Gram of the split is sum_k L[i][k] conj(L[j][k])
  oz_split_rows<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(L, ldl, (int)m, (int)K, (int)Kp, E, expo);
  SR_LAUNCHED();
  Params P{};
  P.nblk = 1;
  P.Kp = Kp;
  P.kstages = (int)(2 * Kp / BKB);
  P.spc = kChunkK / BKB;
  P.expo = expo;
  Blk& B = P.b[0];
  B.col0 = 0;
  B.C = C;
  B.ldc = ldc;
  B.n = (int)m;
  B.RT = (B.n + BM - 1) / BM;
  B.CT = (B.n + BN - 1) / BN;
  B.tile_begin = 0;
  P.total_tiles = 2 * lower_tiles(B.n);
  CUtensorMap ma, mb;
  SR_TRY(make_map(ma, E, Kp, m, BM, kSplitBar ? 1 : kSlices));
  SR_TRY(make_map(mb, E, Kp, m, BN, kSplitBar ? 1 : kSlices));
  return launch_herm(ma, mb, P, 2 * Kp / BKB, st);
}

// ---------------------------------------------------------------- rectangles
// The distributed dense full QGT (parallel.dist_full_qgt) needs rectangles of the Gram,
// C = A[:, row0:row0+m]^H A[:, 0:n] (a panel row of S), and rectangular trailing updates,
// C -= L[row0:row0+m] L[0:n]^H (a rank's panel row against the broadcast panel column).  Both
// are the same engine with one "rect" block: the tile grid is the full m x n rectangle
// (column-major), the A operand starts at row0 of the slice matrix, and the epilogue writes
// (or adds, or subtracts) every element, with no conjugate mirror.

size_t cols_workspace_bytes(long long ns, long long ncols) {
  const long long Kp = pad_k(ns);
  return round256(slice_bytes(Kp, ncols)) + round256((size_t)ncols * 8) + round256((size_t)ncols * 4);
}

sr_status cols_prepare(const double2* A, long long lda, long long ns, long long ncols, void* ws, size_t ws_bytes,
                       cudaStream_t st) {
  if (ws_bytes < cols_workspace_bytes(ns, ncols) || !ws) {
    set_error("cols_prepare: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  SR_TRY(set_attrs());
  const long long Kp = pad_k(ns);
  Arena a(ws, ws_bytes);
  int8_t* E = a.take<int8_t>(slice_bytes(Kp, ncols));
  unsigned long long* mx = a.take<unsigned long long>(ncols);
  int* expo = a.take<int>(ncols);
  SR_CUDA(cudaMemsetAsync(mx, 0, (size_t)ncols * 8, st));
  const int rows_per = 256;
  dim3 g1((unsigned)((ncols + 255) / 256), (unsigned)((ns + rows_per - 1) / rows_per));
  oz_colmax<<<g1, 256, 0, st>>>(A, lda, 0, (int)ncols, ns, rows_per, mx);
  SR_LAUNCHED();
  dim3 g2((unsigned)((ncols + 31) / 32), (unsigned)(Kp / 64));
  oz_split<<<g2, 256, kSplitSmem, st>>>(A, lda, 0, (int)ncols, ns, Kp, mx, E, expo);
  SR_LAUNCHED();
  return SR_OK;
}

sr_status cols_rect_gram(long long ns, long long ncols, void* ws, size_t ws_bytes, long long row0, long long m,
                         long long n, double2* C, long long ldc, bool accumulate, cudaStream_t st) {
  if (m <= 0 || n <= 0) return SR_OK;
  if (row0 < 0 || row0 + m > ncols || n > ncols || ws_bytes < cols_workspace_bytes(ns, ncols) || !ws) {
    set_error("cols_rect_gram: bad range or workspace");
    return SR_ERR_INVALID;
  }
  if (ns == 0) {
    if (!accumulate) SR_CUDA(cudaMemset2DAsync(C, ldc * sizeof(double2), 0, n * sizeof(double2), m, st));
    return SR_OK;
  }
  SR_TRY(set_attrs());
  const long long Kp = pad_k(ns);
  Arena a(ws, ws_bytes);
  int8_t* E = a.take<int8_t>(slice_bytes(Kp, ncols));
  a.take<unsigned long long>(ncols);
  int* expo = a.take<int>(ncols);
  Params P{};
  P.nblk = 1;
  P.Kp = Kp;
  P.spc = kChunkK / BKB;
  P.expo = expo;
  Blk& B = P.b[0];
  B.col0 = 0;
  B.rect = 1;
  B.row0 = row0;
  B.m = (int)m;
  B.n = (int)n;
  B.C = C;
  B.ldc = ldc;
  B.RT = (int)((m + BM - 1) / BM);
  B.CT = (int)((n + BN - 1) / BN);
  B.tile_begin = 0;
  P.total_tiles = 2LL * B.RT * B.CT;
  CUtensorMap ma, mb;
  SR_TRY(make_map(ma, E, Kp, ncols, BM, kSplitBar ? 1 : kSlices));
  SR_TRY(make_map(mb, E, Kp, ncols, BN, kSplitBar ? 1 : kSlices));
  return launch_herm(ma, mb, P, 2 * Kp / BKB, st, accumulate);
}

sr_status rows_rect_sub(long long rows, long long K, long long row0, long long m, long long n, double2* C,
                        long long ldc, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (m <= 0 || n <= 0 || K <= 0) return SR_OK;
  if (row0 < 0 || row0 + m > rows || n > rows || ws_bytes < trail_workspace_bytes(rows, K) || !ws) {
    set_error("rows_rect_sub: bad range or workspace");
    return SR_ERR_INVALID;
  }
  SR_TRY(set_attrs());
  const long long Kp = pad_k(K);
  Arena a(ws, trail_workspace_bytes(rows, K));
  int8_t* E = a.take<int8_t>((size_t)kSlices * 3 * Kp * rows);
  int* expo = a.take<int>(rows);
  Params P{};
  P.nblk = 1;
  P.Kp = Kp;
  P.kstages = (int)(2 * Kp / BKB);
  P.spc = kChunkK / BKB;
  P.expo = expo;
  Blk& B = P.b[0];
  B.col0 = 0;
  B.rect = 1;
  B.row0 = row0;
  B.m = (int)m;
  B.n = (int)n;
  B.C = C;
  B.ldc = ldc;
  B.RT = (int)((m + BM - 1) / BM);
  B.CT = (int)((n + BN - 1) / BN);
  B.tile_begin = 0;
  P.total_tiles = 2LL * B.RT * B.CT;
  CUtensorMap ma, mb;
  SR_TRY(make_map(ma, E, Kp, rows, BM, kSplitBar ? 1 : kSlices));
  SR_TRY(make_map(mb, E, Kp, rows, BN, kSplitBar ? 1 : kSlices));
  const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(P.total_tiles, kNumSMs));
  timer_begin("trail_i8", st);
  gram_i8<MODE_SUB><<<grid, kThreads, kSmem, st>>>(ma, mb, P);
  timer_end(st);
  SR_LAUNCHED();
  return SR_OK;
}

}  // namespace oz
cudaError_t trace_install_ozaki(TraceDev t) { return trace_install_local(t); }
}  // namespace sr
