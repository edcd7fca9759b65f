// gram.cuh — FP64 tensor-core (DMMA.8x8x4) complex tile engine.
//
// One engine serves every dense contraction of the step:
//   stage (4)  S_b = A_b^H A_b         (flavor TN: operands K-major, A conjugated)   PAPER.md Eq. 3
//   full QGT   S   = A^H A              (flavor TN)                                   PAPER.md §2
//   NTK        T   = A A^H              (flavor NH: operands row-major along K, B conjugated)
//   Cholesky   trailing update C -= L_p L_p^H and the panel TRSM L_ip = A_ip Linv^H (flavor NH)
// Tile 64x64 complex per CTA, K step 16, 256 threads = 8 warps (2 x 4), warp tile 32x16
// complex = 4 x 2 DMMA 8x8 sub-tiles, each complex product as 4 real DMMAs (re/im planes
// de-interleaved from the LDS.128 of one complex element).  Operand tiles are staged by
// a 3-stage cp.async pipeline (16-byte copies, zero-fill outside the matrix) into padded
// shared-memory tiles whose strides make every fragment load bank-conflict free.
#pragma once
#include <cuda.h>

#include <algorithm>

#include "common.cuh"

namespace sr {
namespace gram {

constexpr int BM = 64;   // tile rows   (complex)
constexpr int BN = 64;   // tile cols   (complex)
constexpr int BK = 16;   // K per stage (complex)
constexpr int kThreads = 256;
constexpr int kMaxProbs = 24;
constexpr int kBand = 16;     // tile rows per rasterisation band (lower-triangle tile sets)

// Operand storage flavors.
//  TN: a(m,k) = conj(A[k*lda + m]), b(k,n) = B[k*ldb + n]   (tile smem [BK][64+2])
//  NH: a(m,k) = A[m*lda + k],       b(k,n) = conj(B[n*ldb + k]) (tile smem [64][BK+4])
enum Flavor { TN = 0, NH = 1 };
// Epilogues: C = tile with conj-transposed mirror (Hermitian result, diagonal imag = 0);
// C -= tile; C = tile.
enum Epi { HERM_STORE = 0, SUB = 1, STORE = 2 };

struct Prob {
  const double2* A;
  const double2* B;
  double2* C;
  long long lda, ldb, ldc;
  int M, N;           // C is M x N (LOWER tile sets use M == N and tiles I >= J)
  long long K;
  int lower;          // 1: tiles with I >= J only; 0: all Mt x Nt tiles
  int tiles_n;        // Nt (column tiles)
  long long tile_begin;
};

struct ProbSet {
  int count;
  long long total_tiles;
  Prob p[kMaxProbs];
};

constexpr int TN_LD = BM + 2;   // 66 complex = 1056 B per k-row  (1056 mod 128 = 32)
constexpr int NH_LD = BK + 4;   // 20 complex =  320 B per m-row  ( 320 mod 128 = 64)
template <int FL>
constexpr int tile_elems() { return FL == TN ? BK * TN_LD : BM * NH_LD; }   // 1056 / 1280
// Pipeline depth: TN (the QGT Gram, long K) 3 stages = 101 KB; NH (Cholesky TRSM/trailing
// update with K = 64, NTK Gram) 2 stages = 82 KB.  Both fit 2 CTAs per SM.
template <int FL>
constexpr int stages() { return FL == TN ? 3 : 2; }
template <int FL>
constexpr size_t smem_bytes() { return (size_t)stages<FL>() * 2 * tile_elems<FL>() * sizeof(double2); }
template <int FL>
constexpr int min_blocks() { return 2; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Load one K-stage of the operand covering rows/cols [r0, r0+64) of the matrix.
// TN: smem[k][m] <- X[(k0+k)*ld + r0+m];  NH: smem[m][k] <- X[(r0+m)*ld + k0+k].
template <int FL>
__device__ __forceinline__ void load_tile(double2* s, const double2* X, long long ld, int r0, int rmax,
                                          long long k0, long long K) {
#pragma unroll
  for (int it = 0; it < (BK * 64) / kThreads; it++) {
    const int e = threadIdx.x + it * kThreads;
    int kk, mm;
    if (FL == TN) {
      kk = e >> 6;
      mm = e & 63;
    } else {
      mm = e >> 4;
      kk = e & 15;
    }
    const long long gk = k0 + kk;
    const int gm = r0 + mm;
    const bool v = (gk < K) && (gm < rmax);
    const double2* src = v ? (FL == TN ? X + gk * ld + gm : X + (long long)gm * ld + gk) : X;
    double2* dst = FL == TN ? s + kk * TN_LD + mm : s + mm * NH_LD + kk;
    cp_async16(dst, src, v);
  }
}

// Fragment fetch: element (row r, k) of a 64-row operand tile.
template <int FL>
__device__ __forceinline__ double2 frag(const double2* s, int r, int k) {
  return FL == TN ? s[k * TN_LD + r] : s[r * NH_LD + k];
}

__device__ __forceinline__ void tile_of(const ProbSet& ps, long long t, int& pi, int& I, int& J) {
  pi = 0;
#pragma unroll 1
  while (pi + 1 < ps.count && t >= ps.p[pi + 1].tile_begin) pi++;
  const long long lt = t - ps.p[pi].tile_begin;
  if (ps.p[pi].lower) {
    // row of lt in row-major lower-triangle order
    long long i = (long long)((sqrt(8.0 * (double)lt + 1.0) - 1.0) * 0.5);
    while ((i + 1) * (i + 2) / 2 <= lt) i++;
    while (i * (i + 1) / 2 > lt) i--;
    // Band rasterisation: rows are grouped in bands of kBand tile rows and each band is
    // walked column-major, so the CTAs resident at one time share few operand strips
    // (L2 reuse of the K-slabs instead of whole-matrix re-reads from HBM per wave).
    const long long T = ps.p[pi].tiles_n;
    const long long r0 = (i / kBand) * kBand, r1 = min(T, r0 + kBand), nb = r1 - r0;
    const long long u = lt - r0 * (r0 + 1) / 2;
    if (u < (r0 + 1) * nb) {
      J = (int)(u / nb);
      I = (int)(r0 + u % nb);
    } else {
      long long v = u - (r0 + 1) * nb, sz = nb - 1, col = r0 + 1;
      while (v >= sz) {
        v -= sz;
        sz--;
        col++;
      }
      J = (int)col;
      I = (int)(col + v);
    }
  } else {
    I = (int)(lt / ps.p[pi].tiles_n);
    J = (int)(lt % ps.p[pi].tiles_n);
  }
}

template <int FL, int EP>
__global__ void __launch_bounds__(kThreads, min_blocks<FL>()) tile_kernel(const __grid_constant__ ProbSet ps) {
  extern __shared__ __align__(16) double2 smem[];
  int pi, I, J;
  tile_of(ps, blockIdx.x, pi, I, J);
  const Prob& P = ps.p[pi];
  const int m0 = I * BM, n0 = J * BN;
  const long long K = P.K;
  const int KT = (int)((K + BK - 1) / BK);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int lr = lane >> 2, lk = lane & 3;

  double acc_r[4][2][2], acc_i[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 2; b++) {
      acc_r[a][b][0] = acc_r[a][b][1] = 0.0;
      acc_i[a][b][0] = acc_i[a][b][1] = 0.0;
    }

  constexpr int TE = tile_elems<FL>();
  constexpr int kStages = stages<FL>();
  auto sA = [&](int st) { return smem + (size_t)st * 2 * TE; };
  auto sB = [&](int st) { return smem + (size_t)st * 2 * TE + TE; };

#pragma unroll
  for (int s = 0; s < kStages - 1; s++) {
    if (s < KT) {
      load_tile<FL>(sA(s), P.A, P.lda, m0, P.M, (long long)s * BK, K);
      load_tile<FL>(sB(s), P.B, P.ldb, n0, P.N, (long long)s * BK, K);
    }
    cp_commit();
  }

#pragma unroll 1
  for (int kt = 0; kt < KT; kt++) {
    cp_wait<kStages - 2>();
    __syncthreads();
    {
      const int nk = kt + kStages - 1;
      const int st = nk % kStages;
      if (nk < KT) {
        load_tile<FL>(sA(st), P.A, P.lda, m0, P.M, (long long)nk * BK, K);
        load_tile<FL>(sB(st), P.B, P.ldb, n0, P.N, (long long)nk * BK, K);
      }
      cp_commit();
    }
    const double2* a_s = sA(kt % kStages);
    const double2* b_s = sB(kt % kStages);
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double ar[4], ai[4], nai[4], br[2], bi[2];
#pragma unroll
      for (int mi = 0; mi < 4; mi++) {
        const double2 v = frag<FL>(a_s, wm * 32 + mi * 8 + lr, k4 + lk);
        ar[mi] = v.x;
        ai[mi] = FL == TN ? -v.y : v.y;   // a(m,k) = conj(.) in TN
        nai[mi] = -ai[mi];
      }
#pragma unroll
      for (int ni = 0; ni < 2; ni++) {
        const double2 v = frag<FL>(b_s, wn * 16 + ni * 8 + lr, k4 + lk);
        br[ni] = v.x;
        bi[ni] = FL == NH ? -v.y : v.y;   // b(k,n) = conj(.) in NH
      }
#pragma unroll
      for (int mi = 0; mi < 4; mi++)
#pragma unroll
        for (int ni = 0; ni < 2; ni++) {
          // (ar + i ai)(br + i bi) = (ar br - ai bi) + i (ar bi + ai br)
          dmma(acc_r[mi][ni][0], acc_r[mi][ni][1], ar[mi], br[ni]);
          dmma(acc_i[mi][ni][0], acc_i[mi][ni][1], ar[mi], bi[ni]);
          dmma(acc_r[mi][ni][0], acc_r[mi][ni][1], nai[mi], bi[ni]);
          dmma(acc_i[mi][ni][0], acc_i[mi][ni][1], ai[mi], br[ni]);
        }
    }
  }
  cp_wait<0>();

  // Epilogue: lane holds C[m][n], C[m][n+1] of each 8x8 sub-tile, m = .. + lane/4,
  // n = .. + 2*(lane%4).
#pragma unroll
  for (int mi = 0; mi < 4; mi++)
#pragma unroll
    for (int ni = 0; ni < 2; ni++) {
      const int m = m0 + wm * 32 + mi * 8 + lr;
      const int nb = n0 + wn * 16 + ni * 8 + 2 * lk;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int n = nb + h;
        if (m >= P.M || n >= P.N) continue;
        double2 v = make_double2(acc_r[mi][ni][h], acc_i[mi][ni][h]);
        double2* c = P.C + (long long)m * P.ldc + n;
        if (EP == HERM_STORE) {
          // lower entries only (m >= n within diagonal tiles), mirrored: the stored matrix
          // is exactly Hermitian with a real diagonal
          if (I == J && m < n) continue;
          if (m == n) v.y = 0.0;
          *c = v;
          if (m != n) P.C[(long long)n * P.ldc + m] = cconj(v);
        } else if (EP == SUB) {
          *c = csub(*c, v);
        } else {
          *c = v;
        }
      }
    }
}

// ---------------------------------------------------------------- TN with TMA staging
// The TN flavour (the QGT Grams: every problem a column range of ONE row-major matrix X)
// with its K-slabs staged by TMA instead of cp.async: per stage and 64-column panel, eight
// 2-D boxes of 16 rows x 8 complex (128 bytes, 128-byte swizzle), completing on an
// mbarrier; one thread issues the copies.  Element (k, m) of a panel lives at
//   (m / 8) * 2048 + k * 128 + ((m % 8) ^ (k % 8)) * 16
// so the DMMA fragment loads (8 columns x 4 k per quarter-warp) stay bank-conflict free
// without padding.  Rows past K and columns past the matrix read as zero (TMA OOB fill);
// columns past a problem's range belong to its neighbour and only reach masked outputs.
constexpr int TMA_PANEL = BK * BM * 16;            // 16 KB per 64-column panel
constexpr int TMA_STAGES = 3;
constexpr size_t kTmaSmem = (size_t)TMA_STAGES * 2 * TMA_PANEL + 1024 + 64;

__device__ __forceinline__ double2 frag_sw(const uint8_t* panel, int m, int k) {
  return *reinterpret_cast<const double2*>(panel + (m >> 3) * 2048 + k * 128 + (((m & 7) ^ (k & 7)) << 4));
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done)
                 : "r"(bar), "r"(parity)
                 : "memory");
}

template <int EP>
__global__ void __launch_bounds__(kThreads, 2) tn_tma_kernel(const __grid_constant__ ProbSet ps,
                                                             const __grid_constant__ CUtensorMap map,
                                                             const double2* __restrict__ base) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + TMA_STAGES * 2 * TMA_PANEL);
  int pi, I, J;
  tile_of(ps, blockIdx.x, pi, I, J);
  const Prob& P = ps.p[pi];
  const int m0 = I * BM, n0 = J * BN;
  const long long K = P.K;
  const int KT = (int)((K + BK - 1) / BK);
  // column coordinates (in doubles) of the two panels inside the matrix
  const int ca = (int)(2 * ((P.A - base) + m0)), cb = (int)(2 * ((P.B - base) + n0));
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int lr = lane >> 2, lk = lane & 3;
  auto issue = [&](int kt) {   // thread 0: slab kt into stage kt % TMA_STAGES
    const int st = kt % TMA_STAGES;
    const uint32_t bar = bar0 + 8 * st;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(2 * TMA_PANEL) : "memory");
    const uint32_t da = sbase + st * 2 * TMA_PANEL, db = da + TMA_PANEL;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      tma2d(da + q * 2048, &map, ca + 16 * q, kt * BK, bar);
      tma2d(db + q * 2048, &map, cb + 16 * q, kt * BK, bar);
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < TMA_STAGES; s++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0 + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < TMA_STAGES - 1 && s < KT; s++) issue(s);

  double acc_r[4][2][2], acc_i[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 2; b++) {
      acc_r[a][b][0] = acc_r[a][b][1] = 0.0;
      acc_i[a][b][0] = acc_i[a][b][1] = 0.0;
    }
#pragma unroll 1
  for (int kt = 0; kt < KT; kt++) {
    __syncthreads();   // every warp is done with slab kt-1, whose stage the next issue refills
    if (threadIdx.x == 0 && kt + TMA_STAGES - 1 < KT) issue(kt + TMA_STAGES - 1);
    const int st = kt % TMA_STAGES;
    mbar_wait_parity(bar0 + 8 * st, (uint32_t)((kt / TMA_STAGES) & 1));
    const uint8_t* a_s = sm + st * 2 * TMA_PANEL;
    const uint8_t* b_s = a_s + TMA_PANEL;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double ar[4], ai[4], nai[4], br[2], bi[2];
#pragma unroll
      for (int mi = 0; mi < 4; mi++) {
        const double2 v = frag_sw(a_s, wm * 32 + mi * 8 + lr, k4 + lk);
        ar[mi] = v.x;
        ai[mi] = -v.y;   // a(m,k) = conj(A[k][m])
        nai[mi] = v.y;
      }
#pragma unroll
      for (int ni = 0; ni < 2; ni++) {
        const double2 v = frag_sw(b_s, wn * 16 + ni * 8 + lr, k4 + lk);
        br[ni] = v.x;
        bi[ni] = v.y;
      }
#pragma unroll
      for (int mi = 0; mi < 4; mi++)
#pragma unroll
        for (int ni = 0; ni < 2; ni++) {
          dmma(acc_r[mi][ni][0], acc_r[mi][ni][1], ar[mi], br[ni]);
          dmma(acc_i[mi][ni][0], acc_i[mi][ni][1], ar[mi], bi[ni]);
          dmma(acc_r[mi][ni][0], acc_r[mi][ni][1], nai[mi], bi[ni]);
          dmma(acc_i[mi][ni][0], acc_i[mi][ni][1], ai[mi], br[ni]);
        }
    }
  }
#pragma unroll
  for (int mi = 0; mi < 4; mi++)
#pragma unroll
    for (int ni = 0; ni < 2; ni++) {
      const int m = m0 + wm * 32 + mi * 8 + lr;
      const int nb = n0 + wn * 16 + ni * 8 + 2 * lk;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int n = nb + h;
        if (m >= P.M || n >= P.N) continue;
        double2 v = make_double2(acc_r[mi][ni][h], acc_i[mi][ni][h]);
        double2* c = P.C + (long long)m * P.ldc + n;
        if (EP == HERM_STORE) {
          if (I == J && m < n) continue;
          if (m == n) v.y = 0.0;
          *c = v;
          if (m != n) P.C[(long long)n * P.ldc + m] = cconj(v);
        } else if (EP == SUB) {
          *c = csub(*c, v);
        } else {
          *c = v;
        }
      }
    }
}

// Host helpers -----------------------------------------------------------------
inline int tiles(long long n, int b) { return (int)((n + b - 1) / b); }

inline void add_prob(ProbSet& ps, const double2* A, long long lda, const double2* B, long long ldb, double2* C,
                     long long ldc, int M, int N, long long K, bool lower) {
  Prob& p = ps.p[ps.count];
  p.A = A;
  p.B = B;
  p.C = C;
  p.lda = lda;
  p.ldb = ldb;
  p.ldc = ldc;
  p.M = M;
  p.N = N;
  p.K = K;
  p.lower = lower ? 1 : 0;
  const int tm = tiles(M, BM), tn = tiles(N, BN);
  p.tiles_n = tn;
  p.tile_begin = ps.total_tiles;
  ps.total_tiles += lower ? (long long)tm * (tm + 1) / 2 : (long long)tm * tn;
  ps.count++;
}

template <int FL, int EP>
inline sr_status launch(const ProbSet& ps, cudaStream_t st) {
  if (ps.total_tiles == 0) return SR_OK;
  static unsigned long long attr_set = 0;
  if (first_on_device(attr_set)) {
    SR_CUDA(cudaFuncSetAttribute(tile_kernel<FL, EP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem_bytes<FL>()));
  }
  tile_kernel<FL, EP><<<(unsigned)ps.total_tiles, kThreads, smem_bytes<FL>(), st>>>(ps);
  SR_LAUNCHED();
  return SR_OK;
}

// Skinny products of the Cholesky panel chain (flavor NH, K <= 64, N <= 64): the panel
// TRSM L_ip = A_ip Linv_p^H and the in-strip updates C -= L_i L_j^H are M x 64 x 64 with M
// up to the block size.  One 64x64 tile per CTA leaves most SMs idle and its 4-step
// pipeline latency (~20 us) sits on the critical path; here a CTA owns 16 full rows
// (all 64 columns, so the in-place TRSM reads its rows before anyone writes them), the whole
// K = 64 is staged in two cp.async halves, and 4 warps each take 16 columns.
// The off-chain in-strip updates use 32-row CTAs (TM = 32: B staged once per 32 rows).
constexpr int SK_LD = 68;   // 1088 B per row (mod 128 = 64: conflict-free LDS.128 fragments)
constexpr int SK_THREADS = 128;
template <int TM>
constexpr size_t skinny_smem() { return (size_t)(TM + 64) * SK_LD * sizeof(double2); }   // 87 / 104 KB

template <int EP, int SK_TM = 16, bool KLOOP = false>
__global__ void __launch_bounds__(SK_THREADS, 2) skinny_kernel(const __grid_constant__ ProbSet ps) {
  constexpr int MI = SK_TM / 8;
  TraceScope trace_(EP == STORE ? TR_TRSM : TR_SKINNY_SUB, (int)ps.p[0].M);
  extern __shared__ __align__(16) double2 smem[];
  double2* sa = smem;
  double2* sb = smem + SK_TM * SK_LD;
  int pi = 0;
#pragma unroll 1
  while (pi + 1 < ps.count && (long long)blockIdx.x >= ps.p[pi + 1].tile_begin) pi++;
  const Prob& P = ps.p[pi];
  const int m0 = (int)((long long)blockIdx.x - P.tile_begin) * SK_TM;
  const long long K = P.K;
  pdl_wait();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = lane >> 2, lk = lane & 3;
  double acc_r[MI][2][2], acc_i[MI][2][2];
#pragma unroll
  for (int a = 0; a < MI; a++)
#pragma unroll
    for (int b = 0; b < 2; b++) {
      acc_r[a][b][0] = acc_r[a][b][1] = 0.0;
      acc_i[a][b][0] = acc_i[a][b][1] = 0.0;
    }
  // K in chunks of 64: one chunk (straight-line, KLOOP = false) for the chain's K = 64
  // products; the left-looking column updates of a strip have K up to 64 (kStrip - 2)
  const long long kend = KLOOP ? K : 1;
#pragma unroll 1
  for (long long kc = 0; kc < kend; kc += 64) {
    if (kc > 0) __syncthreads();   // the previous chunk has been consumed
#pragma unroll
    for (int h = 0; h < 2; h++) {   // two commit groups: k in [32h, 32h + 32)
#pragma unroll
      for (int it = 0; it < (SK_TM * 32) / SK_THREADS; it++) {
        const int e = threadIdx.x + it * SK_THREADS;
        const int r = e >> 5, k = 32 * h + (e & 31);
        const bool v = (m0 + r < P.M) && (kc + k < K);
        cp_async16(sa + r * SK_LD + k, v ? P.A + (long long)(m0 + r) * P.lda + kc + k : P.A, v);
      }
#pragma unroll
      for (int it = 0; it < (64 * 32) / SK_THREADS; it++) {
        const int e = threadIdx.x + it * SK_THREADS;
        const int r = e >> 5, k = 32 * h + (e & 31);
        const bool v = (r < P.N) && (kc + k < K);
        cp_async16(sb + r * SK_LD + k, v ? P.B + (long long)r * P.ldb + kc + k : P.B, v);
      }
      cp_commit();
    }
#pragma unroll
    for (int h = 0; h < 2; h++) {
      if (h == 0) cp_wait<1>(); else cp_wait<0>();
      __syncthreads();
#pragma unroll
      for (int k4 = 32 * h; k4 < 32 * h + 32; k4 += 4) {
        double ar[MI], ai[MI], nai[MI], br[2], bi[2];
#pragma unroll
        for (int mi = 0; mi < MI; mi++) {
          const double2 v = sa[(mi * 8 + lr) * SK_LD + k4 + lk];
          ar[mi] = v.x;
          ai[mi] = v.y;
          nai[mi] = -v.y;
        }
#pragma unroll
        for (int ni = 0; ni < 2; ni++) {
          const double2 v = sb[(w * 16 + ni * 8 + lr) * SK_LD + k4 + lk];
          br[ni] = v.x;
          bi[ni] = -v.y;   // b(k,n) = conj(B[n][k])
        }
#pragma unroll
        for (int mi = 0; mi < MI; mi++)
#pragma unroll
          for (int ni = 0; ni < 2; ni++) {
            dmma(acc_r[mi][ni][0], acc_r[mi][ni][1], ar[mi], br[ni]);
            dmma(acc_i[mi][ni][0], acc_i[mi][ni][1], ar[mi], bi[ni]);
            dmma(acc_r[mi][ni][0], acc_r[mi][ni][1], nai[mi], bi[ni]);
            dmma(acc_i[mi][ni][0], acc_i[mi][ni][1], ai[mi], br[ni]);
          }
      }
    }
  }
#pragma unroll
  for (int mi = 0; mi < MI; mi++)
#pragma unroll
    for (int ni = 0; ni < 2; ni++) {
      const int m = m0 + mi * 8 + lr;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int n = w * 16 + ni * 8 + 2 * lk + h;
        if (m >= P.M || n >= P.N) continue;
        const double2 v = make_double2(acc_r[mi][ni][h], acc_i[mi][ni][h]);
        double2* c = P.C + (long long)m * P.ldc + n;
        *c = EP == SUB ? csub(*c, v) : v;
      }
    }
  pdl_trigger();
}

// Launch a set of NH problems with N <= 64 and K <= 64 (not lower) on the skinny kernel.
template <int EP, int SK_TM, bool KLOOP>
inline sr_status launch_skinny_k(const ProbSet& ps, long long total, cudaStream_t st, bool pdl) {
  constexpr size_t kSkinnySmem = skinny_smem<SK_TM>();
  static unsigned long long attr_set = 0;
  if (first_on_device(attr_set)) {
    SR_CUDA(cudaFuncSetAttribute(skinny_kernel<EP, SK_TM, KLOOP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSkinnySmem));
  }
  if (pdl)
    SR_CUDA(launch_pdl(skinny_kernel<EP, SK_TM, KLOOP>, dim3((unsigned)total), dim3(SK_THREADS), kSkinnySmem, st, ps));
  else
    skinny_kernel<EP, SK_TM, KLOOP><<<(unsigned)total, SK_THREADS, kSkinnySmem, st>>>(ps);
  SR_LAUNCHED();
  return SR_OK;
}

template <int EP, int SK_TM = 16>
inline sr_status launch_skinny(ProbSet ps, cudaStream_t st, bool pdl = false) {
  static_assert(EP == SUB || EP == STORE, "skinny epilogues: SUB or STORE");
  long long total = 0, kmax = 0;
  for (int i = 0; i < ps.count; i++) {
    if (ps.p[i].N > 64 || ps.p[i].lower || (EP == STORE && ps.p[i].K > 64)) return SR_ERR_INVALID;
    ps.p[i].tile_begin = total;
    total += (ps.p[i].M + SK_TM - 1) / SK_TM;
    kmax = std::max(kmax, (long long)ps.p[i].K);
  }
  if (total == 0) return SR_OK;
  if (kmax > 64) return launch_skinny_k<EP, SK_TM, true>(ps, total, st, pdl);
  return launch_skinny_k<EP, SK_TM, false>(ps, total, st, pdl);
}

using TmaEncode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// TN problems that are all column ranges of one row-major matrix X (ncols columns, K rows,
// leading dimension ld complex) on the TMA-staged kernel.
template <int EP>
inline sr_status launch_tn_tma(const ProbSet& ps, const double2* X, long long ld, long long ncols, long long K,
                               cudaStream_t st) {
  if (ps.total_tiles == 0) return SR_OK;
  // The one tensor map covers X: every problem must be a Hermitian Gram of a column range of
  // X (A == B inside [X, X + ncols), the same ld and K).  Anything else takes the cp.async
  // kernel, which reads each problem's own pointers.
  for (int i = 0; i < ps.count; i++) {
    const Prob& p = ps.p[i];
    const long long c0 = p.A - X;
    if (p.A != p.B || p.lda != ld || p.ldb != ld || p.K != K || c0 < 0 || c0 + p.N > ncols || p.M != p.N)
      return launch<TN, EP>(ps, st);
  }
  static TmaEncode enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    SR_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return SR_ERR_CUDA;
    }
    enc = reinterpret_cast<TmaEncode>(p);
  }
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)(2 * ncols), (cuuint64_t)std::max(1LL, K)};
  const cuuint64_t strides[1] = {(cuuint64_t)(16 * ld)};
  const cuuint32_t box[2] = {16, (cuuint32_t)BK};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double2*>(X), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (FP64 Gram): " + std::to_string((int)r));
    return SR_ERR_CUDA;
  }
  static unsigned long long attr_set = 0;
  if (first_on_device(attr_set)) {
    SR_CUDA(cudaFuncSetAttribute(tn_tma_kernel<EP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem));
  }
  tn_tma_kernel<EP><<<(unsigned)ps.total_tiles, kThreads, kTmaSmem, st>>>(ps, map, X);
  SR_LAUNCHED();
  return SR_OK;
}

}  // namespace gram
}  // namespace sr
