// chol_diag.cuh — the 64x64 diagonal-tile kernel of the blocked Cholesky (chol.cu).  In its
// own header so tools/diag_probe.cu can time its phases (SR_DIAG_PROBE hook, empty here).
#pragma once
#include "chol.cuh"

#ifndef SR_DIAG_PROBE
#define SR_DIAG_PROBE(i)
#endif
#ifndef SR_DIAG_ISOLATE
#define SR_DIAG_ISOLATE 1
#endif
#ifndef SR_DIAG_BS
#define SR_DIAG_BS 8   // diagonal sub-block of the single-warp factor (8 or 16)
#endif

namespace sr {
namespace cholk {

constexpr int NB = 64;

// One CTA per block: factor the 64x64 diagonal tile of panel p, form its inverse
// X = Linv_p and y_p = Linv_p b_p.  Blocked by BS = 8 (the latency of a 64-step column
// recursion with a block barrier per step is what limited the unblocked forms; 8 beat 16,
// tools/diag_probe.cu: 66.6k vs 75.3k cycles):
//   for each BS-column block k (offset o = BS k):
//     (a) warp 0 factors D_k = A[o:o+BS, o:o+BS] in registers, lane r = row r, columns
//         broadcast through shared memory, 1/sqrt of each pivot kept in dinv;
//     (b) rows r >= o+BS solve x D_k^H = A[r, o:o+BS] (a quad per row, right-looking);
//     (c) A[r][s] -= sum_m L[r][o+m] conj(L[s][o+m]) on the trailing lower triangle
//         (2x2 register patches), overlapped with (a) of the next block.
//   inverse: X_kk = D_k^{-1} (warp k, lane j = column j), then by block distance d = 1..3:
//     W_ik = sum_{j=k}^{i-1} L_ij X_jk and X_ik = -X_ii W_ik (i = k + d), 2x2 patches.
constexpr int LDT = NB + 1;   // 1040-byte rows
constexpr size_t kDiagSmem = ((size_t)2 * NB * LDT + 32 * 33) * sizeof(double2);   // T, X, W

__device__ __forceinline__ void cfma_conjb(double2& acc, double2 a, double2 b) {   // acc += a conj(b)
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.y, b.x, acc.y);
  acc.y = fma(-a.x, b.y, acc.y);
}

// (a) warp 0: D = L L^H for the 16x16 block at (o, o) of T, in place.  Lane r < 16 holds
// row r; step c scales column c, publishes it to T (one __syncwarp) and applies the
// rank-1 update to the later columns of its row, reading L[s][c] back as shared-memory
// broadcasts.  Every lane also keeps the running diagonal dg[s] = A_ss - sum_k |L_sk|^2
// (the same arithmetic as the owner's update of its own diagonal entry), so each step's
// pivot is available locally without a broadcast.
template <int BS>
__device__ __forceinline__ void factorb(double2* T, int o, int lane, double* dinv, int* bad) {
  double2 d[BS];
  double dg[BS];
  const int r = lane;
#pragma unroll
  for (int s = 0; s < BS; s++) {
    d[s] = (r < BS && s <= r) ? T[(o + r) * LDT + o + s] : make_double2(0.0, 0.0);
    dg[s] = T[(o + s) * LDT + o + s].x;
  }
#pragma unroll
  for (int c = 0; c < BS; c++) {
    double piv = dg[c];
    if (!(piv > 0.0)) {
      if (lane == 0 && *bad == 0) *bad = o + c + 1;
      piv = 1.0;
    }
    const double isd = rsqrt(piv);
    if (r == c) d[c] = make_double2(piv * isd, 0.0);
    else if (r > c) d[c] = cscale(d[c], isd);
    if (r < BS && r >= c) T[(o + r) * LDT + o + c] = d[c];
    if (lane == 0) dinv[o + c] = isd;
    __syncwarp();
#pragma unroll
    for (int s = 1; s < BS; s++) {
      if (s <= c) continue;
      const double2 ls = T[(o + s) * LDT + o + c];   // L[s][c]
      dg[s] -= ls.x * ls.x + ls.y * ls.y;
      if (r >= s && r < BS) {
        double2 v = d[s];
        v.x -= d[c].x * ls.x + d[c].y * ls.y;
        v.y -= d[c].y * ls.x - d[c].x * ls.y;
        d[s] = v;
      }
    }
  }
}

// (a') BS = 8, the form used: lane r < 8 holds row r of the block in registers; step c
// takes column c from lanes s > c by shuffles (no shared-memory round trip, no redundant
// per-lane diagonal), and lane c+1 forms the next pivot A[c+1][c+1] - |A[c+1][c]|^2 isd^2
// before the rank-1 update.  (Spreading the block over all 32 lanes, two entries per
// lane, measured slower: 3.5k vs 2.9k cycles per 8x8 factor, tools/diag_probe.cu.)
__device__ __forceinline__ void factor8(double2* T, int o, int lane, double* dinv, int* bad) {
  const int r = lane & 7;
  double2 d[8];
#pragma unroll
  for (int s = 0; s < 8; s++) d[s] = s <= r ? T[(o + r) * LDT + o + s] : make_double2(0.0, 0.0);
  double piv = __shfl_sync(0xffffffffu, d[0].x, 0);
#pragma unroll
  for (int c = 0; c < 8; c++) {
    if (!(piv > 0.0)) {
      if (lane == 0 && *bad == 0) *bad = o + c + 1;
      piv = 1.0;
    }
    const double n2 = d[c].x * d[c].x + d[c].y * d[c].y;
    const double isd = rsqrt(piv);
    double pn = 0.0;
    if (c < 7) pn = __shfl_sync(0xffffffffu, d[c < 7 ? c + 1 : 7].x - n2 * (isd * isd), c < 7 ? c + 1 : 7);
    if (r == c) d[c] = make_double2(piv * isd, 0.0);
    else if (r > c) d[c] = cscale(d[c], isd);
    if (lane == 0) dinv[o + c] = isd;
#pragma unroll
    for (int s = c + 1; s < 8; s++) {
      const double lx = __shfl_sync(0xffffffffu, d[c].x, s), ly = __shfl_sync(0xffffffffu, d[c].y, s);
      if (r >= s) {   // d[s] -= L[r][c] conj(L[s][c])
        d[s].x -= d[c].x * lx + d[c].y * ly;
        d[s].y -= d[c].y * lx - d[c].x * ly;
      }
    }
    piv = pn;
  }
  if (lane < 8) {
#pragma unroll
    for (int s = 0; s < 8; s++)
      if (s <= r) T[(o + r) * LDT + o + s] = d[s];
  }
}

// (b) rows below the block solve x D^H = A[r, o:o+16] with D = L[o:o+16, o:o+16]
// (diagonal real, 1/D_cc in dinv): a quad per row, lane q holding entries m = q mod 4;
// step c: x_c = a_c / D_cc from the owner lane, shuffled inside the quad, then
// a_m -= x_c conj(D[m][c]) for m > c.
template <int BS>
__device__ __forceinline__ void trsm_quad(double2* T, int o, int r, int q, const double* dinv) {
  double2 a[BS / 4];
#pragma unroll
  for (int k = 0; k < BS / 4; k++) a[k] = T[r * LDT + o + 4 * k + q];
#pragma unroll
  for (int c = 0; c < BS; c++) {
    if (q == (c & 3)) {   // owner: x_c final, published in place
      a[c >> 2] = cscale(a[c >> 2], dinv[o + c]);
      T[r * LDT + o + c] = a[c >> 2];
    }
    __syncwarp();
    const double2 x = T[r * LDT + o + c];
#pragma unroll
    for (int k = 0; k < BS / 4; k++) {
      const int m = 4 * k + q;
      if (m > c) {
        const double2 dm = T[(o + m) * LDT + o + c];
        a[k].x -= x.x * dm.x + x.y * dm.y;
        a[k].y -= x.y * dm.x - x.x * dm.y;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < BS / 4; k++) T[r * LDT + o + 4 * k + q] = a[k];
}

// Lower-triangle patch index e -> (pi, pj), pi >= pj.
__device__ __forceinline__ void tri_patch(int e, int& pi, int& pj) {
  pi = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  while ((pi + 1) * (pi + 2) / 2 <= e) pi++;
  while (pi * (pi + 1) / 2 > e) pi--;
  pj = e - pi * (pi + 1) / 2;
}

// (c) trailing update of rows/cols [o+BS, 64) by the BS columns L[:, o:o+BS], by threads
// t in [0, nt); with skip_next the BS x BS diagonal block at o+BS is left to syrkb_diag.
template <int BS>
__device__ __forceinline__ void syrkb(double2* T, int o, int t, int nt, bool skip_next) {
  const int b0 = o + BS, P = (NB - b0) / 2, cnt = P * (P + 1) / 2;
  for (int e = t; e < cnt; e += nt) {
    int pi, pj;
    tri_patch(e, pi, pj);
    if (skip_next && pi < BS / 2) continue;   // patch rows (and so columns) inside block o+BS
    const int r0 = b0 + 2 * pi, s0 = b0 + 2 * pj;
    double2 acc[2][2] = {{make_double2(0.0, 0.0), make_double2(0.0, 0.0)},
                         {make_double2(0.0, 0.0), make_double2(0.0, 0.0)}};
#pragma unroll 4
    for (int m = 0; m < BS; m++) {
      const double2 lr0 = T[r0 * LDT + o + m], lr1 = T[(r0 + 1) * LDT + o + m];
      const double2 ls0 = T[s0 * LDT + o + m], ls1 = T[(s0 + 1) * LDT + o + m];
      cfma_conjb(acc[0][0], lr0, ls0);
      cfma_conjb(acc[0][1], lr0, ls1);
      cfma_conjb(acc[1][0], lr1, ls0);
      cfma_conjb(acc[1][1], lr1, ls1);
    }
#pragma unroll
    for (int u = 0; u < 2; u++)
#pragma unroll
      for (int v = 0; v < 2; v++)
        if (r0 + u >= s0 + v) {
          double2& x = T[(r0 + u) * LDT + s0 + v];
          x = csub(x, acc[u][v]);
        }
  }
}

// Warp 0: the diagonal block at o+BS receives block o's update (BS(BS+1)/2 lower entries).
template <int BS>
__device__ __forceinline__ void syrkb_diag(double2* T, int o, int lane) {
  const int b0 = o + BS;
  for (int e = lane; e < BS * (BS + 1) / 2; e += 32) {
    int r, c;
    tri_patch(e, r, c);
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int m = 0; m < BS; m++) cfma_conjb(acc, T[(b0 + r) * LDT + o + m], T[(b0 + c) * LDT + o + m]);
    double2& x = T[(b0 + r) * LDT + b0 + c];
    x = csub(x, acc);
  }
}

// X[o:o+16, o:o+16] = L[o:o+16, o:o+16]^{-1} (lane j < 16 = column j; zeros above the diagonal).
__device__ __forceinline__ void inv16(const double2* T, double2* X, int o, int lane, const double* dinv) {
  if (lane >= 16) return;
  const int j = lane;
  double2 b[16];
#pragma unroll
  for (int i = 0; i < 16; i++) b[i] = make_double2(i == j ? 1.0 : 0.0, 0.0);
#pragma unroll
  for (int i = 0; i < 16; i++) {
    const double2 x = cscale(b[i], dinv[o + i]);
    X[(o + i) * LDT + o + j] = x;
#pragma unroll
    for (int m = i + 1; m < 16; m++) {
      const double2 l = T[(o + m) * LDT + o + i];
      b[m].x -= l.x * x.x - l.y * x.y;
      b[m].y -= l.x * x.y + l.y * x.x;
    }
  }
}

// 8x8 complex tile on DMMA: C += sum_{k in [k0, k1)} A[r][k] B[k][c] for r, c < 8, with A and
// B row-major in shared memory (k0, k1 multiples of 4).  Lane l holds C[l/4][2(l%4) + {0,1}].
constexpr int LDW = 33;
__device__ __forceinline__ void dmma_t(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void tile_mma(const double2* A, int lda, const double2* B, int ldb, int k0, int k1, int lane,
                                         double* cr, double* ci) {
  const int lr = lane >> 2, lk = lane & 3;
#pragma unroll 4
  for (int k = k0; k < k1; k += 4) {
    const double2 a = A[lr * lda + k + lk], b = B[(k + lk) * ldb + lr];
    dmma_t(cr[0], cr[1], a.x, b.x);
    dmma_t(cr[0], cr[1], -a.y, b.y);
    dmma_t(ci[0], ci[1], a.x, b.y);
    dmma_t(ci[0], ci[1], a.y, b.x);
  }
}
__device__ __forceinline__ void tile_put(double2* C, int ldc, int lane, const double* cr, const double* ci, double sg) {
  const int lr = lane >> 2, lk = lane & 3;
  C[lr * ldc + 2 * lk] = make_double2(sg * cr[0], sg * ci[0]);
  C[lr * ldc + 2 * lk + 1] = make_double2(sg * cr[1], sg * ci[1]);
}

// C[r][c] -= sum_{m < 8} L[r][o+m] conj(L[c][o+m]) for the 8x8 tile at (r0, c0), r >= c only.
__device__ __forceinline__ void syrk_tile(double2* T, int o, int r0, int c0, int lane) {
  const int lr = lane >> 2, lk = lane & 3;
  double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
#pragma unroll
  for (int k = 0; k < 8; k += 4) {
    const double2 a = T[(r0 + lr) * LDT + o + k + lk], b = T[(c0 + lr) * LDT + o + k + lk];
    dmma_t(cr[0], cr[1], a.x, b.x);
    dmma_t(cr[0], cr[1], a.y, b.y);
    dmma_t(ci[0], ci[1], a.y, b.x);
    dmma_t(ci[0], ci[1], -a.x, b.y);
  }
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int r = r0 + lr, c = c0 + 2 * lk + h;
    if (r >= c) {
      double2& x = T[r * LDT + c];
      x = make_double2(x.x - cr[h], x.y - ci[h]);
    }
  }
}

// (c') BS = 8 trailing update on DMMA: A[r][s] -= sum_m L[r][o+m] conj(L[s][o+m]) over
// 8x8 tiles (I >= J) of the trailing triangle, one tile per warp at a time; the tile of
// the next diagonal block is left to warp 0 (syrk_diag_mma).
__device__ __forceinline__ void syrk_mma(double2* T, int o, int wi, int nw, int lane) {
  const int b0 = o + 8, nb = (NB - b0) / 8, cnt = nb * (nb + 1) / 2;
  for (int e = wi; e < cnt; e += nw) {
    int I, J;
    tri_patch(e, I, J);
    if (I == 0) continue;
    syrk_tile(T, o, b0 + 8 * I, b0 + 8 * J, lane);
  }
}

// Warp 0: the next diagonal block (o+8, o+8) receives block o's update (one DMMA tile).
__device__ __forceinline__ void syrk_diag_mma(double2* T, int o, int lane) { syrk_tile(T, o, o + 8, o + 8, lane); }

__global__ void __launch_bounds__(256) chol_diag(const CholBlock B, int* info, int p, int p0) {
  extern __shared__ double2 dsm[];
  double2* T = dsm;              // [64][LDT]: A (lower) -> L
  double2* X = dsm + NB * LDT;   // [64][LDT]: Linv (lower)
  __shared__ double dinv[NB];
  __shared__ double2 bsh[NB];
  __shared__ int bad;
  const long long np = B.npad;
  double2* tile = B.Fm + (long long)p * NB * np + (long long)p * NB;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  pdl_wait();
  SR_DIAG_PROBE(0);
  {   // 16 independent loads per thread in flight, then the shared-memory stores
    double2 v[16];
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const int e = t + 256 * u, r = e >> 6, c = e & 63;
      v[u] = c <= r ? tile[(long long)r * np + c] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const int e = t + 256 * u, r = e >> 6, c = e & 63;
      if (c <= r) T[r * LDT + c] = v[u];
    }
  }
  {   // b_p -= sum over the strip's earlier panels q in [p0, p) of L_pq y_q (rows of panel p)
    const int r = t >> 2, q = t & 3;
    const double2* lrow = B.Fm + ((long long)p * NB + r) * np;
    double2 sa[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    const int c0 = p0 * NB + q, c1 = p * NB;   // c1 - c0 + q is a multiple of 64
    for (int c = c0; c < c1; c += 16) {
#pragma unroll
      for (int u = 0; u < 4; u++) cfma(sa[u], lrow[c + 4 * u], B.rhs[c + 4 * u]);
    }
    double2 s2 = cadd(cadd(sa[0], sa[1]), cadd(sa[2], sa[3]));
    s2.x += __shfl_xor_sync(0xffffffffu, s2.x, 1);
    s2.y += __shfl_xor_sync(0xffffffffu, s2.y, 1);
    s2.x += __shfl_xor_sync(0xffffffffu, s2.x, 2);
    s2.y += __shfl_xor_sync(0xffffffffu, s2.y, 2);
    if (q == 0) bsh[r] = csub(B.rhs[(long long)p * NB + r], s2);
  }
  if (t == 0) bad = 0;
  __syncthreads();
  SR_DIAG_PROBE(1);
  // Block k (BS columns): warp 0 applies block k-1's update to the diagonal block k and
  // factors it while warps 1-7 apply block k-1's update to the rest of the trailing
  // triangle (the SYRK is off the critical path); then every warp solves the rows below.
  constexpr int BS = SR_DIAG_BS;
  static_assert(BS == 8 || BS == 16, "diagonal sub-block must be 8 or 16");
  for (int k = 0; k < NB / BS; k++) {
    const int o = BS * k;
    if (warp == 0) {
      if (k > 0) {
        if (BS == 8) syrk_diag_mma(T, o - BS, lane);
        else syrkb_diag<BS>(T, o - BS, lane);
      }
      __syncwarp();
      if (BS == 8) factor8(T, o, lane, dinv, &bad);
      else factorb<BS>(T, o, lane, dinv, &bad);
    } else if (k > 0) {
#if SR_DIAG_ISOLATE
      // warp 4 shares warp 0's scheduler (and FP64 pipe): it stays idle so the factor
      // steps, the critical path, are not slowed by SYRK instructions on that pipe
      if (warp != 4) {
        if (BS == 8) syrk_mma(T, o - BS, warp < 4 ? warp - 1 : warp - 2, 6, lane);
        else syrkb<BS>(T, o - BS, warp < 4 ? t - 32 : t - 64, 192, true);
      }
#else
      syrkb<BS>(T, o - BS, t - 32, 224, true);
#endif
    }
    __syncthreads();
    SR_DIAG_PROBE(17 + 2 * k);
    if (k < NB / BS - 1) {
      if (t < 4 * (NB - o - BS)) trsm_quad<BS>(T, o, o + BS + (t >> 2), t & 3, dinv);
      __syncthreads();
    }
    SR_DIAG_PROBE(18 + 2 * k);
  }
  SR_DIAG_PROBE(2);
  if (t == 0 && bad && info) atomicCAS(info, 0, (int)(B.row_base + (long long)p * NB + bad));
  if (warp < 4) inv16(T, X, 16 * warp, lane, dinv);
  __syncthreads();
  SR_DIAG_PROBE(14);
  // Inverse by recursive doubling on the FP64 tensor cores: X21 = -X22 L21 X11 for the
  // 16-blocks inside each 32-block (both at once), then for the two 32-blocks.  Each warp
  // owns 8x8 output tiles (DMMA 8x8x4, a complex product as 4 real MMAs); X is lower
  // triangular with explicit zeros above the diagonal inside the 16-blocks (inv16), so a
  // tile's K range starts at its column (L X) or ends at its row (X W).
  {
    double2* W = dsm + 2 * NB * LDT;   // [32][LDW] scratch product
    {   // 16 -> 32: W' = L21' X11' (rows 32b+16.., cols 32b..), X21' = -X22' W'
      const int bb = warp >> 2, ti = (warp >> 1) & 1, tj = warp & 1, o = 32 * bb;
      double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
      tile_mma(T + (o + 16 + 8 * ti) * LDT + o, LDT, X + o * LDT + o + 8 * tj, LDT, 8 * tj, 16, lane, cr, ci);
      tile_put(W + (16 * bb + 8 * ti) * LDW + 8 * tj, LDW, lane, cr, ci, 1.0);
      __syncthreads();
      cr[0] = cr[1] = ci[0] = ci[1] = 0.0;
      tile_mma(X + (o + 16 + 8 * ti) * LDT + o + 16, LDT, W + 16 * bb * LDW + 8 * tj, LDW, 0, 8 * ti + 8, lane, cr, ci);
      tile_put(X + (o + 16 + 8 * ti) * LDT + o + 8 * tj, LDT, lane, cr, ci, -1.0);
      __syncthreads();
    }
    {   // 32 -> 64: W = L21 X11 (rows 32.., cols 0..31), X21 = -X22 W; two tiles per warp
      const int ti = warp >> 1;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int tj = 2 * (warp & 1) + h;
        double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
        tile_mma(T + (32 + 8 * ti) * LDT, LDT, X + 8 * tj, LDT, 8 * tj, 32, lane, cr, ci);
        tile_put(W + 8 * ti * LDW + 8 * tj, LDW, lane, cr, ci, 1.0);
      }
      __syncthreads();
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int tj = 2 * (warp & 1) + h;
        double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
        tile_mma(X + (32 + 8 * ti) * LDT + 32, LDT, W + 8 * tj, LDW, 0, 8 * ti + 8, lane, cr, ci);
        tile_put(X + (32 + 8 * ti) * LDT + 8 * tj, LDT, lane, cr, ci, -1.0);
      }
      __syncthreads();
    }
  }
  SR_DIAG_PROBE(15);
  double2* linv = B.linv + (long long)p * NB * NB;
  for (int e = t; e < NB * NB; e += 256) {
    const int r = e >> 6, c = e & 63;
    if (c <= r) tile[(long long)r * np + c] = T[r * LDT + c];
    linv[e] = c <= r ? X[r * LDT + c] : make_double2(0.0, 0.0);
  }
  {
    const int r = t >> 2, q = t & 3;
    double2 y = make_double2(0.0, 0.0);
    for (int c = q; c <= r; c += 4) cfma(y, X[r * LDT + c], bsh[c]);
    y.x += __shfl_xor_sync(0xffffffffu, y.x, 1);
    y.y += __shfl_xor_sync(0xffffffffu, y.y, 1);
    y.x += __shfl_xor_sync(0xffffffffu, y.x, 2);
    y.y += __shfl_xor_sync(0xffffffffu, y.y, 2);
    if (q == 0) B.rhs[(long long)p * NB + r] = y;
  }
  pdl_trigger();
  __syncthreads();
  SR_DIAG_PROBE(16);
}

}  // namespace cholk
}  // namespace sr
