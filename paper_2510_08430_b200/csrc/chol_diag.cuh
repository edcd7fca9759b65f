// chol_diag.cuh — the 64x64 diagonal-tile kernel of the blocked Cholesky (chol.cu).  In its
// own header so tools/diag_probe.cu can time its phases (SR_DIAG_PROBE hook, empty here).
#pragma once
#include "chol.cuh"

#ifndef SR_DIAG_PROBE
#define SR_DIAG_PROBE(i)
#endif
namespace sr {
namespace cholk {

constexpr int NB = 64;

// One CTA per block: factor the 64x64 diagonal tile of panel p, form its inverse
// X = Linv_p and y_p = Linv_p b_p.  Blocked by 8 (a 64-step column recursion with a block
// barrier per step is what limited the unblocked forms):
//   for each 8-column block k (offset o = 8k):
//     (a) warp 0 factors D_k = A[o:o+8, o:o+8] in registers (lane r = row r, columns by
//         shuffles) and, in lanes 8..15 of the same instruction stream, D_k^{-1};
//     (b) rows r >= o+8: L[r, o:o+8] = A[r, o:o+8] D_k^{-H}, 8x8 DMMA tiles;
//     (c) A[r][s] -= sum_m L[r][o+m] conj(L[s][o+m]) on the trailing lower triangle as
//         8x8 DMMA tiles (warps 1-3, 5-7), overlapped with (a) of the next block, whose
//         own diagonal tile warp 0 updates first.
//   inverse: X21 = -X22 L21 X11 by recursive doubling 8 -> 16 -> 32 -> 64 on DMMA.
// Phase timings: tools/diag_probe.cu (66.9k cycles for the first scalar-FP64 version,
// 50.1k with the DMMA SYRK and inverse levels).
constexpr int LDT = NB + 1;   // 1040-byte rows
// T and X (the inverse's scratch W lives in T's unused strict upper triangle): 130 KB, so
// a diagonal tile fits on an SM beside one 87 KB skinny CTA of the off-chain updates
constexpr size_t kDiagSmem = (size_t)2 * NB * LDT * sizeof(double2);

// 8x8 complex tile on DMMA: C += sum_{k in [k0, k1)} A[r][k] B[k][c] for r, c < 8, with A and
// B row-major in shared memory (k0, k1 multiples of 4).  Lane l holds C[l/4][2(l%4) + {0,1}].
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

// (a') warp 0, lanes r < 8: row r of the 8x8 block D in registers; step c takes column c
// from lanes s > c by shuffles (no shared-memory round trip), and lane c+1 forms the next
// pivot A[c+1][c+1] - |A[c+1][c]|^2 isd^2 before the rank-1 update.  Lanes 8 + j run the
// forward substitution D x = e_j on the same broadcasts (x_c = b_c isd_c, then
// b_s -= L[s][c] x_c), so D^{-1} comes out of the same instruction stream and lands in X.
// (Spreading D over all 32 lanes, two entries per lane, measured slower: 3.5k vs 2.9k
// cycles per 8x8 factor, tools/diag_probe.cu.)
__device__ __forceinline__ void factor8(double2* T, double2* X, int o, int lane, double* dinv, int* bad) {
  const int r = lane & 7;
  const bool fl = lane < 8, il = lane >= 8 && lane < 16;   // factor lanes, inverse lanes
  double2 d[8];
#pragma unroll
  for (int s = 0; s < 8; s++)
    d[s] = fl ? (s <= r ? T[(o + r) * LDT + o + s] : make_double2(0.0, 0.0)) : make_double2(s == r ? 1.0 : 0.0, 0.0);
  double piv = __shfl_sync(0xffffffffu, d[0].x, 0);
  const int sgn = fl ? (int)0x80000000 : 0;   // factor lanes multiply by conj(L[s][c])
  const bool upd = !fl;
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
    // No lane-dependent branches around whole steps: the compiler would otherwise unswitch
    // the loop into a factor copy and an inverse copy that the warp runs one after the other.
    d[c] = cscale(d[c], isd);
    if (fl && r == c) d[c] = make_double2(piv * isd, 0.0);
    if (lane == 0) dinv[o + c] = isd;
#pragma unroll
    for (int s = c + 1; s < 8; s++) {
      // factor lanes: d[s] -= L[r][c] conj(L[s][c]); inverse lanes: b_s -= x_c L[s][c]
      const double lx = __shfl_sync(0xffffffffu, d[c].x, s);
      const double ly0 = __shfl_sync(0xffffffffu, d[c].y, s);
      const double ly = __hiloint2double(__double2hiint(ly0) ^ sgn, __double2loint(ly0));
      if (upd || r >= s) {
        d[s].x -= d[c].x * lx - d[c].y * ly;
        d[s].y -= d[c].x * ly + d[c].y * lx;
      }
    }
    piv = pn;
  }
  if (fl) {
#pragma unroll
    for (int s = 0; s < 8; s++)
      if (s <= r) T[(o + r) * LDT + o + s] = d[s];
  } else if (il) {   // X[o+s][o+j] = x_s (zeros above the diagonal)
#pragma unroll
    for (int s = 0; s < 8; s++) X[(o + s) * LDT + o + r] = d[s];
  }
}

// (b') rows below block o: L[r][o:o+8] = A[r][o:o+8] D^{-H}, one 8x8 DMMA tile per warp.
__device__ __forceinline__ void trsm_tile(double2* T, const double2* X, int o, int r0, int lane) {
  const int lr = lane >> 2, lk = lane & 3;
  double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
#pragma unroll
  for (int k = 0; k < 8; k += 4) {   // sum_m A[r][m] conj(Dinv[c][m])
    const double2 a = T[(r0 + lr) * LDT + o + k + lk], b = X[(o + lr) * LDT + o + k + lk];
    dmma_t(cr[0], cr[1], a.x, b.x);
    dmma_t(cr[0], cr[1], a.y, b.y);
    dmma_t(ci[0], ci[1], a.y, b.x);
    dmma_t(ci[0], ci[1], -a.x, b.y);
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; h++) T[(r0 + lr) * LDT + o + 2 * lk + h] = make_double2(cr[h], ci[h]);
}

// Lower-triangle patch index e -> (pi, pj), pi >= pj.
__device__ __forceinline__ void tri_patch(int e, int& pi, int& pj) {
  pi = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  while ((pi + 1) * (pi + 2) / 2 <= e) pi++;
  while (pi * (pi + 1) / 2 > e) pi--;
  pj = e - pi * (pi + 1) / 2;
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
  TraceScope trace_(TR_DIAG, (int)(B.row_base / 64) * 4096 + p);
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
  // Block k: warp 0 applies block k-1's update to the diagonal block k and factors it
  // (with D_k^{-1}) while warps 1-3, 5-7 apply block k-1's update to the rest of the
  // trailing triangle; warp 4 shares warp 0's scheduler and stays idle so the factor, the
  // critical path, does not compete for its FP64 pipe.  Then the rows below are solved.
  for (int k = 0; k < NB / 8; k++) {
    const int o = 8 * k;
    if (warp == 0) {
      if (k > 0) syrk_diag_mma(T, o - 8, lane);
      __syncwarp();
      factor8(T, X, o, lane, dinv, &bad);
    } else if (k > 0 && warp != 4) {
      syrk_mma(T, o - 8, warp < 4 ? warp - 1 : warp - 2, 6, lane);
    }
    __syncthreads();
    SR_DIAG_PROBE(17 + 2 * k);
    if (k < NB / 8 - 1) {
      if (warp < 7 - k) trsm_tile(T, X, o, o + 8 + 8 * warp, lane);
      __syncthreads();
    }
    SR_DIAG_PROBE(18 + 2 * k);
  }
  SR_DIAG_PROBE(2);
  if (t == 0 && bad && info) atomicCAS(info, 0, (int)(B.row_base + (long long)p * NB + bad));
  {   // 8 -> 16: X21 = -X22 (L21 X11) inside each 16-block (warps 0-3, one block each)
    double2* W = T + 32;   // scratch in T's unused strict upper triangle (rows 0-31, cols 32-63)
    if (warp < 4) {
      const int o = 16 * warp;
      double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
      tile_mma(T + (o + 8) * LDT + o, LDT, X + o * LDT + o, LDT, 0, 8, lane, cr, ci);
      tile_put(W + 8 * warp * LDT, LDT, lane, cr, ci, 1.0);
      __syncwarp();
      cr[0] = cr[1] = ci[0] = ci[1] = 0.0;
      tile_mma(X + (o + 8) * LDT + o + 8, LDT, W + 8 * warp * LDT, LDT, 0, 8, lane, cr, ci);
      tile_put(X + (o + 8) * LDT + o, LDT, lane, cr, ci, -1.0);
    }
    __syncthreads();
  }
  SR_DIAG_PROBE(14);
  // Inverse by recursive doubling on the FP64 tensor cores: X21 = -X22 L21 X11 for the
  // 16-blocks inside each 32-block (both at once), then for the two 32-blocks.  Each warp
  // owns 8x8 output tiles (DMMA 8x8x4, a complex product as 4 real MMAs); X is lower
  // triangular with explicit zeros above the diagonal inside the 8-blocks (factor8) and
  // the 16-blocks (the level above), so a tile's K range starts at its column (L X) or ends
  // at its row (X W).
  {
    double2* W = T + 32;   // [32][LDT] scratch product in T's unused strict upper triangle
    {   // 16 -> 32: W' = L21' X11' (rows 32b+16.., cols 32b..), X21' = -X22' W'
      const int bb = warp >> 2, ti = (warp >> 1) & 1, tj = warp & 1, o = 32 * bb;
      double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
      tile_mma(T + (o + 16 + 8 * ti) * LDT + o, LDT, X + o * LDT + o + 8 * tj, LDT, 8 * tj, 16, lane, cr, ci);
      tile_put(W + (16 * bb + 8 * ti) * LDT + 8 * tj, LDT, lane, cr, ci, 1.0);
      __syncthreads();
      cr[0] = cr[1] = ci[0] = ci[1] = 0.0;
      tile_mma(X + (o + 16 + 8 * ti) * LDT + o + 16, LDT, W + 16 * bb * LDT + 8 * tj, LDT, 0, 8 * ti + 8, lane, cr, ci);
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
        tile_put(W + 8 * ti * LDT + 8 * tj, LDT, lane, cr, ci, 1.0);
      }
      __syncthreads();
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int tj = 2 * (warp & 1) + h;
        double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
        tile_mma(X + (32 + 8 * ti) * LDT + 32, LDT, W + 8 * tj, LDT, 0, 8 * ti + 8, lane, cr, ci);
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
