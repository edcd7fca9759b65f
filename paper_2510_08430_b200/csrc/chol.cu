// chol.cu — stage (5): batched, blocked, right-looking Cholesky solve of
// (S_b + lambda I) x_b = F_b for all layer blocks at once (§2: "Each block S_l
// is inverted independently, using a uniform diagonal shift lambda"), also used by the
// full-QGT and NTK comparison paths with a single "block".
//
// Each block is copied into a padded factor matrix (n_pad = 64*ceil(n/64), identity in
// the padding so the padded system decouples).  Panel step p (all blocks with
// p < P_b advance together, one launch per kernel):
//   chol_diag        factor the 64x64 diagonal tile in shared memory, form its inverse
//                    Linv_p, and y_p = Linv_p b_p (forward substitution folded in)
//   trsm (engine)    L_ip = A_ip Linv_p^H for every row tile i > p      (DMMA, NH/STORE)
//   (chol_diag also subtracts the strip's earlier panels from its own 64 rows of b)
//   inner (engine)   A_ij -= L_ip L_jp^H for the strip's later columns j (DMMA, NH/SUB)
// and after every strip of 4 panels chol_rhs_update (b_i -= L_i,strip y_strip for the rows
// below) and one deferred trailing update with K = 256:
//   trail (engine)   A_ij -= L_i,strip L_j,strip^H for i >= j beyond the strip (NH/SUB)
// then back substitution L^H x = y strip by strip (x_p = Linv_p^H y_p inside the strip,
// then y_{<strip} -= L_strip,<^H x_strip) and dtheta = -x.
#include <cstdlib>

#include "chol.cuh"
#include "gram.cuh"
#include "ozaki.cuh"

namespace sr {
namespace {

constexpr int NB = 64;
constexpr int kStrip = 4;   // panels per strip (deferred trailing update with K = 256)

__global__ void chol_init(CholSet cs, double lam, int inplace) {
  const int b = blockIdx.y;
  const CholBlock& B = cs.b[b];
  const long long n = B.n, np = B.npad;
  const long long total = np * np;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / np, c = e % np;
    if (r < n && c < n) {
      if (inplace) {
        if (r == c) B.Fm[e].x += lam;
      } else {
        double2 v = B.S[r * n + c];
        if (r == c) v.x += lam;
        B.Fm[e] = v;
      }
    } else {
      B.Fm[e] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    }
  }
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < np;
       r += (long long)gridDim.x * blockDim.x)
    B.rhs[r] = r < n ? B.F[r] : make_double2(0.0, 0.0);
}

// One CTA per block: factor the 64x64 diagonal tile of panel p, form its inverse
// X = Linv_p and y_p = Linv_p b_p.  Blocked by 16 (the latency of a 64-step column
// recursion with a block barrier per step is what limited the unblocked forms):
//   for each 16-column block k (offset o = 16k):
//     (a) warp 0 factors D_k = A[o:o+16, o:o+16] in registers, lane r = row r, columns
//         broadcast by shuffles, 1/sqrt of each pivot kept in dinv;
//     (b) rows r >= o+16 solve x D_k^H = A[r, o:o+16] (one thread per row, right-looking);
//     (c) A[r][s] -= sum_m L[r][o+m] conj(L[s][o+m]) on the trailing lower triangle
//         (2x2 register patches).
//   inverse: X_kk = D_k^{-1} (warp k, lane j = column j), then by block distance d = 1..3:
//     W_ik = sum_{j=k}^{i-1} L_ij X_jk and X_ik = -X_ii W_ik (i = k + d), 2x2 patches.
constexpr int LDT = NB + 1;   // 1040-byte rows
constexpr size_t kDiagSmem = (size_t)2 * NB * LDT * sizeof(double2);

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
__device__ __forceinline__ void factor16(double2* T, int o, int lane, double* dinv, int* bad) {
  double2 d[16];
  double dg[16];
  const int r = lane;
#pragma unroll
  for (int s = 0; s < 16; s++) {
    d[s] = (r < 16 && s <= r) ? T[(o + r) * LDT + o + s] : make_double2(0.0, 0.0);
    dg[s] = T[(o + s) * LDT + o + s].x;
  }
#pragma unroll
  for (int c = 0; c < 16; c++) {
    double piv = dg[c];
    if (!(piv > 0.0)) {
      if (lane == 0 && *bad == 0) *bad = o + c + 1;
      piv = 1.0;
    }
    const double isd = rsqrt(piv);
    if (r == c) d[c] = make_double2(piv * isd, 0.0);
    else if (r > c) d[c] = cscale(d[c], isd);
    if (r < 16 && r >= c) T[(o + r) * LDT + o + c] = d[c];
    if (lane == 0) dinv[o + c] = isd;
    __syncwarp();
#pragma unroll
    for (int s = 1; s < 16; s++) {
      if (s <= c) continue;
      const double2 ls = T[(o + s) * LDT + o + c];   // L[s][c]
      dg[s] -= ls.x * ls.x + ls.y * ls.y;
      if (r >= s && r < 16) {
        double2 v = d[s];
        v.x -= d[c].x * ls.x + d[c].y * ls.y;
        v.y -= d[c].y * ls.x - d[c].x * ls.y;
        d[s] = v;
      }
    }
  }
}

// (b) rows below the block solve x D^H = A[r, o:o+16] with D = L[o:o+16, o:o+16]
// (diagonal real, 1/D_cc in dinv): a quad per row, lane q holding entries m = q mod 4;
// step c: x_c = a_c / D_cc from the owner lane, shuffled inside the quad, then
// a_m -= x_c conj(D[m][c]) for m > c.
__device__ __forceinline__ void trsm_quad(double2* T, int o, int r, int q, const double* dinv) {
  double2 a[4];
#pragma unroll
  for (int k = 0; k < 4; k++) a[k] = T[r * LDT + o + 4 * k + q];
#pragma unroll
  for (int c = 0; c < 16; c++) {
    if (q == (c & 3)) {   // owner: x_c final, published in place
      a[c >> 2] = cscale(a[c >> 2], dinv[o + c]);
      T[r * LDT + o + c] = a[c >> 2];
    }
    __syncwarp();
    const double2 x = T[r * LDT + o + c];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int m = 4 * k + q;
      if (m > c) {
        const double2 dm = T[(o + m) * LDT + o + c];
        a[k].x -= x.x * dm.x + x.y * dm.y;
        a[k].y -= x.y * dm.x - x.x * dm.y;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 4; k++) T[r * LDT + o + 4 * k + q] = a[k];
}

// Lower-triangle patch index e -> (pi, pj), pi >= pj.
__device__ __forceinline__ void tri_patch(int e, int& pi, int& pj) {
  pi = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  while ((pi + 1) * (pi + 2) / 2 <= e) pi++;
  while (pi * (pi + 1) / 2 > e) pi--;
  pj = e - pi * (pi + 1) / 2;
}

// (c) trailing update of rows/cols [o+16, 64) by the 16 columns L[:, o:o+16].
__device__ __forceinline__ void syrk16(double2* T, int o, int t) {
  const int b0 = o + 16, P = (NB - b0) / 2, cnt = P * (P + 1) / 2;
  for (int e = t; e < cnt; e += 256) {
    int pi, pj;
    tri_patch(e, pi, pj);
    const int r0 = b0 + 2 * pi, s0 = b0 + 2 * pj;
    double2 acc[2][2] = {{make_double2(0.0, 0.0), make_double2(0.0, 0.0)},
                         {make_double2(0.0, 0.0), make_double2(0.0, 0.0)}};
#pragma unroll 4
    for (int m = 0; m < 16; m++) {
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
  for (int e = t; e < NB * NB; e += 256) {
    const int r = e >> 6, c = e & 63;
    if (c <= r) T[r * LDT + c] = tile[(long long)r * np + c];
  }
  {   // b_p -= sum over the strip's earlier panels q in [p0, p) of L_pq y_q (rows of panel p)
    const int r = t >> 2, q = t & 3;
    const double2* lrow = B.Fm + ((long long)p * NB + r) * np;
    double2 s2 = make_double2(0.0, 0.0);
    for (long long c = (long long)p0 * NB + q; c < (long long)p * NB; c += 4) cfma(s2, lrow[c], B.rhs[c]);
    s2.x += __shfl_xor_sync(0xffffffffu, s2.x, 1);
    s2.y += __shfl_xor_sync(0xffffffffu, s2.y, 1);
    s2.x += __shfl_xor_sync(0xffffffffu, s2.x, 2);
    s2.y += __shfl_xor_sync(0xffffffffu, s2.y, 2);
    if (q == 0) bsh[r] = csub(B.rhs[(long long)p * NB + r], s2);
  }
  if (t == 0) bad = 0;
  __syncthreads();
  for (int k = 0; k < 4; k++) {
    const int o = 16 * k;
    if (warp == 0) factor16(T, o, lane, dinv, &bad);
    __syncthreads();
    if (k < 3) {
      if (t < 4 * (NB - o - 16)) trsm_quad(T, o, o + 16 + (t >> 2), t & 3, dinv);
      __syncthreads();
      syrk16(T, o, t);
      __syncthreads();
    }
  }
  if (t == 0 && bad && info) atomicCAS(info, 0, (int)(B.row_base + (long long)p * NB + bad));
  if (warp < 4) inv16(T, X, 16 * warp, lane, dinv);
  __syncthreads();
  for (int d = 1; d < 4; d++) {
    const int nbk = 4 - d;
    const bool act = t < nbk * 64;
    const int kb = t >> 6, ib = kb + d, pr = (t & 63) >> 3, pc = t & 7;
    const int r0 = 16 * ib + 2 * pr, c0 = 16 * kb + 2 * pc;
    double2 acc[2][2] = {{make_double2(0.0, 0.0), make_double2(0.0, 0.0)},
                         {make_double2(0.0, 0.0), make_double2(0.0, 0.0)}};
    if (act) {   // W_ik = sum_{m in blocks k..i-1} L[r][m] X[m][c]
      for (int m = 16 * kb; m < 16 * ib; m++) {
        const double2 l0 = T[r0 * LDT + m], l1 = T[(r0 + 1) * LDT + m];
        const double2 x0 = X[m * LDT + c0], x1 = X[m * LDT + c0 + 1];
        cfma(acc[0][0], l0, x0);
        cfma(acc[0][1], l0, x1);
        cfma(acc[1][0], l1, x0);
        cfma(acc[1][1], l1, x1);
      }
#pragma unroll
      for (int u = 0; u < 2; u++)
#pragma unroll
        for (int v = 0; v < 2; v++) X[(r0 + u) * LDT + c0 + v] = acc[u][v];
    }
    __syncthreads();
    if (act) {   // X_ik = -X_ii W_ik (X_ii lower triangular)
#pragma unroll
      for (int u = 0; u < 2; u++)
#pragma unroll
        for (int v = 0; v < 2; v++) acc[u][v] = make_double2(0.0, 0.0);
      for (int m = 16 * ib; m <= r0 + 1; m++) {
        const double2 w0 = X[m * LDT + c0], w1 = X[m * LDT + c0 + 1];
        const double2 x0 = m <= r0 ? X[r0 * LDT + m] : make_double2(0.0, 0.0);
        const double2 x1 = X[(r0 + 1) * LDT + m];
        cfma(acc[0][0], x0, w0);
        cfma(acc[0][1], x0, w1);
        cfma(acc[1][0], x1, w0);
        cfma(acc[1][1], x1, w1);
      }
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int u = 0; u < 2; u++)
#pragma unroll
        for (int v = 0; v < 2; v++) X[(r0 + u) * LDT + c0 + v] = make_double2(-acc[u][v].x, -acc[u][v].y);
    }
    __syncthreads();
  }
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
}

// b_i -= sum_{c in [c0, c1)} L[i][c] y[c] for rows i >= c1 (the strip's panels applied to the
// right-hand side of every later row at once; one warp per row).
__global__ void chol_rhs_update(const CholBlock B, long long c0, long long c1) {
  const long long np = B.npad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long r = c1 + (long long)blockIdx.x * 8 + warp; r < np; r += (long long)gridDim.x * 8) {
    const double2* row = B.Fm + r * np;
    double2 s = make_double2(0.0, 0.0);
    for (long long c = c0 + lane; c < c1; c += 32) cfma(s, row[c], B.rhs[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    }
    if (lane == 0) B.rhs[r] = csub(B.rhs[r], s);
  }
}

// Back substitution L^H x = y by strips of panels [p0, pend), two launches per strip:
// chol_back_strip (one CTA): for p = pend-1 .. p0: x_p = Linv_p^H y_p, then
//   y_q -= L_pq^H x_p for the strip's earlier panels q in [p0, p);
// chol_back_rest (one CTA per 64 columns c < 64 p0): y_c -= sum_{r in strip} conj(L[r][c]) x_r.
// Reductions run in a fixed order (deterministic).
__global__ void __launch_bounds__(256) chol_back_strip(const CholBlock B, int p0, int pend) {
  __shared__ double2 ys[kStrip][NB];
  __shared__ double2 xs[NB];
  const long long np = B.npad;
  const int t = threadIdx.x, c = t >> 2, q4 = t & 3;
  for (int e = t; e < (pend - p0) * NB; e += 256) ys[e >> 6][e & 63] = B.rhs[(long long)p0 * NB + e];
  __syncthreads();
  for (int p = pend - 1; p >= p0; p--) {
    const double2* linv = B.linv + (long long)p * NB * NB;
    double2 sx = make_double2(0.0, 0.0);
    for (int r = c + q4; r < NB; r += 4) cfma_conj(sx, linv[r * NB + c], ys[p - p0][r]);
    sx.x += __shfl_xor_sync(0xffffffffu, sx.x, 1);
    sx.y += __shfl_xor_sync(0xffffffffu, sx.y, 1);
    sx.x += __shfl_xor_sync(0xffffffffu, sx.x, 2);
    sx.y += __shfl_xor_sync(0xffffffffu, sx.y, 2);
    if (q4 == 0) {
      xs[c] = sx;
      B.xout[(long long)p * NB + c] = sx;
    }
    __syncthreads();
    for (int q = p0; q < p; q++) {   // y_q[c] -= sum_r conj(L[p*64+r][q*64+c]) x_p[r]
      const double2* lp = B.Fm + (long long)p * NB * np + (long long)q * NB + c;
      double2 sy = make_double2(0.0, 0.0);
      for (int r = q4; r < NB; r += 4) cfma_conj(sy, lp[(long long)r * np], xs[r]);
      sy.x += __shfl_xor_sync(0xffffffffu, sy.x, 1);
      sy.y += __shfl_xor_sync(0xffffffffu, sy.y, 1);
      sy.x += __shfl_xor_sync(0xffffffffu, sy.x, 2);
      sy.y += __shfl_xor_sync(0xffffffffu, sy.y, 2);
      if (q4 == 0) ys[q - p0][c] = csub(ys[q - p0][c], sy);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) chol_back_rest(const CholBlock B, int p0, int pend) {
  __shared__ double2 xs[kStrip * NB];
  __shared__ double2 red[4][NB];
  const long long np = B.npad;
  const int t = threadIdx.x, cl = t & 63, rq = t >> 6;
  const int nr = (pend - p0) * NB;
  for (int e = t; e < nr; e += 256) xs[e] = B.xout[(long long)p0 * NB + e];
  __syncthreads();
  const long long ncol = (long long)p0 * NB;
  for (long long cb = (long long)blockIdx.x * NB; cb < ncol; cb += (long long)gridDim.x * NB) {
    const long long c = cb + cl;
    double2 s = make_double2(0.0, 0.0);
    const double2* col = B.Fm + ((long long)p0 * NB) * np + c;
#pragma unroll 4
    for (int r = rq; r < nr; r += 4) cfma_conj(s, col[(long long)r * np], xs[r]);
    red[rq][cl] = s;
    __syncthreads();
    if (rq == 0) {
      const double2 v = cadd(cadd(red[0][cl], red[1][cl]), cadd(red[2][cl], red[3][cl]));
      B.rhs[c] = csub(B.rhs[c], v);
    }
    __syncthreads();
  }
}

__global__ void chol_output(CholSet cs, double sign) {
  const CholBlock& B = cs.b[blockIdx.y];
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < B.n;
       r += (long long)gridDim.x * blockDim.x)
    B.out[r] = cscale(B.xout[r], sign);
}

}  // namespace

void carve_chol(Arena& a, CholSet& cs, const long long* sizes, int nblk) {
  cs.count = nblk;
  long long row_base = 0;
  for (int b = 0; b < nblk; b++) {
    CholBlock& B = cs.b[b];
    B.n = sizes[b];
    B.P = (int)((B.n + NB - 1) / NB);
    B.npad = (long long)B.P * NB;
    B.row_base = row_base;
    row_base += B.n;
    B.Fm = a.take<double2>((size_t)B.npad * B.npad);
    B.rhs = a.take<double2>(B.npad);
    B.xout = a.take<double2>(B.npad);
    B.linv = a.take<double2>((size_t)B.P * NB * NB);
    B.tws_bytes = oz::trail_workspace_bytes(B.npad, (long long)kStrip * NB);
    B.tws = a.take<char>(B.tws_bytes);
  }
}

namespace {

// Persistent-grid cap of the int8 trailing update: with several blocks in flight, leave SMs
// for the other blocks' latency-bound panel chains (SR_TRAIL_CTAS overrides, for tuning).
int trail_ctas(int nblocks) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("SR_TRAIL_CTAS");
    env = e ? atoi(e) : -1;
  }
  if (env >= 0) return env;
  (void)nblocks;
  return 0;   // measured: capping the grid slows the 3-block solve (trailing throughput bound)
}

// Factorisation + substitutions of ONE block on one stream (two-level blocking, see header).
sr_status solve_block(CholSet& cs, int b, cudaStream_t st) {
  const CholBlock& B = cs.b[b];
  // Two-level blocking: strips of kStrip panels.  Inside a strip each panel p is factored
  // (chol_diag), its column solved (TRSM), the RHS updated, and only the strip's own later
  // columns updated (K = 64); the rest of the trailing matrix receives one deferred update
  // per strip with K = 64 * kStrip, which is where the flops are (4x the arithmetic
  // intensity of a per-panel update, 4x fewer passes over the trailing matrix).
  const bool i8 = gram_engine() == SR_GRAM_INT8;
  for (int p0 = 0; p0 < B.P; p0 += kStrip) {
    const int pend = std::min(p0 + kStrip, B.P);
    for (int p = p0; p < pend; p++) {
      timer_begin("chol_diag", st);
      chol_diag<<<1, 256, kDiagSmem, st>>>(B, cs.info, p, p0);
      timer_end(st);
      SR_LAUNCHED();
      const long long m = B.npad - (long long)(p + 1) * NB;
      if (m <= 0) continue;
      gram::ProbSet trsm{}, inner{};
      double2* panel = B.Fm + (long long)(p + 1) * NB * B.npad + (long long)p * NB;
      gram::add_prob(trsm, panel, B.npad, B.linv + (long long)p * NB * NB, NB, panel, B.npad, (int)m, NB, NB, false);
      for (int jj = p + 1; jj < pend; jj++) {   // later columns of the strip, rows i >= jj
        const double2* lrows = B.Fm + (long long)jj * NB * B.npad + (long long)p * NB;
        double2* cblk = B.Fm + (long long)jj * NB * B.npad + (long long)jj * NB;
        gram::add_prob(inner, lrows, B.npad, lrows, B.npad, cblk, B.npad, (int)(B.npad - (long long)jj * NB), NB, NB,
                       false);
      }
      timer_begin("chol_trsm", st);
      SR_TRY((gram::launch<gram::NH, gram::STORE>(trsm, st)));
      timer_end(st);
      timer_begin("chol_inner", st);
      if (inner.count) SR_TRY((gram::launch<gram::NH, gram::SUB>(inner, st)));
      timer_end(st);
    }
    const long long m = B.npad - (long long)pend * NB;
    if (m > 0) {   // the strip's y applied to the right-hand side of all later rows
      dim3 g((unsigned)std::min<long long>((m + 7) / 8, 4 * kNumSMs), 1);
      timer_begin("chol_rhs", st);
      chol_rhs_update<<<g, 256, 0, st>>>(B, (long long)p0 * NB, (long long)pend * NB);
      timer_end(st);
      SR_LAUNCHED();
    }
    if (m > 0) {   // deferred trailing update of the strip, K = 64 * (pend - p0)
      const double2* lp = B.Fm + (long long)pend * NB * B.npad + (long long)p0 * NB;
      double2* trailing = B.Fm + (long long)pend * NB * B.npad + (long long)pend * NB;
      if (i8) {   // int8 digit-slice tcgen05 engine (ozaki.cu), lower triangle
        SR_TRY(oz::trail_update_i8(lp, B.npad, m, (long long)(pend - p0) * NB, trailing, B.npad, B.tws, B.tws_bytes,
                                   trail_ctas(cs.count), st));
      } else {
        gram::ProbSet trail{};
        gram::add_prob(trail, lp, B.npad, lp, B.npad, trailing, B.npad, (int)m, (int)m,
                       (long long)(pend - p0) * NB, true);
        timer_begin("trail_dmma", st);
        SR_TRY((gram::launch<gram::NH, gram::SUB>(trail, st)));
        timer_end(st);
      }
    }
  }
  for (int p0 = (B.P - 1) / kStrip * kStrip; p0 >= 0; p0 -= kStrip) {
    const int pend = std::min(p0 + kStrip, B.P);
    timer_begin("chol_back", st);
    chol_back_strip<<<1, 256, 0, st>>>(B, p0, pend);
    SR_LAUNCHED();
    if (p0 > 0) {
      chol_back_rest<<<(unsigned)std::min(p0, 4 * kNumSMs), 256, 0, st>>>(B, p0, pend);
      SR_LAUNCHED();
    }
    timer_end(st);
  }
  return SR_OK;
}

// Side streams for independent blocks (created once per process; high priority so the
// latency-bound panel chain of one block is scheduled ahead of another block's big update).
constexpr int kSideStreams = 8;
struct SidePool {
  cudaStream_t s[kSideStreams];
  cudaEvent_t fork, join[kSideStreams];
  bool ok = false;
};
sr_status side_pool(SidePool*& out) {
  static SidePool pool;
  if (!pool.ok) {
    int lo = 0, hi = 0;
    SR_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (int i = 0; i < kSideStreams; i++) {
      SR_CUDA(cudaStreamCreateWithPriority(&pool.s[i], cudaStreamNonBlocking, hi));
      SR_CUDA(cudaEventCreateWithFlags(&pool.join[i], cudaEventDisableTiming));
    }
    SR_CUDA(cudaEventCreateWithFlags(&pool.fork, cudaEventDisableTiming));
    pool.ok = true;
  }
  out = &pool;
  return SR_OK;
}

}  // namespace

sr_status chol_solve(CholSet& cs, double lam, bool inplace, double sign, cudaStream_t st) {
  if (cs.info) SR_CUDA(cudaMemsetAsync(cs.info, 0, sizeof(int), st));
  {
    long long mx = 0;
    for (int b = 0; b < cs.count; b++) mx = std::max(mx, cs.b[b].npad * cs.b[b].npad);
    dim3 g((unsigned)std::min<long long>((mx + 255) / 256, 2 * kNumSMs), (unsigned)cs.count);
    chol_init<<<g, 256, 0, st>>>(cs, lam, inplace ? 1 : 0);
    SR_LAUNCHED();
  }
  static bool diag_attr = false;
  if (!diag_attr) {
    SR_CUDA(cudaFuncSetAttribute(chol_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiagSmem));
    diag_attr = true;
  }
  if (cs.count == 1) {
    SR_TRY(solve_block(cs, 0, st));
  } else {
    // independent blocks on side streams, forked from and joined back into `st`
    SidePool* pool;
    SR_TRY(side_pool(pool));
    SR_CUDA(cudaEventRecord(pool->fork, st));
    for (int b = 0; b < cs.count; b++) {
      cudaStream_t sb = pool->s[b % kSideStreams];
      SR_CUDA(cudaStreamWaitEvent(sb, pool->fork, 0));
      SR_TRY(solve_block(cs, b, sb));
    }
    for (int i = 0; i < std::min(cs.count, kSideStreams); i++) {
      SR_CUDA(cudaEventRecord(pool->join[i], pool->s[i]));
      SR_CUDA(cudaStreamWaitEvent(st, pool->join[i], 0));
    }
  }
  {
    long long mx = 0;
    for (int b = 0; b < cs.count; b++) mx = std::max(mx, cs.b[b].n);
    dim3 g((unsigned)std::max<long long>(1, std::min<long long>((mx + 255) / 256, 4 * kNumSMs)),
           (unsigned)cs.count);
    chol_output<<<g, 256, 0, st>>>(cs, sign);
    SR_LAUNCHED();
  }
  return SR_OK;
}

}  // namespace sr
