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
//   chol_rhs_update  b_i -= L_ip y_p
//   trail (engine)   A_ij -= L_ip L_jp^H for i >= j > p                  (DMMA, NH/SUB)
// then back substitution L^H x = y panel by panel (x_p = Linv_p^H y_p, then
// y_{<p} -= L_p,<p^H x_p) and dtheta = -x.
#include "chol.cuh"
#include "gram.cuh"

namespace sr {
namespace {

constexpr int NB = 64;

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

// One CTA per active block: factor the 64x64 diagonal tile of panel p, its inverse Linv_p
// and y_p = Linv_p b_p in ONE sweep of 64 steps.  Step c works on the unscaled column c
// (a_rc, pivot d_c = a_cc):
//   Cholesky trailing part   T[r][s] -= a_rc conj(a_sc) / d_c        (c < s <= r)
//   forward substitution     Y[r][j] -= a_rc Y[c][j] / d_c            (c < r, j <= c; j = 64: b)
// with Y = [I | b] on entry; at the end L[r][c] = a_rc / sqrt(d_c), L[c][c] = sqrt(d_c),
// Linv[r][j] = Y[r][j] / sqrt(d_r), y_r = Y[r][64] / sqrt(d_r).
// Thread (r, q) = (t/4, t%4) keeps the 16 entries s = q + 4k of row r of T and of Y in
// registers.  Column c of T and row c of Y are published to a double-buffered shared strip
// by their owners at the end of step c-1 (inside the unrolled update loop, so no register
// array is ever indexed dynamically); one barrier per step.
__global__ void __launch_bounds__(256) chol_diag(CholSet cs, ActiveList act, int p) {
  __shared__ double2 colc[2][NB];       // T[.][c]   (published column)
  __shared__ double2 rowc[2][NB + 4];   // Y[c][.]   (published row; [NB] = rhs entry)
  __shared__ double piv[NB];
  const CholBlock& B = cs.b[act.idx[blockIdx.x]];
  const long long np = B.npad;
  double2* tile = B.Fm + (long long)p * NB * np + (long long)p * NB;
  const int t = threadIdx.x, r = t >> 2, q = t & 3;
  double2 tr[16], yr[16];
  double2 rhs = make_double2(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < 16; k++) {
    const int s = q + 4 * k;
    tr[k] = s <= r ? tile[(long long)r * np + s] : make_double2(0.0, 0.0);
    yr[k] = make_double2(s == r ? 1.0 : 0.0, 0.0);
  }
  if (q == 0) {
    rhs = B.rhs[(long long)p * NB + r];
    colc[0][r] = tr[0];
  }
  if (r == 0) {
#pragma unroll
    for (int k = 0; k < 16; k++) rowc[0][q + 4 * k] = yr[k];
    if (q == 0) rowc[0][NB] = rhs;
  }
  for (int c = 0; c < NB; c++) {
    const int buf = c & 1, nbuf = buf ^ 1;
    __syncthreads();
    double d = colc[buf][c].x;
    if (!(d > 0.0)) {
      if (t == 0 && cs.info) atomicCAS(cs.info, 0, (int)(B.row_base + (long long)p * NB + c + 1));
      d = 1.0;
    }
    if (t == 0) piv[c] = d;
    if (r > c) {
      const double inv = 1.0 / d;
      const double2 a = colc[buf][r];
      const double2 g = make_double2(a.x * inv, a.y * inv);   // a_rc / d_c
#pragma unroll
      for (int k = 0; k < 16; k++) {
        const int s = q + 4 * k;
        if (s > c && s <= r) {                                // T[r][s] -= g conj(a_sc)
          const double2 bb = colc[buf][s];
          tr[k].x -= g.x * bb.x + g.y * bb.y;
          tr[k].y -= g.y * bb.x - g.x * bb.y;
          if (s == c + 1) colc[nbuf][r] = tr[k];              // publish column c+1
        }
        if (s <= c) {                                         // Y[r][s] -= g Y[c][s]
          const double2 y = rowc[buf][s];
          yr[k].x -= g.x * y.x - g.y * y.y;
          yr[k].y -= g.x * y.y + g.y * y.x;
        }
      }
      if (q == 0) {
        const double2 y = rowc[buf][NB];
        rhs.x -= g.x * y.x - g.y * y.y;
        rhs.y -= g.x * y.y + g.y * y.x;
      }
      if (r == c + 1) {                                       // publish row c+1 of Y (final now)
#pragma unroll
        for (int k = 0; k < 16; k++) rowc[nbuf][q + 4 * k] = yr[k];
        if (q == 0) rowc[nbuf][NB] = rhs;
      }
    }
  }
  __syncthreads();
  double2* linv = B.linv + (long long)p * NB * NB;
  const double isr = 1.0 / sqrt(piv[r]);
#pragma unroll
  for (int k = 0; k < 16; k++) {
    const int s = q + 4 * k;
    if (s < r) tile[(long long)r * np + s] = cscale(tr[k], 1.0 / sqrt(piv[s]));
    else if (s == r) tile[(long long)r * np + s] = make_double2(sqrt(piv[r]), 0.0);
    linv[r * NB + s] = s <= r ? cscale(yr[k], isr) : make_double2(0.0, 0.0);
  }
  if (q == 0) B.rhs[(long long)p * NB + r] = cscale(rhs, isr);
}

// b_i -= sum_c L[i][p*64 + c] y_p[c] for rows i >= (p+1)*64 (one warp per row).
__global__ void chol_rhs_update(CholSet cs, ActiveList act, int p) {
  const CholBlock& B = cs.b[act.idx[blockIdx.y]];
  const long long np = B.npad;
  const long long r0 = (long long)(p + 1) * NB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2* y = B.rhs + (long long)p * NB;
  const double2 y0 = y[lane], y1 = y[lane + 32];
  for (long long r = r0 + (long long)blockIdx.x * 8 + warp; r < np; r += (long long)gridDim.x * 8) {
    const double2* row = B.Fm + r * np + (long long)p * NB;
    double2 s = cmul(row[lane], y0);
    cfma(s, row[lane + 32], y1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    }
    if (lane == 0) B.rhs[r] = csub(B.rhs[r], s);
  }
}

// x_p = Linv_p^H y_p (into xout), then y_c -= sum_c' conj(L[p*64 + c'][c]) x_p[c'] for c < p*64.
// Each CTA owns 64 columns; 256 threads = 64 columns x 4 row quarters, reduced in a fixed
// order through shared memory (deterministic).
__global__ void __launch_bounds__(256) chol_back(CholSet cs, ActiveList act, int p) {
  __shared__ double2 ys[NB];
  __shared__ double2 xs[NB];
  __shared__ double2 red[4][NB];
  const CholBlock& B = cs.b[act.idx[blockIdx.y]];
  const long long np = B.npad;
  const int t = threadIdx.x;
  if (t < NB) ys[t] = B.rhs[(long long)p * NB + t];
  __syncthreads();
  const double2* linv = B.linv + (long long)p * NB * NB;
  {
    const int c = t >> 2, q = t & 3;
    double2 s = make_double2(0.0, 0.0);
    for (int r = c + q; r < NB; r += 4) cfma_conj(s, linv[r * NB + c], ys[r]);
    s.x += __shfl_xor_sync(0xffffffffu, s.x, 1);
    s.y += __shfl_xor_sync(0xffffffffu, s.y, 1);
    s.x += __shfl_xor_sync(0xffffffffu, s.x, 2);
    s.y += __shfl_xor_sync(0xffffffffu, s.y, 2);
    if (q == 0) xs[c] = s;
  }
  __syncthreads();
  if (blockIdx.x == 0 && t < NB) B.xout[(long long)p * NB + t] = xs[t];
  const long long ncol = (long long)p * NB;
  const int cl = t & 63, rq = t >> 6;
  for (long long c0 = (long long)blockIdx.x * NB; c0 < ncol; c0 += (long long)gridDim.x * NB) {
    const long long c = c0 + cl;
    double2 s = make_double2(0.0, 0.0);
    const double2* col = B.Fm + ((long long)p * NB + rq * 16) * np + c;
#pragma unroll 4
    for (int r = 0; r < 16; r++) cfma_conj(s, col[(long long)r * np], xs[rq * 16 + r]);
    red[rq][cl] = s;
    __syncthreads();
    if (rq == 0) {
      double2 v = cadd(cadd(red[0][cl], red[1][cl]), cadd(red[2][cl], red[3][cl]));
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
  }
}

sr_status chol_solve(CholSet& cs, double lam, bool inplace, double sign, cudaStream_t st) {
  int pmax = 0;
  for (int b = 0; b < cs.count; b++) pmax = std::max(pmax, cs.b[b].P);
  if (cs.info) SR_CUDA(cudaMemsetAsync(cs.info, 0, sizeof(int), st));
  {
    long long mx = 0;
    for (int b = 0; b < cs.count; b++) mx = std::max(mx, cs.b[b].npad * cs.b[b].npad);
    dim3 g((unsigned)std::min<long long>((mx + 255) / 256, 2 * kNumSMs), (unsigned)cs.count);
    chol_init<<<g, 256, 0, st>>>(cs, lam, inplace ? 1 : 0);
    SR_LAUNCHED();
  }
  for (int p = 0; p < pmax; p++) {
    ActiveList act;
    act.n = 0;
    long long max_trail = 0;
    for (int b = 0; b < cs.count; b++)
      if (cs.b[b].P > p) {
        act.idx[act.n++] = b;
        max_trail = std::max(max_trail, cs.b[b].npad - (long long)(p + 1) * NB);
      }
    chol_diag<<<act.n, 256, 0, st>>>(cs, act, p);
    SR_LAUNCHED();
    if (max_trail <= 0) continue;
    gram::ProbSet trsm{}, trail{};
    for (int i = 0; i < act.n; i++) {
      const CholBlock& B = cs.b[act.idx[i]];
      const long long m = B.npad - (long long)(p + 1) * NB;
      if (m <= 0) continue;
      double2* panel = B.Fm + (long long)(p + 1) * NB * B.npad + (long long)p * NB;
      gram::add_prob(trsm, panel, B.npad, B.linv + (long long)p * NB * NB, NB, panel, B.npad, (int)m, NB, NB,
                     false);
      double2* trailing = B.Fm + (long long)(p + 1) * NB * B.npad + (long long)(p + 1) * NB;
      gram::add_prob(trail, panel, B.npad, panel, B.npad, trailing, B.npad, (int)m, (int)m, NB, true);
    }
    SR_TRY((gram::launch<gram::NH, gram::STORE>(trsm, st)));
    {
      dim3 g((unsigned)std::min<long long>((max_trail + 7) / 8, 4 * kNumSMs), (unsigned)act.n);
      chol_rhs_update<<<g, 256, 0, st>>>(cs, act, p);
      SR_LAUNCHED();
    }
    SR_TRY((gram::launch<gram::NH, gram::SUB>(trail, st)));
  }
  for (int p = pmax - 1; p >= 0; p--) {
    ActiveList act;
    act.n = 0;
    for (int b = 0; b < cs.count; b++)
      if (cs.b[b].P > p) act.idx[act.n++] = b;
    dim3 g((unsigned)std::max(1, p), (unsigned)act.n);
    chol_back<<<g, 256, 0, st>>>(cs, act, p);
    SR_LAUNCHED();
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
