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
//   inner (engine)   A_ij -= L_ip L_jp^H for the strip's later columns j (DMMA, NH/SUB)
// and after every strip of 4 panels one deferred trailing update with K = 256:
//   trail (engine)   A_ij -= L_i,strip L_j,strip^H for i >= j beyond the strip (NH/SUB)
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

// One CTA per active block: factor the 64x64 diagonal tile of panel p (left-looking), its
// inverse X = Linv_p (row by row) and y_p = Linv_p b_p.  Step c, one barrier:
//   d_c     = A[c][c] - sum_{k<c} |L[c][k]|^2                      (every quad, redundantly)
//   L[r][c] = (A[r][c] - sum_{k<c} L[r][k] conj(L[c][k])) / sqrt(d_c)   rows r > c
//   X[c][j] = -(sum_{j<=k<c} L[c][k] X[k][j]) / sqrt(d_c)               j = r < c
//   L[c][c] = sqrt(d_c), X[c][c] = 1/sqrt(d_c)                          quad r == c
// Quad (r, q) = (t/4, t%4) splits each dot product over k = q mod 4 and reduces with two
// shuffles.  Everything reads only entries finalised in earlier steps.
constexpr int LDS = NB + 4;   // 1088-byte rows: conflict-free quad access
constexpr size_t kDiagSmem = (size_t)2 * NB * LDS * sizeof(double2);
__global__ void __launch_bounds__(256) chol_diag(CholSet cs, ActiveList act, int p) {
  extern __shared__ double2 dsm[];
  double2* T = dsm;              // [64][LDS]: A (lower), columns replaced by L as they finish
  double2* X = dsm + NB * LDS;   // [64][LDS]: Linv rows
  __shared__ double2 bsh[NB];
  const CholBlock& B = cs.b[act.idx[blockIdx.x]];
  const long long np = B.npad;
  double2* tile = B.Fm + (long long)p * NB * np + (long long)p * NB;
  const int t = threadIdx.x, r = t >> 2, q = t & 3;
  for (int e = t; e < NB * NB; e += 256) {
    const int rr = e >> 6, c = e & 63;
    T[rr * LDS + c] = c <= rr ? tile[(long long)rr * np + c] : make_double2(0.0, 0.0);
    X[rr * LDS + c] = make_double2(0.0, 0.0);
  }
  if (t < NB) bsh[t] = B.rhs[(long long)p * NB + t];
  __syncthreads();
  for (int c = 0; c < NB; c++) {
    // pivot: d = A[c][c] - sum_{k<c} |L[c][k]|^2
    double dp0 = 0.0, dp1 = 0.0;
    int k = q;
    for (; k + 4 < c; k += 8) {
      const double2 u = T[c * LDS + k], v = T[c * LDS + k + 4];
      dp0 = fma(u.x, u.x, fma(u.y, u.y, dp0));
      dp1 = fma(v.x, v.x, fma(v.y, v.y, dp1));
    }
    if (k < c) {
      const double2 u = T[c * LDS + k];
      dp0 = fma(u.x, u.x, fma(u.y, u.y, dp0));
    }
    double dsum = dp0 + dp1;
    dsum += __shfl_xor_sync(0xffffffffu, dsum, 1);
    dsum += __shfl_xor_sync(0xffffffffu, dsum, 2);
    double d = T[c * LDS + c].x - dsum;
    if (!(d > 0.0)) {
      if (t == 0 && cs.info) atomicCAS(cs.info, 0, (int)(B.row_base + (long long)p * NB + c + 1));
      d = 1.0;
    }
    const double isd = 1.0 / sqrt(d);
    double2 s0 = make_double2(0.0, 0.0), s1 = s0;
    if (r > c) {
      // sum_{k<c} L[r][k] conj(L[c][k])
      int kk = q;
      for (; kk + 4 < c; kk += 8) {
        cfma_conj(s0, T[c * LDS + kk], T[r * LDS + kk]);
        cfma_conj(s1, T[c * LDS + kk + 4], T[r * LDS + kk + 4]);
      }
      if (kk < c) cfma_conj(s0, T[c * LDS + kk], T[r * LDS + kk]);
    } else if (r < c) {
      // sum_{r<=k<c} L[c][k] X[k][r]
      int kk = r + q;
      for (; kk + 4 < c; kk += 8) {
        cfma(s0, T[c * LDS + kk], X[kk * LDS + r]);
        cfma(s1, T[c * LDS + kk + 4], X[(kk + 4) * LDS + r]);
      }
      if (kk < c) cfma(s0, T[c * LDS + kk], X[kk * LDS + r]);
    }
    double2 sum = cadd(s0, s1);
    sum.x += __shfl_xor_sync(0xffffffffu, sum.x, 1);
    sum.y += __shfl_xor_sync(0xffffffffu, sum.y, 1);
    sum.x += __shfl_xor_sync(0xffffffffu, sum.x, 2);
    sum.y += __shfl_xor_sync(0xffffffffu, sum.y, 2);
    if (q == 0) {
      if (r > c) {
        T[r * LDS + c] = cscale(csub(T[r * LDS + c], sum), isd);
      } else if (r < c) {
        X[c * LDS + r] = make_double2(-sum.x * isd, -sum.y * isd);
      } else {
        T[c * LDS + c] = make_double2(d * isd, 0.0);   // sqrt(d)
        X[c * LDS + c] = make_double2(isd, 0.0);
      }
    }
    __syncthreads();
  }
  double2* linv = B.linv + (long long)p * NB * NB;
  for (int e = t; e < NB * NB; e += 256) {
    const int rr = e >> 6, c = e & 63;
    if (c <= rr) tile[(long long)rr * np + c] = T[rr * LDS + c];
    linv[e] = X[rr * LDS + c];
  }
  {
    double2 y = make_double2(0.0, 0.0);
    for (int c = q; c <= r; c += 4) cfma(y, X[r * LDS + c], bsh[c]);
    y.x += __shfl_xor_sync(0xffffffffu, y.x, 1);
    y.y += __shfl_xor_sync(0xffffffffu, y.y, 1);
    y.x += __shfl_xor_sync(0xffffffffu, y.x, 2);
    y.y += __shfl_xor_sync(0xffffffffu, y.y, 2);
    if (q == 0) B.rhs[(long long)p * NB + r] = y;
  }
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

namespace {

// Factorisation + substitutions of ONE block on one stream (two-level blocking, see header).
sr_status solve_block(CholSet& cs, int b, cudaStream_t st) {
  const CholBlock& B = cs.b[b];
  ActiveList act;
  act.n = 1;
  act.idx[0] = b;
  // Two-level blocking: strips of kStrip panels.  Inside a strip each panel p is factored
  // (chol_diag), its column solved (TRSM), the RHS updated, and only the strip's own later
  // columns updated (K = 64); the rest of the trailing matrix receives one deferred update
  // per strip with K = 64 * kStrip, which is where the flops are (4x the arithmetic
  // intensity of a per-panel update, 4x fewer passes over the trailing matrix).
  constexpr int kStrip = 4;
  for (int p0 = 0; p0 < B.P; p0 += kStrip) {
    const int pend = std::min(p0 + kStrip, B.P);
    for (int p = p0; p < pend; p++) {
      chol_diag<<<1, 256, kDiagSmem, st>>>(cs, act, p);
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
      SR_TRY((gram::launch<gram::NH, gram::STORE>(trsm, st)));
      dim3 g((unsigned)std::min<long long>((m + 7) / 8, 4 * kNumSMs), 1);
      chol_rhs_update<<<g, 256, 0, st>>>(cs, act, p);
      SR_LAUNCHED();
      SR_TRY((gram::launch<gram::NH, gram::SUB>(inner, st)));
    }
    const long long m = B.npad - (long long)pend * NB;
    if (m > 0) {   // deferred trailing update of the strip, K = 64 * (pend - p0)
      gram::ProbSet trail{};
      const double2* lp = B.Fm + (long long)pend * NB * B.npad + (long long)p0 * NB;
      double2* trailing = B.Fm + (long long)pend * NB * B.npad + (long long)pend * NB;
      gram::add_prob(trail, lp, B.npad, lp, B.npad, trailing, B.npad, (int)m, (int)m, (long long)(pend - p0) * NB, true);
      SR_TRY((gram::launch<gram::NH, gram::SUB>(trail, st)));
    }
  }
  for (int p = B.P - 1; p >= 0; p--) {
    dim3 g((unsigned)std::max(1, p), 1);
    chol_back<<<g, 256, 0, st>>>(cs, act, p);
    SR_LAUNCHED();
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
