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
constexpr int LDT = NB + 1;

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

// One CTA per active block.  Factors the diagonal tile of panel p in place, writes
// Linv_p, and replaces b_p by y_p = Linv_p b_p.
__global__ void __launch_bounds__(256) chol_diag(CholSet cs, ActiveList act, int p) {
  extern __shared__ double2 sm[];
  double2* T = sm;              // [64][65]  factor tile
  double2* X = sm + NB * LDT;   // [64][65]  inverse
  __shared__ double2 yb[NB];
  const CholBlock& B = cs.b[act.idx[blockIdx.x]];
  const long long np = B.npad;
  double2* tile = B.Fm + (long long)p * NB * np + (long long)p * NB;
  const int t = threadIdx.x;
  for (int e = t; e < NB * NB; e += 256) {
    const int r = e >> 6, c = e & 63;
    T[r * LDT + c] = c <= r ? tile[(long long)r * np + c] : make_double2(0.0, 0.0);
  }
  if (t < NB) yb[t] = B.rhs[(long long)p * NB + t];
  __syncthreads();
  // unblocked right-looking Cholesky, lower
  const int tr = t >> 2, tq = t & 3;
  for (int c = 0; c < NB; c++) {
    __syncthreads();  // step c-1's trailing update (which wrote T[c][c]) is visible
    double d = T[c * LDT + c].x;
    if (!(d > 0.0)) {
      if (t == 0 && cs.info) atomicCAS(cs.info, 0, (int)(B.row_base + (long long)p * NB + c + 1));
      d = 1.0;
    }
    const double sd = sqrt(d), isd = 1.0 / sd;
    __syncthreads();
    if (t == 0) T[c * LDT + c] = make_double2(sd, 0.0);
    if (t > c && t < NB) T[t * LDT + c] = cscale(T[t * LDT + c], isd);
    __syncthreads();
    if (tr > c) {
      const double2 lrc = T[tr * LDT + c];
      for (int s = c + 1 + tq; s <= tr; s += 4) {
        const double2 lsc = T[s * LDT + c];
        // T[r][s] -= L[r][c] conj(L[s][c])
        double2 v = T[tr * LDT + s];
        v.x -= lrc.x * lsc.x + lrc.y * lsc.y;
        v.y -= lrc.y * lsc.x - lrc.x * lsc.y;
        T[tr * LDT + s] = v;
      }
    }
  }
  __syncthreads();
  // X = L^{-1}: column j per quad of lanes, forward substitution, quad-reduced sums.
  {
    const int j = t >> 2, q = t & 3;
    for (int r = 0; r < NB; r++) {
      double2 s = make_double2(0.0, 0.0);
      if (r >= j)
        for (int k = j + q; k < r; k += 4) cfma(s, T[r * LDT + k], X[k * LDT + j]);
      s.x += __shfl_xor_sync(0xffffffffu, s.x, 1);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, 1);
      s.x += __shfl_xor_sync(0xffffffffu, s.x, 2);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, 2);
      if (q == 0) {
        double2 x = make_double2(0.0, 0.0);
        if (r >= j) {
          const double inv = 1.0 / T[r * LDT + r].x;
          x = make_double2(((r == j ? 1.0 : 0.0) - s.x) * inv, -s.y * inv);
        }
        X[r * LDT + j] = x;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  double2* linv = B.linv + (long long)p * NB * NB;
  for (int e = t; e < NB * NB; e += 256) {
    const int r = e >> 6, c = e & 63;
    if (c <= r) tile[(long long)r * np + c] = T[r * LDT + c];
    linv[e] = X[r * LDT + c];
  }
  if (t < NB) {
    double2 y = make_double2(0.0, 0.0);
    for (int c = 0; c <= t; c++) cfma(y, X[t * LDT + c], yb[c]);
    B.rhs[(long long)p * NB + t] = y;
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
__global__ void __launch_bounds__(256) chol_back(CholSet cs, ActiveList act, int p) {
  __shared__ double2 ys[NB];
  __shared__ double2 xs[NB];
  const CholBlock& B = cs.b[act.idx[blockIdx.y]];
  const long long np = B.npad;
  const int t = threadIdx.x;
  if (t < NB) ys[t] = B.rhs[(long long)p * NB + t];
  __syncthreads();
  const double2* linv = B.linv + (long long)p * NB * NB;
  {
    // 4 lanes per output c, rows r >= c split by r % 4
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
  for (long long c = (long long)blockIdx.x * 256 + t; c < ncol; c += (long long)gridDim.x * 256) {
    double2 s = make_double2(0.0, 0.0);
    const double2* col = B.Fm + (long long)p * NB * np + c;
#pragma unroll 8
    for (int r = 0; r < NB; r++) cfma_conj(s, col[(long long)r * np], xs[r]);
    B.rhs[c] = csub(B.rhs[c], s);
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
  const size_t diag_smem = 2 * NB * LDT * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    SR_CUDA(cudaFuncSetAttribute(chol_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)diag_smem));
    attr = true;
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
    chol_diag<<<act.n, 256, diag_smem, st>>>(cs, act, p);
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
    const long long ncol = (long long)p * NB;
    dim3 g((unsigned)std::max<long long>(1, (ncol + 255) / 256), (unsigned)act.n);
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
