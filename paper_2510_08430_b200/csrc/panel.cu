// panel.cu — building blocks of the distributed dense full-QGT solve (parallel.dist_full_qgt):
// S = A^H A held by block rows across ranks and factorised by a right-looking blocked Cholesky
// whose panels travel between ranks (§2 "S . delta theta = -F" with the full QGT; §1:
// the full QGT "cannot be easily parallelized across multiple devices").
//
//   sr_gram_tn      C = A^H B   (the partial QGT rows A_r[:, rows]^H A_r[:, cols], FP64 DMMA)
//   sr_gram_nh_sub  C -= A B^H  (the trailing update S_qj -= L_qp L_jp^H, FP64 DMMA)
//   sr_chol_inv     M + lambda I = L L^H for one diagonal block (the library's blocked Cholesky)
//                   and L^{-1} explicitly (tile columns of the inverse by forward substitution
//                   with the 64x64 diagonal-tile inverses the factorisation forms), so that
//                   the panel TRSM L_qp = S_qp L_pp^{-H} is one sr_gram_nh on every rank.
#include <algorithm>

#include "chol.cuh"
#include "gram.cuh"
#include "ozaki.cuh"

namespace sr {
namespace {

constexpr int TB = 64;   // tile of the triangular inverse (the Cholesky's diagonal tile)

// X = L^{-1} for the padded factor L (Fm, ld np, T = np/64 tile rows), one CTA per tile
// column j: X_jj = Linv_j (from the factorisation), then for i = j+1 .. T-1
// X_ij = -Linv_i sum_{k=j}^{i-1} L_ik X_kj, the tiles of column j computed in order (each CTA
// reads only its own earlier tiles).  Thread t holds row t/4, columns 16 (t%4) .. +15 of the
// 64x64 accumulator; operand tiles are staged in shared memory.
__global__ void __launch_bounds__(256) tri_inv(const double2* __restrict__ L, long long np,
                                               const double2* __restrict__ linv, double2* __restrict__ X) {
  extern __shared__ __align__(16) double2 sm[];
  double2* sa = sm;               // [64][64] left operand
  double2* sb = sm + TB * TB;     // [64][64] right operand
  const int j = blockIdx.x, T = (int)(np / TB);
  const int t = threadIdx.x, r = t >> 2, c0 = (t & 3) * 16;
  auto tile = [&](auto* base, long long ld, int I, int J) { return base + (long long)I * TB * ld + (long long)J * TB; };
  // X_jj = Linv_j
  for (int e = t; e < TB * TB; e += 256) tile(X, np, j, j)[(e >> 6) * np + (e & 63)] = linv[(long long)j * TB * TB + e];
  for (int i = j + 1; i < T; i++) {
    double2 acc[16];
#pragma unroll
    for (int q = 0; q < 16; q++) acc[q] = make_double2(0.0, 0.0);
    for (int k = j; k < i; k++) {
      __syncthreads();
      const double2* Lik = tile(L, np, i, k);
      const double2* Xkj = tile(X, np, k, j);
      for (int e = t; e < TB * TB; e += 256) {
        sa[e] = Lik[(e >> 6) * np + (e & 63)];
        sb[e] = Xkj[(e >> 6) * np + (e & 63)];
      }
      __syncthreads();
      for (int m = 0; m < TB; m++) {
        const double2 a = sa[r * TB + m];
#pragma unroll
        for (int q = 0; q < 16; q++) cfma(acc[q], a, sb[m * TB + c0 + q]);
      }
    }
    // X_ij = -Linv_i acc
    __syncthreads();
    const double2* li = linv + (long long)i * TB * TB;
    for (int e = t; e < TB * TB; e += 256) sa[e] = li[e];
#pragma unroll
    for (int q = 0; q < 16; q++) sb[r * TB + c0 + q] = acc[q];
    __syncthreads();
    double2 out[16];
#pragma unroll
    for (int q = 0; q < 16; q++) out[q] = make_double2(0.0, 0.0);
    for (int m = 0; m < TB; m++) {
      const double2 a = sa[r * TB + m];
#pragma unroll
      for (int q = 0; q < 16; q++) cfma(out[q], a, sb[m * TB + c0 + q]);
    }
    double2* xij = tile(X, np, i, j);
#pragma unroll
    for (int q = 0; q < 16; q++) xij[(long long)r * np + c0 + q] = make_double2(-out[q].x, -out[q].y);
  }
}

// dst (n x n, ld) = lower triangle of src (ld np), zeros above the diagonal.
__global__ void copy_lower(const double2* __restrict__ src, long long np, double2* __restrict__ dst, long long ld,
                           long long n) {
  const long long total = n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / n, c = e % n;
    dst[r * ld + c] = c <= r ? src[r * np + c] : make_double2(0.0, 0.0);
  }
}

size_t chol_inv_ws(long long n) {
  long long sz = n;
  Arena a(nullptr, 0);
  CholSet cs{};
  carve_chol(a, cs, &sz, 1);
  const long long np = cs.b[0].npad;
  a.take<double2>(np);                    // zero right-hand side
  a.take<double2>(np);                    // discarded solution
  a.take<double2>((size_t)np * np);       // padded inverse
  return a.used;
}

unsigned grid_of(long long n) { return (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 8 * kNumSMs)); }

}  // namespace
}  // namespace sr

using namespace sr;

extern "C" {

SR_API sr_status sr_gram_tn(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B, int64_t ldb,
                            double* C, int64_t ldc, void* stream) {
  SR_CHECK_ARG(m >= 0 && n >= 0 && k >= 0 && m < (1LL << 31) && n < (1LL << 31), "bad sizes");
  SR_CHECK_ARG(lda >= m && ldb >= n && ldc >= n, "leading dimension too small");
  if (m == 0 || n == 0) return SR_OK;
  SR_CHECK_ARG(C && ((A && B) || k == 0), "null pointer");
  gram::ProbSet ps{};
  gram::add_prob(ps, reinterpret_cast<const double2*>(A), lda, reinterpret_cast<const double2*>(B), ldb,
                 reinterpret_cast<double2*>(C), ldc, (int)m, (int)n, k, false);
  return gram::launch<gram::TN, gram::STORE>(ps, (cudaStream_t)stream);
}

SR_API sr_status sr_gram_nh_sub(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                                int64_t ldb, double* C, int64_t ldc, void* stream) {
  SR_CHECK_ARG(m >= 0 && n >= 0 && k >= 0 && m < (1LL << 31) && n < (1LL << 31), "bad sizes");
  SR_CHECK_ARG(lda >= k && ldb >= k && ldc >= n, "leading dimension too small");
  if (m == 0 || n == 0 || k == 0) return SR_OK;
  SR_CHECK_ARG(A && B && C, "null pointer");
  gram::ProbSet ps{};
  gram::add_prob(ps, reinterpret_cast<const double2*>(A), lda, reinterpret_cast<const double2*>(B), ldb,
                 reinterpret_cast<double2*>(C), ldc, (int)m, (int)n, k, false);
  return gram::launch<gram::NH, gram::SUB>(ps, (cudaStream_t)stream);
}

SR_API size_t sr_cols_i8_workspace_bytes(int64_t n_samples, int64_t n_cols) {
  if (n_samples < 0 || n_cols < 1) return 0;
  return oz::cols_workspace_bytes(n_samples, n_cols);
}

SR_API sr_status sr_cols_i8_prepare(int64_t n_samples, int64_t n_cols, const double* A, int64_t lda, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(n_samples >= 0 && n_cols >= 1 && lda >= n_cols && n_cols < (1LL << 31) / oz::kSlices, "bad sizes");
  SR_CHECK_ARG(workspace && (A || n_samples == 0), "null pointer");
  if (n_samples == 0) return SR_OK;
  return oz::cols_prepare(reinterpret_cast<const double2*>(A), lda, n_samples, n_cols, workspace, workspace_bytes,
                          (cudaStream_t)stream);
}

SR_API sr_status sr_cols_i8_gram(int64_t n_samples, int64_t n_cols, int64_t row0, int64_t m, int64_t n, double* C,
                                 int64_t ldc, int accumulate, void* workspace, size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(n_samples >= 0 && n_cols >= 1 && m >= 0 && n >= 0 && ldc >= n, "bad sizes");
  SR_CHECK_ARG(row0 >= 0 && row0 + m <= n_cols && n <= n_cols, "rows / columns outside the prepared matrix");
  SR_CHECK_ARG((C || m == 0 || n == 0) && workspace, "null pointer");
  return oz::cols_rect_gram(n_samples, n_cols, workspace, workspace_bytes, row0, m, n, reinterpret_cast<double2*>(C),
                            ldc, accumulate != 0, (cudaStream_t)stream);
}

SR_API size_t sr_rows_i8_sub_workspace_bytes(int64_t rows, int64_t K) {
  if (rows < 1 || K < 1) return 0;
  return oz::trail_workspace_bytes(rows, K);
}

SR_API sr_status sr_rows_i8_prepare(int64_t rows, int64_t K, const double* L, int64_t ldl, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(rows >= 1 && K >= 1 && K <= 8192 && ldl >= K && rows < (1LL << 31) / oz::kSlices, "bad sizes");
  SR_CHECK_ARG(L && workspace, "null pointer");
  return oz::trail_split_i8(reinterpret_cast<const double2*>(L), ldl, rows, K, workspace, workspace_bytes,
                            (cudaStream_t)stream);
}

SR_API sr_status sr_rows_i8_sub(int64_t rows, int64_t K, int64_t row0, int64_t m, int64_t n, double* C, int64_t ldc,
                                void* workspace, size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(rows >= 1 && K >= 1 && K <= 8192 && m >= 0 && n >= 0 && ldc >= n, "bad sizes");
  SR_CHECK_ARG(row0 >= 0 && row0 + m <= rows && n <= rows, "rows outside L");
  SR_CHECK_ARG((C || m == 0 || n == 0) && workspace, "null pointer");
  return oz::rows_rect_sub(rows, K, row0, m, n, reinterpret_cast<double2*>(C), ldc, workspace, workspace_bytes,
                           (cudaStream_t)stream);
}

SR_API size_t sr_chol_inv_workspace_bytes(int64_t n) { return n < 1 ? 0 : chol_inv_ws(n); }

SR_API sr_status sr_chol_inv(int64_t n, const double* M, double lambda, double* L, int64_t ldl, double* Linv,
                             int64_t ldv, int32_t* info, void* workspace, size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(n >= 1 && n < (1LL << 31) && ldl >= n && ldv >= n, "bad sizes");
  SR_CHECK_ARG(M && L && Linv && workspace, "null pointer");
  SR_CHECK_ARG(lambda >= 0.0, "lambda < 0");
  cudaStream_t st = (cudaStream_t)stream;
  long long sz = n;
  Arena a(workspace, workspace_bytes);
  CholSet cs{};
  cs.info = info;
  carve_chol(a, cs, &sz, 1);
  CholBlock& B = cs.b[0];
  const long long np = B.npad;
  double2* zero = a.take<double2>(np);
  double2* sol = a.take<double2>(np);
  double2* Xp = a.take<double2>((size_t)np * np);
  if (!a.ok()) {
    set_error("sr_chol_inv: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  SR_CUDA(cudaMemsetAsync(zero, 0, np * sizeof(double2), st));
  B.S = reinterpret_cast<const double2*>(M);
  B.F = zero;
  B.out = sol;
  SR_TRY(chol_solve(cs, lambda, false, -1.0, st));   // factorisation (the solve of 0 is a by-product)
  static unsigned long long attr = 0;
  const size_t smem = 2 * TB * TB * sizeof(double2);
  if (first_on_device(attr)) SR_CUDA(cudaFuncSetAttribute(tri_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  tri_inv<<<(unsigned)(np / TB), 256, smem, st>>>(B.Fm, np, B.linv, Xp);
  SR_LAUNCHED();
  copy_lower<<<grid_of(n * n), 256, 0, st>>>(B.Fm, np, reinterpret_cast<double2*>(L), ldl, n);
  SR_LAUNCHED();
  copy_lower<<<grid_of(n * n), 256, 0, st>>>(Xp, np, reinterpret_cast<double2*>(Linv), ldv, n);
  SR_LAUNCHED();
  return SR_OK;
}

}  // extern "C"
