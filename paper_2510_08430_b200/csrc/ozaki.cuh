// ozaki.cuh — stage (4) on the 5th-generation tensor cores (tcgen05 kind::i8), see ozaki.cu.
#pragma once
#include "common.cuh"

namespace sr {
namespace oz {

constexpr int kSlices = 7;   // int8 digits per scaled value (54 bits, DESIGN.md §5 "Ozaki")

// Workspace bytes of block_qgt_i8 for n_samples rows and the given block partition.
size_t workspace_bytes(long long ns, int nblk, const int64_t* offs);

// S_b = A_b^H A_b for every block (same contract as sr_block_qgt), computed from the int8
// digit slices of the column-scaled A with tcgen05 kind::i8 MMAs accumulated exactly in
// TMEM (int32) and recombined in FP64.
sr_status block_qgt_i8(long long ns, int nblk, const int64_t* offs, const double2* A, long long lda, double2* S,
                       void* ws, size_t ws_bytes, cudaStream_t st, long long ldc = 0, bool accumulate = false);
// (accumulate: S += A_b^H A_b instead of S = ..., the sample-chunked step.)
// (ldc > 0, one block: the result is written with that leading dimension, e.g. straight into
// a padded Cholesky matrix -- the full-QGT solve.)

// T = L L^H (both triangles, real diagonal) for the m rows of L (m x K, row-major, ld ldl),
// written with leading dimension ldc: the NTK Gram A A^H of the sample-space solve.  Rows are
// scaled and split like the trailing updates' L; any K (chunked exact accumulation).
size_t rows_workspace_bytes(long long m, long long K);
sr_status gram_rows_i8(const double2* L, long long ldl, long long m, long long K, double2* C, long long ldc, void* ws,
                       size_t ws_bytes, cudaStream_t st);

// Cholesky trailing update C[i][j] -= sum_k L[i][k] conj(L[j][k]) for i >= j < m (lower
// triangle only; C row-major with leading dimension ldc, L row-major along k with ldl),
// by the same digit-slice tcgen05 engine.  K <= 8192.  max_ctas caps the persistent grid
// (0 = one CTA per SM).
size_t trail_workspace_bytes(long long m, long long K);
sr_status trail_update_i8(const double2* L, long long ldl, long long m, long long K, double2* C, long long ldc,
                          void* ws, size_t ws_bytes, int max_ctas, cudaStream_t st);
// The same update in parts (lookahead): trail_split_i8 scales and splits the rows of L
// into the workspace once; trail_apply_i8 then applies C -= L L^H to the lower triangle of
// the trailing square [r0, m) x [r0, m), with jlim > 0 only to its first 64 jlim columns
// (a lower trapezoid).  ctas sets the grid: 0 = one CTA per SM (persistent), n > 0 = n
// CTAs, n < 0 = one CTA per -n tiles (non-persistent: CTAs retire as they finish, so work
// on higher-priority streams gets SMs meanwhile).  The workspace must hold the split of the same L.
sr_status trail_split_i8(const double2* L, long long ldl, long long m, long long K, void* ws, size_t ws_bytes,
                         cudaStream_t st);
sr_status trail_apply_i8(long long m, long long K, double2* C, long long ldc, void* ws, long long r0, int jlim,
                         long long ctas, cudaStream_t st);

// Rectangles of the same engine (the distributed dense full QGT): cols_prepare splits all
// ncols columns of A once; cols_rect_gram then forms C (m x n) (+)= A[:, row0:row0+m]^H A[:, 0:n];
// rows_rect_sub applies C -= L[row0:row0+m] L[0:n]^H for the rows of L (rows x K, K <= 8192)
// split by trail_split_i8 into the same workspace.
size_t cols_workspace_bytes(long long ns, long long ncols);
sr_status cols_prepare(const double2* A, long long lda, long long ns, long long ncols, void* ws, size_t ws_bytes,
                       cudaStream_t st);
sr_status cols_rect_gram(long long ns, long long ncols, void* ws, size_t ws_bytes, long long row0, long long m,
                         long long n, double2* C, long long ldc, bool accumulate, cudaStream_t st);
sr_status rows_rect_sub(long long rows, long long K, long long row0, long long m, long long n, double2* C,
                        long long ldc, void* ws, size_t ws_bytes, cudaStream_t st);

}  // namespace oz
}  // namespace sr
