// chol.cuh — batched blocked Cholesky solve interface (see chol.cu).
#pragma once
#include "common.cuh"

namespace sr {

constexpr int kMaxBlocks = 24;

struct CholBlock {
  const double2* S;   // source matrix (n x n, ld n) unless in place
  const double2* F;   // right-hand side [n]
  double2* out;       // solution destination [n] (sign applied)
  double2* Fm;        // padded factor matrix [npad][npad]
  double2* rhs;       // [npad]: b, then y, then the back-substitution residual
  double2* xout;      // [npad]: x
  double2* linv;      // [P][64][64]: inverses of the diagonal tiles
  void* tws;          // int8 trailing-update workspace (digit slices of one strip)
  size_t tws_bytes;
  long long n, npad, row_base;
  int P;
};

struct CholSet {
  int count;
  int* info;
  bool keep_info;   // true: do not reset *info (a caller solving blocks one call at a time)
  CholBlock b[kMaxBlocks];
};


// Carves Fm/rhs/xout/linv for blocks of the given sizes (S, F, out set by the caller).
void carve_chol(Arena& a, CholSet& cs, const long long* sizes, int nblk);
// Solves (M_b + lam I) x_b = F_b for all blocks; writes out_b = sign * x_b.  With
// inplace, M_b is already in Fm (ld npad, rows/cols < n) and only the diagonal shift
// and the identity padding are applied.  With ready (one event per block), block b's
// copy-in and factorisation wait for ready[b] instead of running after everything queued
// on st before the call (the step overlaps block b's solve with later blocks' Grams).
sr_status chol_solve(CholSet& cs, double lam, bool inplace, double sign, cudaStream_t st,
                     const cudaEvent_t* ready = nullptr);

}  // namespace sr
