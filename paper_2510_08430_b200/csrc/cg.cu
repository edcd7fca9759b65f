// cg.cu — matrix-free full-QGT solve support: (S + lambda I) x = -F with S = A^H A applied
// as A^H (A p), never formed (§2 "S . delta theta = -F"; the full QGT of configs[3]
// is 146 GB and cannot be held or reduced on one B200).  With samples sharded over ranks,
// S p = sum_r A_r^H (A_r p): each rank applies its rows and one all-reduce of n_p values
// sums them (parallel.full_qgt_cg).  Conjugate gradients on the Hermitian positive-definite
// S + lambda I; every vector update is replicated identically on all ranks.
//
// Kernels: av_rows (out = alpha A v, one warp per row, fixed-order lane sums: HBM-bound
// stream of A), zdotc (fixed-order two-level reduction), and the CG updates, which take the
// step scalars as device values (alpha = num / den computed in the kernel, no host round trip).
#include "common.cuh"

namespace sr {
namespace {

constexpr int kDotBlocks = 2 * kNumSMs;

// out[k] = alpha * sum_i A[k][i] v[i]
__global__ void __launch_bounds__(256) av_rows(const double2* __restrict__ A, long long lda, long long nrows,
                                               long long np, const double2* __restrict__ v, double alpha,
                                               double2* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= nrows) return;
  const double2* a = A + row * lda;
  double2 s0 = make_double2(0.0, 0.0), s1 = s0, s2 = s0, s3 = s0;
  long long i = lane;
  for (; i + 96 < np; i += 128) {
    cfma(s0, a[i], v[i]);
    cfma(s1, a[i + 32], v[i + 32]);
    cfma(s2, a[i + 64], v[i + 64]);
    cfma(s3, a[i + 96], v[i + 96]);
  }
  for (; i < np; i += 32) cfma(s0, a[i], v[i]);
  double2 s = cadd(cadd(s0, s1), cadd(s2, s3));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
    s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
  }
  if (lane == 0) out[row] = cscale(s, alpha);
}

__device__ __forceinline__ double2 block_sum(double2 s, double2* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
    s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
  }
  if (lane == 0) sh[warp] = s;
  __syncthreads();
  if (warp == 0) {
    s = lane < (int)(blockDim.x >> 5) ? sh[lane] : make_double2(0.0, 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    }
  }
  return s;
}

// part[b] = sum over this block's fixed strided elements of conj(x) y
__global__ void __launch_bounds__(256) zdotc_partial(long long n, const double2* __restrict__ x,
                                                     const double2* __restrict__ y, double2* __restrict__ part) {
  __shared__ double2 sh[8];
  double2 s = make_double2(0.0, 0.0);
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
    cfma_conj(s, x[i], y[i]);
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(256) zdotc_final(const double2* __restrict__ part, int nparts,
                                                   double2* __restrict__ out) {
  __shared__ double2 sh[8];
  double2 s = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < nparts; i += 256) s = cadd(s, part[i]);
  s = block_sum(s, sh);
  if (threadIdx.x == 0) *out = s;
}

// y += sign * (num / den) * x   (num, den: device complex scalars)
__global__ void cg_axpy(long long n, const double2* __restrict__ x, double2* __restrict__ y,
                        const double2* __restrict__ num, const double2* __restrict__ den, double sign) {
  const double2 a = cscale(cdiv(*num, *den), sign);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    cfma(y[i], a, x[i]);
}

// y = x + (num / den) * y
__global__ void cg_xpby(long long n, const double2* __restrict__ x, double2* __restrict__ y,
                        const double2* __restrict__ num, const double2* __restrict__ den) {
  const double2 b = cdiv(*num, *den);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = cadd(x[i], cmul(b, y[i]));
}

unsigned grid_for(long long n) {
  return (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 4 * kNumSMs));
}

}  // namespace
}  // namespace sr

using namespace sr;

extern "C" {

SR_API sr_status sr_av(int64_t n_rows, int64_t n_p, const double* A, int64_t lda, const double* v, double alpha,
                       double* out, void* stream) {
  SR_CHECK_ARG(n_rows >= 0 && n_p >= 0 && lda >= n_p, "bad sizes");
  if (n_rows == 0) return SR_OK;
  SR_CHECK_ARG(out && (n_p == 0 || (A && v)), "null pointer");
  av_rows<<<(unsigned)((n_rows + 7) / 8), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const double2*>(A), lda, n_rows, n_p, reinterpret_cast<const double2*>(v), alpha,
      reinterpret_cast<double2*>(out));
  SR_LAUNCHED();
  return SR_OK;
}

SR_API size_t sr_zdotc_workspace_bytes(void) { return round256(kDotBlocks * sizeof(double2)); }

SR_API sr_status sr_zdotc(int64_t n, const double* x, const double* y, double* out, void* workspace,
                          size_t workspace_bytes, void* stream) {
  SR_CHECK_ARG(n >= 0, "n < 0");
  SR_CHECK_ARG(out && workspace && (n == 0 || (x && y)), "null pointer");
  SR_CHECK_ARG(workspace_bytes >= kDotBlocks * sizeof(double2), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  double2* part = static_cast<double2*>(workspace);
  zdotc_partial<<<kDotBlocks, 256, 0, st>>>(n, reinterpret_cast<const double2*>(x),
                                            reinterpret_cast<const double2*>(y), part);
  SR_LAUNCHED();
  zdotc_final<<<1, 256, 0, st>>>(part, kDotBlocks, reinterpret_cast<double2*>(out));
  SR_LAUNCHED();
  return SR_OK;
}

SR_API sr_status sr_cg_axpy(int64_t n, const double* x, double* y, const double* num, const double* den, double sign,
                            void* stream) {
  SR_CHECK_ARG(n >= 0, "n < 0");
  if (n == 0) return SR_OK;
  SR_CHECK_ARG(x && y && num && den, "null pointer");
  cg_axpy<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, reinterpret_cast<const double2*>(x),
                                                         reinterpret_cast<double2*>(y),
                                                         reinterpret_cast<const double2*>(num),
                                                         reinterpret_cast<const double2*>(den), sign);
  SR_LAUNCHED();
  return SR_OK;
}

SR_API sr_status sr_cg_xpby(int64_t n, const double* x, double* y, const double* num, const double* den,
                            void* stream) {
  SR_CHECK_ARG(n >= 0, "n < 0");
  if (n == 0) return SR_OK;
  SR_CHECK_ARG(x && y && num && den, "null pointer");
  cg_xpby<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, reinterpret_cast<const double2*>(x),
                                                         reinterpret_cast<double2*>(y),
                                                         reinterpret_cast<const double2*>(num),
                                                         reinterpret_cast<const double2*>(den));
  SR_LAUNCHED();
  return SR_OK;
}

}  // extern "C"
