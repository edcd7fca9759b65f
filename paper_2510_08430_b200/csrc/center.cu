// center.cu — stage (3) sr_center_force and the column reduction y = A^H v it shares
// with the NTK solve.
//
// PAPER.md Eq. 2: Delta O_i = O_i - <O_i>; north_star (3): F = Obar^H (E_loc - <E_loc>)/N_s.
// With sample weights w_k (uniform 1/N_s, or Born weights for full enumeration):
//   E = sum_k w_k E_k,  e_k = sqrt(w_k)(E_k - E),  <O> = sum_k w_k O_k,
//   A_k = sqrt(w_k)(O_k - <O>)  (in place),       F = A^H e.
// O is row-major [N_s][ldo]; every pass streams it with one thread per column (a warp
// reads 512 contiguous bytes of a row), rows split into chunks whose partial sums are
// reduced in a fixed chunk order (deterministic, no atomics).
#include "common.cuh"

namespace sr {
namespace {

constexpr int kColThreads = 256;

// ww[k] = w_k (given, or 1/n_total), sw[k] = sqrt(w_k).
__global__ void weights_prep(const double* __restrict__ weights, long long ns, long long n_total,
                             double* __restrict__ ww, double* __restrict__ sw) {
  const double uni = 1.0 / (double)n_total;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < ns;
       k += (long long)gridDim.x * blockDim.x) {
    const double w = weights ? weights[k] : uni;
    ww[k] = w;
    sw[k] = sqrt(w);
  }
}

// Single CTA: out = sum_k w_k E_k (fixed-order strided sums, then a fixed tree).
__global__ void __launch_bounds__(1024) wsum_energy(const double* __restrict__ ww, const double2* __restrict__ e_loc,
                                                    long long ns, double2* __restrict__ out) {
  __shared__ double2 red[1024];
  double2 s = make_double2(0.0, 0.0);
  for (long long k = threadIdx.x; k < ns; k += 1024) {
    const double w = ww[k];
    const double2 e = e_loc[k];
    s.x = fma(w, e.x, s.x);
    s.y = fma(w, e.y, s.y);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = cadd(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// e_tilde[k] = sqrt(w_k) (E_k - E)
__global__ void e_tilde_kernel(const double* __restrict__ sw, const double2* __restrict__ e_loc,
                               const double2* __restrict__ energy, long long ns, double2* __restrict__ e_tilde) {
  const double2 em = *energy;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < ns;
       k += (long long)gridDim.x * blockDim.x)
    e_tilde[k] = cscale(csub(e_loc[k], em), sw[k]);
}

// part[c_chunk][c] = sum_{k in chunk} w_k O[k][c]
__global__ void __launch_bounds__(kColThreads) colsum_partial(const double2* __restrict__ O, long long ldo,
                                                              long long ns, long long np, long long rows_per_chunk,
                                                              const double* __restrict__ ww,
                                                              double2* __restrict__ part) {
  const long long c = (long long)blockIdx.x * kColThreads + threadIdx.x;
  const long long k0 = (long long)blockIdx.y * rows_per_chunk;
  const long long k1 = min(ns, k0 + rows_per_chunk);
  if (c >= np) return;
  double2 s0 = make_double2(0.0, 0.0), s1 = s0;
  long long k = k0;
  for (; k + 1 < k1; k += 2) {
    const double2 a = O[k * ldo + c], b = O[(k + 1) * ldo + c];
    const double wa = ww[k], wb = ww[k + 1];
    s0.x = fma(wa, a.x, s0.x);
    s0.y = fma(wa, a.y, s0.y);
    s1.x = fma(wb, b.x, s1.x);
    s1.y = fma(wb, b.y, s1.y);
  }
  if (k < k1) {
    const double2 a = O[k * ldo + c];
    s0.x = fma(ww[k], a.x, s0.x);
    s0.y = fma(ww[k], a.y, s0.y);
  }
  part[(long long)blockIdx.y * np + c] = cadd(s0, s1);
}

__global__ void chunk_reduce(const double2* __restrict__ part, long long np, int n_chunks, double scale,
                             double2* __restrict__ out) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < np;
       c += (long long)gridDim.x * blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < n_chunks; q++) s = cadd(s, part[(long long)q * np + c]);
    out[c] = cscale(s, scale);
  }
}

// A[k][c] = sw_k (O[k][c] - mean[c]) in place; part[chunk][c] = sum_k conj(A[k][c]) e[k]
__global__ void __launch_bounds__(kColThreads) center_force_partial(double2* __restrict__ O, long long ldo,
                                                                    long long ns, long long np,
                                                                    long long rows_per_chunk,
                                                                    const double* __restrict__ sw,
                                                                    const double2* __restrict__ mean,
                                                                    const double2* __restrict__ e,
                                                                    double2* __restrict__ part) {
  const long long c = (long long)blockIdx.x * kColThreads + threadIdx.x;
  const long long k0 = (long long)blockIdx.y * rows_per_chunk;
  const long long k1 = min(ns, k0 + rows_per_chunk);
  if (c >= np) return;
  const double2 m = mean[c];
  double2 s = make_double2(0.0, 0.0);
  for (long long k = k0; k < k1; k++) {
    const double2 a = cscale(csub(O[k * ldo + c], m), sw[k]);
    O[k * ldo + c] = a;
    cfma_conj(s, a, e[k]);
  }
  part[(long long)blockIdx.y * np + c] = s;
}

// part[chunk][c] = sum_{k in chunk} conj(A[k][c]) v[k]
__global__ void __launch_bounds__(kColThreads) aHv_partial(const double2* __restrict__ A, long long lda,
                                                           long long ns, long long np, long long rows_per_chunk,
                                                           const double2* __restrict__ v,
                                                           double2* __restrict__ part) {
  const long long c = (long long)blockIdx.x * kColThreads + threadIdx.x;
  const long long k0 = (long long)blockIdx.y * rows_per_chunk;
  const long long k1 = min(ns, k0 + rows_per_chunk);
  if (c >= np) return;
  double2 s0 = make_double2(0.0, 0.0), s1 = s0;
  long long k = k0;
  for (; k + 1 < k1; k += 2) {
    cfma_conj(s0, A[k * lda + c], v[k]);
    cfma_conj(s1, A[(k + 1) * lda + c], v[k + 1]);
  }
  if (k < k1) cfma_conj(s0, A[k * lda + c], v[k]);
  part[(long long)blockIdx.y * np + c] = cadd(s0, s1);
}

struct ChunkPlan {
  long long strips, chunks, rows;
};
ChunkPlan plan_chunks(long long ns, long long np) {
  ChunkPlan p;
  p.strips = (np + kColThreads - 1) / kColThreads;
  long long want = (4LL * kNumSMs + p.strips - 1) / p.strips;   // >= 4 CTAs per SM
  long long max_chunks = std::max<long long>(1, (ns + 31) / 32);  // at least 32 rows per chunk
  p.chunks = std::max<long long>(1, std::min(want, max_chunks));
  p.rows = (ns + p.chunks - 1) / p.chunks;
  p.chunks = (ns + p.rows - 1) / p.rows;
  if (p.chunks < 1) p.chunks = 1;
  return p;
}

}  // namespace

size_t aHv_ws(long long ns, long long np) {
  ChunkPlan p = plan_chunks(ns, np);
  return round256((size_t)p.chunks * np * sizeof(double2));
}

// out[c] = scale * sum_k conj(A[k][c]) v[k]
sr_status aHv_impl(long long ns, long long np, const double2* A, long long lda, const double2* v, double scale,
                   double2* out, void* ws, size_t ws_bytes, cudaStream_t st) {
  ChunkPlan p = plan_chunks(ns, np);
  Arena a(ws, ws_bytes);
  double2* part = a.take<double2>((size_t)p.chunks * np);
  if (!a.ok()) {
    set_error("aHv: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  dim3 g((unsigned)p.strips, (unsigned)p.chunks);
  aHv_partial<<<g, kColThreads, 0, st>>>(A, lda, ns, np, p.rows, v, part);
  SR_LAUNCHED();
  chunk_reduce<<<(unsigned)std::min<long long>((np + 255) / 256, 8 * kNumSMs), 256, 0, st>>>(part, np,
                                                                                            (int)p.chunks,
                                                                                            scale, out);
  SR_LAUNCHED();
  return SR_OK;
}

namespace {
struct CfWs {
  double *ww, *sw;
  double2 *mean, *part, *esum;
};
CfWs carve_cf(Arena& a, long long ns, long long np) {
  ChunkPlan p = plan_chunks(ns, np);
  CfWs w;
  w.ww = a.take<double>(ns);
  w.sw = a.take<double>(ns);
  w.mean = a.take<double2>(np);
  w.esum = a.take<double2>(1);
  w.part = a.take<double2>((size_t)p.chunks * np);
  return w;
}
unsigned grid1d(long long n) { return (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 8 * kNumSMs)); }
}  // namespace

size_t center_force_ws(long long ns, long long np) {
  Arena a(nullptr, 0);
  carve_cf(a, ns, np);
  return a.used;
}

// Local weighted moments: wsum_O[c] = sum_k w_k O[k][c], wsum_E = sum_k w_k E_k  (w = 1/n_total if no weights)
sr_status column_moments_impl(long long ns, long long n_total, long long np, const double* O_d, long long ldo,
                              const double* weights, const double* e_loc, double* wsum_O, double* wsum_E,
                              void* ws, size_t ws_bytes, cudaStream_t st) {
  Arena a(ws, ws_bytes);
  CfWs w = carve_cf(a, ns, np);
  if (!a.ok()) {
    set_error("sr_column_moments: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  ChunkPlan p = plan_chunks(ns, np);
  weights_prep<<<grid1d(ns), 256, 0, st>>>(weights, ns, n_total, w.ww, w.sw);
  SR_LAUNCHED();
  wsum_energy<<<1, 1024, 0, st>>>(w.ww, reinterpret_cast<const double2*>(e_loc), ns,
                                  reinterpret_cast<double2*>(wsum_E));
  SR_LAUNCHED();
  dim3 g((unsigned)p.strips, (unsigned)p.chunks);
  colsum_partial<<<g, kColThreads, 0, st>>>(reinterpret_cast<const double2*>(O_d), ldo, ns, np, p.rows, w.ww,
                                            w.part);
  SR_LAUNCHED();
  chunk_reduce<<<grid1d(np), 256, 0, st>>>(w.part, np, (int)p.chunks, 1.0, reinterpret_cast<double2*>(wsum_O));
  SR_LAUNCHED();
  return SR_OK;
}

// Centre with a given global mean and energy; F_partial = sum_local conj(A) e.
sr_status center_force_global_impl(long long ns, long long n_total, long long np, double* O_d, long long ldo,
                                   const double* weights, const double* e_loc, const double* mean,
                                   const double* energy, double* e_tilde, double* F, void* ws, size_t ws_bytes,
                                   cudaStream_t st) {
  Arena a(ws, ws_bytes);
  CfWs w = carve_cf(a, ns, np);
  if (!a.ok()) {
    set_error("sr_center_force_global: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  ChunkPlan p = plan_chunks(ns, np);
  weights_prep<<<grid1d(ns), 256, 0, st>>>(weights, ns, n_total, w.ww, w.sw);
  SR_LAUNCHED();
  e_tilde_kernel<<<grid1d(ns), 256, 0, st>>>(w.sw, reinterpret_cast<const double2*>(e_loc),
                                             reinterpret_cast<const double2*>(energy), ns,
                                             reinterpret_cast<double2*>(e_tilde));
  SR_LAUNCHED();
  dim3 g((unsigned)p.strips, (unsigned)p.chunks);
  center_force_partial<<<g, kColThreads, 0, st>>>(reinterpret_cast<double2*>(O_d), ldo, ns, np, p.rows, w.sw,
                                                  reinterpret_cast<const double2*>(mean),
                                                  reinterpret_cast<const double2*>(e_tilde), w.part);
  SR_LAUNCHED();
  chunk_reduce<<<grid1d(np), 256, 0, st>>>(w.part, np, (int)p.chunks, 1.0, reinterpret_cast<double2*>(F));
  SR_LAUNCHED();
  return SR_OK;
}

// Single-process stage (3): moments, then centring + force with the local (= global) mean.
sr_status center_force_impl(long long ns, long long np, double* O_d, long long ldo, const double* weights,
                            const double* e_loc, double* energy, double* e_tilde, double* F, void* ws,
                            size_t ws_bytes, cudaStream_t st) {
  Arena a(ws, ws_bytes);
  CfWs w = carve_cf(a, ns, np);
  if (!a.ok()) {
    set_error("sr_center_force: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  double* e_out = energy ? energy : reinterpret_cast<double*>(w.esum);
  SR_TRY(column_moments_impl(ns, ns, np, O_d, ldo, weights, e_loc, reinterpret_cast<double*>(w.mean), e_out, ws,
                             ws_bytes, st));
  return center_force_global_impl(ns, ns, np, O_d, ldo, weights, e_loc, reinterpret_cast<const double*>(w.mean),
                                  e_out, e_tilde, F, ws, ws_bytes, st);
}

}  // namespace sr
