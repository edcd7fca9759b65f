// center.cu — stage (3) sr_center_force (+ its sample-sharded form) and the column
// reduction y = A^H v shared with the NTK solve.
//
// PAPER.md Eq. 2: Delta O_i = O_i - <O_i>; north_star (3): F = Obar^H (E_loc - <E_loc>)/N_s.
// With sample weights w_k (uniform 1/N_s, or given, e.g. Born weights over a sector):
//   E = sum_k w_k E_k,  e_k = sqrt(w_k)(E_k - E),  <O> = sum_k w_k O_k,
//   A_k = sqrt(w_k)(O_k - <O>)  (in place),       F = A^H e.
// Centring precision (reading R7): <O> and E are accumulated in double-double
// (TwoSum / fma-TwoProd) and subtracted as hi then lo, so O - <O> carries one rounding even
// when |<O>| / std(O) ~ 1e6 (nearly constant last-layer bias derivatives).
//
// O is row-major [N_s][ldo]; each pass streams it with one thread per column (a warp reads
// 512 contiguous bytes of a row); rows are split into chunks whose partial sums are reduced
// in a fixed chunk order (deterministic, no atomics).
//
// Moments row layout (complex): [ <O>_hi (n_p) | <O>_lo (n_p) | E_hi | E_lo ]; a sharded run
// all-gathers one row per rank and the centring kernels sum the rows in double-double.
#include "common.cuh"

namespace sr {
namespace {

constexpr int kColThreads = 256;

// ---- double-double helpers (Knuth TwoSum, fma TwoProd) ----
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
__device__ __forceinline__ void dd_add(double& hi, double& lo, double x, double xlo) {
  double s, e;
  two_sum(hi, x, s, e);
  e += lo + xlo;
  hi = s + e;
  lo = e - (hi - s);
}
__device__ __forceinline__ void dd_add_prod(double& hi, double& lo, double w, double x) {
  const double p = w * x;
  dd_add(hi, lo, p, fma(w, x, -p));
}
// (hi, lo) / d for an integer-valued d
__device__ __forceinline__ void dd_div(double& hi, double& lo, double d) {
  const double q1 = hi / d;
  const double r = fma(-q1, d, hi) + lo;
  const double q2 = r / d;
  hi = q1 + q2;
  lo = q2 - (hi - q1);
}

struct CDD {  // complex double-double
  double rh, rl, ih, il;
  __device__ void zero() { rh = rl = ih = il = 0.0; }
  __device__ void add(double2 x) {
    dd_add(rh, rl, x.x, 0.0);
    dd_add(ih, il, x.y, 0.0);
  }
  __device__ void add_w(double w, double2 x) {
    dd_add_prod(rh, rl, w, x.x);
    dd_add_prod(ih, il, w, x.y);
  }
  __device__ void add(const CDD& o) {
    dd_add(rh, rl, o.rh, o.rl);
    dd_add(ih, il, o.ih, o.il);
  }
  __device__ void add_parts(double2 hi, double2 lo) {
    dd_add(rh, rl, hi.x, lo.x);
    dd_add(ih, il, hi.y, lo.y);
  }
  __device__ void div(double d) {
    dd_div(rh, rl, d);
    dd_div(ih, il, d);
  }
  __device__ double2 hi() const { return make_double2(rh, ih); }
  __device__ double2 lo() const { return make_double2(rl, il); }
};

// ww[k] = w_k (given weights only), sw[k] = sqrt(w_k) (given, or 1/n_total)
__global__ void weights_prep(const double* __restrict__ weights, long long ns, long long n_total,
                             double* __restrict__ sw) {
  const double uni = 1.0 / (double)n_total;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < ns;
       k += (long long)gridDim.x * blockDim.x)
    sw[k] = sqrt(weights ? weights[k] : uni);
}

// Single CTA: moments row tail [E_hi, E_lo] = sum_k w_k E_k (uniform: (sum_k E_k) / n_total).
__global__ void __launch_bounds__(1024) wsum_energy(const double* __restrict__ weights,
                                                    const double2* __restrict__ e_loc, long long ns,
                                                    long long n_total, double2* __restrict__ out) {
  __shared__ CDD red[1024];
  CDD s;
  s.zero();
  for (long long k = threadIdx.x; k < ns; k += 1024) {
    if (weights)
      s.add_w(weights[k], e_loc[k]);
    else
      s.add(e_loc[k]);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x].add(red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    CDD t = red[0];
    if (!weights) t.div((double)n_total);
    out[0] = t.hi();
    out[1] = t.lo();
  }
}

// part[chunk][c] (hi, lo) = sum_{k in chunk} w_k O[k][c]  (uniform: plain sums)
__global__ void __launch_bounds__(kColThreads) colsum_partial(const double2* __restrict__ O, long long ldo,
                                                              long long ns, long long np, long long rows_per_chunk,
                                                              const double* __restrict__ weights,
                                                              double2* __restrict__ part_hi,
                                                              double2* __restrict__ part_lo) {
  const long long c = (long long)blockIdx.x * kColThreads + threadIdx.x;
  const long long k0 = (long long)blockIdx.y * rows_per_chunk;
  const long long k1 = min(ns, k0 + rows_per_chunk);
  if (c >= np) return;
  CDD s;
  s.zero();
  long long k = k0;
  for (; k + 3 < k1; k += 4) {  // four loads in flight
    const double2 a = O[k * ldo + c], b = O[(k + 1) * ldo + c], d = O[(k + 2) * ldo + c],
                  e = O[(k + 3) * ldo + c];
    if (weights) {
      s.add_w(weights[k], a);
      s.add_w(weights[k + 1], b);
      s.add_w(weights[k + 2], d);
      s.add_w(weights[k + 3], e);
    } else {
      s.add(a);
      s.add(b);
      s.add(d);
      s.add(e);
    }
  }
  for (; k < k1; k++) {
    if (weights)
      s.add_w(weights[k], O[k * ldo + c]);
    else
      s.add(O[k * ldo + c]);
  }
  part_hi[(long long)blockIdx.y * np + c] = s.hi();
  part_lo[(long long)blockIdx.y * np + c] = s.lo();
}

// moments[c] = hi, moments[np + c] = lo of (sum over chunks) / divisor
__global__ void chunk_reduce_dd(const double2* __restrict__ part_hi, const double2* __restrict__ part_lo,
                                long long np, int n_chunks, double divisor, double2* __restrict__ moments) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < np;
       c += (long long)gridDim.x * blockDim.x) {
    CDD s;
    s.zero();
    for (int q = 0; q < n_chunks; q++) s.add_parts(part_hi[(long long)q * np + c], part_lo[(long long)q * np + c]);
    if (divisor != 1.0) s.div(divisor);
    moments[c] = s.hi();
    moments[np + c] = s.lo();
  }
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

// e_tilde[k] = sqrt(w_k) ((E_k - E_hi) - E_lo) with E summed over the moment rows; energy = E rounded.
__global__ void e_tilde_kernel(const double* __restrict__ sw, const double2* __restrict__ e_loc,
                               const double2* __restrict__ moments, int n_parts, long long row_len,
                               long long np, long long ns, double2* __restrict__ e_tilde,
                               double2* __restrict__ energy) {
  CDD E;
  E.zero();
  for (int p = 0; p < n_parts; p++) E.add_parts(moments[p * row_len + 2 * np], moments[p * row_len + 2 * np + 1]);
  const double2 eh = E.hi(), el = E.lo();
  if (energy && blockIdx.x == 0 && threadIdx.x == 0) *energy = make_double2(eh.x + el.x, eh.y + el.y);
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < ns;
       k += (long long)gridDim.x * blockDim.x)
    e_tilde[k] = cscale(csub(csub(e_loc[k], eh), el), sw[k]);
}

// A[k][c] = sw_k ((O[k][c] - m_hi[c]) - m_lo[c]) in place; part[chunk][c] = sum_k conj(A[k][c]) e[k]
__global__ void __launch_bounds__(kColThreads) center_force_partial(double2* __restrict__ O, long long ldo,
                                                                    long long ns, long long np,
                                                                    long long rows_per_chunk,
                                                                    const double* __restrict__ sw,
                                                                    const double2* __restrict__ moments,
                                                                    int n_parts, long long row_len,
                                                                    const double2* __restrict__ e,
                                                                    double2* __restrict__ part) {
  const long long c = (long long)blockIdx.x * kColThreads + threadIdx.x;
  const long long k0 = (long long)blockIdx.y * rows_per_chunk;
  const long long k1 = min(ns, k0 + rows_per_chunk);
  if (c >= np) return;
  CDD m;
  m.zero();
  for (int p = 0; p < n_parts; p++) m.add_parts(moments[p * row_len + c], moments[p * row_len + np + c]);
  const double2 mh = m.hi(), ml = m.lo();
  double2 s = make_double2(0.0, 0.0);
  for (long long k = k0; k < k1; k++) {
    const double2 a = cscale(csub(csub(O[k * ldo + c], mh), ml), sw[k]);
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
  long long want = (4LL * kNumSMs + p.strips - 1) / p.strips;     // >= 4 CTAs per SM
  long long max_chunks = std::max<long long>(1, (ns + 31) / 32);  // at least 32 rows per chunk
  p.chunks = std::max<long long>(1, std::min(want, max_chunks));
  p.rows = std::max<long long>(1, (ns + p.chunks - 1) / p.chunks);
  p.chunks = std::max<long long>(1, (ns + p.rows - 1) / p.rows);
  return p;
}

unsigned grid1d(long long n) {
  return (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 8 * kNumSMs));
}

struct CfWs {
  double* sw;
  double2 *part_hi, *part_lo, *moments;
};
CfWs carve_cf(Arena& a, long long ns, long long np) {
  ChunkPlan p = plan_chunks(ns, np);
  CfWs w;
  w.sw = a.take<double>(ns);
  w.part_hi = a.take<double2>((size_t)p.chunks * np);
  w.part_lo = a.take<double2>((size_t)p.chunks * np);
  w.moments = a.take<double2>(2 * np + 2);
  return w;
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
  chunk_reduce<<<grid1d(np), 256, 0, st>>>(part, np, (int)p.chunks, scale, out);
  SR_LAUNCHED();
  return SR_OK;
}

size_t center_force_ws(long long ns, long long np) {
  Arena a(nullptr, 0);
  carve_cf(a, ns, np);
  return a.used;
}

// One moments row (see file header) from the local rows.
sr_status column_moments_impl(long long ns, long long n_total, long long np, const double* O_d, long long ldo,
                              const double* weights, const double* e_loc, double* moments_d, void* ws,
                              size_t ws_bytes, cudaStream_t st) {
  Arena a(ws, ws_bytes);
  CfWs w = carve_cf(a, ns, np);
  if (!a.ok()) {
    set_error("sr_column_moments: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  ChunkPlan p = plan_chunks(ns, np);
  double2* moments = reinterpret_cast<double2*>(moments_d);
  wsum_energy<<<1, 1024, 0, st>>>(weights, reinterpret_cast<const double2*>(e_loc), ns, n_total, moments + 2 * np);
  SR_LAUNCHED();
  dim3 g((unsigned)p.strips, (unsigned)p.chunks);
  colsum_partial<<<g, kColThreads, 0, st>>>(reinterpret_cast<const double2*>(O_d), ldo, ns, np, p.rows, weights,
                                            w.part_hi, w.part_lo);
  SR_LAUNCHED();
  chunk_reduce_dd<<<grid1d(np), 256, 0, st>>>(w.part_hi, w.part_lo, np, (int)p.chunks,
                                              weights ? 1.0 : (double)n_total, moments);
  SR_LAUNCHED();
  return SR_OK;
}

// Centre with the summed moment rows; F_partial = sum_local conj(A) e.
sr_status center_force_global_impl(long long ns, long long n_total, long long np, double* O_d, long long ldo,
                                   const double* weights, const double* e_loc, int n_parts, const double* moments_d,
                                   double* energy, double* e_tilde, double* F, void* ws, size_t ws_bytes,
                                   cudaStream_t st) {
  Arena a(ws, ws_bytes);
  CfWs w = carve_cf(a, ns, np);
  if (!a.ok()) {
    set_error("sr_center_force_global: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  ChunkPlan p = plan_chunks(ns, np);
  const double2* moments = reinterpret_cast<const double2*>(moments_d);
  const long long row = 2 * np + 2;
  weights_prep<<<grid1d(ns), 256, 0, st>>>(weights, ns, n_total, w.sw);
  SR_LAUNCHED();
  e_tilde_kernel<<<grid1d(ns), 256, 0, st>>>(w.sw, reinterpret_cast<const double2*>(e_loc), moments, n_parts, row,
                                             np, ns, reinterpret_cast<double2*>(e_tilde),
                                             reinterpret_cast<double2*>(energy));
  SR_LAUNCHED();
  dim3 g((unsigned)p.strips, (unsigned)p.chunks);
  center_force_partial<<<g, kColThreads, 0, st>>>(reinterpret_cast<double2*>(O_d), ldo, ns, np, p.rows, w.sw,
                                                  moments, n_parts, row, reinterpret_cast<const double2*>(e_tilde),
                                                  w.part_hi);
  SR_LAUNCHED();
  chunk_reduce<<<grid1d(np), 256, 0, st>>>(w.part_hi, np, (int)p.chunks, 1.0, reinterpret_cast<double2*>(F));
  SR_LAUNCHED();
  return SR_OK;
}

// Single-process stage (3): moments of all rows, then centring + force.
sr_status center_force_impl(long long ns, long long np, double* O_d, long long ldo, const double* weights,
                            const double* e_loc, double* energy, double* e_tilde, double* F, void* ws,
                            size_t ws_bytes, cudaStream_t st) {
  Arena a(ws, ws_bytes);
  CfWs w = carve_cf(a, ns, np);
  if (!a.ok()) {
    set_error("sr_center_force: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  double* mom = reinterpret_cast<double*>(w.moments);
  SR_TRY(column_moments_impl(ns, ns, np, O_d, ldo, weights, e_loc, mom, ws, ws_bytes, st));
  return center_force_global_impl(ns, ns, np, O_d, ldo, weights, e_loc, 1, mom, energy, e_tilde, F, ws, ws_bytes,
                                  st);
}

}  // namespace sr
