// mlp.cu — stage (1) sr_jacobian and stage (2) sr_local_energy.
//
// The dense layers of both stages run on the FP64 tensor cores (dense_z, net.cuh).
// Stage 1 (§2 Eq. 2, O_i(x) = d_theta_i log psi(x)):
//   jac_forward   rows = samples; z_l = W_l h_l + b_l, stores h_{l+1} = lncosh(z_l) and
//                 tanh(z_l) per layer to [N_s][w] scratch, ln psi = sum_j h_L[j]
//   jac_backward  delta_{L-1} = tanh(z_{L-1}); delta_{l-1} = tanh(z_{l-1}) * (W_l^T delta_l)
//   jac_outer     O[k][off_l + j*fin + i] = delta_l[k][j] h_l[k][i], O[k][.. + j] = delta_l[k][j]
//                 — the HBM-bound stream: every O element written once, 16-byte coalesced.
// Stage 2 (Eq. 1): one row per connected configuration x' of sample k;
//   the first layer is updated from the sample's z_0 by the two flipped spins
//   (z_0(x') = z_0(x) - 2 s_i W_0[:,i] - 2 s_j W_0[:,j]), the remaining layers run
//   densely on the row tile in shared memory, and each row contributes
//   2 J_b exp(ln psi(x') - ln psi(x)); rows of one sample are reduced in bond order.
#include <cstdlib>

#include "net.cuh"

namespace sr {

sr_status make_net(int n_layers, const int32_t* widths, NetDesc* net) {
  SR_CHECK_ARG(widths != nullptr, "widths is null");
  SR_CHECK_ARG(n_layers >= 1 && n_layers <= kMaxLayers, "n_layers must be in [1, 16]");
  net->L = n_layers;
  net->wmax = 0;
  long long p = 0, t = 0, a = 0;
  for (int l = 0; l <= n_layers; l++) {
    SR_CHECK_ARG(widths[l] >= 1 && widths[l] <= kMaxWidth, "every width must be in [1, 256]");
    net->w[l] = widths[l];
    if (widths[l] > net->wmax) net->wmax = widths[l];
  }
  for (int l = 0; l < n_layers; l++) {
    net->woff[l] = p;
    net->boff[l] = p + (long long)widths[l + 1] * widths[l];
    p += (long long)widths[l + 1] * (widths[l] + 1);
    net->toff[l] = t;
    t += (long long)widths[l + 1] * widths[l];
    net->aoff[l] = a;
    a += widths[l + 1];
  }
  net->n_p = p;
  net->n_wt = t;
  net->n_act = a;
  return SR_OK;
}

namespace {

constexpr int kThreads = 256;

// WT_l[i][j] = W_l[j][i] for all layers (coalesced weight reads in the forward pass).
__global__ void transpose_weights(NetDesc net, const double2* __restrict__ theta, double2* __restrict__ wt) {
  for (int l = 0; l < net.L; l++) {
    const int fin = net.w[l], fout = net.w[l + 1];
    const long long n = (long long)fin * fout;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
      const int i = (int)(e / fout), j = (int)(e % fout);
      wt[net.toff[l] + e] = theta[net.woff[l] + (long long)j * fin + i];
    }
  }
}

template <int RB>
__global__ void __launch_bounds__(kThreads) jac_forward(NetDesc net, const double2* __restrict__ theta,
                                                        const double2* __restrict__ wt,
                                                        const int8_t* __restrict__ spins, long long ns,
                                                        double2* __restrict__ hs, double2* __restrict__ ts,
                                                        double2* __restrict__ log_psi) {
  extern __shared__ double2 smem[];
  const int ld = act_ld(net.wmax);
  double2* cur = smem;
  double2* nxt = smem + RB * ld;
  const long long row0 = (long long)blockIdx.x * RB;
  const int n0 = net.w[0];
  for (int e = threadIdx.x; e < RB * n0; e += kThreads) {
    const int r = e / n0, i = e % n0;
    const long long k = row0 + r;
    cur[r * ld + i] = make_double2(k < ns ? (double)spins[k * n0 + i] : 0.0, 0.0);
  }
  __syncthreads();
  for (int l = 0; l < net.L; l++) {
    const int fout = net.w[l + 1];
    double2* hl = hs + net.aoff[l] * ns;
    double2* tl = ts + net.aoff[l] * ns;
    dense_z<RB>(wt + net.toff[l], net.w[l], fout, cur, ld, nxt, ld);
    __syncthreads();
    const double2* bl = theta + net.boff[l];
    for (int e = threadIdx.x; e < RB * fout; e += kThreads) {
      const int r = e / fout, j = e - r * fout;
      double2 h, th;
      lncosh_tanh(cadd(bl[j], nxt[r * ld + j]), h, th);
      nxt[r * ld + j] = h;
      const long long k = row0 + r;
      if (k < ns) {
        hl[k * fout + j] = h;
        tl[k * fout + j] = th;
      }
    }
    __syncthreads();
    double2* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  // ln psi = sum_j h_L[j]: one warp per row, fixed lane order then a fixed shuffle tree.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fl = net.w[net.L];
  for (int r = warp; r < RB; r += kThreads / 32) {
    double2 s = make_double2(0.0, 0.0);
    for (int j = lane; j < fl; j += 32) s = cadd(s, cur[r * ld + j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    }
    const long long k = row0 + r;
    if (lane == 0 && k < ns) log_psi[k] = s;
  }
}

// delta_{l-1} = tanh(z_{l-1}) * (W_l^T delta_l): M = W_l as [w[l+1]][w[l]] row-major.
// ts holds tanh(z_l) on entry and delta_l on exit (delta_{L-1} = tanh(z_{L-1}) as is).
template <int RB>
__global__ void __launch_bounds__(kThreads) jac_backward(NetDesc net, const double2* __restrict__ theta,
                                                         double2* __restrict__ ts, long long ns) {
  extern __shared__ double2 smem[];
  const int ld = act_ld(net.wmax);
  double2* cur = smem;
  double2* nxt = smem + RB * ld;
  const long long row0 = (long long)blockIdx.x * RB;
  {
    const int fl = net.w[net.L];
    const double2* tL = ts + net.aoff[net.L - 1] * ns;
    for (int e = threadIdx.x; e < RB * fl; e += kThreads) {
      const int r = e / fl, j = e % fl;
      const long long k = row0 + r;
      cur[r * ld + j] = k < ns ? tL[k * fl + j] : make_double2(0.0, 0.0);
    }
  }
  __syncthreads();
  for (int l = net.L - 1; l >= 1; l--) {
    const int nout = net.w[l];
    double2* tprev = ts + net.aoff[l - 1] * ns;
    dense_z<RB>(theta + net.woff[l], net.w[l + 1], nout, cur, ld, nxt, ld);
    __syncthreads();
    for (int e = threadIdx.x; e < RB * nout; e += kThreads) {
      const int r = e / nout, i = e - r * nout;
      const long long k = row0 + r;
      double2 d = make_double2(0.0, 0.0);
      if (k < ns) {
        d = cmul(tprev[k * nout + i], nxt[r * ld + i]);
        tprev[k * nout + i] = d;
      }
      nxt[r * ld + i] = d;
    }
    __syncthreads();
    double2* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
}

// One CTA per (sample k, layer l): writes the n_l = fout*(fin+1) row segment of O.
__global__ void __launch_bounds__(kThreads) jac_outer(NetDesc net, const int8_t* __restrict__ spins,
                                                      const double2* __restrict__ hs,
                                                      const double2* __restrict__ ds, long long ns,
                                                      double2* __restrict__ O, long long ldo) {
  __shared__ double2 hin[kMaxWidth];
  __shared__ double2 del[kMaxWidth];
  const long long k = blockIdx.x;
  const int l = blockIdx.y;
  const int fin = net.w[l], fout = net.w[l + 1];
  for (int i = threadIdx.x; i < fin; i += kThreads)
    hin[i] = l == 0 ? make_double2((double)spins[k * fin + i], 0.0) : hs[net.aoff[l - 1] * ns + k * fin + i];
  for (int j = threadIdx.x; j < fout; j += kThreads) del[j] = ds[net.aoff[l] * ns + k * fout + j];
  __syncthreads();
  double2* row = O + k * ldo + net.woff[l];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < fout; j += kThreads / 32) {
    const double2 d = del[j];
    double2* seg = row + (long long)j * fin;
    for (int i = lane; i < fin; i += 32) seg[i] = cmul(d, hin[i]);
  }
  double2* brow = row + (long long)fout * fin;
  for (int j = threadIdx.x; j < fout; j += kThreads) brow[j] = del[j];
}

// ---------------------------------------------------------------- stage 2 ----
// Z0[k][j] = b_0[j] + sum_i W_0[j][i] s_k[i]; diag[k] = sum_b J_b s_i s_j; cnt[k] = #flippable bonds.
__global__ void energy_prepare(NetDesc net, const double2* __restrict__ theta, const double2* __restrict__ wt,
                               const int8_t* __restrict__ spins, long long ns, long long nb,
                               const int2* __restrict__ bij, const double* __restrict__ bj,
                               double2* __restrict__ z0, double* __restrict__ diag, int* __restrict__ cnt) {
  const int n0 = net.w[0], w1 = net.w[1];
  const long long total = ns * w1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long k = e / w1;
    const int j = (int)(e % w1);
    double2 acc = theta[net.boff[0] + j];
    const int8_t* s = spins + k * n0;
    for (int i = 0; i < n0; i++) {
      const double2 w = wt[net.toff[0] + (long long)i * w1 + j];
      const double si = (double)s[i];
      acc.x = fma(w.x, si, acc.x);
      acc.y = fma(w.y, si, acc.y);
    }
    z0[e] = acc;
  }
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < ns;
       k += (long long)gridDim.x * blockDim.x) {
    const int8_t* s = spins + k * n0;
    double d = 0.0;
    int c = 0;
    for (long long b = 0; b < nb; b++) {
      const int2 p = bij[b];
      const int si = s[p.x], sj = s[p.y];
      d = fma(bj[b], (double)(si * sj), d);
      c += si != sj;
    }
    diag[k] = d;
    cnt[k] = c;
  }
}

// Exclusive scan of cnt[0..ns) into off[0..ns] (off[ns] = total rows).  One CTA.
__global__ void __launch_bounds__(1024) scan_counts(const int* __restrict__ cnt, long long ns,
                                                    long long* __restrict__ off) {
  __shared__ long long warp_sums[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (long long base = 0; base < ns; base += 1024) {
    const long long k = base + threadIdx.x;
    long long v = k < ns ? cnt[k] : 0;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      long long s = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      warp_sums[lane] = s;
    }
    __syncthreads();
    const long long incl = x + (warp > 0 ? warp_sums[warp - 1] : 0) + carry;
    if (k < ns) off[k] = incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[ns] = carry;
}

// rows of sample k (in bond order): row_sb[r] = (k, b).
__global__ void energy_rows(const int8_t* __restrict__ spins, long long ns, int n0, long long nb,
                            const int2* __restrict__ bij, const long long* __restrict__ off,
                            longlong2* __restrict__ row_sb) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < ns;
       k += (long long)gridDim.x * blockDim.x) {
    const int8_t* s = spins + k * n0;
    long long r = off[k];
    for (long long b = 0; b < nb; b++) {
      const int2 p = bij[b];
      if (s[p.x] != s[p.y]) row_sb[r++] = make_longlong2(k, b);
    }
  }
}

#ifndef SR_ENERGY_MG
#define SR_ENERGY_MG 1
#endif
// row tiles per weight fragment in energy_eval (dense_z); measured 1 / 2 / 4: configs[1]
// 0.721 / 0.751 / 0.747 ms, configs[2] 35.4 / 33.2 / 33.2 ms
constexpr int kEnergyMG = SR_ENERGY_MG;

// h = lncosh(b_j + z), applied by dense_z to its accumulators in registers (the activation is
// fused into the DMMA pass: no separate shared-memory pass and barrier per layer).
struct LncoshBias {
  const double2* __restrict__ b;
  __device__ __forceinline__ double2 operator()(int j, double2 z) const { return lncosh(cadd(b[j], z)); }
};

#ifndef SR_ENERGY_FUSED
#define SR_ENERGY_FUSED 1
#endif

// Persistent over tiles of RB connected rows: ln psi(x') then 2 J exp(ln psi(x') - ln psi(x)).
#ifndef SR_ENERGY_MINB
#define SR_ENERGY_MINB 3   // 85 registers: 3 CTAs per SM (measured: configs[3] 182 vs 189 ms at 1, 193 at 4; configs[1] 0.61 vs 0.64 ms)
#endif
template <int RB>
__global__ void __launch_bounds__(kThreads, SR_ENERGY_MINB) energy_eval(NetDesc net, const double2* __restrict__ theta,
                                                        const double2* __restrict__ wt,
                                                        const int8_t* __restrict__ spins,
                                                        const int2* __restrict__ bij,
                                                        const double* __restrict__ bj,
                                                        const double2* __restrict__ z0,
                                                        const double2* __restrict__ log_psi,
                                                        const long long* __restrict__ off, long long ns,
                                                        const longlong2* __restrict__ row_sb,
                                                        double2* __restrict__ contrib) {
  extern __shared__ double2 smem[];
  __shared__ longlong2 tile_sb[RB];
  const int ld = act_ld(net.wmax);
  const long long R = off[ns];
  const int n0 = net.w[0], w1 = net.w[1];
  const double2* wt0 = wt + net.toff[0];
  for (long long row0 = (long long)blockIdx.x * RB; row0 < R; row0 += (long long)gridDim.x * RB) {
    double2* cur = smem;
    double2* nxt = smem + RB * ld;
      if (threadIdx.x < RB) {
      const long long r = row0 + threadIdx.x;
      tile_sb[threadIdx.x] = r < R ? row_sb[r] : make_longlong2(-1, 0);
    }
    __syncthreads();
    // first layer from z_0 of the sample and the two flipped spins
    for (int e = threadIdx.x; e < RB * w1; e += kThreads) {
      const int r = e / w1, j = e % w1;
      const longlong2 sb = tile_sb[r];
      double2 h = make_double2(0.0, 0.0);
      if (sb.x >= 0) {
        const int2 p = bij[sb.y];
        const double si = (double)spins[sb.x * n0 + p.x], sj = (double)spins[sb.x * n0 + p.y];
        double2 z = z0[sb.x * w1 + j];
        const double2 wi = wt0[(long long)p.x * w1 + j], wj = wt0[(long long)p.y * w1 + j];
        z.x = fma(-2.0 * si, wi.x, z.x);
        z.y = fma(-2.0 * si, wi.y, z.y);
        z.x = fma(-2.0 * sj, wj.x, z.x);
        z.y = fma(-2.0 * sj, wj.y, z.y);
        h = lncosh(z);
      }
      cur[r * ld + j] = h;
    }
    __syncthreads();
    for (int l = 1; l < net.L; l++) {
      const int fout = net.w[l + 1];
      const double2* bl = theta + net.boff[l];
      if (SR_ENERGY_FUSED) {
        dense_z<RB, (RB / 8 < kEnergyMG ? RB / 8 : kEnergyMG), true>(wt + net.toff[l], net.w[l], fout, cur, ld, nxt,
                                                                      ld, LncoshBias{bl});
        __syncthreads();
      } else {
        dense_z<RB, (RB / 8 < kEnergyMG ? RB / 8 : kEnergyMG), true>(wt + net.toff[l], net.w[l], fout, cur, ld, nxt,
                                                                      ld);
        __syncthreads();
        for (int e = threadIdx.x; e < RB * fout; e += kThreads) {
          const int r = e / fout, j = e - r * fout;
          nxt[r * ld + j] = lncosh(cadd(bl[j], nxt[r * ld + j]));
        }
        __syncthreads();
      }
      double2* tmp = cur;
      cur = nxt;
      nxt = tmp;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fl = net.w[net.L];
    for (int r = warp; r < RB; r += kThreads / 32) {
      double2 s = make_double2(0.0, 0.0);
      for (int j = lane; j < fl; j += 32) s = cadd(s, cur[r * ld + j]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
      }
      const longlong2 sb = tile_sb[r];
      if (lane == 0 && sb.x >= 0) {
        const double2 ratio = cexp(csub(s, log_psi[sb.x]));
        contrib[row0 + r] = cscale(ratio, 2.0 * bj[sb.y]);
      }
    }
    __syncthreads();
  }
}

__global__ void energy_reduce(const double* __restrict__ diag, const long long* __restrict__ off,
                              const double2* __restrict__ contrib, long long ns, double2* __restrict__ e_loc) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < ns;
       k += (long long)gridDim.x * blockDim.x) {
    double2 e = make_double2(diag[k], 0.0);
    for (long long r = off[k]; r < off[k + 1]; r++) e = cadd(e, contrib[r]);
    e_loc[k] = e;
  }
}

size_t tile_smem(const NetDesc& net, int rb) {
  return (size_t)2 * rb * act_ld(net.wmax) * sizeof(double2);
}

template <typename K>
sr_status set_smem(K kernel, size_t bytes) {
  SR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return SR_OK;
}

struct JacWs {
  double2 *wt, *hs, *ts;
};
JacWs carve_jac(Arena& a, const NetDesc& net, long long ns) {
  JacWs w;
  w.wt = a.take<double2>(net.n_wt);
  w.hs = a.take<double2>(net.n_act * ns);
  w.ts = a.take<double2>(net.n_act * ns);
  return w;
}

struct EnWs {
  double2 *wt, *z0, *contrib;
  double* diag;
  int* cnt;
  long long* off;
  longlong2* rows;
  int2* bij;
};
EnWs carve_en(Arena& a, const NetDesc& net, long long ns, long long nb) {
  EnWs w;
  w.wt = a.take<double2>(net.n_wt);
  w.z0 = a.take<double2>((size_t)ns * net.w[1]);
  w.diag = a.take<double>(ns);
  w.cnt = a.take<int>(ns);
  w.off = a.take<long long>(ns + 1);
  w.rows = a.take<longlong2>((size_t)ns * nb);
  w.contrib = a.take<double2>((size_t)ns * nb);
  return w;
}

}  // namespace

template <int RB>
sr_status launch_jac(const NetDesc& net, const double2* theta, const JacWs& w, const int8_t* spins, long long ns,
                     double* log_psi, unsigned grid, size_t sm, cudaStream_t st) {
  SR_TRY(set_smem(jac_forward<RB>, sm));
  SR_TRY(set_smem(jac_backward<RB>, sm));
  jac_forward<RB><<<grid, kThreads, sm, st>>>(net, theta, w.wt, spins, ns, w.hs, w.ts,
                                              reinterpret_cast<double2*>(log_psi));
  SR_LAUNCHED();
  if (net.L > 1) {
    jac_backward<RB><<<grid, kThreads, sm, st>>>(net, theta, w.ts, ns);
    SR_LAUNCHED();
  }
  return SR_OK;
}

sr_status jacobian_impl(const NetDesc& net, const double* theta_d, const int8_t* spins, long long ns,
                        double* log_psi, double* O, long long ldo, void* ws, size_t ws_bytes,
                        cudaStream_t st) {
  Arena a(ws, ws_bytes);
  JacWs w = carve_jac(a, net, ns);
  if (!a.ok()) {
    set_error("sr_jacobian: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  if (ns == 0) return SR_OK;
  const double2* theta = reinterpret_cast<const double2*>(theta_d);
  transpose_weights<<<64, kThreads, 0, st>>>(net, theta, w.wt);
  SR_LAUNCHED();
  // 8-row tiles (measured best with the DMMA dense layers: configs[1] 0.259 ms vs 0.279 / 0.336
  // with 16 / 32 rows; configs[2] 3.70 ms vs 5.35 with 32 rows)
  constexpr int rb = 8;
  SR_TRY(launch_jac<rb>(net, theta, w, spins, ns, log_psi, (unsigned)((ns + rb - 1) / rb), tile_smem(net, rb), st));
  dim3 og((unsigned)ns, (unsigned)net.L);
  jac_outer<<<og, kThreads, 0, st>>>(net, spins, w.hs, w.ts, ns, reinterpret_cast<double2*>(O), ldo);
  SR_LAUNCHED();
  return SR_OK;
}

size_t jacobian_ws(const NetDesc& net, long long ns) {
  Arena a(nullptr, 0);
  carve_jac(a, net, ns);
  return a.used;
}

size_t local_energy_ws(const NetDesc& net, long long ns, long long nb) {
  Arena a(nullptr, 0);
  carve_en(a, net, ns, nb);
  a.take<int2>(nb);
  return a.used;
}

sr_status local_energy_impl(const NetDesc& net, const double* theta_d, long long nb, const int32_t* bonds_ij,
                            const double* bond_j, const int8_t* spins, long long ns, const double* log_psi,
                            double* e_loc, void* ws, size_t ws_bytes, cudaStream_t st) {
  Arena a(ws, ws_bytes);
  EnWs w = carve_en(a, net, ns, nb);
  if (!a.ok()) {
    set_error("sr_local_energy: workspace too small");
    return SR_ERR_WORKSPACE;
  }
  if (ns == 0) return SR_OK;
  const double2* theta = reinterpret_cast<const double2*>(theta_d);
  const int2* bij = reinterpret_cast<const int2*>(bonds_ij);
  transpose_weights<<<64, kThreads, 0, st>>>(net, theta, w.wt);
  SR_LAUNCHED();
  energy_prepare<<<4 * kNumSMs, kThreads, 0, st>>>(net, theta, w.wt, spins, ns, nb, bij, bond_j, w.z0, w.diag,
                                                   w.cnt);
  SR_LAUNCHED();
  scan_counts<<<1, 1024, 0, st>>>(w.cnt, ns, w.off);
  SR_LAUNCHED();
  energy_rows<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(spins, ns, net.w[0], nb, bij, w.off, w.rows);
  SR_LAUNCHED();
  // 16-row tiles: more CTAs per SM hide the L2 latency of the weight stream (measured
  // faster than 32 rows: configs[3] 229 vs 359 ms; 8 rows within noise at configs[3],
  // slower at configs[1]/[2]); SR_ENERGY_RB overrides for tuning.  Forcing 5-6 CTAs per SM
  // (SR_ENERGY_MINB) costs registers and spills: slower (272 / 355 ms at configs[3]).
  int rb = 16;
  if (const char* e = getenv("SR_ENERGY_RB")) rb = atoi(e) == 32 ? 32 : atoi(e) == 24 ? 24 : atoi(e) == 8 ? 8 : 16;
  const size_t sm = tile_smem(net, rb);
  const long long max_tiles = (ns * nb + rb - 1) / rb;
  const double2* lp = reinterpret_cast<const double2*>(log_psi);
  // persistent: as many CTAs as fit on the SMs at once
  auto grid_of = [&](auto kernel) -> unsigned {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, sm) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    if (const char* e = getenv("SR_ENERGY_CTAS_PER_SM")) per_sm = std::max(1, std::min(per_sm, atoi(e)));
    return (unsigned)std::max<long long>(1, std::min<long long>(max_tiles, (long long)per_sm * kNumSMs));
  };
  if (rb == 32) {
    SR_TRY(set_smem(energy_eval<32>, sm));
    const unsigned grid = grid_of(energy_eval<32>);
    energy_eval<32><<<grid, kThreads, sm, st>>>(net, theta, w.wt, spins, bij, bond_j, w.z0, lp, w.off, ns, w.rows,
                                                w.contrib);
  } else if (rb == 24) {
    SR_TRY(set_smem(energy_eval<24>, sm));
    const unsigned grid = grid_of(energy_eval<24>);
    energy_eval<24><<<grid, kThreads, sm, st>>>(net, theta, w.wt, spins, bij, bond_j, w.z0, lp, w.off, ns, w.rows,
                                                w.contrib);
  } else if (rb == 16) {
    SR_TRY(set_smem(energy_eval<16>, sm));
    const unsigned grid = grid_of(energy_eval<16>);
    energy_eval<16><<<grid, kThreads, sm, st>>>(net, theta, w.wt, spins, bij, bond_j, w.z0, lp, w.off, ns, w.rows,
                                                w.contrib);
  } else {
    SR_TRY(set_smem(energy_eval<8>, sm));
    const unsigned grid = grid_of(energy_eval<8>);
    energy_eval<8><<<grid, kThreads, sm, st>>>(net, theta, w.wt, spins, bij, bond_j, w.z0, lp, w.off, ns, w.rows,
                                               w.contrib);
  }
  SR_LAUNCHED();
  energy_reduce<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(w.diag, w.off, w.contrib, ns,
                                                               reinterpret_cast<double2*>(e_loc));
  SR_LAUNCHED();
  return SR_OK;
}

}  // namespace sr
