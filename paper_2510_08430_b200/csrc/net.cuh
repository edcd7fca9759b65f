// net.cuh — network descriptor and the row-batched dense complex layer used by the
// Jacobian (stage 1) and local-energy (stage 2) kernels.
#pragma once
#include "common.cuh"

namespace sr {

constexpr int kMaxLayers = 16;
constexpr int kMaxWidth = 256;

// Layer l (0-based) maps h_l (width w[l]) to h_{l+1} (width w[l+1]);
// W_l is [w[l+1]][w[l]] row-major at theta + woff[l], b_l at theta + boff[l].
struct NetDesc {
  int L;
  int wmax;
  int w[kMaxLayers + 1];
  long long woff[kMaxLayers];  // complex offset of W_l in theta (== O column offset of block l)
  long long boff[kMaxLayers];  // complex offset of b_l
  long long toff[kMaxLayers];  // complex offset of W_l^T in the transposed-weight scratch
  long long aoff[kMaxLayers];  // complex offset of layer-l activations in [N_s][w[l+1]] scratch
  long long n_p;
  long long n_act;             // sum_l w[l+1]
  long long n_wt;              // sum_l w[l]*w[l+1]
};

sr_status make_net(int n_layers, const int32_t* widths, NetDesc* net);

// Leading dimension (complex elements) of the [RB][ld] activation tiles in shared memory:
// ld = 4 (mod 8), so the 8 rows x 4 columns of a DMMA A fragment (16-byte loads) hit
// disjoint bank groups in each 8-lane phase.
__host__ __device__ constexpr int act_ld(int wmax) { return (wmax + 7) / 8 * 8 + 4; }

__device__ __forceinline__ void net_dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// z[r][j] = bias[j] + sum_i hin[r][i] M[i][j] for the rows r < RB held in shared memory
// (ld ldin = act_ld(.)), M row-major [n_in][n_out] complex in global memory (L2/L1
// resident), on the FP64 tensor cores: each complex 8x8x4 product is four real
// mma.sync.m8n8k4.f64 (SASS DMMA) into three accumulators (Re*Re, Im*Im, cross terms), so
// Re z = rr - ii.  Warp g owns the 8-column n-tiles g, g+8, ... and all RB/8 row tiles of
// each; the B fragment (M[k0 + lane%4][n0 + lane/4]) is loaded once per k step and used
// for every row tile.  Ragged n_in / n_out are zero-padded in the fragments.
// epi(r, j, z) is called for every r < RB, j < n_out.
template <int RB, typename Epi>
__device__ __forceinline__ void dense_rows(const double2* __restrict__ M, const double2* __restrict__ bias,
                                           int n_in, int n_out, const double2* hin, int ldin, Epi epi) {
  static_assert(RB % 8 == 0, "RB must be a multiple of 8");
  constexpr int MT = RB / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int gr = lane >> 2, gc = lane & 3;   // fragment row / column-in-group
  const int nt_count = (n_out + 7) >> 3;
  const int k_full = n_in & ~3;
  for (int nt = warp; nt < nt_count; nt += nwarps) {
    const int n = nt * 8 + gr;                 // B-fragment column of this lane
    const bool n_ok = n < n_out;
    double rr[MT][2], ii[MT][2], ri[MT][2];
#pragma unroll
    for (int m = 0; m < MT; m++) rr[m][0] = rr[m][1] = ii[m][0] = ii[m][1] = ri[m][0] = ri[m][1] = 0.0;
    const double2* mcol = M + (n_ok ? n : 0);
    const double2* arow = hin + gr * ldin + gc;
    auto kstep = [&](int k0, bool tail) {
      const int k = k0 + gc;
      const bool k_ok = !tail || k < n_in;
      const double2 b = (n_ok && k_ok) ? __ldg(mcol + (long long)k * n_out) : make_double2(0.0, 0.0);
#pragma unroll
      for (int m = 0; m < MT; m++) {
        const double2 a = k_ok ? arow[m * 8 * ldin + k0] : make_double2(0.0, 0.0);
        net_dmma(rr[m][0], rr[m][1], a.x, b.x);
        net_dmma(ii[m][0], ii[m][1], a.y, b.y);
        net_dmma(ri[m][0], ri[m][1], a.x, b.y);
        net_dmma(ri[m][0], ri[m][1], a.y, b.x);
      }
    };
#pragma unroll 4
    for (int k0 = 0; k0 < k_full; k0 += 4) kstep(k0, false);
    if (k_full < n_in) kstep(k_full, true);
#pragma unroll
    for (int e = 0; e < 2; e++) {
      const int j = nt * 8 + 2 * gc + e;
      if (j < n_out) {
        const double2 b0 = bias ? bias[j] : make_double2(0.0, 0.0);
#pragma unroll
        for (int m = 0; m < MT; m++)
          epi(m * 8 + gr, j, make_double2(b0.x + (rr[m][e] - ii[m][e]), b0.y + ri[m][e]));
      }
    }
  }
}

}  // namespace sr
