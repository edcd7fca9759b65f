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

// z[r][j] = sum_i hin[r][i] M[i][j] for the rows r < RB held in shared memory (ld ldin =
// act_ld(.)), written to zout[r][j] (shared memory, ld ldz), M row-major [n_in][n_out]
// complex in global memory (L2/L1 resident), on the FP64 tensor cores: each complex 8x8x4
// product is four real mma.sync.m8n8k4.f64 (SASS DMMA) into four independent accumulators,
// z = (rr - ii) + i (ri + ir).  Work units (MG 8-row tiles, one 8-column tile)
// go round robin over the warps; the B fragment M[k0 + lane%4][n0 + lane/4] is loaded once
// per k step for the MG row tiles of a unit (MG > 1 cuts the L2 weight traffic when the
// weights do not stay in L1), and units of one column tile sit on consecutive warps.  Ragged n_in / n_out are
// zero-padded in the fragments.  No barrier inside: the caller synchronises before
// reading zout (and the elementwise activation runs as a separate, balanced pass).
// BATCH: the B fragments of 8 k steps are loaded together ahead of their MMAs (8 L2 loads
// in flight; measured: local energy 0.722 -> 0.695 ms at configs[1], 35.5 -> 31.8 ms at
// configs[2]; the Jacobian kernels are faster without it, 0.258 vs 0.299 ms).
#ifndef SR_DENSE_BQ
#define SR_DENSE_BQ 4   // measured with the fused series epilogue: 4 / 8 / 16 -> configs[1] 0.575 / 0.61 / 0.65 ms, configs[3] 180 / 182 / 195 ms
#endif
// Epilogue applied to each output element in registers before it is stored (Identity: z).
struct ZIdentity {
  __device__ __forceinline__ double2 operator()(int /*j*/, double2 z) const { return z; }
};

template <int RB, int MG = 1, bool BATCH = false, class Epi = ZIdentity>
__device__ __forceinline__ void dense_z(const double2* __restrict__ M, int n_in, int n_out, const double2* hin,
                                        int ldin, double2* zout, int ldz, Epi epi = Epi()) {
  static_assert(RB % (8 * MG) == 0, "RB must be a multiple of 8 MG");
  constexpr int MU = RB / (8 * MG);          // row-tile groups; a unit is MG row tiles x 8 columns
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int gr = lane >> 2, gc = lane & 3;   // fragment row / column-in-group
  const int units = MU * ((n_out + 7) >> 3);
  const int k_full = n_in & ~3;
  for (int u = warp; u < units; u += nwarps) {
    const int mu = u % MU, nt = u / MU;
    const int n = nt * 8 + gr;                 // B-fragment column of this lane
    const bool n_ok = n < n_out;
    double rr[MG][2], ii[MG][2], ri[MG][2], ir[MG][2];
#pragma unroll
    for (int g = 0; g < MG; g++)
      rr[g][0] = rr[g][1] = ii[g][0] = ii[g][1] = ri[g][0] = ri[g][1] = ir[g][0] = ir[g][1] = 0.0;
    const double2* mcol = M + (n_ok ? n : 0);
    const double2* arow = hin + (mu * MG * 8 + gr) * ldin + gc;
    auto kstep = [&](int k0, bool tail) {
      const int k = k0 + gc;
      const bool k_ok = !tail || k < n_in;
      const double2 b = (n_ok && k_ok) ? __ldg(mcol + (long long)k * n_out) : make_double2(0.0, 0.0);
#pragma unroll
      for (int g = 0; g < MG; g++) {   // the B fragment serves MG row tiles
        const double2 a = k_ok ? arow[g * 8 * ldin + k0] : make_double2(0.0, 0.0);
        net_dmma(rr[g][0], rr[g][1], a.x, b.x);
        net_dmma(ii[g][0], ii[g][1], a.y, b.y);
        net_dmma(ri[g][0], ri[g][1], a.x, b.y);
        net_dmma(ir[g][0], ir[g][1], a.y, b.x);
      }
    };
    if (BATCH) {
    constexpr int BQ = SR_DENSE_BQ;
    const int k32 = k_full - k_full % (4 * BQ);
    for (int k0 = 0; k0 < k32; k0 += 4 * BQ) {
      double2 bb[BQ];
#pragma unroll
      for (int q = 0; q < BQ; q++) bb[q] = n_ok ? __ldg(mcol + (long long)(k0 + 4 * q + gc) * n_out) : make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < BQ; q++) {
#pragma unroll
        for (int g = 0; g < MG; g++) {
          const double2 a = arow[g * 8 * ldin + k0 + 4 * q];
          net_dmma(rr[g][0], rr[g][1], a.x, bb[q].x);
          net_dmma(ii[g][0], ii[g][1], a.y, bb[q].y);
          net_dmma(ri[g][0], ri[g][1], a.x, bb[q].y);
          net_dmma(ir[g][0], ir[g][1], a.y, bb[q].x);
        }
      }
    }
    for (int k0 = k32; k0 < k_full; k0 += 4) kstep(k0, false);
    } else {
#pragma unroll 8
    for (int k0 = 0; k0 < k_full; k0 += 4) kstep(k0, false);
    }
    if (k_full < n_in) kstep(k_full, true);
#pragma unroll
    for (int g = 0; g < MG; g++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int j = nt * 8 + 2 * gc + e;
        if (j < n_out)
          zout[((mu * MG + g) * 8 + gr) * ldz + j] = epi(j, make_double2(rr[g][e] - ii[g][e], ri[g][e] + ir[g][e]));
      }
  }
}

}  // namespace sr
