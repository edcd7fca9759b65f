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

// z[r][j] = bias[j] + sum_i M[i][j] * hin[r][i] for the rows r < RB held in shared memory,
// M row-major [n_in][n_out] in global memory (L2-resident weights; coalesced across j).
// Thread layout: 256 threads = 64 output lanes x 4 row groups; row r = group + 4q.
// epi(r, j, z) is called for every r < RB, j < n_out.
template <int RB, typename Epi, int UNROLL = 4>
__device__ __forceinline__ void dense_rows(const double2* __restrict__ M, const double2* __restrict__ bias,
                                           int n_in, int n_out, const double2* hin, int ldin, Epi epi) {
  constexpr int RQ = RB / 4;
  const int tj = threadIdx.x & 63;
  const int tr = threadIdx.x >> 6;
  for (int j0 = 0; j0 < n_out; j0 += 64) {
    const int j = j0 + tj;
    const bool jv = j < n_out;
    double2 acc[RQ];
    double2 b0 = (jv && bias) ? bias[j] : make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < RQ; q++) acc[q] = b0;
    const double2* mcol = M + (jv ? j : 0);
#pragma unroll UNROLL
    for (int i = 0; i < n_in; i++) {
      double2 wv = jv ? __ldg(mcol + (long long)i * n_out) : make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < RQ; q++) cfma(acc[q], wv, hin[(tr + 4 * q) * ldin + i]);
    }
    if (jv) {
#pragma unroll
      for (int q = 0; q < RQ; q++) epi(tr + 4 * q, j, acc[q]);
    }
  }
}

}  // namespace sr
