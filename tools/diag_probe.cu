// Phase timing of the Cholesky diagonal-tile kernel (chol_diag.cuh) with clock64 probes:
// factors a random 64x64 Hermitian positive definite tile (npad = 64) repeatedly and
// prints the mean cycles between probe points.  Build and run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/dp tools/diag_probe.cu && /tmp/dp
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ long long g_probe[64];
#define SR_DIAG_PROBE(i) \
  do {                   \
    if (threadIdx.x == 0) g_probe[i] = clock64(); \
  } while (0)
#include "../paper_2510_08430_b200/csrc/chol_diag.cuh"

namespace sr {
void set_error(const std::string&) {}
void count_launch(int) {}
}  // namespace sr

int main() {
  using namespace sr;
  const int n = 64;
  std::vector<double2> A(n * n);
  srand(1);
  std::vector<double2> M(n * n);
  for (auto& v : M) v = make_double2(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
  for (int i = 0; i < n; i++)
    for (int j = 0; j < n; j++) {
      double2 s = make_double2(i == j ? n : 0.0, 0.0);
      for (int k = 0; k < n; k++) {   // M M^H
        s.x += M[i * n + k].x * M[j * n + k].x + M[i * n + k].y * M[j * n + k].y;
        s.y += M[i * n + k].y * M[j * n + k].x - M[i * n + k].x * M[j * n + k].y;
      }
      A[i * n + j] = s;
    }
  double2 *dA, *dF, *dl, *dr;
  cudaMalloc(&dA, n * n * 16);
  cudaMalloc(&dF, n * n * 16);
  cudaMalloc(&dl, n * n * 16);
  cudaMalloc(&dr, n * 16);
  CholBlock B{};
  B.Fm = dF;
  B.linv = dl;
  B.rhs = dr;
  B.n = n;
  B.npad = n;
  B.P = 1;
  cudaFuncSetAttribute(cholk::chol_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cholk::kDiagSmem);
  const int reps = 50;
  std::vector<double> acc(17, 0.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float tot = 0.f;
  for (int r = 0; r < reps; r++) {
    cudaMemcpy(dF, A.data(), n * n * 16, cudaMemcpyHostToDevice);
    cudaMemset(dr, 0, n * 16);
    cudaEventRecord(e0);
    cholk::chol_diag<<<1, 256, cholk::kDiagSmem>>>(B, nullptr, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0) tot += ms;
    long long h[64];
    cudaMemcpyFromSymbol(h, g_probe, sizeof(h));
    if (r > 0) {
      const int ids[6] = {0, 1, 2, 14, 15, 16};
      for (int u = 1; u < 6; u++) acc[ids[u]] += (double)(h[ids[u]] - h[ids[u - 1]]);
    }
  }
  const int ids[5] = {1, 2, 14, 15, 16};
  const char* names[5] = {"load+rhs", "factor (all blocks)", "inv16", "inverse levels", "store+y"};
  double all = 0;
  for (int u = 0; u < 5; u++) {
    printf("%-20s %8.0f cycles\n", names[u], acc[ids[u]] / (reps - 1));
    all += acc[ids[u]] / (reps - 1);
  }
  printf("total %.0f cycles; event time %.2f us per launch\n", all, 1e3 * tot / (reps - 1));
  {   // per-round split of the factor phase (last repetition): factor+syrk | trsm
    long long h[64];
    cudaMemcpyFromSymbol(h, g_probe, sizeof(h));
    long long prev = h[1];
    for (int k = 0; k < 8; k++) {
      printf("round %d: factor/syrk %6lld  trsm %6lld\n", k, h[17 + 2 * k] - prev, h[18 + 2 * k] - h[17 + 2 * k]);
      prev = h[18 + 2 * k];
    }
  }
  {   // optional fine probes 40..50 (inside factor8 for o == 0, when compiled in)
    long long h[64];
    cudaMemcpyFromSymbol(h, g_probe, sizeof(h));
    for (int i = 41; i <= 50; i++)
      if (h[i] && h[i - 1]) printf("probe %d-%d: %lld\n", i - 1, i, h[i] - h[i - 1]);
  }
  // check: L L^H = A and X L = I (lower triangles)
  std::vector<double2> L(n * n), X(n * n);
  cudaMemcpy(L.data(), dF, n * n * 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(X.data(), dl, n * n * 16, cudaMemcpyDeviceToHost);
  double e1m = 0, e2m = 0, an = 0;
  for (int i = 0; i < n; i++)
    for (int j = 0; j <= i; j++) {
      double sx = 0, sy = 0, ix = 0, iy = 0;
      for (int k = 0; k <= j; k++) {   // (L L^H)_ij = sum_k L_ik conj(L_jk)
        sx += L[i * n + k].x * L[j * n + k].x + L[i * n + k].y * L[j * n + k].y;
        sy += L[i * n + k].y * L[j * n + k].x - L[i * n + k].x * L[j * n + k].y;
      }
      for (int k = j; k <= i; k++) {   // (X L)_ij
        ix += X[i * n + k].x * L[k * n + j].x - X[i * n + k].y * L[k * n + j].y;
        iy += X[i * n + k].x * L[k * n + j].y + X[i * n + k].y * L[k * n + j].x;
      }
      e1m = fmax(e1m, fabs(sx - A[i * n + j].x) + fabs(sy - A[i * n + j].y));
      e2m = fmax(e2m, fabs(ix - (i == j)) + fabs(iy));
      an = fmax(an, fabs(A[i * n + j].x));
    }
  printf("max |L L^H - A| / max|A| = %.2e, max |X L - I| = %.2e\n", e1m / an, e2m);
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
