// Dependent-chain latencies on sm_100a (cycles per op): DFMA, DMUL, double rsqrt(),
// MUFU.RSQ64H-based rsqrt, shared-memory round trip, __shfl_sync.  For chol_diag tuning.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lp tools/lat_probe.cu && /tmp/lp
#include <cstdio>
__global__ void k(double* out, long long* cyc, double seed) {
  __shared__ double sh[64];
  double x = seed + threadIdx.x * 1e-3, y = 1.0 + threadIdx.x * 1e-9;
  const int N = 256;
  long long t0, t1;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; i++) x = fma(x, y, 1e-7);
  t1 = clock64();
  cyc[0] = t1 - t0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; i++) x = x * y;
  t1 = clock64();
  cyc[1] = t1 - t0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; i++) x = rsqrt(x) + 0.5;
  t1 = clock64();
  cyc[2] = t1 - t0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; i++) {
    sh[threadIdx.x & 31] = x;
    __syncwarp();
    x = sh[(threadIdx.x + 1) & 31] + 1e-9;
    __syncwarp();
  }
  t1 = clock64();
  cyc[3] = t1 - t0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; i++) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
  t1 = clock64();
  cyc[4] = t1 - t0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; i++) {   // float rsqrt seed + 2 Newton steps in double
    double r = (double)rsqrtf((float)x);
    r = r * fma(-0.5 * x * r, r, 1.5);
    r = r * fma(-0.5 * x * r, r, 1.5);
    x = r + 0.5;
  }
  t1 = clock64();
  cyc[5] = t1 - t0;
  {   // throughput: 8 independent DFMA chains in one warp
    double c0 = x, c1 = x + 1, c2 = x + 2, c3 = x + 3, c4 = x + 4, c5 = x + 5, c6 = x + 6, c7 = x + 7;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) {
      c0 = fma(c0, y, 1e-7); c1 = fma(c1, y, 1e-7); c2 = fma(c2, y, 1e-7); c3 = fma(c3, y, 1e-7);
      c4 = fma(c4, y, 1e-7); c5 = fma(c5, y, 1e-7); c6 = fma(c6, y, 1e-7); c7 = fma(c7, y, 1e-7);
    }
    t1 = clock64();
    cyc[6] = t1 - t0;
    x = c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
  }
  out[threadIdx.x] = x;
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 1024);
  cudaMallocManaged(&c, 128);
  for (int r = 0; r < 3; r++) {
    k<<<1, 32>>>(o, c, 1.3);
    cudaDeviceSynchronize();
  }
  const char* nm[] = {"DFMA", "DMUL", "rsqrt(double)+add", "STS+syncwarp+LDS+add", "SHFL+add", "rsqrtf+2 Newton+add", "8 indep. DFMA (per 8)"};
  for (int i = 0; i < 7; i++) printf("%-24s %6.1f cycles/iter\n", nm[i], c[i] / 256.0);
  return 0;
}
