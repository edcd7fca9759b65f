// Microbenchmark: FP64 DMMA (mma.sync m8n8k4 -> SASS DMMA.8x8x4) and DFMA
// throughput on the B200, to fix the FP64 roofline denominator used in DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>
template<int CH>
__global__ void dmma_loop(double* out, int iters){
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[CH][2];
#pragma unroll
  for (int j = 0; j < CH; j++) { c[j][0] = 0; c[j][1] = 0; }
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < CH; j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < CH; j++) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template<int CH>
__global__ void dfma_loop(double* out, int iters){
  double a = threadIdx.x * 1e-3, b = 1.0 - blockIdx.x * 1e-9;
  double c[CH];
#pragma unroll
  for (int j = 0; j < CH; j++) c[j] = j;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < CH; j++) c[j] = fma(c[j], b, a);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < CH; j++) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main(){
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, p.multiProcessorCount);
  double* out; cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int bpm : {4, 8}) for (int thr : {128, 256}) {
    int grid = p.multiProcessorCount * bpm;
    dmma_loop<8><<<grid, thr>>>(out, 100); cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; r++) {
      cudaEventRecord(e0); dmma_loop<8><<<grid, thr>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 256 * 8 * (double)iters * grid * (thr / 32);
    printf(", \"dmma_tflops_b%d_t%d\": %.2f", bpm, thr, flops / best * 1e-9);
  }
  for (int bpm : {4, 8}) for (int thr : {256}) {
    int grid = p.multiProcessorCount * bpm;
    dfma_loop<8><<<grid, thr>>>(out, 100); cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; r++) {
      cudaEventRecord(e0); dfma_loop<8><<<grid, thr>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * (double)iters * grid * thr;
    printf(", \"dfma_tflops_b%d_t%d\": %.2f", bpm, thr, flops / best * 1e-9);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf(", \"clock_khz\": %d}\n", clk);
  return 0;
}
