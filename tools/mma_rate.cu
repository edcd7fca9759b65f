// Microbenchmark: tcgen05.mma issue-to-completion throughput per SM for kind::i8 and
// kind::f16 at M=128 and several N, operands resident in shared memory (64-byte swizzle,
// K-major), one CTA per SM, 512 TMEM columns.  Prints MACs/clk/SM and chip TOPS.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, int sw) {
  // sw: 4 = SWIZZLE_64B (SBO 512), 2 = SWIZZLE_128B (SBO 1024)
  uint32_t sbo = sw == 4 ? 512 : 1024;
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(sbo >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)sw << 61);
}

template <int KIND>  // 0 = i8, 1 = f16 (bf16)
__global__ void __launch_bounds__(128, 1) bench(int N, int iters, int sw, int nacc, long long* out, int rnd = 0) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x)   // zeros, or random bytes (power runs)
    reinterpret_cast<uint32_t*>(sm)[i] = rnd ? (uint32_t)(i * 2654435761u) ^ (uint32_t)(blockIdx.x * 40503u) : 0u;
  uint32_t baddr = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(baddr));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  uint32_t tmem = slot;
  uint32_t idesc;
  if (KIND == 0) idesc = (2u << 4) | (1u << 7) | (1u << 10);
  else idesc = (1u << 4) | (1u << 7) | (1u << 10);   // f32 acc, bf16 A/B
  idesc |= ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sm);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint64_t a0 = sdesc(s0, sw), b0 = sdesc(s0 + 32768, sw);
    t0 = clock64();
    for (int it = 0; it < iters; it += 8) {
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint64_t a = a0 + (uint64_t)((u & 1) * 2), b = b0 + (uint64_t)((u & 1) * 2);
        const uint32_t dcol = tmem + (uint32_t)((u % 4) * (N < 128 ? N : 128) % 512);
        if (KIND == 0)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dcol), "l"(a), "l"(b), "r"(idesc), "r"(1));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dcol), "l"(a), "l"(b), "r"(idesc), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(baddr));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}\n" : "=r"(done) : "r"(baddr));
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// Power mode: mma_rate power N seconds -- int8 MMAs of M=128 x N x 32 with random operands
// launched back to back for the given time (sample nvidia-smi alongside); prints the
// sustained rate.
int power_mode(int N, double seconds) {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 200000;
  bench<0><<<148, 128, 65536>>>(N, iters, 4, 512 / N, d, 1);
  cudaDeviceSynchronize();
  float ms = 0.f;
  long long launches = 0;
  cudaEventRecord(a);
  while (ms < seconds * 1e3) {
    for (int r = 0; r < 10; r++) bench<0><<<148, 128, 65536>>>(N, iters, 4, 512 / N, d, 1);
    launches += 10;
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  const double ops = 2.0 * 128.0 * N * 32 * iters * 148 * launches;
  printf("i8 N=%d random operands: %.0f T(ops)/s sustained over %.1f s\n", N, ops / (ms * 1e-3) / 1e12, ms / 1e3);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 3 && argv[1][0] == 'p') return power_mode(atoi(argv[2]), atof(argv[3]));
  long long* d;
  cudaMalloc(&d, 148 * 8);
  long long h[148];
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 20000;
  for (int kind = 0; kind < 2; kind++)
    for (int sw : {4, 2})
      for (int N : {32, 64, 128, 256}) {
        int nacc = 512 / N;
        if (kind == 0) bench<0><<<148, 128, 65536>>>(N, iters, sw, nacc, d);
        else bench<1><<<148, 128, 65536>>>(N, iters, sw, nacc, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
        const int K = kind == 0 ? 32 : 16;
        double macs = 128.0 * N * K * iters;
        double per_clk = macs / mx;
        printf("%s sw=%s N=%3d: %.1f clk/MMA, %.0f MAC/clk/SM, %.0f T(ops)/s at %d MHz\n", kind ? "bf16" : "i8  ",
               sw == 4 ? "64 " : "128", N, (double)mx / iters, per_clk, per_clk * 2 * 148 * clk * 1e3 / 1e12, clk / 1000);
      }
  return 0;
}
