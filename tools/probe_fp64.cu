// Device probe: FP64 FMA throughput (DFMA chains, many independent accumulators),
// SMEM limits and SM count. Used to pin the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_peak(double *out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[blockIdx.x] = s;
}

template <int ILP>
__global__ void dfma_latency(double *out, int iters, double a, double b) {
  double acc = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) acc = fma(acc, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = acc; out[1] = (double)(t1 - t0) / iters; }
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("name=%s sms=%d cc=%d.%d smemPerBlockOptin=%zu smemPerSM=%zu regsPerSM=%d l2=%d clockKHz=%d memClockKHz=%d busWidth=%d\n",
         p.name, p.multiProcessorCount, p.major, p.minor, p.sharedMemPerBlockOptin,
         p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor, p.l2CacheSize, p.clockRate,
         p.memoryClockRate, p.memoryBusWidth);
  double *d; cudaMalloc(&d, 1 << 20);
  const int iters = 1 << 16;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    int blocks = p.multiProcessorCount * (2048 / threads) * 4;
    dfma_peak<8><<<blocks, threads>>>(d, 256, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_peak<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * blocks * threads;
    printf("dfma threads=%d blocks=%d : %.3f ms  %.2f TFLOP/s  (%.1f DFMA/clk/SM at %.0f MHz nominal)\n",
           threads, blocks, ms, flops / ms / 1e9, flops / 2 / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3), p.clockRate / 1e3);
  }
  // sustained: 30 back-to-back launches (about 3 s; nvidia-smi samples the clocks meanwhile)
  {
    const int threads = 1024, blocks = p.multiProcessorCount * 2 * 4;
    const double flops = 2.0 * 8 * (double)iters * blocks * threads;
    float best = 1e30f, all[30];
    for (int r = 0; r < 30; ++r) {
      cudaEventRecord(e0);
      dfma_peak<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      all[r] = ms;
      if (ms < best) best = ms;
    }
    for (int i = 0; i < 30; ++i)
      for (int j = i + 1; j < 30; ++j)
        if (all[j] < all[i]) { float t = all[i]; all[i] = all[j]; all[j] = t; }
    printf("{\"dfma_tflops_best\": %.3f, \"dfma_tflops_median\": %.3f, \"launches\": 30, "
           "\"blocks\": %d, \"threads\": %d, \"ilp\": 8}\n",
           flops / best / 1e9, flops / all[15] / 1e9, blocks, threads);
  }
  dfma_latency<1><<<1, 32>>>(d, 4096, 1.0000001, 1e-9);
  double h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("dfma dependent latency: %.2f clk\n", h[1]);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
