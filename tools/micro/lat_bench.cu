// Latency microbenchmarks (cycles): dependent DFMA / DADD chains, LDS round trip,
// cp.async issue + commit + wait_group.   nvcc -arch=sm_100a -O3 lat_bench.cu
#include <cstdio>
__global__ void dfma_chain(long long *out, double *sink, double a, double b, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, a, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (x == -1) sink[0] = x;
}
__global__ void dadd_chain(long long *out, double *sink, double a, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = x + a;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (x == -1) sink[0] = x;
}
__global__ void ffma_chain(long long *out, float *sink, float a, float b, int n) {
  float x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fmaf(x, a, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (x == -1) sink[0] = x;
}
__global__ void lds_chain(long long *out, double *sink, int n) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) p = idx[p];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (p == -1) sink[0] = p;
}
__global__ void cpasync_bench(long long *out, const double *src, int n) {
  __shared__ __align__(16) double ring[8][256 * 2];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    unsigned dst = (unsigned)__cvta_generic_to_shared(&ring[i & 7][threadIdx.x * 2]);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + ((i * 512 + threadIdx.x * 2) & ((1 << 20) - 1))) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 5;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
int main() {
  long long *d, h;
  double *sink, *src;
  float *fs;
  cudaMalloc(&d, 8); cudaMalloc(&sink, 8); cudaMalloc(&fs, 8);
  cudaMalloc(&src, 8 << 20); cudaMemset(src, 0, 8 << 20);
  const int n = 1000;
  for (int nt : {32, 256}) {
    dfma_chain<<<1, nt>>>(d, sink, 0.999, 0.001, n); dfma_chain<<<1, nt>>>(d, sink, 0.999, 0.001, n);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("threads %d DFMA dep latency %.2f cyc\n", nt, (double)h / (16.0 * n));
    dadd_chain<<<1, nt>>>(d, sink, 0.001, n); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("threads %d DADD dep latency %.2f cyc\n", nt, (double)h / (16.0 * n));
    ffma_chain<<<1, nt>>>(d, fs, 0.999f, 0.001f, n); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("threads %d FFMA dep latency %.2f cyc\n", nt, (double)h / (16.0 * n));
    lds_chain<<<1, nt>>>(d, sink, n); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("threads %d LDS dep latency %.2f cyc\n", nt, (double)h / (16.0 * n));
    cpasync_bench<<<1, nt>>>(d, src, n); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("threads %d cp.async16+commit+wait5 %.2f cyc/iter\n", nt, (double)h / n);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
