// Microbenchmark: cost per iteration of the coarse-solve step skeleton (CTA barrier,
// shared-memory publish/read, cluster launch).  nvcc -arch=sm_100a -O3 bar_bench.cu
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void kern(long long *out, int iters, double *sink) {
  __shared__ double buf[2][1024];
  const int t = threadIdx.x;
  buf[0][t] = t; buf[1][t] = t;
  __syncthreads();
  double x = t;
  long long t0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for (int i = 0; i < iters; ++i) {
    if (MODE >= 1) {
      double *cur = buf[i & 1], *nxt = buf[(i + 1) & 1];
      double y = cur[(t + 1) % blockDim.x] + cur[(t + 31) % blockDim.x];
      x = 0.5 * y + 0.25 * x;
      nxt[t] = x;
    }
    if (MODE == 2) __syncwarp();
    else __syncthreads();
  }
  long long t1 = clock64();
  unsigned long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (t == 0) { out[blockIdx.x] = t1 - t0; out[8 + blockIdx.x] = (long long)(g1 - g0); }
  if (x == -1.0) sink[t] = x;
}
template <int MODE>
__global__ void __cluster_dims__(8, 1, 1) kern_cl(long long *out, int iters, double *sink) {
  unsigned long long g0, g1;
  __shared__ double buf[2][1024];
  const int t = threadIdx.x;
  buf[0][t] = t; buf[1][t] = t;
  __syncthreads();
  double x = t;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double *cur = buf[i & 1], *nxt = buf[(i + 1) & 1];
    double y = cur[(t + 1) % blockDim.x] + cur[(t + 31) % blockDim.x];
    x = 0.5 * y + 0.25 * x;
    nxt[t] = x;
    __syncthreads();
  }
  long long t1 = clock64();
  if (t == 0) out[blockIdx.x] = t1 - t0;
  if (x == -1.0) sink[t] = x;
}

int main() {
  long long *d, h[16];
  double *sink;
  cudaMalloc(&d, 128);
  cudaMalloc(&sink, 8192);
  int iters = 4096;
  for (int rep = 0; rep < 3; ++rep) {
    iters = rep == 0 ? 4096 : (rep == 1 ? 400000 : 4000000);
    kern<1><<<8, 288>>>(d, iters, sink); cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
    printf("iters %d: %.1f cyc/iter %.1f ns/iter (%.0f MHz)\n", iters, (double)h[0] / iters, (double)h[8] / iters, (double)h[0] / h[8] * 1e3);
  }
  iters = 4096;
  for (int nt : {64, 128, 288, 416}) {
    kern<0><<<8, nt>>>(d, iters, sink); cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
    kern<0><<<8, nt>>>(d, iters, sink); cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
    printf("threads %4d  bar only        %.1f cyc/iter\n", nt, (double)h[0] / iters);
    kern<1><<<8, nt>>>(d, iters, sink); cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
    printf("threads %4d  lds+sts+bar     %.1f cyc/iter  %.1f ns/iter  (%.0f MHz)\n", nt, (double)h[0] / iters, (double)h[8] / iters, (double)h[0] / h[8] * 1e3);
    kern<2><<<8, nt>>>(d, iters, sink); cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
    printf("threads %4d  lds+sts+syncwarp %.1f cyc/iter\n", nt, (double)h[0] / iters);
    kern_cl<1><<<8, nt>>>(d, iters, sink); cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
    printf("threads %4d  cluster lds+sts+bar %.1f cyc/iter\n", nt, (double)h[0] / iters);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
