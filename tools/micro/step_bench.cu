// Microbenchmark: one step of the sequential coarse solve x_i = Psi x_{i-1} + g_i on one
// CTA (structure-of-arrays state, whole window in registers, NS partial sums, g from a
// shared ring, publish, CTA barrier).  Cycles per step vs threads / P / taps.
// nvcc -arch=sm_100a -O3 -o step_bench step_bench.cu
#include <cstdio>

struct Coef { double c[32]; };
#include <cooperative_groups.h>
template <int P, int NU, int NS, int MODE>
__device__ __forceinline__ void step_body(long long *out, int iters, double *sink, const Coef &cf);
template <int P, int NU, int NS, int MODE>
__global__ void __launch_bounds__(512) step(long long *out, int iters, double *sink, const __grid_constant__ Coef cf) {
  step_body<P, NU, NS, MODE>(out, iters, sink, cf);
}
template <int P, int NU, int NS, int MODE>
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(512) step_cl(long long *out, int iters, double *sink, const __grid_constant__ Coef cf) {
  step_body<P, NU, NS, MODE>(out, iters, sink, cf);
}
template <int P, int NU, int NS, int MODE>
__device__ __forceinline__ void step_body(long long *out, int iters, double *sink, const Coef &cf) {
  constexpr int COLS = 320;
  __shared__ double S[2][P * COLS];
  __shared__ double G[4][512];
  const int t = threadIdx.x;
  for (int q = t; q < 2 * P * COLS; q += blockDim.x) (&S[0][0])[q] = 1e-3 * q;
  for (int q = t; q < 4 * 512; q += blockDim.x) (&G[0][0])[q] = 1e-4 * q;
  __syncthreads();
  double x[P];
#pragma unroll
  for (int p = 0; p < P; ++p) x[p] = 0;
  const int col = t + 8;  // window starts 8 columns left (o0 = -8*P-ish)
  if ((MODE & 4) && t >= (int)blockDim.x - 32) return;  // idle producer warp
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const double *cur = S[i & 1];
    double *nxt = S[(i + 1) & 1];
    double w[P + NU - 1];
#pragma unroll
    for (int r = 0; r < P + NU - 1; ++r) w[r] = cur[(r % P) * COLS + col - 8 + r / P];
    double acc[NS][P];
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int p = 0; p < P; ++p) acc[s][p] = 0.0;
#pragma unroll
    for (int q = 0; q < NU; ++q)
#pragma unroll
      for (int p = 0; p < P; ++p) acc[q % NS][p] = fma(cf.c[q], w[p + q], acc[q % NS][p]);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      double y = acc[0][p];
#pragma unroll
      for (int s = 1; s < NS; ++s) y += acc[s][p];
      x[p] = (MODE & 1) ? y : y + G[i & 3][(t * P + p) & 511];
    }
#pragma unroll
    for (int p = 0; p < P; ++p) nxt[p * COLS + col] = x[p];
    if ((MODE & 8) && (i & 3) == 3) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (MODE & 2) __syncwarp();
    else if (MODE & 4) asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x - 32) : "memory");
    else __syncthreads();
  }
  long long t1 = clock64();
  if (t == 0) out[blockIdx.x] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int p = 0; p < P; ++p) s += x[p];
  if (s == -1.2345) sink[t] = s;
}

template <int P, int NU, int NS, int MODE>
void run_cl(int nt, long long *d, double *sink) {
  Coef coef;
  for (int q = 0; q < 32; ++q) coef.c[q] = 0.01 * q;
  long long h[16];
  const int iters = 20000;
  cudaFuncSetAttribute(step_cl<P, NU, NS, MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  step_cl<P, NU, NS, MODE><<<16, nt>>>(d, iters, sink, coef);
  step_cl<P, NU, NS, MODE><<<16, nt>>>(d, iters, sink, coef);
  cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  printf("CLUSTER16 threads %3d P %d NU %2d NS %d mode %d (4: named bar + idle warp): %6.1f cyc/step  %s\n", nt, P, NU,
         NS, MODE, (double)h[0] / iters, cudaGetErrorString(cudaGetLastError()));
}
template <int P, int NU, int NS, int MODE>
void run(int nt, long long *d, double *sink, const double *) {
  Coef coef;
  for (int q = 0; q < 32; ++q) coef.c[q] = 0.01 * q;
  long long h[16];
  const int iters = 20000;
  step<P, NU, NS, MODE><<<16, nt>>>(d, iters, sink, coef);
  step<P, NU, NS, MODE><<<16, nt>>>(d, iters, sink, coef);
  cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  printf("threads %3d P %d NU %2d NS %d mode %d (1:no g, 2:syncwarp): %6.1f cyc/step\n", nt, P, NU,
         NS, MODE, (double)h[0] / iters);
}

int main() {
  long long *d;
  double *sink, *coef;
  cudaMalloc(&d, 128);
  cudaMalloc(&sink, 1 << 16);
  cudaMalloc(&coef, 64 * 8);
  cudaMemset(coef, 0, 64 * 8);
  run<2, 10, 2, 0>(64, d, sink, coef);
  run<2, 10, 2, 8>(64, d, sink, coef);
  run<4, 32, 2, 0>(128, d, sink, coef);
  run<4, 32, 2, 8>(128, d, sink, coef);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
