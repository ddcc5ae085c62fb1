// levels.cu — FULL-state primitives on a coarse level l >= 1 (mgrit_relax / mgrit_residual
// / mgrit_coarse_solve with level >= 1; include/mgrit.h).
//
// Level l carries Phi_l = Psi_l (a stencil) and a right-hand side g_l (DESIGN.md
// R12: U[0] = g[0], U[n] = Psi U[n-1] + g[n]).  A primitive is a set of independent rows
//   y(n) = Psi U[n-1] + g[n],   n = n0 + j*nstride, j = 0..nrows-1,
// evaluated in one launch (F-relaxation is m-1 such launches, one per F-point position,
// because F-point jm+i depends on jm+i-1).  Not the production path: mgrit_solve keeps the
// levels on chip (coarse.cu); these kernels are plain, coalesced and L2/HBM-bound.
#include "kernels.h"

namespace mg {

__global__ void __launch_bounds__(256) psi_rowstep_kernel(const __grid_constant__ RowStepArgs a) {
  __shared__ double red[8];
  const int nx = a.nx;
  const long long n = a.n0 + (long long)blockIdx.y * a.nstride;
  const int chunk = (nx + a.bpr - 1) / a.bpr;
  const int i0 = blockIdx.x * chunk, i1 = min(nx, i0 + chunk);
  const double *src = a.U + (n - 1) * (long long)nx;
  const double *cur = a.U + n * (long long)nx;
  const double *g = a.g ? a.g + n * (long long)nx : nullptr;
  double s2 = 0.0;
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    double y = 0.0;
    int q = i + a.op.o0;
    if (a.trunc) {   // Toeplitz, no wrap: taps outside [0, nx) read zero
      for (int k = 0; k < a.op.nu; ++k, ++q)
        if ((unsigned)q < (unsigned)nx) y = fma(a.op.psi[k], src[q], y);
    } else {
      q %= nx;
      if (q < 0) q += nx;
      for (int k = 0; k < a.op.nu; ++k) {   // d = o0 + k ascending
        y = fma(a.op.psi[k], src[q], y);
        q = (q + 1 == nx) ? 0 : q + 1;
      }
    }
    if (g) y += g[i];
    if (a.mode == 0) {
      a.dst[n * (long long)nx + i] = y;
    } else {
      const double r = y - cur[i];
      s2 = fma(r, r, s2);
      if (a.rstore) a.rstore[(a.roff + blockIdx.y) * (long long)nx + i] = r;
    }
  }
  if (a.mode == 1 && a.partials) {
    s2 = block_sum<256>(s2, red);
    if (threadIdx.x == 0) a.partials[(long long)blockIdx.y * a.bpr + blockIdx.x] = s2;
  }
}

cudaError_t launch_psi_rowstep(const RowStepArgs &a, cudaStream_t s) {
  if (a.nrows <= 0) return cudaSuccess;
  if (a.nrows > 65535 * 1024 || a.bpr < 1 || a.bpr > 64) return cudaErrorInvalidValue;
  // gridDim.y <= 65535: split long row sets
  RowStepArgs b = a;
  for (int j0 = 0; j0 < a.nrows; j0 += 65535) {
    b.nrows = min(65535, a.nrows - j0);
    b.n0 = a.n0 + (long long)j0 * a.nstride;
    b.roff = a.roff + j0;
    b.partials = a.partials ? a.partials + (long long)j0 * a.bpr : nullptr;
    psi_rowstep_kernel<<<dim3(a.bpr, b.nrows), 256, 0, s>>>(b);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace mg
