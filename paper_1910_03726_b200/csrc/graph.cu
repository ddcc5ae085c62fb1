// graph.cu — device-side loop control of mgrit_solve's CUDA-graph mode (P:218 stopping
// rule on the device).
//
// The iteration body (coarse-grid correction, fused FCF sweep, deterministic norm
// reduction) is captured once into a graph; a conditional WHILE node repeats it.  After
// each iteration `decide` turns the reduced sum of squares into ||r^(k)|| =
// sqrt(dx dt sum r^2), appends it to the device history, and sets the loop's conditional
// handle(s) to 0 once ||r^(k)|| < tol, k == max_iter or the norm is not finite (R2, R15),
// so the host synchronises once per solve instead of once per iteration.
#include "kernels.h"

namespace mg {

__global__ void loop_init_kernel(LoopState *s, double tol, double dxdt, int max_iter, int k0) {
  s->tol = tol;
  s->dxdt = dxdt;
  s->max_iter = max_iter;
  s->k = k0;
  s->stop = 0;
  s->nonfinite = 0;
}

__global__ void loop_decide_kernel(LoopState *s, const double *norm2, double *hist,
                                   cudaGraphConditionalHandle h0, cudaGraphConditionalHandle h1,
                                   int set_h1) {
  const double rk = sqrt(s->dxdt * norm2[0]);
  const int k = s->k + 1;
  s->k = k;
  hist[k] = rk;
  const int nonfinite = !isfinite(rk);
  const int stop = nonfinite || rk < s->tol || k >= s->max_iter;
  s->stop = stop;
  s->nonfinite |= nonfinite;
  cudaGraphSetConditional(h0, stop ? 0u : 1u);
  if (set_h1) cudaGraphSetConditional(h1, stop ? 0u : 1u);
}

cudaError_t launch_loop_init(LoopState *s, double tol, double dxdt, int max_iter, int k0,
                             cudaStream_t st) {
  loop_init_kernel<<<1, 1, 0, st>>>(s, tol, dxdt, max_iter, k0);
  return cudaGetLastError();
}

cudaError_t launch_loop_decide(LoopState *s, const double *norm2, double *hist,
                               cudaGraphConditionalHandle h0, cudaGraphConditionalHandle h1,
                               int set_h1, cudaStream_t st) {
  loop_decide_kernel<<<1, 1, 0, st>>>(s, norm2, hist, h0, h1, set_h1);
  return cudaGetLastError();
}

}  // namespace mg
