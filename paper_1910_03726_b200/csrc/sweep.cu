// sweep.cu — fine-level relaxation sweep.
//
// One CTA = one (item, tile): an interval's spatial window held in registers
// (P points per thread) across all m Runge-Kutta steps and stages; HBM is
// touched only at the start (C-row u_j and the comparison row u_{j+1}) and the
// end (v_{j+1}, r_{j+2}) through coalesced shared-memory staging.
//
// Fused FCF sweep of interval j:
//   w = Phi^m u_j              (F- then C-relaxation)
//   v_{j+1} = w                (stored)
//   delta = w - u_{j+1}        (C-point residual of the current iterate)
//   r_{j+2} = Phi^m delta      (C-point residual after FCF = coarse RHS, by linearity)
// The same kernel also serves the FULL-state primitives (F/C relaxation, the
// all-row residual) and the final F-point materialisation via RowMaps.
#include "kernels.h"

namespace mg {

template <class SC, int NT, int P>
__global__ void __launch_bounds__(NT) rk_sweep_kernel(const __grid_constant__ SweepArgs a) {
  constexpr int SP = Pad<P>::SP;
  constexpr int W = NT * P;
  constexpr int NW = NT / 32;
  extern __shared__ double smem[];
  double *sA = smem;
  double *sB = sA + NT * SP;
  double *edge = sB + NT * SP;
  double *red = edge + 2 * NW * (SC::NL + SC::NR) + 2;

  const int item = blockIdx.x / a.ntiles;
  const int tile = blockIdx.x - item * a.ntiles;
  const int nx = a.nx;
  const int abeg = (int)(((long long)tile * nx) / a.ntiles);
  const int aend = (int)(((long long)(tile + 1) * nx) / a.ntiles);
  const int T = aend - abeg;
  int start = abeg - a.HL;
  if (start < 0) start += nx;
  const int tid = threadIdx.x;
  int phase = 0;

  auto rowp = [&](const RowMap &r, long long j) -> const double * {
    return r.base + (r.off + j * r.stride) * (long long)nx;
  };
  auto load_window = [&](const double *row, double *s) {
    for (int q = tid; q < W; q += NT) {
      int g = start + q;
      if (g >= nx) g -= nx;
      s[pidx<P>(q)] = __ldg(row + g);
    }
  };
  // Store the T owned outputs [abeg, aend) of a register vector (coalesced via sA).
  auto store_slice = [&](double *row, const double(&v)[P]) {
    __syncthreads();
#pragma unroll
    for (int p = 0; p < P; ++p) sA[tid * SP + p] = v[p];
    __syncthreads();
    for (int q = tid; q < T; q += NT) row[abeg + q] = sA[pidx<P>(a.HL + q)];
  };

  if (a.in.base) load_window(rowp(a.in, item), sA);
  if (a.cmp.base) load_window(rowp(a.cmp, item), sB);
  __syncthreads();
  double x[P];
#pragma unroll
  for (int p = 0; p < P; ++p) x[p] = a.in.base ? sA[tid * SP + p] : 0.0;

  // ---- phase 1: nsteps1 steps of Phi --------------------------------------
  if (a.each_first == 0 && a.each_last >= 0)
    store_slice(const_cast<double *>(a.each.base) +
                    (a.each.off + item * a.each.stride) * (long long)nx, x);
#pragma unroll 1
  for (int i = 1; i <= a.nsteps1; ++i) {
    erk_step<SC, P, NT>(x, a.co, edge, phase);
    if (i >= a.each_first && i <= a.each_last)
      store_slice(const_cast<double *>(a.each.base) +
                      (a.each.off + item * a.each.stride + i * a.each_step) * (long long)nx,
                  x);
  }
  if (a.endw.base) store_slice(const_cast<double *>(rowp(a.endw, item)), x);

  if (a.cmp.base) {
    double d[P];
#pragma unroll
    for (int p = 0; p < P; ++p) d[p] = x[p] - sB[tid * SP + p];
    if (a.partials) {
      double s = 0.0;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int l = tid * P + p;
        if (l >= a.HL && l < a.HL + T) s = fma(d[p], d[p], s);
      }
      s = block_sum<NT>(s, red);
      if (tid == 0) a.partials[blockIdx.x] = s;
    }
    if (a.dstore.base) {
      const int jj = item + a.d_phase;
      if (jj % a.d_every == 0)
        store_slice(const_cast<double *>(rowp(a.dstore, jj / a.d_every)), d);
    }
    // ---- phase 2: r = Phi^m delta ------------------------------------------
    if (a.nsteps2 > 0 && item < a.p2_items) {
#pragma unroll
      for (int p = 0; p < P; ++p) x[p] = d[p];
#pragma unroll 1
      for (int i = 1; i <= a.nsteps2; ++i) erk_step<SC, P, NT>(x, a.co, edge, phase);
      store_slice(const_cast<double *>(rowp(a.r2, item)), x);
    }
  }
}

template <class SC> struct SchemeId;

int rk_scheme_reach_left(int scheme) {
  const int t[] = {ERK1U1::NL, ERK2U2::NL, ERK3U3::NL, ERK4U4::NL, ERK5U5::NL};
  return (scheme >= 0 && scheme < 5) ? t[scheme] : -1;
}
int rk_scheme_reach_right(int scheme) {
  const int t[] = {ERK1U1::NR, ERK2U2::NR, ERK3U3::NR, ERK4U4::NR, ERK5U5::NR};
  return (scheme >= 0 && scheme < 5) ? t[scheme] : -1;
}
int rk_scheme_stages(int scheme) {
  const int t[] = {ERK1U1::S, ERK2U2::S, ERK3U3::S, ERK4U4::S, ERK5U5::S};
  return (scheme >= 0 && scheme < 5) ? t[scheme] : -1;
}

template <class SC, int NT, int P>
static cudaError_t launch_one(const SweepArgs &a, cudaStream_t s) {
  constexpr int SP = Pad<P>::SP;
  const size_t smem =
      sizeof(double) * (2 * NT * SP + 2 * (NT / 32) * (SC::NL + SC::NR) + 2 + NT / 32 + 2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(rk_sweep_kernel<SC, NT, P>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const long long grid = (long long)a.nitems * a.ntiles;
  if (grid <= 0) return cudaSuccess;
  rk_sweep_kernel<SC, NT, P><<<(unsigned)grid, NT, smem, s>>>(a);
  return cudaGetLastError();
}

#define MG_CFGS(X)                                                                          \
  X(32, 2) X(32, 4) X(32, 8) X(64, 8) X(128, 8) X(256, 8) X(512, 8) X(128, 11) X(256, 11)

template <class SC>
static cudaError_t dispatch_cfg(SweepCfg c, const SweepArgs &a, cudaStream_t s) {
#define MG_CASE(NT_, P_) \
  if (c.nt_threads == NT_ && c.p == P_) return launch_one<SC, NT_, P_>(a, s);
  MG_CFGS(MG_CASE)
#undef MG_CASE
  return cudaErrorInvalidConfiguration;
}

bool rk_sweep_supported(int scheme, SweepCfg c) {
  if (scheme < 0 || scheme > 4) return false;
#define MG_CASE(NT_, P_) \
  if (c.nt_threads == NT_ && c.p == P_) return true;
  MG_CFGS(MG_CASE)
#undef MG_CASE
  return false;
}

cudaError_t launch_rk_sweep(int scheme, SweepCfg cfg, const SweepArgs &a, cudaStream_t s) {
  switch (scheme) {
    case 0: return dispatch_cfg<ERK1U1>(cfg, a, s);
    case 1: return dispatch_cfg<ERK2U2>(cfg, a, s);
    case 2: return dispatch_cfg<ERK3U3>(cfg, a, s);
    case 3: return dispatch_cfg<ERK4U4>(cfg, a, s);
    case 4: return dispatch_cfg<ERK5U5>(cfg, a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mg
