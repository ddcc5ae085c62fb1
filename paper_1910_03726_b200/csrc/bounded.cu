// bounded.cu — inflow/outflow boundaries (PAPER.md 4.5; SURVEY 8(f) NEXT-4;
// DESIGN.md R20): the fine propagator with the inverse-Lax-Wendroff inflow closure and the
// polynomial outflow extrapolation, and the periodic problem's Psi truncated at the
// boundaries (Toeplitz, no wrap).
//
// MGRIT runs on the right-hand-side form U[n+1] = Phi_h U[n] + b_n (R12, R20):
//  * Phi_h, the homogeneous operator (zero inflow ghosts, extrapolated outflow ghosts): the
//    whole-row relaxation sweep rk_sweep_kernel<..., BND = true> (rows.cuh) — one interval's
//    row in registers across all m steps and stages; the two row-end threads replace the
//    periodic wrap by the closures (device.cuh bounded_ghosts).
//  * b_n = Phi(0; t_n), the inflow forcing: bnd_forcing_kernel evaluates the Taylor /
//    inverse-Lax-Wendroff ghost values of every Runge-Kutta stage from the inflow derivatives
//    g^(r)(t_n) and steps the zero state; b_n is supported on the first S*NL points, so it is
//    stored as a compact row of FORC_LD doubles per time step.
//  * Psi_T: tpsi_seq_kernel (sequential coarse solve), tpsi_level_kernel (V-cycle level
//    sweep / interpolation) — fixed coordinates, the state in shared memory, taps that fall
//    outside [0, nx) read zero.
#include "kernels.h"
#include "rows.cuh"

namespace mg {

// ---------------------------------------------------------------------------
// Fine sweep with the boundary closures: explicit schemes, whole rows, P >= p + 1.
// ---------------------------------------------------------------------------
template <class SC>
static cudaError_t dispatch_bnd(SweepCfg c, const SweepArgs &a, cudaStream_t s) {
#define MG_CASE(NT_, P_)                                      \
  if (c.nt_threads == NT_ && c.p == P_) {                     \
    if constexpr (P_ >= SC::NL + SC::NR + 1)                  \
      return launch_one<SC, NT_, P_, FusedRT, true>(a, s);    \
    else                                                      \
      return cudaErrorInvalidConfiguration;                   \
  }
  MG_CASE(32, 2) MG_CASE(32, 4) MG_CASE(32, 8) MG_CASE(64, 8) MG_CASE(128, 8) MG_CASE(256, 8)
  MG_CASE(512, 8)
#undef MG_CASE
  return cudaErrorInvalidConfiguration;
}

bool rk_sweep_bnd_supported(int scheme, SweepCfg c) {
  if (scheme < 0 || scheme > 4) return false;
  const int p = rk_scheme_reach_left(scheme) + rk_scheme_reach_right(scheme);
  if (c.p < p + 1 || c.p > 8) return false;
  const int nts[] = {32, 64, 128, 256, 512};
  for (int nt : nts)
    if (c.nt_threads == nt && (nt == 32 || c.p == 8)) return true;
  return false;
}

cudaError_t launch_rk_sweep_bnd(int scheme, SweepCfg cfg, const SweepArgs &a, cudaStream_t s) {
  if (a.ntiles != 1 || cfg.nt_threads * cfg.p != a.nx) return cudaErrorInvalidConfiguration;
  switch (scheme) {
    case 0: return dispatch_bnd<ERK1U1>(cfg, a, s);
    case 1: return dispatch_bnd<ERK2U2>(cfg, a, s);
    case 2: return dispatch_bnd<ERK3U3>(cfg, a, s);
    case 3: return dispatch_bnd<ERK4U4>(cfg, a, s);
    case 4: return dispatch_bnd<ERK5U5>(cfg, a, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_rk_coarse_bnd(int scheme, SweepCfg c, const RKCoarseArgs &a, cudaStream_t s) {
  switch (scheme) {
    case 0: return launch_rkc<ERK1U1, true>(c, a, s);
    case 1: return launch_rkc<ERK2U2, true>(c, a, s);
    case 2: return launch_rkc<ERK3U3, true>(c, a, s);
    case 3: return launch_rkc<ERK4U4, true>(c, a, s);
    case 4: return launch_rkc<ERK5U5, true>(c, a, s);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
// Inflow forcing b_n = Phi(0; t_n) (R20).  One thread per time step; the arithmetic follows
// the stage form in the oracle's order with separately rounded products and sums.
//   ghost value of stage i at x_{-k}:  sum_{q<S} sum_{j<=p} (t1[q][i] * t2[k][j]) * dg[n][q+j],
//   t1[q][i] = dt^q (A^q 1)_i,  t2[k][j] = (k dx/alpha)^j / j!
//   k_i = Z y~_i with y_i = sum_{l<i} a_il k_l (u = 0), b_n = sum_i b_i k_i.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) bnd_forcing_kernel(const __grid_constant__ BndCoef c,
                                                          const double *__restrict__ dg,
                                                          long long nt, double *__restrict__ forc) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= nt) return;
  const int S = c.S, NL = c.NL, NR = c.NR, NB = c.S * c.NL;
  const double *d = dg + n * c.nq;
  double k[MAXS][FORC_LD];
  double ext[FORC_LD + 8];   // y~ on array indices a = -NL .. NB + NR - 1 (ext[a + NL])
  for (int i = 0; i < S; ++i) {
    for (int a = 0; a < NB + NR; ++a) {
      double y = 0.0;
      if (a < NB) {
        for (int l = 0; l < i; ++l)
          if (c.A[i][l] != 0.0) y = __dadd_rn(y, __dmul_rn(c.A[i][l], k[l][a]));
      }
      ext[NL + a] = y;
    }
    for (int kk = 0; kk < NL; ++kk) {   // array index -(kk+1) <-> x_{-kk}
      double acc = 0.0;
      for (int q = 0; q < S; ++q)
        for (int j = 0; j <= c.p; ++j)
          acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(c.t1[q][i], c.t2[kk][j]), d[q + j]));
      ext[NL - 1 - kk] = acc;
    }
    for (int a = 0; a < NB; ++a) {
      double out = 0.0;
      for (int t = 0; t <= NL + NR; ++t) {   // d = -NL + t ascending
        const double term = __dmul_rn(c.z[t], ext[a + t]);
        out = (t == 0) ? term : __dadd_rn(out, term);
      }
      k[i][a] = out;
    }
  }
  for (int a = 0; a < FORC_LD; ++a) {
    double out = 0.0;
    if (a < NB)
      for (int i = 0; i < S; ++i)
        if (c.b[i] != 0.0) out = __dadd_rn(out, __dmul_rn(c.b[i], k[i][a]));
    forc[n * FORC_LD + a] = out;
  }
}

cudaError_t launch_bnd_forcing(const BndCoef &c, const double *dg, long long nt, double *forc,
                               cudaStream_t s) {
  if (nt <= 0) return cudaSuccess;
  if (c.S * c.NL > FORC_LD || c.S > MAXS) return cudaErrorInvalidValue;
  bnd_forcing_kernel<<<(unsigned)((nt + 127) / 128), 128, 0, s>>>(c, dg, nt, forc);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Truncated Toeplitz Psi_T: (Psi_T u)_a = sum_{q: 0 <= a+o0+q < nx} psi_q u_{a+o0+q}.
// s holds the row in the padded layout (pidx); thread t produces its points [tP, tP+P).
// ---------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void tpsi_apply(const double *__restrict__ s, int nx, const PsiOp &op,
                                           double (&out)[P]) {
  const int base = threadIdx.x * P + op.o0;
  auto at = [&](int idx) -> double {
    return ((unsigned)idx < (unsigned)nx) ? s[pidx<P>(idx)] : 0.0;
  };
  double w[P + 3];
#pragma unroll
  for (int r = 0; r < P + 3; ++r) w[r] = at(base + r);
#pragma unroll
  for (int p = 0; p < P; ++p) out[p] = 0.0;
  const int nu4 = (op.nu + 3) & ~3;
#pragma unroll 1
  for (int q0 = 0; q0 < nu4; q0 += 4) {
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const double c = op.psi[q0 + qq];   // taps beyond nu are zero (PsiOp is zero-filled)
#pragma unroll
      for (int p = 0; p < P; ++p) out[p] = fma(c, w[p + qq], out[p]);
    }
#pragma unroll
    for (int r = 0; r + 4 < P + 3; ++r) w[r] = w[r + 4];
#pragma unroll
    for (int r = (P - 1 > 0 ? P - 1 : 0); r < P + 3; ++r) w[r] = at(base + q0 + 4 + r);
  }
}

template <int NT, int P>
__device__ __forceinline__ void tpsi_put(double *s, const double (&x)[P]) {
#pragma unroll
  for (int p = 0; p < P; ++p) s[threadIdx.x * Pad<P>::SP + p] = x[p];
}

// Sequential solve x_n = Psi_T x_{n-1} + g_n, out_n = out_n + x_n (out holds v_n),
// n = n0+1 .. n0+nsteps: one CTA, NT*P == nx, one barrier per step (ping-pong state
// buffers); the rows g_n, v_n are loaded D steps ahead into a register ring.
template <int NT, int P>
__global__ void __launch_bounds__(NT, 1) tpsi_seq_kernel(const __grid_constant__ CoarseArgs a) {
  constexpr int SP = Pad<P>::SP;
  extern __shared__ double smem[];
  double *buf0 = smem, *buf1 = smem + NT * SP;
  const int tid = threadIdx.x, nx = a.nx;
  constexpr int D = (16 / P) < 2 ? 2 : (16 / P);
  double x[P];
#pragma unroll
  for (int p = 0; p < P; ++p) x[p] = a.state_in ? a.state_in[tid * P + p] : 0.0;
  auto load = [&](int i, double(&gv)[P], double(&vv)[P]) {
    if (i > a.nsteps) return;
    const double *g = a.g.base + (a.g.off + (a.n0 + i) * a.g.stride) * (long long)nx;
    const double *v = a.out.base + (a.out.off + (a.n0 + i) * a.out.stride) * (long long)nx;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      gv[p] = g[tid * P + p];
      vv[p] = v[tid * P + p];
    }
  };
  double gr[D][P], vr[D][P];
#pragma unroll
  for (int d = 0; d < D; ++d) load(1 + d, gr[d], vr[d]);
#pragma unroll 1
  for (int i0 = 1; i0 <= a.nsteps; i0 += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int i = i0 + d;
      if (i > a.nsteps) break;
      double *sb = (i & 1) ? buf1 : buf0;
      tpsi_put<NT, P>(sb, x);
      __syncthreads();
      double y[P];
      tpsi_apply<P>(sb, nx, a.op, y);
      double *o = const_cast<double *>(a.out.base) + (a.out.off + (a.n0 + i) * a.out.stride) * (long long)nx;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        x[p] = y[p] + gr[d][p];
        o[tid * P + p] = vr[d][p] + x[p];
      }
      load(i + D, gr[d], vr[d]);
    }
  }
  if (a.state_out) {
#pragma unroll
    for (int p = 0; p < P; ++p) a.state_out[tid * P + p] = x[p];
  }
}

// V-cycle level kernel with Psi_T: the semantics of psi_sweep_kernel (kernels.h PsiSweepArgs),
// one CTA per level-l interval, fixed coordinates.
template <int NT, int P>
__global__ void __launch_bounds__(NT, 1) tpsi_level_kernel(const __grid_constant__ PsiSweepArgs a) {
  constexpr int SP = Pad<P>::SP;
  extern __shared__ double smem[];
  double *buf0 = smem, *buf1 = smem + NT * SP;
  const int tid = threadIdx.x, nx = a.nx, m = a.m;
  const int item = blockIdx.x;
  auto rowp = [&](const RowMap &r, long long j) {
    return r.base + (r.off + j * r.stride) * (long long)nx;
  };
  int par = 0;
  auto step = [&](double(&x)[P]) {   // x <- Psi_T x
    double *sb = par ? buf1 : buf0;
    par ^= 1;
    tpsi_put<NT, P>(sb, x);
    __syncthreads();
    tpsi_apply<P>(sb, nx, a.op, x);
  };
  double x[P];
#pragma unroll
  for (int p = 0; p < P; ++p) x[p] = a.u.base ? rowp(a.u, item)[tid * P + p] : 0.0;
  const long long grow0 = a.g.off + (long long)item * a.g.stride;   // row jm
  auto emit = [&](int i) {   // interp: out2[jm+i] = v2[jm+i] + x
    double *o = const_cast<double *>(a.out2.base) + (a.out2.off + (long long)item * a.out2.stride + i) * nx;
    const double *v = a.v2.base ? a.v2.base + (a.v2.off + (long long)item * a.v2.stride + i) * nx : nullptr;
#pragma unroll
    for (int p = 0; p < P; ++p) o[tid * P + p] = v ? v[tid * P + p] + x[p] : x[p];
  };
  if (a.interp) emit(0);
  const int n1 = a.interp ? (m - 1) : m;
#pragma unroll 1
  for (int i = 1; i <= n1; ++i) {
    double g[P];
    const double *gr = a.g.base + (grow0 + i) * nx;
#pragma unroll
    for (int p = 0; p < P; ++p) g[p] = gr[tid * P + p];
    step(x);
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] += g[p];
    if (a.interp) emit(i);
  }
  if (a.interp) return;
  {
    double *v = const_cast<double *>(rowp(a.v, item));
#pragma unroll
    for (int p = 0; p < P; ++p) v[tid * P + p] = x[p];
  }
  if (item >= a.p2_items) return;
  if (a.ucmp.base) {
    const double *uc = rowp(a.ucmp, item);
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] -= uc[tid * P + p];
  }
#pragma unroll 1
  for (int i = 1; i <= m; ++i) step(x);
  double *r = const_cast<double *>(rowp(a.r2, item));
#pragma unroll
  for (int p = 0; p < P; ++p) r[tid * P + p] = x[p];
}

#define MG_TPSI_CFGS(X) X(32, 2) X(32, 4) X(32, 8) X(64, 8) X(128, 8) X(256, 8) X(512, 8) X(1024, 4)

bool tpsi_cfg(int nx, bool seq, SweepCfg &cfg) {
  if (nx == 64) cfg = {32, 2};
  else if (nx == 128) cfg = {32, 4};
  else if (nx == 256) cfg = {32, 8};
  else if (nx == 512) cfg = {64, 8};
  else if (nx == 1024) cfg = {128, 8};
  else if (nx == 2048) cfg = {256, 8};
  else if (nx == 4096) cfg = seq ? SweepCfg{1024, 4} : SweepCfg{512, 8};
  else return false;
  return true;
}

cudaError_t launch_tpsi_seq(SweepCfg c, const CoarseArgs &a, cudaStream_t s) {
  if (a.nsteps <= 0) return cudaSuccess;
#define MG_CASE(NT_, P_)                                                        \
  if (c.nt_threads == NT_ && c.p == P_ && NT_ * P_ == a.nx) {                   \
    const size_t smem = sizeof(double) * 2 * NT_ * Pad<P_>::SP;                 \
    cudaFuncSetAttribute(tpsi_seq_kernel<NT_, P_>,                              \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    tpsi_seq_kernel<NT_, P_><<<1, NT_, smem, s>>>(a);                           \
    return cudaGetLastError();                                                  \
  }
  MG_TPSI_CFGS(MG_CASE)
#undef MG_CASE
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_tpsi_level(SweepCfg c, const PsiSweepArgs &a, cudaStream_t s) {
  if (a.nitems <= 0) return cudaSuccess;
#define MG_CASE(NT_, P_)                                                        \
  if (c.nt_threads == NT_ && c.p == P_ && NT_ * P_ == a.nx) {                   \
    const size_t smem = sizeof(double) * 2 * NT_ * Pad<P_>::SP;                 \
    cudaFuncSetAttribute(tpsi_level_kernel<NT_, P_>,                            \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    tpsi_level_kernel<NT_, P_><<<(unsigned)a.nitems, NT_, smem, s>>>(a);        \
    return cudaGetLastError();                                                  \
  }
  MG_TPSI_CFGS(MG_CASE)
#undef MG_CASE
  return cudaErrorInvalidConfiguration;
}

}  // namespace mg
