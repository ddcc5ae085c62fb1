// coarse.cu — coarse-grid kernels.
//
// Stencil coarse operators Psi are applied in *shifted* coordinates: with
// contiguous offsets o0..o0+nu-1, a CTA's window origin moves by -o0 per step
// and its valid length shrinks by nu-1 from the right, so the characteristic
// shift (up to ~870 points on cfg5's coarsest level) costs no halo.
//
//  * psi_coarse_kernel: sequential solve x_n = Psi x_{n-1} + g_n over a block of
//    steps, out_n = v_n + x_n (coarse error equation eq. (3) P:210 fused with the
//    C-point correction P:212).  Trapezoid tiles: each CTA recomputes the
//    dependency cone of its slice, so a launch needs no inter-CTA communication.
//  * psi_sweep_kernel: FCF relaxation + residual + injection of V-cycle level l>=2
//    (P:618-624), and its interpolation (correction fused into level l-1's C-rows).
//  * rk_coarse_kernel: IDEAL (Phi^m) / REDISC Psi in Runge-Kutta form.
#include "kernels.h"
#include "tma.cuh"
#include "rows.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace mg {

constexpr int PSI_EXT = MAX_PSI + 8;  // shared-memory tail for wrap/overrun reads

// (g mod nx) for |g| < 2^31 (32-bit division; origins are computed once per step/item)
__device__ __forceinline__ int wrapi(long long g, int nx) {
  const int r = (int)g % nx;
  return r < 0 ? r + nx : r;
}

// x'[p] = sum_q psi_q s[base + p + q]  (s holds the current state, unpadded).
template <int P>
__device__ __forceinline__ void psi_apply(const double *__restrict__ s, int base,
                                          const PsiOp &op, double (&out)[P]) {
  double w[P + 3];
#pragma unroll
  for (int r = 0; r < P + 3; ++r) w[r] = s[pidx<P>(base + r)];
#pragma unroll
  for (int p = 0; p < P; ++p) out[p] = 0.0;
  const int nu4 = (op.nu + 3) & ~3;
#pragma unroll 1
  for (int q0 = 0; q0 < nu4; q0 += 4) {
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const double c = op.psi[q0 + qq];
#pragma unroll
      for (int p = 0; p < P; ++p) out[p] = fma(c, w[p + qq], out[p]);
    }
#pragma unroll
    for (int r = 0; r + 4 < P + 3; ++r) w[r] = w[r + 4];
#pragma unroll
    for (int r = P - 1; r < P + 3; ++r) w[r] = s[pidx<P>(base + q0 + 4 + r)];
  }
}

// Same with the tap count NU known at compile time and the window starting at the
// thread's own first point (base = threadIdx.x * P): the whole P + NU - 1 window is read
// once with immediate offsets and the NU * P FMAs (two partial sums) run from registers.
template <int P, int NU>
__device__ __forceinline__ void psi_apply_own(const double *__restrict__ s, const PsiOp &op,
                                              double (&out)[P]) {
  constexpr int SP = Pad<P>::SP;
  const double *s0 = s + threadIdx.x * SP;
  double w[P + NU - 1];
#pragma unroll
  for (int r = 0; r < P + NU - 1; ++r) w[r] = s0[(r / P) * SP + r % P];
  double a0[P], a1[P];
#pragma unroll
  for (int p = 0; p < P; ++p) { a0[p] = 0.0; a1[p] = 0.0; }
#pragma unroll
  for (int q = 0; q < NU; ++q) {
    const double c = op.psi[q];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (q & 1) a1[p] = fma(c, w[p + q], a1[p]);
      else a0[p] = fma(c, w[p + q], a0[p]);
    }
  }
#pragma unroll
  for (int p = 0; p < P; ++p) out[p] = a0[p] + a1[p];
}

// Write the state into s (padded layout) plus the periodic tail: logical
// s[W + e] = s[e mod W] for e < PSI_EXT.
template <int NT, int P>
__device__ __forceinline__ void psi_put(double *s, const double (&x)[P]) {
  constexpr int W = NT * P;
  const int t = threadIdx.x;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int l = t * P + p;
    s[t * Pad<P>::SP + p] = x[p];
    for (int e = l; e < PSI_EXT; e += W) s[pidx<P>(W + e)] = x[p];
  }
}

// Shared-memory sizes (doubles) of the padded buffers.
template <int NT, int P> struct PsiSmem {
  static constexpr int SP = Pad<P>::SP;
  static constexpr int X = (NT + PSI_EXT / P + 2) * SP;  // state + tail
  static constexpr int G = NT * SP;                      // g window / staging
  static constexpr int TOTAL = 2 * X + 2 * G;   // ping-pong state + ping-pong g/staging
};

// fp64 add at L2, no return (fire-and-forget RED).
__device__ __forceinline__ void red_add_f64(double *p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// Sequential solve  x_n = Psi x_{n-1} + g_n,  out_n += x_n  (n = n0+1 .. n0+N).
// The dependent chain runs in one CTA per (trapezoid) tile with no global latency inside a
// step: g rows stream into a ring of R contiguous slots by TMA bulk copies issued R-1 steps
// ahead (mbarrier per slot); each step applies Psi from the padded state buffer, then a
// coalesced pass adds g_n and writes x_n both to the state (padded) and to a contiguous
// staging slot, whose bulk reduce-add performs the C-point correction out_n += x_n at L2
// (out holds v_n).  Two barriers per step, three staging slots, ping-pong state buffers.
template <int NT, int P, int R>
struct CoarseSmem {
  static constexpr int W = NT * P;
  static constexpr int X = PsiSmem<NT, P>::X;        // padded state + tail
  static constexpr int WB = W + 2;                    // contiguous row slot (even)
  static constexpr int TOTAL = 2 * X + R * WB + 3 * WB + 2 * R + 8;
};

template <int NT, int P, int R, int NU>
__global__ void __launch_bounds__(NT, 1) psi_coarse_kernel(const __grid_constant__ CoarseArgs a) {
  using CS = CoarseSmem<NT, P, R>;
  constexpr int W = NT * P, WB = CS::WB;
  extern __shared__ __align__(128) double smem[];
#define SX(b) (smem + (b) * CS::X)
#define GR(k) (smem + 2 * CS::X + (k) * WB)
#define ST(k) (smem + 2 * CS::X + R * WB + (k) * WB)
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 2 * CS::X + (R + 3) * WB);
  const int nx = a.nx, tid = threadIdx.x;
  const int tile = blockIdx.x;
  const int abeg = (int)(((long long)tile * nx) / a.ntiles);
  const int T = (int)(((long long)(tile + 1) * nx) / a.ntiles) - abeg;
  const int N = a.nsteps, o0 = a.op.o0;
  const bool periodic = (a.ntiles == 1 && W == nx);
  auto origin = [&](int i) { return wrapi((long long)abeg + (long long)(N - i) * o0, nx); };
  auto fetch = [&](int i) {  // (thread 0) g row of step i -> ring slot i % R
    if (i > N) return;
    const double *grow = a.g.base + (a.g.off + (a.n0 + i) * a.g.stride) * (long long)nx;
    const int S0 = origin(i) & ~1;
    const int n1 = (S0 + WB <= nx) ? WB : nx - S0;
    uint64_t *b = &bar[i % R];
    mbar_expect_tx(b, (uint32_t)WB * 8u);
    tma_load_1d(GR(i % R), grow + S0, (uint32_t)n1 * 8u, b);
    if (n1 < WB) tma_load_1d(GR(i % R) + n1, grow, (uint32_t)(WB - n1) * 8u, b);
  };
  if (tid == 0) {
    for (int k = 0; k < R; ++k) mbar_init(&bar[k], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int i = 1; i < R; ++i) fetch(i);
  // x_0 into SX(0)
  if (a.state_in) {
    const int S0 = origin(0);
    for (int q = tid; q < W; q += NT) {
      int g = S0 + q;
      if (g >= nx) g -= nx;
      const double v = a.state_in[g];
      SX(0)[pidx<P>(q)] = v;
      if (q < PSI_EXT) SX(0)[pidx<P>(W + q)] = v;
    }
  } else {
    for (int q = tid; q < W + PSI_EXT; q += NT) SX(0)[pidx<P>(q)] = 0.0;
  }
  __syncthreads();
#pragma unroll 1
  for (int i = 1; i <= N; ++i) {
    const double *sprev = SX((i - 1) & 1);
    double *scur = SX(i & 1);
    double y[P];
    if constexpr (NU > 0) psi_apply_own<P, NU>(sprev, a.op, y);
    else psi_apply<P>(sprev, threadIdx.x * P, a.op, y);
    psi_put<NT, P>(scur, y);
    if (tid == 0) {
      fetch(i + R - 1);  // slot (i-1) % R was consumed before the last barrier
      if (i > 3) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // ST((i)%3) free
    }
    __syncthreads();
    // coalesced pass: x_i = y + g_i  (state, tail, staging)
    const int Si = origin(i);
    mbar_wait(&bar[i % R], (uint32_t)(((i - 1) / R) & 1));
    const double *gi = GR(i % R) + (Si & 1);
    double *st = ST(i % 3) + (Si & 1);
    for (int q = tid; q < W; q += NT) {
      const int ix = pidx<P>(q);
      const double v = scur[ix] + gi[q];
      scur[ix] = v;
      if (q < PSI_EXT) scur[pidx<P>(W + q)] = v;
      if (q < T) st[q] = v;
    }
    if (periodic) {  // the tail mirrors the start of the row
      // (entries W + q, q < PSI_EXT were written above from the same q)
    }
    fence_proxy_async();
    __syncthreads();
    // out_i[S_i .. S_i+T) += staging (bulk reduce-add; odd ends by scalar RMW)
    double *orow = const_cast<double *>(a.out.base) + (a.out.off + (a.n0 + i) * a.out.stride) * (long long)nx;
    const double *buf = ST(i % 3);
    const int so = Si & 1;
    int segs[2][2];
    int ns = 1;
    if (Si + T <= nx) { segs[0][0] = Si; segs[0][1] = Si + T; }
    else { segs[0][0] = Si; segs[0][1] = nx; segs[1][0] = 0; segs[1][1] = Si + T - nx; ns = 2; }
    int scalar = 0;
    for (int k = 0; k < ns; ++k) {
      int ga = segs[k][0], gb = segs[k][1];
      const int base = so + (k == 0 ? -Si : nx - Si);
      if (ga < gb && (ga & 1)) {
        if (tid == 1 + scalar) orow[ga] += buf[base + ga];
        ++scalar;
        ++ga;
      }
      if (ga < gb && ((gb - ga) & 1)) {
        if (tid == 1 + scalar) orow[gb - 1] += buf[base + gb - 1];
        ++scalar;
        --gb;
      }
      if (tid == 0 && gb > ga) tma_reduce_add_1d(orow + ga, buf + base + ga, (uint32_t)(gb - ga) * 8u);
    }
    if (tid == 0) bulk_commit();
  }
  if (a.state_out) {  // S_N = abeg: the owned slice [abeg, abeg+T)
    const double *sN = SX(N & 1);
    for (int q = tid; q < T; q += NT) a.state_out[abeg + q] = sN[pidx<P>(q)];
  }
  if (tid == 0) bulk_wait_all();
#undef SX
#undef GR
#undef ST
}

// --------------------------------------------------------------------------
// Periodic single-CTA sequential solve (two-level coarse grid), fixed
// coordinates: thread t owns points [tP, tP+P) of the whole row (NT*P == nx) for the
// stencil, read at base (tP + o0) mod nx from the padded state whose periodic tail
// mirrors its start.  The rows g_n and v_n (the uncorrected C-row) stream into a
// ring of D contiguous slots by TMA bulk copies issued D-1 steps ahead; a coalesced pass
// per step adds g_n into the state and writes u_n = v_n + x_n with coalesced stores.
// Two barriers per step; no global latency inside the chain.
template <int NT, int P, int D>
struct SeqSmem {
  static constexpr int W = NT * P;
  static constexpr int X = PsiSmem<NT, P>::X;
  static constexpr size_t BYTES = sizeof(double) * (2 * (size_t)X + 2 * (size_t)D * W) + 8 * D + 64;
};

template <int NT, int P, int D>
__global__ void __launch_bounds__(NT, 1) psi_seq_periodic_kernel(const __grid_constant__ CoarseArgs a) {
  using SS = SeqSmem<NT, P, D>;
  constexpr int W = NT * P;
  extern __shared__ __align__(128) double smem[];
  double *S0 = smem, *S1 = smem + SS::X;
  double *ring = smem + 2 * SS::X;                 // [D][2][W]: g, v (contiguous)
  uint64_t *bar = reinterpret_cast<uint64_t *>(ring + 2 * (size_t)D * W);
  const int tid = threadIdx.x;
  const int N = a.nsteps;
  int rb = (tid * P + a.op.o0) % W;
  if (rb < 0) rb += W;
  const double *gbase = a.g.base + (a.g.off + a.n0 * a.g.stride) * (long long)W;
  double *obase = const_cast<double *>(a.out.base) + (a.out.off + a.n0 * a.out.stride) * (long long)W;
  const long long gst = a.g.stride * (long long)W, ost = a.out.stride * (long long)W;
  auto fetch = [&](int i) {  // thread 0: rows g_i, v_i -> slot i % D
    if (i > N) return;
    double *gs = ring + (size_t)(i % D) * 2 * W;
    mbar_expect_tx(&bar[i % D], (uint32_t)(2 * W) * 8u);
    tma_load_1d(gs, gbase + i * gst, (uint32_t)W * 8u, &bar[i % D]);
    tma_load_1d(gs + W, obase + i * ost, (uint32_t)W * 8u, &bar[i % D]);
  };
  if (tid == 0) {
    for (int k = 0; k < D; ++k) mbar_init(&bar[k], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int i = 1; i < D; ++i) fetch(i);
  double x[P];
  if (a.state_in) {
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = a.state_in[tid * P + p];
  } else {
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = 0.0;
  }
  psi_put<NT, P>(S0, x);
  __syncthreads();
#pragma unroll 1
  for (int i = 1; i <= N; ++i) {
    const double *sprev = (i & 1) ? S0 : S1;
    double *scur = (i & 1) ? S1 : S0;
    double y[P];
    psi_apply<P>(sprev, rb, a.op, y);
#pragma unroll
    for (int p = 0; p < P; ++p) scur[tid * Pad<P>::SP + p] = y[p];
    if (tid == 0) fetch(i + D - 1);              // slot (i-1) % D was consumed last step
    __syncthreads();
    mbar_wait(&bar[i % D], (uint32_t)(((i - 1) / D) & 1));
    const double *gs = ring + (size_t)(i % D) * 2 * W;
    const double *vs = gs + W;
    double *orow = obase + i * ost;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int q = tid + k * NT;
      const int ix = pidx<P>(q);
      const double xv = scur[ix] + gs[q];       // x_i = Psi x_{i-1} + g_i
      scur[ix] = xv;
      if (q < PSI_EXT) scur[pidx<P>(W + q)] = xv;
      orow[q] = vs[q] + xv;                     // u_i = v_i + e_i
    }
    __syncthreads();
  }
  if (a.state_out) {
    const double *sN = (N & 1) ? S1 : S0;
    for (int q = tid; q < W; q += NT) a.state_out[q] = sN[pidx<P>(q)];
  }
}

template <int NT, int P, int D>
static cudaError_t launch_seq_periodic_d(const CoarseArgs &a, cudaStream_t s) {
  const size_t smem = SeqSmem<NT, P, D>::BYTES;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(psi_seq_periodic_kernel<NT, P, D>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  psi_seq_periodic_kernel<NT, P, D><<<1, NT, smem, s>>>(a);
  return cudaGetLastError();
}

// prefetch depth: up to 8 steps where shared memory allows
template <int NT, int P>
static cudaError_t launch_seq_periodic(const CoarseArgs &a, cudaStream_t s) {
  if constexpr (SeqSmem<NT, P, 8>::BYTES <= 220 * 1024) return launch_seq_periodic_d<NT, P, 8>(a, s);
  else if constexpr (SeqSmem<NT, P, 4>::BYTES <= 220 * 1024) return launch_seq_periodic_d<NT, P, 4>(a, s);
  else return launch_seq_periodic_d<NT, P, 2>(a, s);
}

// --------------------------------------------------------------------------
// Cluster-wide periodic sequential solve (two-level coarse grid): the periodic
// row is split over the CL CTAs of one thread-block cluster (CTA c owns [c*Wc, (c+1)*Wc),
// Wc = NT*P), so a step's nu*nx FMAs run on CL SMs.  Per step i: Psi from the CTA's
// buffer B[(i-1)&1] (own values + left/right halos of x_{i-1}), x_i = Psi x_{i-1} + g_i,
// u_i = v_i + x_i.  Own x_i goes to the local buffer B[i&1]; the boundary values
// are written straight into the neighbours' B[i&1] halos with st.async, each completing
// bytes on the receiver's halo mbarrier hb[i&1] -- point-to-point, no cluster barrier and
// no memory fence in the loop.  WAR safety by causality: a neighbour writes my B[i&1]
// (step i) only after receiving my x_{i-1}, sent after this CTA's __syncthreads that
// follows every read of B[i&1] (step i-1).
// Global memory is touched only by the async proxy: TMA bulk loads of g_i / v_i into a
// D-deep ring and bulk stores of u_i from a 3-deep staging ring, issued by thread 0.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  mg_jitter(6);
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  mg_jitter(7);
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

template <int NT, int P> struct ClusterSmem {
  static constexpr int HMAX = 64;  // max halo per side (host-checked)
  static constexpr int Wc = NT * P;
  static constexpr int BL = ((HMAX + Wc + HMAX + PSI_EXT) / P + 2) * Pad<P>::SP;
  static constexpr size_t BYTES = sizeof(double) * 2 * BL + 24;  // 2 state buffers, 3 mbarriers
};

// y_p = sum_q psi_q x[base + p + q], q < NU4 (coefficients zero-padded past nu): the whole
// window is loaded at once and each output keeps two partial sums (short FMA chains).
template <int P, int NU4>
__device__ __forceinline__ void psi_apply_pad2(const double *__restrict__ s, int base,
                                                const PsiOp &op, double (&out)[P]) {
  double w[P + NU4 - 1];
#pragma unroll
  for (int r = 0; r < P + NU4 - 1; ++r) w[r] = s[pidx<P>(base + r)];
  double acc0[P], acc1[P];
#pragma unroll
  for (int p = 0; p < P; ++p) { acc0[p] = 0.0; acc1[p] = 0.0; }
#pragma unroll
  for (int q = 0; q < NU4; q += 2) {
    const double c0 = op.psi[q], c1 = op.psi[q + 1];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      acc0[p] = fma(c0, w[p + q], acc0[p]);
      acc1[p] = fma(c1, w[p + q + 1], acc1[p]);
    }
  }
#pragma unroll
  for (int p = 0; p < P; ++p) out[p] = acc0[p] + acc1[p];
}

// Register-ring version: each thread prefetches g_i and v_i of its own P points D steps
// ahead with plain loads and stores u_i directly (no fence anywhere in the loop, so the
// stores are fire-and-forget).  The halo senders and the halo readers of each side lie in
// one warp (host-checked), so a __syncwarp -- not the CTA barrier -- orders a warp's
// reads of B[(i-1)&1] before its sends of x_i: the inter-CTA chain per step is
// halo wait -> window load -> NU4/2 FMAs -> st.async.
template <int NT, int P, int CL, int D, int NU4>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT, 1)
    psi_seq_cluster_kernel(const __grid_constant__ CoarseArgs a) {
  static_assert(P % 2 == 0, "P even (16-byte vector loads)");
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  using CS = ClusterSmem<NT, P>;
  constexpr int Wc = CS::Wc, HMAX = CS::HMAX, BL = CS::BL;
  extern __shared__ __align__(128) double smem[];
  // Halo mbarriers: x_s lands on hb[s % 3].  Three, not two: the boundary warps run
  // ahead of the CTA barrier, so the neighbours' x_{i+1} can complete while a warp of this
  // CTA is still waiting for x_{i-1}; with two barriers that phase would alias.
  uint64_t *hb = reinterpret_cast<uint64_t *>(smem + 2 * BL);
  const uint32_t rank = cluster.block_rank();
  const int tid = threadIdx.x;
  const int N = a.nsteps, o0 = a.op.o0, nu = a.op.nu;
  // Halo widths, at least one point each way even for a one-sided stencil: the exchange
  // must be mutual every step, else a CTA could run ahead of the neighbour it feeds (the
  // ring only bounds the lead by CL steps) and overwrite halos / mbarrier phases that
  // neighbour has not consumed.  A point past the stencil is read with a zero weight.
  const int HL = o0 < 0 ? max(-o0, 1) : 1;         // left halo (points before the slice)
  const int HR = max(o0 + nu - 1, 1);
  const uint32_t hbytes = (uint32_t)(HL + HR) * 8u;
  const int gx0 = rank * Wc + tid * P;             // global index of the thread's first point
  const double *gb = a.g.base + (a.g.off + a.n0 * a.g.stride) * (long long)a.nx + gx0;
  double *ob = const_cast<double *>(a.out.base) + (a.out.off + a.n0 * a.out.stride) * (long long)a.nx + gx0;
  const long long gst = a.g.stride * (long long)a.nx, ost = a.out.stride * (long long)a.nx;
  const uint32_t rprev = (rank + CL - 1) % CL, rnext = (rank + 1) % CL;
  const uint32_t s_base = smem_u32(smem);
  const uint32_t p_base = mapa_shared(s_base, rprev), n_base = mapa_shared(s_base, rnext);
  const uint32_t p_hb = mapa_shared(smem_u32(hb), rprev), n_hb = mapa_shared(smem_u32(hb), rnext);
  // local buffer index: HMAX + l for own point l; l < 0 left halo, l >= Wc right halo
  auto publish_local = [&](int k, const double(&x)[P]) {
    double *bk = smem + k * BL;
#pragma unroll
    for (int p = 0; p < P; ++p) bk[pidx<P>(HMAX + tid * P + p)] = x[p];
  };
  auto send_halo = [&](int k, int h, const double(&x)[P]) {  // buffer k, mbarrier h
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int l = tid * P + p;
      if (l < HR)            // prev's right halo
        st_async_f64(p_base + 8u * (uint32_t)(k * BL + pidx<P>(HMAX + Wc + l)), x[p], p_hb + 8u * h);
      if (l >= Wc - HL)      // next's left halo
        st_async_f64(n_base + 8u * (uint32_t)(k * BL + pidx<P>(HMAX + l - Wc)), x[p], n_hb + 8u * h);
    }
  };
  for (int q = tid; q < 2 * BL; q += NT) smem[q] = 0.0;  // over-read slots stay finite
  if (tid == 0) {
    for (int k = 0; k < 3; ++k) mbar_init(&hb[k], 1);
    fence_mbar_init();
    for (int k = 0; k < 3; ++k) mbar_expect_tx(&hb[k], hbytes);  // halos of x_0, x_1, x_2
  }
  double x[P];
  if (a.state_in) {
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = a.state_in[gx0 + p];
  } else {
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = 0.0;
  }
  double gq[D][P], vq[D][P];
  auto load = [&](int d, int i) {
#pragma unroll
    for (int p = 0; p < P; p += 2) {
      const double2 g2 = __ldg(reinterpret_cast<const double2 *>(gb + i * gst + p));
      const double2 v2 = __ldg(reinterpret_cast<const double2 *>(ob + i * ost + p));
      gq[d][p] = g2.x; gq[d][p + 1] = g2.y;
      vq[d][p] = v2.x; vq[d][p + 1] = v2.y;
    }
  };
#pragma unroll
  for (int d = 0; d < D; ++d)
    if (1 + d <= N) load(d, 1 + d);
  cluster.sync();  // buffers zeroed, barriers armed everywhere before any remote store
  publish_local(0, x);
  send_halo(0, 0, x);
  __syncthreads();
  int hp = 0;                                      // (i - 1) % 3
  const int base = HMAX + tid * P + o0;
  const bool edge_warp = (tid >> 5) == 0 || (tid >> 5) == NT / 32 - 1;
#pragma unroll 1
  for (int i0 = 1; i0 <= N; i0 += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int i = i0 + d;
      if (i <= N) {
        const int kp = (i - 1) & 1, kc = i & 1;
        // halos of x_{i-1}: only the boundary warps read them (the others read their own
        // region, ordered by the CTA barrier).  The st.async data lands in this CTA's
        // shared memory and completes on its own mbarrier, so a CTA-scope acquire (no L1
        // invalidation) suffices, as for a TMA load.
        if (edge_warp) mbar_wait(&hb[hp], (uint32_t)(((i - 1) / 3) & 1));
        double y[P];
        psi_apply_pad2<P, NU4>(smem + kp * BL, base, a.op, y);
#pragma unroll
        for (int p = 0; p < P; ++p) x[p] = y[p] + gq[d][p];          // x_i = Psi x_{i-1} + g_i
        __syncwarp();                               // this warp's reads of B[kp] done
        const int hc = hp == 2 ? 0 : hp + 1;      // i % 3
        send_halo(kc, hc, x);
        publish_local(kc, x);
        double *orow = ob + i * ost;
#pragma unroll
        for (int p = 0; p < P; p += 2)              // u_i = v_i + e_i
          *reinterpret_cast<double2 *>(orow + p) = make_double2(vq[d][p] + x[p], vq[d][p + 1] + x[p + 1]);
        if (i + D <= N) load(d, i + D);             // refill this ring slot D steps ahead
        if (tid == 0) mbar_expect_tx(&hb[hp], hbytes);  // re-arm for the halos of x_{i+2}
        hp = hc;
        __syncthreads();                            // B[kc] complete; B[kp] reads done
      }
    }
  }
  if (a.state_out) {
#pragma unroll
    for (int p = 0; p < P; ++p) a.state_out[gx0 + p] = x[p];
  }
  // the halos of x_N may still be landing here: wait for them, and keep every CTA's
  // shared memory alive until all have
  mbar_wait_cluster(&hb[N % 3], (uint32_t)((N / 3) & 1));
  cluster.sync();
}

template <int NT, int P, int CL, int NU4, int D = 4>
static cudaError_t launch_seq_cluster_nu(const CoarseArgs &a, cudaStream_t s) {
  const size_t smem = ClusterSmem<NT, P>::BYTES;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(psi_seq_cluster_kernel<NT, P, CL, D, NU4>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (CL > 8)
      cudaFuncSetAttribute(psi_seq_cluster_kernel<NT, P, CL, D, NU4>,
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  psi_seq_cluster_kernel<NT, P, CL, D, NU4><<<CL, NT, smem, s>>>(a);
  return cudaGetLastError();
}

template <int NT, int P, int CL>
static cudaError_t launch_seq_cluster(const CoarseArgs &a, cudaStream_t s) {
  const int nu = a.op.nu;
  if (nu <= 12) return launch_seq_cluster_nu<NT, P, CL, 12>(a, s);
  if (nu <= 16) return launch_seq_cluster_nu<NT, P, CL, 16>(a, s);
  if (nu <= 20) return launch_seq_cluster_nu<NT, P, CL, 20>(a, s);
  if (nu <= 24) return launch_seq_cluster_nu<NT, P, CL, 24>(a, s);
  if (nu <= 32) return launch_seq_cluster_nu<NT, P, CL, 32>(a, s);
  if (nu <= 40) return launch_seq_cluster_nu<NT, P, CL, 40>(a, s);
  if (nu <= 48) return launch_seq_cluster_nu<NT, P, CL, 48>(a, s);
  return launch_seq_cluster_nu<NT, P, CL, 64>(a, s);
}

// Host check for the cluster path: nx == cl*NT*P, halos <= 64 and each side's halo
// senders and readers inside one warp.
bool seq_cluster_ok(int cl, SweepCfg c, int nx, int o0, int nu) {
  if (cl < 2 || cl > 16 || cl * c.nt_threads * c.p != nx) return false;
  const int hl = std::max(1, -o0), hr = std::max(1, o0 + nu - 1);
  int nu4 = 64;
  for (int v : {12, 16, 20, 24, 32, 40, 48})
    if (nu <= v) { nu4 = v; break; }
  const int wpts = 32 * c.p;  // points per warp
  return hl <= 64 && hr <= 64 && hl <= wpts && hr <= wpts && c.nt_threads >= 64 &&
         nu4 + c.p + 2 + std::max(o0, 0) <= wpts && std::max(-o0, 0) <= wpts;
}

// --------------------------------------------------------------------------
// Communication-avoiding cluster solve (s-step halos).  Same chain and split as above, but
// the CTA also keeps an extended halo of EL >= S*HL points on the left and ER >= S*HR on
// the right and advances the whole extended region S steps between exchanges: after k
// local steps the values are exact on [-(S-k)HL, Wc+(S-k)HR), so after S steps the own
// region [0, Wc) is exact and only then are EL / ER boundary points exchanged (st.async
// into the neighbours' receive buffers, complete_tx on their mbarriers).  The inter-SM
// latency is paid once per S steps; the price is (EL+ER)/Wc redundant FMAs.
// Threads: t covers local points l = -EL + t*P + p; own threads are t in [EL/P, EL/P+NT).
// Per super-step j (steps jS+1..jS+S): halo threads wait for exchange j (x_{jS} of the
// neighbours' boundary points) and copy it from the receive buffer R[j&1] into the state
// buffer; then S local steps, each one CTA barrier.  R is separate from the state
// buffers, so a neighbour that runs ahead cannot overwrite halo values still being read.
template <int NT, int P> struct CaSmem {
  static constexpr int EMAX = 256;                  // EL + ER <= EMAX (host-checked)
  static constexpr int MARG = 64;                   // left over-read (-o0 <= 64), multiple of P
  static constexpr int MARGR = 160;                 // right over-read (HR + NU4 padding + P)
  static constexpr int Wc = NT * P;
  static constexpr int COLS = (MARG + EMAX + Wc + MARGR) / P + 1;
  static constexpr int BL = COLS * P;               // state buffer, structure of arrays [P][COLS]
  static constexpr int D = 6;                       // cp.async ring depth (steps)
  static constexpr int GW = EMAX + Wc;              // g ring row (extended region), v: Wc
  static constexpr size_t BYTES =
      sizeof(double) * (2 * (size_t)BL + 2 * EMAX + (size_t)D * (GW + Wc)) + 24;
};

// Stencil window from a [P][COLS] structure-of-arrays buffer: logical slot q lives at
// (q % P) * COLS + q / P, so for every window offset the 32 lanes of a warp read 32
// consecutive doubles (no bank conflicts).  Whole window in registers, two partial sums.
template <int P, int COLS, int NU4>
__device__ __forceinline__ void psi_soa_fixed(const double *__restrict__ s, int base,
                                              const PsiOp &op, double (&out)[P]) {
  double w[P + NU4 - 1];
#pragma unroll
  for (int r = 0; r < P + NU4 - 1; ++r) w[r] = s[((base + r) % P) * COLS + (base + r) / P];
  double acc0[P], acc1[P];
#pragma unroll
  for (int p = 0; p < P; ++p) { acc0[p] = 0.0; acc1[p] = 0.0; }
#pragma unroll
  for (int q = 0; q < NU4; q += 2) {
    const double c0 = op.psi[q], c1 = op.psi[q + 1];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      acc0[p] = fma(c0, w[p + q], acc0[p]);
      acc1[p] = fma(c1, w[p + q + 1], acc1[p]);
    }
  }
#pragma unroll
  for (int p = 0; p < P; ++p) out[p] = acc0[p] + acc1[p];
}
// Same with the window's phase REM = base % P known at compile time: s0 points at column
// base / P, every load has an immediate offset (no per-tap index arithmetic).
template <int P, int COLS, int NU4, int REM>
__device__ __forceinline__ void psi_soa_rem(const double *__restrict__ s0, const PsiOp &op,
                                            double (&out)[P]) {
  double w[P + NU4 - 1];
#pragma unroll
  for (int r = 0; r < P + NU4 - 1; ++r) w[r] = s0[((REM + r) % P) * COLS + (REM + r) / P];
  double acc0[P], acc1[P];
#pragma unroll
  for (int p = 0; p < P; ++p) { acc0[p] = 0.0; acc1[p] = 0.0; }
#pragma unroll
  for (int q = 0; q < NU4; q += 2) {
    const double c0 = op.psi[q], c1 = op.psi[q + 1];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      acc0[p] = fma(c0, w[p + q], acc0[p]);
      acc1[p] = fma(c1, w[p + q + 1], acc1[p]);
    }
  }
#pragma unroll
  for (int p = 0; p < P; ++p) out[p] = acc0[p] + acc1[p];
}
template <int P, int COLS, int NU4>
__device__ __forceinline__ void psi_soa_dispatch(const double *__restrict__ s, int base,
                                                 const PsiOp &op, double (&out)[P]) {
  const int rem = base % P;           // base >= 0
  const double *s0 = s + base / P;
  if constexpr (P == 2) {
    if (rem == 0) psi_soa_rem<P, COLS, NU4, 0>(s0, op, out);
    else psi_soa_rem<P, COLS, NU4, 1>(s0, op, out);
  } else if constexpr (P == 4) {
    if (rem == 0) psi_soa_rem<P, COLS, NU4, 0>(s0, op, out);
    else if (rem == 1) psi_soa_rem<P, COLS, NU4, 1>(s0, op, out);
    else if (rem == 2) psi_soa_rem<P, COLS, NU4, 2>(s0, op, out);
    else psi_soa_rem<P, COLS, NU4, 3>(s0, op, out);
  } else {
    psi_soa_fixed<P, COLS, NU4>(s, base, op, out);
  }
}
// Wide stencils: the window streamed through registers four taps at a time.
template <int P, int COLS>
__device__ __forceinline__ void psi_soa_chunked(const double *__restrict__ s, int base,
                                                const PsiOp &op, double (&out)[P]) {
  auto ld = [&](int q) { return s[(q % P) * COLS + q / P]; };
  double w[P + 3];
#pragma unroll
  for (int r = 0; r < P + 3; ++r) w[r] = ld(base + r);
#pragma unroll
  for (int p = 0; p < P; ++p) out[p] = 0.0;
  const int nu4 = (op.nu + 3) & ~3;
#pragma unroll 1
  for (int q0 = 0; q0 < nu4; q0 += 4) {
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const double c = op.psi[q0 + qq];
#pragma unroll
      for (int p = 0; p < P; ++p) out[p] = fma(c, w[p + qq], out[p]);
    }
#pragma unroll
    for (int r = 0; r + 4 < P + 3; ++r) w[r] = w[r + 4];
#pragma unroll
    for (int r = P - 1; r < P + 3; ++r) w[r] = ld(base + q0 + 4 + r);
  }
}
__device__ __forceinline__ void cp_async16(void *dst_s, const void *src_g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst_s)), "l"(src_g)
               : "memory");
}

// The g_i / v_i rows come in through a per-thread cp.async ring (D steps deep): unlike
// register prefetches, cp.async copies are not waited for by the per-step CTA barrier
// (a plain load in flight must complete before bar.sync releases), so the DRAM latency
// stays off the step chain.
template <int NT, int P, int CL, int NU4>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT + 128, 1)
    psi_seq_cluster_ca_kernel(const __grid_constant__ CoarseArgs a, int S) {
  static_assert(P % 2 == 0, "P even (16-byte copies)");
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  using CS = CaSmem<NT, P>;
  constexpr int Wc = CS::Wc, BL = CS::BL, COLS = CS::COLS, MARG = CS::MARG, D = CS::D, GW = CS::GW;
  extern __shared__ __align__(128) double smem[];
  double *R = smem + 2 * BL;                        // receive buffers [2][EL + ER]
  double *gring = R + 2 * CS::EMAX;                 // [D][GW]
  double *vring = gring + (size_t)D * GW;           // [D][Wc]
  uint64_t *hb = reinterpret_cast<uint64_t *>(vring + (size_t)D * Wc);  // exchange j: hb[j % 3]
  const uint32_t rank = cluster.block_rank();
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int N = a.nsteps, o0 = a.op.o0, nu = a.op.nu;
  const int HL = o0 < 0 ? max(-o0, 1) : 1, HR = max(o0 + nu - 1, 1);
  const int EL = ((S * HL + P - 1) / P) * P, ER = ((S * HR + P - 1) / P) * P;
  const uint32_t hbytes = (uint32_t)(EL + ER) * 8u;
  const int l0 = -EL + tid * P;                    // first local point of this thread
  const bool active = l0 < Wc + ER;
  const bool own = l0 >= 0 && l0 < Wc;
  const bool lhalo = l0 < 0, rhalo = l0 >= Wc && active;
  int gx = (int)rank * Wc + l0;                    // global index (periodic)
  if (gx < 0) gx += a.nx;
  if (gx >= a.nx) gx -= a.nx;
  const double *gb = a.g.base + (a.g.off + a.n0 * a.g.stride) * (long long)a.nx + gx;
  double *ob = const_cast<double *>(a.out.base) + (a.out.off + a.n0 * a.out.stride) * (long long)a.nx + gx;
  const long long gst = a.g.stride * (long long)a.nx, ost = a.out.stride * (long long)a.nx;
  const uint32_t rprev = (rank + CL - 1) % CL, rnext = (rank + 1) % CL;
  const uint32_t r_loc = smem_u32(R), hb_loc = smem_u32(hb);
  const uint32_t p_R = mapa_shared(r_loc, rprev), n_R = mapa_shared(r_loc, rnext);
  const uint32_t p_hb = mapa_shared(hb_loc, rprev), n_hb = mapa_shared(hb_loc, rnext);
  const int q0 = MARG + EL + l0;                   // logical slot of point l0 (multiple of P)
  const int col = q0 / P;
  auto put = [&](double *b, const double(&x)[P]) {
#pragma unroll
    for (int p = 0; p < P; ++p) b[p * COLS + col] = x[p];
  };
  // R layout: [0, EL) = left halo l = -EL + q; [EL, EL+ER) = right halo l = Wc + (q - EL)
  auto send = [&](int j, const double(&x)[P]) {   // exchange j: own boundary points
    if (!own) return;
    const int rb = (j & 1) * CS::EMAX;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int l = l0 + p;
      if (l < ER)            // prev's right halo, slot EL + l
        st_async_f64(p_R + 8u * (uint32_t)(rb + EL + l), x[p], p_hb + 8u * (uint32_t)(j % 3));
      if (l >= Wc - EL)      // next's left halo, slot l - (Wc - EL)
        st_async_f64(n_R + 8u * (uint32_t)(rb + l - (Wc - EL)), x[p], n_hb + 8u * (uint32_t)(j % 3));
    }
  };
  const double *gpf = gb + gst;                    // rows of the next prefetch (step 1, 2, ...)
  const double *vpf = ob + ost;
  auto prefetch = [&](int i) {  // this thread's g_i (and v_i) points -> ring slot i % D
    if (i <= N && active) {
      double *gs = gring + (i % D) * GW + tid * P;
#pragma unroll
      for (int p = 0; p < P; p += 2) cp_async16(gs + p, gpf + p);
      if (own) {
        double *vs = vring + (i % D) * Wc + l0;
#pragma unroll
        for (int p = 0; p < P; p += 2) cp_async16(vs + p, vpf + p);
      }
    }
    gpf += gst;
    vpf += ost;
    cp_async_commit();
  };
  for (int q = tid; q < 2 * BL; q += nthr) smem[q] = 0.0;  // margins stay finite
  if (tid == 0) {
    for (int k = 0; k < 3; ++k) mbar_init(&hb[k], 1);
    fence_mbar_init();
    for (int k = 0; k < 3; ++k) mbar_expect_tx(&hb[k], hbytes);
  }
  double x[P];
#pragma unroll
  for (int p = 0; p < P; ++p) x[p] = (own && a.state_in) ? a.state_in[gx + p] : 0.0;
  for (int i = 1; i < D; ++i) prefetch(i);
  cluster.sync();  // buffers zeroed, barriers armed everywhere before any remote store
  if (own) put(smem, x);
  send(0, x);
  int j = 0, k = 0;                                // super-step j, local step k (1..S)
#pragma unroll 1
  for (int i = 1; i <= N; ++i) {
    double *cur = smem + ((i - 1) & 1) * BL, *nxt = smem + (i & 1) * BL;
    if (k == 0) {  // start of super-step j: halo threads take x_{jS} from R[j&1]
      if (lhalo || rhalo) {
        mbar_wait(&hb[j % 3], (uint32_t)((j / 3) & 1));
        const double *rj = R + (j & 1) * CS::EMAX + (lhalo ? EL + l0 : EL + (l0 - Wc));
        double h[P];
#pragma unroll
        for (int p = 0; p < P; ++p) h[p] = rj[p];
        put(cur, h);
      }
      if (tid == 0) mbar_expect_tx(&hb[j % 3], hbytes);  // re-arm for exchange j + 3
      __syncthreads();
    }
    ++k;
    prefetch(i + D - 1);
    cp_async_wait<D - 1>();                        // this thread's rows of step i landed
    if (active) {
      double y[P];
      if constexpr (NU4 <= 32) {
        psi_soa_dispatch<P, COLS, NU4>(cur, q0 + o0, a.op, y);
      } else {
        psi_soa_chunked<P, COLS>(cur, q0 + o0, a.op, y);
      }
      const double *gs = gring + (i % D) * GW + tid * P;
#pragma unroll
      for (int p = 0; p < P; ++p) x[p] = y[p] + gs[p];   // x_i = Psi x_{i-1} + g_i
      put(nxt, x);
      if (own) {
        if (k == S || i == N) send(j + 1, x);      // exact own values of x_{(j+1)S}
        const double *vs = vring + (i % D) * Wc + l0;
        double *orow = ob + (long long)i * ost;
#pragma unroll
        for (int p = 0; p < P; p += 2)             // u_i = v_i + e_i
          *reinterpret_cast<double2 *>(orow + p) = make_double2(vs[p] + x[p], vs[p + 1] + x[p + 1]);
      }
    }
    if (k == S) { k = 0; ++j; }
    __syncthreads();
  }
  cp_async_wait<0>();
  if (own && a.state_out) {
#pragma unroll
    for (int p = 0; p < P; ++p) a.state_out[gx + p] = x[p];
  }
  // the last exchange may still be landing here: wait for it, keep shared memory alive
  const int jl = k == 0 ? j : j + 1;
  if (tid == 0) mbar_wait(&hb[jl % 3], (uint32_t)((jl / 3) & 1));
  cluster.sync();
}

template <int NT, int P, int CL, int NU4>
static cudaError_t launch_seq_ca_nu(const CoarseArgs &a, int S, int nthr, cudaStream_t s) {
  const size_t smem = CaSmem<NT, P>::BYTES;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(psi_seq_cluster_ca_kernel<NT, P, CL, NU4>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (CL > 8)
      cudaFuncSetAttribute(psi_seq_cluster_ca_kernel<NT, P, CL, NU4>,
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  psi_seq_cluster_ca_kernel<NT, P, CL, NU4><<<CL, nthr, smem, s>>>(a, S);
  return cudaGetLastError();
}

template <int NT, int P, int CL>
static cudaError_t launch_seq_ca(const CoarseArgs &a, int S, cudaStream_t s) {
  const int o0 = a.op.o0, nu = a.op.nu;
  const int HL = o0 < 0 ? std::max(-o0, 1) : 1, HR = std::max(o0 + nu - 1, 1);
  const int EL = ((S * HL + P - 1) / P) * P, ER = ((S * HR + P - 1) / P) * P;
  const int nthr = NT + (((EL + ER) / P + 31) / 32) * 32;
  if (nu <= 12) return launch_seq_ca_nu<NT, P, CL, 12>(a, S, nthr, s);
  if (nu <= 16) return launch_seq_ca_nu<NT, P, CL, 16>(a, S, nthr, s);
  if (nu <= 20) return launch_seq_ca_nu<NT, P, CL, 20>(a, S, nthr, s);
  if (nu <= 24) return launch_seq_ca_nu<NT, P, CL, 24>(a, S, nthr, s);
  if (nu <= 28) return launch_seq_ca_nu<NT, P, CL, 28>(a, S, nthr, s);
  if (nu <= 32) return launch_seq_ca_nu<NT, P, CL, 32>(a, S, nthr, s);
  return launch_seq_ca_nu<NT, P, CL, 64>(a, S, nthr, s);
}

// Largest s-step depth S <= smax with EL + ER <= 256 (and EL, ER <= Wc); 0: not possible.
int seq_ca_depth(int cl, SweepCfg c, int nx, int o0, int nu, int smax) {
  if (cl < 2 || cl > 16 || cl * c.nt_threads * c.p != nx || c.p % 2) return 0;
  const int HL = o0 < 0 ? std::max(-o0, 1) : 1, HR = std::max(o0 + nu - 1, 1);
  const int Wc = c.nt_threads * c.p;
  for (int S = smax; S >= 2; --S) {
    const int EL = ((S * HL + c.p - 1) / c.p) * c.p, ER = ((S * HR + c.p - 1) / c.p) * c.p;
    if (EL + ER <= 256 && EL <= Wc && ER <= Wc && (EL + ER) / c.p <= 128) return S;
  }
  return 0;
}

cudaError_t launch_psi_seq_cluster_ca(int cl, SweepCfg c, int S, const CoarseArgs &a, cudaStream_t s) {
  if (a.nsteps <= 0) return cudaSuccess;
  if (cl == 8 && c.nt_threads == 64 && c.p == 2) return launch_seq_ca<64, 2, 8>(a, S, s);
  if (cl == 16 && c.nt_threads == 128 && c.p == 2) return launch_seq_ca<128, 2, 16>(a, S, s);
  if (cl == 8 && c.nt_threads == 256 && c.p == 2) return launch_seq_ca<256, 2, 8>(a, S, s);
  if (cl == 16 && c.nt_threads == 32 && c.p == 2) return launch_seq_ca<32, 2, 16>(a, S, s);
  if (cl == 8 && c.nt_threads == 128 && c.p == 4) return launch_seq_ca<128, 4, 8>(a, S, s);
  if (cl == 16 && c.nt_threads == 64 && c.p == 4) return launch_seq_ca<64, 4, 16>(a, S, s);
  if (cl == 8 && c.nt_threads == 32 && c.p == 4) return launch_seq_ca<32, 4, 8>(a, S, s);
  // wider rows (two-level solves beyond nx = 4096): 2048, 8192, 16384 points per cluster
  if (cl == 16 && c.nt_threads == 64 && c.p == 2) return launch_seq_ca<64, 2, 16>(a, S, s);
  if (cl == 16 && c.nt_threads == 128 && c.p == 4) return launch_seq_ca<128, 4, 16>(a, S, s);
  if (cl == 16 && c.nt_threads == 256 && c.p == 4) return launch_seq_ca<256, 4, 16>(a, S, s);
  return cudaErrorInvalidConfiguration;
}

// --------------------------------------------------------------------------
// Communication-avoiding cluster solve, warp-specialised ("lean step").  Same split,
// s-step halos and point-to-point DSMEM exchange as psi_seq_cluster_ca_kernel, but the
// compute warps' per-step instruction stream -- which sets the step latency of this
// sequential chain -- carries no global-memory work at all:
//  * a producer warp streams the g rows into a ring of 3 sets x 4 rows (extended region
//    EL+Wc+ER per row) with bulk copies, up to 12 steps ahead;
//  * the correction u_n = v_n + e_n is a bulk reduce-add of the own slice of e_n
//    into the C-row (which holds v_n): compute threads stage e_n in a 3 x 4-row ring, the
//    producer issues the reduce-adds and frees the set once they have read it;
//  * compute warps synchronise with a named barrier (the producer never joins it) and
//    meet the producer through mbarriers once per 4 steps: g set full / free, staging set
//    full / free;
//  * the stencil window's phase (o0 mod P) is a template parameter, fixed for the launch.
// Per step: window loads, NU4*P FMAs (2 partial sums), + g, publish, one named barrier.
template <int NT, int P> struct TbSmem {
  using CS = CaSmem<NT, P>;
  static constexpr int Wc = NT * P, GW = CS::EMAX + Wc, NS = 12;
  static constexpr size_t BYTES =
      sizeof(double) * (2 * (size_t)CS::BL + 2 * CS::EMAX + (size_t)NS * (GW + Wc)) + 128;
};

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  mg_jitter(8);
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int NT, int P, int CL, int NU4, int REM>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT + 160, 1)
    psi_seq_cluster_tb_kernel(const __grid_constant__ CoarseArgs a, int S) {
  static_assert(P % 2 == 0, "P even (16-byte rows)");
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  using CS = CaSmem<NT, P>;
  using TS = TbSmem<NT, P>;
  constexpr int Wc = CS::Wc, BL = CS::BL, COLS = CS::COLS, MARG = CS::MARG, GW = TS::GW;
  extern __shared__ __align__(128) double smem[];
  double *R = smem + 2 * BL;                        // receive buffers [2][EMAX]
  double *gring = R + 2 * CS::EMAX;                 // [12][GW]
  double *oring = gring + (size_t)TS::NS * GW;      // [12][Wc]
  uint64_t *hb = reinterpret_cast<uint64_t *>(oring + (size_t)TS::NS * Wc);  // [3] exchange
  uint64_t *gfull = hb + 3, *gfree = hb + 6, *ofull = hb + 9, *ofree = hb + 12;
  const uint32_t rank = cluster.block_rank();
  const int tid = threadIdx.x, nthr = blockDim.x, ncomp = nthr - 32;
  const bool producer = tid >= ncomp;
  const int N = a.nsteps, nx = a.nx, o0 = a.op.o0, nu = a.op.nu;
  const int H = (N + 3) / 4;                        // halves of 4 steps
  const int HL = o0 < 0 ? max(-o0, 1) : 1, HR = max(o0 + nu - 1, 1);
  const int EL = ((S * HL + P - 1) / P) * P, ER = ((S * HR + P - 1) / P) * P;
  const int GWa = EL + Wc + ER;                     // extended row length (even)
  const uint32_t hbytes = (uint32_t)(EL + ER) * 8u;
  const int l0 = -EL + tid * P;
  const bool active = !producer && l0 < Wc + ER;
  const bool own = !producer && l0 >= 0 && l0 < Wc;
  const bool lhalo = !producer && l0 < 0, rhalo = !producer && l0 >= Wc && active;
  // truncated Psi: the halo points of the first / last CTA lie beyond the row
  // ends; they hold zero at every step (whatever the wrap neighbour sends or g contains there)
  const bool ghost = a.trunc && ((rank == 0 && lhalo) || (rank == CL - 1 && rhalo));
  const int own0 = (int)rank * Wc;                  // global index of local point 0
  int gx = own0 + l0;
  if (gx < 0) gx += nx;
  if (gx >= nx) gx -= nx;
  int seg0 = own0 - EL;                             // extended segment start (periodic)
  if (seg0 < 0) seg0 += nx;
  const uint32_t rprev = (rank + CL - 1) % CL, rnext = (rank + 1) % CL;
  const uint32_t r_loc = smem_u32(R), hb_loc = smem_u32(hb);
  const uint32_t p_R = mapa_shared(r_loc, rprev), n_R = mapa_shared(r_loc, rnext);
  const uint32_t p_hb = mapa_shared(hb_loc, rprev), n_hb = mapa_shared(hb_loc, rnext);
  const int col = (MARG + tid * P) / P;             // SoA column of point l0
  const int wcol = (MARG + tid * P + o0 - REM) / P; // window column (phase REM = o0 mod P)
  auto put = [&](double *b, const double(&x)[P]) {
#pragma unroll
    for (int p = 0; p < P; ++p) b[p * COLS + col] = x[p];
  };
  auto send = [&](int j, const double(&x)[P]) {
    if (!own) return;
    const int rb = (j & 1) * CS::EMAX;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int l = l0 + p;
      if (l < ER)
        st_async_f64(p_R + 8u * (uint32_t)(rb + EL + l), x[p], p_hb + 8u * (uint32_t)(j % 3));
      if (l >= Wc - EL)
        st_async_f64(n_R + 8u * (uint32_t)(rb + l - (Wc - EL)), x[p], n_hb + 8u * (uint32_t)(j % 3));
    }
  };
  for (int q = tid; q < 2 * BL; q += nthr) smem[q] = 0.0;  // margins stay finite
  if (tid == 0) {
    for (int k = 0; k < 15; ++k) mbar_init(&hb[k], 1);
    fence_mbar_init();
    for (int k = 0; k < 3; ++k) mbar_expect_tx(&hb[k], hbytes);
  }
  double x[P];
#pragma unroll
  for (int p = 0; p < P; ++p) x[p] = (own && a.state_in) ? a.state_in[gx + p] : 0.0;
  cluster.sync();  // buffers zeroed, barriers armed everywhere before any remote store

  if (producer) {
    // ---- producer warp: lanes q = 0..3 handle row 4t+1+q of half t --------------------
    const int q = tid - ncomp;
    const int n1g = (seg0 + GWa <= nx) ? GWa : nx - seg0;
    // gate (speculative chain): rows up to 4t+4 needed -> floor(row / wait_every) + 1 chunks
    // of the producing sweep complete.  Lane 0 polls the flag (acquire, system scope: the
    // stream wrote it after the producing kernel completed); a proxy fence orders the bulk
    // copies (async proxy) behind it.  Rows only grow with t, so the gate of issue_g(t)
    // also covers the reduce-adds of the halves before it.
    int gate_done = 0;
    auto gate = [&](int t) {
      if (!a.wait_flag) return;
      const int row = min(N, 4 * t + 4);
      const int need = min(a.wait_chunks, row / a.wait_every + 1);
      if (need > gate_done) {
        mg_jitter(10);
        if (q == 0) {
          // The producing sweeps run concurrently on other SMs.  If kernels are being
          // serialised (a profiler's kernel replay, CUDA_LAUNCH_BLOCKING=1) they never run
          // while this kernel is resident: give up after 10 s with a launch failure instead
          // of hanging the GPU (use MGRIT_OPT_OVERLAP = C, 0 under such tools).
          unsigned long long v, t0, t1;
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
          do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a.wait_flag) : "memory");
            if (v < a.wait_base + (unsigned long long)need) {
              __nanosleep(256);
              asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
              if (t1 - t0 > 10000000000ull) __trap();
            }
          } while (v < a.wait_base + (unsigned long long)need);
        }
        __syncwarp();
        asm volatile("fence.proxy.async;" ::: "memory");
        gate_done = need;
      }
    };
    auto issue_g = [&](int t) {  // half t -> set t % 3
      gate(t);
      if (q == 0) mbar_expect_tx(&gfull[t % 3], (uint32_t)((min(N, 4 * t + 4) - 4 * t) * GWa) * 8u);
      __syncwarp();
      const int r = 4 * t + 1 + q;
      if (q < 4 && r <= N) {
        double *dst = gring + (size_t)((r - 1) % TS::NS) * GW;
        const double *src = a.g.base + (a.g.off + (a.n0 + r) * a.g.stride) * (long long)nx;
        tma_load_1d(dst, src + seg0, (uint32_t)n1g * 8u, &gfull[t % 3]);
        if (n1g < GWa) tma_load_1d(dst + n1g, src, (uint32_t)(GWa - n1g) * 8u, &gfull[t % 3]);
      }
    };
    for (int t = 0; t < 3 && t < H; ++t) issue_g(t);
    for (int t = 0; t < H; ++t) {
      // staging set of half t full -> reduce-add into out, free the set once read
      mbar_wait(&ofull[t % 3], (uint32_t)((t / 3) & 1));
      const int r = 4 * t + 1 + q;
      if (q < 4 && r <= N) {
        double *dst = const_cast<double *>(a.out.base) +
                      (a.out.off + (a.n0 + r) * a.out.stride) * (long long)nx + own0;
        tma_reduce_add_1d(dst, oring + (size_t)((r - 1) % TS::NS) * Wc, (uint32_t)Wc * 8u);
      }
      bulk_commit();
      bulk_wait_read_all();
      __syncwarp();
      if (q == 0) mbar_arrive(&ofree[t % 3]);
      // progress: rows <= n0 + 4(t+1) of this CTA's slice are complete in global memory once
      // the issuing lanes' bulk groups have completed (not only read); release at system
      // scope for the stream-ordered wait
      if (a.progress && (4 * (t + 1)) % a.prog_every == 0) {
        mg_jitter(9);
        bulk_wait_all();
        __syncwarp();
        if (q == 0) {
          __threadfence_system();
          atomicAdd_system(a.progress, 1ull);
        }
      }
      // g set of half t read by every compute thread -> reload it with half t + 3
      if (t + 3 < H) {
        mbar_wait(&gfree[t % 3], (uint32_t)((t / 3) & 1));
        issue_g(t + 3);
      }
    }
    bulk_wait_all();
  } else {
    // ---- compute warps ---------------------------------------------------------------
    if (own) put(smem, x);
    send(0, x);
    int j = 0, k = 0;                              // super-step j, local step k (1..S)
    int h = 0, kh = 0, slot = 0;                   // half h, step in the half, (i-1) % 12
#pragma unroll 1
    for (int i = 1; i <= N; ++i) {
      double *cur = smem + ((i - 1) & 1) * BL, *nxt = smem + (i & 1) * BL;
      if (k == 0) {  // start of super-step j: halo threads take x_{jS} from R[j&1]
        if (lhalo || rhalo) {
          mbar_wait(&hb[j % 3], (uint32_t)((j / 3) & 1));
          const double *rj = R + (j & 1) * CS::EMAX + (lhalo ? EL + l0 : EL + (l0 - Wc));
          double hv[P];
#pragma unroll
          for (int p = 0; p < P; ++p) hv[p] = ghost ? 0.0 : rj[p];
          put(cur, hv);
        }
        if (tid == 0) mbar_expect_tx(&hb[j % 3], hbytes);  // re-arm for exchange j + 3
        named_bar(1, ncomp);
      }
      ++k;
      if (kh == 0) {  // start of half h: hand half h-1's sets back, take half h's
        if (tid == 0 && h > 0) {
          mbar_arrive(&gfree[(h - 1) % 3]);
          mbar_arrive(&ofull[(h - 1) % 3]);
        }
        mbar_wait(&gfull[h % 3], (uint32_t)((h / 3) & 1));
        if (own && h >= 3) mbar_wait(&ofree[h % 3], (uint32_t)(((h - 3) / 3) & 1));
      }
      if (active) {
        double w[P + NU4 - 1];
        const double *s0 = cur + wcol;
#pragma unroll
        for (int r = 0; r < P + NU4 - 1; ++r) w[r] = s0[((REM + r) % P) * COLS + (REM + r) / P];
        double acc0[P], acc1[P];
#pragma unroll
        for (int p = 0; p < P; ++p) { acc0[p] = 0.0; acc1[p] = 0.0; }
#pragma unroll
        for (int qq = 0; qq < NU4; qq += 2) {
          const double c0 = a.op.psi[qq], c1 = a.op.psi[qq + 1];
#pragma unroll
          for (int p = 0; p < P; ++p) {
            acc0[p] = fma(c0, w[p + qq], acc0[p]);
            acc1[p] = fma(c1, w[p + qq + 1], acc1[p]);
          }
        }
        const double *gs = gring + (size_t)slot * GW + tid * P;
#pragma unroll
        for (int p = 0; p < P; ++p) x[p] = ghost ? 0.0 : (acc0[p] + acc1[p]) + gs[p];  // x_i = Psi x_{i-1} + g_i
        put(nxt, x);
        if (own) {
          double *os = oring + (size_t)slot * Wc + l0;
#pragma unroll
          for (int p = 0; p < P; ++p) os[p] = x[p];
          if (kh == 3 || i == N) fence_proxy_async();  // the half's staged rows -> async proxy
          if (k == S || i == N) send(j + 1, x);        // exact own values of x_{(j+1)S}
        }
      }
      if (k == S) { k = 0; ++j; }
      if (++kh == 4) { kh = 0; ++h; }
      if (++slot == TS::NS) slot = 0;
      named_bar(1, ncomp);
    }
    if (tid == 0) mbar_arrive(&ofull[(H - 1) % 3]);  // the last half is staged
    if (own && a.state_out) {
#pragma unroll
      for (int p = 0; p < P; ++p) a.state_out[gx + p] = x[p];
    }
    const int jl = k == 0 ? j : j + 1;
    if (tid == 0) mbar_wait(&hb[jl % 3], (uint32_t)((jl / 3) & 1));
  }
  cluster.sync();
}

template <int NT, int P, int CL, int NU4, int REM>
static cudaError_t launch_seq_tb_rem(const CoarseArgs &a, int S, int nthr, cudaStream_t s) {
  const size_t smem = TbSmem<NT, P>::BYTES;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(psi_seq_cluster_tb_kernel<NT, P, CL, NU4, REM>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (CL > 8)
      cudaFuncSetAttribute(psi_seq_cluster_tb_kernel<NT, P, CL, NU4, REM>,
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  psi_seq_cluster_tb_kernel<NT, P, CL, NU4, REM><<<CL, nthr, smem, s>>>(a, S);
  return cudaGetLastError();
}

template <int NT, int P, int CL, int NU4>
static cudaError_t launch_seq_tb_nu(const CoarseArgs &a, int S, int nthr, cudaStream_t s) {
  const int rem = ((a.op.o0 % P) + P) % P;
  if constexpr (P == 2) {
    if (rem == 0) return launch_seq_tb_rem<NT, P, CL, NU4, 0>(a, S, nthr, s);
    return launch_seq_tb_rem<NT, P, CL, NU4, 1>(a, S, nthr, s);
  } else {
    if (rem == 0) return launch_seq_tb_rem<NT, P, CL, NU4, 0>(a, S, nthr, s);
    if (rem == 1) return launch_seq_tb_rem<NT, P, CL, NU4, 1>(a, S, nthr, s);
    if (rem == 2) return launch_seq_tb_rem<NT, P, CL, NU4, 2>(a, S, nthr, s);
    return launch_seq_tb_rem<NT, P, CL, NU4, 3>(a, S, nthr, s);
  }
}

template <int NT, int P, int CL>
static cudaError_t launch_seq_tb(const CoarseArgs &a, int S, cudaStream_t s) {
  const int o0 = a.op.o0, nu = a.op.nu;
  const int HL = o0 < 0 ? std::max(-o0, 1) : 1, HR = std::max(o0 + nu - 1, 1);
  const int EL = ((S * HL + P - 1) / P) * P, ER = ((S * HR + P - 1) / P) * P;
  const int nthr = NT + (((EL + ER) / P + 31) / 32) * 32 + 32;  // + producer warp
  if (nu <= 10) return launch_seq_tb_nu<NT, P, CL, 10>(a, S, nthr, s);
  if (nu <= 12) return launch_seq_tb_nu<NT, P, CL, 12>(a, S, nthr, s);
  if (nu <= 16) return launch_seq_tb_nu<NT, P, CL, 16>(a, S, nthr, s);
  if (nu <= 32) return launch_seq_tb_nu<NT, P, CL, 32>(a, S, nthr, s);
  return cudaErrorInvalidValue;
}

// Same configurations / depth rule as the CA kernel (seq_ca_depth); windows up to 32 taps.
cudaError_t launch_psi_seq_cluster_tb(int cl, SweepCfg c, int S, const CoarseArgs &a, cudaStream_t s) {
  if (a.nsteps <= 0) return cudaSuccess;
  if (a.op.nu > 32) return cudaErrorInvalidValue;
  if (cl == 16 && c.nt_threads == 128 && c.p == 2) return launch_seq_tb<128, 2, 16>(a, S, s);
  if (cl == 16 && c.nt_threads == 32 && c.p == 2) return launch_seq_tb<32, 2, 16>(a, S, s);
  if (cl == 16 && c.nt_threads == 64 && c.p == 4) return launch_seq_tb<64, 4, 16>(a, S, s);
  if (cl == 16 && c.nt_threads == 128 && c.p == 4) return launch_seq_tb<128, 4, 16>(a, S, s);
  return cudaErrorInvalidConfiguration;
}

bool seq_cluster_tb_supported(int cl, SweepCfg c) {
  return cl == 16 && ((c.nt_threads == 128 && c.p == 2) || (c.nt_threads == 32 && c.p == 2) ||
                      (c.nt_threads == 64 && c.p == 4) || (c.nt_threads == 128 && c.p == 4));
}

// nx = CL * NT * P; the halos (-o0, o0+nu-1) must be <= 64 and <= NT*P (host-checked).
cudaError_t launch_psi_seq_cluster(int cl, SweepCfg c, const CoarseArgs &a, cudaStream_t s) {
  if (a.nsteps <= 0) return cudaSuccess;
  if (cl == 8 && c.nt_threads == 128 && c.p == 4) return launch_seq_cluster<128, 4, 8>(a, s);
  if (cl == 16 && c.nt_threads == 64 && c.p == 4) return launch_seq_cluster<64, 4, 16>(a, s);
  if (cl == 8 && c.nt_threads == 64 && c.p == 2) return launch_seq_cluster<64, 2, 8>(a, s);
  if (cl == 16 && c.nt_threads == 128 && c.p == 2) return launch_seq_cluster<128, 2, 16>(a, s);
  if (cl == 8 && c.nt_threads == 256 && c.p == 2) return launch_seq_cluster<256, 2, 8>(a, s);
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_psi_seq_periodic(SweepCfg c, const CoarseArgs &a, cudaStream_t s) {
  if (a.nsteps <= 0) return cudaSuccess;
  if (c.nt_threads == 32 && c.p == 2) return launch_seq_periodic<32, 2>(a, s);
  if (c.nt_threads == 32 && c.p == 4) return launch_seq_periodic<32, 4>(a, s);
  if (c.nt_threads == 32 && c.p == 8) return launch_seq_periodic<32, 8>(a, s);
  if (c.nt_threads == 64 && c.p == 8) return launch_seq_periodic<64, 8>(a, s);
  if (c.nt_threads == 128 && c.p == 8) return launch_seq_periodic<128, 8>(a, s);
  if (c.nt_threads == 256 && c.p == 8) return launch_seq_periodic<256, 8>(a, s);
  if (c.nt_threads == 512 && c.p == 8) return launch_seq_periodic<512, 8>(a, s);
  if (c.nt_threads == 1024 && c.p == 4) return launch_seq_periodic<1024, 4>(a, s);
  if (c.nt_threads == 256 && c.p == 4) return launch_seq_periodic<256, 4>(a, s);
  return cudaErrorInvalidConfiguration;
}

// --------------------------------------------------------------------------
template <int NT, int P>
__global__ void __launch_bounds__(NT, 1) psi_sweep_kernel(const __grid_constant__ PsiSweepArgs a) {
  constexpr int W = NT * P;
  extern __shared__ double smem[];
  constexpr int SP = Pad<P>::SP;
  double *sx = smem;
  double *sg = sx + PsiSmem<NT, P>::X;
  double *so = sg + PsiSmem<NT, P>::G;
  const int nx = a.nx, tid = threadIdx.x, m = a.m;
  const int item = blockIdx.x / a.ntiles;
  const int tile = blockIdx.x - item * a.ntiles;
  const int abeg = (int)(((long long)tile * nx) / a.ntiles);
  const int T = (int)(((long long)(tile + 1) * nx) / a.ntiles) - abeg;
  const int o0 = a.op.o0;
  const bool p2 = !a.interp && item < a.p2_items;
  // total steps in this CTA and the origin of step i: S_i = abeg + (N - i) o0
  const int N = a.interp ? (m - 1) : (p2 ? 2 * m : m);
  auto origin = [&](int i) { return wrapi((long long)abeg + (long long)(N - i) * o0, nx); };
  auto rowp = [&](const RowMap &r, long long j) {
    return r.base + (r.off + j * r.stride) * (long long)nx;
  };
  auto load = [&](const double *row, int S, double *s) {
    for (int q = tid; q < W; q += NT) {
      int g = S + q;
      if (g >= nx) g -= nx;
      s[pidx<P>(q)] = __ldg(row + g);
    }
  };
  // out[S..S+T) = (add ? add : 0) + x   (x staged through so)
  auto store = [&](double *row, const double *add, int S, const double(&v)[P]) {
    __syncthreads();
#pragma unroll
    for (int p = 0; p < P; ++p) so[tid * SP + p] = v[p];
    __syncthreads();
    for (int q = tid; q < T; q += NT) {
      int g = S + q;
      if (g >= nx) g -= nx;
      row[g] = add ? add[g] + so[pidx<P>(q)] : so[pidx<P>(q)];
    }
  };

  double x[P];
  if (a.u.base) {
    load(rowp(a.u, item), origin(0), sx);
    __syncthreads();
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = sx[tid * SP + p];
  } else {
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = 0.0;
  }
  const long long grow0 = a.g.off + (long long)item * a.g.stride;   // row jm
  if (a.interp) {
    const long long orow0 = a.out2.off + (long long)item * a.out2.stride;
    const long long vrow0 = a.v2.off + (long long)item * a.v2.stride;
    store(const_cast<double *>(a.out2.base) + orow0 * nx, a.v2.base ? a.v2.base + vrow0 * nx : nullptr,
          origin(0), x);
  }
  const int n1 = a.interp ? (m - 1) : m;
#pragma unroll 1
  for (int i = 1; i <= n1; ++i) {
    __syncthreads();
    psi_put<NT, P>(sx, x);
    load(a.g.base + (grow0 + i) * nx, origin(i), sg);
    __syncthreads();
    double y[P];
    psi_apply<P>(sx, tid * P, a.op, y);
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = y[p] + sg[tid * SP + p];
    if (a.interp) {
      const long long orow = a.out2.off + (long long)item * a.out2.stride + i;
      const long long vrow = a.v2.off + (long long)item * a.v2.stride + i;
      store(const_cast<double *>(a.out2.base) + orow * nx, a.v2.base ? a.v2.base + vrow * nx : nullptr,
            origin(i), x);
    }
  }
  if (a.interp) return;
  // v_{j+1}
  store(const_cast<double *>(rowp(a.v, item)), nullptr, origin(m), x);
  if (!p2) return;
  if (a.ucmp.base) {
    __syncthreads();
    load(rowp(a.ucmp, item), origin(m), sg);
    __syncthreads();
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] -= sg[tid * SP + p];
  }
#pragma unroll 1
  for (int i = m + 1; i <= 2 * m; ++i) {
    __syncthreads();
    psi_put<NT, P>(sx, x);
    __syncthreads();
    psi_apply<P>(sx, tid * P, a.op, x);
  }
  store(const_cast<double *>(rowp(a.r2, item)), nullptr, origin(2 * m), x);
}

// --------------------------------------------------------------------------
// Tile-mode level kernel (odd P => contiguous shared windows) with bulk-copy I/O.
// All rows an item needs (g rows, u_j, u_{j+1}, v2 rows) are requested by one
// thread at CTA start (1-2 TMA copies each, completion on one mbarrier per row)
// so HBM streaming overlaps the Psi steps; outputs leave through two alternating
// staging buffers with bulk stores (unaligned ends by scalar stores).  Windows
// start at the even address below the step origin; `off` = origin & 1.
// --------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void psi_apply_c(const double *__restrict__ s, int base,
                                            const PsiOp &op, double (&out)[P]) {
  const double *sp = s + base;
  double w[P + 3];
#pragma unroll
  for (int r = 0; r < P + 3; ++r) w[r] = sp[r];
#pragma unroll
  for (int p = 0; p < P; ++p) out[p] = 0.0;
  const int nu = op.nu, nu4 = nu & ~3;
  int q0 = 0;
#pragma unroll 1
  for (; q0 < nu4; q0 += 4) {
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const double c = op.psi[q0 + qq];
#pragma unroll
      for (int p = 0; p < P; ++p) out[p] = fma(c, w[p + qq], out[p]);
    }
#pragma unroll
    for (int r = 0; r + 4 < P + 3; ++r) w[r] = w[r + 4];
#pragma unroll
    for (int r = P - 1; r < P + 3; ++r) w[r] = sp[q0 + 4 + r];
  }
#pragma unroll 1
  for (; q0 < nu; ++q0) {
    const double c = op.psi[q0];
#pragma unroll
    for (int p = 0; p < P; ++p) out[p] = fma(c, w[p], out[p]);
#pragma unroll
    for (int r = 0; r < P + 2; ++r) w[r] = w[r + 1];
    w[P + 2] = sp[q0 + P + 3];
  }
}

// Publish a thread's P values of a shifted-coordinate window.  No periodic tail: the
// windows are tiles (W <= nx, T <= W - halo), and the reads past W only feed outputs
// beyond the valid length, which shrinks by nu-1 per step.
template <int P>
__device__ __forceinline__ void psi_put_window(double *s, const double (&x)[P]) {
  double *st = s + threadIdx.x * P;
#pragma unroll
  for (int p = 0; p < P; ++p) st[p] = x[p];
}

// Compile-time tap count: the thread's whole input window (P + NU - 1 values) is read
// once from shared memory and the NU*P FMAs run from registers.
template <int P, int NU>
__device__ __forceinline__ void psi_apply_fixed(const double *__restrict__ s, int base,
                                                const PsiOp &op, double (&out)[P]) {
  const double *sp = s + base;
  double w[P + NU - 1];
#pragma unroll
  for (int r = 0; r < P + NU - 1; ++r) w[r] = sp[r];
#pragma unroll
  for (int p = 0; p < P; ++p) out[p] = 0.0;
#pragma unroll
  for (int q = 0; q < NU; ++q) {
    const double c = op.psi[q];
#pragma unroll
    for (int p = 0; p < P; ++p) out[p] = fma(c, w[p + q], out[p]);
  }
}

template <int P, int NU>
__device__ __forceinline__ void psi_apply_any(const double *s, int base, const PsiOp &op,
                                              double (&out)[P]) {
  if constexpr (NU > 0)
    psi_apply_fixed<P, NU>(s, base, op, out);
  else
    psi_apply_c<P>(s, base, op, out);
}

template <int NT, int P> struct LevelSmem {
  static constexpr int W = NT * P;
  static constexpr int WB = W + 2;                 // even
  static constexpr int X = (W + PSI_EXT + 1) & ~1;
  static constexpr int NROW_MAX = 8;
  static size_t bytes(int nrow) { return sizeof(double) * (2 * X + (size_t)nrow * WB + 2 * NROW_MAX) + 64; }
};

// Rows of an item (slots, dense):
//   sweep : g rows jm+1..jm+m, then u_{j+1} (if ucmp), then u_j (if u)
//   interp: u_j, g rows jm+1..jm+m-1, v2 rows jm+i (i = 0..m-1, if v2)
// Output staging reuses consumed row buffers: v_{j+1} -> slot of g_1, r_{j+2} -> slot of
// g_2, interpolated rows in place of their v2 row.
template <int NT, int P, int NU>
__global__ void __launch_bounds__(NT, 1) psi_level_kernel(const __grid_constant__ PsiSweepArgs a) {
  static_assert(P % 2 == 1, "contiguous windows need odd P");
  using L = LevelSmem<NT, P>;
  constexpr int W = L::W, WB = L::WB;
  extern __shared__ __align__(128) double smem[];
  double *X = smem;             // two state buffers (ping-pong): one barrier per step
  double *RB = smem + 2 * L::X;
  const int nx = a.nx, tid = threadIdx.x, m = a.m;
  const bool interp = a.interp != 0;
  const int nrow = interp ? m : (m + (a.ucmp.base ? 1 : 0) + (a.u.base ? 1 : 0));
  uint64_t *bar = reinterpret_cast<uint64_t *>(RB + nrow * WB);
  const int item = blockIdx.x / a.ntiles;
  const int tile = blockIdx.x - item * a.ntiles;
  const int half = nx >> 1;
  const int abeg = 2 * (int)(((long long)tile * half) / a.ntiles);
  const int T = 2 * (int)(((long long)(tile + 1) * half) / a.ntiles) - abeg;
  const int o0 = a.op.o0;
  const bool p2 = !interp && item < a.p2_items;
  const int N = interp ? (m - 1) : (p2 ? 2 * m : m);
  auto origin = [&](int i) { return wrapi((long long)abeg + (long long)(N - i) * o0, nx); };
  auto rowp = [&](const RowMap &r, long long j) {
    return r.base + (r.off + j * r.stride) * (long long)nx;
  };
  const long long g0 = a.g.off + (long long)item * a.g.stride;
  const int k_ucmp = m, k_u = m + (a.ucmp.base ? 1 : 0);
  auto slot_row = [&](int k, const double *&row, int &S) {
    if (!interp) {
      if (k < m) { row = a.g.base + (g0 + k + 1) * nx; S = origin(k + 1); }
      else if (a.ucmp.base && k == k_ucmp) { row = rowp(a.ucmp, item); S = origin(m); }
      else { row = rowp(a.u, item); S = origin(0); }
      return;
    }
    if (k == 0) { row = rowp(a.u, item); S = origin(0); }
    else { row = a.g.base + (g0 + k) * nx; S = origin(k); }
  };
  // lane k of warp 0 requests row k (in parallel: a serial issue loop by one thread held
  // every warp of the CTA at the barrier below for ~15 % of the kernel's time)
  if (tid < nrow) {
    const int k = tid;
    mbar_init(&bar[k], 1);
    fence_mbar_init();
    const double *row;
    int S;
    slot_row(k, row, S);
    if (interp || p2 || !a.ucmp.base || k != k_ucmp) {  // else: not needed
      const int S0 = S & ~1;
      const int n1 = (S0 + WB <= nx) ? WB : nx - S0;
      mbar_expect_tx(&bar[k], (uint32_t)WB * 8u);
      tma_load_1d(RB + k * WB, row + S0, (uint32_t)n1 * 8u, &bar[k]);
      if (n1 < WB) tma_load_1d(RB + k * WB + n1, row, (uint32_t)(WB - n1) * 8u, &bar[k]);
    }
  }
  __syncthreads();
  auto slot = [&](int k, int S) -> double * {  // element q of slot k's window at origin S
    mbar_wait(&bar[k], 0);
    return RB + k * WB + (S & 1);
  };
  // parity of origin(i) (abeg and nx are even): all the step loop needs to find a slot
  auto opar = [&](int i) { return ((N - i) * o0) & 1; };
  // out[S .. S+T) = v[q]  (or out += v[q] with `acc`: bulk reduce-add at L2), staged in
  // buffer `buf`, a consumed row.  No barrier before staging: each thread overwrites only
  // buffer positions it read itself in this step (same origin), or positions of a row
  // consumed at least one barrier ago.
  auto store = [&](double *row, int S, const double(&v)[P], bool acc, double *buf) {
    const int so = S & 1;
    double *st = buf + so;
#pragma unroll
    for (int p = 0; p < P; ++p) st[tid * P + p] = v[p];
    fence_proxy_async();
    __syncthreads();
    int segs[2][2];
    int ns = 1;
    if (S + T <= nx) { segs[0][0] = S; segs[0][1] = S + T; }
    else { segs[0][0] = S; segs[0][1] = nx; segs[1][0] = 0; segs[1][1] = S + T - nx; ns = 2; }
    int scalar = 0;
    for (int k = 0; k < ns; ++k) {
      int ga = segs[k][0], gb = segs[k][1];
      const int base = so + (k == 0 ? -S : nx - S);   // buffer index of global g = base + g
      if (ga < gb && (ga & 1)) {
        if (tid == 1 + scalar) row[ga] = acc ? row[ga] + buf[base + ga] : buf[base + ga];
        ++scalar;
        ++ga;
      }
      if (ga < gb && ((gb - ga) & 1)) {
        if (tid == 1 + scalar)
          row[gb - 1] = acc ? row[gb - 1] + buf[base + gb - 1] : buf[base + gb - 1];
        ++scalar;
        --gb;
      }
      if (tid == 0 && gb > ga) {
        if (acc) tma_reduce_add_1d(row + ga, buf + base + ga, (uint32_t)(gb - ga) * 8u);
        else tma_store_1d(row + ga, buf + base + ga, (uint32_t)(gb - ga) * 8u);
      }
    }
    if (tid == 0) bulk_commit();
  };

  double x[P];
  if (a.u.base) {
    const double *su = slot(interp ? 0 : k_u, origin(0));
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = su[tid * P + p];
  } else {
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = 0.0;
  }
  if (interp)  // out[jm] += u_j  (staged in place of the consumed u row)
    store(const_cast<double *>(a.out2.base) + (a.out2.off + (long long)item * a.out2.stride) * nx,
          origin(0), x, true, RB);
  const int n1 = interp ? (m - 1) : m;
  int sx = 0;
  // One Psi step: publish x in X[sx&1], one barrier, read the neighbours' values.  The
  // buffer written next was last read two steps ago, before the previous barrier.
  auto psi_step = [&](double(&y)[P]) {
    double *Xb = X + (sx & 1) * L::X;
    psi_put_window<P>(Xb, x);
    __syncthreads();
    psi_apply_any<P, NU>(Xb, tid * P, a.op, y);
    ++sx;
  };
#pragma unroll 1
  for (int i = 1; i <= n1; ++i) {
    double y[P];
    psi_step(y);
    const int kg = interp ? i : i - 1;
    const double *sg = slot(kg, opar(i));
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = y[p] + sg[tid * P + p];
    if (interp)  // out[jm+i] += x_i  (staged in place of the consumed g row)
      store(const_cast<double *>(a.out2.base) +
                (a.out2.off + (long long)item * a.out2.stride + i) * nx,
            origin(i), x, true, RB + kg * WB);
  }
  if (!interp) {
    store(const_cast<double *>(rowp(a.v, item)), origin(m), x, false, RB);  // slot of g_1
    if (p2) {
      if (a.ucmp.base) {
        const double *sc = slot(k_ucmp, opar(m));
#pragma unroll
        for (int p = 0; p < P; ++p) x[p] -= sc[tid * P + p];
      }
#pragma unroll 1
      for (int i = m + 1; i <= 2 * m; ++i) {
        double y[P];
        psi_step(y);
#pragma unroll
        for (int p = 0; p < P; ++p) x[p] = y[p];
      }
      store(const_cast<double *>(rowp(a.r2, item)), origin(2 * m), x, false,
            RB + (m >= 2 ? 1 : 0) * WB);  // slot of g_2
    }
  }
  if (tid == 0) bulk_wait_all();
}

template <int NT, int P, int NU>
static cudaError_t launch_level_one(const PsiSweepArgs &a, cudaStream_t s) {
  using L = LevelSmem<NT, P>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(psi_level_kernel<NT, P, NU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)L::bytes(L::NROW_MAX));
    cudaFuncSetAttribute(psi_level_kernel<NT, P, NU>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  const int m = a.m;
  const int nrow = a.interp ? m : (m + (a.ucmp.base ? 1 : 0) + (a.u.base ? 1 : 0));
  const long long grid = (long long)a.nitems * a.ntiles;
  if (grid <= 0) return cudaSuccess;
  psi_level_kernel<NT, P, NU><<<(unsigned)grid, NT, L::bytes(nrow), s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_psi_level_tma(SweepCfg c, const PsiSweepArgs &a, cudaStream_t s) {
  if (a.m > 4 || (a.nx & 1)) return cudaErrorInvalidValue;
  if (c.nt_threads != 128 || c.p != 9) return cudaErrorInvalidConfiguration;
  switch (a.op.nu) {
    case 9: return launch_level_one<128, 9, 9>(a, s);
    case 13: return launch_level_one<128, 9, 13>(a, s);
    case 17: return launch_level_one<128, 9, 17>(a, s);
    case 21: return launch_level_one<128, 9, 21>(a, s);
    case 25: return launch_level_one<128, 9, 25>(a, s);
    default: return launch_level_one<128, 9, 0>(a, s);
  }
}

// --------------------------------------------------------------------------
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) reduce_kernel(const double *__restrict__ p, long long n,
                                                      double *out) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += 1024) s += p[i];
  s = block_sum<1024>(s, red);
  if (threadIdx.x == 0) out[0] = s;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// One CTA per row chunk: blockIdx.y strides over rows, threads over the row's points (two
// per thread, 16-byte stores), so there is no per-element 64-bit division.
__global__ void fill_guess_kernel(double *dst, long long row0, long long rows, int nx,
                                  uint64_t seed, int lo_kind, const double *u0) {
  auto value = [&](long long n, int i) {
    if (n == 0 && u0) return u0[i];
    const uint64_t idx = (uint64_t)n * (uint64_t)nx + (uint64_t)i;
    const uint64_t k = splitmix64(idx + seed * 0x632BE59BD9B4E019ull) >> 11;
    return lo_kind == 0 ? (double)((long long)k - (1ll << 52)) * 0x1p-52 : (double)k * 0x1p-53;
  };
  const bool pairs = (nx & 1) == 0;
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    const long long n = row0 + r;
    double *row = dst + r * (long long)nx;
    if (pairs) {
      for (int i = 2 * threadIdx.x; i < nx; i += 2 * blockDim.x)
        *reinterpret_cast<double2 *>(row + i) = make_double2(value(n, i), value(n, i + 1));
    } else {
      for (int i = threadIdx.x; i < nx; i += blockDim.x) row[i] = value(n, i);
    }
  }
}

// --------------------------------------------------------------------------
#define MG_PSI_CFGS(X) \
  X(32, 2) X(32, 4) X(32, 8) X(64, 8) X(128, 8) X(256, 8) X(512, 8)

template <int NT, int P, int R, int NU>
static cudaError_t launch_coarse_ring(const CoarseArgs &a, cudaStream_t s) {
  const size_t smem = sizeof(double) * CoarseSmem<NT, P, R>::TOTAL;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(psi_coarse_kernel<NT, P, R, NU>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  psi_coarse_kernel<NT, P, R, NU><<<a.ntiles, NT, smem, s>>>(a);
  return cudaGetLastError();
}

// ring depth: 8 slots where shared memory allows, else 4.  The V-cycle coarsest level of
// the cfg5 hierarchy (256 x 8 tiles) gets compile-time tap counts (nu_l = 9 .. 25).
template <int NT, int P>
static cudaError_t launch_coarse_one(const CoarseArgs &a, cudaStream_t s) {
  if constexpr (sizeof(double) * CoarseSmem<NT, P, 8>::TOTAL <= 220 * 1024) {
    if constexpr (NT == 256 && P == 8) {
      switch (a.op.nu) {
        case 9: return launch_coarse_ring<NT, P, 8, 9>(a, s);
        case 13: return launch_coarse_ring<NT, P, 8, 13>(a, s);
        case 17: return launch_coarse_ring<NT, P, 8, 17>(a, s);
        case 21: return launch_coarse_ring<NT, P, 8, 21>(a, s);
        case 25: return launch_coarse_ring<NT, P, 8, 25>(a, s);
        default: break;
      }
    }
    return launch_coarse_ring<NT, P, 8, 0>(a, s);
  } else {
    return launch_coarse_ring<NT, P, 4, 0>(a, s);
  }
}

template <int NT, int P>
static cudaError_t launch_psisweep_one(const PsiSweepArgs &a, cudaStream_t s) {
  const size_t smem = sizeof(double) * PsiSmem<NT, P>::TOTAL;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(psi_sweep_kernel<NT, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  const long long grid = (long long)a.nitems * a.ntiles;
  if (grid <= 0) return cudaSuccess;
  psi_sweep_kernel<NT, P><<<(unsigned)grid, NT, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_psi_coarse(SweepCfg c, const CoarseArgs &a, cudaStream_t s) {
  if (a.nsteps <= 0) return cudaSuccess;
#define MG_CASE(NT_, P_) \
  if (c.nt_threads == NT_ && c.p == P_) return launch_coarse_one<NT_, P_>(a, s);
  MG_PSI_CFGS(MG_CASE)
#undef MG_CASE
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_psi_sweep(SweepCfg c, const PsiSweepArgs &a, cudaStream_t s) {
#define MG_CASE(NT_, P_) \
  if (c.nt_threads == NT_ && c.p == P_) return launch_psisweep_one<NT_, P_>(a, s);
  MG_PSI_CFGS(MG_CASE)
#undef MG_CASE
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_rk_coarse(int scheme, SweepCfg c, const RKCoarseArgs &a, cudaStream_t s) {
  switch (scheme) {
    case 0: return launch_rkc<ERK1U1>(c, a, s);
    case 1: return launch_rkc<ERK2U2>(c, a, s);
    case 2: return launch_rkc<ERK3U3>(c, a, s);
    case 3: return launch_rkc<ERK4U4>(c, a, s);
    case 4: return launch_rkc<ERK5U5>(c, a, s);
    case 5: return launch_rkc<SDIRK1U1>(c, a, s);
    case 6: return launch_rkc<SDIRK2U2>(c, a, s);
    case 7: return launch_rkc<SDIRK3U3>(c, a, s);
    case 8: return launch_rkc<SDIRK4U4>(c, a, s);
    default: return cudaErrorInvalidValue;
  }
}

// Deterministic two-pass sum: pass 1 sums fixed contiguous chunks (one block each), pass 2
// sums the chunk results in order (same value for the same input, any launch timing).
__global__ void __launch_bounds__(256) reduce_chunks_kernel(const double *__restrict__ p, long long n,
                                                            long long chunk, double *part) {
  __shared__ double red[8];
  const long long b0 = blockIdx.x * chunk, b1 = b0 + chunk < n ? b0 + chunk : n;
  double s = 0.0;
  for (long long i = b0 + threadIdx.x; i < b1; i += 256) s += p[i];
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

cudaError_t launch_reduce(const double *partials, long long n, double *out, cudaStream_t s) {
  constexpr long long kChunks = 512;
  if (n <= 65536) {
    reduce_kernel<<<1, 1024, 0, s>>>(partials, n, out);
    return cudaGetLastError();
  }
  const long long chunk = (n + kChunks - 1) / kChunks;
  // chunk sums go to out[1 .. kChunks] (the caller's scalar area holds >= 64 doubles;
  // the partials buffer tail is used instead to stay in bounds)
  double *tmp = const_cast<double *>(partials) + n;  // workspace reserves room after n
  reduce_chunks_kernel<<<(unsigned)kChunks, 256, 0, s>>>(partials, n, chunk, tmp);
  reduce_kernel<<<1, 1024, 0, s>>>(tmp, kChunks, out);
  return cudaGetLastError();
}

cudaError_t launch_fill_guess(double *dst, long long row0, long long rows, int nx, uint64_t seed,
                              int lo_kind, const double *u0, cudaStream_t s) {
  if (rows <= 0 || nx <= 0) return cudaSuccess;
  long long blocks = rows < 148 * 32 ? rows : 148 * 32;
  fill_guess_kernel<<<(unsigned)blocks, 256, 0, s>>>(dst, row0, rows, nx, seed, lo_kind, u0);
  return cudaGetLastError();
}

}  // namespace mg
