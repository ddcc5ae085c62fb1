// kernels.h — host-visible launch interfaces of the MGRIT kernels (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "sdirk.cuh"

namespace mg {

// Row addressing: row(j) = base + (off + j*stride) * nx.  base == nullptr disables.
struct RowMap {
  const double *base;
  long long off;
  long long stride;
};

// ---- RK sweep (fine level, fixed coordinates, halo tiles or whole periodic rows) ----
struct SweepArgs {
  int nx;
  int nitems;      // items (intervals or rows) j = 0..nitems-1
  int ntiles;      // spatial tiles per item (1 = whole periodic row)
  int HL;          // left halo (points) of the window in tile mode
  int nsteps1;     // phase-1 steps of Phi
  int nsteps2;     // phase-2 steps (applied to delta), 0 = none
  int p2_items;    // phase 2 only for items j < p2_items
  int load_after;  // TMA kernel: issue the next item's prefetch after this phase-1 step
  int defer_v;     // TMA kernel: store v_{j+1} together with r_{j+2} (one fence per item)
  int each_first;  // write phase-1 states i = each_first..each_last into `each` rows
  int each_last;   //   (each_last < each_first: none); i = 0 is the input state
  long long each_step;  // row(j,i) = each.base + (each.off + j*each.stride + i*each_step)*nx
  RowMap in;       // input state (base null: zero)
  RowMap cmp;      // delta = x - cmp (base null: no delta)
  RowMap endw;     // store the phase-1 result
  RowMap each;
  RowMap dstore;   // store delta of item j at row (j+d_phase)/d_every if divisible
  int d_every, d_phase;
  RowMap r2;       // phase-2 result
  double *partials;  // [nitems*ntiles] sum(delta^2) over each tile's own outputs
  RKCoeffs co;
  SdirkCoef sd;      // implicit schemes: factored periodic stage solve (sdirk.cuh)
  // inflow/outflow rows (bounded.cu): compact forcing rows b_n (FORC_LD doubles each, nb
  // used); phase-1 step i of item j adds row f_off + j*f_stride + i - 1 (null: homogeneous)
  const double *forc;
  int nb;
  long long f_off, f_stride;
  // SMs left free for a concurrently running kernel (the overlapped two-level coarse
  // solve's 16-CTA cluster): the persistent grid is sized for sms - reserve_sms
  int reserve_sms;
  // at most this many CTAs per SM in the persistent grid (0: what fits), leaving registers
  // and shared memory to a concurrent kernel (the overlapped V-cycle's level kernels)
  int max_per_sm;
};
constexpr int FORC_LD = 24;   // >= S*NL of every explicit scheme (ERK5+U5: 18)

struct SweepCfg {
  int nt_threads;  // NT
  int p;           // points per thread
  int minb = 0;    // TMA kernel: __launch_bounds__ min blocks per SM (0 = default)
};

// scheme: 0 ERK1U1, 1 ERK2U2, 2 ERK3U3, 3 ERK4U4, 4 ERK5U5, 5 SDIRK1U1 .. 8 SDIRK4U4
cudaError_t launch_rk_sweep(int scheme, SweepCfg cfg, const SweepArgs &a, cudaStream_t s);
bool rk_sweep_supported(int scheme, SweepCfg cfg);
// Persistent TMA-pipelined sweep for halo-tile mode (odd P, even nx; no per-step writes).
// Tile boundaries are 2*floor(t*(nx/2)/ntiles); HL must be even.
cudaError_t launch_rk_sweep_tma(int scheme, SweepCfg cfg, const SweepArgs &a, cudaStream_t s);
// All-row residual of consecutive rows in.row(n-1) -> in.row(n), n = 1..a.nitems, in
// (tile, chunk-of-rows) work items; one per-warp partial per item.
cudaError_t launch_rk_residual_tma(int scheme, SweepCfg cfg, const SweepArgs &a, int chunk,
                                   cudaStream_t s);
int rk_scheme_reach_left(int scheme);
int rk_scheme_reach_right(int scheme);
int rk_scheme_stages(int scheme);
bool rk_scheme_implicit(int scheme);

// ---- Stencil (Psi) kernels in shifted coordinates ----
constexpr int MAX_PSI = 64;
struct PsiOp {
  int nu;        // taps, contiguous offsets o0 .. o0+nu-1
  int o0;
  double psi[MAX_PSI];
};

// Sequential (coarsest-level) solve over steps n0+1..n0+nsteps of
//   x_n = Psi x_{n-1} + g_n,   out_n += x_n      (out holds v_n)
// in trapezoid tiles (no inter-CTA communication inside a launch).
struct CoarseArgs {
  int nx, ntiles, nsteps;
  long long n0;
  RowMap g;        // g row n  (n = n0+i)
  RowMap out;      // out row n (accumulated)
  const double *state_in;  // x_{n0} (nx), null: zero
  double *state_out;       // x_{n0+nsteps} (nx), null: not stored
  // progress counter (psi_seq_cluster_tb_kernel; null: none): every CTA of the cluster adds 1
  // once its slice of the rows out_n, n <= n0 + k*prog_every, is complete in global memory
  // (k = 1, 2, ...); a stream-ordered cuStreamWaitValue64 releases dependent work
  unsigned long long *progress;
  int prog_every;          // steps per publication (multiple of 4, divides nsteps)
  // input gate of a chain launched ahead of its inputs (speculative chain of the next
  // iteration): the rows g_n, out_n with n <= k*wait_every - 1 may be touched
  // once *wait_flag >= wait_base + k (all rows once it is >= wait_base + wait_chunks); the
  // flag is written by the stream after each producer kernel (cuStreamWriteValue64)
  const unsigned long long *wait_flag;
  unsigned long long wait_base;
  int wait_every, wait_chunks;
  // 1: Psi truncated at the row ends (Toeplitz, no wrap; inflow/outflow rows, bounded.cu):
  // psi_seq_cluster_tb_kernel keeps the halo points beyond the row ends at zero
  int trunc;
  PsiOp op;
};
cudaError_t launch_psi_coarse(SweepCfg cfg, const CoarseArgs &a, cudaStream_t s);
// Periodic whole-row single-CTA variant (NT*P == nx), fixed coordinates, per-thread
// cp.async streaming of g and out rows.
cudaError_t launch_psi_seq_periodic(SweepCfg cfg, const CoarseArgs &a, cudaStream_t s);
// Thread-block-cluster variant: the row split over `cl` CTAs (DSMEM halos, one cluster
// barrier per step).  nx == cl * NT * P.
cudaError_t launch_psi_seq_cluster(int cl, SweepCfg cfg, const CoarseArgs &a, cudaStream_t s);
bool seq_cluster_ok(int cl, SweepCfg cfg, int nx, int o0, int nu);
// Communication-avoiding variant: S steps per halo exchange (extended halos S*HL, S*HR).
cudaError_t launch_psi_seq_cluster_ca(int cl, SweepCfg cfg, int S, const CoarseArgs &a, cudaStream_t s);
int seq_ca_depth(int cl, SweepCfg cfg, int nx, int o0, int nu, int smax);
// Same split and s-step halos with batched TMA I/O (g ring, reduce-add correction), the
// launch's window phase as a template parameter; nu <= 32.
cudaError_t launch_psi_seq_cluster_tb(int cl, SweepCfg cfg, int S, const CoarseArgs &a, cudaStream_t s);
bool seq_cluster_tb_supported(int cl, SweepCfg cfg);

// Level-l (l >= 2) relaxation sweep of the V-cycle with Psi_l and RHS g (u = 0 start):
//   phase 1: x_i = Psi x_{i-1} + g[jm+i], i=1..m, x_0 = u_j (null: 0) -> v_{j+1}
//   delta = x_m - u_{j+1} (null: x_m); phase 2: m homogeneous steps -> r_{j+2}.
// Interp mode: x_0 = u_j, x_i = Psi x_{i-1} + g[jm+i] for i = 1..m-1,
//   out[jm+i] = v2[jm+i] + x_i for i = 0..m-1.
struct PsiSweepArgs {
  int nx, nitems, ntiles, m;
  int interp;
  RowMap u;        // level-l C-rows (null: zero)
  RowMap ucmp;     // u_{j+1} (null: zero)
  RowMap g;        // level-l rhs rows, row(j) = base + (off + j*stride) and + i
  RowMap v;        // v_{j+1}
  RowMap r2;       // r_{j+2}
  int p2_items;
  RowMap v2;       // interp: addend rows of level l-1 (row jm+i) (periodic kernel)
  RowMap out2;     // interp: output rows of level l-1 (row jm+i)
  int accumulate;  // interp (TMA kernel): out2 += x (bulk reduce-add), v2 unused
  PsiOp op;
};
cudaError_t launch_psi_sweep(SweepCfg cfg, const PsiSweepArgs &a, cudaStream_t s);
// Tile-mode variant with bulk-copy I/O (odd P, even nx, m <= 4); even tile boundaries.
cudaError_t launch_psi_level_tma(SweepCfg cfg, const PsiSweepArgs &a, cudaStream_t s);

// RK-form coarse operator (IDEAL = q fine steps, REDISC = one step at CFL m*c),
// sequential over nsteps, whole periodic row, one CTA.
struct RKCoarseArgs {
  int nx, nsteps, q;
  int ring_b;        // > 0: g / v rows through a shared-memory block ring of ring_b steps (set by the launcher)
  RowMap g, v, out;
  RKCoeffs co;
  SdirkCoef sd;      // implicit schemes: the coarse step's factored stage solve
};
cudaError_t launch_rk_coarse(int scheme, SweepCfg cfg, const RKCoarseArgs &a, cudaStream_t s);

// ---- Inflow/outflow boundaries (bounded.cu; PAPER.md 4.5, R20) ----
// Host-derived tables of the inflow closure: t1[q][i] = dt^q (A^q 1)_i, t2[k][j] =
// (k dx/alpha)^j / j!; z, A, b as in RKCoeffs; p = order of U_p, nq = p + S derivatives
// g^(0..nq-1)(t_n) per time step.
struct BndCoef {
  int S, NL, NR, p, nq;
  double t1[MAXS][MAXS];
  double t2[4][MAXS];
  double z[MAXZ];
  double A[MAXS][MAXS];
  double b[MAXS];
};
// b_n = Phi(0; t_n), n = 0..nt-1, from dg (nt x nq, device) into forc (nt x FORC_LD, device).
cudaError_t launch_bnd_forcing(const BndCoef &c, const double *dg, long long nt, double *forc,
                               cudaStream_t s);
// Whole-row sweep with the boundary closures (explicit schemes; NT*P == nx, P >= p + 1).
cudaError_t launch_rk_sweep_bnd(int scheme, SweepCfg cfg, const SweepArgs &a, cudaStream_t s);
bool rk_sweep_bnd_supported(int scheme, SweepCfg cfg);
cudaError_t launch_rk_coarse_bnd(int scheme, SweepCfg c, const RKCoarseArgs &a, cudaStream_t s);
// Truncated-Toeplitz Psi: sequential solve (CoarseArgs semantics, out accumulated) and the
// V-cycle level sweep / interpolation (PsiSweepArgs semantics of launch_psi_sweep).
bool tpsi_cfg(int nx, bool seq, SweepCfg &cfg);
cudaError_t launch_tpsi_seq(SweepCfg c, const CoarseArgs &a, cudaStream_t s);
cudaError_t launch_tpsi_level(SweepCfg c, const PsiSweepArgs &a, cudaStream_t s);

// Level-l (l >= 1) FULL-state primitives (levels.cu): rows n = n0 + j*nstride,
// j = 0..nrows-1, y = Psi U[n-1] + g[n] (g null: 0).  mode 0: dst[n] = y;  mode 1:
// r = y - U[n], per-block sum r^2 -> partials[j*bpr + b] (nullable), and if rstore is
// set, r -> rstore row (roff + j).  bpr blocks of 256 threads per row (1..64).
struct RowStepArgs {
  int nx, nrows, bpr, mode;
  int trunc;       // 1: Psi truncated at the boundaries (no wrap), bounded.cu
  long long n0, nstride;
  const double *U;
  double *dst;
  const double *g;
  double *partials;
  double *rstore;
  long long roff;
  PsiOp op;
};
cudaError_t launch_psi_rowstep(const RowStepArgs &a, cudaStream_t s);

// Device-side loop control of the CUDA-graph solve (graph.cu).
struct LoopState {
  double tol, dxdt;
  int k, max_iter, stop, nonfinite;
};
cudaError_t launch_loop_init(LoopState *s, double tol, double dxdt, int max_iter, int k0,
                             cudaStream_t st);
// ||r^(k)|| = sqrt(dxdt * norm2[0]) -> hist[k]; handles h0 (and h1 if set_h1) := !stop
cudaError_t launch_loop_decide(LoopState *s, const double *norm2, double *hist,
                               cudaGraphConditionalHandle h0, cudaGraphConditionalHandle h1,
                               int set_h1, cudaStream_t st);

// Deterministic reduction of partials -> out[0] (single block, fixed order).
cudaError_t launch_reduce(const double *partials, long long n, double *out, cudaStream_t s);

// Counter-based SplitMix64 uniform generator (R4).
cudaError_t launch_fill_guess(double *dst, long long row0, long long rows, int nx,
                              uint64_t seed, int lo_kind, const double *u0, cudaStream_t s);

}  // namespace mg
