/*
 * mgrit.h — C ABI of the B200 MGRIT/Parareal library (libmgrit.so) for the 1D
 * constant-coefficient linear advection equation u_t + alpha u_x = 0, periodic or
 * with inflow/outflow boundaries (mgrit_set_inflow).
 *
 * Paper: De Sterck, Falgout, Friedhoff, Krzysik, MacLachlan, "Optimizing MGRIT and
 * Parareal coarse-grid operators for linear advection", arXiv:1910.03726.
 * "P:n" = line n of PAPER.md; "S:n" = line n of SPEC.md.
 *
 * Conventions (apply to every entry point)
 *  - All floating point is IEEE fp64.  Space-time arrays are row-major [t][x]: row n
 *    (time t^n = n dt) holds nx contiguous doubles, x_i = -1 + i*2/nx (periodic).
 *  - "_dev" pointers are CUDA device pointers, "_host" pointers host pointers.
 *  - Ownership: the caller owns ALL device memory (the workspace, the guess, outputs)
 *    and the CUDA stream.  The library never calls cudaMalloc/cudaFree; it carves the
 *    caller's workspace.  Host arrays passed to mgrit_setup are copied.
 *  - Every call is asynchronous on the context's stream except those that return host
 *    values (mgrit_residual with norm_host, mgrit_solve, mgrit_profile_read), which
 *    synchronise the stream.
 *  - Errors: a negative mgrit_status; mgrit_last_error(ctx) gives a message.
 *  - Stencil index convention: a circulant operator A is a stencil {d: a_d} with
 *    (A u)_i = sum_d a_d u_{(i+d) mod nx}.
 */
#ifndef MGRIT_H
#define MGRIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGRIT_MAX_LEVELS 8
#define MGRIT_MAX_PSI_TAPS 64

typedef enum {
  MGRIT_OK = 0,
  MGRIT_EINVAL = -1,      /* invalid argument (sizes, divisibility, pointers) */
  MGRIT_ENOMEM = -2,      /* workspace too small */
  MGRIT_ECUDA = -3,       /* CUDA launch/runtime error */
  MGRIT_ENONFINITE = -4,  /* residual became NaN/Inf; history filled up to that point */
  MGRIT_EUNSUPPORTED = -5, /* valid but not implemented combination */
  MGRIT_ECOMM = -6         /* a time-shard communication callback failed */
} mgrit_status;

/* Runge-Kutta tableaux of Appendix A.  Order p pairs RK_p with U_p. */
typedef enum {
  MGRIT_TAB_ERK1 = 0,       /* Euler */
  MGRIT_TAB_ERK2 = 1,       /* SSP RK2 */
  MGRIT_TAB_ERK3_SSP = 2,   /* SSP RK3 */
  MGRIT_TAB_ERK3_KUTTA = 3, /* Kutta RK3 (BASELINE.json cfg2) */
  MGRIT_TAB_ERK4 = 4,       /* classical RK4 */
  MGRIT_TAB_ERK5 = 5,       /* Butcher (236a) */
  MGRIT_TAB_SDIRK1 = 6,     /* backward Euler */
  MGRIT_TAB_SDIRK2 = 7,
  MGRIT_TAB_SDIRK3 = 8,     /* P:999, zeta = 0.43586652150845899942 */
  MGRIT_TAB_SDIRK4 = 9      /* Hairer-Wanner (6.16) */
} mgrit_tableau;

typedef enum { MGRIT_RELAX_F = 0, MGRIT_RELAX_C = 1, MGRIT_RELAX_FCF = 2 } mgrit_relax_kind;

/* Multilevel cycle of mgrit_solve: V-cycle (default) or F-cycle, in which
 * each coarse problem is solved by one F-cycle followed by one V-cycle (R19). */
typedef enum { MGRIT_CYCLE_V = 0, MGRIT_CYCLE_F = 1 } mgrit_cycle_kind;

/* Coarse-grid time stepper Psi. */
typedef enum {
  MGRIT_PSI_STENCIL = 0, /* sparse circulant, e.g. the LSQ fit of eq. (LSQ_1D_problem) */
  MGRIT_PSI_IDEAL = 1,   /* Psi = Phi^m */
  MGRIT_PSI_REDISC = 2   /* Phi rediscretised with time step m dt, i.e. CFL redisc_cfl */
} mgrit_psi_kind;

typedef struct {
  int kind;              /* mgrit_psi_kind */
  int nnz;               /* STENCIL: number of taps (1..MGRIT_MAX_PSI_TAPS) */
  const int *offsets;    /* STENCIL: host, nnz strictly increasing offsets d */
  const double *coeffs;  /* STENCIL: host, nnz coefficients psi_d */
  double redisc_cfl;     /* REDISC: CFL number of the coarse operator (m*c) */
} mgrit_psi;

typedef struct mgrit_ctx mgrit_ctx;

/*
 * Workspace size (bytes) for a problem; see mgrit_setup for the arguments.
 * Returns 0 for invalid sizes.
 */
size_t mgrit_workspace_bytes(int nx, int nt, int m, int levels);

/*
 * mgrit_setup — create a solver context (north_star: mgrit_setup(nx, nt, m, alpha, CFL,
 * scheme, levels, psi_coeffs)).
 *   nx, nt      spatial points (periodic) and time steps; nt % m^(levels-1) == 0.
 *   m           coarsening factor (>= 2) on every level.
 *   alpha, cfl  wave speed (> 0) and CFL number c = alpha dt/dx; dx = 2/nx.
 *   order       p of the upwind stencil U_p, 1..5.
 *   tableau     mgrit_tableau; explicit tableaux need ERK, implicit SDIRK.
 *   levels      2 = two-level MGRIT/Parareal; > 2 = multilevel V-cycle.
 *   psi         host array of levels-1 coarse operators Psi_2..Psi_L (copied).  IDEAL
 *               (Phi^m) and REDISC (Phi at CFL redisc_cfl) are only valid for
 *               levels == 2 and nx in {64, 128, ..., 4096}; with an SDIRK tableau the coarse
 *               step solves its own stages (factored as for the fine step).
 *   relax       production relaxation of mgrit_solve: MGRIT_RELAX_F (Parareal) or
 *               MGRIT_RELAX_FCF.
 *   workspace_dev / workspace_bytes   caller-owned device memory, >= mgrit_workspace_bytes.
 *   stream      cudaStream_t (NULL = legacy default stream).
 * Errors: EINVAL (sizes, divisibility, tableau/order mismatch, nx too small for a stencil),
 *         ENOMEM (workspace), EUNSUPPORTED (SDIRK needs whole periodic rows: nx in
 *         {64, 128, ..., 4096}; RK-form Psi outside the sizes above; a Psi stencil wider
 *         than MGRIT_MAX_PSI_TAPS or nx/2).
 */
int mgrit_setup(mgrit_ctx **ctx, int nx, int nt, int m, double alpha, double cfl, int order,
                int tableau, int levels, const mgrit_psi *psi, int relax,
                void *workspace_dev, size_t workspace_bytes, void *stream);

void mgrit_destroy(mgrit_ctx *ctx);
const char *mgrit_last_error(const mgrit_ctx *ctx);

/*
 * The library's fp64 coefficients (host-only, no GPU needed): z_d of Z = dt L
 * (z_d = (-c w_d)/den, R3), the tableau (A row-major s x s, b), and, for a
 * STENCIL Psi of level l, its dense contiguous window.  Sizes: z[8], A[36], b[6].
 */
int mgrit_get_coefficients(const mgrit_ctx *ctx, int *s, int *z_lo, int *z_n, double *z,
                           double *A, double *b);

/*
 * Same coefficients without a context (host-only): U_p stencil at CFL `cfl` and the
 * tableau `tableau`.  Returns EINVAL for unknown ids.
 */
int mgrit_scheme_coefficients(int order, int tableau, double cfl, int *s, int *z_lo, int *z_n,
                              double *z, double *A, double *b);

/*
 * mgrit_set_guess — register the initial space-time iterate: a FULL
 * (nt+1) x nx device array whose row 0 is u0.  It is read, never written; the caller
 * keeps it alive while solving.
 */
int mgrit_set_guess(mgrit_ctx *ctx, const double *guess_dev);

/*
 * FULL-state primitives on a caller-owned device array U_dev of level `level`, in place
 * (P:206-212).  Level 0 is the fine grid: U_dev is (nt+1) x nx, Phi_0 = Phi (the RK step),
 * row 0 = u0 is never written.  Level l >= 1 (multilevel hierarchy, P:618-624;
 * stencil Psi only) is (nt_l+1) x nx with nt_l = nt/m^l, Phi_l = Psi_l, and the equations
 * U[n] = Psi_l U[n-1] + g_l[n] (R12) with the right-hand side registered by
 * mgrit_set_rhs (none: g_l = 0); row 0 is not written either.
 *   mgrit_relax:        kind F: U[jm+i] = Phi_l U[jm+i-1] (+ g_l[jm+i]), i = 1..m-1;
 *                       C: U[(j+1)m] = Phi_l U[(j+1)m-1] (+ g_l); FCF: F then C then F.
 *   mgrit_residual:     norm_host (nullable) = sqrt(dx dt_l sum_{n>=1} |r[n]|^2), dt_l = m^l dt,
 *                       r[n] = (g_l[n] +) Phi_l U[n-1] - U[n] over ALL rows (DESIGN.md
 *                       R1); r_dev (nullable, (nt_l/m+1) x nx) receives the C-point
 *                       residuals r_j = r[jm], r_0 = 0.
 *   mgrit_coarse_solve: coarse-grid correction of level l by level l+1 solved exactly
 *                       (sequentially): r_j as above, e_j = Psi_{l+1} e_{j-1} + r_j, e_0 = 0
 *                       (eq. 3), U[jm] += e_j, then F-relaxation ("ideal
 *                       interpolation").  Needs l + 1 < levels.
 * Errors: EINVAL (null pointers, level out of range, nt_l not a multiple of m),
 *         EUNSUPPORTED (level >= 1 with an IDEAL/REDISC Psi), ECUDA.
 */
int mgrit_relax(mgrit_ctx *ctx, int level, int kind, double *U_dev);
int mgrit_residual(mgrit_ctx *ctx, int level, const double *U_dev, double *norm_host,
                   double *r_dev);
int mgrit_coarse_solve(mgrit_ctx *ctx, int level, double *U_dev);

/*
 * mgrit_set_rhs — right-hand side g_l ((nt_l+1) x nx device array, read only, caller-owned;
 * NULL = zero) used by the level-l FULL primitives above, 1 <= level < levels.  Level 0 has
 * no right-hand side (g_0 = (u0, 0, ..., 0) is implied by row 0 of U).  Errors: EINVAL.
 */
int mgrit_set_rhs(mgrit_ctx *ctx, int level, const double *g_dev);

/*
 * mgrit_set_inflow — inflow/outflow boundaries instead of the periodic one (PAPER.md 4.5,
 * P:672-680; R20).  The row then holds the nx unknowns u_1..u_nx at x_i = -1 + i dx,
 * x_0 = -1 is the inflow point (its value is data), x_nx = 1 the outflow point.
 *   enable   0: back to periodic rows.  1: every fine step is Phi(u; t_n) = Phi_h u + b_n:
 *            Phi_h uses zero inflow ghosts and degree-p polynomial extrapolation of every
 *            stage vector at the outflow; b_n = Phi(0; t_n) carries the inflow data through
 *            the Taylor / inverse-Lax-Wendroff ghost values of each Runge-Kutta stage
 *            (Carpenter et al.); every stencil Psi_l is truncated at the boundaries (Toeplitz,
 *            no wrap), IDEAL/REDISC Psi use the same closures.
 *   dg_dev   device, nt x (order + s) row-major: the inflow derivatives g^(r)(t_n),
 *            r = 0..order+s-1, at t_n = n dt, n = 0..nt-1 (s = stages); read during the call
 *            only (the forcing rows b_n go to the workspace).  NULL: homogeneous inflow.
 * All entry points then act on the affine system U[n+1] = Phi_h U[n] + b_n (mgrit_relax,
 * mgrit_residual, mgrit_coarse_solve, mgrit_solve; coarse levels are error equations and
 * stay homogeneous).  Asynchronous on the context's stream.
 * Errors: EUNSUPPORTED (SDIRK tableau; time shards; a row that does not fit one CTA with
 * more points per thread than the order: nx in {64, 128, ..., 4096}, nx >= 128 for order
 * 3-4, nx >= 256 for order 5; RK-form Psi with nx = 4096), ECUDA.
 * mgrit_get_forcing copies the nt x MGRIT_FORCING_LD forcing rows (b_n on the first
 * s*|d_min| points of the row, zero-padded) to out_dev.
 */
#define MGRIT_FORCING_LD 24
int mgrit_set_inflow(mgrit_ctx *ctx, int enable, const double *dg_dev);
int mgrit_get_forcing(mgrit_ctx *ctx, double *out_dev);

/*
 * mgrit_solve — MGRIT iterations from the registered guess until ||r^(k)|| < tol or
 * k == max_iter (R2, R15).  Production engine: C-point storage, fused
 * relax+residual+restriction sweeps, sequential (or V-cycle) coarse solve.
 *   out_dev       nullable; FULL (nt+1) x nx solution (F-points materialised by an
 *                 F-relaxation from the final C-points).
 *   iters         iterations performed K.
 *   hist_host     nullable, >= max_iter+1 doubles: ||r^(0)|| .. ||r^(K)||.
 *   converged     1 if ||r^(K)|| < tol.
 *   crows_hist_dev  nullable, max_iter x (nt/m+1) x nx: C-rows after every iteration.
 * Returns MGRIT_ENONFINITE if the residual became NaN/Inf (history filled so far).
 */
int mgrit_solve(mgrit_ctx *ctx, double tol, int max_iter, double *out_dev, int *iters,
                double *hist_host, int *converged, double *crows_hist_dev);

/*
 * mgrit_set_cycle — cycle of mgrit_solve's coarse-grid correction for levels >= 3:
 * MGRIT_CYCLE_V (default) or MGRIT_CYCLE_F (R19).
 * Two-level solves are unaffected (the coarse solve is exact).  Host-only setter.
 * Errors: EINVAL for another value or a null context.
 */
int mgrit_set_cycle(mgrit_ctx *ctx, int cycle);

/*
 * mgrit_set_final_sweep — how mgrit_solve (with out_dev non-NULL) measures the residual
 * of the iterate it returns.  The sweep that measures ||r^(k)|| normally also computes
 * the next coarse right-hand side r = Phi^m delta; if iteration k is the last, that work
 * is unused and the FULL solution needs a separate F-relaxation pass.  A check sweep
 * instead writes the F-relaxed iterate (all rows) into out_dev while measuring the norm
 * (identical partial sums, so identical history and K).  Modes:
 *   MGRIT_FINAL_OFF      never (always the fused sweep, then a materialisation pass);
 *   MGRIT_FINAL_PREDICT  (default) when k == max_iter, or when the geometric
 *                        extrapolation ||r^(k-1)||^2/||r^(k-2)|| of a decreasing history
 *                        is below tol; if the check does not converge, the fused sweep
 *                        is run after it (results unchanged, one extra phase-1 pass);
 *   MGRIT_FINAL_ALWAYS   every iteration (tests the misprediction path).
 * Host-only setter.  Errors: EINVAL for another value or a null context.
 */
enum { MGRIT_FINAL_OFF = 0, MGRIT_FINAL_PREDICT = 1, MGRIT_FINAL_ALWAYS = 2 };
int mgrit_set_final_sweep(mgrit_ctx *ctx, int mode);

/*
 * mgrit_set_option — replace a measured kernel-configuration default by another valid
 * one (tuning scans, tests of alternative kernels).  Results stay correct for every
 * accepted value; a configuration that no kernel supports makes the next call that needs
 * it return MGRIT_EUNSUPPORTED.  n = 0 restores the default.  Host-only; the library
 * reads no environment variables.
 *   MGRIT_OPT_FINE_TILE      NT, P[, minBlocks]  tile of the fused FCF fine sweep (halo tiles)
 *   MGRIT_OPT_WHOLE_ROW      NT, P               whole-periodic-row sweep tried first
 *   MGRIT_OPT_SEQ_CLUSTER    CL, NT, P           two-level coarse solve: cluster split (CL = 0:
 *                                                no cluster -> single-CTA solve)
 *   MGRIT_OPT_SEQ_S          S                   s-step depth limit (S < 2: exchange every step)
 *   MGRIT_OPT_COARSE_KERNEL  0 | 1               warp-specialised (default) | cp.async variant
 *   MGRIT_OPT_SEQ_CFG        NT, P               single-CTA coarse solve configuration
 *   MGRIT_OPT_SDIRK_PRODUCT  0 | 1               1: product-form SDIRK stage solves only
 *   MGRIT_OPT_GRAPH          0 | 1               mgrit_solve's iterations as one CUDA graph with
 *                                                a device-side WHILE loop (one host sync per
 *                                                solve) | per-iteration host loop; default:
 *                                                graph for nx*nt <= 2^23 (latency-bound)
 *                                                unless the overlapped iteration with a
 *                                                speculative chain applies (MGRIT_OPT_OVERLAP),
 *                                                host loop otherwise (it predicts the last
 *                                                iteration and fuses materialisation)
 *   MGRIT_OPT_STAGE_FORM     0 | 1               1: explicit steps in the plain Runge-Kutta
 *                                                stage form (no folded last stage, no
 *                                                Shu-Osher SSP-RK3; R5)
 *   MGRIT_OPT_OVERLAP        C[, spec]           two-level host-loop solves: the sequential
 *                                                coarse chain runs on a private high-priority
 *                                                stream and publishes its progress every
 *                                                nc/C steps; the next iteration's sweep over
 *                                                the intervals already corrected follows
 *                                                beside it, released by stream-ordered memory
 *                                                waits (bitwise the serial iteration); 0 or
 *                                                1: serial; default 16 / 8 chunks for chains
 *                                                of >= 2048 / >= 1024 steps, halved with a
 *                                                speculative chain (mgrit_overlap_plan).
 *                                                Optional second value: 1 / 0 = speculative
 *                                                chain on / off (FCF: the chain of iteration
 *                                                k+1 is launched behind the sweep chunks of
 *                                                iteration k, gated on a flag the stream
 *                                                writes after each chunk; default: on when
 *                                                the chain is estimated >= 1.5x the sweep).
 *                                                The speculative chain needs concurrent
 *                                                kernels: under tools that serialise them
 *                                                (profiler kernel replay, launch blocking)
 *                                                use C, 0 -- its gate otherwise gives up
 *                                                after 10 s with a launch failure
 *   MGRIT_OPT_VOVERLAP       C[, n[, spec]]      V-cycle host-loop solves (halo-tile kernels):
 *                                                the HBM-bound level-1 interpolation in C
 *                                                chunks on a high-priority stream, the
 *                                                FP64-bound fine sweep over the corrected
 *                                                intervals beside it with at most n CTAs per
 *                                                SM, and (spec = 1) the next V-cycle's level-1
 *                                                sweep behind it; ordered by events, bitwise
 *                                                the serial iteration; C = 0 or 1: serial
 *                                                (the default: measured gain <= 1.5 %,
 *                                                DESIGN.md 6.11)
 * Errors: EINVAL (unknown option, wrong count, negative value); EUNSUPPORTED if the new
 * whole-row / SDIRK setting cannot factor the stage solves (the old setting is kept).
 */
typedef enum {
  MGRIT_OPT_FINE_TILE = 0,
  MGRIT_OPT_WHOLE_ROW = 1,
  MGRIT_OPT_SEQ_CLUSTER = 2,
  MGRIT_OPT_SEQ_S = 3,
  MGRIT_OPT_COARSE_KERNEL = 4,
  MGRIT_OPT_SEQ_CFG = 5,
  MGRIT_OPT_SDIRK_PRODUCT = 6,
  MGRIT_OPT_STAGE_FORM = 7,
  MGRIT_OPT_GRAPH = 8,
  MGRIT_OPT_OVERLAP = 9,
  MGRIT_OPT_VOVERLAP = 10,
  MGRIT_OPT_COUNT = 11
} mgrit_option;
int mgrit_set_option(mgrit_ctx *ctx, int option, const int *values, int n);

/*
 * mgrit_overlap_plan — the chunking the overlapped two-level iteration (MGRIT_OPT_OVERLAP)
 * uses for a coarse chain of nc steps when `want` chunks are asked for (host-only, no GPU):
 * *chunks = C (0: serial), and for i < C the fine intervals [j0[i], j1[i]) of sweep chunk i
 * (j0, j1 nullable; room for `want` entries).  Chain chunk i covers the steps iL+1..(i+1)L,
 * L = nc/C; sweep chunk i is shifted by one interval so that it reads C-rows <= (i+1)L and
 * overwrites coarse right-hand-side rows <= (i+1)L only.  Errors: EINVAL.
 */
int mgrit_overlap_plan(long long nc, int want, int *chunks, long long *j0, long long *j1);

/*
 * ---- Time-parallel MGRIT over several GPUs (the paper parallelises time
 * only, with contiguous blocks of time per processor) ----
 *
 * mgrit_setup_shard creates the context of time shard `rank` of `nranks`: the global
 * problem has nt steps; this rank owns steps [rank*nt/nranks, (rank+1)*nt/nranks] (its
 * fine C-intervals j in [rank*nc, (rank+1)*nc), nc = nt/(m*nranks)), with nt/nranks
 * divisible by m^(levels-1).  Every level's sweep, residual injection and interpolation run
 * on the rank's own intervals; the sequential coarsest-level solve is pipelined across the
 * ranks (state x passed rank to rank).  Exchanges per iteration, each one row of nx doubles
 * through the caller-owned staging rows stage_send_dev / stage_recv_dev:
 *   - the current iterate's C-row at the block start (halo, from rank-1) before each fine
 *     sweep, the corrected level-l C-row at the block start before each interpolation;
 *   - the coarse right-hand side r_{nc+1} of the block's last interval (to rank+1) after
 *     each sweep;
 *   - the coarsest chain's state (rank-1 -> rank);
 *   - the squared residual norm (allreduce_sum of one double).
 * The caller provides the communication (NCCL/gloo through torch.distributed, or an
 * in-process emulation) as callbacks:
 *   shift(user, has_send, has_recv, stream): if has_send, send stage_send_dev (written on
 *     `stream` before the call; the callback orders itself after it) to rank+1; if has_recv,
 *     receive rank-1's row into stage_recv_dev, complete before returning.  Called by every
 *     rank at the same points (flags 0 for the missing neighbour).  0 on success.
 *   allreduce_sum(user, vals, n): in-place sum of n host doubles over all ranks.
 * The guess (mgrit_set_guess) and out_dev are the rank's local FULL block of
 * nt/nranks + 1 rows whose row 0 is global row rank*nt/nranks (u0 on rank 0).  Stencil Psi
 * and the V-cycle only (EUNSUPPORTED otherwise); the history is the global one, identical
 * on every rank.  nranks = 1 is an ordinary solve through the same code path.
 */
typedef struct {
  void *user;
  int (*shift)(void *user, int has_send, int has_recv, void *stream);
  int (*allreduce_sum)(void *user, double *vals, int n);
} mgrit_comm;
size_t mgrit_workspace_bytes_shard(int nx, int nt, int m, int levels, int nranks);
int mgrit_setup_shard(mgrit_ctx **ctx, int nx, int nt, int m, double alpha, double cfl,
                      int order, int tableau, int levels, const mgrit_psi *psi, int relax,
                      int rank, int nranks, double *stage_send_dev, double *stage_recv_dev,
                      void *workspace_dev, size_t workspace_bytes, void *stream);
int mgrit_solve_shard(mgrit_ctx *ctx, const mgrit_comm *comm, double tol, int max_iter,
                      double *out_dev, int *iters, double *hist_host, int *converged);

/*
 * ---- Coarse-operator synthesis on the GPU (§4) ----
 * mgrit_psi_fit computes Psi_2..Psi_levels by the weighted linear least-squares fit of
 * eq. (LSQ_1D_problem) (w(z) = 1/(1 - z + 1e-6)^2 at |eigenvalues| of the
 * operator being coarsened), recursively Psi_{l+1} ~ Psi_l^m, for the
 * scheme (order, tableau, cfl) on nx points:
 *   widths      levels-1 window widths nu_l: contiguous offsets centred on
 *               round_half_away(-m^l cfl) (R8); NULL with eta > 0:
 *   eta         > 0: two-level threshold pattern, the contiguous hull of the entries of
 *               the first column of Phi^m with magnitude >= eta * max.
 * Outputs (host): nnz_out[levels-1], offsets_out / coeffs_out [(levels-1) x
 * MGRIT_MAX_PSI_TAPS] (row l: nnz_out[l] increasing offsets), imag_out (nullable,
 * levels-1): the P:394 flag, the largest imaginary component of the complex problem's
 * solution (fits with imag > 1e-8 are not accepted by the paper).  The normal equations
 * are formed and solved in double-double arithmetic on the device (csrc/psifit.cu).
 * workspace_dev: caller-owned device memory of mgrit_psi_fit_workspace_bytes(nx).
 * Synchronous on `stream`.  Errors: EINVAL (sizes, ids, pattern), ENOMEM, ECUDA.
 */
size_t mgrit_psi_fit_workspace_bytes(int nx);
int mgrit_psi_fit(int nx, int order, int tableau, double cfl, int m, int levels,
                  const int *widths, double eta, int *offsets_out, int *nnz_out,
                  double *coeffs_out, double *imag_out, void *workspace_dev,
                  size_t workspace_bytes, void *stream);

/*
 * mgrit_psi_fit_nl — the nonlinear least-squares coarse operator of PAPER.md Appendix B
 * (eq. (nlsq)) on the device: minimise F(psi) = (1/nx) sum_k ||E_k(psi)||^2 with
 * ||E_k|| the two-level FCF estimate (Dobrev_bounds) P:283-293 of Fourier mode k, over the
 * real nonzeros psi of a circulant Psi with the contiguous pattern `offsets`, by
 * Levenberg-Marquardt (identity scaling, l_0 = 0.01, x10 / /10, stop at relative decrease
 * or step 1e-6, at most max_iter trials; the paper allows 30) from the start value in
 * `coeffs` (the linear fit of mgrit_psi_fit).  Explicit tableaux, two-level.
 *   coeffs          host, nnz: start value in, result out.
 *   iters_out       nullable: trials used.   objective_out  nullable: F at the result.
 *   history_out     nullable, max_iter + 1: F after every trial (entry 0: the start value).
 * The modes are evaluated one thread per k (the geometric sum of the estimate by Horner), the
 * Gauss-Newton matrix J^T J and J^T r are accumulated and factored in double-double.
 * Synchronous on `stream`.  Errors: EINVAL, ENOMEM, EUNSUPPORTED (SDIRK), ECUDA.
 */
size_t mgrit_psi_fit_nl_workspace_bytes(int nx);
int mgrit_psi_fit_nl(int nx, int order, int tableau, double cfl, int m, int nt, int nnz,
                     const int *offsets, double *coeffs, int max_iter, int *iters_out,
                     double *objective_out, double *history_out, void *workspace_dev,
                     size_t workspace_bytes, void *stream);

/* C-rows (nt/m+1) x nx of the current iterate after mgrit_solve. */
int mgrit_get_crows(mgrit_ctx *ctx, double *out_dev);

/*
 * Input generation (not part of the method; R4): fills rows [row0, row0+rows)
 * of an iterate with the counter-based SplitMix64 uniform variates of (seed, n*nx+i);
 * lo_kind 0: U[-1,1), 1: U[0,1).  If u0_dev is non-NULL and row0 == 0, row 0 := u0.
 */
int mgrit_fill_guess(double *dst_dev, long long row0, long long rows, int nx, uint64_t seed,
                     int lo_kind, const double *u0_dev, void *stream);

/*
 * Profiling (bench.py): when enabled, every kernel launch is bracketed by CUDA events on
 * the launching stream; mgrit_profile_read returns, per kernel class, the number of
 * launches and the summed device milliseconds since the last reset.
 * Classes: 0 fine sweep, 1 coarse-level sweeps, 2 coarse/sequential solves,
 *          3 interpolation/materialisation, 4 residual, 5 reductions/other.
 */
#define MGRIT_PROF_CLASSES 6
int mgrit_profile_enable(mgrit_ctx *ctx, int on);
int mgrit_profile_read(mgrit_ctx *ctx, long long *launches, double *ms);
/* Human-readable launch configuration of the fine sweep / level kernels (host-only). */
int mgrit_describe(const mgrit_ctx *ctx, char *buf, size_t len);
/* Total kernel launches since setup (or the last profile reset). */
long long mgrit_launch_count(const mgrit_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* MGRIT_H */
