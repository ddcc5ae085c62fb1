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
#include "tma.cuh"
#include "rows.cuh"

#include <algorithm>
#include <type_traits>

namespace mg {

// ---------------------------------------------------------------------------
// Persistent, TMA-pipelined variant for halo-tile mode (odd P => contiguous
// shared-memory windows).  Each CTA walks work items (interval, tile) with a
// grid stride; while the FP64 pipes run the m RK steps of item i, the bulk-copy
// engine prefetches the windows of item i+1 into the other buffer pair and
// drains the stores (v_{j+1}, r_{j+2}) of item i-1.  Tile boundaries are even so
// every bulk copy is 16-byte aligned.  Modes: in/cmp/endw/dstore/r2/partials
// (the production sweeps and the all-row residual) and per-step writes (each).
// ---------------------------------------------------------------------------
template <class SC, int NT, int P, int MINB>
__global__ void __launch_bounds__(NT, MINB) rk_sweep_tma_kernel(const __grid_constant__ SweepArgs a) {
  static_assert(P % 2 == 1, "contiguous windows need odd P");
  constexpr int W = NT * P;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(128) double smem[];
  // buffers: IN(b) = smem + b*W (double-buffered prefetch), CM = smem + 2W (the comparison
  // row u_{j+1}, loaded at item start and consumed after phase 1).  Macros, not pointer
  // arrays (those would live in local memory).
#define IN(b) (smem + (b) * W)
  double *CM = smem + 2 * W;
  double *edge = smem + 3 * W;
  double *red = edge + 2 * NT * (SC::NL + SC::NR) + 2;
  uint64_t *bar = reinterpret_cast<uint64_t *>(red + NW + 2);  // bar[0..1] in, bar[2] cmp
  const int tid = threadIdx.x;
  const int nx = a.nx;
  const int total = a.nitems * a.ntiles;
  const int half = nx >> 1;

  auto tile_beg = [&](int t) { return 2 * (int)(((long long)t * half) / a.ntiles); };
  auto rowp = [&](const RowMap &r, long long j) -> const double * {
    return r.base + (r.off + j * r.stride) * (long long)nx;
  };
  // window loads (one thread): `in` rows of item w into IN(b), `cmp` rows into CM
  auto window = [&](int w, int &start, int &n1) {
    const int tile = w % a.ntiles;
    start = tile_beg(tile) - a.HL;
    if (start < 0) start += nx;
    n1 = (start + W <= nx) ? W : nx - start;
  };
  auto issue_in = [&](int w, int b) {
    int start, n1;
    window(w, start, n1);
    mbar_expect_tx(&bar[b], (uint32_t)W * 8u);
    const double *row = rowp(a.in, w / a.ntiles);
    tma_load_1d(IN(b), row + start, (uint32_t)n1 * 8u, &bar[b]);
    if (n1 < W) tma_load_1d(IN(b) + n1, row, (uint32_t)(W - n1) * 8u, &bar[b]);
  };
  auto issue_cmp = [&](int w, double *dst) {
    int start, n1;
    window(w, start, n1);
    mbar_expect_tx(&bar[2], (uint32_t)W * 8u);
    const double *row = rowp(a.cmp, w / a.ntiles);
    tma_load_1d(dst, row + start, (uint32_t)n1 * 8u, &bar[2]);
    if (n1 < W) tma_load_1d(dst + n1, row, (uint32_t)(W - n1) * 8u, &bar[2]);
  };
  // wait until at most n of this thread's bulk groups are still reading shared memory
  auto wait_read_upto = [&](int n) {
    if (n <= 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    else if (n == 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    else if (n == 2) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
    else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
  };
  // check sweep (per-step writes AND comparison rows): IN(b) and CM alternate as staging,
  // and the comparison row is loaded after the last per-step store, into the buffer the
  // store before it used (phase-1's last step covers the load)
  const bool chk = a.cmp.base && a.each_last >= a.each_first;
  // stage x into buf, then bulk-store the owned slice [HL, HL+T) to row[abeg..].  The
  // leading barrier is needed only when buf was read by other threads since the last
  // barrier (per-step staging after thread 0's read-completion wait); the production
  // stores stage into windows last read many barriers ago or in place.
  auto store = [&](double *row, double *buf, const double(&v)[P], int abeg, int T,
                   bool lead_barrier) {
    if (lead_barrier) __syncthreads();
#pragma unroll
    for (int p = 0; p < P; ++p) buf[tid * P + p] = v[p];
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tma_store_1d(row + abeg, buf + a.HL, (uint32_t)T * 8u);
      bulk_commit();
    }
  };

  if (tid == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && (int)blockIdx.x < total) issue_in(blockIdx.x, 0);
  int phase = 0;
  int it = 0;
  int nstage = 0;
#pragma unroll 1
  for (int w = blockIdx.x; w < total; w += gridDim.x, ++it) {
    const int b = it & 1;
    const uint32_t par = (uint32_t)((it >> 1) & 1);
    const int nw = w + gridDim.x;
    const int nstage0 = nstage;
    double *CMP = CM;                               // where the comparison row lands
    // Prefetch of item it+1 into IN(b^1) and the comparison row of item it into CM: both
    // buffers held the staged stores of item it-1, so thread 0 must first wait for those
    // bulk stores to finish reading shared memory.  Doing that at item start would hold
    // warp 0 (and, through the next barrier, the whole CTA); it is deferred until after
    // the first RK step unless the item has a single step.
    auto issue_loads = [&]() {
      if (tid == 0) {
        wait_read_upto(nstage - nstage0);          // only this item's own stores may still read
        if (nw < total) issue_in(nw, b ^ 1);
        if (a.cmp.base && !chk) issue_cmp(w, CM);
      }
    };
    const bool early = a.nsteps1 < 2;
    if (early) issue_loads();
    const int item = w / a.ntiles, tile = w - item * a.ntiles;
    const int abeg = tile_beg(tile);
    const int T = tile_beg(tile + 1) - abeg;
    mbar_wait(&bar[b], par);
    double x[P];
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = IN(b)[tid * P + p];
    // per-step writes (F-relaxation / materialisation / check sweep): IN(b) and CM
    // alternate as staging; a buffer is reused once the store before last has read it.
    auto each_store = [&](int i) {
      if (tid == 0 && nstage >= 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      double *row = const_cast<double *>(a.each.base) +
                    (a.each.off + (long long)item * a.each.stride + (long long)i * a.each_step) *
                        (long long)nx;
      store(row, (nstage & 1) ? CM : IN(b), x, abeg, T, true);
      ++nstage;
      if (chk && i == a.each_last) {
        CMP = (nstage & 1) ? CM : IN(b);           // the buffer of the store before last
        if (tid == 0) {
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          issue_cmp(w, CMP);
        }
      }
    };
    // The steps before and after the thread-0 prefetch run in separate loops so the
    // divergent issue region does not sit inside a step loop (a reconvergence point per
    // step); per-step writes get their own loops for the same reason.
    if (a.each_first == 0 && a.each_last >= 0) each_store(0);
    const int la = early ? 0 : min(max(a.load_after, 1), a.nsteps1);
    if (a.each_last >= a.each_first) {
#pragma unroll 1
      for (int i = 1; i <= la; ++i) {
        erk_step<SC, P, NT>(x, a.co, edge, phase);
        if (i >= a.each_first && i <= a.each_last) each_store(i);
      }
      if (!early) issue_loads();
#pragma unroll 1
      for (int i = la + 1; i <= a.nsteps1; ++i) {
        erk_step<SC, P, NT>(x, a.co, edge, phase);
        if (i >= a.each_first && i <= a.each_last) each_store(i);
      }
    } else {
#pragma unroll 1
      for (int i = 1; i <= la; ++i) erk_step<SC, P, NT>(x, a.co, edge, phase);
      if (!early) issue_loads();
#pragma unroll 1
      for (int i = la + 1; i <= a.nsteps1; ++i) erk_step<SC, P, NT>(x, a.co, edge, phase);
    }
    // v_{j+1}: with a phase 2 to follow, staged in place now and stored together with
    // r_{j+2} (one fence and one barrier per item); otherwise stored right away
    const bool defer_v = a.endw.base && a.cmp.base && a.nsteps2 > 0 && item < a.p2_items &&
                         a.defer_v;
    if (defer_v) {
#pragma unroll
      for (int p = 0; p < P; ++p) IN(b)[tid * P + p] = x[p];
    } else if (a.endw.base) {
      store(const_cast<double *>(rowp(a.endw, item)), IN(b), x, abeg, T, false);
    }
    if (a.cmp.base) {
      mbar_wait(&bar[2], (uint32_t)(it & 1));
      double d[P];
#pragma unroll
      for (int p = 0; p < P; ++p) d[p] = x[p] - CMP[tid * P + p];
      if (a.partials) {
        double sacc = 0.0;
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const int l = tid * P + p;
          if (l >= a.HL && l < a.HL + T) sacc = fma(d[p], d[p], sacc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(FULL, sacc, o);
        if ((tid & 31) == 0) a.partials[((long long)item * a.ntiles + tile) * NW + (tid >> 5)] = sacc;
      }
      if (a.dstore.base) {
        const int jj = item + a.d_phase;
        if (jj % a.d_every == 0)
          store(const_cast<double *>(rowp(a.dstore, jj / a.d_every)), CM, d, abeg, T, false);
      }
      if (a.nsteps2 > 0 && item < a.p2_items) {
#pragma unroll
        for (int p = 0; p < P; ++p) x[p] = d[p];
#pragma unroll 1
        for (int i = 1; i <= a.nsteps2; ++i) erk_step<SC, P, NT>(x, a.co, edge, phase);
        if (defer_v) {
#pragma unroll
          for (int p = 0; p < P; ++p) CM[tid * P + p] = x[p];
          fence_proxy_async();
          __syncthreads();
          if (tid == 0) {
            tma_store_1d(const_cast<double *>(rowp(a.endw, item)) + abeg, IN(b) + a.HL, (uint32_t)T * 8u);
            tma_store_1d(const_cast<double *>(rowp(a.r2, item)) + abeg, CM + a.HL, (uint32_t)T * 8u);
            bulk_commit();
          }
        } else {
          store(const_cast<double *>(rowp(a.r2, item)), CM, x, abeg, T, false);
        }
      }
    }
  }
  if (tid == 0) bulk_wait_all();
#undef IN
}

template <class SC, int NT, int P, int MINB>
static cudaError_t launch_tma_one(const SweepArgs &a, cudaStream_t s) {
  constexpr int W = NT * P;
  const size_t smem =
      sizeof(double) * (3 * W + 2 * NT * (SC::NL + SC::NR) + 2 + NT / 32 + 2) +
      4 * sizeof(uint64_t) + 16;
  static int blocks_per_sm = 0;
  if (!blocks_per_sm) {
    cudaFuncSetAttribute(rk_sweep_tma_kernel<SC, NT, P, MINB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 116 * 1024));
    cudaFuncSetAttribute(rk_sweep_tma_kernel<SC, NT, P, MINB>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm,
                                                  rk_sweep_tma_kernel<SC, NT, P, MINB>, NT, smem);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long total = (long long)a.nitems * a.ntiles;
  if (total <= 0) return cudaSuccess;
  // max_per_sm == 3 (overlapped V-cycle): the grid alone does not keep a fourth
  // CTA off an SM, so the launch asks for just enough shared memory that four CTAs no longer
  // fit (4 x (57472 + 1024) > 228 KiB) while three of them leave room for one 128 x 9 level
  // kernel CTA (3 x 58496 + 57728 <= 233472 bytes)
  size_t smem_l = smem;
  int per_sm = blocks_per_sm;
  if (a.max_per_sm > 0 && a.max_per_sm < blocks_per_sm) {
    per_sm = a.max_per_sm;
    // smallest request (multiple of 128) with (per_sm + 1) x (request + 1 KiB) > 228 KiB
    const size_t need = ((233472 / (per_sm + 1) - 1024) / 128 + 1) * 128;
    smem_l = std::max(smem, need);
  }
  const long long grid = std::min<long long>(total, (long long)std::max(1, sms - a.reserve_sms) * per_sm);
  rk_sweep_tma_kernel<SC, NT, P, MINB><<<(unsigned)grid, NT, smem_l, s>>>(a);
  return cudaGetLastError();
}

#define MG_TMA_CFGS(X) X(128, 15) X(256, 11) X(64, 15) X(32, 31)

template <class SC>
static cudaError_t dispatch_tma(SweepCfg c, const SweepArgs &a, cudaStream_t s) {
// default: no min-blocks hint (ptxas picks 128 registers for 128x15 -> 4 CTAs/SM)
#define MG_CASE(NT_, P_) \
  if (c.nt_threads == NT_ && c.p == P_ && c.minb == 0) \
    return launch_tma_one<SC, NT_, P_, 0>(a, s);
  MG_TMA_CFGS(MG_CASE)
#undef MG_CASE
  if (c.nt_threads == 128 && c.p == 15 && c.minb == 3) return launch_tma_one<SC, 128, 15, 3>(a, s);
  if (c.nt_threads == 128 && c.p == 15 && c.minb == 2) return launch_tma_one<SC, 128, 15, 2>(a, s);
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_rk_sweep_tma(int scheme, SweepCfg cfg, const SweepArgs &a, cudaStream_t s) {
  switch (scheme) {
    case 0: return dispatch_tma<ERK1U1>(cfg, a, s);
    case 1: return dispatch_tma<ERK2U2>(cfg, a, s);
    case 2: return dispatch_tma<ERK3U3>(cfg, a, s);
    case 3: return dispatch_tma<ERK4U4>(cfg, a, s);
    case 4: return dispatch_tma<ERK5U5>(cfg, a, s);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
// All-row residual r_n = Phi U[n-1] - U[n] (hist[0]) in halo tiles: a work item
// is a (tile, chunk of consecutive rows); the CTA streams the chunk's rows through a
// ring of three windows (TMA), so every row is loaded once and serves first as the
// comparison row and then as the next input.  Per-warp partial sums of r^2.
// ---------------------------------------------------------------------------
template <class SC, int NT, int P>
__global__ void __launch_bounds__(NT, 4) rk_residual_tma_kernel(const __grid_constant__ SweepArgs a,
                                                             int chunk) {
  static_assert(P % 2 == 1, "contiguous windows need odd P");
  constexpr int W = NT * P;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(128) double smem[];
  double *edge = smem + 3 * W;
  uint64_t *bar = reinterpret_cast<uint64_t *>(edge + 2 * NT * (SC::NL + SC::NR) + 2);
  const int tid = threadIdx.x;
  const int nx = a.nx, half = nx >> 1;
  const int nrows = a.nitems;                       // residual rows n = 1..nrows
  const int nchunks = (nrows + chunk - 1) / chunk;
  const int total = nchunks * a.ntiles;
  auto tile_beg = [&](int t) { return 2 * (int)(((long long)t * half) / a.ntiles); };
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  unsigned parity = 0;  // bit s = parity of the next completion of ring slot s
  int phase = 0;
#pragma unroll 1
  for (int w = blockIdx.x; w < total; w += gridDim.x) {
    const int tile = w % a.ntiles, ch = w / a.ntiles;
    const int r0 = ch * chunk, r1 = min(nrows, r0 + chunk);  // residual rows r0+1 .. r1
    const int abeg = tile_beg(tile), T = tile_beg(tile + 1) - abeg;
    int start = abeg - a.HL;
    if (start < 0) start += nx;
    const int n1 = (start + W <= nx) ? W : nx - start;
    auto issue = [&](int row, int slot) {  // thread 0: guess row `row` -> ring slot
      const double *src = a.in.base + (a.in.off + (long long)row * a.in.stride) * (long long)nx;
      double *dst = smem + slot * W;
      mbar_expect_tx(&bar[slot], (uint32_t)W * 8u);
      tma_load_1d(dst, src + start, (uint32_t)n1 * 8u, &bar[slot]);
      if (n1 < W) tma_load_1d(dst + n1, src, (uint32_t)(W - n1) * 8u, &bar[slot]);
    };
    __syncthreads();  // previous item's readers are done with every slot
    if (tid == 0) {
      issue(r0, 0);
      issue(r0 + 1, 1);
    }
    double sacc = 0.0;
    int s_in = 0;
#pragma unroll 1
    for (int n = r0; n < r1; ++n) {
      const int s_cmp = (s_in + 1) % 3, s_next = (s_in + 2) % 3;
      mbar_wait(&bar[s_in], (parity >> s_in) & 1u);
      double x[P];
#pragma unroll
      for (int p = 0; p < P; ++p) x[p] = smem[s_in * W + tid * P + p];
      if (tid == 0 && n + 2 <= r1) issue(n + 2, s_next);   // slot s_next was read last row
      erk_step<SC, P, NT>(x, a.co, edge, phase);
      mbar_wait(&bar[s_cmp], (parity >> s_cmp) & 1u);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const double d = x[p] - smem[s_cmp * W + tid * P + p];
        const int l = tid * P + p;
        if (l >= a.HL && l < a.HL + T) sacc = fma(d, d, sacc);
      }
      parity ^= 1u << s_in;  // the input slot's completion is consumed
      s_in = s_cmp;
    }
    parity ^= 1u << s_in;  // ... and the last comparison row's
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(FULL, sacc, o);
    if ((tid & 31) == 0) a.partials[((long long)ch * a.ntiles + tile) * NW + (tid >> 5)] = sacc;
  }
}

template <class SC, int NT, int P>
static cudaError_t launch_residual_one(const SweepArgs &a, int chunk, cudaStream_t s) {
  constexpr int W = NT * P;
  const size_t smem = sizeof(double) * (3 * W + 2 * NT * (SC::NL + SC::NR) + 4) + 64;
  static int blocks_per_sm = 0;
  if (!blocks_per_sm) {
    cudaFuncSetAttribute(rk_residual_tma_kernel<SC, NT, P>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, rk_residual_tma_kernel<SC, NT, P>,
                                                  NT, smem);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long total = (long long)((a.nitems + chunk - 1) / chunk) * a.ntiles;
  if (total <= 0) return cudaSuccess;
  const long long grid = std::min<long long>(
      total, (long long)std::max(1, sms - a.reserve_sms) *
                 (a.max_per_sm > 0 ? std::min(a.max_per_sm, blocks_per_sm) : blocks_per_sm));
  rk_residual_tma_kernel<SC, NT, P><<<(unsigned)grid, NT, smem, s>>>(a, chunk);
  return cudaGetLastError();
}

template <class SC>
static cudaError_t dispatch_residual(SweepCfg c, const SweepArgs &a, int chunk, cudaStream_t s) {
#define MG_CASE(NT_, P_) \
  if (c.nt_threads == NT_ && c.p == P_) return launch_residual_one<SC, NT_, P_>(a, chunk, s);
  MG_TMA_CFGS(MG_CASE)
#undef MG_CASE
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_rk_residual_tma(int scheme, SweepCfg cfg, const SweepArgs &a, int chunk,
                                   cudaStream_t s) {
  switch (scheme) {
    case 0: return dispatch_residual<ERK1U1>(cfg, a, chunk, s);
    case 1: return dispatch_residual<ERK2U2>(cfg, a, chunk, s);
    case 2: return dispatch_residual<ERK3U3>(cfg, a, chunk, s);
    case 3: return dispatch_residual<ERK4U4>(cfg, a, chunk, s);
    case 4: return dispatch_residual<ERK5U5>(cfg, a, chunk, s);
    default: return cudaErrorInvalidValue;
  }
}

template <class SC> struct SchemeId;

int rk_scheme_reach_left(int scheme) {
  const int t[] = {ERK1U1::NL, ERK2U2::NL, ERK3U3::NL, ERK4U4::NL, ERK5U5::NL,
                   SDIRK1U1::NL, SDIRK2U2::NL, SDIRK3U3::NL, SDIRK4U4::NL};
  return (scheme >= 0 && scheme < 9) ? t[scheme] : -1;
}
int rk_scheme_reach_right(int scheme) {
  const int t[] = {ERK1U1::NR, ERK2U2::NR, ERK3U3::NR, ERK4U4::NR, ERK5U5::NR,
                   SDIRK1U1::NR, SDIRK2U2::NR, SDIRK3U3::NR, SDIRK4U4::NR};
  return (scheme >= 0 && scheme < 9) ? t[scheme] : -1;
}
int rk_scheme_stages(int scheme) {
  const int t[] = {ERK1U1::S, ERK2U2::S, ERK3U3::S, ERK4U4::S, ERK5U5::S,
                   SDIRK1U1::S, SDIRK2U2::S, SDIRK3U3::S, SDIRK4U4::S};
  return (scheme >= 0 && scheme < 9) ? t[scheme] : -1;
}
bool rk_scheme_implicit(int scheme) { return scheme >= 5 && scheme < 9; }

#define MG_CFGS(X)                                                                          \
  X(32, 2) X(32, 4) X(32, 8) X(64, 8) X(128, 8) X(256, 8) X(512, 8) X(128, 11) X(256, 11) X(128, 15)

template <class SC>
static cudaError_t dispatch_cfg(SweepCfg c, const SweepArgs &a, cudaStream_t s) {
#define MG_CASE(NT_, P_) \
  if (c.nt_threads == NT_ && c.p == P_) return launch_one<SC, NT_, P_>(a, s);
  MG_CFGS(MG_CASE)
#undef MG_CASE
  return cudaErrorInvalidConfiguration;
}

#define MG_IMPL_CFGS(X) X(32, 2) X(32, 4) X(32, 8) X(64, 8) X(128, 8) X(256, 8) X(512, 8) X(256, 16)
template <class SC>
static cudaError_t dispatch_implicit(SweepCfg c, const SweepArgs &a, cudaStream_t s) {
  // cfg4's production shape (SDIRK3+U3, 4096-point rows, three real factors, scan depth 8,
  // warp-local carries): the fused solve's structure fixed at compile time
  if constexpr (std::is_same<SC, SDIRK3U3>::value) {
    if (c.nt_threads == 256 && c.p == 16 && a.sd.fused && a.sd.ncrec == 0 && a.sd.dmax == 8 &&
        a.sd.warp_local)
      return launch_one<SC, 256, 16, FusedSpec<8, 1, 0, 1>>(a, s);
  }
#define MG_CASE(NT_, P_) \
  if (c.nt_threads == NT_ && c.p == P_) return launch_one<SC, NT_, P_>(a, s);
  MG_IMPL_CFGS(MG_CASE)
#undef MG_CASE
  return cudaErrorInvalidConfiguration;
}

bool rk_sweep_supported(int scheme, SweepCfg c) {
  if (scheme < 0 || scheme > 8) return false;
  if (scheme >= 5 && c.p == 11) return false;  // implicit: whole periodic rows only
  if (c.nt_threads == 256 && c.p == 16) return scheme >= 5;  // implicit-only configuration
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
    case 5: return dispatch_implicit<SDIRK1U1>(cfg, a, s);
    case 6: return dispatch_implicit<SDIRK2U2>(cfg, a, s);
    case 7: return dispatch_implicit<SDIRK3U3>(cfg, a, s);
    case 8: return dispatch_implicit<SDIRK4U4>(cfg, a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mg
