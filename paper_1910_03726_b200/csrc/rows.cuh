// rows.cuh — the whole-row / per-thread-copy relaxation sweep kernel (rk_sweep_kernel) and its
// launcher, shared by sweep.cu (periodic rows, halo tiles) and bounded.cu (inflow/outflow
// rows, BND = true; PAPER.md 4.5, R20).
#pragma once
#include "kernels.h"
#include "tma.cuh"

#include <algorithm>

namespace mg {

// One step of Phi: explicit stage form, or SDIRK with periodic banded stage solves.
template <class SC, int P, int NT, class FS = FusedRT, bool BND = false>
__device__ __forceinline__ void phi_step(double (&x)[P], const SweepArgs &a, double *edge,
                                         int &phase, double *wbuf, int &wphase) {
  if constexpr (SC::implicit)
    dirk_step<SC, P, NT, FS>(x, a.co, a.sd, edge, phase, wbuf, wphase);
  else
    erk_step<SC, P, NT, BND>(x, a.co, edge, phase);
}

// Persistent: each CTA walks work items (item, tile) with a grid stride and prefetches
// the next item's input / comparison windows with per-thread cp.async copies (padded
// layout) into the other buffer pair while it computes the current one, so a whole-row
// CTA (one per SM for the 512-thread SDIRK and ERK5 rows) never idles on a cold load.
// BND (inflow/outflow rows, ntiles == 1, W == nx): Phi = Phi_h + forcing.  Phase-1 step i of
// item j is U[n+1] = Phi_h U[n] + b_n with n = f_off + j*f_stride + i - 1, b_n the compact
// forcing row a.forc[n*FORC_LD .. +nb) on the row's first nb points (null: homogeneous);
// phase 2 acts on delta and is homogeneous.
template <class SC, int NT, int P, class FS = FusedRT, bool BND = false>
__global__ void __launch_bounds__(NT, 1) rk_sweep_kernel(const __grid_constant__ SweepArgs a) {
  constexpr int SP = Pad<P>::SP;
  constexpr int W = NT * P;
  constexpr int NW = NT / 32;
  extern __shared__ double smem[];
  double *bufA = smem;                   // [2][NT*SP] input windows
  double *bufB = bufA + 2 * NT * SP;     // [2][NT*SP] comparison windows
  double *edge = bufB + 2 * NT * SP;
  double *red = edge + 2 * NT * (SC::NL + SC::NR) + 2;
  double *wbuf = red + NW + 2;  // 16*NW (SDIRK recurrences: 2 phases x <= 8 slots) + lane tables
  int wphase = 0;
  const int nx = a.nx;
  const int total = a.nitems * a.ntiles;
  const int tid = threadIdx.x;
  int phase = 0;

  auto rowp = [&](const RowMap &r, long long j) -> const double * {
    return r.base + (r.off + j * r.stride) * (long long)nx;
  };
  auto span = [&](int w, int &item, int &abeg, int &T, int &start) {
    item = w / a.ntiles;
    const int tile = w - item * a.ntiles;
    abeg = (int)(((long long)tile * nx) / a.ntiles);
    T = (int)(((long long)(tile + 1) * nx) / a.ntiles) - abeg;
    start = abeg - a.HL;
    if (start < 0) start += nx;
  };
  // this thread's copies of item w's windows into buffer pair b (one cp.async group)
  auto issue = [&](int w, int b) {
    if (w < total) {
      int item, abeg, T, start;
      span(w, item, abeg, T, start);
      const double *ri = a.in.base ? rowp(a.in, item) : nullptr;
      const double *rc = a.cmp.base ? rowp(a.cmp, item) : nullptr;
      for (int q = tid; q < W; q += NT) {
        int g = start + q;
        if (g >= nx) g -= nx;
        if (ri) cp_async8(bufA + b * NT * SP + pidx<P>(q), ri + g);
        if (rc) cp_async8(bufB + b * NT * SP + pidx<P>(q), rc + g);
      }
    }
    cp_async_commit();
  };
  if constexpr (SC::implicit)
    if (a.sd.fused) fused_lane_tables<SC::NL, SC::NR, NT>(a.sd, wbuf);
  issue(blockIdx.x, 0);
  int it = 0;
#pragma unroll 1
  for (int w = blockIdx.x; w < total; w += gridDim.x, ++it) {
    const int b = it & 1;
    issue(w + gridDim.x, b ^ 1);          // buffers b^1 were released by the last barrier
    cp_async_wait<1>();                   // this thread's copies of item w landed
    __syncthreads();                      // ... and everybody else's
    double *sA = bufA + b * NT * SP, *sB = bufB + b * NT * SP;
    int item, abeg, T, start;
    span(w, item, abeg, T, start);
    // Store the T owned outputs [abeg, aend) of a register vector (coalesced via sA).
    auto store_slice = [&](double *row, const double(&v)[P]) {
      __syncthreads();
#pragma unroll
      for (int p = 0; p < P; ++p) sA[tid * SP + p] = v[p];
      __syncthreads();
      for (int q = tid; q < T; q += NT) row[abeg + q] = sA[pidx<P>(a.HL + q)];
    };
    double x[P];
#pragma unroll
    for (int p = 0; p < P; ++p) x[p] = a.in.base ? sA[tid * SP + p] : 0.0;

    // ---- phase 1: nsteps1 steps of Phi --------------------------------------
    if (a.each_first == 0 && a.each_last >= 0)
      store_slice(const_cast<double *>(a.each.base) +
                      (a.each.off + item * a.each.stride) * (long long)nx, x);
#pragma unroll 1
    for (int i = 1; i <= a.nsteps1; ++i) {
      double fb[P];
      if constexpr (BND) {  // forcing row of this step, in flight during the step
        const double *fr = a.forc ? a.forc + (a.f_off + item * a.f_stride + (i - 1)) * FORC_LD : nullptr;
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const int l = tid * P + p;
          fb[p] = (fr && l < a.nb) ? __ldg(fr + l) : 0.0;
        }
      }
      phi_step<SC, P, NT, FS, BND>(x, a, edge, phase, wbuf, wphase);
      if constexpr (BND) {
#pragma unroll
        for (int p = 0; p < P; ++p) x[p] += fb[p];
      }
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
        if (tid == 0) a.partials[w] = s;
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
        for (int i = 1; i <= a.nsteps2; ++i)
          phi_step<SC, P, NT, FS, BND>(x, a, edge, phase, wbuf, wphase);
        store_slice(const_cast<double *>(rowp(a.r2, item)), x);
      }
    }
    __syncthreads();                      // buffers b (and the staging in sA) are free
  }
  cp_async_wait<0>();
}


template <class SC, int NT, int P, class FS = FusedRT, bool BND = false>
static cudaError_t launch_one(const SweepArgs &a, cudaStream_t s) {
  constexpr int SP = Pad<P>::SP;
  const size_t smem = sizeof(double) * (4 * NT * SP + 2 * NT * (SC::NL + SC::NR) + 2 +
                                        NT / 32 + 2 + 16 * (NT / 32) + 8 * 32 + 2);
  static int blocks_per_sm = 0;
  if (!blocks_per_sm) {
    cudaFuncSetAttribute(rk_sweep_kernel<SC, NT, P, FS, BND>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, rk_sweep_kernel<SC, NT, P, FS, BND>, NT, smem);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long total = (long long)a.nitems * a.ntiles;
  if (total <= 0) return cudaSuccess;
  const long long grid = std::min<long long>(
      total, (long long)std::max(1, sms - a.reserve_sms) *
                 (a.max_per_sm > 0 ? std::min(a.max_per_sm, blocks_per_sm) : blocks_per_sm));
  rk_sweep_kernel<SC, NT, P, FS, BND><<<(unsigned)grid, NT, smem, s>>>(a);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------
// RK-form coarse operator (IDEAL = q fine steps, REDISC = one step at CFL m*c),
// sequential over nsteps, whole row, one CTA.  BND: the homogeneous inflow/outflow operator.
template <class SC, int NT, int P, bool BND = false>
__global__ void __launch_bounds__(NT, 1) rk_coarse_kernel(const __grid_constant__ RKCoarseArgs a) {
  extern __shared__ double smem[];
  double *edge = smem;
  double *wbuf = edge + 2 * NT * (SC::NL + SC::NR) + 2;  // SDIRK recurrences + lane tables
  int wphase = 0;
  const int tid = threadIdx.x, nx = a.nx;
  int phase = 0;
  if constexpr (SC::implicit) {
    if (a.sd.fused) fused_lane_tables<SC::NL, SC::NR, NT>(a.sd, wbuf);
    __syncthreads();
  }
  // one coarse step = q steps of the (explicit or SDIRK) Runge-Kutta propagator
  auto rk = [&](double(&x)[P]) {
    if constexpr (SC::implicit) dirk_step<SC, P, NT>(x, a.co, a.sd, edge, phase, wbuf, wphase);
    else erk_step<SC, P, NT, BND>(x, a.co, edge, phase);
  };
  double x[P];
#pragma unroll
  for (int p = 0; p < P; ++p) x[p] = 0.0;
  // Short rows (ring_b > 0: nx <= 512, contiguous g and v rows): a step takes a few tens of
  // nanoseconds, far less than a global load, so the rows come in blocks of ring_b steps by
  // bulk copies into a double-buffered shared-memory ring (one mbarrier per buffer), one
  // block ahead of the chain; a step then only reads shared memory.
  if (a.ring_b > 0) {
    const int B = a.ring_b, N = a.nsteps;
    double *ring = wbuf + 16 * (NT / 32) + 8 * 32 + 2;
    ring += (reinterpret_cast<uintptr_t>(ring) & 8) ? 1 : 0;            // 16-byte aligned
    uint64_t *bar = reinterpret_cast<uint64_t *>(ring + 4 * (size_t)B * nx);
    auto issue = [&](int blk) {  // thread 0: rows n0 .. n0+cnt-1 of g (and v) -> buffer blk & 1
      const int n0 = 1 + blk * B;
      if (n0 > N) return;
      const int cnt = min(B, N - n0 + 1), buf = blk & 1;
      const uint32_t bytes = (uint32_t)cnt * (uint32_t)nx * 8u;
      mbar_expect_tx(&bar[buf], a.v.base ? 2u * bytes : bytes);
      tma_load_1d(ring + (size_t)(2 * buf) * B * nx, a.g.base + (a.g.off + n0) * (long long)nx, bytes, &bar[buf]);
      if (a.v.base)
        tma_load_1d(ring + (size_t)(2 * buf + 1) * B * nx, a.v.base + (a.v.off + n0) * (long long)nx, bytes,
                    &bar[buf]);
    };
    if (tid == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
      issue(0);
      issue(1);
    }
#pragma unroll 1
    for (int blk = 0; 1 + blk * B <= N; ++blk) {
      const int n0 = 1 + blk * B, cnt = min(B, N - n0 + 1), buf = blk & 1;
      mbar_wait(&bar[buf], (uint32_t)((blk >> 1) & 1));
      const double *gs = ring + (size_t)(2 * buf) * B * nx + tid * P;
      const double *vs = gs + (size_t)B * nx;
      // the next step's g and v values are read from shared memory before the current step's
      // arithmetic (a lone warp issues in order: the load latency then hides behind the step)
      double *o = const_cast<double *>(a.out.base) + (a.out.off + (long long)n0 * a.out.stride) * nx + tid * P;
      const long long ostep = a.out.stride * (long long)nx;
      double gn[P], vn[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        gn[p] = gs[p];
        vn[p] = a.v.base ? vs[p] : 0.0;
      }
#pragma unroll 2
      for (int d = 0; d < cnt; ++d) {
        double gc[P], vc[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          gc[p] = gn[p];
          vc[p] = vn[p];
        }
        if (d + 1 < cnt) {
#pragma unroll
          for (int p = 0; p < P; ++p) {
            gn[p] = gs[(d + 1) * nx + p];
            vn[p] = a.v.base ? vs[(d + 1) * nx + p] : 0.0;
          }
        }
#pragma unroll 1
        for (int r = 0; r < a.q; ++r) rk(x);
#pragma unroll
        for (int p = 0; p < P; ++p) {
          x[p] = x[p] + gc[p];
          o[p] = vc[p] + x[p];
        }
        o += ostep;
      }
      __syncthreads();                    // every thread has read buffer `buf`
      if (tid == 0) issue(blk + 2);
    }
    return;
  }
  // g_n and v_n do not depend on the chain: a register ring loads them D steps ahead, so
  // their latency (~1 us) overlaps D coarse steps (one-warp rows exchange by shuffles, no
  // barrier).  The ring is indexed at compile time: steps run in blocks of D.
  constexpr int D = SC::implicit ? 2 : ((16 / P) < 2 ? 2 : (16 / P));
  auto load = [&](int n, double(&gv)[P], double(&vv)[P]) {
    if (n > a.nsteps) return;
    const double *g = a.g.base + (a.g.off + (long long)n * a.g.stride) * nx;
    const double *v = a.v.base ? a.v.base + (a.v.off + (long long)n * a.v.stride) * nx : nullptr;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      gv[p] = g[tid * P + p];
      vv[p] = v ? v[tid * P + p] : 0.0;
    }
  };
  double gr[D][P], vr[D][P];
#pragma unroll
  for (int d = 0; d < D; ++d) load(1 + d, gr[d], vr[d]);
#pragma unroll 1
  for (int n0 = 1; n0 <= a.nsteps; n0 += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int n = n0 + d;
      if (n > a.nsteps) break;
#pragma unroll 1
      for (int r = 0; r < a.q; ++r) rk(x);
      double *o = const_cast<double *>(a.out.base) + (a.out.off + (long long)n * a.out.stride) * nx;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        x[p] = x[p] + gr[d][p];
        o[tid * P + p] = a.v.base ? vr[d][p] + x[p] : x[p];
      }
      load(n + D, gr[d], vr[d]);                  // slot d: D - 1 steps of lead
    }
  }
}

template <class SC, bool BND = false>
static cudaError_t launch_rkc(SweepCfg c, const RKCoarseArgs &a, cudaStream_t s) {
  size_t smem = sizeof(double) * (2 * c.nt_threads * (SC::NL + SC::NR) + 4 +
                                  16 * (c.nt_threads / 32) + 8 * 32 + 2);
  // short contiguous rows: shared-memory block ring of ring_b steps (4 arrays of <= 2048 doubles)
  RKCoarseArgs b = a;
  b.ring_b = 0;
  if (a.nx <= 512 && a.nx % 2 == 0 && a.g.stride == 1 && (!a.v.base || a.v.stride == 1) &&
      a.nsteps >= 16) {
    b.ring_b = std::min(32, 2048 / a.nx);
    smem += sizeof(double) * (4 * (size_t)b.ring_b * a.nx + 2) + 2 * sizeof(uint64_t) + 16;
  }
#define MG_RKC(NT_, P_)                                                      \
  if (c.nt_threads == NT_ && c.p == P_) {                                    \
    if constexpr (!BND || P_ >= SC::NL + SC::NR + 1) {                       \
      if (smem > 48 * 1024)                                                  \
        cudaFuncSetAttribute(rk_coarse_kernel<SC, NT_, P_, BND>,             \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      rk_coarse_kernel<SC, NT_, P_, BND><<<1, NT_, smem, s>>>(b);            \
      return cudaGetLastError();                                             \
    } else {                                                                 \
      return cudaErrorInvalidConfiguration;                                  \
    }                                                                        \
  }
  MG_RKC(32, 2) MG_RKC(32, 4) MG_RKC(32, 8) MG_RKC(64, 8) MG_RKC(128, 8) MG_RKC(256, 8)
  MG_RKC(256, 16)
#undef MG_RKC
  return cudaErrorInvalidConfiguration;
}

}  // namespace mg
