// sdirk.cuh — batched periodic banded stage solves of SDIRK Runge-Kutta steps
// (PAPER.md P:135).
//
// Each SDIRK stage solves (I - a_ii Z) y = rhs with Z = dt L the periodic U_p stencil:
// a circulant band matrix M = sum_d m_d E^d (E = shift).  On the host its symbol
// polynomial is factored, M = (1/gamma) prod_in (1 - r E^-1) prod_out (1 - rho E),
// so M^-1 is a product of first-order *periodic* bidiagonal solves
//     forward   x_i = rho x_{i-1} + f_i      (|rho| < 1, roots inside the unit circle)
//     backward  x_i = rho x_{i+1} + f_i      (rho = 1/r, roots outside)
// Each bidiagonal solve is a parallel cyclic reduction (recursive doubling) across
// the CTA: a sequential pass over the thread's P points, a warp-shuffle scan of the
// chunk carries, a cross-warp pass, and the rank-1 periodic (Sherman-Morrison)
// closure c_0 = S / (1 - rho^N).  One __syncthreads per bidiagonal solve.
// A complex-conjugate root pair (SDIRK2+U2, SDIRK4+U4) is one complex recurrence on the
// real right-hand side: by partial fractions
//   (1 - rho s)^-1 (1 - conj(rho) s)^-1 f = Im(rho y) / Im(rho),  y = (1 - rho s)^-1 f
// (s = E^-1 forward, E backward), since (1 - conj(rho) s)^-1 f = conj(y) for real f.
#pragma once
#include "device.cuh"

namespace mg {

constexpr int MAXP = 16;
constexpr int MAXREC = 4;

struct RecCoef {
  double rpow[MAXP + 1];   // rho^k, k = 0..P
  double rchunk[33];       // (rho^P)^j, j = 0..32
  double rwarp[17];        // (rho^(32P))^w, w = 0..16 (fused form: cross-warp scan)
  double closure;          // 1 / (1 - rho^N), N = nx
  double alpha;            // fused form: gamma * partial-fraction weight of this factor
  int backward;            // 0: x_i = rho x_{i-1} + f_i ; 1: x_i = rho x_{i+1} + f_i
  int pad;
};

constexpr int MAXCREC = 2;

struct CRecCoef {            // complex rho = (re, im), |rho| < 1
  double rpr[MAXP + 1], rpi[MAXP + 1];   // rho^k
  double rcr[33], rci[33];               // (rho^P)^j
  double rwr[17], rwi[17];               // (rho^(32P))^w (fused form)
  double clr, cli;                       // 1 / (1 - rho^N)
  double ratio;                          // Re(rho) / Im(rho)
  double ar, ai;                         // fused form: 2 * gamma * weight (complex)
  int backward;
  int pad;
};

struct SdirkCoef {
  int nrec;
  int ncrec;
  int fused;               // 1: partial-fraction form (fused_stage_solve), 0: product form
  int nrf;                 // fused form: forward real factors in rec[0..nrf), backward after
  double gamma;            // M^-1 = gamma * prod (bidiagonal inverses)
  double beta;             // fused form: gamma * constant term of the partial fractions
  int dmax;                // fused form: warp-scan distances d < dmax (farther lanes' weights
                           //   (rho^P)^d < 2^-70 are below fp64 resolution), power of 2
  int warp_local;          // fused form: 1 if (rho^(32P)) < 2^-70 for every factor, so the
                           //   carry entering a warp is the previous warp's total alone
  RecCoef rec[MAXREC];
  CRecCoef crec[MAXCREC];  // one per complex-conjugate root pair
};

// In-place periodic first-order recurrence over the CTA's whole row (W == nx).
template <int P, int NT>
__device__ __forceinline__ void periodic_recurrence(double (&f)[P], const RecCoef &rc,
                                                    double *wbuf, int &wphase) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double rho = rc.rpow[1];
  const double mu32 = rc.rchunk[32];
  double *wb = wbuf + wphase * NW;
  if (!rc.backward) {
    double l[P];
    l[0] = f[0];
#pragma unroll
    for (int p = 1; p < P; ++p) l[p] = fma(rho, l[p - 1], f[p]);
    double A = l[P - 1];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double v = __shfl_up_sync(FULL, A, d);
      if (lane >= d) A = fma(rc.rchunk[d], v, A);
    }
    if (lane == 31) wb[warp] = A;
    __syncthreads();
    double tot = 0.0;
#pragma unroll 1
    for (int v = 0; v < NW; ++v) tot = fma(mu32, tot, wb[v]);
    double c = tot * rc.closure;                     // carry entering warp 0 (periodic)
#pragma unroll 1
    for (int v = 0; v < warp; ++v) c = fma(mu32, c, wb[v]);
    const double Aprev = __shfl_up_sync(FULL, A, 1);
    const double cin = (lane == 0) ? c : fma(rc.rchunk[lane], c, Aprev);
#pragma unroll
    for (int p = 0; p < P; ++p) f[p] = fma(rc.rpow[p + 1], cin, l[p]);
  } else {
    double l[P];
    l[P - 1] = f[P - 1];
#pragma unroll
    for (int p = P - 2; p >= 0; --p) l[p] = fma(rho, l[p + 1], f[p]);
    double B = l[0];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double v = __shfl_down_sync(FULL, B, d);
      if (lane + d < 32) B = fma(rc.rchunk[d], v, B);
    }
    if (lane == 0) wb[warp] = B;
    __syncthreads();
    double tot = 0.0;
#pragma unroll 1
    for (int v = NW - 1; v >= 0; --v) tot = fma(mu32, tot, wb[v]);
    double c = tot * rc.closure;                     // carry entering the last warp
#pragma unroll 1
    for (int v = NW - 1; v > warp; --v) c = fma(mu32, c, wb[v]);
    const double Bnext = __shfl_down_sync(FULL, B, 1);
    const double cin = (lane == 31) ? c : fma(rc.rchunk[31 - lane], c, Bnext);
#pragma unroll
    for (int p = 0; p < P; ++p) f[p] = fma(rc.rpow[P - p], cin, l[p]);
  }
  wphase ^= 1;
}

// Complex multiply-add helpers: (ar + i ai)(br + i bi) + (cr + i ci).
__device__ __forceinline__ void cfma(double ar, double ai, double br, double bi, double &cr,
                                     double &ci) {
  const double r = fma(ar, br, fma(-ai, bi, cr));
  ci = fma(ar, bi, fma(ai, br, ci));
  cr = r;
}

// In-place periodic complex-pair solve over the CTA's whole row: f <- Im(rho y)/Im(rho)
// with y the periodic solution of y_i = rho y_{i-1} + f_i (backward: y_{i+1}).
template <int P, int NT>
__device__ __forceinline__ void periodic_recurrence_cplx(double (&f)[P], const CRecCoef &rc,
                                                         double *wbuf, int &wphase) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double rr = rc.rpr[1], ri = rc.rpi[1];
  const double mr = rc.rcr[32], mi = rc.rci[32];
  double *wb = wbuf + wphase * 2 * NW;            // [NW] re, [NW] im
  double lr[P], li[P];
  const bool bwd = rc.backward != 0;
  if (!bwd) {
    lr[0] = f[0];
    li[0] = 0.0;
#pragma unroll
    for (int p = 1; p < P; ++p) {
      lr[p] = f[p];
      li[p] = 0.0;
      cfma(rr, ri, lr[p - 1], li[p - 1], lr[p], li[p]);
    }
  } else {
    lr[P - 1] = f[P - 1];
    li[P - 1] = 0.0;
#pragma unroll
    for (int p = P - 2; p >= 0; --p) {
      lr[p] = f[p];
      li[p] = 0.0;
      cfma(rr, ri, lr[p + 1], li[p + 1], lr[p], li[p]);
    }
  }
  // chunk carry of this thread, scanned across the warp
  double Ar = bwd ? lr[0] : lr[P - 1], Ai = bwd ? li[0] : li[P - 1];
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double vr = bwd ? __shfl_down_sync(FULL, Ar, d) : __shfl_up_sync(FULL, Ar, d);
    const double vi = bwd ? __shfl_down_sync(FULL, Ai, d) : __shfl_up_sync(FULL, Ai, d);
    if (bwd ? (lane + d < 32) : (lane >= d)) cfma(rc.rcr[d], rc.rci[d], vr, vi, Ar, Ai);
  }
  if (lane == (bwd ? 0 : 31)) {
    wb[warp] = Ar;
    wb[NW + warp] = Ai;
  }
  __syncthreads();
  double tr = 0.0, ti = 0.0;
  if (!bwd) {
#pragma unroll 1
    for (int v = 0; v < NW; ++v) {
      double nr = wb[v], ni = wb[NW + v];
      cfma(mr, mi, tr, ti, nr, ni);
      tr = nr; ti = ni;
    }
  } else {
#pragma unroll 1
    for (int v = NW - 1; v >= 0; --v) {
      double nr = wb[v], ni = wb[NW + v];
      cfma(mr, mi, tr, ti, nr, ni);
      tr = nr; ti = ni;
    }
  }
  double cr = 0.0, ci = 0.0;                       // carry entering the first warp
  cfma(tr, ti, rc.clr, rc.cli, cr, ci);
  if (!bwd) {
#pragma unroll 1
    for (int v = 0; v < warp; ++v) {
      double nr = wb[v], ni = wb[NW + v];
      cfma(mr, mi, cr, ci, nr, ni);
      cr = nr; ci = ni;
    }
  } else {
#pragma unroll 1
    for (int v = NW - 1; v > warp; --v) {
      double nr = wb[v], ni = wb[NW + v];
      cfma(mr, mi, cr, ci, nr, ni);
      cr = nr; ci = ni;
    }
  }
  const double Pr = bwd ? __shfl_down_sync(FULL, Ar, 1) : __shfl_up_sync(FULL, Ar, 1);
  const double Pi = bwd ? __shfl_down_sync(FULL, Ai, 1) : __shfl_up_sync(FULL, Ai, 1);
  double inr = cr, ini = ci;
  if (lane != (bwd ? 31 : 0)) {
    const int k = bwd ? 31 - lane : lane;
    inr = Pr;
    ini = Pi;
    cfma(rc.rcr[k], rc.rci[k], cr, ci, inr, ini);
  }
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int k = bwd ? P - p : p + 1;
    double yr = lr[p], yi = li[p];
    cfma(rc.rpr[k], rc.rpi[k], inr, ini, yr, yi);
    f[p] = fma(rc.ratio, yi, yr);                   // Im(rho y) / Im(rho)
  }
  wphase ^= 1;
}

// ---------------------------------------------------------------------------
// Fused (partial-fraction) stage solve.  The inverse symbol of the stage matrix,
//   1/m(z) = gamma prod_k 1/(1 - a_k z^-1) prod_l 1/(1 - b_l z)     (|a_k|, |b_l| < 1),
// is, for distinct roots, beta + sum_k A_k/(1 - a_k z^-1) + sum_l B_l/(1 - b_l z), so
// M^-1 f = beta f + sum of INDEPENDENT first-order periodic recurrences on the same f
// (weights computed on the host, mgrit_api.cu make_sdirk; used only when they are well
// conditioned).  All recurrences run in one pass: interleaved local chains, interleaved
// warp scans, ONE barrier, a shuffle scan of the warp carries (log2 NW steps instead of
// a serial loop), and the carry fix-up accumulates straight into y.
// Slots in wbuf (per phase): NL forward real (absent ones have rho = alpha = 0), then
// 2 per complex pair, then NR backward real.
// ---------------------------------------------------------------------------
template <int NW>
__device__ __forceinline__ double warp_carry_fwd(double t, const double *mu, double closure,
                                                 int warp, int lane) {
  // t = this lane's warp total (lane v < NW holds warp v's); returns the carry entering
  // `warp`: mu^warp * tot * closure + sum_{v<warp} mu^(warp-1-v) t_v
  double S = (lane < NW) ? t : 0.0;
#pragma unroll
  for (int d = 1; d < NW; d <<= 1) {
    const double v = __shfl_up_sync(FULL, S, d);
    if (lane >= d) S = fma(mu[d], v, S);
  }
  const double tot = __shfl_sync(FULL, S, NW - 1);
  const double prev = __shfl_sync(FULL, S, (warp + 31) & 31);
  return fma(mu[warp], tot * closure, warp ? prev : 0.0);
}

template <int NW>
__device__ __forceinline__ double warp_carry_bwd(double t, const double *mu, double closure,
                                                 int warp, int lane) {
  // carry entering `warp` from the right: mu^(NW-1-warp) * tot * closure
  //   + sum_{v>warp} mu^(v-warp-1) t_v,   tot = sum_v mu^v t_v
  double S = (lane < NW) ? t : 0.0;
#pragma unroll
  for (int d = 1; d < NW; d <<= 1) {
    const double v = __shfl_down_sync(FULL, S, d);
    if (lane + d < NW) S = fma(mu[d], v, S);
  }
  const double tot = __shfl_sync(FULL, S, 0);
  const double next = __shfl_sync(FULL, S, (warp + 1) & 31);
  return fma(mu[NW - 1 - warp], tot * closure, warp < NW - 1 ? next : 0.0);
}

template <int NW>
__device__ __forceinline__ void warp_carry_cplx(double tr, double ti, const CRecCoef &rc,
                                                int warp, int lane, double &cr, double &ci) {
  double Sr = (lane < NW) ? tr : 0.0, Si = (lane < NW) ? ti : 0.0;
#pragma unroll
  for (int d = 1; d < NW; d <<= 1) {
    const double vr = __shfl_up_sync(FULL, Sr, d);
    const double vi = __shfl_up_sync(FULL, Si, d);
    if (lane >= d) cfma(rc.rwr[d], rc.rwi[d], vr, vi, Sr, Si);
  }
  const double totr = __shfl_sync(FULL, Sr, NW - 1), toti = __shfl_sync(FULL, Si, NW - 1);
  const double pr = __shfl_sync(FULL, Sr, (warp + 31) & 31);
  const double pi = __shfl_sync(FULL, Si, (warp + 31) & 31);
  double c0r = 0.0, c0i = 0.0;
  cfma(totr, toti, rc.clr, rc.cli, c0r, c0i);
  cr = warp ? pr : 0.0;
  ci = warp ? pi : 0.0;
  cfma(rc.rwr[warp], rc.rwi[warp], c0r, c0i, cr, ci);
}

// Per-lane carry multipliers of the fused solve, built once per CTA in shared memory
// (lane-indexed constant-bank loads would serialise across the warp): slot k < NL:
// (rho_k^P)^lane; pair slots NL, NL+1: Re/Im (rho^P)^lane; backward slots:
// (rho^P)^(31-lane).  Layout [slot][32] at wbuf + 16*NW.
template <int NL, int NR, int NT>
__device__ __forceinline__ void fused_lane_tables(const SdirkCoef &sd, double *wbuf) {
  constexpr int NW = NT / 32;
  constexpr int NSLOT = NL + 2 * (NL / 2) + NR;
  double *lt = wbuf + 2 * 8 * NW;
  for (int t = threadIdx.x; t < NSLOT * 32; t += NT) {
    const int slot = t >> 5, l = t & 31;
    double v;
    if (slot < NL) v = sd.rec[slot].rchunk[l];
    else if (slot < NL + 2 * (NL / 2)) v = (slot == NL) ? sd.crec[0].rcr[l] : sd.crec[0].rci[l];
    else v = sd.rec[NL + (slot - NL - 2 * (NL / 2))].rchunk[31 - l];
    lt[t] = v;
  }
}

// Compile-time specialisation of the fused solve for a launch whose factor structure is
// known on the host (mgrit_api.cu make_sdirk): DMAX > 0 fixes the warp-scan depth, WL / PAIR
// >= 0 fix warp_local / the complex pair, FUSED = 1 drops the product-form branch.  The
// defaults read those fields at run time (every shape; FusedRT).
template <int DMAX = 0, int WL = -1, int PAIR = -1, int FUSED = 0>
struct FusedSpec {
  static constexpr int dmax = DMAX, wl = WL, pair = PAIR, fused = FUSED;
};
using FusedRT = FusedSpec<>;

template <int NL, int NR, int P, int NT, class FS = FusedRT>
__device__ __forceinline__ void fused_stage_solve(double (&f)[P], const SdirkCoef &sd,
                                                  double *wbuf, int &wphase) {
  constexpr int NW = NT / 32;
  constexpr int NSLOT = NL + 2 * (NL / 2) + NR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool pair = (NL >= 2) && (FS::pair >= 0 ? FS::pair == 1 : sd.ncrec > 0);  // warp-uniform
  double *wb = wbuf + wphase * NSLOT * NW;
  const double *lt = wbuf + 2 * 8 * NW;            // lane tables (fused_lane_tables)
  double y[P];
#pragma unroll
  for (int p = 0; p < P; ++p) y[p] = sd.beta * f[p];
  // ---- local chains (interleaved) -------------------------------------------------
  double A[NL], Br[NR > 0 ? NR : 1];
  double Cr = 0.0, Ci = 0.0;
#pragma unroll
  for (int k = 0; k < NL; ++k) A[k] = f[0];
#pragma unroll
  for (int p = 0; p < P; ++p) {
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      if (p > 0) A[k] = fma(sd.rec[k].rpow[1], A[k], f[p]);
      y[p] = fma(sd.rec[k].alpha, A[k], y[p]);
    }
  }
  if constexpr (NL >= 2) {
    if (pair) {
      const CRecCoef &rc = sd.crec[0];
      Cr = f[0];
      Ci = 0.0;
      y[0] = fma(rc.ar, Cr, y[0]);
#pragma unroll
      for (int p = 1; p < P; ++p) {
        double nr = f[p], ni = 0.0;
        cfma(rc.rpr[1], rc.rpi[1], Cr, Ci, nr, ni);
        Cr = nr;
        Ci = ni;
        y[p] = fma(rc.ar, Cr, fma(-rc.ai, Ci, y[p]));
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    const RecCoef &rc = sd.rec[NL + k];
    Br[k] = f[P - 1];
    y[P - 1] = fma(rc.alpha, Br[k], y[P - 1]);
#pragma unroll
    for (int p = P - 2; p >= 0; --p) {
      Br[k] = fma(rc.rpow[1], Br[k], f[p]);
      y[p] = fma(rc.alpha, Br[k], y[p]);
    }
  }
  // ---- warp scans of the chunk totals (interleaved) --------------------------------
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    if (d >= (FS::dmax > 0 ? FS::dmax : sd.dmax)) break;  // warp-uniform
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const double v = __shfl_up_sync(FULL, A[k], d);
      if (lane >= d) A[k] = fma(sd.rec[k].rchunk[d], v, A[k]);
    }
    if constexpr (NL >= 2) {
      if (pair) {
        const double vr = __shfl_up_sync(FULL, Cr, d), vi = __shfl_up_sync(FULL, Ci, d);
        if (lane >= d) cfma(sd.crec[0].rcr[d], sd.crec[0].rci[d], vr, vi, Cr, Ci);
      }
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      const double v = __shfl_down_sync(FULL, Br[k], d);
      if (lane + d < 32) Br[k] = fma(sd.rec[NL + k].rchunk[d], v, Br[k]);
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int k = 0; k < NL; ++k) wb[k * NW + warp] = A[k];
    if constexpr (NL >= 2) {
      wb[NL * NW + warp] = Cr;
      wb[(NL + 1) * NW + warp] = Ci;
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NR; ++k) wb[(NL + 2 * (NL / 2) + k) * NW + warp] = Br[k];
  }
  __syncthreads();
  const int ld = lane < NW ? lane : 0;
  const bool wl = FS::wl >= 0 ? FS::wl == 1 : sd.warp_local != 0;
  const int wprev = (warp + NW - 1) % NW, wnext = (warp + 1) % NW;
  // ---- carries entering the warp, then entering the lane; fix-up into y ------------
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    const RecCoef &rc = sd.rec[k];
    const double cw = wl ? wb[k * NW + wprev] * (warp ? 1.0 : rc.closure)
                         : warp_carry_fwd<NW>(wb[k * NW + ld], rc.rwarp, rc.closure, warp, lane);
    const double Ap = __shfl_up_sync(FULL, A[k], 1);
    const double cin = (lane == 0) ? cw : fma(lt[k * 32 + lane], cw, Ap);
    const double ac = rc.alpha * cin;
#pragma unroll
    for (int p = 0; p < P; ++p) y[p] = fma(rc.rpow[p + 1], ac, y[p]);
  }
  if constexpr (NL >= 2) {
    if (pair) {
      const CRecCoef &rc = sd.crec[0];
      double cr, ci;
      if (wl) {
        const double tr = wb[NL * NW + wprev], ti = wb[(NL + 1) * NW + wprev];
        cr = tr;
        ci = ti;
        if (!warp) {
          cr = 0.0;
          ci = 0.0;
          cfma(tr, ti, rc.clr, rc.cli, cr, ci);
        }
      } else {
        warp_carry_cplx<NW>(wb[NL * NW + ld], wb[(NL + 1) * NW + ld], rc, warp, lane, cr, ci);
      }
      const double Pr = __shfl_up_sync(FULL, Cr, 1), Pi = __shfl_up_sync(FULL, Ci, 1);
      double inr = cr, ini = ci;
      if (lane != 0) {
        inr = Pr;
        ini = Pi;
        cfma(lt[NL * 32 + lane], lt[(NL + 1) * 32 + lane], cr, ci, inr, ini);
      }
      double acr = 0.0, aci = 0.0;                   // (2 gamma A) * cin
      cfma(rc.ar, rc.ai, inr, ini, acr, aci);
#pragma unroll
      for (int p = 0; p < P; ++p) y[p] = fma(rc.rpr[p + 1], acr, fma(-rc.rpi[p + 1], aci, y[p]));
    }
  }
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    const RecCoef &rc = sd.rec[NL + k];
    const int slot = NL + 2 * (NL / 2) + k;
    const double cw = wl ? wb[slot * NW + wnext] * (warp < NW - 1 ? 1.0 : rc.closure)
                         : warp_carry_bwd<NW>(wb[slot * NW + ld], rc.rwarp, rc.closure, warp, lane);
    const double Bn = __shfl_down_sync(FULL, Br[k], 1);
    const double cin = (lane == 31) ? cw : fma(lt[slot * 32 + lane], cw, Bn);
    const double ac = rc.alpha * cin;
#pragma unroll
    for (int p = 0; p < P; ++p) y[p] = fma(rc.rpow[P - p], ac, y[p]);
  }
#pragma unroll
  for (int p = 0; p < P; ++p) f[p] = y[p];
  wphase ^= 1;
}

template <int P, int NT>
__device__ __forceinline__ void stage_solve(double (&y)[P], const SdirkCoef &sd, double *wbuf,
                                            int &wphase) {
#pragma unroll 1
  for (int k = 0; k < sd.nrec; ++k) periodic_recurrence<P, NT>(y, sd.rec[k], wbuf, wphase);
#pragma unroll 1
  for (int k = 0; k < sd.ncrec; ++k) periodic_recurrence_cplx<P, NT>(y, sd.crec[k], wbuf, wphase);
#pragma unroll
  for (int p = 0; p < P; ++p) y[p] *= sd.gamma;
}

// One SDIRK step in stage form (b-form update, R14):
//   (I - a_ii Z) y_i = x + sum_{l<i} a_il k_l,   k_i = Z y_i,   x <- x + sum_i b_i k_i.
template <class SC, int P, int NT, class FS = FusedRT>
__device__ __forceinline__ void dirk_step(double (&x)[P], const RKCoeffs &c, const SdirkCoef &sd,
                                          double *edge, int &phase, double *wbuf, int &wphase) {
  constexpr int S = SC::S;
  double acc[S][P];
  double out[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    out[p] = x[p];
#pragma unroll
    for (int i = 0; i < S; ++i) acc[i][p] = x[p];
  }
#pragma unroll
  for (int i = 0; i < S; ++i) {
    if (FS::fused == 1 || sd.fused)
      fused_stage_solve<SC::NL, SC::NR, P, NT, FS>(acc[i], sd, wbuf, wphase);
    else
      stage_solve<P, NT>(acc[i], sd, wbuf, wphase);
    double k[P];
    apply_Z<SC::NL, SC::NR, P, NT>(acc[i], k, c.z, edge, phase);
#pragma unroll
    for (int l = i + 1; l < S; ++l) {
      if (SC::a_nz(l, i)) {
#pragma unroll
        for (int p = 0; p < P; ++p) acc[l][p] = fma(c.A[l][i], k[p], acc[l][p]);
      }
    }
    if (SC::b_nz(i)) {
#pragma unroll
      for (int p = 0; p < P; ++p) out[p] = fma(c.b[i], k[p], out[p]);
    }
  }
#pragma unroll
  for (int p = 0; p < P; ++p) x[p] = out[p];
}

// SDIRKp + Up pairs (strictly-lower A pattern; the diagonal is the stage solve).
using SDIRK1U1 = Scheme<1, 1, 0, 0ull, 0x1u, true>;
using SDIRK2U2 = Scheme<2, 2, 0, abit(1, 0), 0x3u, true>;
using SDIRK3U3 = Scheme<3, 2, 1, abit(1, 0) | abit(2, 0) | abit(2, 1), 0x7u, true>;
using SDIRK4U4 = Scheme<5, 3, 1,
                        abit(1, 0) | abit(2, 0) | abit(2, 1) | abit(3, 0) | abit(3, 1) |
                            abit(3, 2) | abit(4, 0) | abit(4, 1) | abit(4, 2) | abit(4, 3),
                        0x1Fu, true>;

}  // namespace mg
