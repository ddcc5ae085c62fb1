// mgrit_api.cu — C ABI (include/mgrit.h): validation, workspace carving, kernel
// orchestration of the MGRIT iteration.
//
// Production iteration:
//   hist[0] = ||r|| over all rows of the guess (R1)
//   sweep(u)             : v_{j+1} = Phi^m u_j, delta_{j+1} = v_{j+1} - u_{j+1} (norm),
//                          r_{j+2} = Phi^m delta_{j+1}              (FCF)
//   repeat: coarse correction (two-level sequential, or V-cycle)  -> u
//           sweep(u) -> ||r^(k)|| ; stop when < tol                (R2)
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges per solve / iteration / level / kernel class

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/mgrit.h"
#include "kernels.h"

using namespace mg;

cudaError_t mg_add_rows(double *dst, const double *a, const double *b, int n, cudaStream_t s);

namespace {

// Upwind stencils U1..U5: weights w_d for d = dmin..dmax and den.
struct Upwind {
  int dmin, dmax, den;
  int w[6];
};
const Upwind kUpwind[6] = {
    {0, 0, 1, {0}},
    {-1, 0, 1, {-1, 1}},                       // U1: u_i - u_{i-1}
    {-2, 0, 2, {1, -4, 3}},                    // U2: 3u_i - 4u_{i-1} + u_{i-2}
    {-2, 1, 6, {1, -6, 3, 2}},                 // U3: 2u_{i+1} + 3u_i - 6u_{i-1} + u_{i-2}
    {-3, 1, 12, {-1, 6, -18, 10, 3}},          // U4
    {-3, 2, 60, {-2, 15, -60, 20, 30, -3}},    // U5
};

struct Tab {
  int s;
  bool implicit;
  double A[MAXS][MAXS];
  double b[MAXS];
};

// Butcher tableaux (App. A).  Built at run time with plain IEEE
// operations (host compiled with -ffp-contract=off), R3.
bool make_tableau(int id, Tab &t) {
  std::memset(&t, 0, sizeof(t));
  switch (id) {
    case MGRIT_TAB_ERK1:
      t.s = 1; t.b[0] = 1.0; return true;
    case MGRIT_TAB_ERK2:
      t.s = 2; t.A[1][0] = 1.0; t.b[0] = 1.0 / 2.0; t.b[1] = 1.0 / 2.0; return true;
    case MGRIT_TAB_ERK3_SSP:
      t.s = 3; t.A[1][0] = 1.0; t.A[2][0] = 1.0 / 4.0; t.A[2][1] = 1.0 / 4.0;
      t.b[0] = 1.0 / 6.0; t.b[1] = 1.0 / 6.0; t.b[2] = 2.0 / 3.0; return true;
    case MGRIT_TAB_ERK3_KUTTA:
      t.s = 3; t.A[1][0] = 1.0 / 2.0; t.A[2][0] = -1.0; t.A[2][1] = 2.0;
      t.b[0] = 1.0 / 6.0; t.b[1] = 2.0 / 3.0; t.b[2] = 1.0 / 6.0; return true;
    case MGRIT_TAB_ERK4:
      t.s = 4; t.A[1][0] = 1.0 / 2.0; t.A[2][1] = 1.0 / 2.0; t.A[3][2] = 1.0;
      t.b[0] = 1.0 / 6.0; t.b[1] = 1.0 / 3.0; t.b[2] = 1.0 / 3.0; t.b[3] = 1.0 / 6.0; return true;
    case MGRIT_TAB_ERK5:
      t.s = 6;
      t.A[1][0] = 1.0 / 4.0;
      t.A[2][0] = 1.0 / 8.0; t.A[2][1] = 1.0 / 8.0;
      t.A[3][2] = 1.0 / 2.0;
      t.A[4][0] = 3.0 / 16.0; t.A[4][1] = -3.0 / 8.0; t.A[4][2] = 3.0 / 8.0; t.A[4][3] = 9.0 / 16.0;
      t.A[5][0] = -3.0 / 7.0; t.A[5][1] = 8.0 / 7.0; t.A[5][2] = 6.0 / 7.0;
      t.A[5][3] = -12.0 / 7.0; t.A[5][4] = 8.0 / 7.0;
      t.b[0] = 7.0 / 90.0; t.b[1] = 0.0; t.b[2] = 32.0 / 90.0; t.b[3] = 12.0 / 90.0;
      t.b[4] = 32.0 / 90.0; t.b[5] = 7.0 / 90.0;
      return true;
    case MGRIT_TAB_SDIRK1:
      t.s = 1; t.implicit = true; t.A[0][0] = 1.0; t.b[0] = 1.0; return true;
    case MGRIT_TAB_SDIRK2: {
      t.s = 2; t.implicit = true;
      const double g = 1.0 - std::sqrt(2.0) / 2.0, h = std::sqrt(2.0) / 2.0;
      t.A[0][0] = g; t.A[1][0] = h; t.A[1][1] = g; t.b[0] = h; t.b[1] = g; return true;
    }
    case MGRIT_TAB_SDIRK3: {
      t.s = 3; t.implicit = true;
      volatile double zeta = 0.43586652150845899942;
      const double beta = (1.0 - zeta) / 2.0;
      const double gamma = -1.5 * zeta * zeta + 4.0 * zeta - 0.25;
      const double eps = 1.5 * zeta * zeta - 5.0 * zeta + 1.25;
      t.A[0][0] = zeta; t.A[1][0] = beta; t.A[1][1] = zeta;
      t.A[2][0] = gamma; t.A[2][1] = eps; t.A[2][2] = zeta;
      t.b[0] = gamma; t.b[1] = eps; t.b[2] = zeta; return true;
    }
    case MGRIT_TAB_SDIRK4: {
      t.s = 5; t.implicit = true;
      const double A[5][5] = {{1.0 / 4.0, 0, 0, 0, 0},
                              {1.0 / 2.0, 1.0 / 4.0, 0, 0, 0},
                              {17.0 / 50.0, -1.0 / 25.0, 1.0 / 4.0, 0, 0},
                              {371.0 / 1360.0, -137.0 / 2720.0, 15.0 / 544.0, 1.0 / 4.0, 0},
                              {25.0 / 24.0, -49.0 / 48.0, 125.0 / 16.0, -85.0 / 12.0, 1.0 / 4.0}};
      for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j) t.A[i][j] = A[i][j];
      for (int j = 0; j < 5; ++j) t.b[j] = A[4][j];
      return true;
    }
  }
  return false;
}

// z_d = (-c * w_d) / den, d = dmin..dmax (R3), stored at index d - dmin.
void make_z(int order, double cfl, double *z, int *zlo, int *zn) {
  const Upwind &u = kUpwind[order];
  for (int d = u.dmin; d <= u.dmax; ++d) {
    const volatile double wd = (double)u.w[d - u.dmin];
    z[d - u.dmin] = (-cfl * wd) / (double)u.den;
  }
  *zlo = u.dmin;
  *zn = u.dmax - u.dmin + 1;
}

// b_{S-1} z_d for the explicit step's folded last stage, and the Shu-Osher-type form of
// a 3-stage ERK (SSP-RK3: a10 = 1, a20 = a21 = 1/4, b0 = b1 = 1/6, b2 = 2/3; device.cuh
// erk_step): y2 = x + a21 Z(x + y1) and x' = x + b0 Z(x + y1) + b2 Z y2
// = (1 - b0/a21) x + (b0/a21)(y2 + Z y2) when b0/a21 == b2 (R5, 6.1).  The form is
// used only when every coefficient it needs is exact in fp64 -- b0/a21 == b2 exactly,
// 1 - b2 + b2 == 1, a10 and a21 powers of two (so a10 z_d, a21 z_d are exact) -- because
// then it applies exactly the operator of the oracle's stage form with the same fp64
// coefficients (4 fl(1/6) = fl(2/3)); a rounded product coefficient would bias every step
// and drift linearly with nt (the measured 1.2e-12 at 65536 steps of the
// earlier form with b2 z_d products).
static bool pow2(double v) {
  int e;
  return v != 0.0 && std::fabs(std::frexp(v, &e)) == 0.5;
}
// Step forms (MGRIT_OPT_STAGE_FORM): 0 = production default, 1 = plain stage form,
// 2 = stage form with the folded last stage, 3 = Shu-Osher exact-operator form,
// 4 = incremental Shu-Osher form.
// Default: the incremental form (4).  Measured against the full-length cfg5 golden
// (8192 x 65536, tools/golden_forms.py): 1: 2.3e-13, 2: 1.7e-13, 3: 1.19e-12 (the product
// so0 * x rounds a full-size value every step, a bias the coarse chain accumulates), 4:
// 2.5e-13, at the speed of 3 (15 FP64 instructions per point-step for U3).
constexpr int kDefaultForm = 4;
static void fold_last_stage(RKCoeffs &co, int s, int form = 0) {
  if (form == 0) form = kDefaultForm;
  for (int d = 0; d < MAXZ; ++d) co.bz[d] = (s > 0) ? co.b[s - 1] * co.z[d] : 0.0;
  co.so3 = 0;
  co.fold = form == 1 ? 0 : 1;
  if (form <= 2) return;
  if (s != 3 || co.mdiag[0] != 0.0) return;
  const double a10 = co.A[1][0], a20 = co.A[2][0], a21 = co.A[2][1];
  const double b0 = co.b[0], b1 = co.b[1], b2 = co.b[2];
  if (a21 == 0.0 || a20 != a21 || b0 != b1 || !pow2(a10) || !pow2(a21)) return;
  const volatile double q = b0 / a21;
  const volatile double one_minus = 1.0 - b2;
  if (q != b2 || one_minus + b2 != 1.0) return;
  if (form == 4 && a10 != 1.0) return;
  co.so[1] = b2;
  co.so[0] = one_minus;
  for (int d = 0; d < MAXZ; ++d) {
    co.soz[0][d] = a10 * co.z[d];
    co.soz[1][d] = a21 * co.z[d];
    co.soz[2][d] = 0.0;
  }
  co.so3 = form == 4 ? 2 : 1;
}

int scheme_id(int tableau) {
  switch (tableau) {
    case MGRIT_TAB_ERK1: return 0;
    case MGRIT_TAB_ERK2: return 1;
    case MGRIT_TAB_ERK3_SSP:
    case MGRIT_TAB_ERK3_KUTTA: return 2;
    case MGRIT_TAB_ERK4: return 3;
    case MGRIT_TAB_ERK5: return 4;
    case MGRIT_TAB_SDIRK1: return 5;
    case MGRIT_TAB_SDIRK2: return 6;
    case MGRIT_TAB_SDIRK3: return 7;
    case MGRIT_TAB_SDIRK4: return 8;
    default: return -1;
  }
}

int tableau_order(int tableau) {
  switch (tableau) {
    case MGRIT_TAB_ERK1: case MGRIT_TAB_SDIRK1: return 1;
    case MGRIT_TAB_ERK2: case MGRIT_TAB_SDIRK2: return 2;
    case MGRIT_TAB_ERK3_SSP: case MGRIT_TAB_ERK3_KUTTA: case MGRIT_TAB_SDIRK3: return 3;
    case MGRIT_TAB_ERK4: case MGRIT_TAB_SDIRK4: return 4;
    case MGRIT_TAB_ERK5: return 5;
  }
  return -1;
}

// Roots of sum_k c[k] x^k (degree n <= 5) by Durand-Kerner in long double, polished by
// Newton steps; deterministic.
std::vector<std::complex<long double>> poly_roots(const std::vector<long double> &c) {
  typedef std::complex<long double> C;
  const int n = (int)c.size() - 1;
  std::vector<C> r(n);
  const C seed(0.4L, 0.9L);
  for (int k = 0; k < n; ++k) r[k] = std::pow(seed, k);
  auto eval = [&](C x) {
    C v = c[n];
    for (int k = n - 1; k >= 0; --k) v = v * x + (long double)c[k];
    return v;
  };
  auto deriv = [&](C x) {
    C v = (long double)n * c[n];
    for (int k = n - 1; k >= 1; --k) v = v * x + (long double)k * c[k];
    return v;
  };
  for (int it = 0; it < 500; ++it) {
    for (int k = 0; k < n; ++k) {
      C den = c[n];
      for (int j = 0; j < n; ++j)
        if (j != k) den *= (r[k] - r[j]);
      r[k] -= eval(r[k]) / den;
    }
  }
  for (int k = 0; k < n; ++k)
    for (int it = 0; it < 4; ++it) {
      const C d = deriv(r[k]);
      if (std::abs(d) > 0) r[k] -= eval(r[k]) / d;
    }
  return r;
}

// Factor M = I - a Z (periodic, stencil z_d at d = zlo..zlo+zn-1) into first-order periodic
// recurrences for the device stage solve (sdirk.cuh).  Returns false if the factorisation is
// not supported (complex roots, or winding number != 0).
// Partial-fraction (fused) form of the stage-matrix inverse (sdirk.cuh,
// fused_stage_solve).  With inside roots a_k (forward factors 1/(1 - a_k z^-1)) and
// b_l = 1/r_l for the outside roots r_l (backward factors 1/(1 - b_l z)):
//   A_k = prod_{j!=k} 1/(1 - a_j/a_k) prod_l 1/(1 - b_l a_k)   (residue at z = a_k)
//   B_l = prod_{j!=l} 1/(1 - b_j/b_l) prod_k 1/(1 - a_k b_l)   (residue at z = 1/b_l)
//   const = F(inf) - sum_k A_k,  F(inf) = 1 if there is no outside root, else 0.
// Used only when the weights are well conditioned (sum of |weights| <= 64), so the
// rounding of the sum stays within a few ulps of the product form's.
// Power tables of one real first-order factor of the fused form (host only).
static void fill_real_factor(RecCoef &rc, long double rho, long double alpha, bool bwd, int P,
                             int nx) {
  long double pk = 1.0L;
  for (int i = 0; i <= MAXP; ++i) {
    rc.rpow[i] = (i <= P) ? (double)pk : 0.0;
    pk *= rho;
  }
  const long double rP = powl(rho, (long double)P);
  long double pj = 1.0L;
  for (int j = 0; j <= 32; ++j) { rc.rchunk[j] = (double)pj; pj *= rP; }
  const long double mu = powl(rho, (long double)(32 * P));
  long double pw = 1.0L;
  for (int w = 0; w <= 16; ++w) { rc.rwarp[w] = (double)pw; pw *= mu; }
  rc.closure = (double)(1.0L / (1.0L - powl(rho, (long double)nx)));
  rc.alpha = (double)alpha;
  rc.backward = bwd ? 1 : 0;
}

void make_sdirk_fused(const std::vector<std::complex<long double>> &roots, long double gamma,
                      int NL, int P, int nx, SdirkCoef &sd) {
  typedef std::complex<long double> C;
  const C one(1.0L, 0.0L);
  std::vector<C> a, b;
  for (auto &r : roots) {
    if (std::abs(r) < 1.0L) a.push_back(r);
    else b.push_back(one / r);
  }
  const int NR = (int)b.size();
  std::vector<C> A(a.size()), B(b.size());
  long double cond = 0.0L;
  C cst = (NR == 0) ? one : C(0.0L, 0.0L);
  for (size_t k = 0; k < a.size(); ++k) {
    C w = one;
    for (size_t j = 0; j < a.size(); ++j)
      if (j != k) w /= (one - a[j] / a[k]);
    for (auto &bl : b) w /= (one - bl * a[k]);
    A[k] = w;
    cst -= w;
    cond += std::abs(w);
  }
  for (size_t l = 0; l < b.size(); ++l) {
    C w = one;
    for (size_t j = 0; j < b.size(); ++j)
      if (j != l) w /= (one - b[j] / b[l]);
    for (auto &ak : a) w /= (one - ak * b[l]);
    B[l] = w;
    cond += std::abs(w);
  }
  cond += std::abs(cst);
  sd.fused = 0;
  if (!(cond <= 64.0L) || NR > 1 || (int)a.size() != NL || NL + NR > MAXREC) return;
  // slots: rec[0..NL) forward real (then zero dummies), rec[NL..NL+NR) backward real,
  // crec[0] the complex pair (member with Im > 0)
  SdirkCoef f = sd;
  for (int k = 0; k < MAXREC; ++k) std::memset(&f.rec[k], 0, sizeof(RecCoef));
  for (int k = 0; k < MAXCREC; ++k) std::memset(&f.crec[k], 0, sizeof(CRecCoef));
  auto fill_real = [&](RecCoef &rc, long double rho, long double alpha, bool bwd) {
    fill_real_factor(rc, rho, alpha, bwd, P, nx);
  };
  int nrf = 0, npair = 0;
  std::vector<std::pair<long double, long double>> fr;  // (rho, alpha) forward real
  for (size_t k = 0; k < a.size(); ++k) {
    const long double im = a[k].imag();
    if (std::fabs((double)im) <= 1e-12 * std::max(1.0, (double)std::abs(a[k]))) {
      fr.push_back({a[k].real(), (gamma * A[k]).real()});
    } else if (im > 0) {
      if (npair >= 1) return;
      CRecCoef &rc = f.crec[npair++];
      const C rho = a[k];
      C pk = one;
      for (int i = 0; i <= MAXP; ++i) {
        rc.rpr[i] = (i <= P) ? (double)pk.real() : 0.0;
        rc.rpi[i] = (i <= P) ? (double)pk.imag() : 0.0;
        pk *= rho;
      }
      const C rP = std::pow(rho, (long double)P);
      C pj = one;
      for (int j = 0; j <= 32; ++j) { rc.rcr[j] = (double)pj.real(); rc.rci[j] = (double)pj.imag(); pj *= rP; }
      const C mu = std::pow(rho, (long double)(32 * P));
      C pw = one;
      for (int w = 0; w <= 16; ++w) { rc.rwr[w] = (double)pw.real(); rc.rwi[w] = (double)pw.imag(); pw *= mu; }
      const C cl = one / (one - std::pow(rho, (long double)nx));
      rc.clr = (double)cl.real();
      rc.cli = (double)cl.imag();
      const C w2 = 2.0L * gamma * A[k];
      rc.ar = (double)w2.real();
      rc.ai = (double)w2.imag();
    }
  }
  std::sort(fr.begin(), fr.end(), [](const std::pair<long double, long double> &x,
                                     const std::pair<long double, long double> &y) {
    return std::fabs(x.first) < std::fabs(y.first);
  });
  for (auto &pr : fr) fill_real(f.rec[nrf++], pr.first, pr.second, false);
  for (int k = nrf; k < NL; ++k) fill_real(f.rec[k], 0.0L, 0.0L, false);  // dummies
  for (int l = 0; l < NR; ++l) fill_real(f.rec[NL + l], b[l].real(), (gamma * B[l]).real(), true);
  f.nrf = nrf;
  f.ncrec = npair;
  f.nrec = NL + NR;
  f.beta = (double)(gamma * cst).real();
  // scan truncation: weights (rho^P)^d below 2^-70 are beyond fp64 resolution
  long double rmax = 0.0L;
  for (auto &x : a) rmax = std::max(rmax, (long double)std::abs(x));
  for (auto &x : b) rmax = std::max(rmax, (long double)std::abs(x));
  const long double tiny = ldexpl(1.0L, -70);
  f.dmax = 32;
  for (int d = 1; d < 32; d <<= 1)
    if (powl(rmax, (long double)(P * d)) < tiny) { f.dmax = d; break; }
  f.warp_local = powl(rmax, (long double)(32 * P)) < tiny ? 1 : 0;
  f.fused = 1;
  sd = f;
}

bool make_sdirk(const double *z, int zlo, int zn, double a, int P, int nx, SdirkCoef &sd,
                std::string &why, bool allow_fused) {
  std::memset(&sd, 0, sizeof(sd));
  // m_d = delta_d0 - a z_d; polynomial q(x) = sum_d m_d x^(d - zlo)
  std::vector<long double> q(zn);
  for (int k = 0; k < zn; ++k) {
    const int d = zlo + k;
    q[k] = -(long double)a * (long double)z[k] + (d == 0 ? 1.0L : 0.0L);
  }
  while (q.size() > 1 && q.back() == 0.0L) q.pop_back();
  const int deg = (int)q.size() - 1;
  const int NL = -zlo;
  auto roots = poly_roots(q);
  std::complex<long double> gamma_inv = q[deg];
  // real roots -> first-order factors; complex roots come in conjugate pairs -> one complex
  // factor each (sdirk.cuh), represented by the member with positive imaginary part
  std::vector<long double> rs;
  std::vector<std::complex<long double>> cs;
  int nin = 0;
  for (auto &r : roots) {
    const bool inside = std::abs(r) < 1.0L;
    if (inside) ++nin;
    if (std::fabs((double)r.imag()) <= 1e-12 * std::max(1.0, (double)std::abs(r))) {
      if (!inside) gamma_inv *= -r.real();
      rs.push_back(r.real());
    } else {
      if (!inside) gamma_inv *= -r;  // the pair contributes |r|^2 (real)
      if (r.imag() > 0) cs.push_back(r);
    }
  }
  if (2 * cs.size() + rs.size() != roots.size()) {
    why = "unpaired complex roots in the SDIRK stage matrix";
    return false;
  }
  if (nin != NL) {
    why = "stage matrix winding number != 0";
    return false;
  }
  if ((int)rs.size() > MAXREC || (int)cs.size() > MAXCREC) {
    why = "too many stage-matrix factors";
    return false;
  }
  sd.gamma = (double)(1.0L / gamma_inv.real());
  sd.nrec = (int)rs.size();
  sd.ncrec = (int)cs.size();
  int k = 0;
  // forward (inside) factors first, then backward (outside), in increasing |root|
  std::sort(rs.begin(), rs.end(), [](long double x, long double y) { return std::fabs(x) < std::fabs(y); });
  for (long double rr : rs) {
    RecCoef &rc = sd.rec[k++];
    const bool bwd = std::fabs(rr) >= 1.0L;
    const long double rho = bwd ? 1.0L / rr : rr;
    rc.backward = bwd ? 1 : 0;
    long double pk = 1.0L;
    for (int i = 0; i <= P; ++i) {
      rc.rpow[i] = (double)pk;
      pk *= rho;
    }
    const long double rP = powl(rho, (long double)P);
    long double pj = 1.0L;
    for (int j = 0; j <= 32; ++j) {
      rc.rchunk[j] = (double)pj;
      pj *= rP;
    }
    rc.closure = (double)(1.0L / (1.0L - powl(rho, (long double)nx)));
  }
  k = 0;
  for (auto &r : cs) {
    CRecCoef &rc = sd.crec[k++];
    const bool bwd = std::abs(r) >= 1.0L;
    const std::complex<long double> one(1.0L, 0.0L);
    const std::complex<long double> rho = bwd ? one / r : r;
    rc.backward = bwd ? 1 : 0;
    std::complex<long double> pk = one;
    for (int i = 0; i <= P; ++i) {
      rc.rpr[i] = (double)pk.real();
      rc.rpi[i] = (double)pk.imag();
      pk *= rho;
    }
    const std::complex<long double> rP = std::pow(rho, (long double)P);
    std::complex<long double> pj = one;
    for (int j = 0; j <= 32; ++j) {
      rc.rcr[j] = (double)pj.real();
      rc.rci[j] = (double)pj.imag();
      pj *= rP;
    }
    const std::complex<long double> cl = one / (one - std::pow(rho, (long double)nx));
    rc.clr = (double)cl.real();
    rc.cli = (double)cl.imag();
    rc.ratio = (double)(rho.real() / rho.imag());
  }
  if (allow_fused) make_sdirk_fused(roots, 1.0L / gamma_inv.real(), NL, P, nx, sd);
  return true;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Whole-row configuration of the RK-form coarse solve (rk_coarse_kernel): one CTA per row.
bool rk_coarse_cfg(int nx, SweepCfg &cfg) {
  if (nx == 64) cfg = {32, 2};
  else if (nx == 128) cfg = {32, 4};
  else if (nx == 256) cfg = {32, 8};
  else if (nx == 512) cfg = {64, 8};
  else if (nx == 1024) cfg = {128, 8};
  else if (nx == 2048) cfg = {256, 8};
  else if (nx == 4096) cfg = {256, 16};
  else return false;
  return true;
}

// Longest history the CUDA-graph solve keeps on the device (max_iter < kGraphHist).
constexpr int kGraphHist = 4096;

// Layout of the workspace (doubles unless noted).
struct Layout {
  size_t u0, v0, g[MGRIT_MAX_LEVELS], u2[MGRIT_MAX_LEVELS], ul[MGRIT_MAX_LEVELS];
  size_t partials, scal, sa, sb, hist, lstate, st_in, st_out, forc, prog, total;
  long long npart;
};

bool make_layout(int nx, int nt, int m, int levels, Layout &L) {
  if (nx < 2 || nt < 1 || m < 2 || levels < 2 || levels > MGRIT_MAX_LEVELS) return false;
  long long q = 1;
  for (int l = 0; l < levels - 1; ++l) {
    q *= m;
    if (q > nt || nt % q) return false;
  }
  size_t off = 0;
  const size_t row = (size_t)nx * sizeof(double);
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes); return o; };
  const long long nc0 = nt / m;
  L.u0 = take((nc0 + 1) * row);
  L.v0 = take((nc0 + 1) * row);
  long long ntl = nt;
  for (int l = 1; l < levels; ++l) {
    ntl /= m;  // nt at level l
    L.g[l] = take((ntl + 2) * row);   // + the outbox row of a time shard (r_{nc+1})
    if (l < levels - 1) {
      L.ul[l] = take((ntl / m + 1) * row);
      L.u2[l] = take((ntl / m + 1) * row);   // F-cycle: C-rows of the second (V) visit
    } else {
      L.u2[l] = L.ul[l] = 0;
    }
  }
  // partials: largest sweep = all nt rows x up to 64 tiles
  L.npart = (long long)(nt + 1) * 64;
  L.partials = take((L.npart + 1024) * sizeof(double));  // + room for the reduction chunks
  L.scal = take(64 * sizeof(double));
  L.hist = take(kGraphHist * sizeof(double));   // device history of the graph-mode solve
  L.lstate = take(64);
  L.sa = take(row);
  L.sb = take(row);
  L.st_in = take(row);    // time shards: coarsest-chain state from the left neighbour
  L.st_out = take(row);   //              and to the right neighbour
  L.forc = take((size_t)nt * FORC_LD * sizeof(double));   // inflow forcing rows b_n (R20)
  L.prog = take(64);      // progress counter of the overlapped two-level chain
  L.total = off;
  return true;
}

}  // namespace

struct mgrit_ctx {
  int nx, nt, m, levels, order, tableau, relax, scheme;
  int cycle = MGRIT_CYCLE_V;
  // inflow/outflow boundaries (mgrit_set_inflow; PAPER.md 4.5, R20): Phi = Phi_h +
  // forcing rows, every Psi truncated at the boundaries
  int bc = 0;
  double *forc = nullptr;   // workspace: nt x FORC_LD
  int final_sweep = MGRIT_FINAL_PREDICT;  // mgrit_set_final_sweep
  // mgrit_set_option: explicit replacements of measured defaults (n = 0: default)
  int opt_n[MGRIT_OPT_COUNT] = {0};
  int opt_v[MGRIT_OPT_COUNT][4] = {{0}};
  bool implicit;
  double alpha, cfl, dx, dt;
  cudaStream_t stream;
  long long ntl[MGRIT_MAX_LEVELS];  // nt at level l
  int psi_kind;
  PsiOp op[MGRIT_MAX_LEVELS];       // stencil Psi of level l >= 1
  double redisc_cfl;
  RKCoeffs fine, coarse_rk;
  SdirkCoef sd;
  SdirkCoef coarse_sd;              // RK-form Psi of an SDIRK scheme: the coarse stage solve
  int coarse_q;
  int zlo, zn;
  Tab tab;
  Layout lay;
  char *ws;
  double *u0b, *v0b, *g[MGRIT_MAX_LEVELS], *u2[MGRIT_MAX_LEVELS], *ul[MGRIT_MAX_LEVELS];
  double *partials, *scal, *sa, *sb;
  double *hist_dev;       // graph mode: ||r^(k)|| on the device
  // time sharding (mgrit_setup_shard): this context holds fine intervals
  // [rank*nc, (rank+1)*nc) of a global problem of nranks*nc intervals
  int rank = 0, nranks = 1;
  double *stage_send = nullptr, *stage_recv = nullptr;   // caller-owned, nx doubles each
  const mgrit_comm *comm = nullptr;                       // during mgrit_solve_shard
  double *st_in = nullptr, *st_out = nullptr;
  LoopState *lstate;      // graph mode: k, stop flags, tol
  cudaGraphExec_t gexec = nullptr;   // cached loop graph (invalidated by setters)
  long long glaunch[2] = {0, 0};     // kernels per captured iteration body (A, B)
  // overlapped two-level iteration: the coarse chain's chunks run on a private
  // high-priority stream while the next sweep's chunks follow on the caller's stream
  cudaStream_t hstream[2] = {nullptr, nullptr};   // chains alternate (two may be in flight)
  std::vector<cudaEvent_t> hev;
  unsigned long long *prog = nullptr;      // workspace: prog[0], prog[1] chain progress counters,
                                           //   prog[2] the sweep-chunk flag of a speculative chain
  void *wait_value_fn = nullptr;           // cuStreamWaitValue64 (driver entry point)
  void *write_value_fn = nullptr;          // cuStreamWriteValue64
  bool lsweep1_done = false;               // overlapped V-cycle: the next level-1 sweep already ran
  cudaStream_t gstream = nullptr;    // private capture/launch stream (the caller's may be
  cudaEvent_t gevent = nullptr;      //   the legacy default stream, which cannot capture)
  double *ucur, *unext;   // fine C-rows: current iterate / next (FCF ping-pong of u0b, v0b)
  const double *guess;
  const double *rhs[MGRIT_MAX_LEVELS] = {nullptr};  // mgrit_set_rhs: g_l of level-l primitives
  bool have_iterate;   // u0b holds the iterate (after >= 1 iteration)
  std::string err;
  // profiling
  bool prof;
  std::vector<cudaEvent_t> evpool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  long long prof_launch[MGRIT_PROF_CLASSES];
  double prof_ms[MGRIT_PROF_CLASSES];
  long long launches;
};

namespace {

bool opt(const mgrit_ctx *c, int key, int need = 1) { return c->opt_n[key] >= need; }
int stage_form(const mgrit_ctx *c) {
  return opt(c, MGRIT_OPT_STAGE_FORM) ? c->opt_v[MGRIT_OPT_STAGE_FORM][0] : 0;
}

int fail(mgrit_ctx *c, int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

// Status of an asynchronous runtime call (memcpy/memset on the context's stream): a
// failure is reported where it happens, not at the next synchronisation.
#define MG_CK(c, expr)                                                                     \
  do {                                                                                     \
    const cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess) return fail((c), MGRIT_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

cudaEvent_t get_event(mgrit_ctx *c) {
  if (!c->evpool.empty()) {
    cudaEvent_t e = c->evpool.back();
    c->evpool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  return e;
}

// NVTX range (RAII): visible in Nsight Systems / ncu --nvtx; a no-op without a tool.
struct Range {
  explicit Range(const char *name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};
const char *const kClassName[MGRIT_PROF_CLASSES] = {"fine_sweep", "level_sweep", "coarse_solve",
                                                    "interp", "residual", "other"};

// Run a launch, counting it and (if profiling) bracketing it with events.
template <class F>
int run(mgrit_ctx *c, int cls, F &&f) {
  Range nv(kClassName[cls]);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->prof) {
    e0 = get_event(c);
    e1 = get_event(c);
    if (!e0 || !e1) return fail(c, MGRIT_ECUDA, "cudaEventCreate failed");
    MG_CK(c, cudaEventRecord(e0, c->stream));
  }
  cudaError_t st = f();
  if (st != cudaSuccess) return fail(c, MGRIT_ECUDA, "kernel launch failed: %s", cudaGetErrorString(st));
  c->launches++;
  if (c->prof) {
    MG_CK(c, cudaEventRecord(e1, c->stream));
    c->pending.push_back({cls, {e0, e1}});
  }
  return MGRIT_OK;
}

void collect(mgrit_ctx *c) {
  for (auto &p : c->pending) {
    float ms = 0.f;
    cudaEventSynchronize(p.second.second);
    cudaEventElapsedTime(&ms, p.second.first, p.second.second);
    c->prof_ms[p.first] += ms;
    c->prof_launch[p.first] += 1;
    c->evpool.push_back(p.second.first);
    c->evpool.push_back(p.second.second);
  }
  c->pending.clear();
}

// ---- launch configuration of the fine RK sweep --------------------------------
struct FineCfg {
  SweepCfg cfg;
  int ntiles, HL;
};

// Choose (NT, P, tiles) for a sweep of `steps` total Phi applications per item.
bool choose_fine(const mgrit_ctx *c, int steps, FineCfg &f) {
  const int nx = c->nx;
  // periodic whole-row mode: W == nx exactly
  // SDIRK rows of 4096 points: 256 threads x 16 points (twice the work per scan and
  // barrier of 512 x 8; measured 1.02 vs 1.10 ms per cfg4 sweep)
  int cand[][2] = {{256, 16}, {512, 8}, {256, 8}, {128, 8}, {64, 8}, {32, 8}, {32, 4}, {32, 2}};
  if (opt(c, MGRIT_OPT_WHOLE_ROW, 2)) {  // mgrit_set_option: (NT, P) tried first
    cand[0][0] = c->opt_v[MGRIT_OPT_WHOLE_ROW][0];
    cand[0][1] = c->opt_v[MGRIT_OPT_WHOLE_ROW][1];
  }
  if (c->bc) {  // inflow/outflow: whole rows whose last thread owns the p+1 extrapolation nodes
    for (auto &cc : cand) {
      if (cc[0] * cc[1] == nx && rk_sweep_bnd_supported(c->scheme, {cc[0], cc[1]})) {
        f.cfg = {cc[0], cc[1]};
        f.ntiles = 1;
        f.HL = 0;
        return true;
      }
    }
    return false;
  }
  for (auto &cc : cand) {
    if (cc[0] * cc[1] == nx && rk_sweep_supported(c->scheme, {cc[0], cc[1]})) {
      f.cfg = {cc[0], cc[1]};
      f.ntiles = 1;
      f.HL = 0;
      return true;
    }
  }
  if (rk_scheme_implicit(c->scheme)) return false;  // implicit stage solves need whole rows
  // tile mode with halos: window W = NT*P >= T + HL + HR.  HL is rounded up to even and
  // tiles are even-aligned (2*floor(t*(nx/2)/ntiles)) so the TMA kernel's bulk copies are
  // 16-byte aligned.
  const int S = rk_scheme_stages(c->scheme);
  int HL = steps * S * rk_scheme_reach_left(c->scheme);
  HL += HL & 1;
  const int HR = steps * S * rk_scheme_reach_right(c->scheme);
  int tcand[][3] = {{128, 15, 0}, {256, 11, 0}};
  if (steps == 2 * c->m && opt(c, MGRIT_OPT_FINE_TILE, 2)) {  // FCF sweep: (NT, P[, minBlocks])
    tcand[0][0] = c->opt_v[MGRIT_OPT_FINE_TILE][0];
    tcand[0][1] = c->opt_v[MGRIT_OPT_FINE_TILE][1];
    tcand[0][2] = c->opt_n[MGRIT_OPT_FINE_TILE] >= 3 ? c->opt_v[MGRIT_OPT_FINE_TILE][2] : 0;
  }
  for (auto &cc : tcand) {
    const int W = cc[0] * cc[1];
    if (W > nx) continue;
    const int Tmax = W - HL - HR;
    if (Tmax < 64) continue;
    int ntiles = (nx + Tmax - 1) / Tmax;
    while (2 * ((nx / 2 + ntiles - 1) / ntiles) + 1 > Tmax) ++ntiles;
    f.cfg = {cc[0], cc[1], cc[2]};
    f.ntiles = ntiles;
    f.HL = HL;
    return true;
  }
  return false;
}

// ---- launch configuration of the stencil (Psi) kernels -------------------------
struct PsiCfg {
  SweepCfg cfg;
  int ntiles;
};
bool choose_psi(int nx, int halo, bool allow_periodic, PsiCfg &f) {
  const int cand[][2] = {{512, 8}, {256, 8}, {128, 8}, {64, 8}, {32, 8}, {32, 4}, {32, 2}};
  if (allow_periodic) {
    for (auto &cc : cand)
      if (cc[0] * cc[1] == nx) {
        f.cfg = {cc[0], cc[1]};
        f.ntiles = 1;
        return true;
      }
  }
  // tiles: smallest window that leaves >= max(halo, 128) outputs, preferring many tiles
  const int tc[][2] = {{256, 8}, {512, 8}};
  for (auto &cc : tc) {
    const int W = cc[0] * cc[1];
    const int Tmax = W - halo;
    if (Tmax < std::min(128, nx) || W > nx) continue;
    int ntiles = (nx + Tmax - 1) / Tmax;
    if ((nx + ntiles - 1) / ntiles > Tmax) ++ntiles;
    f.cfg = {cc[0], cc[1]};
    f.ntiles = ntiles;
    return true;
  }
  // fall back to periodic whole row if it exists
  for (auto &cc : cand)
    if (cc[0] * cc[1] == nx) {
      f.cfg = {cc[0], cc[1]};
      f.ntiles = 1;
      return true;
    }
  return false;
}

// Tile-mode TMA level kernel: (NT, P) = (128, 9), even tile boundaries.
bool choose_level_tma(int nx, int m, int halo, PsiCfg &f) {
  if ((nx & 1) || m > 4) return false;
  const int W = 128 * 9;
  if (W > nx) return false;
  const int Tmax = W - halo;
  if (Tmax < 128) return false;
  int ntiles = (nx + Tmax - 1) / Tmax;
  while (2 * ((nx / 2 + ntiles - 1) / ntiles) > Tmax) ++ntiles;
  f.cfg = {128, 9};
  f.ntiles = ntiles;
  return true;
}

RowMap rm(const double *b, long long off, long long stride) { return RowMap{b, off, stride}; }
const RowMap kNone = {nullptr, 0, 0};

SweepArgs base_sweep(const mgrit_ctx *c) {
  SweepArgs a;
  std::memset(&a, 0, sizeof(a));
  a.nx = c->nx;
  a.each_first = 1;
  a.each_last = 0;  // none
  a.d_every = 1;
  a.load_after = 1;  // issue the next item's prefetch after phase-1 step 1 (DESIGN 6.6)
  a.defer_v = 1;     // v_{j+1} stored with r_{j+2} (measured: -0.3 % per cfg5 solve)
  a.co = c->fine;
  a.sd = c->sd;
  a.in = a.cmp = a.endw = a.each = a.dstore = a.r2 = kNone;
  return a;
}

int sweep(mgrit_ctx *c, int cls, SweepArgs a, int total_steps) {
  FineCfg f;
  if (!choose_fine(c, total_steps, f))
    return fail(c, MGRIT_EUNSUPPORTED, "no fine-sweep configuration for nx=%d", c->nx);
  a.ntiles = f.ntiles;
  a.HL = f.HL;
  if (a.partials && (long long)a.nitems * a.ntiles > c->lay.npart)
    return fail(c, MGRIT_ENOMEM, "partials buffer too small");
  if (c->bc) {  // forcing rows: phase-1 step i of item j adds b_n, n = f_off + j*f_stride + i - 1
    a.forc = c->forc;
    a.nb = c->tab.s * rk_scheme_reach_left(c->scheme);
    return run(c, cls, [&] { return launch_rk_sweep_bnd(c->scheme, f.cfg, a, c->stream); });
  }
  // halo tiles, even nx, no per-step writes: persistent TMA-pipelined kernel
  const bool tma = f.ntiles > 1 && (c->nx % 2 == 0) && (f.cfg.p % 2 == 1) && a.in.base;
  if (a.partials && tma && (long long)a.nitems * a.ntiles * (f.cfg.nt_threads / 32) > c->lay.npart)
    return fail(c, MGRIT_ENOMEM, "partials buffer too small");
  if (tma) return run(c, cls, [&] { return launch_rk_sweep_tma(c->scheme, f.cfg, a, c->stream); });
  return run(c, cls, [&] { return launch_rk_sweep(c->scheme, f.cfg, a, c->stream); });
}

// Number of norm partials a sweep of `items` items writes (per tile; the TMA kernel writes
// one per warp).
long long partial_count(const mgrit_ctx *c, long long items, int total_steps) {
  FineCfg f;
  if (!choose_fine(c, total_steps, f)) return 0;
  const bool tma = f.ntiles > 1 && (c->nx % 2 == 0) && (f.cfg.p % 2 == 1);
  const int per = tma ? f.cfg.nt_threads / 32 : 1;
  return items * f.ntiles * per;
}

int reduce_norm(mgrit_ctx *c, long long n, double *norm2_host) {
  int st = run(c, 5, [&] { return launch_reduce(c->partials, n, c->scal, c->stream); });
  if (st) return st;
  if (n > 65536) c->launches++;  // two-pass reduction = two kernels
  if (norm2_host) {
    cudaError_t e = cudaMemcpyAsync(norm2_host, c->scal, sizeof(double), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return fail(c, MGRIT_ECUDA, "norm readback: %s", cudaGetErrorString(e));
  }
  return MGRIT_OK;
}

// Sequential coarse solve on level l (= levels-1, the coarsest) for steps 1..ntl:
//   x_n = Psi x_{n-1} + g_n, out_n = v_n + x_n  (stencil Psi: v == out, accumulated).
// Launch plan of the stencil-Psi sequential solve on level l.  Short chains (the
// V-cycle's coarsest level): trapezoid tiles, one launch, no inter-CTA communication.
// Long chains (two-level): the row split over a thread-block cluster (DSMEM halos), else
// one periodic CTA.
// ---- chunking of the overlapped two-level iteration --------------------
// Number of chunks actually used for a chain of nc steps when `want` are asked for: the
// largest C <= want with nc % C == 0, chunk length L = nc/C a multiple of 4 (the chain
// publishes per half of 4 steps) and L >= 32; 0 if there is none above 1.
int overlap_chunks(long long nc, int want) {
  while (want > 1 && (nc % want || (nc / want) % 4 || nc / want < 32)) --want;
  return want > 1 ? want : 0;
}
// Sweep chunk i of C (chunk length L = nc/C): the fine intervals [j0, j1).  Shifted by one
// interval against the chain's chunks so that it reads only C-rows <= (i+1)L (corrected by
// chain chunk i) and overwrites only coarse right-hand-side rows <= (i+1)L (consumed by it).
void overlap_sweep_chunk(long long nc, int C, int i, long long *j0, long long *j1) {
  const long long L = nc / C;
  *j0 = i == 0 ? 0 : i * L - 1;
  *j1 = i + 1 < C ? (i + 1) * L - 1 : nc;
}

struct CoarsePlan {
  enum Kind { NONE, TILES, CLUSTER, CLUSTER_CA, SEQ, TILES_SEG } kind = NONE;
  SweepCfg cfg = {0, 0};
  int ntiles = 1, cl = 0, S = 0;
  int seg = 0;       // TILES_SEG: steps per launch (trapezoid tiles, state row carried over)
  bool tb = false;   // CLUSTER_CA: warp-specialised variant (psi_seq_cluster_tb_kernel)
};

static CoarsePlan plan_coarse(const mgrit_ctx *c, int l) {
  CoarsePlan pl;
  const PsiOp &op = c->op[l];
  const long long cone = c->ntl[l] * (long long)(op.nu - 1);
  PsiCfg pc;
  // trapezoid tiles of the coarse kernel: 256 x 8 windows (the 512 x 8 ring exceeds the
  // shared memory of one SM), so the cone must leave >= 128 outputs of 2048
  if (cone <= 2048 - 128 && c->nx >= 2048 && choose_psi(c->nx, (int)cone, false, pc)) {
    pl.kind = CoarsePlan::TILES;
    pl.cfg = pc.cfg;
    pl.ntiles = pc.ntiles;
    return pl;
  }
  const bool whole = choose_psi(c->nx, 0, true, pc) && pc.ntiles == 1 &&
                     pc.cfg.nt_threads * pc.cfg.p == c->nx;
  // 16-CTA clusters (measured with tools/probe_cfgs.sh): the warp-
  // specialised kernel (nu <= 32) prefers 4 points per thread at nx = 4096 (half the
  // shared-memory window loads per output) and deeper s-steps; the cp.async variant
  // (wider stencils) keeps 2 points per thread and depth 4 for wide stencils.  Rows wider
  // than one CTA can hold (nx = 8192, 16384) are split 16 ways as well (512 / 1024 points
  // per SM; the warp-specialised ring does not fit 1024-point slices in shared memory).
  const bool want_tb = op.nu <= 32 && !(opt(c, MGRIT_OPT_COARSE_KERNEL) &&
                                        c->opt_v[MGRIT_OPT_COARSE_KERNEL][0] == 1);
  int cl = 0, smax = 8;
  SweepCfg cc = {0, 0};
  if (c->nx == 4096) {
    cl = 16;
    cc = (op.nu <= 16 || want_tb) ? SweepCfg{64, 4} : SweepCfg{128, 2};
    smax = op.nu <= 16 ? 8 : (want_tb ? 6 : 4);
  } else if (c->nx == 1024) {
    cl = 16;
    cc = {32, 2};
    smax = want_tb ? 12 : 8;
  } else if (c->nx == 2048) {
    cl = 16;
    cc = {64, 2};
  } else if (c->nx == 8192) {
    cl = 16;
    cc = {128, 4};
    smax = 6;
  } else if (c->nx == 16384) {
    cl = 16;
    cc = {256, 4};
    smax = 6;
  }
  if (opt(c, MGRIT_OPT_SEQ_CLUSTER, 3)) {
    cl = c->opt_v[MGRIT_OPT_SEQ_CLUSTER][0];
    cc = {c->opt_v[MGRIT_OPT_SEQ_CLUSTER][1], c->opt_v[MGRIT_OPT_SEQ_CLUSTER][2]};
  }
  if (opt(c, MGRIT_OPT_SEQ_S)) smax = c->opt_v[MGRIT_OPT_SEQ_S][0];
  if (smax >= 2) {
    const int S = seq_ca_depth(cl, cc, c->nx, op.o0, op.nu, smax);
    if (S >= 2) {
      pl.kind = CoarsePlan::CLUSTER_CA;
      pl.cfg = cc;
      pl.cl = cl;
      pl.S = S;
      pl.tb = want_tb && seq_cluster_tb_supported(cl, cc);
      return pl;
    }
  }
  if (seq_cluster_ok(cl, cc, c->nx, op.o0, op.nu)) {
    pl.kind = CoarsePlan::CLUSTER;
    pl.cfg = cc;
    pl.cl = cl;
    return pl;
  }
  if (!whole) {
    // any other width: the chain in segments of `seg` steps whose trapezoid cone fits a
    // 4096- (or 2048-) point window; the state row x_n is carried between launches
    for (const int W : {2048}) {
      if (W > c->nx) continue;
      const int seg = (W - 128) / std::max(1, op.nu - 1);
      if (seg < 1) continue;
      if (!choose_psi(c->nx, seg * (op.nu - 1), false, pc)) continue;
      pl.kind = CoarsePlan::TILES_SEG;
      pl.cfg = pc.cfg;
      pl.ntiles = pc.ntiles;
      pl.seg = (int)std::min<long long>(seg, c->ntl[l]);
      return pl;
    }
    return pl;
  }
  SweepCfg sc = pc.cfg;  // more threads per row for the latency-bound chain
  if (c->nx == 4096) sc = {1024, 4};
  else if (c->nx == 1024) sc = {256, 4};
  if (opt(c, MGRIT_OPT_SEQ_CFG, 2)) sc = {c->opt_v[MGRIT_OPT_SEQ_CFG][0], c->opt_v[MGRIT_OPT_SEQ_CFG][1]};
  pl.kind = CoarsePlan::SEQ;
  pl.cfg = sc;
  return pl;
}

// (n0, nsteps >= 0): only steps n0+1 .. n0+nsteps of the chain (a chunk of the overlapped
// two-level iteration; stencil Psi with a cluster / single-CTA plan), nsteps < 0: all.
int coarse_solve_level(mgrit_ctx *c, int l, RowMap v, RowMap out,
                       const double *state_in = nullptr, double *state_out = nullptr,
                       long long n0 = 0, long long nsteps = -1,
                       unsigned long long *progress = nullptr, int prog_every = 0,
                       const unsigned long long *wait_flag = nullptr,
                       unsigned long long wait_base = 0, int wait_chunks = 0) {
  const long long N = nsteps >= 0 ? nsteps : c->ntl[l];
  if (c->psi_kind != MGRIT_PSI_STENCIL) {
    RKCoarseArgs a;
    std::memset(&a, 0, sizeof(a));
    a.nx = c->nx;
    a.nsteps = (int)N;
    a.q = c->coarse_q;
    a.g = rm(c->g[l], 0, 1);
    a.v = v;
    a.out = out;
    a.co = c->coarse_rk;
    a.sd = c->coarse_sd;
    SweepCfg cfg;
    if (!rk_coarse_cfg(c->nx, cfg))
      return fail(c, MGRIT_EUNSUPPORTED, "RK-form Psi supports nx in {64,128,...,4096}");
    if (c->bc) {  // Psi = Phi_h^q with the boundary closures
      if (c->nx == 4096 || !rk_sweep_bnd_supported(c->scheme, cfg))
        return fail(c, MGRIT_EUNSUPPORTED, "inflow/outflow RK-form Psi: nx in {64,...,2048} and "
                                           "points per thread > order");
      return run(c, 2, [&] { return launch_rk_coarse_bnd(c->scheme, cfg, a, c->stream); });
    }
    return run(c, 2, [&] { return launch_rk_coarse(c->scheme, cfg, a, c->stream); });
  }
  // truncated Toeplitz Psi on a long chain: the warp-specialised 16-CTA cluster kernel with the
  // halo points beyond the row ends held at zero (CoarseArgs::trunc); otherwise one CTA
  const bool bc_cluster = c->bc && [&] {
    const CoarsePlan pl = plan_coarse(c, l);
    return pl.kind == CoarsePlan::CLUSTER_CA && pl.tb;
  }();
  if (c->bc && !bc_cluster) {  // one CTA, fixed coordinates (bounded.cu)
    if (progress) return fail(c, MGRIT_EUNSUPPORTED, "progress counter: cluster solve only");
    SweepCfg cfg;
    if (!tpsi_cfg(c->nx, true, cfg))
      return fail(c, MGRIT_EUNSUPPORTED, "inflow/outflow: nx in {64,128,...,4096}");
    CoarseArgs a;
    std::memset(&a, 0, sizeof(a));
    a.nx = c->nx;
    a.ntiles = 1;
    a.nsteps = (int)N;
    a.g = rm(c->g[l], 0, 1);
    a.out = out;
    a.state_in = state_in;
    a.state_out = state_out;
    a.op = c->op[l];
    return run(c, 2, [&] { return launch_tpsi_seq(cfg, a, c->stream); });
  }
  const CoarsePlan pl = plan_coarse(c, l);
  if (pl.kind == CoarsePlan::NONE)
    return fail(c, MGRIT_EUNSUPPORTED, "no coarse-solve configuration for nx=%d", c->nx);
  CoarseArgs a;
  std::memset(&a, 0, sizeof(a));
  a.nx = c->nx;
  a.ntiles = pl.ntiles;
  a.nsteps = (int)N;
  a.n0 = n0;
  a.g = rm(c->g[l], 0, 1);
  a.out = out;
  a.state_in = state_in;
  a.state_out = state_out;
  a.op = c->op[l];
  a.trunc = c->bc;
  if (progress) {
    if (!(pl.kind == CoarsePlan::CLUSTER_CA && pl.tb))
      return fail(c, MGRIT_EUNSUPPORTED, "progress counter: warp-specialised cluster solve only");
    a.progress = progress;
    a.prog_every = prog_every;
    a.wait_flag = wait_flag;
    a.wait_base = wait_base;
    a.wait_every = prog_every;
    a.wait_chunks = wait_chunks;
  }
  switch (pl.kind) {
    case CoarsePlan::CLUSTER:
      return run(c, 2, [&] { return launch_psi_seq_cluster(pl.cl, pl.cfg, a, c->stream); });
    case CoarsePlan::CLUSTER_CA:
      if (pl.tb)
        return run(c, 2, [&] { return launch_psi_seq_cluster_tb(pl.cl, pl.cfg, pl.S, a, c->stream); });
      return run(c, 2, [&] { return launch_psi_seq_cluster_ca(pl.cl, pl.cfg, pl.S, a, c->stream); });
    case CoarsePlan::SEQ:
      return run(c, 2, [&] { return launch_psi_seq_periodic(pl.cfg, a, c->stream); });
    case CoarsePlan::TILES_SEG: {
      // segments n0 = 0, seg, 2 seg, ...: x_{n0} in / x_{n0+seg} out through sa / sb
      double *st[2] = {c->sa, c->sb};
      int k = 0;
      for (long long n0 = 0; n0 < N; n0 += pl.seg, ++k) {
        a.n0 = n0;
        a.nsteps = (int)std::min<long long>(pl.seg, N - n0);
        a.state_in = n0 == 0 ? state_in : st[(k + 1) & 1];
        a.state_out = n0 + a.nsteps < N ? st[k & 1] : state_out;
        const int s = run(c, 2, [&] { return launch_psi_coarse(pl.cfg, a, c->stream); });
        if (s) return s;
      }
      return MGRIT_OK;
    }
    default:
      return run(c, 2, [&] { return launch_psi_coarse(pl.cfg, a, c->stream); });
  }
}

// Level-l (1 <= l <= levels-2) FCF sweep with RHS g_l, zero initial guess:
// v_l rows 1..nc, g_{l+1} rows 2..nc.
// uin: C-rows of a nonzero level-l iterate (F-cycle's second visit), null: zero guess;
// the FCF C-rows v go to vout rows 1..nc, r_{j+2} = Psi^m delta to g_{l+1} rows 2..nc.
// Phase 2 (the coarse right-hand side r_{j+2}) of the last interval: the global problem has
// no C-point nc+1, but a time shard that is not the last one computes its right
// neighbour's first coarse RHS row into the outbox row nc+1 of g_{l+1}.
int p2_count(const mgrit_ctx *c, long long nc) {
  return (int)(c->rank < c->nranks - 1 ? nc : nc - 1);
}

// (J0, cnt >= 0): only the level-l intervals J0 .. J0+cnt-1 (a chunk of the overlapped V-cycle).
int level_sweep(mgrit_ctx *c, int l, const double *uin, double *vout, long long J0 = 0,
                long long cnt = -1) {
  const PsiOp &op = c->op[l];
  const int m = c->m;
  const long long nc = c->ntl[l] / m;
  if (cnt < 0) cnt = nc - J0;
  PsiCfg pc;
  const bool tma = !c->bc && choose_level_tma(c->nx, m, 2 * m * (op.nu - 1), pc);
  if (c->bc) {
    pc.ntiles = 1;
    if (!tpsi_cfg(c->nx, false, pc.cfg))
      return fail(c, MGRIT_EUNSUPPORTED, "inflow/outflow: nx in {64,128,...,4096}");
  } else if (!tma && !choose_psi(c->nx, 2 * m * (op.nu - 1), true, pc))
    return fail(c, MGRIT_EUNSUPPORTED, "no level-sweep configuration");
  PsiSweepArgs a;
  std::memset(&a, 0, sizeof(a));
  a.nx = c->nx;
  a.nitems = (int)cnt;
  a.ntiles = pc.ntiles;
  a.m = m;
  a.interp = 0;
  a.u = uin ? rm(uin, J0, 1) : kNone;
  a.ucmp = uin ? rm(uin, J0 + 1, 1) : kNone;
  a.g = rm(c->g[l], J0 * m, m);
  a.v = rm(vout, J0 + 1, 1);   // v_{j+1} is the uncorrected C-row; the coarse levels add E
  a.r2 = rm(c->g[l + 1], J0 + 2, 1);
  a.p2_items = (int)std::max<long long>(0, std::min<long long>(cnt, p2_count(c, nc) - J0));
  a.v2 = a.out2 = kNone;
  a.op = op;
  if (c->bc) return run(c, 1, [&] { return launch_tpsi_level(pc.cfg, a, c->stream); });
  if (tma) return run(c, 1, [&] { return launch_psi_level_tma(pc.cfg, a, c->stream); });
  return run(c, 1, [&] { return launch_psi_sweep(pc.cfg, a, c->stream); });
}

// Level-l interpolation: from corrected C-rows u_l, F-relax with g_l and add the level-l
// values to level l-1's C-rows in place: out_{l-1}[n] += U_l[n], n = 0..nt_l (out_{l-1}
// holds v_{l-1} written by the level-(l-1) sweep; P:212 correction fused).
// (J0, cnt >= 0): only the level-l intervals J0 .. J0+cnt-1; the last point n = nt_l is added
// with the chunk that ends at nc.
int level_interp(mgrit_ctx *c, int l, const double *usrc_rows, RowMap out_prev, long long J0 = 0,
                 long long cnt = -1) {
  const PsiOp &op = c->op[l];
  const int m = c->m;
  const long long nc = c->ntl[l] / m;
  if (cnt < 0) cnt = nc - J0;
  PsiCfg pc;
  const bool tma = !c->bc && choose_level_tma(c->nx, m, (m - 1) * (op.nu - 1), pc);
  if (c->bc) {
    pc.ntiles = 1;
    if (!tpsi_cfg(c->nx, false, pc.cfg))
      return fail(c, MGRIT_EUNSUPPORTED, "inflow/outflow: nx in {64,128,...,4096}");
  } else if (!tma && !choose_psi(c->nx, (m - 1) * (op.nu - 1), true, pc))
    return fail(c, MGRIT_EUNSUPPORTED, "no interpolation configuration");
  PsiSweepArgs a;
  std::memset(&a, 0, sizeof(a));
  a.nx = c->nx;
  a.nitems = (int)cnt;
  a.ntiles = pc.ntiles;
  a.m = m;
  a.interp = 1;
  a.accumulate = 1;
  a.u = rm(usrc_rows, J0, 1);
  a.ucmp = kNone;
  a.g = rm(c->g[l], J0 * m, m);
  a.v = a.r2 = kNone;
  a.out2 = RowMap{out_prev.base, out_prev.off + J0 * m * out_prev.stride, out_prev.stride * m};
  a.v2 = tma ? kNone : a.out2;   // periodic kernel: out = v2 + x with v2 == out (in place)
  a.op = op;
  int st = c->bc ? run(c, 3, [&] { return launch_tpsi_level(pc.cfg, a, c->stream); })
           : tma ? run(c, 3, [&] { return launch_psi_level_tma(pc.cfg, a, c->stream); })
                 : run(c, 3, [&] { return launch_psi_sweep(pc.cfg, a, c->stream); });
  if (st || J0 + cnt < nc) return st;
  // the last point n = nt_l (level l's last C-row): out[nt_l] += u_l[nc]
  const long long ntl = c->ntl[l];
  double *dst = const_cast<double *>(out_prev.base) +
                (out_prev.off + ntl * out_prev.stride) * (long long)c->nx;
  const double *usrc = usrc_rows + nc * (long long)c->nx;
  return run(c, 3, [&] { return mg_add_rows(dst, dst, usrc, c->nx, c->stream); });
}

// Level-l coarse cycle with zero initial guess and RHS g_l; the level-l result is ADDED to
// dst (the C-rows of level l-1, which hold that level's uncorrected v).
//   V: sweep(l); cycle_V(l+1) -> ul[l]; interp(l) -> dst
//   F: sweep(l); cycle_F(l+1) -> ul[l]  [= MG_F(l, 0)];
//      then one V-cycle on level l from that iterate: sweep(l, iterate ul[l]) -> u2[l];
//      cycle_V(l+1) -> u2[l]; interp(l) from u2[l] -> dst               (R19)
// The coarsest level is the sequential solve (its F- and V-visits coincide).
int level_cycle(mgrit_ctx *c, int l, bool fcyc, RowMap dst) {
  static const char *const kLevel[MGRIT_MAX_LEVELS] = {"level 0", "level 1", "level 2", "level 3",
                                                       "level 4", "level 5", "level 6", "level 7"};
  Range nv(kLevel[l]);
  const int L = c->levels;
  if (l == L - 1) return coarse_solve_level(c, l, dst, dst);
  int st = MGRIT_OK;
  if (l == 1 && c->lsweep1_done) c->lsweep1_done = false;   // ran behind the last fine sweep
  else st = level_sweep(c, l, nullptr, c->ul[l]);
  if (st) return st;
  st = level_cycle(c, l + 1, fcyc, rm(c->ul[l], 0, 1));
  if (st) return st;
  if (!fcyc) return level_interp(c, l, c->ul[l], dst);
  st = level_sweep(c, l, c->ul[l], c->u2[l]);
  if (st) return st;
  st = level_cycle(c, l + 1, false, rm(c->u2[l], 0, 1));
  if (st) return st;
  return level_interp(c, l, c->u2[l], dst);
}

// Coarse-grid correction below level 0 after the fine sweep (g_1 = r): the fine C-rows
// `out0` hold v and receive += E (two-level: the sequential solve; multilevel: a V- or
// F-cycle on level 1).
int coarse_correction(mgrit_ctx *c, RowMap out0) {
  if (c->levels == 2) return coarse_solve_level(c, 1, out0, out0);
  return level_cycle(c, 1, c->cycle == MGRIT_CYCLE_F, out0);
}

// ---- level >= 1 FULL-state primitives (levels.cu) ----------------------------------
int level_check(mgrit_ctx *c, int level, bool need_coarser) {
  if (level < 1 || level >= c->levels || (need_coarser && level + 1 >= c->levels))
    return fail(c, MGRIT_EINVAL, "level %d out of range for %d levels", level, c->levels);
  if (c->psi_kind != MGRIT_PSI_STENCIL)
    return fail(c, MGRIT_EUNSUPPORTED, "level >= 1 primitives need stencil Psi operators");
  if (c->ntl[level] % c->m)
    return fail(c, MGRIT_EINVAL, "level %d has nt = %lld, not a multiple of m", level, c->ntl[level]);
  return MGRIT_OK;
}

RowStepArgs rowstep(const mgrit_ctx *c, int level, const double *U) {
  RowStepArgs a;
  std::memset(&a, 0, sizeof(a));
  a.nx = c->nx;
  a.bpr = std::max(1, std::min(64, (c->nx + 1023) / 1024));
  a.U = U;
  a.dst = const_cast<double *>(U);
  a.g = c->rhs[level];
  a.op = c->op[level];
  a.trunc = c->bc;
  return a;
}

// F- (positions i = 1..m-1) or C-relaxation (position m) of a level-l FULL array.
int level_relax_rows(mgrit_ctx *c, int level, double *U, int i_first, int i_last) {
  const int m = c->m;
  const long long nc = c->ntl[level] / m;
  for (int i = i_first; i <= i_last; ++i) {
    RowStepArgs a = rowstep(c, level, U);
    a.mode = 0;
    a.n0 = i;
    a.nstride = m;
    a.nrows = (int)nc;
    int st = run(c, 1, [&] { return launch_psi_rowstep(a, c->stream); });
    if (st) return st;
  }
  return MGRIT_OK;
}


// ---- CUDA-graph loop (graph.cu) --------------------------------------------------------
void drop_graph(mgrit_ctx *c) {
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  c->gexec = nullptr;
}

// Leaf nodes (no dependents) of a graph: the dependencies of a node appended after it.
std::vector<cudaGraphNode_t> graph_leaves(cudaGraph_t g) {
  size_t n = 0;
  cudaGraphGetNodes(g, nullptr, &n);
  std::vector<cudaGraphNode_t> nodes(n), leaves;
  if (n) cudaGraphGetNodes(g, nodes.data(), &n);
  for (auto nd : nodes) {
    size_t d = 0;
    cudaGraphNodeGetDependentNodes(nd, nullptr, &d);
    if (d == 0) leaves.push_back(nd);
  }
  return leaves;
}

// Capture `body` followed by the decide kernel into graph `g` (appended to its nodes).
template <class F>
int capture_into(mgrit_ctx *c, cudaGraph_t g, F &&body, cudaGraphConditionalHandle h0,
                 cudaGraphConditionalHandle h1, int set_h1, long long &nlaunch) {
  MG_CK(c, cudaStreamBeginCaptureToGraph(c->stream, g, nullptr, nullptr, 0,
                                         cudaStreamCaptureModeRelaxed));
  const long long l0 = c->launches;
  int st = body();
  if (!st) {
    const cudaError_t e = launch_loop_decide(c->lstate, c->scal, c->hist_dev, h0, h1, set_h1,
                                             c->stream);
    if (e != cudaSuccess) st = fail(c, MGRIT_ECUDA, "decide: %s", cudaGetErrorString(e));
  }
  nlaunch = c->launches - l0 + 1;
  c->launches = l0;                       // counted per executed iteration instead
  cudaGraph_t out = g;
  const cudaError_t e = cudaStreamEndCapture(c->stream, &out);
  if (st) return st;
  if (e != cudaSuccess) return fail(c, MGRIT_ECUDA, "graph capture: %s", cudaGetErrorString(e));
  return MGRIT_OK;
}

// WHILE(h_w) { A; decide -> h_w, h_i; IF(h_i) { B; decide -> h_w } } for FCF (A and B are
// the two buffer parities of the C-row ping-pong), WHILE(h_w) { A; decide } for F.
template <class F>
int build_loop_graph(mgrit_ctx *c, bool fcf, F &&iteration) {
  cudaGraph_t g = nullptr;
  MG_CK(c, cudaGraphCreate(&g, 0));
  auto cleanup = [&](int st) {
    cudaGraphDestroy(g);
    return st;
  };
  cudaGraphConditionalHandle hw, hi = 0;
  if (cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault) != cudaSuccess)
    return cleanup(fail(c, MGRIT_ECUDA, "conditional handle"));
  alignas(cudaGraphNodeParams) unsigned char wbuf[sizeof(cudaGraphNodeParams)];
  std::memset(wbuf, 0, sizeof(wbuf));
  cudaGraphNodeParams &wp = *reinterpret_cast<cudaGraphNodeParams *>(wbuf);
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wn;
  if (cudaGraphAddNode(&wn, g, nullptr, 0, &wp) != cudaSuccess)
    return cleanup(fail(c, MGRIT_ECUDA, "while node"));
  cudaGraph_t bw = wp.conditional.phGraph_out[0];
  if (fcf && cudaGraphConditionalHandleCreate(&hi, bw, 0, cudaGraphCondAssignDefault) != cudaSuccess)
    return cleanup(fail(c, MGRIT_ECUDA, "conditional handle"));
  int st = capture_into(c, bw, iteration, hw, hi, fcf ? 1 : 0, c->glaunch[0]);
  if (st) return cleanup(st);
  c->glaunch[1] = 0;
  if (fcf) {
    std::vector<cudaGraphNode_t> deps = graph_leaves(bw);
    alignas(cudaGraphNodeParams) unsigned char ibuf[sizeof(cudaGraphNodeParams)];
    std::memset(ibuf, 0, sizeof(ibuf));
    cudaGraphNodeParams &ip = *reinterpret_cast<cudaGraphNodeParams *>(ibuf);
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hi;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t in;
    if (cudaGraphAddNode(&in, bw, deps.data(), deps.size(), &ip) != cudaSuccess)
      return cleanup(fail(c, MGRIT_ECUDA, "if node"));
    st = capture_into(c, ip.conditional.phGraph_out[0], iteration, hw, hw, 0, c->glaunch[1]);
    if (st) return cleanup(st);
  }
  const cudaError_t e = cudaGraphInstantiate(&c->gexec, g, 0);
  if (e != cudaSuccess) {
    c->gexec = nullptr;
    return cleanup(fail(c, MGRIT_ECUDA, "graph instantiate: %s", cudaGetErrorString(e)));
  }
  return cleanup(MGRIT_OK);
}


// ---- time shards (mgrit_setup_shard / mgrit_solve_shard) ------------------------------
double *row_ptr(const mgrit_ctx *c, double *base, long long r) { return base + r * (long long)c->nx; }

// Neighbour exchange through the staging rows: send_row -> rank+1, rank-1 -> recv_row.
int comm_shift(mgrit_ctx *c, const double *send_row, double *recv_row) {
  if (c->nranks == 1) return MGRIT_OK;
  const bool hs = send_row && c->rank < c->nranks - 1;
  const bool hr = recv_row && c->rank > 0;
  const size_t row = (size_t)c->nx * sizeof(double);
  if (hs) MG_CK(c, cudaMemcpyAsync(c->stage_send, send_row, row, cudaMemcpyDeviceToDevice, c->stream));
  if (c->comm->shift(c->comm->user, hs ? 1 : 0, hr ? 1 : 0, c->stream))
    return fail(c, MGRIT_ECOMM, "mgrit_comm.shift failed (rank %d)", c->rank);
  if (hr) MG_CK(c, cudaMemcpyAsync(recv_row, c->stage_recv, row, cudaMemcpyDeviceToDevice, c->stream));
  return MGRIT_OK;
}

int comm_sum(mgrit_ctx *c, double *v, int n) {
  if (c->nranks == 1) return MGRIT_OK;
  if (c->comm->allreduce_sum(c->comm->user, v, n))
    return fail(c, MGRIT_ECOMM, "mgrit_comm.allreduce_sum failed (rank %d)", c->rank);
  return MGRIT_OK;
}

// V-cycle on level l of a time shard (zero initial guess, RHS g_l; result added to dst,
// the level-(l-1) C-rows).  As level_cycle, plus: the right neighbour's first coarse RHS
// row after the sweep, the corrected C-row at the block start before the interpolation,
// and the coarsest chain's state rank -> rank+1.
int level_cycle_shard(mgrit_ctx *c, int l, RowMap dst) {
  const int L = c->levels;
  const bool first = c->rank == 0, last = c->rank == c->nranks - 1;
  if (l == L - 1) {
    int st = first ? MGRIT_OK : comm_shift(c, nullptr, c->st_in);
    if (st) return st;
    st = coarse_solve_level(c, l, dst, dst, first ? nullptr : c->st_in, last ? nullptr : c->st_out);
    if (st) return st;
    return last ? MGRIT_OK : comm_shift(c, c->st_out, nullptr);
  }
  const long long nc = c->ntl[l] / c->m;
  int st = level_sweep(c, l, nullptr, c->ul[l]);
  if (st) return st;
  st = comm_shift(c, row_ptr(c, c->g[l + 1], nc + 1), row_ptr(c, c->g[l + 1], 1));
  if (st) return st;
  st = level_cycle_shard(c, l + 1, rm(c->ul[l], 0, 1));
  if (st) return st;
  st = comm_shift(c, row_ptr(c, c->ul[l], nc), row_ptr(c, c->ul[l], 0));
  if (st) return st;
  return level_interp(c, l, c->ul[l], dst);
}


}  // namespace

// Factored SDIRK stage solves (sdirk.cuh) of the fine step and, for an RK-form Psi, of the
// coarse step (Phi at CFL m*c or Phi^m).  Depends on the whole-row configuration
// (points per thread) and on MGRIT_OPT_SDIRK_PRODUCT, so mgrit_set_option re-runs it.
int setup_sdirk(mgrit_ctx *c, std::string &why) {
  std::memset(&c->sd, 0, sizeof(c->sd));
  std::memset(&c->coarse_sd, 0, sizeof(c->coarse_sd));
  if (!c->implicit) return MGRIT_OK;
  const bool fused = !(opt(c, MGRIT_OPT_SDIRK_PRODUCT) && c->opt_v[MGRIT_OPT_SDIRK_PRODUCT][0] == 1);
  FineCfg f;
  if (!choose_fine(c, 1, f)) {
    why = "SDIRK needs nx in {64,128,256,...,4096} (whole-row CTAs)";
    return MGRIT_EUNSUPPORTED;
  }
  if (!make_sdirk(c->fine.z, c->zlo, c->zn, c->tab.A[0][0], f.cfg.p, c->nx, c->sd, why, fused))
    return MGRIT_EUNSUPPORTED;
  if (c->psi_kind != MGRIT_PSI_STENCIL) {
    SweepCfg rc;
    if (!rk_coarse_cfg(c->nx, rc)) {
      why = "RK-form Psi supports nx in {64,128,...,4096}";
      return MGRIT_EUNSUPPORTED;
    }
    if (!make_sdirk(c->coarse_rk.z, c->zlo, c->zn, c->tab.A[0][0], rc.p, c->nx, c->coarse_sd, why,
                    fused))
      return MGRIT_EUNSUPPORTED;
  }
  return MGRIT_OK;
}

__global__ void mg_add_rows_kernel(double *dst, const double *a, const double *b, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = a[i] + b[i];
}
cudaError_t mg_add_rows(double *dst, const double *a, const double *b, int n, cudaStream_t s) {
  mg_add_rows_kernel<<<(n + 255) / 256 < 148 ? (n + 255) / 256 : 148, 256, 0, s>>>(dst, a, b, n);
  return cudaGetLastError();
}

// =============================================================================
extern "C" {

size_t mgrit_workspace_bytes(int nx, int nt, int m, int levels) {
  Layout L;
  if (!make_layout(nx, nt, m, levels, L)) return 0;
  return L.total;
}

const char *mgrit_last_error(const mgrit_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int mgrit_setup(mgrit_ctx **out, int nx, int nt, int m, double alpha, double cfl, int order,
                int tableau, int levels, const mgrit_psi *psi, int relax, void *workspace_dev,
                size_t workspace_bytes, void *stream) {
  if (!out) return MGRIT_EINVAL;
  *out = nullptr;
  mgrit_ctx *c = new mgrit_ctx();
  c->err.clear();
  c->nx = nx; c->nt = nt; c->m = m; c->levels = levels; c->order = order;
  c->tableau = tableau; c->relax = relax; c->alpha = alpha; c->cfl = cfl;
  c->stream = (cudaStream_t)stream;
  c->prof = false;
  c->launches = 0;
  std::memset(c->prof_launch, 0, sizeof(c->prof_launch));
  std::memset(c->prof_ms, 0, sizeof(c->prof_ms));
  auto bad = [&](int code, const char *msg) {
    fprintf(stderr, "mgrit_setup: %s\n", msg);
    delete c;
    return code;
  };
  if (!(alpha > 0)) return bad(MGRIT_EINVAL, "alpha must be > 0");
  if (!(cfl > 0)) return bad(MGRIT_EINVAL, "cfl must be > 0");
  if (order < 1 || order > 5) return bad(MGRIT_EINVAL, "order must be 1..5");
  if (tableau_order(tableau) != order) return bad(MGRIT_EINVAL, "tableau order != stencil order");
  if (relax != MGRIT_RELAX_F && relax != MGRIT_RELAX_FCF) return bad(MGRIT_EINVAL, "relax must be F or FCF");
  if (!make_tableau(tableau, c->tab)) return bad(MGRIT_EINVAL, "unknown tableau");
  c->implicit = c->tab.implicit;
  c->scheme = scheme_id(tableau);
  if (c->scheme < 0) return bad(MGRIT_EUNSUPPORTED, "unsupported tableau");
  if (!make_layout(nx, nt, m, levels, c->lay)) return bad(MGRIT_EINVAL, "invalid nx/nt/m/levels (nt % m^(levels-1) != 0?)");
  if (workspace_bytes < c->lay.total || !workspace_dev) return bad(MGRIT_ENOMEM, "workspace too small");
  const Upwind &up = kUpwind[order];
  if (nx < 4 * (up.dmax - up.dmin + 1)) return bad(MGRIT_EINVAL, "nx too small for the stencil");
  if (!psi) return bad(MGRIT_EINVAL, "psi is NULL");
  c->dx = 2.0 / nx;
  c->dt = cfl * c->dx / alpha;
  c->ntl[0] = nt;
  for (int l = 1; l < levels; ++l) c->ntl[l] = c->ntl[l - 1] / m;
  // fine coefficients
  std::memset(&c->fine, 0, sizeof(c->fine));
  make_z(order, cfl, c->fine.z, &c->zlo, &c->zn);
  for (int i = 0; i < MAXS; ++i) {
    c->fine.b[i] = c->tab.b[i];
    c->fine.mdiag[i] = c->tab.A[i][i];
    for (int j = 0; j < MAXS; ++j) c->fine.A[i][j] = c->tab.A[i][j];
  }
  fold_last_stage(c->fine, c->tab.s, stage_form(c));
  // coarse operators
  c->psi_kind = psi[0].kind;
  for (int l = 1; l < levels; ++l) {
    const mgrit_psi &p = psi[l - 1];
    if (p.kind != c->psi_kind) return bad(MGRIT_EINVAL, "mixed Psi kinds across levels");
    if (p.kind == MGRIT_PSI_STENCIL) {
      if (p.nnz < 1 || p.nnz > MGRIT_MAX_PSI_TAPS || !p.offsets || !p.coeffs)
        return bad(MGRIT_EINVAL, "bad stencil Psi");
      const int o0 = p.offsets[0], o1 = p.offsets[p.nnz - 1];
      const int nu = o1 - o0 + 1;
      if (nu > MAX_PSI || nu > nx / 2) return bad(MGRIT_EINVAL, "Psi stencil too wide");
      PsiOp &op = c->op[l];
      std::memset(&op, 0, sizeof(op));
      op.nu = nu;
      op.o0 = o0;
      for (int k = 0; k < p.nnz; ++k) {
        if (k > 0 && p.offsets[k] <= p.offsets[k - 1]) return bad(MGRIT_EINVAL, "Psi offsets must increase");
        op.psi[p.offsets[k] - o0] = p.coeffs[k];
      }
    } else {
      if (levels != 2) return bad(MGRIT_EINVAL, "IDEAL/REDISC Psi only for two levels");
      std::memset(&c->coarse_rk, 0, sizeof(c->coarse_rk));
      c->coarse_rk = c->fine;
      if (p.kind == MGRIT_PSI_IDEAL) {
        c->coarse_q = m;
      } else if (p.kind == MGRIT_PSI_REDISC) {
        int zlo, zn;
        make_z(order, p.redisc_cfl, c->coarse_rk.z, &zlo, &zn);
        fold_last_stage(c->coarse_rk, c->tab.s, stage_form(c));
        c->coarse_q = 1;
        c->redisc_cfl = p.redisc_cfl;
      } else {
        return bad(MGRIT_EINVAL, "unknown Psi kind");
      }
    }
  }
  {
    std::string why;
    const int st = setup_sdirk(c, why);
    if (st) return bad(st, why.c_str());
  }
  // carve the workspace
  c->ws = (char *)workspace_dev;
  c->u0b = (double *)(c->ws + c->lay.u0);
  c->v0b = (double *)(c->ws + c->lay.v0);
  for (int l = 1; l < levels; ++l) {
    c->g[l] = (double *)(c->ws + c->lay.g[l]);
    c->ul[l] = (l < levels - 1) ? (double *)(c->ws + c->lay.ul[l]) : nullptr;
    c->u2[l] = (l < levels - 1) ? (double *)(c->ws + c->lay.u2[l]) : nullptr;
  }
  c->ucur = c->u0b;
  c->unext = c->v0b;
  c->partials = (double *)(c->ws + c->lay.partials);
  c->scal = (double *)(c->ws + c->lay.scal);
  c->sa = (double *)(c->ws + c->lay.sa);
  c->sb = (double *)(c->ws + c->lay.sb);
  c->hist_dev = (double *)(c->ws + c->lay.hist);
  c->st_in = (double *)(c->ws + c->lay.st_in);
  c->st_out = (double *)(c->ws + c->lay.st_out);
  c->forc = (double *)(c->ws + c->lay.forc);
  c->prog = (unsigned long long *)(c->ws + c->lay.prog);
  if (cudaMemsetAsync(c->prog, 0, 64, c->stream) != cudaSuccess)
    return bad(MGRIT_ECUDA, "memset of the progress counter failed");
  c->lstate = (LoopState *)(c->ws + c->lay.lstate);
  c->guess = nullptr;
  c->have_iterate = false;
  // constant rows: g_l rows 0 and 1 (r_1 = 0), coarse v_l/u_l row 0
  const size_t row = (size_t)nx * sizeof(double);
  for (int l = 1; l < levels; ++l) {
    cudaError_t e = cudaMemsetAsync(c->g[l], 0, 2 * row, c->stream);
    if (e == cudaSuccess && l < levels - 1) e = cudaMemsetAsync(c->ul[l], 0, row, c->stream);
    if (e == cudaSuccess && l < levels - 1) e = cudaMemsetAsync(c->u2[l], 0, row, c->stream);
    if (e != cudaSuccess) return bad(MGRIT_ECUDA, cudaGetErrorString(e));
  }
  *out = c;
  return MGRIT_OK;
}

void mgrit_destroy(mgrit_ctx *c) {
  if (!c) return;
  for (auto &p : c->pending) {
    cudaEventDestroy(p.second.first);
    cudaEventDestroy(p.second.second);
  }
  for (auto e : c->evpool) cudaEventDestroy(e);
  drop_graph(c);
  if (c->gevent) cudaEventDestroy(c->gevent);
  if (c->gstream) cudaStreamDestroy(c->gstream);
  for (auto e : c->hev) cudaEventDestroy(e);
  for (auto hs : c->hstream) if (hs) cudaStreamDestroy(hs);
  delete c;
}

int mgrit_get_coefficients(const mgrit_ctx *c, int *s, int *z_lo, int *z_n, double *z, double *A,
                           double *b) {
  if (!c) return MGRIT_EINVAL;
  if (s) *s = c->tab.s;
  if (z_lo) *z_lo = c->zlo;
  if (z_n) *z_n = c->zn;
  if (z) for (int k = 0; k < c->zn; ++k) z[k] = c->fine.z[k];
  if (A) for (int i = 0; i < MAXS; ++i) for (int j = 0; j < MAXS; ++j) A[i * MAXS + j] = c->tab.A[i][j];
  if (b) for (int i = 0; i < MAXS; ++i) b[i] = c->tab.b[i];
  return MGRIT_OK;
}

int mgrit_scheme_coefficients(int order, int tableau, double cfl, int *s, int *z_lo, int *z_n,
                              double *z, double *A, double *b) {
  Tab t;
  if (order < 1 || order > 5 || tableau_order(tableau) != order || !make_tableau(tableau, t))
    return MGRIT_EINVAL;
  double zz[MAXZ] = {0};
  int lo, n;
  make_z(order, cfl, zz, &lo, &n);
  if (s) *s = t.s;
  if (z_lo) *z_lo = lo;
  if (z_n) *z_n = n;
  if (z) for (int k = 0; k < n; ++k) z[k] = zz[k];
  if (A) for (int i = 0; i < MAXS; ++i) for (int j = 0; j < MAXS; ++j) A[i * MAXS + j] = t.A[i][j];
  if (b) for (int i = 0; i < MAXS; ++i) b[i] = t.b[i];
  return MGRIT_OK;
}

int mgrit_set_guess(mgrit_ctx *c, const double *guess_dev) {
  if (!c || !guess_dev) return MGRIT_EINVAL;
  c->guess = guess_dev;
  c->have_iterate = false;
  return MGRIT_OK;
}

int mgrit_set_inflow(mgrit_ctx *c, int enable, const double *dg_dev) {
  if (!c) return MGRIT_EINVAL;
  drop_graph(c);
  if (!enable) {
    c->bc = 0;
    return MGRIT_OK;
  }
  if (c->implicit) return fail(c, MGRIT_EUNSUPPORTED, "inflow/outflow: explicit tableaux only (P:680)");
  if (c->nranks > 1) return fail(c, MGRIT_EUNSUPPORTED, "inflow/outflow: not in time-shard mode");
  const int old = c->bc;
  c->bc = 1;
  FineCfg f;
  SweepCfg tc;
  if (!choose_fine(c, c->m, f) || !tpsi_cfg(c->nx, true, tc)) {
    c->bc = old;
    return fail(c, MGRIT_EUNSUPPORTED,
                "inflow/outflow needs whole rows: nx in {64,128,...,4096} with nx/32 > order "
                "(nx >= 256 for order 5)");
  }
  if (!dg_dev) {  // homogeneous inflow u(-1, t) = 0
    MG_CK(c, cudaMemsetAsync(c->forc, 0, (size_t)c->nt * FORC_LD * sizeof(double), c->stream));
    return MGRIT_OK;
  }
  // tables of the Taylor / inverse-Lax-Wendroff ghost stage values (R20)
  BndCoef b;
  std::memset(&b, 0, sizeof(b));
  const int S = c->tab.s;
  b.S = S;
  b.NL = rk_scheme_reach_left(c->scheme);
  b.NR = rk_scheme_reach_right(c->scheme);
  b.p = c->order;
  b.nq = c->order + S;
  double v[MAXS], w[MAXS];
  for (int i = 0; i < S; ++i) v[i] = 1.0;
  for (int q = 0; q < S; ++q) {   // v = A^q 1
    for (int i = 0; i < S; ++i) b.t1[q][i] = std::pow(c->dt, q) * v[i];
    for (int i = 0; i < S; ++i) {
      double acc = 0.0;
      for (int l = 0; l < S; ++l) acc += c->tab.A[i][l] * v[l];
      w[i] = acc;
    }
    for (int i = 0; i < S; ++i) v[i] = w[i];
  }
  for (int k = 0; k < b.NL; ++k) {
    double fact = 1.0;
    for (int j = 0; j <= b.p; ++j) {
      if (j > 0) fact *= j;
      b.t2[k][j] = std::pow(k * c->dx / c->alpha, j) / fact;
    }
  }
  std::memcpy(b.z, c->fine.z, sizeof(b.z));
  for (int i = 0; i < MAXS; ++i) {
    b.b[i] = c->tab.b[i];
    for (int j = 0; j < MAXS; ++j) b.A[i][j] = c->tab.A[i][j];
  }
  return run(c, 5, [&] { return launch_bnd_forcing(b, dg_dev, c->nt, c->forc, c->stream); });
}

int mgrit_get_forcing(mgrit_ctx *c, double *out_dev) {
  if (!c || !out_dev) return MGRIT_EINVAL;
  if (!c->bc) return fail(c, MGRIT_EINVAL, "mgrit_set_inflow first");
  MG_CK(c, cudaMemcpyAsync(out_dev, c->forc, (size_t)c->nt * FORC_LD * sizeof(double),
                           cudaMemcpyDeviceToDevice, c->stream));
  return MGRIT_OK;
}

int mgrit_set_rhs(mgrit_ctx *c, int level, const double *g_dev) {
  if (!c) return MGRIT_EINVAL;
  if (level < 1 || level >= c->levels) return fail(c, MGRIT_EINVAL, "rhs level %d out of range", level);
  c->rhs[level] = g_dev;
  return MGRIT_OK;
}

int mgrit_relax(mgrit_ctx *c, int level, int kind, double *U) {
  if (!c || !U) return MGRIT_EINVAL;
  if (kind != MGRIT_RELAX_F && kind != MGRIT_RELAX_C && kind != MGRIT_RELAX_FCF)
    return fail(c, MGRIT_EINVAL, "relax kind");
  if (level != 0) {  // Phi_l = Psi_l with RHS g_l (P:206 on level l; R12)
    int st = level_check(c, level, false);
    if (st) return st;
    const int m = c->m;
    if (kind != MGRIT_RELAX_C) st = level_relax_rows(c, level, U, 1, m - 1);
    if (!st && kind != MGRIT_RELAX_F) st = level_relax_rows(c, level, U, m, m);
    if (!st && kind == MGRIT_RELAX_FCF) st = level_relax_rows(c, level, U, 1, m - 1);
    return st;
  }
  const int m = c->m;
  const long long nc = c->nt / m;
  auto frelax = [&]() {
    SweepArgs a = base_sweep(c);
    a.nitems = (int)nc;
    a.nsteps1 = m - 1;
    a.in = rm(U, 0, m);
    a.f_off = 0;
    a.f_stride = m;
    a.each = rm(U, 0, m);
    a.each_step = 1;
    a.each_first = 1;
    a.each_last = m - 1;
    return sweep(c, 0, a, m - 1);
  };
  auto crelax = [&]() {
    SweepArgs a = base_sweep(c);
    a.nitems = (int)nc;
    a.nsteps1 = 1;
    a.in = rm(U, m - 1, m);
    a.f_off = m - 1;
    a.f_stride = m;
    a.endw = rm(U, m, m);
    return sweep(c, 0, a, 1);
  };
  int st = MGRIT_OK;
  if (kind == MGRIT_RELAX_F) st = frelax();
  else if (kind == MGRIT_RELAX_C) st = crelax();
  else if (kind == MGRIT_RELAX_FCF) {
    st = frelax();
    if (!st) st = crelax();
    if (!st) st = frelax();
  } else st = fail(c, MGRIT_EINVAL, "relax kind");
  return st;
}

// Rows per work item of the streaming all-row residual kernel.
constexpr int kResidualChunk = 64;

// Level-0 all-row residual: sum of squares over rows 1..nt (n2_host, nullable: no
// readback) and, if r_dev, the C-point residuals.
static int residual0(mgrit_ctx *c, const double *U, double *n2_host, double *r_dev) {
  FineCfg f;
  if (!r_dev && choose_fine(c, 1, f) && f.ntiles > 1 && (c->nx % 2 == 0) && (f.cfg.p % 2 == 1)) {
    // norm only: streaming kernel, every row loaded once
    SweepArgs a = base_sweep(c);
    a.nitems = c->nt;
    a.in = rm(U, 0, 1);
    a.ntiles = f.ntiles;
    a.HL = f.HL;
    a.partials = c->partials;
    const long long np = (long long)((c->nt + kResidualChunk - 1) / kResidualChunk) * f.ntiles *
                         (f.cfg.nt_threads / 32);
    if (np > c->lay.npart) return fail(c, MGRIT_ENOMEM, "partials buffer too small");
    int st = run(c, 4, [&] {
      return launch_rk_residual_tma(c->scheme, f.cfg, a, kResidualChunk, c->stream);
    });
    if (st) return st;
    return reduce_norm(c, np, n2_host);
  }
  SweepArgs a = base_sweep(c);
  a.nitems = c->nt;
  a.nsteps1 = 1;
  a.in = rm(U, 0, 1);
  a.f_off = 0;
  a.f_stride = 1;
  a.cmp = rm(U, 1, 1);
  a.partials = c->partials;
  if (r_dev) {
    MG_CK(c, cudaMemsetAsync(r_dev, 0, (size_t)c->nx * sizeof(double), c->stream));
    a.dstore = rm(r_dev, 0, 1);
    a.d_every = c->m;
    a.d_phase = 1;
  }
  int st = sweep(c, 4, a, 1);
  if (st) return st;
  return reduce_norm(c, partial_count(c, c->nt, 1), n2_host);
}


int mgrit_residual(mgrit_ctx *c, int level, const double *U, double *norm_host, double *r_dev) {
  if (!c || !U) return MGRIT_EINVAL;
  if (level != 0) {  // r[n] = g[n] + Psi U[n-1] - U[n], n = 1..nt_l; dt_l = m^l dt
    int st = level_check(c, level, false);
    if (st) return st;
    const long long ntl = c->ntl[level];
    RowStepArgs a = rowstep(c, level, U);
    a.mode = 1;
    a.n0 = 1;
    a.nstride = 1;
    a.nrows = (int)ntl;
    a.partials = c->partials;
    const long long np = ntl * a.bpr;
    if (np > c->lay.npart) return fail(c, MGRIT_ENOMEM, "partials buffer too small");
    st = run(c, 4, [&] { return launch_psi_rowstep(a, c->stream); });
    if (st) return st;
    double n2 = 0;
    st = reduce_norm(c, np, norm_host ? &n2 : nullptr);
    if (st) return st;
    if (norm_host) {
      double dtl = c->dt;
      for (int l = 0; l < level; ++l) dtl *= c->m;
      *norm_host = std::sqrt(c->dx * dtl * n2);
    }
    if (r_dev) {  // C-point residuals r_j = g[jm] + Psi U[jm-1] - U[jm], r_0 = 0
      MG_CK(c, cudaMemsetAsync(r_dev, 0, (size_t)c->nx * sizeof(double), c->stream));
      RowStepArgs b = rowstep(c, level, U);
      b.mode = 1;
      b.n0 = c->m;
      b.nstride = c->m;
      b.nrows = (int)(ntl / c->m);
      b.rstore = r_dev;
      b.roff = 1;
      st = run(c, 4, [&] { return launch_psi_rowstep(b, c->stream); });
    }
    return st;
  }
  double n2 = 0;
  const int st = residual0(c, U, norm_host ? &n2 : nullptr, r_dev);
  if (st) return st;
  if (norm_host) *norm_host = std::sqrt(c->dx * c->dt * n2);
  return MGRIT_OK;
}

int mgrit_set_final_sweep(mgrit_ctx *c, int mode) {
  if (!c) return MGRIT_EINVAL;
  if (mode != MGRIT_FINAL_OFF && mode != MGRIT_FINAL_PREDICT && mode != MGRIT_FINAL_ALWAYS)
    return fail(c, MGRIT_EINVAL, "final-sweep mode must be OFF, PREDICT or ALWAYS");
  c->final_sweep = mode;
  return MGRIT_OK;
}

int mgrit_set_option(mgrit_ctx *c, int option, const int *values, int n) {
  if (!c) return MGRIT_EINVAL;
  static const int kMin[MGRIT_OPT_COUNT] = {2, 2, 3, 1, 1, 2, 1, 1, 1, 1, 1};
  static const int kMax[MGRIT_OPT_COUNT] = {3, 2, 3, 1, 1, 2, 1, 1, 1, 2, 3};
  if (option < 0 || option >= MGRIT_OPT_COUNT) return fail(c, MGRIT_EINVAL, "unknown option %d", option);
  if (n != 0 && (n < kMin[option] || n > kMax[option] || !values))
    return fail(c, MGRIT_EINVAL, "option %d takes %d..%d values", option, kMin[option], kMax[option]);
  for (int i = 0; i < n; ++i)
    if (values[i] < 0) return fail(c, MGRIT_EINVAL, "option %d: negative value", option);
  if ((option == MGRIT_OPT_COARSE_KERNEL || option == MGRIT_OPT_SDIRK_PRODUCT ||
       option == MGRIT_OPT_GRAPH) && n && values[0] > 1)
    return fail(c, MGRIT_EINVAL, "option %d takes 0 or 1", option);
  if (option == MGRIT_OPT_STAGE_FORM && n && values[0] > 4)
    return fail(c, MGRIT_EINVAL, "option %d takes 0 or 1", option);
  const int old_n = c->opt_n[option];
  int old_v[4];
  std::memcpy(old_v, c->opt_v[option], sizeof(old_v));
  drop_graph(c);
  c->opt_n[option] = n;
  for (int i = 0; i < 4; ++i) c->opt_v[option][i] = i < n ? values[i] : 0;
  if (option == MGRIT_OPT_STAGE_FORM) {  // re-derive the step coefficients in the new form
    fold_last_stage(c->fine, c->tab.s, stage_form(c));
    if (c->psi_kind != MGRIT_PSI_STENCIL) {
      if (c->coarse_q == 1) {  // REDISC: own z at the coarse CFL
        int zlo, zn;
        make_z(c->order, c->redisc_cfl, c->coarse_rk.z, &zlo, &zn);
      } else {
        std::memcpy(c->coarse_rk.z, c->fine.z, sizeof(c->fine.z));
      }
      fold_last_stage(c->coarse_rk, c->tab.s, stage_form(c));
    }
  }
  if (option == MGRIT_OPT_WHOLE_ROW || option == MGRIT_OPT_SDIRK_PRODUCT) {
    std::string why;
    const int st = setup_sdirk(c, why);
    if (st) {  // restore the previous (valid) state
      c->opt_n[option] = old_n;
      std::memcpy(c->opt_v[option], old_v, sizeof(old_v));
      std::string why2;
      setup_sdirk(c, why2);
      return fail(c, st, "%s", why.c_str());
    }
  }
  return MGRIT_OK;
}

int mgrit_overlap_plan(long long nc, int want, int *chunks, long long *j0, long long *j1) {
  if (nc < 1 || want < 0 || !chunks) return MGRIT_EINVAL;
  const int C = overlap_chunks(nc, want);
  *chunks = C;
  for (int i = 0; i < C && j0 && j1; ++i) overlap_sweep_chunk(nc, C, i, &j0[i], &j1[i]);
  return MGRIT_OK;
}

int mgrit_set_cycle(mgrit_ctx *c, int cycle) {
  if (!c) return MGRIT_EINVAL;
  if (cycle != MGRIT_CYCLE_V && cycle != MGRIT_CYCLE_F) return fail(c, MGRIT_EINVAL, "cycle must be V or F");
  drop_graph(c);
  c->cycle = cycle;
  return MGRIT_OK;
}

int mgrit_coarse_solve(mgrit_ctx *c, int level, double *U) {
  if (!c || !U) return MGRIT_EINVAL;
  if (level != 0) {  // level l: r_j -> g_{l+1}; e = sequential Psi_{l+1} solve; U[jm] += e_j; F
    int st = level_check(c, level, true);
    if (st) return st;
    RowStepArgs a = rowstep(c, level, U);
    a.mode = 1;
    a.n0 = c->m;
    a.nstride = c->m;
    a.nrows = (int)(c->ntl[level] / c->m);
    a.rstore = c->g[level + 1];
    a.roff = 1;
    st = run(c, 4, [&] { return launch_psi_rowstep(a, c->stream); });
    if (st) return st;
    st = coarse_solve_level(c, level + 1, rm(U, 0, c->m), rm(U, 0, c->m));
    if (st) return st;
    return mgrit_relax(c, level, MGRIT_RELAX_F, U);
  }
  if (c->psi_kind != MGRIT_PSI_STENCIL && c->levels != 2)
    return fail(c, MGRIT_EUNSUPPORTED, "RK-form Psi: two levels only");
  const int m = c->m;
  const long long nc = c->nt / m;
  // r_j = Phi U[jm-1] - U[jm], j = 1..nc  -> g_1 rows 1..nc
  SweepArgs a = base_sweep(c);
  a.nitems = (int)nc;
  a.nsteps1 = 1;
  a.in = rm(U, m - 1, m);
  a.f_off = m - 1;
  a.f_stride = m;
  a.cmp = rm(U, m, m);
  a.dstore = rm(c->g[1], 1, 1);
  int st = sweep(c, 4, a, 1);
  if (st) return st;
  // e_j = Psi e_{j-1} + r_j ; U[jm] += e_j
  st = coarse_solve_level(c, 1, rm(U, 0, m), rm(U, 0, m));
  if (st) return st;
  // ideal interpolation: F-relaxation
  return mgrit_relax(c, 0, MGRIT_RELAX_F, U);
}

int mgrit_solve(mgrit_ctx *c, double tol, int max_iter, double *out_dev, int *iters,
                double *hist, int *converged, double *crows_hist) {
  if (!c) return MGRIT_EINVAL;
  if (!c->guess) return fail(c, MGRIT_EINVAL, "mgrit_set_guess first");
  if (max_iter < 0) return fail(c, MGRIT_EINVAL, "max_iter < 0");
  Range nv_solve("mgrit_solve");
  const int m = c->m, nx = c->nx;
  const long long nc = c->nt / m;
  const size_t row = (size_t)nx * sizeof(double);
  const bool fcf = c->relax == MGRIT_RELAX_FCF;
  int st;
  // row 0 of the C-row buffers = u0
  c->ucur = c->u0b;
  c->unext = c->v0b;
  MG_CK(c, cudaMemcpyAsync(c->u0b, c->guess, row, cudaMemcpyDeviceToDevice, c->stream));
  MG_CK(c, cudaMemcpyAsync(c->v0b, c->guess, row, cudaMemcpyDeviceToDevice, c->stream));
  // hist[0]: all-row residual of the guess
  double r0;
  st = mgrit_residual(c, 0, c->guess, &r0, nullptr);
  if (st) return st;
  if (hist) hist[0] = r0;
  if (!fcf)  // Parareal: the coarse correction updates the C-rows in place (v = u)
    MG_CK(c, cudaMemcpy2DAsync(c->ucur, row, c->guess, row * m, row, nc + 1,
                               cudaMemcpyDeviceToDevice, c->stream));
  int k = 0;
  bool conv = r0 < tol;
  bool nonfinite = !std::isfinite(r0);
  c->have_iterate = false;
  FineCfg f;
  if (!choose_fine(c, fcf ? 2 * m : m, f)) return fail(c, MGRIT_EUNSUPPORTED, "no sweep cfg");
  // FCF sweep: reads the current C-rows (the guess's at k = 0), writes v into `unext`
  // (the next iterate before its coarse correction), delta norm, r -> g_1.
  // (j0, cnt): only the intervals j0 .. j0+cnt-1 (a chunk of the overlapped iteration, with
  // `reserve` SMs left to the concurrent coarse chain); cnt < 0: all.
  auto do_sweep = [&](bool first, bool want_norm, long long j0 = 0, long long cnt = -1,
                      int reserve = 0, int per_sm = 0) -> int {
    if (cnt < 0) cnt = nc - j0;
    SweepArgs a = base_sweep(c);
    a.nitems = (int)cnt;
    a.nsteps1 = m;
    a.f_off = j0 * m;
    a.f_stride = m;
    a.reserve_sms = reserve;
    a.max_per_sm = per_sm;
    if (first && fcf) {
      a.in = rm(c->guess, j0 * m, m);
      a.cmp = rm(c->guess, (j0 + 1) * m, m);
    } else {
      a.in = rm(c->ucur, j0, 1);
      a.cmp = rm(c->ucur, j0 + 1, 1);
    }
    a.partials = want_norm ? c->partials + partial_count(c, j0, fcf ? 2 * m : m) : nullptr;
    if (fcf) {
      a.endw = rm(c->unext, j0 + 1, 1);
      a.nsteps2 = m;
      a.p2_items = (int)std::max<long long>(0, std::min<long long>(cnt, nc - 1 - j0));
      a.r2 = rm(c->g[1], j0 + 2, 1);
    } else {
      a.dstore = rm(c->g[1], j0 + 1, 1);
      a.d_every = 1;
      a.d_phase = 0;
    }
    return sweep(c, 0, a, fcf ? 2 * m : m);
  };
  // Check+materialise sweep: phase 1 of the fused sweep (same tiles, so the same norm
  // partials, bit for bit) with per-step writes of the FULL iterate into out_dev and no
  // coarse RHS.  Used for the sweep that measures ||r^(k)|| when iteration k is known
  // (k == max_iter) or predicted to be the last, so a converged solve needs neither the
  // unused r = Phi^m delta nor a separate materialisation pass.
  auto check_sweep = [&](long long j0 = 0, long long cnt = -1, int reserve = 0) -> int {
    if (cnt < 0) cnt = nc - j0;
    SweepArgs a = base_sweep(c);
    a.nitems = (int)cnt;
    a.nsteps1 = m;
    a.f_off = j0 * m;
    a.f_stride = m;
    a.reserve_sms = reserve;
    a.in = rm(c->ucur, j0, 1);
    a.cmp = rm(c->ucur, j0 + 1, 1);
    a.partials = c->partials + partial_count(c, j0, fcf ? 2 * m : m);
    a.each = rm(out_dev, j0 * m, m);
    a.each_step = 1;
    a.each_first = 0;
    a.each_last = m - 1;
    return sweep(c, 3, a, fcf ? 2 * m : m);
  };
  // Overlapped two-level iteration (option MGRIT_OPT_OVERLAP = number of chunks C, default 8
  // for long chains): the sequential coarse chain runs as ONE launch of the 16-CTA
  // cluster kernel on a private high-priority stream and publishes a progress counter every
  // L = nc/C steps; as soon as chunk i's C-rows are corrected, the next iteration's fused
  // sweep over those intervals follows on the caller's stream, beside the running chain, on
  // the SMs the cluster leaves free.  The sweeps are released by stream-ordered memory waits
  // (cuStreamWaitValue64 on the counter): no kernel waits on another, so there is no
  // co-residency requirement.
  // Sweep chunk i covers the intervals [iL-1, (i+1)L-1) (the last one up to nc): it reads
  // the C-rows <= (i+1)L, which chunk i has corrected, and overwrites the coarse right-hand
  // side rows <= (i+1)L, which chunk i has consumed.  Same kernels on the same data in the
  // same order per row: results are bitwise those of the serial iteration.
  int nchunks = 0;
  // Speculation pays when the chain is much longer than the sweep it hides behind (two chains
  // in flight cost the sweeps 32 SMs): cost model fitted to the measured kernels
  // (profiles/r02_overlap_ab.txt) -- chain step = 230 ns + 4.5 x its FP64 floor (nu * nx/16
  // FMAs per SM at 64 per clock), sweep = stage-form flops at 23 TF/s (explicit) or 10 TF/s
  // (SDIRK).  cfg3: 0.75 vs 0.60 ms -> no; cfg4: 2.1 vs 0.7 ms -> yes.
  bool spec_default = false;
  double sweep_est_ms = 0.0;
  if (c->levels == 2 && c->psi_kind == MGRIT_PSI_STENCIL) {
    const double floor_ns = c->op[1].nu * (nx / 16.0) / 64.0 / 1.965;
    const double chain_ms = nc * (230.0 + 4.5 * floor_ns) * 1e-6;
    int nnz = 0;
    for (int i = 0; i < c->tab.s; ++i) {
      nnz += c->tab.b[i] != 0.0;
      for (int l = 0; l < c->tab.s; ++l) nnz += c->tab.A[i][l] != 0.0;
    }
    const double flops = c->tab.s * (2.0 * c->zn - 1.0) + 2.0 * nnz;
    const double sweep_ms = (double)nc * m * (fcf ? 2 : 1) * nx * flops / (c->implicit ? 10e12 : 23e12) * 1e3;
    spec_default = chain_ms >= 1.5 * sweep_ms;
    sweep_est_ms = sweep_ms;
  }
  if (c->levels == 2 && c->psi_kind == MGRIT_PSI_STENCIL && !c->prof && c->nranks == 1) {
    const CoarsePlan pl = plan_coarse(c, 1);
    const bool chain = pl.kind == CoarsePlan::CLUSTER_CA && pl.tb;
    // default (measured, profiles/r02_overlap_ab.txt): 16 chunks of >= 128 steps, 8 with a
    // speculative chain (its sweeps run on fewer SMs: coarser chunks quantise better)
    const bool sp = spec_default && fcf;
    int want = opt(c, MGRIT_OPT_OVERLAP) ? c->opt_v[MGRIT_OPT_OVERLAP][0]
                                         : (nc >= 2048 ? (sp ? 8 : 16) : (nc >= 1024 ? (sp ? 4 : 8) : 0));
    want = overlap_chunks(nc, want);
    if (chain && want > 1) nchunks = want;
    if (nchunks && !c->wait_value_fn) {   // stream-ordered memory operations (driver entry points)
      cudaDriverEntryPointQueryResult qr;
      void *fn = nullptr, *fn2 = nullptr;
      if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
          qr != cudaDriverEntryPointSuccess || !fn ||
          cudaGetDriverEntryPoint("cuStreamWriteValue64", &fn2, cudaEnableDefault, &qr) != cudaSuccess ||
          qr != cudaDriverEntryPointSuccess || !fn2) {
        cudaGetLastError();
        nchunks = 0;                      // not available: serial iteration
      } else {
        c->wait_value_fn = fn;
        c->write_value_fn = fn2;
      }
    }
  }
  // Speculative chain (FCF only; option MGRIT_OPT_OVERLAP second value 0 disables): while
  // iteration k's sweep chunks run, the chain of iteration k+1 is already resident on the
  // other high-priority stream; its producer warps are gated, chunk by chunk, on a flag the
  // caller's stream writes after each sweep chunk (cuStreamWriteValue64).  It only modifies
  // the buffer of iterate k+1 (v' + e), never iterate k, so a solve that converges at k simply
  // ignores it.  Two chains in flight halve the iteration period.
  typedef int (*mem_fn_t)(cudaStream_t, unsigned long long, unsigned long long, unsigned int);
  if (nchunks > 1)   // sweep-chunk flag := 0 (the previous solve's drain left it released)
    MG_CK(c, cudaMemsetAsync(c->prog + 2, 0, sizeof(unsigned long long), c->stream));
  const bool spec_ok = nchunks > 1 && fcf &&
                       (opt(c, MGRIT_OPT_OVERLAP, 2) ? c->opt_v[MGRIT_OPT_OVERLAP][1] != 0 : spec_default);
  bool spec_inflight = false;       // the chain of the next correction is already launched
  int spec_par = 0;                 // ... on hstream[spec_par] with counter prog[spec_par]
  unsigned long long flag_seq = 0;  // value of the sweep-chunk flag prog[2] after the last write
  // release and drain a chain in flight (error paths, end of the solve)
  auto drain_chains = [&]() {
    if (c->write_value_fn && nchunks > 1)
      ((mem_fn_t)c->write_value_fn)(c->stream, (unsigned long long)(uintptr_t)(c->prog + 2),
                                   1ull << 62, 0u);
    for (auto hs : c->hstream) if (hs) cudaStreamSynchronize(hs);
    spec_inflight = false;
    c->lsweep1_done = false;
  };
  struct Drain {
    std::function<void()> f;
    ~Drain() { f(); }
  } drain_guard{drain_chains};
  auto ensure_streams = [&]() -> int {
    for (auto &hs : c->hstream) {
      if (hs) continue;
      int lo = 0, hi = 0;
      MG_CK(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
      MG_CK(c, cudaStreamCreateWithPriority(&hs, cudaStreamNonBlocking, hi));
    }
    while ((int)c->hev.size() < 2) {
      cudaEvent_t e = nullptr;
      MG_CK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->hev.push_back(e);
    }
    return MGRIT_OK;
  };
  // wait on the caller's stream until the chain with counter prog[par] has published `chunks`
  auto wait_chain = [&](int par, int chunks) -> int {
    const int wr = ((mem_fn_t)c->wait_value_fn)(c->stream, (unsigned long long)(uintptr_t)(c->prog + par),
                                                16ull * (unsigned long long)chunks, 0u /* GEQ */);
    return wr ? fail(c, MGRIT_ECUDA, "cuStreamWaitValue64 failed (%d)", wr) : MGRIT_OK;
  };
  // correction k (k = the iteration being performed, already incremented) overlapped with the
  // sweep that measures ||r^(k)||; may_spec: iteration k+1 may follow (k < max_iter)
  // final: the sweep chunks are check-sweep chunks (residual + FULL solution, no coarse RHS)
  auto overlapped_iteration = [&](bool may_spec, bool final = false) -> int {
    const int C_ = nchunks;
    const long long L = nc / C_;
    int s2 = ensure_streams();
    if (s2) return s2;
    const cudaStream_t user = c->stream;
    double *corr = fcf ? c->unext : c->ucur;   // C-rows receiving += e
    int par;
    if (spec_inflight) {
      par = spec_par;                          // chain k is already running
      spec_inflight = false;
    } else {
      par = spec_par ^ 1;
      spec_par = par;
      // counter := 0 on the caller's stream, before the event the chain waits for and before
      // the memory waits below (so no wait can see an earlier chain's value)
      MG_CK(c, cudaMemsetAsync(c->prog + par, 0, sizeof(unsigned long long), user));
      MG_CK(c, cudaEventRecord(c->hev[par], user));          // the previous sweep is complete
      MG_CK(c, cudaStreamWaitEvent(c->hstream[par], c->hev[par], 0));
      c->stream = c->hstream[par];
      s2 = coarse_solve_level(c, 1, rm(corr, 0, 1), rm(corr, 0, 1), nullptr, nullptr, 0, -1,
                              c->prog + par, (int)L);
      c->stream = user;
      if (s2) return s2;
    }
    if (fcf) std::swap(c->ucur, c->unext);                  // the sweeps below read `corr`
    const bool spec = spec_ok && may_spec && !final;
    if (spec) {  // chain k+1: corrects the rows the sweep chunks below write (now `unext`)
      const int p2 = par ^ 1;
      MG_CK(c, cudaMemsetAsync(c->prog + p2, 0, sizeof(unsigned long long), user));
      MG_CK(c, cudaEventRecord(c->hev[p2], user));
      MG_CK(c, cudaStreamWaitEvent(c->hstream[p2], c->hev[p2], 0));
      c->stream = c->hstream[p2];
      s2 = coarse_solve_level(c, 1, rm(c->unext, 0, 1), rm(c->unext, 0, 1), nullptr, nullptr, 0, -1,
                              c->prog + p2, (int)L, c->prog + 2, flag_seq, C_);
      c->stream = user;
      if (s2) return s2;
      spec_inflight = true;
      spec_par = p2;
    }
    for (int i = 0; i < C_; ++i) {
      s2 = wait_chain(par, i + 1);
      if (s2) return s2;
      long long j0, j1;
      overlap_sweep_chunk(nc, C_, i, &j0, &j1);
      const int reserve = i + 1 < C_ ? (spec ? 32 : 16) : (spec ? 16 : 0);
      s2 = final ? check_sweep(j0, j1 - j0, reserve) : do_sweep(false, true, j0, j1 - j0, reserve);
      if (s2) return s2;
      if (spec) {
        const int wr = ((mem_fn_t)c->write_value_fn)(user, (unsigned long long)(uintptr_t)(c->prog + 2),
                                                     ++flag_seq, 0u);
        if (wr) return fail(c, MGRIT_ECUDA, "cuStreamWriteValue64 failed (%d)", wr);
      }
    }
    return MGRIT_OK;
  };
  // Overlapped V-cycle (option MGRIT_OPT_VOVERLAP = C chunks, CTAs per SM of the concurrent
  // fine sweep, speculative level-1 sweep 0/1; OFF by default): the top of the V-cycle is
  // HBM-bound (level-1 interpolation: 86 % of the DRAM peak, no FP64 work to speak of) and the
  // fused fine sweep is FP64-bound (HBM at 40 %), so in principle they can run side by side.
  // Measured (profiles/r02_voverlap.txt): co-resident, the two kernels slow each other down by
  // as much as the overlap saves (cfg5 34.65 -> 34.1-34.2 ms at best, the gain coming from
  // filled kernel tails), so the serial iteration stays the default.  The level-1 interpolation goes in C chunks on a high-priority stream; after the
  // event of chunk i the fine sweep over the fine intervals [4iL-2, 4(i+1)L-2) follows on the
  // caller's stream with one CTA slot per SM left free; behind it, on a second stream, the
  // level-1 sweep of the NEXT V-cycle over the level-1 intervals [iL-1, (i+1)L-1) (it only
  // writes coarse scratch rows, so it is harmless if the solve stops).  The shifted chunk
  // boundaries make every read see rows that are final and every write hit rows that are
  // consumed (same argument as the two-level overlap).  CUDA events only.  Same kernels on the
  // same rows: bitwise the serial iteration.
  int vchunks = 0, v_per_sm = 3;
  bool v_spec = true;
  c->lsweep1_done = false;
  if (c->levels >= 3 && c->psi_kind == MGRIT_PSI_STENCIL && c->cycle == MGRIT_CYCLE_V && fcf &&
      !c->bc && !c->prof && c->nranks == 1 && f.ntiles > 1) {
    const long long nc1 = c->ntl[1] / m;
    PsiCfg pc;
    int want = opt(c, MGRIT_OPT_VOVERLAP) ? c->opt_v[MGRIT_OPT_VOVERLAP][0] : 0;
    if (opt(c, MGRIT_OPT_VOVERLAP, 2)) v_per_sm = c->opt_v[MGRIT_OPT_VOVERLAP][1];
    if (opt(c, MGRIT_OPT_VOVERLAP, 3)) v_spec = c->opt_v[MGRIT_OPT_VOVERLAP][2] != 0;
    while (want > 1 && (nc1 % want || nc1 / want < 64)) --want;
    if (want > 1 && choose_level_tma(nx, m, 2 * m * (c->op[1].nu - 1), pc)) vchunks = want;
  }
  bool v_side_pending = false;   // work on the side streams the caller's stream has not joined
  auto v_join = [&]() -> int {   // caller's stream waits for both side streams
    if (!v_side_pending) return MGRIT_OK;
    for (int sidx = 0; sidx < 2; ++sidx) {
      MG_CK(c, cudaEventRecord(c->hev[sidx], c->hstream[sidx]));
      MG_CK(c, cudaStreamWaitEvent(c->stream, c->hev[sidx], 0));
    }
    v_side_pending = false;
    return MGRIT_OK;
  };
  auto vcycle_overlapped = [&](bool may_spec) -> int {
    const int C_ = vchunks;
    const long long nc1 = c->ntl[1] / m, L = nc1 / C_;
    int s2 = ensure_streams();
    if (s2) return s2;
    while ((int)c->hev.size() < 2 + 2 * C_) {
      cudaEvent_t e = nullptr;
      MG_CK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->hev.push_back(e);
    }
    const cudaStream_t user = c->stream, hi = c->hstream[0], hs = c->hstream[1];
    double *dst = c->unext;     // holds v of the last fine sweep, receives += E
    s2 = v_join();              // the speculative level-1 sweep (if any) is complete
    if (s2) return s2;
    // down leg and the levels below level 1: serial on the caller's stream
    if (c->lsweep1_done) c->lsweep1_done = false;
    else s2 = level_sweep(c, 1, nullptr, c->ul[1]);
    if (!s2) s2 = level_cycle(c, 2, false, rm(c->ul[1], 0, 1));
    if (s2) return s2;
    std::swap(c->ucur, c->unext);                 // the fine sweep chunks read `dst`
#ifdef MG_TRACE
    std::vector<cudaEvent_t> tev(3 * C_ + 1);
    for (auto &e : tev) cudaEventCreate(&e);
    cudaEventRecord(tev[3 * C_], user);
#endif
    MG_CK(c, cudaEventRecord(c->hev[0], user));
    MG_CK(c, cudaStreamWaitEvent(hi, c->hev[0], 0));
    const bool spec = v_spec && may_spec;
    for (int i = 0; i < C_; ++i) {
      c->stream = hi;
      s2 = level_interp(c, 1, c->ul[1], rm(dst, 0, 1), i * L, L);
      c->stream = user;
      if (s2) return s2;
      cudaEvent_t ei = c->hev[2 + 2 * i], fi = c->hev[3 + 2 * i];
      MG_CK(c, cudaEventRecord(ei, hi));
#ifdef MG_TRACE
      cudaEventRecord(tev[3 * i], hi);
#endif
      MG_CK(c, cudaStreamWaitEvent(user, ei, 0));
      const long long j0 = i == 0 ? 0 : 4 * i * L - 2;
      const long long j1 = i + 1 < C_ ? 4 * (i + 1) * L - 2 : nc;
      s2 = do_sweep(false, true, j0, j1 - j0, 0, i + 1 < C_ || spec ? v_per_sm : 0);
      if (s2) return s2;
#ifdef MG_TRACE
      cudaEventRecord(tev[3 * i + 1], user);
#endif
      if (spec) {  // the next V-cycle's level-1 sweep over the intervals whose g_1 rows are final
        MG_CK(c, cudaEventRecord(fi, user));
        MG_CK(c, cudaStreamWaitEvent(hs, fi, 0));
        const long long J0 = i == 0 ? 0 : i * L - 1;
        const long long J1 = i + 1 < C_ ? (i + 1) * L - 1 : nc1;
        c->stream = hs;
        s2 = level_sweep(c, 1, nullptr, c->ul[1], J0, J1 - J0);
        c->stream = user;
        if (s2) return s2;
#ifdef MG_TRACE
        cudaEventRecord(tev[3 * i + 2], hs);
#endif
      }
    }
#ifdef MG_TRACE
    cudaDeviceSynchronize();
    fprintf(stderr, "voverlap trace (ms since the fork): interp end / fine sweep end / level-1 sweep end\n");
    for (int i = 0; i < C_; ++i) {
      float a = 0, b = 0, d = 0;
      cudaEventElapsedTime(&a, tev[3 * C_], tev[3 * i]);
      cudaEventElapsedTime(&b, tev[3 * C_], tev[3 * i + 1]);
      if (spec) cudaEventElapsedTime(&d, tev[3 * C_], tev[3 * i + 2]);
      fprintf(stderr, "  chunk %d: %.3f / %.3f / %.3f\n", i, a, b, d);
    }
    for (auto &e : tev) cudaEventDestroy(e);
#endif
    v_side_pending = true;
    if (spec) c->lsweep1_done = true;
    return MGRIT_OK;
  };
  bool materialised = false;
  std::vector<double> h(1, r0);
  // graph mode (option MGRIT_OPT_GRAPH; default: latency-bound problems): the iterations run
  // as one CUDA graph with a device-side WHILE loop (graph.cu), one host sync per solve
  const bool graph = !c->prof && !crows_hist && max_iter < kGraphHist &&
                     (opt(c, MGRIT_OPT_GRAPH) ? c->opt_v[MGRIT_OPT_GRAPH][0] == 1
                                              : ((long long)nx * c->nt <= (1ll << 23) && !spec_ok));
  // one iteration after the first sweep: coarse correction, (FCF: swap), fused sweep, norm
  auto iteration = [&]() -> int {
    int s2 = coarse_correction(c, rm(fcf ? c->unext : c->ucur, 0, 1));
    if (s2) return s2;
    if (fcf) std::swap(c->ucur, c->unext);
    s2 = do_sweep(false, true);
    if (s2) return s2;
    return reduce_norm(c, partial_count(c, nc, fcf ? 2 * m : m), nullptr);
  };
  if (!conv && !nonfinite && max_iter > 0 && graph) {
    st = do_sweep(true, false);
    if (st) return st;
    c->ucur = c->u0b;
    c->unext = c->v0b;
    // capture and launch on the context's private stream, ordered after the caller's
    if (!c->gstream) {
      MG_CK(c, cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking));
      MG_CK(c, cudaEventCreateWithFlags(&c->gevent, cudaEventDisableTiming));
    }
    const cudaStream_t user = c->stream;
    MG_CK(c, cudaEventRecord(c->gevent, user));
    MG_CK(c, cudaStreamWaitEvent(c->gstream, c->gevent, 0));
    c->stream = c->gstream;
    auto graph_run = [&](LoopState &ls, std::vector<double> &hd) -> int {
      if (!c->gexec) {
        const int s2 = build_loop_graph(c, fcf, iteration);
        c->ucur = c->u0b;
        c->unext = c->v0b;
        if (s2) return s2;
      }
      MG_CK(c, launch_loop_init(c->lstate, tol, c->dx * c->dt, max_iter, 0, c->stream));
      MG_CK(c, cudaGraphLaunch(c->gexec, c->stream));
      MG_CK(c, cudaMemcpyAsync(&ls, c->lstate, sizeof(ls), cudaMemcpyDeviceToHost, c->stream));
      MG_CK(c, cudaMemcpyAsync(hd.data(), c->hist_dev, (max_iter + 1) * sizeof(double),
                               cudaMemcpyDeviceToHost, c->stream));
      MG_CK(c, cudaStreamSynchronize(c->stream));
      return MGRIT_OK;
    };
    LoopState ls;
    std::vector<double> hd(max_iter + 1);
    st = graph_run(ls, hd);
    c->stream = user;
    if (st) return st;
    k = ls.k;
    for (int i = 1; i <= k; ++i) {
      if (hist) hist[i] = hd[i];
      h.push_back(hd[i]);
    }
    nonfinite = ls.nonfinite != 0;
    conv = !nonfinite && hd[k] < tol;
    c->launches += (long long)((k + 1) / 2) * c->glaunch[0] + (long long)(k / 2) * c->glaunch[1] + 1;
    if (fcf && (k & 1)) std::swap(c->ucur, c->unext);   // odd k: the iterate is in v0b
    c->have_iterate = true;
  } else if (!conv && !nonfinite && max_iter > 0) {
    // (worth the extra launches only for sweeps of some length: cfg2's 26 us sweep is not)
    if (spec_ok && sweep_est_ms >= 0.1 &&
        !(out_dev && c->final_sweep != MGRIT_FINAL_OFF &&
          (max_iter <= 1 || c->final_sweep == MGRIT_FINAL_ALWAYS))) {
      // the chain of iteration 1 is launched first, gated on the chunks of the first sweep
      const int C_ = nchunks;
      const long long L = nc / C_;
      st = ensure_streams();
      if (st) return st;
      const int p2 = spec_par ^ 1;
      MG_CK(c, cudaMemsetAsync(c->prog + p2, 0, sizeof(unsigned long long), c->stream));
      MG_CK(c, cudaEventRecord(c->hev[p2], c->stream));
      MG_CK(c, cudaStreamWaitEvent(c->hstream[p2], c->hev[p2], 0));
      const cudaStream_t user = c->stream;
      c->stream = c->hstream[p2];
      st = coarse_solve_level(c, 1, rm(c->unext, 0, 1), rm(c->unext, 0, 1), nullptr, nullptr, 0, -1,
                              c->prog + p2, (int)L, c->prog + 2, flag_seq, C_);
      c->stream = user;
      if (st) return st;
      spec_inflight = true;
      spec_par = p2;
      for (int i = 0; i < C_; ++i) {
        long long j0, j1;
        overlap_sweep_chunk(nc, C_, i, &j0, &j1);
        st = do_sweep(true, false, j0, j1 - j0, 16);
        if (st) return st;
        const int wr = ((mem_fn_t)c->write_value_fn)(user, (unsigned long long)(uintptr_t)(c->prog + 2),
                                                     ++flag_seq, 0u);
        if (wr) return fail(c, MGRIT_ECUDA, "cuStreamWriteValue64 failed (%d)", wr);
      }
    } else {
      st = do_sweep(true, false);
      if (st) return st;
    }
    while (true) {
      Range nv_it("iteration");
      // coarse-grid correction: (FCF) unext += E, then unext becomes the iterate;
      // (F) ucur += e in place
      // residual of iterate k+1 (computed by the next sweep).  Predicted last: the
      // previous two residuals extrapolated geometrically fall below tol.
      ++k;
      bool last = false;
      if (out_dev && c->final_sweep != MGRIT_FINAL_OFF) {
        if (k >= max_iter || c->final_sweep == MGRIT_FINAL_ALWAYS) last = true;
        else if (k >= 2 && h[k - 1] < h[k - 2]) last = h[k - 1] * (h[k - 1] / h[k - 2]) < tol;
      }
      // short sweeps (cfg2: 26 us) are not worth chunking for the last iteration
      const bool ovl = (nchunks > 1 && !(last && sweep_est_ms < 0.1)) || (vchunks > 1 && !last);
      if (ovl && vchunks > 1) {
        st = vcycle_overlapped(k < max_iter);      // level-1 interpolation || fine sweep || next level-1 sweep
      } else if (ovl) {
        // chain || the sweep chunks that measure ||r^(k)|| (check-sweep chunks if predicted last)
        st = overlapped_iteration(k < max_iter, last);
      } else if (spec_inflight) {  // the correction is already running (speculative chain)
        st = wait_chain(spec_par, nchunks);
        spec_inflight = false;
        if (!st && fcf) std::swap(c->ucur, c->unext);
      } else {
        st = v_join();
        if (!st) st = coarse_correction(c, rm(fcf ? c->unext : c->ucur, 0, 1));
        if (!st && fcf) std::swap(c->ucur, c->unext);
      }
      if (st) return st;
      c->have_iterate = true;
      if (crows_hist)
        MG_CK(c, cudaMemcpyAsync(crows_hist + (size_t)(k - 1) * (nc + 1) * nx, c->ucur,
                                 (nc + 1) * row, cudaMemcpyDeviceToDevice, c->stream));
      if (!ovl) st = last ? check_sweep() : do_sweep(false, true);
      if (st) return st;
      double n2;
      st = reduce_norm(c, partial_count(c, nc, fcf ? 2 * m : m), &n2);
      if (st) return st;
      const double rk = std::sqrt(c->dx * c->dt * n2);
      if (hist) hist[k] = rk;
      h.push_back(rk);
      const bool stop = !std::isfinite(rk) || rk < tol || k >= max_iter;
      if (last && stop) materialised = true;
      if (!std::isfinite(rk)) { nonfinite = true; break; }
      if (rk < tol) { conv = true; break; }
      if (k >= max_iter) break;
      if (last) {  // mispredicted: the fused sweep for the next coarse correction
        st = do_sweep(false, false);
        if (st) return st;
      }
    }
  }
  if (iters) *iters = k;
  if (converged) *converged = conv ? 1 : 0;
  if (out_dev) {
    if (!c->have_iterate) {
      MG_CK(c, cudaMemcpyAsync(out_dev, c->guess, (size_t)(c->nt + 1) * row,
                               cudaMemcpyDeviceToDevice, c->stream));
    } else if (materialised) {
      MG_CK(c, cudaMemcpyAsync(out_dev + (size_t)c->nt * nx, c->ucur + (size_t)nc * nx, row,
                               cudaMemcpyDeviceToDevice, c->stream));
    } else {
      SweepArgs a = base_sweep(c);
      a.nitems = (int)nc;
      a.nsteps1 = m - 1;
      a.f_off = 0;
      a.f_stride = m;
      a.in = rm(c->ucur, 0, 1);
      a.each = rm(out_dev, 0, m);
      a.each_step = 1;
      a.each_first = 0;
      a.each_last = m - 1;
      st = sweep(c, 3, a, m - 1);
      if (st) return st;
      MG_CK(c, cudaMemcpyAsync(out_dev + (size_t)c->nt * nx, c->ucur + (size_t)nc * nx, row,
                               cudaMemcpyDeviceToDevice, c->stream));
    }
  }
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return fail(c, MGRIT_ECUDA, "solve: %s", cudaGetErrorString(e));
  if (c->prof) collect(c);
  if (nonfinite) return fail(c, MGRIT_ENONFINITE, "residual became non-finite at iteration %d", k);
  return MGRIT_OK;
}

int mgrit_get_crows(mgrit_ctx *c, double *out_dev) {
  if (!c || !out_dev) return MGRIT_EINVAL;
  const long long nc = c->nt / c->m;
  const size_t row = (size_t)c->nx * sizeof(double);
  if (c->have_iterate)
    MG_CK(c, cudaMemcpyAsync(out_dev, c->ucur, (nc + 1) * row, cudaMemcpyDeviceToDevice, c->stream));
  else
    MG_CK(c, cudaMemcpy2DAsync(out_dev, row, c->guess, row * c->m, row, nc + 1,
                               cudaMemcpyDeviceToDevice, c->stream));
  return MGRIT_OK;
}

int mgrit_fill_guess(double *dst, long long row0, long long rows, int nx, uint64_t seed, int lo_kind,
                     const double *u0, void *stream) {
  if (!dst || nx < 1 || rows < 0 || (lo_kind != 0 && lo_kind != 1)) return MGRIT_EINVAL;
  cudaError_t e = launch_fill_guess(dst, row0, rows, nx, seed, lo_kind, u0, (cudaStream_t)stream);
  return e == cudaSuccess ? MGRIT_OK : MGRIT_ECUDA;
}

int mgrit_profile_enable(mgrit_ctx *c, int on) {
  if (!c) return MGRIT_EINVAL;
  cudaStreamSynchronize(c->stream);
  collect(c);
  c->prof = on != 0;
  std::memset(c->prof_launch, 0, sizeof(c->prof_launch));
  std::memset(c->prof_ms, 0, sizeof(c->prof_ms));
  c->launches = 0;
  return MGRIT_OK;
}

int mgrit_profile_read(mgrit_ctx *c, long long *launches, double *ms) {
  if (!c) return MGRIT_EINVAL;
  cudaStreamSynchronize(c->stream);
  collect(c);
  for (int i = 0; i < MGRIT_PROF_CLASSES; ++i) {
    if (launches) launches[i] = c->prof_launch[i];
    if (ms) ms[i] = c->prof_ms[i];
  }
  return MGRIT_OK;
}

long long mgrit_launch_count(const mgrit_ctx *c) { return c ? c->launches : -1; }

int mgrit_describe(const mgrit_ctx *c, char *buf, size_t len) {
  if (!c || !buf || len == 0) return MGRIT_EINVAL;
  FineCfg f;
  const int m = c->m;
  const bool ok = choose_fine(c, c->relax == MGRIT_RELAX_FCF ? 2 * m : m, f);
  const bool tma = ok && f.ntiles > 1 && (c->nx % 2 == 0) && (f.cfg.p % 2 == 1);
  const char *kern = !ok ? "none" : (tma ? "rk_sweep_tma_kernel" : "rk_sweep_kernel");
  char coarse[96] = "rk_coarse_kernel";
  if (c->psi_kind == MGRIT_PSI_STENCIL) {
    const CoarsePlan pl = plan_coarse(c, c->levels - 1);
    if (pl.kind == CoarsePlan::CLUSTER_CA)
      snprintf(coarse, sizeof(coarse), "%s<NT=%d,P=%d,CL=%d,S=%d>",
               pl.tb ? "psi_seq_cluster_tb_kernel" : "psi_seq_cluster_ca_kernel",
               pl.cfg.nt_threads, pl.cfg.p, pl.cl, pl.S);
    else if (pl.kind == CoarsePlan::CLUSTER)
      snprintf(coarse, sizeof(coarse), "psi_seq_cluster_kernel<NT=%d,P=%d,CL=%d>", pl.cfg.nt_threads,
               pl.cfg.p, pl.cl);
    else if (pl.kind == CoarsePlan::SEQ)
      snprintf(coarse, sizeof(coarse), "psi_seq_periodic_kernel<NT=%d,P=%d>", pl.cfg.nt_threads, pl.cfg.p);
    else if (pl.kind == CoarsePlan::TILES)
      snprintf(coarse, sizeof(coarse), "psi_coarse_kernel<NT=%d,P=%d> tiles=%d", pl.cfg.nt_threads,
               pl.cfg.p, pl.ntiles);
    else if (pl.kind == CoarsePlan::TILES_SEG)
      snprintf(coarse, sizeof(coarse), "psi_coarse_kernel<NT=%d,P=%d> tiles=%d seg=%d",
               pl.cfg.nt_threads, pl.cfg.p, pl.ntiles, pl.seg);
    else
      snprintf(coarse, sizeof(coarse), "none");
  }
  snprintf(buf, len, "fine=%s<scheme%d,NT=%d,P=%d> tiles=%d halo=%d levels=%d coarse=%s", kern,
           c->scheme, ok ? f.cfg.nt_threads : 0, ok ? f.cfg.p : 0, ok ? f.ntiles : 0, ok ? f.HL : 0,
           c->levels, coarse);
  return MGRIT_OK;
}

// ---- time shards ---------------------------------------------------------------------
size_t mgrit_workspace_bytes_shard(int nx, int nt, int m, int levels, int nranks) {
  if (nranks < 1 || nt % nranks) return 0;
  return mgrit_workspace_bytes(nx, nt / nranks, m, levels);
}

int mgrit_setup_shard(mgrit_ctx **out, int nx, int nt, int m, double alpha, double cfl, int order,
                      int tableau, int levels, const mgrit_psi *psi, int relax, int rank,
                      int nranks, double *stage_send, double *stage_recv, void *workspace_dev,
                      size_t workspace_bytes, void *stream) {
  if (!out) return MGRIT_EINVAL;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks || nt % nranks) {
    fprintf(stderr, "mgrit_setup_shard: bad rank/nranks or nt %% nranks != 0\n");
    return MGRIT_EINVAL;
  }
  if (nranks > 1 && (!stage_send || !stage_recv)) {
    fprintf(stderr, "mgrit_setup_shard: staging rows required\n");
    return MGRIT_EINVAL;
  }
  const int st = mgrit_setup(out, nx, nt / nranks, m, alpha, cfl, order, tableau, levels, psi,
                             relax, workspace_dev, workspace_bytes, stream);
  if (st) return st;
  (*out)->rank = rank;
  (*out)->nranks = nranks;
  (*out)->stage_send = stage_send;
  (*out)->stage_recv = stage_recv;
  return MGRIT_OK;
}

int mgrit_solve_shard(mgrit_ctx *c, const mgrit_comm *comm, double tol, int max_iter,
                      double *out_dev, int *iters, double *hist, int *converged) {
  if (!c) return MGRIT_EINVAL;
  if (!c->guess) return fail(c, MGRIT_EINVAL, "mgrit_set_guess first");
  if (max_iter < 0) return fail(c, MGRIT_EINVAL, "max_iter < 0");
  if (c->nranks > 1 && (!comm || !comm->shift || !comm->allreduce_sum))
    return fail(c, MGRIT_EINVAL, "time shards need a mgrit_comm");
  if (c->psi_kind != MGRIT_PSI_STENCIL || c->cycle != MGRIT_CYCLE_V)
    return fail(c, MGRIT_EUNSUPPORTED, "time shards: stencil Psi and V-cycles only");
  Range nv_solve("mgrit_solve_shard");
  c->comm = comm;
  struct Reset {
    mgrit_ctx *c;
    ~Reset() { c->comm = nullptr; }
  } reset{c};
  const int m = c->m, nx = c->nx;
  const long long nc = c->nt / m;
  const size_t row = (size_t)nx * sizeof(double);
  const bool fcf = c->relax == MGRIT_RELAX_FCF;
  const double dxdt = c->dx * c->dt;
  c->ucur = c->u0b;
  c->unext = c->v0b;
  MG_CK(c, cudaMemcpyAsync(c->u0b, c->guess, row, cudaMemcpyDeviceToDevice, c->stream));
  MG_CK(c, cudaMemcpyAsync(c->v0b, c->guess, row, cudaMemcpyDeviceToDevice, c->stream));
  // hist[0]: the guess's residual over the block's rows, summed over the ranks
  double n2 = 0.0;
  int st = residual0(c, c->guess, &n2, nullptr);
  if (st) return st;
  st = comm_sum(c, &n2, 1);
  if (st) return st;
  const double r0 = std::sqrt(dxdt * n2);
  if (hist) hist[0] = r0;
  if (!fcf)
    MG_CK(c, cudaMemcpy2DAsync(c->ucur, row, c->guess, row * m, row, nc + 1,
                               cudaMemcpyDeviceToDevice, c->stream));
  auto do_sweep = [&](bool first, bool want_norm) -> int {
    SweepArgs a = base_sweep(c);
    a.nitems = (int)nc;
    a.nsteps1 = m;
    a.f_off = 0;
    a.f_stride = m;
    if (first && fcf) {
      a.in = rm(c->guess, 0, m);
      a.cmp = rm(c->guess, m, m);
    } else {
      a.in = rm(c->ucur, 0, 1);
      a.cmp = rm(c->ucur, 1, 1);
    }
    a.partials = want_norm ? c->partials : nullptr;
    if (fcf) {
      a.endw = rm(c->unext, 1, 1);
      a.nsteps2 = m;
      a.p2_items = p2_count(c, nc);
      a.r2 = rm(c->g[1], 2, 1);
    } else {
      a.dstore = rm(c->g[1], 1, 1);
      a.d_every = 1;
      a.d_phase = 0;
    }
    int s2 = sweep(c, 0, a, fcf ? 2 * m : m);
    if (s2) return s2;
    // the right neighbour's first coarse RHS row r_{nc+1} (FCF; Parareal's r_j are local)
    return fcf ? comm_shift(c, row_ptr(c, c->g[1], nc + 1), row_ptr(c, c->g[1], 1)) : MGRIT_OK;
  };
  int k = 0;
  bool conv = r0 < tol, nonfinite = !std::isfinite(r0);
  c->have_iterate = false;
  if (!conv && !nonfinite && max_iter > 0) {
    st = do_sweep(true, false);
    if (st) return st;
    while (true) {
      Range nv_it("iteration");
      st = level_cycle_shard(c, 1, rm(fcf ? c->unext : c->ucur, 0, 1));
      if (st) return st;
      if (fcf) std::swap(c->ucur, c->unext);
      c->have_iterate = true;
      ++k;
      // the corrected C-row at the block start belongs to rank-1
      st = comm_shift(c, row_ptr(c, c->ucur, nc), row_ptr(c, c->ucur, 0));
      if (st) return st;
      st = do_sweep(false, true);
      if (st) return st;
      st = reduce_norm(c, partial_count(c, nc, fcf ? 2 * m : m), &n2);
      if (st) return st;
      st = comm_sum(c, &n2, 1);
      if (st) return st;
      const double rk = std::sqrt(dxdt * n2);
      if (hist) hist[k] = rk;
      if (!std::isfinite(rk)) { nonfinite = true; break; }
      if (rk < tol) { conv = true; break; }
      if (k >= max_iter) break;
    }
  }
  if (iters) *iters = k;
  if (converged) *converged = conv ? 1 : 0;
  if (out_dev) {
    if (!c->have_iterate) {
      MG_CK(c, cudaMemcpyAsync(out_dev, c->guess, (size_t)(c->nt + 1) * row,
                               cudaMemcpyDeviceToDevice, c->stream));
    } else {
      SweepArgs a = base_sweep(c);
      a.nitems = (int)nc;
      a.nsteps1 = m - 1;
      a.f_off = 0;
      a.f_stride = m;
      a.in = rm(c->ucur, 0, 1);
      a.each = rm(out_dev, 0, m);
      a.each_step = 1;
      a.each_first = 0;
      a.each_last = m - 1;
      st = sweep(c, 3, a, m - 1);
      if (st) return st;
      MG_CK(c, cudaMemcpyAsync(out_dev + (size_t)c->nt * nx, c->ucur + (size_t)nc * nx, row,
                               cudaMemcpyDeviceToDevice, c->stream));
    }
  }
  const cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return fail(c, MGRIT_ECUDA, "solve_shard: %s", cudaGetErrorString(e));
  if (nonfinite) return fail(c, MGRIT_ENONFINITE, "residual became non-finite at iteration %d", k);
  return MGRIT_OK;
}

}  // extern "C"
