// psifit.cu — GPU synthesis of the coarse operators Psi_l (§4,
// eq. (LSQ_1D_problem), weights P:338-342, patterns P:568 / P:786, recursion
// P:620).  The host numpy fit (paper_1910_03726_b200/psi.py) stays the reference input
// path; this is the same weighted linear least-squares problem solved on the device.
//
// For a contiguous pattern d_a = o0 + a, a = 0..nu-1, the real minimiser of
//   || W^{1/2} (lambda^m - mu(psi)) ||_2,   mu_k = sum_a psi_a e^{i theta_k d_a},
// satisfies the normal equations (Lemma 3's proof)  G psi = h  with
//   G_ab = sum_k w_k Re(e^{-i theta_k d_a} e^{i theta_k d_b})
//   h_a  = sum_k w_k Re(e^{-i theta_k d_a} lambda_k^m),
// w_k = 1/(1 - |lambda_k| + eps)^2, eps = 1e-6.  The weights span ~12 orders of magnitude
// (w_0 = 1e12 at |lambda_0| = 1), so G is formed and factored in double-double arithmetic
// (error-free TwoSum / TwoProd via FMA): the sums keep the small-weight modes that an fp64
// sum would round away, and the Cholesky factorisation of the ill-conditioned G stays
// accurate (tests/test_oracle_pins.py pins the same equations at 50 digits).  The P:394
// flag is the imaginary part of the complex problem's solution, G^-1 h_I with
// h_I,a = sum_k w_k Im(e^{-i theta_k d_a} lambda_k^m) (zero in exact arithmetic, Lemma 3).
//
// Kernels: symbol (lambda_k, lambda_k^m, w_k per frequency), partial sums per k-chunk
// (one thread per output entry and chunk, fixed order), a one-thread double-double Cholesky
// solve, and a direct inverse DFT for the eta-threshold pattern (first column of Phi^m).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/mgrit.h"
#include "kernels.h"

namespace mg {
namespace {

struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_norm(double hi, double lo) {
  const double s = hi + lo;
  return {s, lo - (s - hi)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = dd_norm(s.hi, s.lo);
  s.lo += t.lo;
  return dd_norm(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e = fma(a.hi, b.lo, e);
  e = fma(a.lo, b.hi, e);
  return dd_norm(p, e);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  const double p = a.hi * b;
  double e = fma(a.hi, b, -p);
  e = fma(a.lo, b, e);
  return dd_norm(p, e);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_div(dd a, dd b) {
  const double q1 = a.hi / b.hi;
  const dd r = dd_add(a, dd_neg(dd_mul_d(b, q1)));
  const double q2 = r.hi / b.hi;
  const dd r2 = dd_add(r, dd_neg(dd_mul_d(b, q2)));
  const double q3 = r2.hi / b.hi;
  return dd_add(dd_norm(q1, q2), {q3, 0.0});
}
__device__ __forceinline__ dd dd_sqrt(dd a) {
  const double x = sqrt(a.hi);
  const dd x2 = dd_mul({x, 0.0}, {x, 0.0});
  const dd r = dd_add(a, dd_neg(x2));
  return dd_add({x, 0.0}, {r.hi / (2.0 * x), 0.0});
}
// w * t accumulated into s (t a double, w a double): error-free product then dd add
__device__ __forceinline__ dd dd_fma_acc(dd s, double w, double t) {
  const double p = w * t;
  return dd_add(s, dd_norm(p, fma(w, t, -p)));
}

// e^{i theta_k q} with exact argument reduction: theta_k q = 2 pi ((k q) mod nx) / nx.
__device__ __forceinline__ void expi(long long k, long long q, int nx, double &c, double &s) {
  long long r = (k * q) % nx;
  if (r < 0) r += nx;
  sincospi(2.0 * (double)r / (double)nx, &s, &c);
}

struct FitSym {
  int nx, m, s, implicit;   // s > 0: Runge-Kutta symbol from (z, A, b); s == 0: stencil
  int zlo, zn;
  double z[MAX_PSI];
  double A[MAXS][MAXS];
  double b[MAXS];
};

// lambda_k (Runge-Kutta: R(zhat_k) by forward substitution of (I - zA) x = 1, P:142-152;
// stencil: sum_d z_d e^{i theta_k d}), t_k = lambda_k^m, w_k.
__global__ void fit_symbol_kernel(const __grid_constant__ FitSym a, double *lam_re,
                                  double *lam_im, double *t_re, double *t_im, double *w) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= a.nx) return;
  double zr = 0.0, zi = 0.0;
  for (int j = 0; j < a.zn; ++j) {
    double c, s;
    expi(k, a.zlo + j, a.nx, c, s);
    zr = fma(a.z[j], c, zr);
    zi = fma(a.z[j], s, zi);
  }
  double lr = zr, li = zi;
  if (a.s > 0) {
    double xr[MAXS], xi[MAXS];
    double ur = 0.0, ui = 0.0;                    // sum_i b_i x_i
    for (int i = 0; i < a.s; ++i) {
      double nr = 1.0, ni = 0.0;                  // 1 + z sum_{j<i} A_ij x_j
      double sr = 0.0, si = 0.0;
      for (int j = 0; j < i; ++j) {
        sr = fma(a.A[i][j], xr[j], sr);
        si = fma(a.A[i][j], xi[j], si);
      }
      nr += zr * sr - zi * si;
      ni += zr * si + zi * sr;
      const double dr = 1.0 - a.A[i][i] * zr, di = -a.A[i][i] * zi;
      const double den = dr * dr + di * di;
      xr[i] = (nr * dr + ni * di) / den;
      xi[i] = (ni * dr - nr * di) / den;
      ur = fma(a.b[i], xr[i], ur);
      ui = fma(a.b[i], xi[i], ui);
    }
    lr = 1.0 + (zr * ur - zi * ui);
    li = zr * ui + zi * ur;
  }
  double pr = 1.0, pi = 0.0;
  for (int q = 0; q < a.m; ++q) {
    const double nr = pr * lr - pi * li, ni = pr * li + pi * lr;
    pr = nr;
    pi = ni;
  }
  const double ww = 1.0 / ((1.0 - hypot(lr, li) + 1e-6) * (1.0 - hypot(lr, li) + 1e-6));
  lam_re[k] = lr;
  lam_im[k] = li;
  t_re[k] = pr;
  t_im[k] = pi;
  w[k] = ww;
}

constexpr int kChunk = 256;

// Output entries: G_ab for the np = nu(nu+1)/2 pairs a <= b (row-packed), then h_a, then
// h_I,a; partial[e * nchunks + c] = double-double sum over the k in chunk c.  G is formed
// from the same fp64 basis values e^{i theta_k d_a} as h (G_ab = sum_k w_k (c_a c_b +
// s_a s_b), exact products): the normal equations of ONE least-squares problem.  (The
// Toeplitz shortcut g(d_b - d_a) = sum_k w_k cos(theta_k (d_b - d_a)) is the same matrix in
// exact arithmetic but, from rounded basis values, not the Gram matrix of the basis h uses;
// with the smooth modes weighted 1e12 that inconsistency moved psi by ~1e-7.)
__device__ __forceinline__ dd dd_prod(double a, double b) {
  const double p = a * b;
  return {p, fma(a, b, -p)};
}
__global__ void fit_sums_kernel(int nx, int nu, int o0, const double *t_re, const double *t_im,
                                const double *w, double *part_hi, double *part_lo, int nchunks) {
  const int e = blockIdx.y * blockDim.x + threadIdx.x;
  const int c = blockIdx.x;
  const int np = nu * (nu + 1) / 2;
  if (e >= np + 2 * nu) return;
  int ia = 0, ib = 0;
  if (e < np) {  // row-packed (a, b), b <= a: e = a(a+1)/2 + b
    while ((ia + 1) * (ia + 2) / 2 <= e) ++ia;
    ib = e - ia * (ia + 1) / 2;
  }
  dd s = {0.0, 0.0};
  const int k0 = c * kChunk, k1 = min(nx, k0 + kChunk);
  for (int k = k0; k < k1; ++k) {
    dd term;
    if (e < np) {
      double ca, sa, cb, sb;
      expi(k, o0 + ia, nx, ca, sa);
      expi(k, o0 + ib, nx, cb, sb);
      term = dd_add(dd_prod(ca, cb), dd_prod(sa, sb));
    } else {
      const int a = e < np + nu ? e - np : e - np - nu;
      double ca, sa;
      expi(k, o0 + a, nx, ca, sa);
      // e^{-i theta d} t = (ca - i sa)(tr + i ti): Re = ca tr + sa ti, Im = ca ti - sa tr
      term = e < np + nu ? dd_add(dd_prod(ca, t_re[k]), dd_prod(sa, t_im[k]))
                         : dd_add(dd_prod(ca, t_im[k]), dd_neg(dd_prod(sa, t_re[k])));
    }
    s = dd_add(s, dd_mul_d(term, w[k]));
  }
  part_hi[e * nchunks + c] = s.hi;
  part_lo[e * nchunks + c] = s.lo;
}

// One thread: sum the chunks (fixed order), build G, Cholesky in double-double, solve for
// psi and the imaginary diagnostic.  out[0..nu): psi, out[nu]: max |imag part|.
constexpr size_t kSolveSmem = sizeof(double) * 2 * (MAX_PSI * (MAX_PSI + 1) / 2 + 2 * MAX_PSI);

__global__ void fit_solve_kernel(int nu, const double *part_hi, const double *part_lo,
                                 int nchunks, double *out) {
  // the factor and right-hand sides live in shared memory (a 36 KB per-thread stack
  // would make the driver reserve local memory for every resident thread of the GPU)
  extern __shared__ dd sm[];
  if (threadIdx.x || blockIdx.x) return;
  dd *h = sm, *hI = h + MAX_PSI, *G = hI + MAX_PSI;     // G row-packed, then factored in place
  const int np = nu * (nu + 1) / 2;
  for (int e = 0; e < np + 2 * nu; ++e) {
    dd s = {0.0, 0.0};
    for (int c = 0; c < nchunks; ++c) s = dd_add(s, {part_hi[e * nchunks + c], part_lo[e * nchunks + c]});
    if (e < np) G[e] = s;
    else if (e < np + nu) h[e - np] = s;
    else hI[e - np - nu] = s;
  }
  // Cholesky G = L L^T in place (row-packed lower triangle: entry (i, j), j <= i)
  auto at = [&](int i, int j) -> dd & { return G[i * (i + 1) / 2 + j]; };
  for (int j = 0; j < nu; ++j) {
    dd d = at(j, j);
    for (int k = 0; k < j; ++k) d = dd_add(d, dd_neg(dd_mul(at(j, k), at(j, k))));
    const dd ljj = dd_sqrt(d);
    at(j, j) = ljj;
    for (int i = j + 1; i < nu; ++i) {
      dd v = at(i, j);
      for (int k = 0; k < j; ++k) v = dd_add(v, dd_neg(dd_mul(at(i, k), at(j, k))));
      at(i, j) = dd_div(v, ljj);
    }
  }
  auto solve = [&](dd *b) {  // L L^T x = b in place
    for (int i = 0; i < nu; ++i) {
      dd v = b[i];
      for (int k = 0; k < i; ++k) v = dd_add(v, dd_neg(dd_mul(at(i, k), b[k])));
      b[i] = dd_div(v, at(i, i));
    }
    for (int i = nu - 1; i >= 0; --i) {
      dd v = b[i];
      for (int k = i + 1; k < nu; ++k) v = dd_add(v, dd_neg(dd_mul(at(k, i), b[k])));
      b[i] = dd_div(v, at(i, i));
    }
  };
  solve(h);
  solve(hI);
  double imag = 0.0;
  for (int a = 0; a < nu; ++a) {
    out[a] = h[a].hi + h[a].lo;
    imag = fmax(imag, fabs(hI[a].hi + hI[a].lo));
  }
  out[nu] = imag;
}

// ---------------------------------------------------------------------------
// Nonlinear least squares (Appendix B, eq. (nlsq); R21):
//   F(psi) = (1/nx) sum_k |r_k|^2,  r_k = C_k g(|mu_k|) (lambda_k^m - mu_k),
//   C_k = sqrt(m) |lambda_k|^m,  g(a) = sum_{j=0}^{N-2} a^j (N = nt/m; Horner),
// the two-level FCF estimate (Dobrev_bounds) P:283-293 per Fourier mode.
// nl_mode_kernel: one thread per mode k -> mu_k, r_k and the two factors of the Jacobian row
//   dr_k/dpsi_a = P_k rho_ka - Q_k E_ka,  E_ka = e^{i theta_k d_a},  rho_ka = Re(conj(mu_k) E_ka),
//   P_k = C_k g'(a_k)/a_k (lambda_k^m - mu_k)  (complex),  Q_k = C_k g(a_k)  (real).
// nl_sums_kernel: double-double partial sums per k-chunk of G_ab = sum_k Re(conj(J_ka) J_kb),
//   h_a = sum_k Re(conj(J_ka) r_k) and sum_k |r_k|^2 (fixed order).
// nl_step_kernel: one thread, (G + l I) delta = -h by Cholesky in double-double,
//   psi_trial = psi + delta, |delta|, |psi|.
// ---------------------------------------------------------------------------
__global__ void nl_mode_kernel(int nx, int nu, int o0, int m, int nterms, const double *psi,
                               const double *lam_re, const double *lam_im, const double *t_re,
                               const double *t_im, double *mu_re, double *mu_im, double *r_re,
                               double *r_im, double *P_re, double *P_im, double *Q) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nx) return;
  double mr = 0.0, mi = 0.0;
  for (int a = 0; a < nu; ++a) {
    double c, s;
    expi(k, o0 + a, nx, c, s);
    mr = fma(psi[a], c, mr);
    mi = fma(psi[a], s, mi);
  }
  const double am = hypot(mr, mi);
  double g = 1.0, dg = 0.0;
  for (int j = 1; j < nterms; ++j) {
    dg = fma(dg, am, g);
    g = fma(g, am, 1.0);
  }
  const double al = hypot(lam_re[k], lam_im[k]);
  double C = sqrt((double)m);
  for (int q = 0; q < m; ++q) C *= al;
  const double dr = t_re[k] - mr, di = t_im[k] - mi;
  mu_re[k] = mr;
  mu_im[k] = mi;
  r_re[k] = C * g * dr;
  r_im[k] = C * g * di;
  const double pf = am > 0.0 ? C * dg / am : 0.0;
  P_re[k] = pf * dr;
  P_im[k] = pf * di;
  Q[k] = C * g;
}

// entries: G_ab (np = nu(nu+1)/2 row-packed pairs b <= a), h_a (nu), F (1)
__global__ void nl_sums_kernel(int nx, int nu, int o0, const double *mu_re, const double *mu_im,
                               const double *r_re, const double *r_im, const double *P_re,
                               const double *P_im, const double *Q, double *part_hi,
                               double *part_lo, int nchunks, int f_only) {
  const int e = blockIdx.y * blockDim.x + threadIdx.x;
  const int c = blockIdx.x;
  const int np = nu * (nu + 1) / 2;
  if (e >= np + nu + 1) return;
  if (f_only && e != np + nu) return;
  int ia = 0, ib = 0;
  if (e < np) {
    while ((ia + 1) * (ia + 2) / 2 <= e) ++ia;
    ib = e - ia * (ia + 1) / 2;
  } else if (e < np + nu) {
    ia = e - np;
  }
  dd s = {0.0, 0.0};
  const int k0 = c * kChunk, k1 = min(nx, k0 + kChunk);
  for (int k = k0; k < k1; ++k) {
    if (e == np + nu) {
      s = dd_add(s, dd_add(dd_prod(r_re[k], r_re[k]), dd_prod(r_im[k], r_im[k])));
      continue;
    }
    double ca, sa;
    expi(k, o0 + ia, nx, ca, sa);
    const double rho_a = mu_re[k] * ca + mu_im[k] * sa;          // Re(conj(mu) E_a)
    const double ja_re = P_re[k] * rho_a - Q[k] * ca, ja_im = P_im[k] * rho_a - Q[k] * sa;
    if (e < np) {
      double cb, sb;
      expi(k, o0 + ib, nx, cb, sb);
      const double rho_b = mu_re[k] * cb + mu_im[k] * sb;
      const double jb_re = P_re[k] * rho_b - Q[k] * cb, jb_im = P_im[k] * rho_b - Q[k] * sb;
      s = dd_add(s, dd_add(dd_prod(ja_re, jb_re), dd_prod(ja_im, jb_im)));
    } else {
      s = dd_add(s, dd_add(dd_prod(ja_re, r_re[k]), dd_prod(ja_im, r_im[k])));
    }
  }
  part_hi[e * nchunks + c] = s.hi;
  part_lo[e * nchunks + c] = s.lo;
}

// out[0..nu): psi + delta, out[nu]: |delta|, out[nu+1]: |psi|, out[nu+2]: sum |r|^2 (of the
// point the sums were formed at).  sum_only: just out[nu+2].
__global__ void nl_step_kernel(int nu, const double *psi, double lmb, const double *part_hi,
                               const double *part_lo, int nchunks, int sum_only, double *out) {
  extern __shared__ dd sm[];
  if (threadIdx.x || blockIdx.x) return;
  dd *h = sm, *G = h + MAX_PSI;
  const int np = nu * (nu + 1) / 2;
  for (int e = sum_only ? np + nu : 0; e < np + nu + 1; ++e) {
    dd s = {0.0, 0.0};
    for (int c = 0; c < nchunks; ++c) s = dd_add(s, {part_hi[e * nchunks + c], part_lo[e * nchunks + c]});
    if (e < np) G[e] = s;
    else if (e < np + nu) h[e - np] = dd_neg(s);
    else out[nu + 2] = s.hi + s.lo;
  }
  if (sum_only) return;
  auto at = [&](int i, int j) -> dd & { return G[i * (i + 1) / 2 + j]; };
  for (int j = 0; j < nu; ++j) at(j, j) = dd_add(at(j, j), {lmb, 0.0});
  for (int j = 0; j < nu; ++j) {
    dd d = at(j, j);
    for (int k = 0; k < j; ++k) d = dd_add(d, dd_neg(dd_mul(at(j, k), at(j, k))));
    const dd ljj = dd_sqrt(d);
    at(j, j) = ljj;
    for (int i = j + 1; i < nu; ++i) {
      dd v = at(i, j);
      for (int k = 0; k < j; ++k) v = dd_add(v, dd_neg(dd_mul(at(i, k), at(j, k))));
      at(i, j) = dd_div(v, ljj);
    }
  }
  for (int i = 0; i < nu; ++i) {
    dd v = h[i];
    for (int k = 0; k < i; ++k) v = dd_add(v, dd_neg(dd_mul(at(i, k), h[k])));
    h[i] = dd_div(v, at(i, i));
  }
  for (int i = nu - 1; i >= 0; --i) {
    dd v = h[i];
    for (int k = i + 1; k < nu; ++k) v = dd_add(v, dd_neg(dd_mul(at(k, i), h[k])));
    h[i] = dd_div(v, at(i, i));
  }
  double nd = 0.0, npsi = 0.0;
  for (int a = 0; a < nu; ++a) {
    const double d = h[a].hi + h[a].lo;
    out[a] = psi[a] + d;
    nd = fma(d, d, nd);
    npsi = fma(psi[a], psi[a], npsi);
  }
  out[nu] = sqrt(nd);
  out[nu + 1] = sqrt(npsi);
}

// Real part of the first column of Phi^m: col_j = (1/nx) sum_k t_k e^{2 pi i jk/nx}.
__global__ void fit_idft_kernel(int nx, const double *t_re, const double *t_im, double *col) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nx) return;
  double s = 0.0;
  for (int k = 0; k < nx; ++k) {
    double c, sn;
    expi(k, j, nx, c, sn);
    s = fma(t_re[k], c, fma(-t_im[k], sn, s));
  }
  col[j] = s / nx;
}

}  // namespace
}  // namespace mg

using namespace mg;

namespace {
int round_half_away(double x) {
  const int r = (int)std::floor(std::fabs(x) + 0.5);
  return x >= 0 ? r : -r;
}
}  // namespace

extern "C" {

size_t mgrit_psi_fit_workspace_bytes(int nx) {
  if (nx < 2) return 0;
  const size_t nch = (size_t)(nx + kChunk - 1) / kChunk;
  const size_t ne = (size_t)MAX_PSI * (MAX_PSI + 1) / 2 + 2 * MAX_PSI;
  return sizeof(double) * (6 * (size_t)nx + 2 * ne * nch + MAX_PSI + 8) + 256;
}

int mgrit_psi_fit(int nx, int order, int tableau, double cfl, int m, int levels,
                  const int *widths, double eta, int *offsets_out, int *nnz_out,
                  double *coeffs_out, double *imag_out, void *workspace_dev,
                  size_t workspace_bytes, void *stream_) {
  if (nx < 8 || m < 2 || levels < 2 || levels > MGRIT_MAX_LEVELS || !offsets_out || !nnz_out ||
      !coeffs_out || !workspace_dev || (!widths && !(eta > 0.0)))
    return MGRIT_EINVAL;
  if (workspace_bytes < mgrit_psi_fit_workspace_bytes(nx)) return MGRIT_ENOMEM;
  if (eta > 0.0 && levels != 2) return MGRIT_EINVAL;   // threshold patterns: two levels
  cudaStream_t st = (cudaStream_t)stream_;
  int s = 0, zlo = 0, zn = 0;
  double z[8], A[36], b[6];
  if (mgrit_scheme_coefficients(order, tableau, cfl, &s, &zlo, &zn, z, A, b)) return MGRIT_EINVAL;
  const int nch = (nx + kChunk - 1) / kChunk;
  double *w0 = (double *)workspace_dev;
  double *lr = w0, *li = lr + nx, *tr = li + nx, *ti = tr + nx, *ww = ti + nx, *col = ww + nx;
  const size_t ne = (size_t)MAX_PSI * (MAX_PSI + 1) / 2 + 2 * MAX_PSI;
  double *phi = col + nx, *plo = phi + ne * nch, *res = plo + ne * nch;
  FitSym sym;
  std::memset(&sym, 0, sizeof(sym));
  sym.nx = nx;
  sym.m = m;
  sym.s = s;
  sym.zlo = zlo;
  sym.zn = zn;
  for (int j = 0; j < zn; ++j) sym.z[j] = z[j];
  for (int i = 0; i < s; ++i) {
    sym.b[i] = b[i];
    for (int j = 0; j < s; ++j) sym.A[i][j] = A[i * 6 + j];
  }
  std::vector<double> hcol(nx), hout(MAX_PSI + 1);
  for (int l = 0; l < levels - 1; ++l) {
    fit_symbol_kernel<<<(nx + 255) / 256, 256, 0, st>>>(sym, lr, li, tr, ti, ww);
    if (cudaGetLastError() != cudaSuccess) return MGRIT_ECUDA;
    int o0, nu;
    if (eta > 0.0) {   // contiguous hull of |col_j| >= eta max|col| (d = -j wrapped)
      fit_idft_kernel<<<(nx + 127) / 128, 128, 0, st>>>(nx, tr, ti, col);
      if (cudaMemcpyAsync(hcol.data(), col, nx * sizeof(double), cudaMemcpyDeviceToHost, st) !=
              cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess)
        return MGRIT_ECUDA;
      double mx = 0.0;
      for (int j = 0; j < nx; ++j) mx = std::max(mx, std::fabs(hcol[j]));
      int dlo = nx, dhi = -nx;
      for (int j = 0; j < nx; ++j)
        if (std::fabs(hcol[j]) >= eta * mx) {
          const int d = ((-j + nx / 2) % nx + nx) % nx - nx / 2;
          dlo = std::min(dlo, d);
          dhi = std::max(dhi, d);
        }
      o0 = dlo;
      nu = dhi - dlo + 1;
    } else {            // window of widths[l] centred on -m^(l+1) c (R8)
      nu = widths[l];
      const int centre = round_half_away(-std::pow((double)m, l + 1) * cfl);
      o0 = centre - (nu - 1) / 2;
    }
    if (nu < 1 || nu > MGRIT_MAX_PSI_TAPS || nu > nx / 2) return MGRIT_EINVAL;
    dim3 grid(nch, (nu * (nu + 1) / 2 + 2 * nu + 127) / 128);
    fit_sums_kernel<<<grid, 128, 0, st>>>(nx, nu, o0, tr, ti, ww, phi, plo, nch);
    fit_solve_kernel<<<1, 32, kSolveSmem, st>>>(nu, phi, plo, nch, res);
    if (cudaGetLastError() != cudaSuccess) return MGRIT_ECUDA;
    if (cudaMemcpyAsync(hout.data(), res, (nu + 1) * sizeof(double), cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return MGRIT_ECUDA;
    nnz_out[l] = nu;
    for (int a = 0; a < nu; ++a) {
      offsets_out[l * MGRIT_MAX_PSI_TAPS + a] = o0 + a;
      coeffs_out[l * MGRIT_MAX_PSI_TAPS + a] = hout[a];
    }
    if (imag_out) imag_out[l] = hout[nu];
    // the next level coarsens Psi_l: its symbol is the stencil's
    std::memset(&sym, 0, sizeof(sym));
    sym.nx = nx;
    sym.m = m;
    sym.s = 0;
    sym.zlo = o0;
    sym.zn = nu;
    for (int a = 0; a < nu; ++a) sym.z[a] = hout[a];
  }
  return MGRIT_OK;
}

size_t mgrit_psi_fit_nl_workspace_bytes(int nx) {
  if (nx < 2) return 0;
  const size_t nch = (size_t)(nx + kChunk - 1) / kChunk;
  const size_t ne = (size_t)MAX_PSI * (MAX_PSI + 1) / 2 + MAX_PSI + 1;
  return sizeof(double) * (12 * (size_t)nx + 2 * ne * nch + 3 * MAX_PSI + 16) + 256;
}

int mgrit_psi_fit_nl(int nx, int order, int tableau, double cfl, int m, int nt, int nnz,
                     const int *offsets, double *coeffs, int max_iter, int *iters_out,
                     double *objective_out, double *history_out, void *workspace_dev,
                     size_t workspace_bytes, void *stream_) {
  if (nx < 8 || m < 2 || nt < 2 * m || nt % m || nnz < 1 || nnz > MGRIT_MAX_PSI_TAPS || nnz > nx / 2 ||
      !offsets || !coeffs || !workspace_dev || max_iter < 0)
    return MGRIT_EINVAL;
  for (int a = 1; a < nnz; ++a)
    if (offsets[a] != offsets[0] + a) return MGRIT_EINVAL;   // contiguous patterns (R8, P:786 hull)
  if (workspace_bytes < mgrit_psi_fit_nl_workspace_bytes(nx)) return MGRIT_ENOMEM;
  cudaStream_t st = (cudaStream_t)stream_;
  int s = 0, zlo = 0, zn = 0;
  double z[8], A[36], b[6];
  if (mgrit_scheme_coefficients(order, tableau, cfl, &s, &zlo, &zn, z, A, b)) return MGRIT_EINVAL;
  if (tableau >= MGRIT_TAB_SDIRK1) return MGRIT_EUNSUPPORTED;   // explicit schemes only
  const int nch = (nx + kChunk - 1) / kChunk, nu = nnz, o0 = offsets[0];
  const int np = nu * (nu + 1) / 2, nent = np + nu + 1;
  double *w0 = (double *)workspace_dev;
  double *lr = w0, *li = lr + nx, *tr = li + nx, *ti = tr + nx, *ww = ti + nx;
  double *mur = ww + nx, *mui = mur + nx, *rr = mui + nx, *ri = rr + nx, *Pr = ri + nx, *Pi = Pr + nx,
         *Qq = Pi + nx;
  const size_t ne = (size_t)MAX_PSI * (MAX_PSI + 1) / 2 + MAX_PSI + 1;
  double *phi = Qq + nx, *plo = phi + ne * nch, *psi_d = plo + ne * nch, *trial_d = psi_d + MAX_PSI,
         *res = trial_d + MAX_PSI;
  FitSym sym;
  std::memset(&sym, 0, sizeof(sym));
  sym.nx = nx;
  sym.m = m;
  sym.s = s;
  sym.zlo = zlo;
  sym.zn = zn;
  for (int j = 0; j < zn; ++j) sym.z[j] = z[j];
  for (int i = 0; i < s; ++i) {
    sym.b[i] = b[i];
    for (int j = 0; j < s; ++j) sym.A[i][j] = A[i * 6 + j];
  }
  fit_symbol_kernel<<<(nx + 255) / 256, 256, 0, st>>>(sym, lr, li, tr, ti, ww);
  if (cudaGetLastError() != cudaSuccess) return MGRIT_ECUDA;
  const int nterms = nt / m - 1;
  const size_t smem = sizeof(double) * 2 * (MAX_PSI * (MAX_PSI + 1) / 2 + MAX_PSI);
  std::vector<double> psi(coeffs, coeffs + nu), hout(nu + 3);
#define NL_CK(x) do { if ((x) != cudaSuccess) return MGRIT_ECUDA; } while (0)
  // modes and sums at `p` (device array); f_only: just sum |r|^2
  auto eval = [&](const double *p, int f_only) -> cudaError_t {
    nl_mode_kernel<<<(nx + 127) / 128, 128, 0, st>>>(nx, nu, o0, m, nterms, p, lr, li, tr, ti, mur, mui,
                                                   rr, ri, Pr, Pi, Qq);
    dim3 grid(nch, (nent + 127) / 128);
    nl_sums_kernel<<<grid, 128, 0, st>>>(nx, nu, o0, mur, mui, rr, ri, Pr, Pi, Qq, phi, plo, nch, f_only);
    return cudaGetLastError();
  };
  auto sum_f = [&](double &F) -> cudaError_t {
    nl_step_kernel<<<1, 32, smem, st>>>(nu, psi_d, 0.0, phi, plo, nch, 1, res);
    cudaError_t e = cudaMemcpyAsync(hout.data(), res, (nu + 3) * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    F = hout[nu + 2] / nx;
    return e;
  };
  NL_CK(cudaMemcpyAsync(psi_d, psi.data(), nu * sizeof(double), cudaMemcpyHostToDevice, st));
  NL_CK(eval(psi_d, 0));
  double F = 0.0;
  NL_CK(sum_f(F));
  if (history_out) history_out[0] = F;
  double lmb = 0.01;
  int it = 0;
  bool done = false;
  while (it < max_iter && !done) {
    // G, h, F are those of psi_d (formed by the last full eval)
    while (it < max_iter) {
      ++it;
      nl_step_kernel<<<1, 32, smem, st>>>(nu, psi_d, lmb, phi, plo, nch, 0, res);
      NL_CK(cudaGetLastError());
      NL_CK(cudaMemcpyAsync(hout.data(), res, (nu + 3) * sizeof(double), cudaMemcpyDeviceToHost, st));
      NL_CK(cudaStreamSynchronize(st));
      const double nd = hout[nu], npsi = hout[nu + 1];
      std::vector<double> trial(hout.begin(), hout.begin() + nu);
      // the sums of psi_d are still needed if the trial is rejected: evaluate the trial's
      // F into the upper half of the partial arrays' F entry only (f_only touches entry F)
      NL_CK(cudaMemcpyAsync(trial_d, trial.data(), nu * sizeof(double), cudaMemcpyHostToDevice, st));
      NL_CK(eval(trial_d, 1));
      double Fn = 0.0;
      NL_CK(sum_f(Fn));
      if (Fn < F) {
        const bool small = (F - Fn) <= 1e-6 * F || nd <= 1e-6 * (1.0 + npsi);
        psi = trial;
        NL_CK(cudaMemcpyAsync(psi_d, trial_d, nu * sizeof(double), cudaMemcpyDeviceToDevice, st));
        F = Fn;
        lmb /= 10.0;
        if (history_out) history_out[it] = F;
        done = small;
        if (!done && it < max_iter) NL_CK(eval(psi_d, 0));   // G, h at the accepted point
        break;
      }
      lmb *= 10.0;
      if (history_out) history_out[it] = Fn;
      // rejected: the mode arrays hold the trial's values, but G and h (partials) are intact;
      // only the F entry of the partials was overwritten, and F is kept on the host
    }
  }
#undef NL_CK
  for (int a = 0; a < nu; ++a) coeffs[a] = psi[a];
  if (iters_out) *iters_out = it;
  if (objective_out) *objective_out = F;
  return MGRIT_OK;
}

}  // extern "C"
