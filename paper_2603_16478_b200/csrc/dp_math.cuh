// Per-element and per-contact FP64 device math of the implicit step.
//
// Restates, for one element / one contact per thread, the reference
// functions cited inline (paths under /root/reference/pkg/src/diffproj).
// No tensor cores: everything here is scalar FP64 on the CUDA cores.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace dp {

// element status codes (host maps them to the reference's exceptions)
enum : int { ST_OK = 0, ST_NONFINITE = 1, ST_INVERTED = 2, ST_NH_STALL = 4, ST_PENETRATION = 8 };

constexpr double kInvSqrt2 = 0.70710678118654752440;

// ---------------------------------------------------------------------------
// 3x3 helpers (row-major m[r][c])

__device__ __forceinline__ double det3(const double a[3][3]) {
  return a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) -
         a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
         a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
}

// Solve J x = b (3x3 or 2x2) by Gaussian elimination with partial pivoting,
// the algorithm of LAPACK dgesv that np.linalg.solve calls (elasticity.py:212).
template <int D>
__device__ __forceinline__ void solve_pp(double J[D][D], double b[D], double x[D]) {
#pragma unroll
  for (int k = 0; k < D; ++k) {
    int p = k;
    double best = fabs(J[k][k]);
#pragma unroll
    for (int r = k + 1; r < D; ++r) {
      double v = fabs(J[r][k]);
      if (v > best) { best = v; p = r; }
    }
    // row swap with compile-time indices (keeps J, b in registers)
#pragma unroll
    for (int r = k + 1; r < D; ++r) {
      if (p == r) {
#pragma unroll
        for (int c = 0; c < D; ++c) { double t = J[k][c]; J[k][c] = J[r][c]; J[r][c] = t; }
        double t = b[k]; b[k] = b[r]; b[r] = t;
      }
    }
#pragma unroll
    for (int r = k + 1; r < D; ++r) {
      double f = J[r][k] / J[k][k];
#pragma unroll
      for (int c = k; c < D; ++c) J[r][c] -= f * J[k][c];
      b[r] -= f * b[k];
    }
  }
#pragma unroll
  for (int k = D - 1; k >= 0; --k) {
    double s = b[k];
#pragma unroll
    for (int c = k + 1; c < D; ++c) s -= J[k][c] * x[c];
    x[k] = s / J[k][k];
  }
}

// ---------------------------------------------------------------------------
// SVD with the reference conventions (svd_polar, elasticity.py:137-165):
// sigma descending, det U = det V = +1 for 3x3, det V = +1 for thin 3x2.
// One-sided (Hestenes) Jacobi on the columns of F: high relative accuracy,
// no F^T F squaring.  F is 3 x D, U is 3 x D, V is D x D.

template <int D>
__device__ __forceinline__ void jacobi_rotate_cols(double A[3][D], double V[D][D], int p, int q) {
  double al = A[0][p] * A[0][p] + A[1][p] * A[1][p] + A[2][p] * A[2][p];
  double be = A[0][q] * A[0][q] + A[1][q] * A[1][q] + A[2][q] * A[2][q];
  double ga = A[0][p] * A[0][q] + A[1][p] * A[1][q] + A[2][p] * A[2][q];
  if (fabs(ga) <= 1e-17 * sqrt(al * be) || ga == 0.0) return;
  double zeta = (be - al) / (2.0 * ga);
  double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  double c = 1.0 / sqrt(1.0 + t * t);
  double s = c * t;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    double ap = A[r][p], aq = A[r][q];
    A[r][p] = c * ap - s * aq;
    A[r][q] = s * ap + c * aq;
  }
#pragma unroll
  for (int r = 0; r < D; ++r) {
    double vp = V[r][p], vq = V[r][q];
    V[r][p] = c * vp - s * vq;
    V[r][q] = s * vp + c * vq;
  }
}

template <int D>
__device__ __forceinline__ void swap_cols(double A[3][D], double V[D][D], double s[D], int p, int q) {
#pragma unroll
  for (int r = 0; r < 3; ++r) { double t = A[r][p]; A[r][p] = A[r][q]; A[r][q] = t; }
#pragma unroll
  for (int r = 0; r < D; ++r) { double t = V[r][p]; V[r][p] = V[r][q]; V[r][q] = t; }
  double t = s[p]; s[p] = s[q]; s[q] = t;
}

// returns status (ST_OK / ST_NONFINITE / ST_INVERTED)
__device__ __forceinline__ int svd3(const double F[3][3], double U[3][3], double sig[3], double V[3][3]) {
  bool finite = true;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) finite = finite && isfinite(F[r][c]);
  if (!finite) return ST_NONFINITE;
  if (!(det3(F) > 0.0)) return ST_INVERTED;      // elasticity.py:148-149
  double A[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) { A[r][c] = F[r][c]; V[r][c] = (r == c) ? 1.0 : 0.0; }
  for (int sweep = 0; sweep < 10; ++sweep) {
    jacobi_rotate_cols<3>(A, V, 0, 1);
    jacobi_rotate_cols<3>(A, V, 0, 2);
    jacobi_rotate_cols<3>(A, V, 1, 2);
    // off-diagonal measure of A^T A relative to column norms
    double n0 = A[0][0] * A[0][0] + A[1][0] * A[1][0] + A[2][0] * A[2][0];
    double n1 = A[0][1] * A[0][1] + A[1][1] * A[1][1] + A[2][1] * A[2][1];
    double n2 = A[0][2] * A[0][2] + A[1][2] * A[1][2] + A[2][2] * A[2][2];
    double g01 = A[0][0] * A[0][1] + A[1][0] * A[1][1] + A[2][0] * A[2][1];
    double g02 = A[0][0] * A[0][2] + A[1][0] * A[1][2] + A[2][0] * A[2][2];
    double g12 = A[0][1] * A[0][2] + A[1][1] * A[1][2] + A[2][1] * A[2][2];
    if (g01 * g01 <= 1e-32 * n0 * n1 && g02 * g02 <= 1e-32 * n0 * n2 && g12 * g12 <= 1e-32 * n1 * n2) break;
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) sig[c] = sqrt(A[0][c] * A[0][c] + A[1][c] * A[1][c] + A[2][c] * A[2][c]);
  // sort descending; each swap flips det V
  int flips = 0;
  if (sig[0] < sig[1]) { swap_cols<3>(A, V, sig, 0, 1); ++flips; }
  if (sig[1] < sig[2]) { swap_cols<3>(A, V, sig, 1, 2); ++flips; }
  if (sig[0] < sig[1]) { swap_cols<3>(A, V, sig, 0, 1); ++flips; }
  if (flips & 1) {
#pragma unroll
    for (int r = 0; r < 3; ++r) { V[r][2] = -V[r][2]; A[r][2] = -A[r][2]; }
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    double inv = 1.0 / sig[c];
#pragma unroll
    for (int r = 0; r < 3; ++r) U[r][c] = A[r][c] * inv;
  }
  // smallest-singular-value column from the cross product: exact det U = +1
  U[0][2] = U[1][0] * U[2][1] - U[2][0] * U[1][1];
  U[1][2] = U[2][0] * U[0][1] - U[0][0] * U[2][1];
  U[2][2] = U[0][0] * U[1][1] - U[1][0] * U[0][1];
  return ST_OK;
}

// thin SVD of a 3x2 F (elasticity.py:156-164): U 3x2, V 2x2 with det V > 0
__device__ __forceinline__ int svd32(const double F[3][2], double U[3][2], double sig[2], double V[2][2]) {
  bool finite = true;
#pragma unroll
  for (int r = 0; r < 3; ++r) finite = finite && isfinite(F[r][0]) && isfinite(F[r][1]);
  if (!finite) return ST_NONFINITE;
  double A[3][2];
#pragma unroll
  for (int r = 0; r < 3; ++r) { A[r][0] = F[r][0]; A[r][1] = F[r][1]; }
  V[0][0] = 1.0; V[0][1] = 0.0; V[1][0] = 0.0; V[1][1] = 1.0;
  for (int sweep = 0; sweep < 4; ++sweep) jacobi_rotate_cols<2>(A, V, 0, 1);
  sig[0] = sqrt(A[0][0] * A[0][0] + A[1][0] * A[1][0] + A[2][0] * A[2][0]);
  sig[1] = sqrt(A[0][1] * A[0][1] + A[1][1] * A[1][1] + A[2][1] * A[2][1]);
  if (sig[0] < sig[1]) swap_cols<2>(A, V, sig, 0, 1);
  if (!(sig[1] > 0.0)) return ST_INVERTED;        // rank-deficient surface element
  if (V[0][0] * V[1][1] - V[0][1] * V[1][0] < 0.0) {
    V[0][1] = -V[0][1]; V[1][1] = -V[1][1];
    A[0][1] = -A[0][1]; A[1][1] = -A[1][1]; A[2][1] = -A[2][1];
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    double inv = 1.0 / sig[c];
#pragma unroll
    for (int r = 0; r < 3; ++r) U[r][c] = A[r][c] * inv;
  }
  return ST_OK;
}

// ---------------------------------------------------------------------------
// Neo-Hookean projection: damped Newton on
//   g(theta) = 2 mu (theta - sigma) + mu (theta - 1/theta) + lam log(J)/theta
// (project_neohookean, elasticity.py:195-242; _nh_residual :181-184;
// _nh_jacobian :187-192).  Returns ST_OK or ST_NH_STALL.

// logj_out = sum_i log(theta_i), returned for reuse: the Newton step's
// Jacobian and W need exactly this value at the accepted theta, and the
// logarithms are the largest single cost of the element kernel (ncu source
// view: 30% of its instructions before this reuse).
template <int D>
__device__ __forceinline__ void nh_g(const double th[D], const double sig[D], double mu, double lam,
                                     double g[D], double& nrm, double& logj_out) {
  double logj = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) logj += log(th[i]);
  logj_out = logj;
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    g[i] = 2.0 * mu * (th[i] - sig[i]) + mu * (th[i] - 1.0 / th[i]) + lam * logj / th[i];
    s += g[i] * g[i];
  }
  nrm = sqrt(s);
}

template <int D>
__device__ __forceinline__ int nh_project(const double sig[D], double mu, double lam, double th[D],
                                          double W[D][D]) {
  const double thr = 1e-11 * fmax(1.0, mu);
  double g[D], rn, logj_th;   // logj_th = sum log(th) at the current theta
#pragma unroll
  for (int i = 0; i < D; ++i) th[i] = sig[i];
  nh_g<D>(th, sig, mu, lam, g, rn, logj_th);
  bool conv = false;
  for (int it = 0; it < 50; ++it) {
    if (rn <= thr) { conv = true; break; }
    const double logj = logj_th;
    double J[D][D], b[D], step[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
#pragma unroll
      for (int j = 0; j < D; ++j) J[i][j] = lam * (1.0 / th[i]) * (1.0 / th[j]);
      J[i][i] += 3.0 * mu + (mu - lam * logj) / (th[i] * th[i]);
      b[i] = -g[i];
    }
    solve_pp<D>(J, b, step);
    double t = 1.0;
    bool acc = false;
    for (int ls = 0; ls < 40; ++ls) {
      double cand[D];
      bool pos = true;
#pragma unroll
      for (int i = 0; i < D; ++i) { cand[i] = th[i] + t * step[i]; pos = pos && (cand[i] > 0.0); }
      if (pos) {
        double gc[D], rc, lc;
        nh_g<D>(cand, sig, mu, lam, gc, rc, lc);
        if (rc < rn) {
#pragma unroll
          for (int i = 0; i < D; ++i) { th[i] = cand[i]; g[i] = gc[i]; }
          rn = rc;
          logj_th = lc;
          acc = true;
          break;
        }
      }
      t *= 0.5;
    }
    if (!acc) return ST_NH_STALL;
  }
  if (!conv && !(rn <= thr)) return ST_NH_STALL;
  // W = dtheta/dsigma, Sherman-Morrison form (elasticity.py:231-237)
  const double logj = logj_th;
  double dinv[D], du[D], udu = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    dinv[i] = 1.0 / (3.0 * mu + (mu - lam * logj) / (th[i] * th[i]));
    double u = 1.0 / th[i];
    du[i] = dinv[i] * u;
    udu += u * du[i];
  }
  double denom = 1.0 + lam * udu;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j)
      W[i][j] = 2.0 * mu * (((i == j) ? dinv[i] : 0.0) - du[i] * du[j] * lam / denom);
  return ST_OK;
}

// energy density zeta(theta) (elasticity.py:175-178)
template <int D>
__device__ __forceinline__ double nh_energy(const double th[D], double mu, double lam) {
  double i1 = 0.0, logj = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) { i1 += th[i] * th[i]; logj += log(th[i]); }
  return 0.5 * mu * (i1 - 2.0 * logj - D) + 0.5 * lam * logj * logj;
}

// dtheta/dmu and dtheta/dlambda (dP_dlame, elasticity.py:309-324)
template <int D>
__device__ __forceinline__ void nh_dtheta_dlame(const double th[D], const double sig[D], double mu, double lam,
                                                double dmu[D], double dlam[D]) {
  double logj = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) logj += log(th[i]);
  double J[D][D], J2[D][D], b1[D], b2[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
#pragma unroll
    for (int j = 0; j < D; ++j) J[i][j] = lam * (1.0 / th[i]) * (1.0 / th[j]);
    J[i][i] += 3.0 * mu + (mu - lam * logj) / (th[i] * th[i]);
    b1[i] = -(3.0 * th[i] - 2.0 * sig[i] - 1.0 / th[i]);
    b2[i] = -(logj / th[i]);
  }
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) J2[i][j] = J[i][j];
  solve_pp<D>(J, b1, dmu);
  solve_pp<D>(J2, b2, dlam);
}

// ---------------------------------------------------------------------------
// Off-diagonal coefficients of dP/dF in the singular basis with the
// within-block-commutation limits (proj_jacobian, elasticity.py:262-300).
// For pair (i,j) returns m = M_ij and n = N_ij (both symmetric in i,j).
__device__ __forceinline__ void mn_pair(double si, double sj, double ti, double tj, double Wii, double Wjj,
                                        double Wij, double tau, double& m, double& n) {
  if (fabs(si - sj) > tau) {
    double den = si * si - sj * sj;
    m = (si * ti - sj * tj) / den;
    n = (sj * ti - si * tj) / den;
  } else {
    double wd = 0.5 * (Wii + Wjj);
    double ts = (ti + tj) / (si + sj);
    m = 0.5 * (wd - Wij + ts);
    n = 0.5 * (wd - Wij - ts);
  }
}

// ---------------------------------------------------------------------------
// Contacts: closed-form condensation and derivative block
// (solve_multipliers contact.py:139-165, build_R :186-209,
//  contact_block :212-248, contact_residual :168-183).

struct ContactLocal {
  double lam[3], delta[3], s;
  int capped;
  double Kc[3][3];   // local frame, row-major
  double kmu[3];
};

__device__ __forceinline__ double fb_smooth(double x, double y, double eps2) {
  return x + y - sqrt(x * x + y * y + eps2);
}

// dn, df already computed by the caller (with the reference arithmetic).
// Returns ST_OK or ST_PENETRATION.
__device__ __forceinline__ int contact_local(double dn, double df0, double df1, double mu, double eps2,
                                             ContactLocal& c) {
  const double tau = 1e-9;   // TAU_FALLBACK, contact.py:25
  const double eps_sq = 0.5 * eps2;
  c.delta[0] = dn; c.delta[1] = df0; c.delta[2] = df1;
  if (!(dn > 0.0)) return ST_PENETRATION;
  double lam_n = eps_sq / dn;
  double nf = sqrt(df0 * df0 + df1 * df1);
  double nfg = fmax(nf, tau);
  double s = mu * lam_n - eps_sq / nfg;
  int capped = 0;
  if (s < -mu * lam_n) { s = -mu * lam_n; capped = 1; }
  double h0 = df0 / nfg, h1 = df1 / nfg;
  double lf0 = -s * h0, lf1 = -s * h1;
  c.lam[0] = lam_n; c.lam[1] = lf0; c.lam[2] = lf1;
  c.s = s; c.capped = capped;
  // rotation R (contact.py:186-209)
  double R[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  double nl = sqrt(lf0 * lf0 + lf1 * lf1);
  if (nf > tau) {
    double a = df0 / nf, b = df1 / nf;
    R[1][1] = a; R[1][2] = b; R[2][1] = -b; R[2][2] = a;
  } else if (nl > tau) {
    double a = lf0 / nl, b = lf1 / nl;
    R[1][1] = -a; R[1][2] = -b; R[2][1] = b; R[2][2] = -a;
  }
  double sign = capped ? -1.0 : 1.0;
  double B[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double kv1;
  B[0][0] = lam_n / dn;
  if (nf >= tau) {
    double a22 = capped ? 0.0 : (mu * lam_n - s) / nf;
    B[1][0] = -sign * mu * lam_n / dn;
    B[1][1] = a22;
    B[2][2] = s / nf;
    kv1 = lam_n;
  } else {
    double ratio = nf / tau;
    B[1][0] = -sign * mu * lam_n / dn * ratio;
    B[1][1] = s / tau;
    B[2][2] = s / tau;
    kv1 = lam_n * ratio;
  }
  // Kc = R^T B R
  double BR[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) BR[i][j] = B[i][0] * R[0][j] + B[i][1] * R[1][j] + B[i][2] * R[2][j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c.Kc[i][j] = R[0][i] * BR[0][j] + R[1][i] * BR[1][j] + R[2][i] * BR[2][j];
  // k_mu = sign * R^T (0, kv1, 0)
#pragma unroll
  for (int i = 0; i < 3; ++i) c.kmu[i] = sign * R[1][i] * kv1;
  return ST_OK;
}

__device__ __forceinline__ void contact_residual_rows(const ContactLocal& c, double mu, double eps2, double out[3]) {
  double nf = sqrt(c.delta[1] * c.delta[1] + c.delta[2] * c.delta[2]);
  double nl = sqrt(c.lam[1] * c.lam[1] + c.lam[2] * c.lam[2]);
  out[0] = fb_smooth(c.delta[0], c.lam[0], eps2);
  out[1] = fb_smooth(nf, mu * c.lam[0] - nl, eps2);
  double a0 = nl * c.delta[1] + nf * c.lam[1];
  double a1 = nl * c.delta[2] + nf * c.lam[2];
  out[2] = sqrt(a0 * a0 + a1 * a1);
}

}  // namespace dp
