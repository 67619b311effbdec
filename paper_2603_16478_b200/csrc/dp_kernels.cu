// Element, assembly, SpMV, Krylov and backprop kernels of libdiffproj_b200.
//
// Data layout:
//  * vectors: flat FP64, xyz-interleaved per vertex (the reference layout);
//  * element inputs: SoA (Dm^-1 as [9][E], w/mu/lam/model as [E]) and the
//    four vertex ids as one int4 per element (one 16-byte load);
//  * element outputs: residual contributions fe[E][NV][3] and the NP
//    unique 3x3 blocks of the symmetric element Hessian, written into a
//    block stream H ordered by the assembly's slot runs (store_hpair);
//  * system matrix: SELL-32 block-sparse (3x3 FP64 blocks), slices of 32
//    block rows, block k of lane l at slot base_s + 32k + l; block values
//    component-major inside a slice so each warp load is 32 consecutive
//    doubles (256 B).
// Assembly is a deterministic stream (no atomics): every canonical SELL slot
// (row <= col) owns a contiguous run of H in element order, and slot (j, i)
// reads the run of (i, j) transposed.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <algorithm>
#include <stdio.h>
#include <stdlib.h>

#include "dp_common.cuh"
#include "dp_internal.h"
#include "dp_math.cuh"

#ifndef DP_ELEM_MINB
#define DP_ELEM_MINB 4
#endif
#ifndef DP_JAC_SMEM
#define DP_JAC_SMEM 1
#endif

namespace dp {

// PCG SpMV slots through a TMA bulk-copy ring (DP_SPMV_BULK=1; measured: in
// situ 23.9 -> 23.1 us per launch, the step rate within noise: off)
static const int g_spmv_bulk = getenv("DP_SPMV_BULK") ? atoi(getenv("DP_SPMV_BULK")) : 0;

// ---------------------------------------------------------------------------
// element kernel

// Gt_a J G_b in the singular basis: U~ C U~^T with C built from W, the
// (M, N) pair coefficients and (triangles) the out-of-plane term.
template <int D>
struct ElemJac {
  double U3[3][3];      // [U | u3] for triangles, U for tets
  double W[D][D];
  double m[3], n[3];    // pairs (0,1), (0,2), (1,2) (tets) / (0,1) (tris)
  double oop[2];        // theta/sigma (triangles)
};

template <int D>
__device__ __forceinline__ void jac_block(const ElemJac<D>& J, const double aa[D], const double ab[D], double out[3][3]) {
  double C[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
  for (int k = 0; k < D; ++k)
#pragma unroll
    for (int l = 0; l < D; ++l) C[k][l] = aa[k] * J.W[k][l] * ab[l];
  if (D == 3) {
    const int pk[3] = {0, 0, 1}, pl[3] = {1, 2, 2};
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const int k = pk[p], l = pl[p];
      C[l][l] += J.m[p] * aa[k] * ab[k];
      C[k][k] += J.m[p] * aa[l] * ab[l];
      C[l][k] += J.n[p] * aa[k] * ab[l];
      C[k][l] += J.n[p] * aa[l] * ab[k];
    }
  } else {
    C[1][1] += J.m[0] * aa[0] * ab[0];
    C[0][0] += J.m[0] * aa[1] * ab[1];
    C[1][0] += J.n[0] * aa[0] * ab[1];
    C[0][1] += J.n[0] * aa[1] * ab[0];
    C[2][2] = J.oop[0] * aa[0] * ab[0] + J.oop[1] * aa[1] * ab[1];
  }
  // out = U C U^T
  double T[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int l = 0; l < 3; ++l) T[i][l] = J.U3[i][0] * C[0][l] + J.U3[i][1] * C[1][l] + J.U3[i][2] * C[2][l];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) out[i][j] = T[i][0] * J.U3[j][0] + T[i][1] * J.U3[j][1] + T[i][2] * J.U3[j][2];
}

// Full per-element projection: F -> SVD -> theta, W -> P (+ jacobian data).
// F is 3 x D.  Returns status.
template <int D>
__device__ __forceinline__ int project_full(const double F[3][D], int model, double mu, double lam, double tau_rel,
                                            double U[3][D], double sig[D], double V[D][D], double th[D],
                                            double W[D][D]) {
  int st;
  if (D == 3) st = svd3((const double(*)[3])F, (double(*)[3])U, sig, (double(*)[3])V);
  else st = svd32((const double(*)[2])F, (double(*)[2])U, sig, (double(*)[2])V);
  if (st) return st;
  if (model == DP_MODEL_NEOHOOKEAN) {
    st = nh_project<D>(sig, mu, lam, th, W);
    if (st) return st;
  } else {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      th[i] = 1.0;
#pragma unroll
      for (int j = 0; j < D; ++j) W[i][j] = 0.0;
    }
  }
  return ST_OK;
}

template <int D>
__device__ __forceinline__ void make_jac(const double U[3][D], const double sig[D], const double th[D],
                                         const double W[D][D], double tau_rel, ElemJac<D>& J) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < D; ++k) J.U3[i][k] = U[i][k];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) J.W[i][j] = W[i][j];
  const double tau = tau_rel * sig[0];
  if (D == 3) {
    mn_pair(sig[0], sig[1], th[0], th[1], W[0][0], W[1][1], W[0][1], tau, J.m[0], J.n[0]);
    mn_pair(sig[0], sig[2], th[0], th[2], W[0][0], W[2][2], W[0][2], tau, J.m[1], J.n[1]);
    mn_pair(sig[1], sig[2], th[1], th[2], W[1][1], W[2][2], W[1][2], tau, J.m[2], J.n[2]);
  } else {
    mn_pair(sig[0], sig[1], th[0], th[1], W[0][0], W[1][1], W[0][1], tau, J.m[0], J.n[0]);
    J.m[1] = J.m[2] = J.n[1] = J.n[2] = 0.0;
    // u3 = u1 x u2 completes the basis (elasticity.py:302-305)
    J.U3[0][2] = U[1][0] * U[2][1] - U[2][0] * U[1][1];
    J.U3[1][2] = U[2][0] * U[0][1] - U[0][0] * U[2][1];
    J.U3[2][2] = U[0][0] * U[1][1] - U[1][0] * U[0][1];
    J.oop[0] = th[0] / sig[0];
    J.oop[1] = th[1] / sig[1];
  }
}

#ifndef ASM_CHUNK
#define ASM_CHUNK 4
#endif

// b += block, or its transpose
__device__ __forceinline__ void acc_block(double b[9], const double src[9], bool transposed) {
  if (!transposed) {
#pragma unroll
    for (int c = 0; c < 9; ++c) b[c] += src[c];
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) b[i * 3 + j] += src[j * 3 + i];
  }
}

// 256-bit global accesses (sm_100): one full 32-byte sector per access
__device__ __forceinline__ void st256(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
__device__ __forceinline__ void ld256(const double* p, double o[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
}
// the same without an L1 allocation: streams whose every 32-byte entry is
// read by one lane exactly once (the residual gather's element-force runs,
// the assembly's block-stream runs); measured k_residual 36.2 -> 33.8 us
#ifndef DP_RES_NA
#define DP_RES_NA 1
#endif
__device__ __forceinline__ void ld256_na(const double* p, double o[4]) {
#if DP_RES_NA
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
               : "l"(p));
#else
  ld256(p, o);
#endif
}
__device__ __forceinline__ void ld256f_na(const float* p, float o[8]) {
#if DP_RES_NA
  asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]), "=f"(o[4]), "=f"(o[5]), "=f"(o[6]), "=f"(o[7])
               : "l"(p));
#else
  ld256f(p, o);
#endif
}

// h^2 w [(beta_a.beta_b) I - blk] for the element's local pair p = (a, b),
// a <= b, written once into the slot-ordered block stream, at its position t
// in the run of the canonical slot (min(i, j), max(i, j)) of its vertices
// i = vid[a], j = vid[b] (epos, built at setup in run order; ~t: i > j, the
// block is stored transposed).  A block is split into its first 8 doubles,
// Hs[t] (64 B: two full-sector 256-bit stores), and its last, Ht[t] (the
// (2,2) entry, transpose-invariant).  The assembly reads each slot's run as
// one contiguous stream, the (j, i) slots the (i, j) run transposed.
template <int NV>
__device__ __forceinline__ void store_hpair(double* __restrict__ Hs, double* __restrict__ Ht,
                                            const int* __restrict__ epos, int e, int p, double hw, double bb,
                                            const double blk[3][3]) {
  constexpr int NP = NV * (NV + 1) / 2;
  double v[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) v[i * 3 + j] = hw * (((i == j) ? bb : 0.0) - blk[i][j]);
  const int tc = __ldg(epos + (size_t)e * NP + p);
  const int t = tc >= 0 ? tc : ~tc;
  double* o = Hs + (size_t)t * kHS;
  if (tc >= 0) {
    st256(o, v[0], v[1], v[2], v[3]);
    st256(o + 4, v[4], v[5], v[6], v[7]);
  } else {
    st256(o, v[0], v[3], v[6], v[1]);
    st256(o + 4, v[4], v[7], v[2], v[5]);
  }
  Ht[t] = v[8];
}

// FP32 block stream (frictionless forward steps, EV_H32): the same block,
// rounded to FP32, 8 floats in one 256-bit store + the tail float, in the
// first half of the FP64 stream's storage (half the stream traffic of the
// element kernel and the assembly; the forward solves run on the FP32
// operator anyway)
template <int NV>
__device__ __forceinline__ void store_hpair32(double* __restrict__ Hs, double* __restrict__ Ht,
                                              const int* __restrict__ epos, int e, int p, double hw, double bb,
                                              const double blk[3][3]) {
  constexpr int NP = NV * (NV + 1) / 2;
  float v[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) v[i * 3 + j] = (float)(hw * (((i == j) ? bb : 0.0) - blk[i][j]));
  const int tc = __ldg(epos + (size_t)e * NP + p);
  const int t = tc >= 0 ? tc : ~tc;
  float* o = reinterpret_cast<float*>(Hs) + (size_t)t * 8;
  if (tc >= 0) {
    const float f8[8] = {v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]};
    st256f(o, f8);
  } else {
    const float f8[8] = {v[0], v[3], v[6], v[1], v[4], v[7], v[2], v[5]};
    st256f(o, f8);
  }
  reinterpret_cast<float*>(Ht)[t] = v[8];
}

// One thread per element.  NV = vertices per element (4 tet, 3 tri).  The
// mode is a template parameter: the residual-only instantiation (line-search
// trials) does not carry the Jacobian path's registers (168 -> fewer), so it
// runs at a higher occupancy; the Jacobian instantiations are register-capped
// at 128 (4 CTAs of 128 per SM: measured faster than 3 CTAs without spills).
template <int NV, int MODE>
__global__ void __launch_bounds__(128, DP_ELEM_MINB)
    k_elements(const int4* __restrict__ ev, const double* __restrict__ Bm, const double* __restrict__ w,
               const double* __restrict__ mu, const double* __restrict__ lam, const int* __restrict__ model, int E,
               const double* __restrict__ q, double h2, double tau_rel, double* __restrict__ fe,
               const int* __restrict__ fe_pos,
               double* __restrict__ H, double* __restrict__ Ht, const int* __restrict__ epos,
               double* __restrict__ Pst,
               int* __restrict__ status, const int* __restrict__ skip, const int* __restrict__ list, const int* __restrict__ list_n) {
  constexpr int mode = MODE;
  if (skip && *(volatile const int*)skip) return;   // line-search trial needing no evaluation
  constexpr int D = NV - 1;
  constexpr int NP = NV * (NV + 1) / 2;
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (mode & EV_LIST) {
    // an element subset (line-search pre-check): same arithmetic as the full pass
    if (e >= min(*list_n, kWatchElemMax)) return;
    e = list[e];
    if (e < 0) return;
  }
  if (e >= E) return;
  const int4 vv = ev[e];
  const int vid[4] = {vv.x, vv.y, vv.z, vv.w};
  double beta[NV][D];
#pragma unroll
  for (int k = 1; k < NV; ++k)
#pragma unroll
    for (int c = 0; c < D; ++c) beta[k][c] = __ldg(Bm + (size_t)((k - 1) * D + c) * E + e);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    double s = 0.0;
#pragma unroll
    for (int k = 1; k < NV; ++k) s += beta[k][c];
    beta[0][c] = -s;
  }
  double x[NV][3];
#pragma unroll
  for (int a = 0; a < NV; ++a)
#pragma unroll
    for (int i = 0; i < 3; ++i) x[a][i] = q[3 * (size_t)vid[a] + i];
  double F[3][D];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < NV; ++a) s += x[a][i] * beta[a][c];
      F[i][c] = s;
    }
  const double hw = h2 * w[e];
  const int mdl = model[e];
  const double emu = mu[e], elam = lam[e];

  double U[3][D], sig[D], V[D][D], th[D], W[D][D];
  int st = ST_OK;
  if (mode & EV_AMAT) {
#pragma unroll
    for (int i = 0; i < D; ++i) { sig[i] = 1.0; th[i] = 1.0; }
  } else {
    st = project_full<D>(F, mdl, emu, elam, tau_rel, U, sig, V, th, W);
  }
  if (st) {
    atomicOr(status, st);
#pragma unroll
    for (int a = 0; a < NV; ++a) st256(fe + (size_t)__ldg(fe_pos + (size_t)e * NV + a) * kFeS, 0.0, 0.0, 0.0, 0.0);
    return;
  }
  if (!(mode & EV_AMAT)) {
    // P = U diag(theta) V^T ; fe_a = h^2 w (F - P) beta_a  (internal_force_and_rhs, elasticity.py:386-396)
    double P[3][D];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s += U[i][k] * th[k] * V[c][k];
        P[i][c] = s;
      }
    // written at the (e, a) entry's position in vertex a's incidence run
    // (fe_pos), one full-sector 256-bit store: k_residual streams the runs
#pragma unroll
    for (int a = 0; a < NV; ++a) {
      double f3[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) s += (F[i][c] - P[i][c]) * beta[a][c];
        f3[i] = hw * s;
      }
      st256(fe + (size_t)__ldg(fe_pos + (size_t)e * NV + a) * kFeS, f3[0], f3[1], f3[2], 0.0);
    }
    if (mode & EV_STOREP) {
      double* o = Pst + (size_t)e * 27;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int c = 0; c < D; ++c) o[i * 3 + c] = P[i][c];
      double dmu[D], dlm[D];
      if (mdl == DP_MODEL_NEOHOOKEAN) {
        nh_dtheta_dlame<D>(th, sig, emu, elam, dmu, dlm);
      } else {
#pragma unroll
        for (int k = 0; k < D; ++k) dmu[k] = dlm[k] = 0.0;
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int c = 0; c < D; ++c) {
          double s1 = 0.0, s2 = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) { s1 += U[i][k] * dmu[k] * V[c][k]; s2 += U[i][k] * dlm[k] * V[c][k]; }
          o[9 + i * 3 + c] = s1;
          o[18 + i * 3 + c] = s2;
        }
    }
  }
  if ((mode & EV_JAC) && !(mode & EV_AMAT) && DP_JAC_SMEM) {
    // Block phase through shared memory: the projection's registers are dead
    // here, and the Jacobian data (J, alpha) is re-read from this thread's
    // shared-memory row one block at a time instead of being held live
    // across the ten unrolled blocks (which spilled at the 128-register cap).
    // Same arithmetic, term by term, as the register path below.
    constexpr int NOOP = (D == 2) ? 2 : 0;
    constexpr int NJ = 9 + D * D + 3 + 3 + NOOP + NV * D + NP;
    // thread-interleaved (field-major) rows: consecutive threads read
    // consecutive doubles, so the 64-bit accesses are bank-conflict free
    // (the row-per-thread layout, stride NJ = 46 doubles, measured 26M
    // shared bank conflicts per C5 launch)
    __shared__ double jsm[NJ][128];
    volatile double* js = &jsm[0][threadIdx.x];
    {
      ElemJac<D> J;
      make_jac<D>(U, sig, th, W, tau_rel, J);
      int f = 0;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) js[(f++) * 128] = J.U3[i][k];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int k = 0; k < D; ++k) js[(f++) * 128] = J.W[i][k];
#pragma unroll
      for (int i = 0; i < 3; ++i) js[(f++) * 128] = J.m[i];
#pragma unroll
      for (int i = 0; i < 3; ++i) js[(f++) * 128] = J.n[i];
      if (NOOP) {
        js[(f++) * 128] = J.oop[0];
        js[(f++) * 128] = J.oop[1];
      }
#pragma unroll
      for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int k = 0; k < D; ++k) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < D; ++c) s += V[c][k] * beta[a][c];
          js[(f++) * 128] = s;
        }
#pragma unroll
      for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int b = a; b < NV; ++b) {
          double bb = 0.0;
#pragma unroll
          for (int c = 0; c < D; ++c) bb += beta[a][c] * beta[b][c];
          js[(f++) * 128] = bb;
        }
    }
    int p = 0;
    constexpr int FA = 9 + D * D + 3 + 3 + NOOP;
    constexpr int FB = FA + NV * D;
#pragma unroll 1
    for (int a = 0; a < NV; ++a) {
#pragma unroll 1
      for (int b = a; b < NV; ++b, ++p) {
        ElemJac<D> J;
        int f = 0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k) J.U3[i][k] = js[(f++) * 128];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
          for (int k = 0; k < D; ++k) J.W[i][k] = js[(f++) * 128];
#pragma unroll
        for (int i = 0; i < 3; ++i) J.m[i] = js[(f++) * 128];
#pragma unroll
        for (int i = 0; i < 3; ++i) J.n[i] = js[(f++) * 128];
        if (NOOP) {
          J.oop[0] = js[(f++) * 128];
          J.oop[1] = js[(f++) * 128];
        } else {
          J.oop[0] = J.oop[1] = 0.0;
        }
        double aa[D], ab[D];
#pragma unroll
        for (int k = 0; k < D; ++k) { aa[k] = js[(FA + a * D + k) * 128]; ab[k] = js[(FA + b * D + k) * 128]; }
        const double bb = js[(FB + p) * 128];
        double blk[3][3];
        jac_block<D>(J, aa, ab, blk);
        if (mode & EV_H32) store_hpair32<NV>(H, Ht, epos, e, p, hw, bb, blk);
        else store_hpair<NV>(H, Ht, epos, e, p, hw, bb, blk);
      }
    }
    return;
  }
  if (mode & EV_JAC) {
    ElemJac<D> J;
    double alpha[NV][D];
    const bool amat = (mode & EV_AMAT) != 0;
    if (!amat) {
      make_jac<D>(U, sig, th, W, tau_rel, J);
#pragma unroll
      for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int k = 0; k < D; ++k) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < D; ++c) s += V[c][k] * beta[a][c];
          alpha[a][k] = s;
        }
    }
    int p = 0;
#pragma unroll
    for (int a = 0; a < NV; ++a)
#pragma unroll
      for (int b = a; b < NV; ++b, ++p) {
        double bb = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) bb += beta[a][c] * beta[b][c];
        double blk[3][3];
        if (amat) {
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) blk[i][j] = 0.0;
        } else {
          jac_block<D>(J, alpha[a], alpha[b], blk);
        }
        if (mode & EV_H32) store_hpair32<NV>(H, Ht, epos, e, p, hw, bb, blk);
        else store_hpair<NV>(H, Ht, epos, e, p, hw, bb, blk);
      }
  }
}

template <int NV>
static void launch_elements_nv(dp_scene* s, const double* q, int mode, int* status, int nb, int nt, double h2) {
#define DP_ELEM_CASE(M)                                                                                       \
  case M:                                                                                                     \
    k_elements<NV, M><<<nb, nt, 0, s->stream>>>(s->ev, s->B, s->w, s->mu, s->lam, s->model, s->E, q, h2, 1e-6, \
                                                s->fe, s->fe_pos, s->H, s->Ht, s->epos, s->Pst, status, s->eval_skip, nullptr, nullptr); \
    break;
  switch (mode) {
    DP_ELEM_CASE(0)
    DP_ELEM_CASE(EV_JAC)
    DP_ELEM_CASE(EV_JAC | EV_H32)
    DP_ELEM_CASE(EV_JAC | EV_STOREP)
    DP_ELEM_CASE(EV_JAC | EV_AMAT)
    DP_ELEM_CASE(EV_STOREP)
    default:
      break;
  }
#undef DP_ELEM_CASE
}

void launch_elements(dp_scene* s, const double* q, int mode, int* status) {
  if (s->E == 0) return;
  const int nt = 128;
  const int nb = grid_for(s->E, nt);
  const double h2 = s->h * s->h;
  const int kt = (mode & EV_JAC) ? KT_ELEM_JAC : KT_ELEM_RES;
  ktm_begin(s, kt);
  if (s->NV == 4) launch_elements_nv<4>(s, q, mode, status, nb, nt, h2);
  else launch_elements_nv<3>(s, q, mode, status, nb, nt, h2);
  ktm_end(s, kt);
  s->launches++;
}

// ---------------------------------------------------------------------------
// residual gather: r = M (q - q_hat) + sum_e fe - h^2 J_b^T lam_b - h^2 J_c^T lam_c
// (momentum_residual, forward.py:101-110), plus max|r| (forward.py:202).

constexpr int kVT = 256;

#ifndef DP_RES_GROUP
#define DP_RES_GROUP 8
#endif
constexpr int kResG = DP_RES_GROUP;   // fe loads in flight per row (measured 4 -> 8)

// one row of the momentum residual (momentum_residual, forward.py:101-110):
// M (q - q_hat) + element contributions (incidence order, 4 loads in flight)
// + bindings + contact forces; shared by the full residual and the
// line-search pre-check so both produce the same bits
__device__ __forceinline__ void residual_row(int i, const double* __restrict__ mass, const double* __restrict__ q,
                                             const double* __restrict__ q_hat, const int* __restrict__ inc_ptr,
                                             const int* __restrict__ inc, const double* __restrict__ fe,
                                             const int* __restrict__ b_ptr, const int* __restrict__ b_idx,
                                             const double* __restrict__ b_target, const double* __restrict__ b_comp,
                                             const int* __restrict__ c_count, const int* __restrict__ c_off,
                                             const double* __restrict__ c_force, int has_contacts, double h2,
                                             double& r0, double& r1, double& r2) {
    const double m = mass[i];
    r0 = m * (q[3 * i] - q_hat[3 * i]);
    r1 = m * (q[3 * i + 1] - q_hat[3 * i + 1]);
    r2 = m * (q[3 * i + 2] - q_hat[3 * i + 2]);
    // element contributions: the vertex's incidence run of the fe stream
    // (incidence order), in groups of 4 (all loads of a group in flight
    // before the in-order accumulation)
    int k = inc_ptr[i];
    const int k1 = inc_ptr[i + 1];
    for (; k + kResG <= k1; k += kResG) {
      double f[kResG][4];
#pragma unroll
      for (int g = 0; g < kResG; ++g) ld256_na(fe + (size_t)(k + g) * kFeS, f[g]);
#pragma unroll
      for (int g = 0; g < kResG; ++g) { r0 += f[g][0]; r1 += f[g][1]; r2 += f[g][2]; }
    }
    for (; k < k1; ++k) {
      double f[4];
      ld256_na(fe + (size_t)k * kFeS, f);
      r0 += f[0]; r1 += f[1]; r2 += f[2];
    }
    if (b_ptr) {
      for (int k = b_ptr[i]; k < b_ptr[i + 1]; ++k) {
        const int b = b_idx[k];
        const double c = h2 / b_comp[b];
        r0 += c * (q[3 * i] - b_target[3 * b]);
        r1 += c * (q[3 * i + 1] - b_target[3 * b + 1]);
        r2 += c * (q[3 * i + 2] - b_target[3 * b + 2]);
      }
    }
    if (has_contacts) {
      const int c0 = c_off[i], cn = c_count[i];
      for (int c = c0; c < c0 + cn; ++c) {
        r0 += c_force[3 * c]; r1 += c_force[3 * c + 1]; r2 += c_force[3 * c + 2];
      }
    }
}

__global__ void __launch_bounds__(kVT) k_residual(int V, const double* __restrict__ mass, const double* __restrict__ q,
                                                  const double* __restrict__ q_hat, const int* __restrict__ inc_ptr,
                                                  const int* __restrict__ inc, const double* __restrict__ fe,
                                                  const int* __restrict__ b_ptr, const int* __restrict__ b_idx,
                                                  const double* __restrict__ b_target, const double* __restrict__ b_comp,
                                                  const int* __restrict__ c_count, const int* __restrict__ c_off,
                                                  const double* __restrict__ c_force, int has_contacts, double h2,
                                                  double* __restrict__ r, double* partial, unsigned int* counter,
                                                  EvalScalars* esc, const int* __restrict__ skip) {
  __shared__ double sh[32];
  if (skip && *(volatile const int*)skip) return;
  const int i = blockIdx.x * kVT + threadIdx.x;
  double amax = 0.0, sq = 0.0;
  if (i < V) {
    double r0, r1, r2;
    residual_row(i, mass, q, q_hat, inc_ptr, inc, fe, b_ptr, b_idx, b_target, b_comp, c_count, c_off, c_force,
                 has_contacts, h2, r0, r1, r2);
    r[3 * i] = r0; r[3 * i + 1] = r1; r[3 * i + 2] = r2;
    amax = fmax(fabs(r0), fmax(fabs(r1), fabs(r2)));
    if (!(amax == amax)) amax = INFINITY;   // NaN propagates as +inf
    sq = r0 * r0 + r1 * r1 + r2 * r2;
  }
  double bm = block_max<kVT>(amax, sh);
  double bs = block_sum<kVT>(sq, sh);
  if (threadIdx.x == 0) { partial[2 * blockIdx.x] = bm; partial[2 * blockIdx.x + 1] = bs; }
  if (last_block(counter)) {
    __shared__ double out[2];
    double m = 0.0, t = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kVT) {
      m = fmax(m, __ldcg(partial + 2 * b));
      t += __ldcg(partial + 2 * b + 1);
    }
    m = block_max<kVT>(m, sh);
    t = block_sum<kVT>(t, sh);
    if (threadIdx.x == 0) { esc->rmax = m; esc->rnorm2 = t; *counter = 0; }
  }
}

void launch_residual(dp_scene* s, const double* q, const double* q_hat, double* r, EvalScalars* esc) {
  const int nb = grid_for(s->V, kVT);
  const int has_c = contact_sources(s) > 0;
  k_residual<<<nb, kVT, 0, s->stream>>>(s->V, s->mass, q, q_hat, s->inc_ptr, s->inc, s->fe, s->nb ? s->b_ptr : nullptr,
                                        s->b_idx, s->b_target, s->b_comp, s->c_count, s->c_off, s->c_force, has_c,
                                        s->h * s->h, r, s->red.partial, s->red.counter, esc, s->eval_skip);
  s->launches++;
}

// ---------------------------------------------------------------------------
// line-search pre-check (forward.py:214-234 accepts a trial iff max|r_try| <
// max|r| and nothing is inverted/penetrating).  Rows that were large at the
// Newton evaluation are watched; before a trial's full evaluation, the
// elements incident to them are evaluated (same k_elements code) and their
// rows summed (same residual_row); if one of them already reaches max|r|
// the full evaluation could only confirm the rejection, so it is skipped.
// Accept/reject decisions are identical to always evaluating fully; a
// watched NH stall leaves the decision to the full evaluation (which raises,
// as the reference does).

__global__ void k_watch_select(int V, int NV, const double* __restrict__ r, const int* __restrict__ inc_ptr,
                               const int* __restrict__ inc, double frac, int* __restrict__ watch_v,
                               int* __restrict__ watch_e, EvalScalars* esc) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const double a = fmax(fabs(r[3 * v]), fmax(fabs(r[3 * v + 1]), fabs(r[3 * v + 2])));
  if (!(a >= frac * esc->rmax)) return;
  const int k0 = inc_ptr[v], deg = inc_ptr[v + 1] - k0;
  const int slot = atomicAdd(&esc->n_watch, 1);
  if (slot >= kWatchMax) return;
  // the row is checked only if all its elements fit in the element list
  const int base = atomicAdd(&esc->n_watch_elem, deg);
  if (base + deg > kWatchElemMax) {
    watch_v[slot] = -1;
    for (int k = base; k < kWatchElemMax; ++k) watch_e[k] = -1;
    return;
  }
  for (int k = 0; k < deg; ++k) watch_e[base + k] = inc[k0 + k] / NV;
  watch_v[slot] = v;
}

__global__ void k_watch_check(const int* __restrict__ watch_v, const double* __restrict__ mass,
                              const double* __restrict__ q, const double* __restrict__ q_hat,
                              const int* __restrict__ inc_ptr, const int* __restrict__ inc,
                              const double* __restrict__ fe, const int* __restrict__ b_ptr,
                              const int* __restrict__ b_idx, const double* __restrict__ b_target,
                              const double* __restrict__ b_comp, const int* __restrict__ c_count,
                              const int* __restrict__ c_off, const double* __restrict__ c_force, int has_contacts,
                              double h2, double rmax_prev, EvalScalars* esc) {
  if (*(volatile const int*)&esc->skip) return;
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= min(esc->n_watch, kWatchMax)) return;
  // a watched element that stalled in its NH projection: let the full
  // evaluation run (and raise)
  if (*(volatile const int*)&esc->status & ST_NH_STALL) return;
  const int v = watch_v[w];
  if (v < 0) return;
  double r0, r1, r2;
  residual_row(v, mass, q, q_hat, inc_ptr, inc, fe, b_ptr, b_idx, b_target, b_comp, c_count, c_off, c_force,
               has_contacts, h2, r0, r1, r2);
  const double a = fmax(fabs(r0), fmax(fabs(r1), fabs(r2)));
  if (!(a < rmax_prev)) {   // >= or NaN: max|r_try| cannot drop below max|r|
    esc->precheck = 1;
    esc->skip = 1;
  }
}

void launch_watch_select(dp_scene* s, const double* r, double frac) {
  cudaMemsetAsync(&s->esc->n_watch, 0, 2 * sizeof(int), s->stream);
  k_watch_select<<<grid_for(s->V, 256), 256, 0, s->stream>>>(s->V, s->NV, r, s->inc_ptr, s->inc, frac, s->watch_v,
                                                             s->watch_e, s->esc);
  s->launches++;
}

void launch_watch_elements(dp_scene* s, const double* q) {
  if (s->E == 0 || s->NV != 4) return;
  const double h2 = s->h * s->h;
  k_elements<4, EV_LIST><<<grid_for(kWatchElemMax, 128), 128, 0, s->stream>>>(
      s->ev, s->B, s->w, s->mu, s->lam, s->model, s->E, q, h2, 1e-6, s->fe, s->fe_pos, s->H, s->Ht, s->epos, s->Pst, &s->esc->status,
      &s->esc->skip, s->watch_e, &s->esc->n_watch_elem);
  s->launches++;
}

void launch_watch_check(dp_scene* s, const double* q, double rmax_prev) {
  const int has_c = contact_sources(s) > 0;
  k_watch_check<<<grid_for(kWatchMax, 128), 128, 0, s->stream>>>(
      s->watch_v, s->mass, q, s->q_hat, s->inc_ptr, s->inc, s->fe, s->nb ? s->b_ptr : nullptr, s->b_idx, s->b_target,
      s->b_comp, s->c_count, s->c_off, s->c_force, has_c, s->h * s->h, rmax_prev, s->esc);
  s->launches++;
}

// ---------------------------------------------------------------------------
// assembly gather into SELL-32 + block-Jacobi inverses
// (fill_pattern core.py:367-376 / assemble_system_jacobian forward.py:113-149
//  / assemble_adjoint_operator adjoint.py:93-120)

__device__ __forceinline__ void inv3_guarded(const double a[9], double o[9]) {
  double c00 = a[4] * a[8] - a[5] * a[7];
  double c01 = a[5] * a[6] - a[3] * a[8];
  double c02 = a[3] * a[7] - a[4] * a[6];
  double det = a[0] * c00 + a[1] * c01 + a[2] * c02;
  double scale = fabs(a[0]) + fabs(a[4]) + fabs(a[8]);
  if (!(fabs(det) > 1e-14 * scale * scale * scale) || !isfinite(det)) {
    // fall back to the scalar Jacobi of the reference (linsolve.py:216-227)
#pragma unroll
    for (int k = 0; k < 9; ++k) o[k] = 0.0;
    o[0] = 1.0 / a[0]; o[4] = 1.0 / a[4]; o[8] = 1.0 / a[8];
    return;
  }
  double id = 1.0 / det;
  o[0] = c00 * id;
  o[1] = (a[2] * a[7] - a[1] * a[8]) * id;
  o[2] = (a[1] * a[5] - a[2] * a[4]) * id;
  o[3] = c01 * id;
  o[4] = (a[0] * a[8] - a[2] * a[6]) * id;
  o[5] = (a[2] * a[3] - a[0] * a[5]) * id;
  o[6] = c02 * id;
  o[7] = (a[1] * a[6] - a[0] * a[7]) * id;
  o[8] = (a[0] * a[4] - a[1] * a[3]) * id;
}

__global__ void __launch_bounds__(256) k_assemble(int V, int S, const int* __restrict__ slice_base,
                                                  const int* __restrict__ slice_width, const int* __restrict__ diag_slot,
                                                  const int2* __restrict__ rinfo, const int* __restrict__ tslot,
                                                  const double* __restrict__ H, const double* __restrict__ Ht,
                                                  const double* __restrict__ mass,
                                                  const int* __restrict__ b_ptr, const int* __restrict__ b_idx,
                                                  const double* __restrict__ b_comp, const int* __restrict__ c_count,
                                                  const int* __restrict__ c_off, const double* __restrict__ c_blk,
                                                  int use_extras, double h2, double* __restrict__ val,
                                                  double* __restrict__ minv, float* __restrict__ val32,
                                                  float* __restrict__ minv32, unsigned short* __restrict__ val16,
                                                  float* __restrict__ sc16, int h32) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= S) return;
  const int row = gw * kSlice + lane;
  const int base = slice_base[gw];
  const int K = slice_width[gw];
  const int dslot = (row < V) ? diag_slot[row] : -1;
  double* vs = val ? val + (size_t)base * 9 : nullptr;   // null: FP32 copy only
  for (int k = 0; k < K; ++k) {
    const int slot = base + k * kSlice + lane;
    double b[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) b[c] = 0.0;
    // the slot's contributions: one contiguous run of the block stream,
    // summed in list order (transposed for the i > j slots); the loads of a
    // group of ASM_CHUNK blocks are issued before the accumulation
    const int2 ri = rinfo[slot];
    const bool tr = ri.y < 0;
    // with tslot: a (j, i) slot is written by its canonical partner (i, j)
    // (the transposed run sum is the transpose of the run sum, entry by
    // entry the same additions), padding slots keep their zeros
    if (tslot && (tr || (ri.y == 0 && slot != dslot))) continue;
    const int n = tr ? -ri.y : ri.y;
    const double* hs = H + (size_t)ri.x * kHS;
    const double* ht = Ht + ri.x;
    int t = 0;
    if (h32) {
      // FP32 block stream (EV_H32): 32 B + 4 B per block
      const float* hs32 = reinterpret_cast<const float*>(H) + (size_t)ri.x * 8;
      const float* ht32 = reinterpret_cast<const float*>(Ht) + ri.x;
      for (; t + ASM_CHUNK <= n; t += ASM_CHUNK) {
        // the group's blocks held as floats (half the registers of doubles),
        // widened exactly when accumulated
        float fs[ASM_CHUNK][9];
#pragma unroll
        for (int g = 0; g < ASM_CHUNK; ++g) {
          ld256f_na(hs32 + (size_t)(t + g) * 8, fs[g]);
          fs[g][8] = __ldg(ht32 + t + g);
        }
#pragma unroll
        for (int g = 0; g < ASM_CHUNK; ++g) {
          double src[9];
#pragma unroll
          for (int c = 0; c < 9; ++c) src[c] = fs[g][c];
          acc_block(b, src, tr);
        }
      }
      for (; t < n; ++t) {
        double src[9];
        float f[8];
        ld256f_na(hs32 + (size_t)t * 8, f);
#pragma unroll
        for (int c = 0; c < 8; ++c) src[c] = f[c];
        src[8] = __ldg(ht32 + t);
        acc_block(b, src, tr);
      }
    } else {
    for (; t + ASM_CHUNK <= n; t += ASM_CHUNK) {
      double src[ASM_CHUNK][9];
#pragma unroll
      for (int g = 0; g < ASM_CHUNK; ++g) {
        ld256_na(hs + (size_t)(t + g) * kHS, &src[g][0]);
        ld256_na(hs + (size_t)(t + g) * kHS + 4, &src[g][4]);
        src[g][8] = __ldg(ht + t + g);
      }
#pragma unroll
      for (int g = 0; g < ASM_CHUNK; ++g) acc_block(b, src[g], tr);
    }
    for (; t < n; ++t) {
      double src[9];
      ld256_na(hs + (size_t)t * kHS, &src[0]);
      ld256_na(hs + (size_t)t * kHS + 4, &src[4]);
      src[8] = __ldg(ht + t);
      acc_block(b, src, tr);
    }
    }
    if (slot == dslot) {
      const double m = mass[row];
      b[0] += m; b[4] += m; b[8] += m;
      if (use_extras) {
        if (b_ptr) {
          for (int t = b_ptr[row]; t < b_ptr[row + 1]; ++t) {
            const double kb = h2 / b_comp[b_idx[t]];
            b[0] += kb; b[4] += kb; b[8] += kb;
          }
        }
        if (c_count) {
          const int c0 = c_off[row], cn = c_count[row];
          for (int c = c0; c < c0 + cn; ++c)
#pragma unroll
            for (int u = 0; u < 9; ++u) b[u] += c_blk[(size_t)c * 9 + u];
        }
      }
      double o[9];
      inv3_guarded(b, o);
#pragma unroll
      for (int u = 0; u < 9; ++u) minv[(size_t)u * V + row] = o[u];
      if (minv32) {
#pragma unroll
        for (int u = 0; u < 9; ++u) minv32[(size_t)u * V + row] = (float)o[u];
      }
    }
    if (vs) {
#pragma unroll
      for (int c = 0; c < 9; ++c) vs[(k * 9 + c) * kSlice + lane] = b[c];
    }
    if (val32) {
      // FP32 copy for the multigrid smoother: 12 floats per slot (9 + pad),
      // slot-major, so a lane reads its block as three 16-byte loads and a
      // warp reads 1.5 KB contiguous
#if DP_VAL32_PACKED == 2
      const float f8[8] = {(float)b[0], (float)b[1], (float)b[2], (float)b[3],
                           (float)b[4], (float)b[5], (float)b[6], (float)b[7]};
      st256f(val32 + (size_t)slot * 8, f8);
      val32[(size_t)slice_base[S] * 8 + slot] = (float)b[8];
#elif DP_VAL32_PACKED
      float4* v4 = reinterpret_cast<float4*>(val32 + (size_t)slot * 12);
      v4[0] = make_float4((float)b[0], (float)b[1], (float)b[2], (float)b[3]);
      v4[1] = make_float4((float)b[4], (float)b[5], (float)b[6], (float)b[7]);
      v4[2] = make_float4((float)b[8], 0.f, 0.f, 0.f);
#else
      float* v32 = val32 + (size_t)base * 9;
#pragma unroll
      for (int c = 0; c < 9; ++c) v32[(k * 9 + c) * kSlice + lane] = (float)b[c];
#endif
    }
    if (tslot) {
      const int t = tslot[slot];
      if (t >= 0) {
        const size_t tb = (size_t)(t - (t % kSlice)) * 9 + (t % kSlice);   // component 0 of slot t
        if (val) {
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) val[tb + (size_t)(r * 3 + c) * kSlice] = b[c * 3 + r];
        }
        if (val32) {
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) val32[tb + (size_t)(r * 3 + c) * kSlice] = (float)b[c * 3 + r];
        }
      }
    }
    if (val16) {
      // FP16 copy for the fine smoother: values / block max |a| (in [-1, 1])
      double mx = 0.0;
#pragma unroll
      for (int c = 0; c < 9; ++c) mx = fmax(mx, fabs(b[c]));
      const float scf = mx > 0.0 ? (float)mx : 1.0f;
      sc16[slot] = scf;
      unsigned short* v16 = val16 + (size_t)base * 9;
#pragma unroll
      for (int c = 0; c < 9; ++c)
        v16[(k * 9 + c) * kSlice + lane] = __half_as_ushort(__float2half_rn((float)(b[c] / (double)scf)));
    }
  }
}

static const int g_asm_tslot = getenv("DP_ASM_TSLOT") ? atoi(getenv("DP_ASM_TSLOT")) : 1;

void launch_assemble(dp_scene* s, double* val, int transpose_contacts, int amat, int h32) {
  (void)transpose_contacts;   // contact blocks are already stored transposed by the contact kernel
  const int nt = 256;
  const int nb = grid_for((int64_t)s->S * 32, nt);
  const int has_c = (contact_sources(s) > 0) && !amat;
  ktm_begin(s, KT_ASSEMBLE);
  // canonical-slot assembly (each run read once, the transpose written by
  // the same lane): not for the FP16 copy or the mass-matrix pass
  const int* tslot = (g_asm_tslot && !amat && !s->val16 && DP_VAL32_PACKED == 0) ? s->tslot : nullptr;
  k_assemble<<<nb, nt, 0, s->stream>>>(s->V, s->S, s->slice_base, s->slice_width, s->diag_slot, s->rinfo, tslot,
                                       s->H, s->Ht, s->mass, s->nb ? s->b_ptr : nullptr, s->b_idx, s->b_comp,
                                       has_c ? s->c_count : nullptr, s->c_off, s->c_blk, amat ? 0 : 1,
                                       s->h * s->h, h32 ? nullptr : val, s->minv, amat ? nullptr : s->val32,
                                       amat ? nullptr : s->minv32, amat ? nullptr : s->val16,
                                       amat ? nullptr : s->sc16, h32);
  ktm_end(s, KT_ASSEMBLE);
  if (!amat && s->val32) s->val32_src = val;   // the FP32 copy now mirrors `val`
  if (!amat) s->val64_valid = !h32;              // false: only the FP32 copy of `val` is current
  s->launches++;
}

// ---------------------------------------------------------------------------
// SELL-32 BSR SpMV: one warp per slice of 32 block rows, one lane per row.

template <bool PRECOND, class TV>
__device__ __forceinline__ void spmv_row(int V, int slice, int lane, const int* __restrict__ slice_base,
                                         const int* __restrict__ slice_width, const int* __restrict__ col,
                                         const TV* __restrict__ val, const double* __restrict__ x, double y[3]) {
  const int base = slice_base[slice];
  const int K = slice_width[slice];
  const TV* vs = val + (size_t)base * 9 + lane;
  const int* cs = col + base + lane;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll 2
  for (int k = 0; k < K; ++k) {
    const int j = __ldg(cs + k * kSlice);
    const TV* v = vs + k * 9 * kSlice;
    const double x0 = __ldg(x + 3 * j), x1 = __ldg(x + 3 * j + 1), x2 = __ldg(x + 3 * j + 2);
    a0 += (double)__ldcs(v + 0 * kSlice) * x0 + (double)__ldcs(v + 1 * kSlice) * x1 +
          (double)__ldcs(v + 2 * kSlice) * x2;
    a1 += (double)__ldcs(v + 3 * kSlice) * x0 + (double)__ldcs(v + 4 * kSlice) * x1 +
          (double)__ldcs(v + 5 * kSlice) * x2;
    a2 += (double)__ldcs(v + 6 * kSlice) * x0 + (double)__ldcs(v + 7 * kSlice) * x1 +
          (double)__ldcs(v + 8 * kSlice) * x2;
  }
  y[0] = a0; y[1] = a1; y[2] = a2;
}

template <class TV>
__global__ void __launch_bounds__(256) k_spmv(int V, int S, const int* __restrict__ slice_base,
                                              const int* __restrict__ slice_width, const int* __restrict__ col,
                                              const TV* __restrict__ val, const double* __restrict__ x,
                                              double* __restrict__ y) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= S) return;
  double a[3];
  spmv_row<false>(V, gw, lane, slice_base, slice_width, col, val, x, a);
  const int row = gw * kSlice + lane;
  if (row < V) { y[3 * row] = a[0]; y[3 * row + 1] = a[1]; y[3 * row + 2] = a[2]; }
}

void launch_spmv(dp_scene* s, const double* val, const double* x, double* y) {
  const int nb = grid_for((int64_t)s->S * 32, 256);
  ktm_begin(s, KT_SPMV);
  if (val == s->val32_src && !s->val64_valid)   // FP32-only forward operator (EV_H32)
    k_spmv<float><<<nb, 256, 0, s->stream>>>(s->V, s->S, s->slice_base, s->slice_width, s->col, s->val32, x, y);
  else
    k_spmv<double><<<nb, 256, 0, s->stream>>>(s->V, s->S, s->slice_base, s->slice_width, s->col, val, x, y);
  ktm_end(s, KT_SPMV);
  s->launches++;
}

// ---------------------------------------------------------------------------
// Chronopoulos-Gear PCG (one grid reduction phase per iteration) with
// 3x3 block-Jacobi preconditioning.  Two kernels per iteration:
//   KA: p = u + b p; s = w + b s; x += a p; r -= a s; u = Minv r; (r,u), (r,r)
//   KB: w = A u; (w,u); last block updates alpha/beta and the done flag.

__device__ __forceinline__ void minv_apply(const double* __restrict__ minv, int V, int i, const double r[3], double u[3]) {
  const double m0 = minv[0 * (size_t)V + i], m1 = minv[1 * (size_t)V + i], m2 = minv[2 * (size_t)V + i];
  const double m3 = minv[3 * (size_t)V + i], m4 = minv[4 * (size_t)V + i], m5 = minv[5 * (size_t)V + i];
  const double m6 = minv[6 * (size_t)V + i], m7 = minv[7 * (size_t)V + i], m8 = minv[8 * (size_t)V + i];
  u[0] = m0 * r[0] + m1 * r[1] + m2 * r[2];
  u[1] = m3 * r[0] + m4 * r[1] + m5 * r[2];
  u[2] = m6 * r[0] + m7 * r[1] + m8 * r[2];
}

__device__ __forceinline__ int ldflag(const int* p) { return *(volatile const int*)p; }

// init: x = 0, p = s = 0, r = b, u = Minv r; gamma = (r,u), rho = (r,r)
__global__ void __launch_bounds__(kVT) k_cg_init(int V, const double* __restrict__ b, const double* __restrict__ minv,
                                                 double* x, double* r, double* u, double* p, double* s, double rtol,
                                                 double* partial, unsigned int* counter, KrylovScalars* ks) {
  __shared__ double sh[32];
  __shared__ double out[2];
  const int i = blockIdx.x * kVT + threadIdx.x;
  double ru = 0.0, rr = 0.0;
  if (i < V) {
    double rv[3] = {b[3 * i], b[3 * i + 1], b[3 * i + 2]};
    double uv[3];
    minv_apply(minv, V, i, rv, uv);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      x[3 * i + c] = 0.0; p[3 * i + c] = 0.0; s[3 * i + c] = 0.0;
      r[3 * i + c] = rv[c]; u[3 * i + c] = uv[c];
      ru += rv[c] * uv[c]; rr += rv[c] * rv[c];
    }
  }
  double t0 = block_sum<kVT>(ru, sh);
  double t1 = block_sum<kVT>(rr, sh);
  if (threadIdx.x == 0) { partial[2 * blockIdx.x] = t0; partial[2 * blockIdx.x + 1] = t1; }
  if (last_block(counter)) {
    fold_partials<kVT, 2>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) {
      ks->gamma = out[0];
      ks->rho = out[1];
      ks->bnorm2 = out[1];
      ks->tol2 = rtol * rtol * out[1];
      ks->alpha = 0.0; ks->beta = 0.0; ks->delta = 0.0;
      ks->iters = 0;
      ks->done = (out[1] == 0.0) ? 1 : 0;
      ks->pad[0] = out[0];   // gamma_new
      *counter = 0;
    }
  }
}

// KB: w = A u; delta = (w, u); last block computes alpha, beta
__global__ void __launch_bounds__(256) k_cg_spmv(int V, int S, const int* __restrict__ slice_base,
                                                 const int* __restrict__ slice_width, const int* __restrict__ col,
                                                 const double* __restrict__ val, const double* __restrict__ u,
                                                 double* __restrict__ w, double* partial, unsigned int* counter,
                                                 KrylovScalars* ks, int first) {
  __shared__ double sh[32];
  __shared__ double out[1];
  if (ldflag(&ks->done)) return;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  double wu = 0.0;
  if (gw < S) {
    double a[3];
    spmv_row<false>(V, gw, lane, slice_base, slice_width, col, val, u, a);
    const int row = gw * kSlice + lane;
    if (row < V) {
      w[3 * row] = a[0]; w[3 * row + 1] = a[1]; w[3 * row + 2] = a[2];
      wu = a[0] * u[3 * row] + a[1] * u[3 * row + 1] + a[2] * u[3 * row + 2];
    }
  }
  double t = block_sum<256>(wu, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block(counter)) {
    fold_partials<256, 1>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) {
      const double delta = out[0];
      const double gnew = ks->pad[0];
      if (first) {
        ks->beta = 0.0;
        if (!(delta > 0.0)) ks->done = 2;
        else ks->alpha = gnew / delta;
      } else {
        const double beta = gnew / ks->gamma;
        const double den = delta - beta * gnew / ks->alpha;
        ks->beta = beta;
        if (!(den > 0.0)) ks->done = 2;     // p^T A p <= 0: breakdown (linsolve.py:89-91)
        else ks->alpha = gnew / den;
      }
      ks->gamma = gnew;
      ks->delta = delta;
      *counter = 0;
    }
  }
}

// KA: vector updates + preconditioner + (r,u), (r,r)
__global__ void __launch_bounds__(kVT) k_cg_update(int V, const double* __restrict__ minv, double* x, double* r,
                                                   double* u, const double* __restrict__ w, double* p, double* s,
                                                   double* partial, unsigned int* counter, KrylovScalars* ks) {
  __shared__ double sh[32];
  __shared__ double out[2];
  if (ldflag(&ks->done)) return;
  const double alpha = ks->alpha, beta = ks->beta;
  const int i = blockIdx.x * kVT + threadIdx.x;
  double ru = 0.0, rr = 0.0;
  if (i < V) {
    double rv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int k = 3 * i + c;
      const double pk = u[k] + beta * p[k];
      const double sk = w[k] + beta * s[k];
      p[k] = pk; s[k] = sk;
      x[k] += alpha * pk;
      rv[c] = r[k] - alpha * sk;
      r[k] = rv[c];
    }
    double uv[3];
    minv_apply(minv, V, i, rv, uv);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      u[3 * i + c] = uv[c];
      ru += rv[c] * uv[c];
      rr += rv[c] * rv[c];
    }
  }
  double t0 = block_sum<kVT>(ru, sh);
  double t1 = block_sum<kVT>(rr, sh);
  if (threadIdx.x == 0) { partial[2 * blockIdx.x] = t0; partial[2 * blockIdx.x + 1] = t1; }
  if (last_block(counter)) {
    fold_partials<kVT, 2>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) {
      ks->pad[0] = out[0];
      ks->rho = out[1];
      ks->iters += 1;
      if (out[1] <= ks->tol2) ks->done = 1;
      *counter = 0;
    }
  }
}

// r = b - A x ; returns partial |r|^2 -> scalar (used for true residuals)
template <class TV>
__global__ void __launch_bounds__(256) k_resid_true(int V, int S, const int* __restrict__ slice_base,
                                                    const int* __restrict__ slice_width, const int* __restrict__ col,
                                                    const TV* __restrict__ val, const double* __restrict__ x,
                                                    const double* __restrict__ b, double* __restrict__ r,
                                                    double* partial, unsigned int* counter, double* result) {
  __shared__ double sh[32];
  __shared__ double out[1];
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  if (gw < S) {
    double a[3];
    spmv_row<false>(V, gw, lane, slice_base, slice_width, col, val, x, a);
    const int row = gw * kSlice + lane;
    if (row < V) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double v = b[3 * row + c] - a[c];
        r[3 * row + c] = v;
        acc += v * v;
      }
    }
  }
  double t = block_sum<256>(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block(counter)) {
    fold_partials<256, 1>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) { *result = out[0]; *counter = 0; }
  }
}

__global__ void __launch_bounds__(kVT) k_norm2(int n, const double* __restrict__ x, double* partial,
                                               unsigned int* counter, double* result) {
  __shared__ double sh[32];
  __shared__ double out[1];
  double acc = 0.0;
  for (int i = blockIdx.x * kVT + threadIdx.x; i < n; i += gridDim.x * kVT) acc += x[i] * x[i];
  double t = block_sum<kVT>(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block(counter)) {
    fold_partials<kVT, 1>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) { *result = out[0]; *counter = 0; }
  }
}

__global__ void k_axpy_to(int n, double* out, const double* a, double t, const double* b) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = a[i] + t * b[i];
}

void launch_axpy_to(dp_scene* s, double* out, const double* a, double t, const double* b) {
  const int n = 3 * s->V;
  k_axpy_to<<<grid_for(n, 256), 256, 0, s->stream>>>(n, out, a, t, b);
  s->launches++;
}

double device_norm2(dp_scene* s, const double* x) {
  const int n = 3 * s->V;
  int nb = grid_for(n, kVT);
  if (nb > 1024) nb = 1024;
  double* res = s->red.partial + s->red.cap_blocks * s->red.width - 1;
  k_norm2<<<nb, kVT, 0, s->stream>>>(n, x, s->red.partial, s->red.counter, res);
  s->launches++;
  double h = 0.0;
  cudaMemcpyAsync(&s->h_ksc->pad[1], res, sizeof(double), cudaMemcpyDeviceToHost, s->stream);
  host_sync(s);
  h = s->h_ksc->pad[1];
  return h;
}

// true relative residual |b - A x| / |b| (synchronous)
// |x|^2 -> *host (pinned) without a sync: the value is valid after the
// caller's next host_sync (second reduction slot, see device_norm2)
static void norm2_async(dp_scene* s, const double* x, double* host) {
  const int n = 3 * s->V;
  int nb = grid_for(n, kVT);
  if (nb > 1024) nb = 1024;
  double* res = s->red.partial + s->red.cap_blocks * s->red.width - 2;
  k_norm2<<<nb, kVT, 0, s->stream>>>(n, x, s->red.partial, s->red.counter, res);
  s->launches++;
  cudaMemcpyAsync(host, res, sizeof(double), cudaMemcpyDeviceToHost, s->stream);
}

// launch half of true_relres: r = b - A x and |r|^2 -> h_ksc->pad[1] (async)
static void true_relres_launch(dp_scene* s, const double* val, const double* b, const double* x, double* r) {
  const int nb = grid_for((int64_t)s->S * 32, 256);
  double* res = s->red.partial + s->red.cap_blocks * s->red.width - 1;
  if (val == s->val32_src && !s->val64_valid)   // FP32-only forward operator (EV_H32)
    k_resid_true<float><<<nb, 256, 0, s->stream>>>(s->V, s->S, s->slice_base, s->slice_width, s->col, s->val32, x,
                                                   b, r, s->red.partial, s->red.counter, res);
  else
    k_resid_true<double><<<nb, 256, 0, s->stream>>>(s->V, s->S, s->slice_base, s->slice_width, s->col, val, x, b,
                                                    r, s->red.partial, s->red.counter, res);
  s->launches++;
  cudaMemcpyAsync(&s->h_ksc->pad[1], res, sizeof(double), cudaMemcpyDeviceToHost, s->stream);
}

static double true_relres(dp_scene* s, const double* val, const double* b, const double* x, double* r, double bnorm) {
  const int nb = grid_for((int64_t)s->S * 32, 256);
  double* res = s->red.partial + s->red.cap_blocks * s->red.width - 1;
  if (val == s->val32_src && !s->val64_valid)   // FP32-only forward operator (EV_H32)
    k_resid_true<float><<<nb, 256, 0, s->stream>>>(s->V, s->S, s->slice_base, s->slice_width, s->col, s->val32, x,
                                                   b, r, s->red.partial, s->red.counter, res);
  else
    k_resid_true<double><<<nb, 256, 0, s->stream>>>(s->V, s->S, s->slice_base, s->slice_width, s->col, val, x, b,
                                                    r, s->red.partial, s->red.counter, res);
  s->launches++;
  cudaMemcpyAsync(&s->h_ksc->pad[1], res, sizeof(double), cudaMemcpyDeviceToHost, s->stream);
  host_sync(s);
  return sqrt(s->h_ksc->pad[1]) / bnorm;
}

static void read_ksc(dp_scene* s) {
  cudaMemcpyAsync(s->h_ksc, s->ksc, sizeof(KrylovScalars), cudaMemcpyDeviceToHost, s->stream);
  host_sync(s);
}

// Solve A x = b to rtol (true relative residual).  Returns 0 ok, 1 not
// converged, 2 breakdown (A not SPD).  x is overwritten.
int cg_solve(dp_scene* s, const double* val, const double* b, double* x, double rtol, int max_iter, int* iters,
             double* relres, int* breakdown) {
  const int V = s->V;
  const int nbv = grid_for(V, kVT);
  const int nbs = grid_for((int64_t)s->S * 32, 256);
  *iters = 0;
  *breakdown = 0;
  double bnorm = sqrt(device_norm2(s, b));
  if (bnorm == 0.0) {
    cudaMemsetAsync(x, 0, sizeof(double) * 3 * V, s->stream);
    *relres = 0.0;
    return 0;
  }
  // restarts on the true residual: x = x0 + d, A d = b - A x0
  double* bb = s->tmp;   // current rhs of the correction solve
  double* xc = s->kx;
  cudaMemsetAsync(x, 0, sizeof(double) * 3 * V, s->stream);
  cudaMemcpyAsync(bb, b, sizeof(double) * 3 * V, cudaMemcpyDeviceToDevice, s->stream);
  double rel = 1.0;
  for (int restart = 0; restart < 4; ++restart) {
    double inner_rtol = rtol / rel * 0.5;
    if (inner_rtol > 0.5) inner_rtol = 0.5;
    if (inner_rtol < 1e-15) inner_rtol = 1e-15;
    k_cg_init<<<nbv, kVT, 0, s->stream>>>(V, bb, s->minv, xc, s->kr, s->ku, s->kp, s->ks, inner_rtol, s->red.partial,
                                          s->red.counter, s->ksc);
    k_cg_spmv<<<nbs, 256, 0, s->stream>>>(V, s->S, s->slice_base, s->slice_width, s->col, val, s->ku, s->kw,
                                          s->red.partial, s->red.counter, s->ksc, 1);
    s->launches += 2;
    int done = 0, launched = 0;
    int chunk = 8;
    while (!done && *iters + launched < max_iter) {
      int n = chunk;
      if (*iters + launched + n > max_iter) n = max_iter - *iters - launched;
      for (int k = 0; k < n; ++k) {
        k_cg_update<<<nbv, kVT, 0, s->stream>>>(V, s->minv, xc, s->kr, s->ku, s->kw, s->kp, s->ks, s->red.partial,
                                                s->red.counter, s->ksc);
        k_cg_spmv<<<nbs, 256, 0, s->stream>>>(V, s->S, s->slice_base, s->slice_width, s->col, val, s->ku, s->kw,
                                              s->red.partial, s->red.counter, s->ksc, 0);
      }
      s->launches += 2 * n;
      launched += n;
      read_ksc(s);
      done = s->h_ksc->done;
      if (chunk < 64) chunk *= 2;
    }
    *iters += s->h_ksc->iters;
    if (s->h_ksc->done == 2) {
      *breakdown = 1;
      // keep the progress so far
      launch_axpy_to(s, x, x, 1.0, xc);
      *relres = true_relres(s, val, b, x, s->tmp, bnorm);
      return 2;
    }
    launch_axpy_to(s, x, x, 1.0, xc);
    rel = true_relres(s, val, b, x, bb, bnorm);   // bb <- b - A x
    if (rel <= rtol || *iters >= max_iter) break;
  }
  *relres = rel;
  return rel <= rtol ? 0 : 1;
}

// ---------------------------------------------------------------------------
// GMRES(m) (gmres, linsolve.py:108-197), device-driven: the column index j,
// the Hessenberg matrix, the Givens rotations and the stop decision live in
// GmresScalars on the device.  Every column kernel reads j from there, and
// k_gm_loopctl advances it and sets the condition of a CUDA-graph WHILE node,
// so a whole restart cycle (up to 50 columns, incl. the multigrid V-cycles)
// is ONE graph launch with no host round trip.  Classical Gram-Schmidt fused
// into the SpMV pass, conditional second pass for tight solves.

constexpr int kGT = 256;
constexpr int kGM1 = kMaxRestart + 1;

__device__ __forceinline__ bool gm_idle(const GmresScalars* gs) {
  return ldflag(&gs->done) || !ldflag(&gs->active);
}

// Left block-Jacobi column kernel, one warp per SELL slice:
//   v_j = w_prev / hn            (own rows, written to the basis)
//   w   = Minv A v_j             (SpMV on the gathered w_prev / hn)
//   coef_i = (w, v_i), i <= j and |w|^2   (block partials, last block folds)
__global__ void __launch_bounds__(256) k_gm_spmvdot(int V, int S, const int* __restrict__ slice_base,
                                                    const int* __restrict__ slice_width, const int* __restrict__ col,
                                                    const double* __restrict__ val, const double* __restrict__ minv,
                                                    double* W0, double* W1, double* Vb, size_t ld, double* partial,
                                                    unsigned int* counter, GmresScalars* gs) {
  __shared__ double sh[8][kGM1 + 1];
  if (gm_idle(gs)) return;
  const int j = gs->j;
  const double* wprev = (j & 1) ? W1 : W0;
  double* wnew = (j & 1) ? W0 : W1;
  double* vj = Vb + (size_t)j * ld;
  const double inv = 1.0 / gs->hn;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * 8 + warp;
  const int row = gw * kSlice + lane;
  double u[3] = {0.0, 0.0, 0.0}, vr[3] = {0.0, 0.0, 0.0};
  if (gw < S) {
    double a[3];
    spmv_row<false>(V, gw, lane, slice_base, slice_width, col, val, wprev, a);
    if (row < V) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        a[c] *= inv;
        vr[c] = wprev[3 * row + c] * inv;
        vj[3 * row + c] = vr[c];
      }
      minv_apply(minv, V, row, a, u);
#pragma unroll
      for (int c = 0; c < 3; ++c) wnew[3 * row + c] = u[c];
    }
  }
  const bool live = (gw < S) && (row < V);
  for (int i0 = 0; i0 <= j + 1; i0 += 8) {
    double d[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = i0 + t;
      double v = 0.0;
      if (live && i <= j + 1) {
        if (i < j) {
          const double* vi = Vb + (size_t)i * ld + 3 * (size_t)row;
          v = u[0] * vi[0] + u[1] * vi[1] + u[2] * vi[2];
        } else if (i == j) {
          v = u[0] * vr[0] + u[1] * vr[1] + u[2] * vr[2];
        } else {
          v = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
        }
      }
      d[t] = v;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const double r = warp_sum(d[t]);
      if (lane == 0 && i0 + t <= j + 1) sh[warp][i0 + t] = r;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= j + 1; i += blockDim.x) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += sh[w][i];
    partial[(size_t)blockIdx.x * (kGM1 + 1) + i] = t;
  }
  if (last_block(counter)) {
    __shared__ double res[kGM1 + 1];
    fold_multi<256>(partial, kGM1 + 1, gridDim.x, j + 2, res);
    for (int i = threadIdx.x; i <= j + 1; i += blockDim.x) {
      if (i <= j) {
        gs->coef[i] = res[i];
        gs->H[(size_t)j * kGM1 + i] = res[i];
      } else {
        gs->wn2_before = res[i];
      }
    }
    if (threadIdx.x == 0) *counter = 0;
  }
}

// coef_i = (w, v_i), i <= j (+ |w|^2 on the first pass), one read of the basis.
// first = 0: re-orthogonalisation pass (only when flagged), added to H.
template <typename TB>
__global__ void __launch_bounds__(kGT) k_gm_dots(int n, const TB* __restrict__ Vb, size_t ld, TB* W0,
                                                 TB* W1, double* partial, unsigned int* counter,
                                                 GmresScalars* gs, int first) {
  __shared__ double sh[kGT / 32][kGM1 + 1];
  if (gm_idle(gs)) return;
  if (!first && !ldflag(&gs->reorth)) return;
  const int j = gs->j;
  const TB* w = ((j + 1) & 1) ? W1 : W0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nd = first ? j + 2 : j + 1;
  for (int i0 = 0; i0 < nd; i0 += 8) {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = blockIdx.x * kGT + threadIdx.x; k < n; k += gridDim.x * kGT) {
      const double wk = (double)w[k];
      double vv[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) vv[t] = (double)Vb[(size_t)min(i0 + t, j) * ld + k];
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] += wk * ((i0 + t <= j) ? vv[t] : wk);
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const double d = warp_sum(acc[t]);
      if (lane == 0 && i0 + t < nd) sh[warp][i0 + t] = d;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nd; i += kGT) {
    double t = 0.0;
#pragma unroll
    for (int ww = 0; ww < kGT / 32; ++ww) t += sh[ww][i];
    partial[(size_t)blockIdx.x * (kGM1 + 1) + i] = t;
  }
  if (last_block(counter)) {
    __shared__ double res[kGM1 + 1];
    fold_multi<kGT>(partial, kGM1 + 1, gridDim.x, nd, res);
    for (int i = threadIdx.x; i < nd; i += kGT) {
      if (i <= j) {
        gs->coef[i] = res[i];
        if (first) gs->H[(size_t)j * kGM1 + i] = res[i];
        else gs->H[(size_t)j * kGM1 + i] += res[i];
      } else {
        gs->wn2_before = res[i];
      }
    }
    if (threadIdx.x == 0) *counter = 0;
  }
}

// left multigrid column kernel (host-driven path only): v_j = w/hn, t = A v_j
__global__ void __launch_bounds__(256) k_gm_spmvnorm(int V, int S, const int* __restrict__ slice_base,
                                                     const int* __restrict__ slice_width, const int* __restrict__ col,
                                                     const double* __restrict__ val, double* W0, double* W1,
                                                     double* Vb, size_t ld, double* __restrict__ t,
                                                     const GmresScalars* gs) {
  if (gm_idle(gs)) return;
  const int j = gs->j;
  const double* wprev = (j & 1) ? W1 : W0;
  double* vj = Vb + (size_t)j * ld;
  const double inv = 1.0 / gs->hn;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= S) return;
  double a[3];
  spmv_row<false>(V, gw, lane, slice_base, slice_width, col, val, wprev, a);
  const int row = gw * kSlice + lane;
  if (row < V) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      vj[3 * row + c] = wprev[3 * row + c] * inv;
      t[3 * row + c] = a[c] * inv;
    }
  }
}

__device__ void gm_finish_column(GmresScalars* gs, int j, double wn2) {
  double* Hc = gs->H + (size_t)j * kGM1;
  const double hn = sqrt(wn2);
  gs->hn = hn;
  Hc[j + 1] = hn;
  for (int i = 0; i < j; ++i) {
    const double t = gs->cs[i] * Hc[i] + gs->sn[i] * Hc[i + 1];
    Hc[i + 1] = -gs->sn[i] * Hc[i] + gs->cs[i] * Hc[i + 1];
    Hc[i] = t;
  }
  const double den = hypot(Hc[j], Hc[j + 1]);
  gs->cs[j] = den != 0.0 ? Hc[j] / den : 1.0;
  gs->sn[j] = den != 0.0 ? Hc[j + 1] / den : 0.0;
  Hc[j] = den;
  Hc[j + 1] = 0.0;
  gs->g[j + 1] = -gs->sn[j] * gs->g[j];
  gs->g[j] = gs->cs[j] * gs->g[j];
  gs->used = j + 1;
  gs->est = fabs(gs->g[j + 1]) / gs->nmb;
  if (fabs(gs->g[j + 1]) <= gs->thr) gs->done = 1;
  else if (!(hn > 1e-300)) gs->done = 2;
}

// w -= sum_i coef_i v_i ; |w|^2 ; the last block finishes column j unless a
// second orthogonalisation pass is needed.
template <typename TB>
__global__ void __launch_bounds__(kGT) k_gm_update(int n, int pass, const TB* __restrict__ Vb, size_t ld,
                                                   TB* W0, TB* W1, double* partial, unsigned int* counter,
                                                   GmresScalars* gs) {
  __shared__ double sh[32];
  __shared__ double coef[kGM1];
  __shared__ double out[1];
  if (gm_idle(gs)) return;
  if (pass == 1 && !ldflag(&gs->reorth)) return;
  const int j = gs->j;
  TB* w = ((j + 1) & 1) ? W1 : W0;
  for (int i = threadIdx.x; i <= j; i += kGT) coef[i] = gs->coef[i];
  __syncthreads();
  double acc = 0.0;
  for (int k = blockIdx.x * kGT + threadIdx.x; k < n; k += gridDim.x * kGT) {
    double v = (double)w[k];
    int i = 0;
    for (; i + 4 <= j + 1; i += 4) {
      const double a0 = (double)Vb[(size_t)i * ld + k], a1 = (double)Vb[(size_t)(i + 1) * ld + k];
      const double a2 = (double)Vb[(size_t)(i + 2) * ld + k], a3 = (double)Vb[(size_t)(i + 3) * ld + k];
      v -= coef[i] * a0 + coef[i + 1] * a1 + coef[i + 2] * a2 + coef[i + 3] * a3;
    }
    for (; i <= j; ++i) v -= coef[i] * (double)Vb[(size_t)i * ld + k];
    const TB vs = (TB)v;
    w[k] = vs;
    acc += (double)vs * (double)vs;
  }
  double t = block_sum<kGT>(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block(counter)) {
    fold_partials<kGT, 1>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) {
      *counter = 0;
      const double wn2 = out[0];
      if (pass == 0 && wn2 < gs->reorth_thr * gs->wn2_before) {
        gs->reorth = 1;
      } else {
        gs->reorth = 0;
        gm_finish_column(gs, j, wn2);
      }
    }
  }
}

// end of a column: advance j and decide whether the cycle continues; in the
// graph path this sets the WHILE node's condition.
__global__ void k_gm_loopctl(GmresScalars* gs, cudaGraphConditionalHandle handle, int use_cond) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned int cont = 0;
  if (!gs->done && gs->active) {
    gs->j += 1;
    cont = (gs->j < gs->m && gs->used < gs->maxit) ? 1u : 0u;
    if (!cont) gs->active = 0;
  }
  if (use_cond) cudaGraphSetConditional(handle, cont);
}

// cycle start: v0 = (Minv) r (unnormalised) and |v0|^2 -> beta, g, thresholds
template <typename TB>
__global__ void __launch_bounds__(kVT) k_gm_start(double reorth_thr, int V, const double* __restrict__ minv,
                                                  const double* __restrict__ r,
                                                  TB* __restrict__ v0, double* partial, unsigned int* counter,
                                                  GmresScalars* gs, double tol, int set_nmb, int m, int maxit) {
  __shared__ double sh[32];
  __shared__ double out[1];
  const int i = blockIdx.x * kVT + threadIdx.x;
  double acc = 0.0;
  if (i < V) {
    double rv[3] = {r[3 * i], r[3 * i + 1], r[3 * i + 2]}, u[3] = {rv[0], rv[1], rv[2]};
    if (minv) minv_apply(minv, V, i, rv, u);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const TB us = (TB)u[c];
      if (v0) v0[3 * i + c] = us;
      acc += (double)us * (double)us;
    }
  }
  double t = block_sum<kVT>(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block(counter)) {
    fold_partials<kVT, 1>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) {
      *counter = 0;
      const double beta = sqrt(out[0]);
      if (set_nmb) {
        gs->nmb = beta != 0.0 ? beta : 1.0;   // |(M^-1) b| (linsolve.py:180)
      } else {
        gs->beta = beta;
        for (int k = 0; k <= kMaxRestart; ++k) gs->g[k] = 0.0;
        gs->g[0] = beta;
        gs->hn = beta;
        gs->thr = 0.1 * tol * gs->nmb;
        gs->done = (beta == 0.0) ? 2 : 0;
        gs->reorth = 0;
        // tight solves (adjoint, 1e-10) need CGS2-level orthogonality; the
        // inexact Newton solves only re-orthogonalise on severe cancellation
        gs->reorth_thr = (tol < 1e-7) ? reorth_thr : 0.0;
        gs->used = 0;
        gs->est = beta / gs->nmb;
        gs->j = 0;
        gs->m = m;
        gs->maxit = maxit;
        gs->active = (maxit > 0) ? 1 : 0;
      }
    }
  }
}

// x += sum_i y_i v_i   (or x = sum when accumulate == 0)
template <typename TB>
__global__ void k_gm_combine(int n, int used, const double* __restrict__ y, const TB* __restrict__ Vb, size_t ld,
                             double* __restrict__ x, int accumulate) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < used; ++i) acc += y[i] * (double)Vb[(size_t)i * ld + k];
    x[k] = accumulate ? x[k] + acc : acc;
  }
}

// Right-preconditioned column, step 1: v_j = w_prev / hn; z = Minv v_j
// (block-Jacobi) or, with multigrid, a copy of v_j into the V-cycle's fixed
// input buffer.
template <typename TB>
__global__ void k_gm_prec(int V, TB* W0, TB* W1, TB* Vb, size_t ld, const double* __restrict__ minv,
                          double* __restrict__ z, double* __restrict__ vcopy, const GmresScalars* gs,
                          const float* __restrict__ minv32, double omega, double* __restrict__ xa) {
  if (gm_idle(gs)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int j = gs->j;
  const TB* wprev = (j & 1) ? W1 : W0;
  TB* vj = Vb + (size_t)j * ld;
  const double inv = 1.0 / gs->hn;
  double v[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const TB vs = (TB)((double)wprev[3 * i + c] * inv);
    v[c] = (double)vs;
    vj[3 * i + c] = vs;
    if (vcopy) vcopy[3 * i + c] = v[c];
  }
  if (xa) {
    // the V-cycle's first fine sweep from zero, x = omega Minv v (k_mg_jacobi0<float>)
    const double r[3] = {v[0], v[1], v[2]};
    double u[3];
    u[0] = minv32[0 * (size_t)V + i] * r[0] + minv32[1 * (size_t)V + i] * r[1] + minv32[2 * (size_t)V + i] * r[2];
    u[1] = minv32[3 * (size_t)V + i] * r[0] + minv32[4 * (size_t)V + i] * r[1] + minv32[5 * (size_t)V + i] * r[2];
    u[2] = minv32[6 * (size_t)V + i] * r[0] + minv32[7 * (size_t)V + i] * r[1] + minv32[8 * (size_t)V + i] * r[2];
    xa[3 * i] = omega * u[0]; xa[3 * i + 1] = omega * u[1]; xa[3 * i + 2] = omega * u[2];
  }
  if (minv) {
    double u[3];
    minv_apply(minv, V, i, v, u);
#pragma unroll
    for (int c = 0; c < 3; ++c) z[3 * i + c] = u[c];
  }
}

// step 2 (one warp per SELL slice): w = A z, coef_i = (w, v_i) for i <= j,
// |w|^2; last block folds into the Hessenberg column.
// SpMV row with the packed FP32 copy of the operator (12 floats per slot)
__device__ __forceinline__ void spmv_row32(int S, int slice, int lane, const int* __restrict__ slice_base,
                                           const int* __restrict__ slice_width, const int* __restrict__ col,
                                           const float* __restrict__ val, const double* __restrict__ x, double y[3]) {
  const int base = slice_base[slice];
  const int K = slice_width[slice];
  const int* cs = col + base + lane;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#if DP_VAL32_PACKED == 2
  const float* tail = val + (size_t)slice_base[S] * 8;
#pragma unroll 2
  for (int k = 0; k < K; ++k) {
    const int slot = base + k * kSlice + lane;
    const int j = __ldg(cs + k * kSlice);
    float m[8];
    ld256f(val + (size_t)slot * 8, m);
    const float m8 = __ldg(tail + slot);
    const double x0 = __ldg(x + 3 * j), x1 = __ldg(x + 3 * j + 1), x2 = __ldg(x + 3 * j + 2);
    a0 += (double)m[0] * x0 + (double)m[1] * x1 + (double)m[2] * x2;
    a1 += (double)m[3] * x0 + (double)m[4] * x1 + (double)m[5] * x2;
    a2 += (double)m[6] * x0 + (double)m[7] * x1 + (double)m8 * x2;
  }
#elif DP_VAL32_PACKED
  const float4* p4 = reinterpret_cast<const float4*>(val) + (size_t)(base + lane) * 3;
#pragma unroll 2
  for (int k = 0; k < K; ++k) {
    const int j = __ldg(cs + k * kSlice);
    const float4* p = p4 + (size_t)k * kSlice * 3;
    const float4 q0 = __ldcs(p), q1 = __ldcs(p + 1), q2 = __ldcs(p + 2);
    const double x0 = __ldg(x + 3 * j), x1 = __ldg(x + 3 * j + 1), x2 = __ldg(x + 3 * j + 2);
    a0 += (double)q0.x * x0 + (double)q0.y * x1 + (double)q0.z * x2;
    a1 += (double)q0.w * x0 + (double)q1.x * x1 + (double)q1.y * x2;
    a2 += (double)q1.z * x0 + (double)q1.w * x1 + (double)q2.x * x2;
  }
#else
  const float* vs = val + (size_t)base * 9 + lane;
#pragma unroll 2
  for (int k = 0; k < K; ++k) {
    const int j = __ldg(cs + k * kSlice);
    const float* v = vs + k * 9 * kSlice;
    const double x0 = __ldg(x + 3 * j), x1 = __ldg(x + 3 * j + 1), x2 = __ldg(x + 3 * j + 2);
    a0 += (double)__ldcs(v + 0 * kSlice) * x0 + (double)__ldcs(v + 1 * kSlice) * x1 + (double)__ldcs(v + 2 * kSlice) * x2;
    a1 += (double)__ldcs(v + 3 * kSlice) * x0 + (double)__ldcs(v + 4 * kSlice) * x1 + (double)__ldcs(v + 5 * kSlice) * x2;
    a2 += (double)__ldcs(v + 6 * kSlice) * x0 + (double)__ldcs(v + 7 * kSlice) * x1 + (double)__ldcs(v + 8 * kSlice) * x2;
  }
#endif
  y[0] = a0; y[1] = a1; y[2] = a2;
}

template <typename TB, typename TV>
__global__ void __launch_bounds__(256) k_gm_spmvdot_r(int V, int S, const int* __restrict__ slice_base,
                                                      const int* __restrict__ slice_width,
                                                      const int* __restrict__ col, const TV* __restrict__ val,
                                                      const double* __restrict__ z, TB* W0, TB* W1,
                                                      const TB* __restrict__ Vb, size_t ld, double* partial,
                                                      unsigned int* counter, GmresScalars* gs,
                                                      double* __restrict__ Zb) {
  __shared__ double sh[8][kGM1 + 1];
  if (gm_idle(gs)) return;
  const int j = gs->j;
  TB* wnew = ((j + 1) & 1) ? W1 : W0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * 8 + warp;
  const int row = gw * kSlice + lane;
  double u[3] = {0.0, 0.0, 0.0};
  if (gw < S) {
    if constexpr (sizeof(TV) == 4) spmv_row32(S, gw, lane, slice_base, slice_width, col, val, z, u);
    else spmv_row<false>(V, gw, lane, slice_base, slice_width, col, val, z, u);
    if (row < V) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const TB us = (TB)u[c];
        wnew[3 * row + c] = us;
        u[c] = (double)us;
      }
      if (Zb) {   // keep z_j = M v_j: the cycle's update is then x += Z y
        double* zj = Zb + (size_t)j * ld + 3 * (size_t)row;
        zj[0] = z[3 * row]; zj[1] = z[3 * row + 1]; zj[2] = z[3 * row + 2];
      }
    } else {
      u[0] = u[1] = u[2] = 0.0;
    }
  }
  const bool live = (gw < S) && (row < V);
  for (int i0 = 0; i0 <= j + 1; i0 += 8) {
    double d[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = i0 + t;
      double v = 0.0;
      if (live && i <= j + 1) {
        if (i <= j) {
          const TB* vi = Vb + (size_t)i * ld + 3 * (size_t)row;
          v = u[0] * (double)vi[0] + u[1] * (double)vi[1] + u[2] * (double)vi[2];
        } else {
          v = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
        }
      }
      d[t] = v;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const double r = warp_sum(d[t]);
      if (lane == 0 && i0 + t <= j + 1) sh[warp][i0 + t] = r;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= j + 1; i += blockDim.x) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += sh[w][i];
    partial[(size_t)blockIdx.x * (kGM1 + 1) + i] = t;
  }
  if (last_block(counter)) {
    __shared__ double res[kGM1 + 1];
    fold_multi<256>(partial, kGM1 + 1, gridDim.x, j + 2, res);
    for (int i = threadIdx.x; i <= j + 1; i += blockDim.x) {
      if (i <= j) {
        gs->coef[i] = res[i];
        gs->H[(size_t)j * kGM1 + i] = res[i];
      } else {
        gs->wn2_before = res[i];
      }
    }
    if (threadIdx.x == 0) *counter = 0;
  }
}

// x += Minv t (block-Jacobi right preconditioner applied to the update)
__global__ void k_minv_axpy(int V, const double* __restrict__ minv, const double* __restrict__ t, double* x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  double v[3] = {t[3 * i], t[3 * i + 1], t[3 * i + 2]}, u[3];
  minv_apply(minv, V, i, v, u);
#pragma unroll
  for (int c = 0; c < 3; ++c) x[3 * i + c] += u[c];
}

// re-orthogonalise (tight solves only) when |w|^2 drops below this fraction
static const double g_reorth_thr = getenv("DP_REORTH") ? atof(getenv("DP_REORTH")) : 0.01;
static const int g_use_graphs = getenv("DP_GRAPHS") ? atoi(getenv("DP_GRAPHS")) : 1;
static const int g_gm_fp32 = getenv("DP_GM_FP32") ? atoi(getenv("DP_GM_FP32")) : 0;
static const int g_prejac = getenv("DP_PREJAC") ? atoi(getenv("DP_PREJAC")) : 1;
static const int g_zbasis = getenv("DP_GM_ZBASIS") ? atoi(getenv("DP_GM_ZBASIS")) : 1;

static int gm_grid(const dp_scene* s, int n) {
  // grid-stride over the basis rows with 4 CTAs per SM: every basis load of
  // a thread is independent (MLP = j+1), and the per-CTA fixed cost (coefficient
  // staging, block reduction, completion ticket) is paid 592 times instead of
  // once per 256 rows (measured: k_gm_update 18.6 -> 12.7 us at C5)
  return std::min(grid_for(n, kGT), 4 * s->nsm);
}

__global__ void k_gm_copy_wnew(int n, const double* __restrict__ src, double* W0, double* W1,
                               const GmresScalars* gs) {
  if (gm_idle(gs)) return;
  double* wn = ((gs->j + 1) & 1) ? W1 : W0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) wn[k] = src[k];
}

// Kernels of one GMRES column (j read on device).  Returns the number of
// kernel launches issued.
static int gm_column(dp_scene* s, const double* val, int use_mg, int left, bool tight, bool lowp, bool zbasis,
                     cudaGraphConditionalHandle h, int use_cond) {
  const int V = s->V, n = 3 * V;
  const size_t ld = (size_t)n;
  const int nbs = grid_for((int64_t)s->S * 32, 256);
  const int nbg = gm_grid(s, n);
  double* Vb = s->gm_V;
  double* z = s->ku;
  int k = 0;
  if (left && !use_mg) {
    k_gm_spmvdot<<<nbs, 256, 0, s->stream>>>(V, s->S, s->slice_base, s->slice_width, s->col, val, s->minv, s->kw,
                                             s->kp, Vb, ld, s->red.partial, s->red.counter, s->gsc);
    k += 1;
  } else if (left) {
    k_gm_spmvnorm<<<nbs, 256, 0, s->stream>>>(V, s->S, s->slice_base, s->slice_width, s->col, val, s->kw, s->kp, Vb,
                                              ld, z, s->gsc);
    // the V-cycle output must be the j-dependent w_new: copy through a fixed buffer
    mg_apply(s, val, z, s->q_try, &s->gsc->done);
    k_gm_copy_wnew<<<grid_for(n, 256), 256, 0, s->stream>>>(n, s->q_try, s->kw, s->kp, s->gsc);
    k_gm_dots<<<nbg, kGT, 0, s->stream>>>(n, Vb, ld, s->kw, s->kp, s->red.partial, s->red.counter, s->gsc, 1);
    k += 3;
  } else if (lowp) {
    // FP32 Krylov basis and FP32 operator copy (inexact Newton solves with
    // the V-cycle; the residual is recomputed in FP64 every cycle)
    float* Vf = reinterpret_cast<float*>(Vb);
    float* W0 = reinterpret_cast<float*>(s->kw);
    float* W1 = reinterpret_cast<float*>(s->kp);
    k_gm_prec<float><<<grid_for(V, 256), 256, 0, s->stream>>>(V, W0, W1, Vf, ld, nullptr, z, s->tmp, s->gsc,
                                                               nullptr, 0.0, nullptr);
    mg_apply(s, val, s->tmp, z, &s->gsc->done);
    k_gm_spmvdot_r<float, float><<<nbs, 256, 0, s->stream>>>(V, s->S, s->slice_base, s->slice_width, s->col,
                                                             s->val32, z, W0, W1, Vf, ld, s->red.partial,
                                                             s->red.counter, s->gsc, nullptr);
    k_gm_update<float><<<nbg, kGT, 0, s->stream>>>(n, 0, Vf, ld, W0, W1, s->red.partial, s->red.counter, s->gsc);
    k_gm_loopctl<<<1, 32, 0, s->stream>>>(s->gsc, h, use_cond);
    return k + 4;
  } else {
    const float* m32 = nullptr;
    double* xa = nullptr;
    double om = 0.0;
    if (use_mg && g_prejac) mg_fine_jacobi0_target(s, &m32, &xa, &om);
    k_gm_prec<double><<<grid_for(V, 256), 256, 0, s->stream>>>(V, s->kw, s->kp, Vb, ld, use_mg ? nullptr : s->minv,
                                                               z, use_mg ? s->tmp : nullptr, s->gsc, m32, om, xa);
    if (use_mg) {
      if (xa) mg_apply_prejac(s, val, s->tmp, z, &s->gsc->done);
      else mg_apply(s, val, s->tmp, z, &s->gsc->done);
    }
    k_gm_spmvdot_r<double, double><<<nbs, 256, 0, s->stream>>>(V, s->S, s->slice_base, s->slice_width, s->col, val,
                                                               z, s->kw, s->kp, Vb, ld, s->red.partial,
                                                               s->red.counter, s->gsc,
                                                               (use_mg && zbasis) ? s->gm_Z : nullptr);
    k += 2;
  }
  k_gm_update<double><<<nbg, kGT, 0, s->stream>>>(n, 0, Vb, ld, s->kw, s->kp, s->red.partial, s->red.counter,
                                                  s->gsc);
  k += 1;
  if (tight) {   // conditional second Gram-Schmidt pass (kernels exit unless flagged)
    k_gm_dots<<<nbg, kGT, 0, s->stream>>>(n, Vb, ld, s->kw, s->kp, s->red.partial, s->red.counter, s->gsc, 0);
    k_gm_update<double><<<nbg, kGT, 0, s->stream>>>(n, 1, Vb, ld, s->kw, s->kp, s->red.partial, s->red.counter,
                                                    s->gsc);
    k += 2;
  }
  k_gm_loopctl<<<1, 32, 0, s->stream>>>(s->gsc, h, use_cond);
  return k + 1;
}

// One restart cycle as a CUDA graph: a WHILE node whose body is one column.
// Cached per (operator, preconditioner side/type, tightness).
struct GmGraph {
  cudaGraphExec_t exec = nullptr;
  int nodes = 0;
};

static GmGraph* gm_graph(dp_scene* s, const double* val, int use_mg, int left, bool tight, bool lowp,
                         bool zbasis) {
  const uint64_t key = (uint64_t)(uintptr_t)val ^ ((uint64_t)use_mg << 1) ^ ((uint64_t)left << 2) ^
                       ((uint64_t)tight << 3) ^ ((uint64_t)lowp << 4) ^ ((uint64_t)zbasis << 5);
  for (auto& e : s->gm_graphs)
    if (e.first == key) return (GmGraph*)e.second;
  std::lock_guard<std::recursive_mutex> api_lock(api_mutex());
  cudaGraph_t g = nullptr;
  if (cudaGraphCreate(&g, 0) != cudaSuccess) return nullptr;
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) {
    cudaGraphDestroy(g);
    return nullptr;
  }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, g, nullptr, 0, &cp) != cudaSuccess) {
    cudaGraphDestroy(g);
    return nullptr;
  }
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  int nodes = 0;
  const int64_t launches0 = s->launches;
  if (cudaStreamBeginCaptureToGraph(s->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
      cudaSuccess) {
    cudaGraphDestroy(g);
    return nullptr;
  }
  const int timing_saved = s->timing;   // no timing events inside a captured graph
  s->timing = 0;
  nodes = gm_column(s, val, use_mg, left, tight, lowp, zbasis, h, 1);
  s->timing = timing_saved;
  cudaGraph_t captured = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(s->stream, &captured);
  nodes += (int)(s->launches - launches0);   // V-cycle kernels count themselves
  s->launches = launches0;
  GmGraph* gg = new GmGraph();
  if (ce != cudaSuccess || cudaGraphInstantiate(&gg->exec, g, 0) != cudaSuccess) {
    cudaGetLastError();
    cudaGraphDestroy(g);
    delete gg;
    return nullptr;
  }
  cudaGraphDestroy(g);
  gg->nodes = nodes;
  s->gm_graphs.push_back({key, (void*)gg});
  return gg;
}

void gm_graphs_destroy(dp_scene* s) {
  for (auto& e : s->gm_graphs) {
    GmGraph* gg = (GmGraph*)e.second;
    if (gg->exec) cudaGraphExecDestroy(gg->exec);
    delete gg;
  }
  s->gm_graphs.clear();
}

// Restarted GMRES(m), right (block-Jacobi or multigrid V-cycle) or left
// preconditioning.  With right preconditioning the Arnoldi estimate is the
// true residual, so the inner stop test and the Newton forcing use the same
// norm as the recomputed residual (linsolve.py:108-197 uses left
// preconditioning; the converged solution is the same).  x = 0 initially.
// Returns 0 converged, 1 not converged.
int gmres_solve(dp_scene* s, const double* val, const double* b, double* x, double rtol, int max_iter, int restart,
                int* iters, double* relres, double min_cycle_gain, int use_mg, int left, int use_x0) {
  const int V = s->V, n = 3 * V;
  if (restart > kMaxRestart) restart = kMaxRestart;
  if (restart > n) restart = n;
  if (restart < 1) restart = 1;
  const size_t ld = (size_t)n;
  const int nbv = grid_for(V, kVT);
  const int nbg = gm_grid(s, n);
  double* Vb = s->gm_V;
  double* r = s->kr;
  double* z = s->ku;       // M^-1 v_j
  double* t = s->kx;       // V y at the end of a cycle
  double* y_dev = s->ks;   // scratch (>= restart doubles)
  const bool tight = rtol < 1e-7;   // inexact Newton solves skip re-orthogonalisation
  // inexact solves with the V-cycle run in FP32 (basis + operator copy)
  const bool fp32_only = s->val32 != nullptr && val == s->val32_src && !s->val64_valid;   // EV_H32 forward
  const bool lowp = (fp32_only || g_gm_fp32) && use_mg && !left && !tight && s->val32 != nullptr &&
                    val == s->val32_src;
  if (fp32_only && !lowp) {
    set_error("GMRES needs the FP64 operator, the last assembly wrote only its FP32 copy");
    return 1;
  }
  *iters = 0;
  // x = 0, or the caller's initial guess (use_x0) when it beats x = 0
  if (!use_x0) cudaMemsetAsync(x, 0, sizeof(double) * n, s->stream);
  const double bnorm = sqrt(device_norm2(s, b));
  if (bnorm == 0.0) {
    cudaMemsetAsync(x, 0, sizeof(double) * n, s->stream);
    *relres = 0.0;
    return 0;
  }
  bool x_zero = !use_x0;
  if (use_x0 && true_relres(s, val, b, x, s->kr, bnorm) >= 1.0) {
    cudaMemsetAsync(x, 0, sizeof(double) * n, s->stream);
    x_zero = true;
  }
  // nmb = |b| (right) or |M^-1 b| (left, the reference's normalisation)
  if (left && use_mg) {
    mg_apply(s, val, b, z, nullptr);
    k_gm_start<double><<<nbv, kVT, 0, s->stream>>>(g_reorth_thr, V, nullptr, z, nullptr, s->red.partial,
                                                   s->red.counter, s->gsc, rtol, 1, 0, 0);
  } else {
    k_gm_start<double><<<nbv, kVT, 0, s->stream>>>(g_reorth_thr, V, left ? s->minv : nullptr, b, nullptr,
                                                   s->red.partial, s->red.counter, s->gsc, rtol, 1, 0, 0);
  }
  s->launches++;
  // right multigrid: keep the preconditioned basis and update x += Z y
  // (saves the end-of-cycle V-cycle)
  const bool zbasis = g_zbasis && use_mg && !left && !lowp;
  if (zbasis && !s->gm_Z) {
    if (cudaMalloc((void**)&s->gm_Z, sizeof(double) * (size_t)(kMaxRestart + 1) * n) != cudaSuccess) {
      cudaGetLastError();
      s->gm_Z = nullptr;
    }
  }
  const bool zb = zbasis && s->gm_Z;
  GmGraph* gg = (g_use_graphs && !(left && use_mg)) ? gm_graph(s, val, use_mg, left, tight, lowp, zb) : nullptr;
  int total = 0;
  double rel = 1.0;
  int m = restart;   // cycle length; grows when a cycle stagnates
  const int m_cap = std::min(kMaxRestart, n);
  bool have_rel = false;   // r and rel already hold b - A x (end of the previous cycle)
  while (total < max_iter) {
    if (!have_rel) {
      if (x_zero) {
        // x = 0: r = b exactly, no SpMV
        cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s->stream);
        rel = 1.0;
      } else {
        rel = true_relres(s, val, b, x, r, bnorm);
      }
    }
    have_rel = false;
    if (rel <= rtol) break;
    const double cycle_start = rel;
    const int budget = max_iter - total;
    const size_t gsc_bytes = offsetof(GmresScalars, H) + sizeof(double) * (size_t)m * kGM1;
    if (left && use_mg) {
      mg_apply(s, val, r, z, nullptr);
      k_gm_start<double><<<nbv, kVT, 0, s->stream>>>(g_reorth_thr, V, nullptr, z, s->kw, s->red.partial, s->red.counter,
                                             s->gsc, rtol, 0, m, budget);
    } else {
      if (lowp)
        k_gm_start<float><<<nbv, kVT, 0, s->stream>>>(g_reorth_thr, V, nullptr, r, reinterpret_cast<float*>(s->kw),
                                                      s->red.partial, s->red.counter, s->gsc, rtol, 0, m, budget);
      else
      k_gm_start<double><<<nbv, kVT, 0, s->stream>>>(g_reorth_thr, V, left ? s->minv : nullptr, r, s->kw, s->red.partial,
                                             s->red.counter, s->gsc, rtol, 0, m, budget);
    }
    s->launches++;
    if (gg) {
      // the whole cycle on the device: one graph launch, one sync
      cudaGraphLaunch(gg->exec, s->stream);
      cudaMemcpyAsync(s->h_gsc, s->gsc, gsc_bytes, cudaMemcpyDeviceToHost, s->stream);
      host_sync(s);
      s->launches += (int64_t)gg->nodes * std::max(1, s->h_gsc->used);
    } else {
      // host-driven columns, polled every 8
      bool stop = false;
      int launched = 0;
      while (!stop && launched < m && launched < budget) {
        int chunk = std::min(8, std::min(m, budget) - launched);
        for (int c = 0; c < chunk; ++c) s->launches += gm_column(s, val, use_mg, left, tight, lowp, zb, 0, 0);
        launched += chunk;
        cudaMemcpyAsync(s->h_gsc, s->gsc, gsc_bytes, cudaMemcpyDeviceToHost, s->stream);
        host_sync(s);
        stop = s->h_gsc->done || !s->h_gsc->active;
      }
    }
    const GmresScalars* hg = s->h_gsc;
    const int used = hg->used;
    *iters += used;
    total = *iters;
    if (used > 0) {
      // back substitution H[:used,:used] y = g[:used]; x += (M^-1) V y
      double y[kMaxRestart];
      for (int i = used - 1; i >= 0; --i) {
        double acc = hg->g[i];
        for (int k = i + 1; k < used; ++k) acc -= hg->H[(size_t)k * kGM1 + i] * y[k];
        y[i] = acc / hg->H[(size_t)i * kGM1 + i];
      }
      cudaMemcpyAsync(y_dev, y, sizeof(double) * used, cudaMemcpyHostToDevice, s->stream);
      if (zb) k_gm_combine<double><<<nbg, kGT, 0, s->stream>>>(n, used, y_dev, s->gm_Z, ld, x, 1);
      else if (lowp) k_gm_combine<float><<<nbg, kGT, 0, s->stream>>>(n, used, y_dev, reinterpret_cast<const float*>(Vb), ld, t, 0);
      else k_gm_combine<double><<<nbg, kGT, 0, s->stream>>>(n, used, y_dev, Vb, ld, left ? x : t, left ? 1 : 0);
      if (left || zb) {
      } else if (use_mg) {
        mg_apply(s, val, t, z, nullptr);
        launch_axpy_to(s, x, x, 1.0, z);
      } else {
        k_minv_axpy<<<grid_for(V, 256), 256, 0, s->stream>>>(V, s->minv, t, x);
      }
      s->launches += 2;
    }
    rel = true_relres(s, val, b, x, r, bnorm);
    have_rel = true;
    if (rel <= rtol) break;
    if (used == 0) break;
    // a cycle that gains less than min_cycle_gain (inexact Newton use), or
    // nothing at all (linsolve.py:187-188), means GMRES(m) is stagnating:
    // lengthen the cycle (restarting discards the Krylov space that an
    // indefinite operator needs), and return the best iterate once the
    // cycle is at its cap
    const bool stalled = (rel >= cycle_start * (1.0 - 1e-12)) ||
                         (min_cycle_gain > 0.0 && rel > cycle_start / min_cycle_gain);
    if (stalled) {
      if (m >= m_cap) break;
      m = std::min(m_cap, 4 * m);
    }
  }
  *relres = rel;
  return rel <= rtol ? 0 : 1;
}

// ---------------------------------------------------------------------------
// PCG with the multigrid V-cycle as preconditioner (symmetric operators).
// Device-resident scalars; the host only polls `done` every few iterations.

// Three launches per iteration besides the V-cycle's own (round 2; the
// round-1 loop had V-cycle + rz + p + spmv + xr):
//   V-cycle    z = M r; its last fine sweep also forms gamma = (r, z) and
//              beta (k_mg_smooth<..., DOT>, mg_set_pcg_dot)
//   spmv_p     p' = z + beta p evaluated on the fly in the gathers (each row
//              also writes its own p'), q = A p', delta = (p', q), alpha;
//              FP32 operator copy for the inexact Newton solves
//   xr_j0      x += alpha p', r -= alpha q, rho = |r|^2 -> done; and the
//              next V-cycle's first fine Jacobi sweep x0 = omega Minv32 r
// p is double-buffered (p' never overwrites a p another warp still gathers).

__device__ __forceinline__ void minv32_apply(const float* __restrict__ minv, int V, int i, const double r[3],
                                             double u[3]) {
  u[0] = minv[0 * (size_t)V + i] * r[0] + minv[1 * (size_t)V + i] * r[1] + minv[2 * (size_t)V + i] * r[2];
  u[1] = minv[3 * (size_t)V + i] * r[0] + minv[4 * (size_t)V + i] * r[1] + minv[5 * (size_t)V + i] * r[2];
  u[2] = minv[6 * (size_t)V + i] * r[0] + minv[7 * (size_t)V + i] * r[1] + minv[8 * (size_t)V + i] * r[2];
}

// x = 0, r = b, p = 0, rho = |b|^2 (tolerances); xa = omega Minv32 b (the
// first V-cycle's fine Jacobi sweep from zero) when xa != nullptr
__global__ void __launch_bounds__(kVT) k_pcg_init(int V, const double* __restrict__ b, double* x, double* r, double* p,
                                                  double rtol, double* partial, unsigned int* counter,
                                                  KrylovScalars* ks, const float* __restrict__ minv32, double omega,
                                                  double* __restrict__ xa, int maxit) {
  __shared__ double sh[32];
  __shared__ double out[1];
  const int i = blockIdx.x * kVT + threadIdx.x;
  double acc = 0.0;
  if (i < V) {
    double rr[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double v = b[3 * i + c];
      x[3 * i + c] = 0.0; p[3 * i + c] = 0.0; r[3 * i + c] = v;
      rr[c] = v;
      acc += v * v;
    }
    if (xa) {
      double u[3];
      minv32_apply(minv32, V, i, rr, u);
      xa[3 * i] = omega * u[0]; xa[3 * i + 1] = omega * u[1]; xa[3 * i + 2] = omega * u[2];
    }
  }
  double t = block_sum<kVT>(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block(counter)) {
    fold_partials<kVT, 1>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) {
      ks->bnorm2 = out[0];
      ks->rho = out[0];
      ks->tol2 = rtol * rtol * out[0];
      ks->gamma = 0.0; ks->beta = 0.0; ks->alpha = 0.0;
      ks->iters = 0;
      ks->maxit = maxit;
      ks->done = (out[0] == 0.0) ? 1 : 0;
      *counter = 0;
    }
  }
}

// graph loop control: continue while not done and within the budget
__global__ void k_pcg_loopctl(const KrylovScalars* ks, cudaGraphConditionalHandle handle) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  cudaGraphSetConditional(handle, (!ks->done && ks->iters < ks->maxit) ? 1u : 0u);
}

// gamma' = (r, z); beta = gamma'/gamma (0 on the first iteration): the
// stand-alone form of the reduction k_mg_smooth<..., DOT> fuses, for fine
// levels too small for the one-warp-per-slice smoother (mg_pcg_rz)
__global__ void __launch_bounds__(kVT) k_pcg_rz(int V, const double* __restrict__ r, const double* __restrict__ z,
                                                double* partial, unsigned int* counter, KrylovScalars* ks) {
  __shared__ double sh[32];
  __shared__ double out[1];
  if (ldflag(&ks->done)) return;
  const int i = blockIdx.x * kVT + threadIdx.x;
  double acc = 0.0;
  if (i < V) acc = r[3 * i] * z[3 * i] + r[3 * i + 1] * z[3 * i + 1] + r[3 * i + 2] * z[3 * i + 2];
  double t = block_sum<kVT>(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block(counter)) {
    fold_partials<kVT, 1>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) {
      const double g = out[0];
      ks->beta = (ks->iters == 0) ? 0.0 : g / ks->gamma;
      ks->gamma = g;
      if (!(g > 0.0)) ks->done = 2;     // preconditioner not SPD on this residual
      *counter = 0;
    }
  }
}

void launch_pcg_rz(dp_scene* s, const double* r, const double* z, double* partial, unsigned int* counter,
                   KrylovScalars* ks) {
  k_pcg_rz<<<grid_for(s->V, kVT), kVT, 0, s->stream>>>(s->V, r, z, partial, counter, ks);
  s->launches++;
}

// p' = z + beta p (rows gathered on the fly, own row written); q = A p';
// delta = (p', q); alpha = gamma / delta
template <class TV, int BULK = 0>
__global__ void __launch_bounds__(256) k_pcg_spmv_p(int V, int S, const int* __restrict__ slice_base,
                                                    const int* __restrict__ slice_width, const int* __restrict__ col,
                                                    const TV* __restrict__ val, const double* __restrict__ z,
                                                    const double* __restrict__ p_old, double* __restrict__ p_new,
                                                    double* __restrict__ q, double* partial, unsigned int* counter,
                                                    KrylovScalars* ks) {
  __shared__ double sh[32];
  __shared__ double out[1];
  if (ldflag(&ks->done)) return;
  const double beta = ks->beta;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  double pq = 0.0;
  if (gw < S) {
    const int base = slice_base[gw];
    const int K = slice_width[gw];
    const TV* vs = val + (size_t)base * 9 + lane;
    const int* cs = col + base + lane;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    if constexpr (BULK > 0 && sizeof(TV) == 4) {
      // slots streamed through a per-warp shared-memory ring filled by TMA
      // bulk copies (as the fine smoother); same values, same order
      __shared__ __align__(128) float sv[8][BULK][9 * kSlice];
      __shared__ __align__(128) int sc[8][BULK][kSlice];
      __shared__ __align__(8) uint64_t mb[8][BULK];
      const int w = threadIdx.x >> 5;
      const float* gv = reinterpret_cast<const float*>(val) + (size_t)base * 9;
      const int* gc = col + base;
      if (lane == 0) {
#pragma unroll
        for (int d = 0; d < BULK; ++d) mbar_init(&mb[w][d], 1);
        mbar_fence_init();
      }
      __syncwarp();
      auto issue = [&](int kk) {
        if (kk < K && lane == 0) {
          const int d = kk % BULK;
          mbar_expect_tx(&mb[w][d], (9 + 1) * kSlice * 4);
          bulk_g2s(sv[w][d], gv + (size_t)kk * 9 * kSlice, 9 * kSlice * 4, &mb[w][d]);
          bulk_g2s(sc[w][d], gc + (size_t)kk * kSlice, kSlice * 4, &mb[w][d]);
        }
      };
#pragma unroll
      for (int kk = 0; kk < BULK; ++kk) issue(kk);
      for (int k = 0; k < K; ++k) {
        const int d = k % BULK;
        mbar_wait(&mb[w][d], (uint32_t)((k / BULK) & 1));
        const float* vv = sv[w][d];
        const int j = sc[w][d][lane];
        const double x0 = __ldg(z + 3 * j) + beta * __ldg(p_old + 3 * j);
        const double x1 = __ldg(z + 3 * j + 1) + beta * __ldg(p_old + 3 * j + 1);
        const double x2 = __ldg(z + 3 * j + 2) + beta * __ldg(p_old + 3 * j + 2);
        a0 += (double)vv[0 * kSlice + lane] * x0 + (double)vv[1 * kSlice + lane] * x1 +
              (double)vv[2 * kSlice + lane] * x2;
        a1 += (double)vv[3 * kSlice + lane] * x0 + (double)vv[4 * kSlice + lane] * x1 +
              (double)vv[5 * kSlice + lane] * x2;
        a2 += (double)vv[6 * kSlice + lane] * x0 + (double)vv[7 * kSlice + lane] * x1 +
              (double)vv[8 * kSlice + lane] * x2;
        __syncwarp();
        issue(k + BULK);
      }
    } else
#pragma unroll 2
    for (int k = 0; k < K; ++k) {
      const int j = __ldg(cs + k * kSlice);
      const TV* v = vs + k * 9 * kSlice;
      const double x0 = __ldg(z + 3 * j) + beta * __ldg(p_old + 3 * j);
      const double x1 = __ldg(z + 3 * j + 1) + beta * __ldg(p_old + 3 * j + 1);
      const double x2 = __ldg(z + 3 * j + 2) + beta * __ldg(p_old + 3 * j + 2);
      a0 += (double)__ldcs(v + 0 * kSlice) * x0 + (double)__ldcs(v + 1 * kSlice) * x1 +
            (double)__ldcs(v + 2 * kSlice) * x2;
      a1 += (double)__ldcs(v + 3 * kSlice) * x0 + (double)__ldcs(v + 4 * kSlice) * x1 +
            (double)__ldcs(v + 5 * kSlice) * x2;
      a2 += (double)__ldcs(v + 6 * kSlice) * x0 + (double)__ldcs(v + 7 * kSlice) * x1 +
            (double)__ldcs(v + 8 * kSlice) * x2;
    }
    const int row = gw * kSlice + lane;
    if (row < V) {
      const double p0 = __ldg(z + 3 * row) + beta * __ldg(p_old + 3 * row);
      const double p1 = __ldg(z + 3 * row + 1) + beta * __ldg(p_old + 3 * row + 1);
      const double p2 = __ldg(z + 3 * row + 2) + beta * __ldg(p_old + 3 * row + 2);
      p_new[3 * row] = p0; p_new[3 * row + 1] = p1; p_new[3 * row + 2] = p2;
      q[3 * row] = a0; q[3 * row + 1] = a1; q[3 * row + 2] = a2;
      pq = a0 * p0 + a1 * p1 + a2 * p2;
    }
  }
  double t = block_sum<256>(pq, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block(counter)) {
    fold_partials<256, 1>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) {
      if (!(out[0] > 0.0)) ks->done = 2;   // p^T A p <= 0 (linsolve.py:89-91)
      else ks->alpha = ks->gamma / out[0];
      ks->delta = out[0];
      *counter = 0;
    }
  }
}

// x += alpha p ; r -= alpha q ; rho = |r|^2 ; done when rho <= tol^2 |b|^2;
// xa = omega Minv32 r (next V-cycle's first fine Jacobi sweep)
__global__ void __launch_bounds__(kVT) k_pcg_xr_j0(int V, double* x, double* r, const double* __restrict__ p,
                                                   const double* __restrict__ q, const float* __restrict__ minv32,
                                                   double omega, double* __restrict__ xa, double* partial,
                                                   unsigned int* counter, KrylovScalars* ks) {
  __shared__ double sh[32];
  __shared__ double out[1];
  if (ldflag(&ks->done)) return;
  const double alpha = ks->alpha;
  const int i = blockIdx.x * kVT + threadIdx.x;
  double acc = 0.0;
  if (i < V) {
    double rr[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int k = 3 * i + c;
      x[k] += alpha * p[k];
      const double v = r[k] - alpha * q[k];
      r[k] = v;
      rr[c] = v;
      acc += v * v;
    }
    double u[3];
    minv32_apply(minv32, V, i, rr, u);
    xa[3 * i] = omega * u[0]; xa[3 * i + 1] = omega * u[1]; xa[3 * i + 2] = omega * u[2];
  }
  double t = block_sum<kVT>(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block(counter)) {
    fold_partials<kVT, 1>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) {
      ks->rho = out[0];
      ks->iters += 1;
      if (out[0] <= ks->tol2) ks->done = 1;
      *counter = 0;
    }
  }
}

static const int g_pcg_fp32 = getenv("DP_PCG_FP32") ? atoi(getenv("DP_PCG_FP32")) : 1;

int pcg_mg_solve_impl(dp_scene* s, const double* val, const double* b, double* x, double rtol, int max_iter,
                      int* iters, double* relres, int* breakdown, int fp32, const double* x0);

// CG needs a symmetric preconditioner: force the symmetric V(nu,nu) cycle.
// fp32: apply the operator from its FP32 copy inside the iteration (inexact
// Newton solves: the operator's 1e-7 relative rounding is far below the
// forcing term; the true residual that ends the solve is FP64)
int pcg_mg_solve(dp_scene* s, const double* val, const double* b, double* x, double rtol, int max_iter, int* iters,
                 double* relres, int* breakdown, int fp32, const double* x0) {
  mg_set_symmetric(s, 1);
  mg_set_pcg_dot(s, s->red.partial, s->red.counter, s->ksc);
  const int rc = pcg_mg_solve_impl(s, val, b, x, rtol, max_iter, iters, relres, breakdown,
                                   fp32 && g_pcg_fp32 && s->val32 != nullptr && s->val32_src == val, x0);
  mg_set_pcg_dot(s, nullptr, nullptr, nullptr);
  mg_set_symmetric(s, 0);
  return rc;
}

// one PCG iteration (V-cycle, fused p-update SpMV, fused x/r update + the
// next V-cycle's first Jacobi sweep) reading p from pin and writing pout
static void pcg_iteration(dp_scene* s, const double* val, int fp32, const double* pin, double* pout,
                          const float* minv32, double omega, double* xa) {
  const int V = s->V;
  const int nbv = grid_for(V, kVT);
  const int nbs = grid_for((int64_t)s->S * 32, 256);
  double *r = s->kr, *z = s->ku, *q = s->kw, *xc = s->kx;
  mg_apply_prejac(s, val, r, z, &s->ksc->done);
  ktm_begin(s, KT_PCG_SPMV);
  if (fp32) {
    if (g_spmv_bulk)
      k_pcg_spmv_p<float, 2><<<nbs, 256, 0, s->stream>>>(V, s->S, s->slice_base, s->slice_width, s->col, s->val32, z,
                                                         pin, pout, q, s->red.partial, s->red.counter, s->ksc);
    else
      k_pcg_spmv_p<float><<<nbs, 256, 0, s->stream>>>(V, s->S, s->slice_base, s->slice_width, s->col, s->val32, z,
                                                      pin, pout, q, s->red.partial, s->red.counter, s->ksc);
  } else {
    k_pcg_spmv_p<double><<<nbs, 256, 0, s->stream>>>(V, s->S, s->slice_base, s->slice_width, s->col, val, z, pin,
                                                     pout, q, s->red.partial, s->red.counter, s->ksc);
  }
  ktm_end(s, KT_PCG_SPMV);
  k_pcg_xr_j0<<<nbv, kVT, 0, s->stream>>>(V, xc, r, pout, q, minv32, omega, xa, s->red.partial, s->red.counter,
                                          s->ksc);
  s->launches += 2;
}

// Device-driven PCG loop: a CUDA graph whose WHILE node runs two iterations
// (the two p-buffer parities) per pass until done or the budget is spent, so
// a whole inexact Newton solve is one graph launch and one host sync.
static GmGraph* pcg_graph(dp_scene* s, const double* val, int fp32) {
  const uint64_t key = (uint64_t)(uintptr_t)val ^ ((uint64_t)fp32 << 6) ^ (1ull << 7);
  for (auto& e : s->gm_graphs)
    if (e.first == key) return (GmGraph*)e.second;
  std::lock_guard<std::recursive_mutex> api_lock(api_mutex());
  const float* minv32 = nullptr;
  double* xa = nullptr;
  double omega = 0.0;
  mg_fine_jacobi0_target(s, &minv32, &xa, &omega);
  cudaGraph_t g = nullptr;
  if (cudaGraphCreate(&g, 0) != cudaSuccess) return nullptr;
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) {
    cudaGraphDestroy(g);
    return nullptr;
  }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, g, nullptr, 0, &cp) != cudaSuccess) {
    cudaGraphDestroy(g);
    return nullptr;
  }
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  const int64_t launches0 = s->launches;
  if (cudaStreamBeginCaptureToGraph(s->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
      cudaSuccess) {
    cudaGraphDestroy(g);
    return nullptr;
  }
  const int timing_saved = s->timing;   // no timing events inside a captured graph
  s->timing = 0;
  pcg_iteration(s, val, fp32, s->kp, s->ks, minv32, omega, xa);
  pcg_iteration(s, val, fp32, s->ks, s->kp, minv32, omega, xa);
  k_pcg_loopctl<<<1, 32, 0, s->stream>>>(s->ksc, h);
  s->launches++;
  s->timing = timing_saved;
  cudaGraph_t captured = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(s->stream, &captured);
  const int nodes = (int)(s->launches - launches0);
  s->launches = launches0;
  GmGraph* gg = new GmGraph();
  if (ce != cudaSuccess || cudaGraphInstantiate(&gg->exec, g, 0) != cudaSuccess) {
    cudaGetLastError();
    cudaGraphDestroy(g);
    delete gg;
    return nullptr;
  }
  cudaGraphDestroy(g);
  gg->nodes = nodes;
  s->gm_graphs.push_back({key, (void*)gg});
  return gg;
}

int pcg_mg_solve_impl(dp_scene* s, const double* val, const double* b, double* x, double rtol, int max_iter,
                      int* iters, double* relres, int* breakdown, int fp32, const double* x0) {
  const int V = s->V, n = 3 * V;
  const int nbv = grid_for(V, kVT);
  const int nbs = grid_for((int64_t)s->S * 32, 256);
  *iters = 0;
  *breakdown = 0;
  // |b| comes back with the first sync of the solve (no sync of its own);
  // a zero rhs runs no iteration (the stop test holds at init) and returns
  // x = 0 once |b| is known
  norm2_async(s, b, &s->h_aux[0]);
  double bnorm = -1.0;
  const float* minv32 = nullptr;
  double* xa = nullptr;
  double omega = 0.0;
  mg_fine_jacobi0_target(s, &minv32, &xa, &omega);
  double* bb = s->tmp;     // rhs of the current correction solve
  double* xc = s->kx;
  double *r = s->kr, *z = s->ku, *q = s->kw;
  double* pb[2] = {s->kp, s->ks};
  double rel = 1.0;
  bool guess = false;
  if (x0) {
    // initial guess: solve A e = b - A x0 for the correction; keep it only
    // when it reduces the residual (else start from zero)
    launch_spmv(s, val, x0, bb);
    launch_axpy_to(s, bb, b, -1.0, bb);
    const double rg = sqrt(device_norm2(s, bb));   // this sync also brings |b|
    bnorm = sqrt(s->h_aux[0]);
    if (bnorm == 0.0) {
      cudaMemsetAsync(x, 0, sizeof(double) * n, s->stream);
      *relres = 0.0;
      return 0;
    }
    rel = rg / bnorm;
    guess = rel < 1.0;
    if (guess) cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, s->stream);
    else rel = 1.0;
    if (guess && rel <= rtol) {
      *relres = rel;
      return 0;
    }
  }
  if (!guess) {
    cudaMemsetAsync(x, 0, sizeof(double) * n, s->stream);
    cudaMemcpyAsync(bb, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s->stream);
  }
  for (int restart = 0; restart < 6; ++restart) {
    double inner = rtol / rel * 0.5;
    inner = fmin(0.5, fmax(inner, 1e-15));
    // FP32 operator inside the iteration: a pass cannot push the FP64 true
    // residual below ~1e-7 of its start (operator rounding), so each pass
    // stops at 1e-5 and the outer loop (FP64 true residual, corrected rhs)
    // refines - mixed-precision iterative refinement for tight solves
    if (fp32) inner = fmax(inner, 1e-5);
    int par = 0;
    k_pcg_init<<<nbv, kVT, 0, s->stream>>>(V, bb, xc, r, pb[0], inner, s->red.partial, s->red.counter, s->ksc, minv32,
                                           omega, xa, max_iter - *iters);
    s->launches++;
    int done = 0, launched = 0, chunk = 4;
    bool fused = false;   // Krylov scalars and the true residual came back in one sync
    GmGraph* gg = (g_use_graphs && !s->timing) ? pcg_graph(s, val, fp32) : nullptr;
    if (gg) {
      // the whole solve on the device: one graph launch, then x += xc and the
      // FP64 true residual queued behind it, one sync for all of it
      cudaGraphLaunch(gg->exec, s->stream);
      cudaMemcpyAsync(s->h_ksc, s->ksc, sizeof(KrylovScalars), cudaMemcpyDeviceToHost, s->stream);
      launch_axpy_to(s, x, x, 1.0, xc);
      true_relres_launch(s, val, b, x, bb);   // bb == s->tmp (the breakdown branch's buffer too)
      host_sync(s);
      done = 1;
      fused = true;
      s->launches += (int64_t)(gg->nodes / 2) * std::max(1, s->h_ksc->iters);
    }
    while (!done && *iters + launched < max_iter) {
      int m = chunk;
      if (*iters + launched + m > max_iter) m = max_iter - *iters - launched;
      for (int k = 0; k < m; ++k) {
        mg_apply_prejac(s, val, r, z, &s->ksc->done);
        ktm_begin(s, KT_PCG_SPMV);
        if (fp32) {
          if (g_spmv_bulk)
            k_pcg_spmv_p<float, 2><<<nbs, 256, 0, s->stream>>>(V, s->S, s->slice_base, s->slice_width, s->col,
                                                               s->val32, z, pb[par], pb[par ^ 1], q, s->red.partial,
                                                               s->red.counter, s->ksc);
          else
            k_pcg_spmv_p<float><<<nbs, 256, 0, s->stream>>>(V, s->S, s->slice_base, s->slice_width, s->col, s->val32,
                                                            z, pb[par], pb[par ^ 1], q, s->red.partial, s->red.counter,
                                                            s->ksc);
        } else {
          k_pcg_spmv_p<double><<<nbs, 256, 0, s->stream>>>(V, s->S, s->slice_base, s->slice_width, s->col, val, z,
                                                           pb[par], pb[par ^ 1], q, s->red.partial, s->red.counter,
                                                           s->ksc);
        }
        ktm_end(s, KT_PCG_SPMV);
        k_pcg_xr_j0<<<nbv, kVT, 0, s->stream>>>(V, xc, r, pb[par ^ 1], q, minv32, omega, xa, s->red.partial,
                                                s->red.counter, s->ksc);
        par ^= 1;
        s->launches += 2;
      }
      launched += m;
      read_ksc(s);
      done = s->h_ksc->done;
      if (chunk < 16) chunk *= 2;
    }
    *iters += s->h_ksc->iters;
    if (bnorm < 0.0) {   // first pass: |b| arrived with its sync
      bnorm = sqrt(s->h_aux[0]);
      if (bnorm == 0.0) {
        cudaMemsetAsync(x, 0, sizeof(double) * n, s->stream);
        *relres = 0.0;
        return 0;
      }
    }
    if (!fused) launch_axpy_to(s, x, x, 1.0, xc);
    const double rel_f = fused ? sqrt(s->h_ksc->pad[1]) / bnorm : 0.0;
    if (s->h_ksc->done == 2) {
      *breakdown = 1;
      *relres = fused ? rel_f : true_relres(s, val, b, x, s->tmp, bnorm);
      return 2;
    }
    rel = fused ? rel_f : true_relres(s, val, b, x, bb, bnorm);
    if (rel <= rtol || *iters >= max_iter) break;
  }
  *relres = rel;
  return rel <= rtol ? 0 : 1;
}

// ---------------------------------------------------------------------------
// step prologue (core.predict core.py:392-397, _residual_scale
// forward.py:169-171) and epilogue (v = (q - q_bar)/h, forward.py:241)

__global__ void __launch_bounds__(kVT) k_predict(int V, const double* __restrict__ q_bar, const double* __restrict__ v_bar,
                                                 const double* __restrict__ mass, const double* __restrict__ fext,
                                                 int has_fext, double h, double g0, double g1, double g2,
                                                 double* __restrict__ q_hat, double* __restrict__ q,
                                                 double* partial, unsigned int* counter, EvalScalars* esc) {
  __shared__ double sh[32];
  const int i = blockIdx.x * kVT + threadIdx.x;
  double amax = 0.0;
  if (i < V) {
    const double m = mass[i];
    const double hh_minv = __dmul_rn(__dmul_rn(h, h), 1.0 / m);
    const double g[3] = {g0, g1, g2};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int k = 3 * i + c;
      const double f = __dadd_rn(has_fext ? fext[k] : 0.0, __dmul_rn(m, g[c]));
      const double qb = q_bar[k];
      const double qh = __dadd_rn(__dadd_rn(qb, __dmul_rn(h, v_bar[k])), __dmul_rn(hh_minv, f));
      // q still holds the previous step's output: a rollout continuation?
      if (q[k] != qb) esc->discont = 1;
      q_hat[k] = qh;
      q[k] = qh;
      amax = fmax(amax, fabs(m * qh));
    }
  }
  double bm = block_max<kVT>(amax, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = bm;
  if (last_block(counter)) {
    __shared__ double out[1];
    fold_partials<kVT, 1>(partial, gridDim.x, out, sh, true);
    if (threadIdx.x == 0) { esc->scale_max = out[0]; *counter = 0; }
  }
}

void launch_predict(dp_scene* s) {
  k_predict<<<grid_for(s->V, kVT), kVT, 0, s->stream>>>(s->V, s->q_bar, s->v_bar, s->mass, s->fext, s->has_fext,
                                                         s->h, s->grav[0], s->grav[1], s->grav[2], s->q_hat, s->q,
                                                         s->red.partial, s->red.counter, s->esc);
  s->launches++;
}

__global__ void k_velocity(int n, const double* q, const double* q_bar, double h, double* v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = (q[i] - q_bar[i]) / h;
}

void launch_velocity(dp_scene* s, const double* q, const double* q_bar, double* v) {
  const int n = 3 * s->V;
  k_velocity<<<grid_for(n, 256), 256, 0, s->stream>>>(n, q, q_bar, s->h, v);
  s->launches++;
}

__global__ void k_reset_eval(EvalScalars* esc) {
  esc->rmax = 0.0;
  esc->status = 0;
  esc->penetrating = 0;
  esc->asym = 0;
}

void launch_reset_eval(dp_scene* s, EvalScalars* esc) {
  k_reset_eval<<<1, 1, 0, s->stream>>>(esc);
  s->launches++;
}

// ---------------------------------------------------------------------------
// backprop_step (adjoint.py:154-219)

// per vertex: dqbar = m z - dL_dv / h + contact q_bar term; dvbar = h m z;
// dfext = h^2 z (adjoint.py:166-176, _contact_qbar_term :142-151)
__global__ void __launch_bounds__(kVT) k_bp_vertex(int V, const double* __restrict__ mass, const double* __restrict__ z,
                                                   const double* __restrict__ dL_dv, double h,
                                                   const int* __restrict__ c_count, const int* __restrict__ c_off,
                                                   const double* __restrict__ c_frame, const double* __restrict__ c_kc,
                                                   int has_contacts, double* __restrict__ dqbar,
                                                   double* __restrict__ dvbar, double* __restrict__ dfext) {
  const int i = blockIdx.x * kVT + threadIdx.x;
  if (i >= V) return;
  const double m = mass[i], h2 = h * h;
  const double zi[3] = {z[3 * i], z[3 * i + 1], z[3 * i + 2]};
  double out[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) out[c] = m * zi[c] - dL_dv[3 * i + c] / h;
  if (has_contacts) {
    const int c0 = c_off[i], cn = c_count[i];
    for (int c = c0; c < c0 + cn; ++c) {
      const double* fr = c_frame + (size_t)c * 9;
      const double* K = c_kc + (size_t)c * 9;
      double zc[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) zc[a] = fr[a * 3] * zi[0] + fr[a * 3 + 1] * zi[1] + fr[a * 3 + 2] * zi[2];
      // t = P_f^T Kc^T zc, P_f = diag(0, 1, 1)
      double t1 = K[0 * 3 + 1] * zc[0] + K[1 * 3 + 1] * zc[1] + K[2 * 3 + 1] * zc[2];
      double t2 = K[0 * 3 + 2] * zc[0] + K[1 * 3 + 2] * zc[1] + K[2 * 3 + 2] * zc[2];
#pragma unroll
      for (int a = 0; a < 3; ++a) out[a] += h2 * (fr[1 * 3 + a] * t1 + fr[2 * 3 + a] * t2);
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    dqbar[3 * i + c] = out[c];
    dvbar[3 * i + c] = h * (m * zi[c]);
    dfext[3 * i + c] = h2 * zi[c];
  }
}

// per contact: dL/dmu_friction += -h^2 k_mu . (frame z)  (adjoint.py:187-191)
__global__ void __launch_bounds__(kVT) k_bp_contacts(int C, const int* __restrict__ vtx, const double* __restrict__ frame,
                                                     const double* __restrict__ kmu, const double* __restrict__ z,
                                                     double h2, double* partial, unsigned int* counter, double* acc) {
  __shared__ double sh[32];
  __shared__ double out[1];
  const int c = blockIdx.x * kVT + threadIdx.x;
  double v = 0.0;
  if (c < C) {
    const int i = vtx[c];
    const double* fr = frame + (size_t)c * 9;
    double zc[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) zc[a] = fr[a * 3] * z[3 * i] + fr[a * 3 + 1] * z[3 * i + 1] + fr[a * 3 + 2] * z[3 * i + 2];
    v = -h2 * (kmu[3 * c] * zc[0] + kmu[3 * c + 1] * zc[1] + kmu[3 * c + 2] * zc[2]);
  }
  double t = block_sum<kVT>(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (last_block(counter)) {
    fold_partials<kVT, 1>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) { acc[0] += out[0]; *counter = 0; }
  }
}

// per binding (adjoint.py:178-184)
__global__ void k_bp_bindings(int nb, const int* __restrict__ vtx, const double* __restrict__ target,
                              const double* __restrict__ comp, const double* __restrict__ q,
                              const double* __restrict__ z, double h2, double* dEb, double* ddb) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int i = vtx[b];
  const double Eb = comp[b];
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double lam_b = -(q[3 * i + c] - target[3 * b + c]) / Eb;
    const double zb = z[3 * i + c];
    acc += zb * (-h2 * lam_b / Eb);
    ddb[3 * b + c] += h2 / Eb * zb;
  }
  dEb[b] += acc;
}

// per element (adjoint.py:193-210): base = (G z).(p - G q_new); ARAP dL/dw,
// dL/dstiffness; NH dmu, dlambda partials.
template <int NV>
__global__ void __launch_bounds__(128) k_bp_elements(const int4* __restrict__ ev, const double* __restrict__ Bm,
                                                     const double* __restrict__ w, const double* __restrict__ vol,
                                                     const int* __restrict__ model, int E, const double* __restrict__ q,
                                                     const double* __restrict__ z, const double* __restrict__ Pst,
                                                     double h2, double* __restrict__ dw, double* partial,
                                                     unsigned int* counter, double* acc) {
  constexpr int D = NV - 1;
  __shared__ double sh[32];
  __shared__ double out[3];
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  double s_stiff = 0.0, s_mu = 0.0, s_lam = 0.0;
  if (e < E) {
    const int4 vv = ev[e];
    const int vid[4] = {vv.x, vv.y, vv.z, vv.w};
    double beta[NV][D];
#pragma unroll
    for (int k = 1; k < NV; ++k)
#pragma unroll
      for (int c = 0; c < D; ++c) beta[k][c] = Bm[(size_t)((k - 1) * D + c) * E + e];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double s = 0.0;
#pragma unroll
      for (int k = 1; k < NV; ++k) s += beta[k][c];
      beta[0][c] = -s;
    }
    const double* P = Pst + (size_t)e * 27;
    double base = 0.0, gzmu = 0.0, gzlam = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        double gz = 0.0, gq = 0.0;
#pragma unroll
        for (int a = 0; a < NV; ++a) {
          gz += z[3 * (size_t)vid[a] + i] * beta[a][c];
          gq += q[3 * (size_t)vid[a] + i] * beta[a][c];
        }
        base += gz * (P[i * 3 + c] - gq);
        gzmu += gz * P[9 + i * 3 + c];
        gzlam += gz * P[18 + i * 3 + c];
      }
    if (model[e] == DP_MODEL_ARAP) {
      dw[e] += h2 * base;
      s_stiff = h2 * base * vol[e];
    } else {
      s_mu = h2 * (2.0 * vol[e] * base + w[e] * gzmu);
      s_lam = h2 * w[e] * gzlam;
    }
  }
  double t0 = block_sum<128>(s_stiff, sh);
  double t1 = block_sum<128>(s_mu, sh);
  double t2 = block_sum<128>(s_lam, sh);
  if (threadIdx.x == 0) {
    partial[3 * blockIdx.x] = t0;
    partial[3 * blockIdx.x + 1] = t1;
    partial[3 * blockIdx.x + 2] = t2;
  }
  if (last_block(counter)) {
    fold_partials<128, 3>(partial, gridDim.x, out, sh);
    if (threadIdx.x == 0) {
      acc[1] += out[0];
      acc[2] += out[1];
      acc[3] += out[2];
      *counter = 0;
    }
  }
}

void launch_backprop(dp_scene* s, const dp_cache* c, const double* z, const double* dL_dv, double* dqbar, double* dvbar,
                     double* dfext) {
  const int has_c = c->n_contacts > 0;
  k_bp_vertex<<<grid_for(s->V, kVT), kVT, 0, s->stream>>>(s->V, s->mass, z, dL_dv, s->h, s->c_count, s->c_off,
                                                          s->c_frame, s->c_kc, has_c, dqbar, dvbar, dfext);
  s->launches++;
  const double h2 = s->h * s->h;
  if (has_c) {
    k_bp_contacts<<<grid_for(c->n_contacts, kVT), kVT, 0, s->stream>>>(
        c->n_contacts, s->c_vertex, s->c_frame, s->c_kmu, z, h2, s->red.partial, s->red.counter, s->g_scal);
    s->launches++;
  }
  if (s->nb) {
    k_bp_bindings<<<grid_for(s->nb, 128), 128, 0, s->stream>>>(s->nb, s->b_vertex, s->b_target, s->b_comp, c->q_new,
                                                               z, h2, s->g_dEb, s->g_ddb);
    s->launches++;
  }
  if (s->E) {
    const int nb = grid_for(s->E, 128);
    if (s->NV == 4)
      k_bp_elements<4><<<nb, 128, 0, s->stream>>>(s->ev, s->B, s->w, s->vol, s->model, s->E, c->q_new, z, s->Pst, h2,
                                                  s->g_dw, s->red.partial, s->red.counter, s->g_scal);
    else
      k_bp_elements<3><<<nb, 128, 0, s->stream>>>(s->ev, s->B, s->w, s->vol, s->model, s->E, c->q_new, z, s->Pst, h2,
                                                  s->g_dw, s->red.partial, s->red.counter, s->g_scal);
    s->launches++;
  }
}

// ---------------------------------------------------------------------------
// batched unit kernels (dp_project_batch): project_element + proj_jacobian +
// dP_dlame for a list of F (elasticity.py:137-324)

template <int D>
__global__ void k_project_batch(int n, const double* __restrict__ F, const int* __restrict__ model,
                                const double* __restrict__ mu, const double* __restrict__ lam, double tau_rel,
                                double* sigma, double* theta, double* Wout, double* Pout, double* J, double* dPmu,
                                double* dPlam, int* status) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double Fm[3][D];
  // input F is (3, D) row-major per item
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int c = 0; c < D; ++c) Fm[i][c] = F[(size_t)e * 3 * D + i * D + c];
  double U[3][D], sig[D], V[D][D], th[D], W[D][D];
  int st = project_full<D>(Fm, model[e], mu[e], lam[e], tau_rel, U, sig, V, th, W);
  status[e] = st;
  if (st) return;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    sigma[(size_t)e * D + k] = sig[k];
    theta[(size_t)e * D + k] = th[k];
#pragma unroll
    for (int l = 0; l < D; ++l) Wout[(size_t)e * D * D + k * D + l] = W[k][l];
  }
  double dmu[D], dlm[D];
  if (model[e] == DP_MODEL_NEOHOOKEAN) nh_dtheta_dlame<D>(th, sig, mu[e], lam[e], dmu, dlm);
  else {
#pragma unroll
    for (int k = 0; k < D; ++k) dmu[k] = dlm[k] = 0.0;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double p = 0.0, pm = 0.0, pl = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        p += U[i][k] * th[k] * V[c][k];
        pm += U[i][k] * dmu[k] * V[c][k];
        pl += U[i][k] * dlm[k] * V[c][k];
      }
      Pout[(size_t)e * 3 * D + i * D + c] = p;
      dPmu[(size_t)e * 3 * D + i * D + c] = pm;
      dPlam[(size_t)e * 3 * D + i * D + c] = pl;
    }
  // dP/dF in the column-stacked basis: J[(c,i),(c',j)] = [Gt_a J G_b]_{ij}
  // with beta_a = e_c, beta_b = e_c'  ->  alpha = row c of V.
  ElemJac<D> Jm;
  make_jac<D>(U, sig, th, W, tau_rel, Jm);
  const int N = 3 * D;
#pragma unroll
  for (int c = 0; c < D; ++c)
#pragma unroll
    for (int c2 = 0; c2 < D; ++c2) {
      double aa[D], ab[D];
#pragma unroll
      for (int k = 0; k < D; ++k) { aa[k] = V[c][k]; ab[k] = V[c2][k]; }
      double blk[3][3];
      jac_block<D>(Jm, aa, ab, blk);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) J[(size_t)e * N * N + (c * 3 + i) * N + (c2 * 3 + j)] = blk[i][j];
    }
}

void launch_project_batch(int n, int d, const double* F, const int* model, const double* mu, const double* lam,
                          double tau_rel, double* sigma, double* theta, double* W, double* P, double* J, double* dPmu,
                          double* dPlam, int* status) {
  if (d == 3)
    k_project_batch<3><<<grid_for(n, 64), 64>>>(n, F, model, mu, lam, tau_rel, sigma, theta, W, P, J, dPmu, dPlam,
                                               status);
  else
    k_project_batch<2><<<grid_for(n, 64), 64>>>(n, F, model, mu, lam, tau_rel, sigma, theta, W, P, J, dPmu, dPlam,
                                               status);
}

// per-element projection export (dp_cache_get_projections)
template <int NV>
__global__ void k_export_proj(const int4* __restrict__ ev, const double* __restrict__ Bm,
                              const double* __restrict__ mu, const double* __restrict__ lam,
                              const int* __restrict__ model, int E, const double* __restrict__ q, double* sigma,
                              double* theta, double* Pout, double* energy) {
  constexpr int D = NV - 1;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int4 vv = ev[e];
  const int vid[4] = {vv.x, vv.y, vv.z, vv.w};
  double beta[NV][D];
  for (int k = 1; k < NV; ++k)
    for (int c = 0; c < D; ++c) beta[k][c] = Bm[(size_t)((k - 1) * D + c) * E + e];
  for (int c = 0; c < D; ++c) {
    double s = 0.0;
    for (int k = 1; k < NV; ++k) s += beta[k][c];
    beta[0][c] = -s;
  }
  double F[3][D];
  for (int i = 0; i < 3; ++i)
    for (int c = 0; c < D; ++c) {
      double s = 0.0;
      for (int a = 0; a < NV; ++a) s += q[3 * (size_t)vid[a] + i] * beta[a][c];
      F[i][c] = s;
    }
  double U[3][D], sig[D], V[D][D], th[D], W[D][D];
  int st = project_full<D>(F, model[e], mu[e], lam[e], 1e-6, U, sig, V, th, W);
  if (st) {
    for (int k = 0; k < D; ++k) sigma[(size_t)e * D + k] = theta[(size_t)e * D + k] = NAN;
    return;
  }
  for (int k = 0; k < D; ++k) { sigma[(size_t)e * D + k] = sig[k]; theta[(size_t)e * D + k] = th[k]; }
  for (int i = 0; i < 3; ++i)
    for (int c = 0; c < D; ++c) {
      double p = 0.0;
      for (int k = 0; k < D; ++k) p += U[i][k] * th[k] * V[c][k];
      Pout[(size_t)e * 3 * D + i * D + c] = p;
    }
  energy[e] = (model[e] == DP_MODEL_NEOHOOKEAN) ? nh_energy<D>(th, mu[e], lam[e]) : 0.0;
}

void launch_export_proj(dp_scene* s, const double* q, double* sigma, double* theta, double* P, double* energy) {
  if (!s->E) return;
  if (s->NV == 4)
    k_export_proj<4><<<grid_for(s->E, 128), 128, 0, s->stream>>>(s->ev, s->B, s->mu, s->lam, s->model, s->E, q,
                                                                  sigma, theta, P, energy);
  else
    k_export_proj<3><<<grid_for(s->E, 128), 128, 0, s->stream>>>(s->ev, s->B, s->mu, s->lam, s->model, s->E, q,
                                                                  sigma, theta, P, energy);
  s->launches++;
}

}  // namespace dp
