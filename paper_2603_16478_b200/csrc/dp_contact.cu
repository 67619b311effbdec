// Contact kernels: detection, pullback, penetration test, per-contact
// condensation.  Compiled with -fmad=false: every fused multiply-add below is
// an explicit fma() placed where the reference's arithmetic fuses (numpy's
// 3-vector dot `n @ x` rounds as fma(a2,b2,fma(a1,b1,a0*b0)) on the CPU the
// reference runs on), everything else rounds per
// operation like the reference's scalar Python/numpy expressions, so contact
// sets are bit-exact (detect_contacts, contact.py:115-136).
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "dp_common.cuh"
#include "dp_internal.h"
#include "dp_math.cuh"

namespace dp {

__device__ __forceinline__ double dot3(const double a[3], const double b[3]) {
  return fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
}

// HalfSpace.gap_normal core.py:110-112, Sphere.gap_normal core.py:133-139
__device__ __forceinline__ double gap_normal(const ColliderSet& cs, int j, const double x[3], double n[3]) {
  if (cs.kind[j] == DP_COLLIDER_HALFSPACE) {
    n[0] = cs.vec[j][0]; n[1] = cs.vec[j][1]; n[2] = cs.vec[j][2];
    return dot3(n, x) - cs.scalar[j];
  }
  double d[3] = {x[0] - cs.vec[j][0], x[1] - cs.vec[j][1], x[2] - cs.vec[j][2]};
  const double r = sqrt(dot3(d, d));
  if (r < 1e-14) {
    n[0] = 0.0; n[1] = 0.0; n[2] = 1.0;
    return -cs.scalar[j];
  }
  n[0] = d[0] / r; n[1] = d[1] / r; n[2] = d[2] / r;
  return r - cs.scalar[j];
}

// _tangent_basis, contact.py:102-112
__device__ __forceinline__ void tangent_basis(const double n[3], double t1[3], double t2[3]) {
  const double a0 = fabs(n[0]), a1 = fabs(n[1]), a2 = fabs(n[2]);
  int k = 0;
  double best = a0;
  if (a1 < best) { best = a1; k = 1; }
  if (a2 < best) { k = 2; }
  const double nk = n[k];   // axis @ n with a unit axis is exactly n[k]
#pragma unroll
  for (int i = 0; i < 3; ++i) t1[i] = ((i == k) ? 1.0 : 0.0) - nk * n[i];
  const double nrm = sqrt(dot3(t1, t1));
#pragma unroll
  for (int i = 0; i < 3; ++i) t1[i] = t1[i] / nrm;
  t2[0] = n[1] * t1[2] - n[2] * t1[1];
  t2[1] = n[2] * t1[0] - n[0] * t1[2];
  t2[2] = n[0] * t1[1] - n[1] * t1[0];
}

// ---------------------------------------------------------------------------
// pullback (forward._pullback, forward.py:63-83)
__global__ void k_pullback(int V, const ColliderSet* __restrict__ csp, double* __restrict__ q,
                           const double* __restrict__ q_bar, double margin) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const ColliderSet& cs = *csp;
  double x[3] = {q[3 * v], q[3 * v + 1], q[3 * v + 2]};
  bool moved = false;
  for (int j = 0; j < cs.n; ++j) {
    double n[3];
    const double gap = gap_normal(cs, j, x, n);
    if (gap <= 0.0) {
      double target = margin;
      if (q_bar) {
        double xb[3] = {q_bar[3 * v], q_bar[3 * v + 1], q_bar[3 * v + 2]}, nb[3];
        const double gp = gap_normal(cs, j, xb, nb);
        if (gp > 0.0) target = fmin(margin, gp);
      }
      target = fmax(target, 1e-12);
      const double d = target - gap;
#pragma unroll
      for (int i = 0; i < 3; ++i) x[i] = x[i] + d * n[i];
      moved = true;
    }
  }
  if (moved) { q[3 * v] = x[0]; q[3 * v + 1] = x[1]; q[3 * v + 2] = x[2]; }
}

void launch_pullback(dp_scene* s, double* q, const double* q_bar, double margin) {
  if (s->colliders.n == 0) return;
  k_pullback<<<grid_for(s->V, 256), 256, 0, s->stream>>>(s->V, s->d_colliders, q, q_bar, margin);
  s->launches++;
}

// _any_penetration (forward.py:86-93)
__global__ void k_penetration(int V, const ColliderSet* __restrict__ csp, const double* __restrict__ q,
                              EvalScalars* esc) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const ColliderSet& cs = *csp;
  const double x[3] = {q[3 * v], q[3 * v + 1], q[3 * v + 2]};
  for (int j = 0; j < cs.n; ++j) {
    double n[3];
    if (gap_normal(cs, j, x, n) <= 0.0) { esc->penetrating = 1; esc->skip = 1; return; }
  }
}

void launch_penetration(dp_scene* s, const double* q, EvalScalars* esc) {
  if (s->colliders.n == 0) return;
  k_penetration<<<grid_for(s->V, 256), 256, 0, s->stream>>>(s->V, s->d_colliders, q, esc);
  s->launches++;
}

// ---------------------------------------------------------------------------
// detection: count -> exclusive scan -> write (order: vertex, then collider)
__global__ void k_detect_count(int V, const ColliderSet* __restrict__ csp, const double* __restrict__ q, double act,
                               int* __restrict__ count) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v > V) return;
  if (v == V) { count[V] = 0; return; }
  const ColliderSet& cs = *csp;
  const double x[3] = {q[3 * v], q[3 * v + 1], q[3 * v + 2]};
  int c = 0;
  for (int j = 0; j < cs.n; ++j) {
    double n[3];
    if (!(gap_normal(cs, j, x, n) > act)) ++c;
  }
  count[v] = c;
}

__global__ void k_detect_write(int V, const ColliderSet* __restrict__ csp, const double* __restrict__ q, double act,
                               const int* __restrict__ off, int* __restrict__ cvtx, int* __restrict__ ccol,
                               double* __restrict__ cframe, double* __restrict__ cdn, double* __restrict__ cmu,
                               EvalScalars* esc) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v == 0) esc->n_contacts = off[V];
  if (v >= V) return;
  int o = off[v];
  if (off[v + 1] == o) return;
  const ColliderSet& cs = *csp;
  const double x[3] = {q[3 * v], q[3 * v + 1], q[3 * v + 2]};
  for (int j = 0; j < cs.n; ++j) {
    double n[3];
    const double gap = gap_normal(cs, j, x, n);
    if (gap > act) continue;
    double t1[3], t2[3];
    tangent_basis(n, t1, t2);
    cvtx[o] = v;
    ccol[o] = j;
    double* fr = cframe + (size_t)o * 9;
#pragma unroll
    for (int i = 0; i < 3; ++i) { fr[i] = n[i]; fr[3 + i] = t1[i]; fr[6 + i] = t2[i]; }
    cdn[o] = dot3(n, x) - gap;
    cmu[o] = cs.mu[j];
    ++o;
  }
}

int contact_scan_setup(dp_scene* s) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, s->c_count, s->c_off, s->V + 1, s->stream);
  if (bytes > s->scan_tmp_bytes) {
    if (s->scan_tmp) cudaFree(s->scan_tmp);
    DP_CUDA(cudaMalloc(&s->scan_tmp, bytes));
    s->scan_tmp_bytes = bytes;
  }
  return 0;
}

void launch_detect(dp_scene* s, const double* q) {
  const int V = s->V;
  if (s->colliders.n == 0) {
    cudaMemsetAsync(&s->esc->n_contacts, 0, sizeof(int), s->stream);
    return;
  }
  k_detect_count<<<grid_for(V + 1, 256), 256, 0, s->stream>>>(V, s->d_colliders, q, s->act, s->c_count);
  size_t bytes = s->scan_tmp_bytes;
  cub::DeviceScan::ExclusiveSum(s->scan_tmp, bytes, s->c_count, s->c_off, V + 1, s->stream);
  k_detect_write<<<grid_for(V, 256), 256, 0, s->stream>>>(V, s->d_colliders, q, s->act, s->c_off, s->c_vertex,
                                                          s->c_collider, s->c_frame, s->c_dn, s->c_mu, s->esc);
  s->launches += 3;
}

// ---------------------------------------------------------------------------
// per-contact condensation (solve_multipliers contact.py:139-165 +
// contact_block :212-248).  Outputs: delta, local Kc, k_mu, global block
// h^2 fr^T Kc fr (transposed for the adjoint, adjoint.py:45-50) and the
// residual contribution -h^2 fr^T lam (forward.py:108-109).
__global__ void k_contacts(const int* __restrict__ n_ptr, int n_fixed, const double* __restrict__ q,
                           const double* __restrict__ q_bar, const int* __restrict__ vtx,
                           const double* __restrict__ frame, const double* __restrict__ dnv,
                           const double* __restrict__ muv, double eps2, double h2, int from_delta, int transpose,
                           double* __restrict__ delta, double* __restrict__ kc, double* __restrict__ kmu,
                           double* __restrict__ blk, double* __restrict__ force, EvalScalars* esc,
                           const int* __restrict__ skip) {
  if (skip && *(volatile const int*)skip) return;   // penetrating line-search trial: no evaluation
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = n_ptr ? *n_ptr : n_fixed;
  if (c >= n) return;
  const double* fr = frame + (size_t)c * 9;
  const double mu = muv[c];
  double dn, df0, df1;
  if (from_delta) {
    dn = delta[3 * c]; df0 = delta[3 * c + 1]; df1 = delta[3 * c + 2];
  } else {
    const int v = vtx[c];
    const double x[3] = {q[3 * v], q[3 * v + 1], q[3 * v + 2]};
    const double d[3] = {x[0] - q_bar[3 * v], x[1] - q_bar[3 * v + 1], x[2] - q_bar[3 * v + 2]};
    dn = dot3(fr, x) - dnv[c];                 // ContactPoint.gaps, contact.py:84-90
    df0 = dot3(fr + 3, d);
    df1 = dot3(fr + 6, d);
    delta[3 * c] = dn; delta[3 * c + 1] = df0; delta[3 * c + 2] = df1;
  }
  ContactLocal L;
  const int st = contact_local(dn, df0, df1, mu, eps2, L);
  if (st) {
    atomicOr(&esc->status, st);
    return;
  }
  if (mu != 0.0) esc->asym = 1;
#pragma unroll
  for (int i = 0; i < 9; ++i) kc[(size_t)c * 9 + i] = L.Kc[i / 3][i % 3];
#pragma unroll
  for (int i = 0; i < 3; ++i) kmu[3 * c + i] = L.kmu[i];
  // global block G = h^2 fr^T K fr (K or K^T)
  double KF[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < 3; ++b) s = fma(transpose ? L.Kc[b][a] : L.Kc[a][b], fr[b * 3 + j], s);
      KF[a][j] = s;
    }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) s = fma(fr[a * 3 + i], KF[a][j], s);
      blk[(size_t)c * 9 + i * 3 + j] = h2 * s;
    }
#pragma unroll
  for (int i = 0; i < 3; ++i)
    force[3 * c + i] = -h2 * fma(fr[6 + i], L.lam[2], fma(fr[3 + i], L.lam[1], fr[i] * L.lam[0]));
}

void launch_contacts(dp_scene* s, const double* q, const double* q_bar, int n_contacts, const int* vtx,
                     const double* frame, const double* dn, const double* mu, double* delta_out, int from_delta,
                     int transpose, EvalScalars* esc) {
  if (s->colliders.n == 0 && n_contacts <= 0) return;
  // n_contacts < 0: the count lives on device (esc->n_contacts), launch over capacity
  const int cap = n_contacts >= 0 ? n_contacts : s->ccap;
  if (cap == 0) return;
  k_contacts<<<grid_for(cap, 128), 128, 0, s->stream>>>(n_contacts >= 0 ? nullptr : &s->esc->n_contacts, n_contacts,
                                                        q, q_bar, vtx, frame, dn, mu, s->eps_fb, s->h * s->h,
                                                        from_delta, transpose, delta_out, s->c_kc, s->c_kmu, s->c_blk,
                                                        s->c_force, esc, s->eval_skip);
  s->launches++;
}

// ---------------------------------------------------------------------------
// unit batch: solve_multipliers + contact_block + contact_residual
__global__ void k_contact_batch(int n, const double* __restrict__ frame, const double* __restrict__ dnv,
                                const double* __restrict__ mu, const double* __restrict__ eps2,
                                const double* __restrict__ x, const double* __restrict__ xb, double* lam,
                                double* delta, double* s_signed, int* capped, double* Kc, double* kmu,
                                double* residual, int* status) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const double* fr = frame + (size_t)c * 9;
  const double xv[3] = {x[3 * c], x[3 * c + 1], x[3 * c + 2]};
  const double d[3] = {xv[0] - xb[3 * c], xv[1] - xb[3 * c + 1], xv[2] - xb[3 * c + 2]};
  const double dn = dot3(fr, xv) - dnv[c];
  const double df0 = dot3(fr + 3, d), df1 = dot3(fr + 6, d);
  ContactLocal L;
  const int st = contact_local(dn, df0, df1, mu[c], eps2[c], L);
  status[c] = st;
  for (int i = 0; i < 3; ++i) delta[3 * c + i] = L.delta[i];
  if (st) return;
  for (int i = 0; i < 3; ++i) { lam[3 * c + i] = L.lam[i]; kmu[3 * c + i] = L.kmu[i]; }
  for (int i = 0; i < 9; ++i) Kc[(size_t)c * 9 + i] = L.Kc[i / 3][i % 3];
  s_signed[c] = L.s;
  capped[c] = L.capped;
  double res[3];
  contact_residual_rows(L, mu[c], eps2[c], res);
  for (int i = 0; i < 3; ++i) residual[3 * c + i] = res[i];
}

void launch_contact_batch(int n, const double* frame, const double* dn, const double* mu, const double* eps2,
                          const double* x, const double* xb, double* lam, double* delta, double* s_signed, int* capped,
                          double* Kc, double* kmu, double* residual, int* status) {
  k_contact_batch<<<grid_for(n, 128), 128>>>(n, frame, dn, mu, eps2, x, xb, lam, delta, s_signed, capped, Kc, kmu,
                                             residual, status);
}

}  // namespace dp
