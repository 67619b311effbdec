// Contact kernels: detection, pullback, penetration test, per-contact
// condensation.  Compiled with -fmad=false: every fused multiply-add below is
// an explicit fma() placed where the reference's arithmetic fuses (numpy's
// 3-vector dot `n @ x` rounds as fma(a2,b2,fma(a1,b1,a0*b0)) on the CPU the
// reference runs on), everything else rounds per
// operation like the reference's scalar Python/numpy expressions, so contact
// sets are bit-exact (detect_contacts, contact.py:115-136).
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
// self-contact (SelfContact in dp_internal.h).  No FMA anywhere (this file is
// compiled -fmad=false) and every dot product is ((x0 y0 + x1 y1) + x2 y2),
// so oracle/self_contact_oracle.py reproduces pair sets and distances
// bit for bit.

__device__ __forceinline__ double sdot(const double a[3], const double b[3]) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// squared distance from p to triangle (a, b, c): Voronoi-region closest
// point (Ericson, Real-Time Collision Detection 5.1.5)
__device__ double tri_dist2(const double p[3], const double a[3], const double b[3], const double c[3]) {
  double ab[3], ac[3], ap[3], q[3];
  for (int i = 0; i < 3; ++i) { ab[i] = b[i] - a[i]; ac[i] = c[i] - a[i]; ap[i] = p[i] - a[i]; }
  const double d1 = sdot(ab, ap), d2 = sdot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) {
    for (int i = 0; i < 3; ++i) q[i] = a[i];
  } else {
    double bp[3];
    for (int i = 0; i < 3; ++i) bp[i] = p[i] - b[i];
    const double d3 = sdot(ab, bp), d4 = sdot(ac, bp);
    const double vc = d1 * d4 - d3 * d2;
    double cp[3];
    for (int i = 0; i < 3; ++i) cp[i] = p[i] - c[i];
    const double d5 = sdot(ab, cp), d6 = sdot(ac, cp);
    const double vb = d5 * d2 - d1 * d6;
    const double va = d3 * d6 - d5 * d4;
    if (d3 >= 0.0 && d4 <= d3) {
      for (int i = 0; i < 3; ++i) q[i] = b[i];
    } else if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
      const double v = d1 / (d1 - d3);
      for (int i = 0; i < 3; ++i) q[i] = a[i] + v * ab[i];
    } else if (d6 >= 0.0 && d5 <= d6) {
      for (int i = 0; i < 3; ++i) q[i] = c[i];
    } else if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
      const double w = d2 / (d2 - d6);
      for (int i = 0; i < 3; ++i) q[i] = a[i] + w * ac[i];
    } else if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
      const double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
      for (int i = 0; i < 3; ++i) q[i] = b[i] + w * (c[i] - b[i]);
    } else {
      const double denom = 1.0 / (va + vb + vc);
      const double v = vb * denom, w = vc * denom;
      for (int i = 0; i < 3; ++i) q[i] = a[i] + ab[i] * v + ac[i] * w;
    }
  }
  double d[3];
  for (int i = 0; i < 3; ++i) d[i] = p[i] - q[i];
  return sdot(d, d);
}

__device__ __forceinline__ long long cell_of(double x, double hc) { return (long long)floor(x / hc); }

__device__ __forceinline__ int cell_hash(long long cx, long long cy, long long cz, int H) {
  const unsigned long long h = (unsigned long long)(cx * 73856093LL) ^ (unsigned long long)(cy * 19349663LL) ^
                               (unsigned long long)(cz * 83492791LL);
  return (int)(h & (unsigned long long)(H - 1));
}

__device__ __forceinline__ bool in_ring(const SelfContact& sc, int v, int u) {
  for (int k = sc.adj_ptr[v]; k < sc.adj_ptr[v + 1]; ++k)
    if (sc.adj[k] == u) return true;
  return false;
}

// candidate of vertex v: the nearest non-adjacent surface triangle (at q_bar)
// to its q_bar position within radius R (distance^2 <= R^2; ties to the lower
// index), scanning the cells within ceil(R / cell) of it; -1 if none
__device__ int self_nearest(const SelfContact& sc, int v, const double x[3], double R, double* d2_out) {
  const double hc = sc.hc[0];
  const long long cx = cell_of(x[0], hc), cy = cell_of(x[1], hc), cz = cell_of(x[2], hc);
  const int k = min(4, max(1, (int)ceil(R / hc)));
  double best = R * R;
  int bt = -1;
  for (int dz = -k; dz <= k; ++dz)
    for (int dy = -k; dy <= k; ++dy)
      for (int dx = -k; dx <= k; ++dx) {
        const int h = cell_hash(cx + dx, cy + dy, cz + dz, sc.H);
        for (int j = sc.cell_start[h]; j < sc.cell_start[h + 1]; ++j) {
          const int t = sc.items[j];
          if (bt >= 0 && t == bt) continue;
          const int ia = sc.tri[3 * t], ib = sc.tri[3 * t + 1], ic = sc.tri[3 * t + 2];
          const double a[3] = {sc.qb[3 * ia], sc.qb[3 * ia + 1], sc.qb[3 * ia + 2]};
          const double b[3] = {sc.qb[3 * ib], sc.qb[3 * ib + 1], sc.qb[3 * ib + 2]};
          const double c[3] = {sc.qb[3 * ic], sc.qb[3 * ic + 1], sc.qb[3 * ic + 2]};
          const double d2 = tri_dist2(x, a, b, c);
          if (!(d2 < best || (d2 == best && (bt < 0 || t < bt)))) continue;
          if (in_ring(sc, v, ia) || in_ring(sc, v, ib) || in_ring(sc, v, ic)) continue;
          best = d2;
          bt = t;
        }
      }
  if (d2_out) *d2_out = best;
  return bt;
}

// gap of vertex v at x against its self-contact plane (valid if cand >= 0)
__device__ __forceinline__ double self_gap(const SelfContact& sc, int v, const double x[3], double n[3]) {
  n[0] = sc.pn[3 * v]; n[1] = sc.pn[3 * v + 1]; n[2] = sc.pn[3 * v + 2];
  return sdot(n, x) - sc.pd[v];
}

// per vertex, once per step (after the prediction): candidate triangle and
// its oriented plane
__global__ void k_self_candidates(SelfContact sc, int V, const double* __restrict__ q_pred, double act) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const double xb[3] = {sc.qb[3 * v], sc.qb[3 * v + 1], sc.qb[3 * v + 2]};
  const double dp[3] = {q_pred[3 * v] - xb[0], q_pred[3 * v + 1] - xb[1], q_pred[3 * v + 2] - xb[2]};
  const double R = act + sqrt(sdot(dp, dp));
  double d2 = 0.0;
  const int t = self_nearest(sc, v, xb, R, &d2);
  sc.cand[v] = t;
  sc.cd2[v] = t >= 0 ? d2 : -1.0;
  if (t < 0) return;
  const int ia = sc.tri[3 * t];
  const double a[3] = {sc.qb[3 * ia], sc.qb[3 * ia + 1], sc.qb[3 * ia + 2]};
  const double m[3] = {sc.tn[3 * t], sc.tn[3 * t + 1], sc.tn[3 * t + 2]};
  const double rel[3] = {xb[0] - a[0], xb[1] - a[1], xb[2] - a[2]};
  const double sg = sdot(m, rel) < 0.0 ? -1.0 : 1.0;
  const double n[3] = {sg * m[0], sg * m[1], sg * m[2]};
  for (int i = 0; i < 3; ++i) sc.pn[3 * v + i] = n[i];
  sc.pd[v] = sdot(n, a);
}

void launch_self_candidates(dp_scene* s, const double* q_pred) {
  if (!s->self.enabled || s->self.n_tri == 0) return;
  k_self_candidates<<<grid_for(s->V, 128), 128, 0, s->stream>>>(s->self, s->V, q_pred, s->act);
  s->launches++;
}

// per-step build at q_bar --------------------------------------------------
__global__ void k_self_radius(SelfContact sc, unsigned long long* rmax_bits) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= sc.n_tri) return;
  const int id[3] = {sc.tri[3 * t], sc.tri[3 * t + 1], sc.tri[3 * t + 2]};
  double P[3][3], c[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < 3; ++k)
    for (int i = 0; i < 3; ++i) { P[k][i] = sc.qb[3 * id[k] + i]; c[i] += P[k][i]; }
  for (int i = 0; i < 3; ++i) c[i] /= 3.0;
  double r2 = 0.0;
  for (int k = 0; k < 3; ++k) {
    double d[3] = {P[k][0] - c[0], P[k][1] - c[1], P[k][2] - c[2]};
    r2 = fmax(r2, sdot(d, d));
  }
  // normal (unit) at q_bar
  double e1[3], e2[3], nn[3];
  for (int i = 0; i < 3; ++i) { e1[i] = P[1][i] - P[0][i]; e2[i] = P[2][i] - P[0][i]; }
  nn[0] = e1[1] * e2[2] - e1[2] * e2[1];
  nn[1] = e1[2] * e2[0] - e1[0] * e2[2];
  nn[2] = e1[0] * e2[1] - e1[1] * e2[0];
  const double l = sqrt(sdot(nn, nn));
  for (int i = 0; i < 3; ++i) sc.tn[3 * t + i] = l > 0.0 ? nn[i] / l : 0.0;
  atomicMax(rmax_bits, (unsigned long long)__double_as_longlong(sqrt(r2)));   // r >= 0: bit order = value order
}

__global__ void k_self_cellsize(SelfContact sc, const unsigned long long* rmax_bits, double act) {
  // cell >= activation + largest centroid radius (and never 0)
  sc.hc[0] = fmax((__longlong_as_double((long long)*rmax_bits) + act) * 1.000001, 1e-12);
}

__global__ void k_self_count(SelfContact sc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= sc.n_tri) return;
  const double hc = sc.hc[0];
  double c[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < 3; ++k)
    for (int i = 0; i < 3; ++i) c[i] += sc.qb[3 * sc.tri[3 * t + k] + i];
  for (int i = 0; i < 3; ++i) c[i] /= 3.0;
  const int h = cell_hash(cell_of(c[0], hc), cell_of(c[1], hc), cell_of(c[2], hc), sc.H);
  sc.tcell[t] = h;
  atomicAdd(&sc.cell_fill[h], 1);
}

// exclusive scan of the H bucket counts in one CTA; cell_fill becomes the
// fill cursor (0)
__global__ void __launch_bounds__(1024) k_self_scan(SelfContact sc) {
  __shared__ int part[1024];
  const int H = sc.H, nt = blockDim.x, t = threadIdx.x;
  const int per = (H + nt - 1) / nt, lo = t * per, hi = min(H, lo + per);
  int sum = 0;
  for (int i = lo; i < hi; ++i) sum += sc.cell_fill[i];
  part[t] = sum;
  __syncthreads();
  for (int off = 1; off < nt; off <<= 1) {
    const int v = (t >= off) ? part[t - off] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int run = part[t] - sum;
  for (int i = lo; i < hi; ++i) {
    const int c = sc.cell_fill[i];
    sc.cell_start[i] = run;
    sc.cell_fill[i] = 0;
    run += c;
  }
  if (t == nt - 1) sc.cell_start[H] = part[nt - 1];
}

__global__ void k_self_fill(SelfContact sc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= sc.n_tri) return;
  const int h = sc.tcell[t];
  sc.items[sc.cell_start[h] + atomicAdd(&sc.cell_fill[h], 1)] = t;
}

void launch_self_build(dp_scene* s) {
  SelfContact& sc = s->self;
  if (!sc.enabled || sc.n_tri == 0) return;
  sc.qb = s->q_bar;
  unsigned long long* rbits = reinterpret_cast<unsigned long long*>(sc.hc + 1);
  cudaMemsetAsync(rbits, 0, sizeof(unsigned long long), s->stream);
  cudaMemsetAsync(sc.cell_fill, 0, sizeof(int) * sc.H, s->stream);
  const int nb = grid_for(sc.n_tri, 256);
  k_self_radius<<<nb, 256, 0, s->stream>>>(sc, rbits);
  k_self_cellsize<<<1, 1, 0, s->stream>>>(sc, rbits, s->act);
  k_self_count<<<nb, 256, 0, s->stream>>>(sc);
  k_self_scan<<<1, 1024, 0, s->stream>>>(sc);
  k_self_fill<<<nb, 256, 0, s->stream>>>(sc);
  s->launches += 5;
}

// ---------------------------------------------------------------------------
// pullback (forward._pullback, forward.py:63-83)
__global__ void k_pullback(int V, const ColliderSet* __restrict__ csp, double* __restrict__ q,
                           const double* __restrict__ q_bar, double margin, SelfContact sc, double act) {
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
  if (sc.enabled && sc.cand[v] >= 0) {
    // the self "collider" after the analytic ones, the HalfSpace rule
    double n[3];
    const double gap = self_gap(sc, v, x, n);
    if (gap <= 0.0) {
      double target = margin;
      if (q_bar) {
        const double xb[3] = {q_bar[3 * v], q_bar[3 * v + 1], q_bar[3 * v + 2]};
        double nb[3];
        const double gp = self_gap(sc, v, xb, nb);
        if (gp > 0.0) target = fmin(margin, gp);
      }
      target = fmax(target, 1e-12);
      const double d = target - gap;
      for (int i = 0; i < 3; ++i) x[i] = x[i] + d * n[i];
      moved = true;
    }
  }
  if (moved) { q[3 * v] = x[0]; q[3 * v + 1] = x[1]; q[3 * v + 2] = x[2]; }
}

void launch_pullback(dp_scene* s, double* q, const double* q_bar, double margin) {
  if (contact_sources(s) == 0) return;
  k_pullback<<<grid_for(s->V, 256), 256, 0, s->stream>>>(s->V, s->d_colliders, q, q_bar, margin, s->self, s->act);
  s->launches++;
}

// _any_penetration (forward.py:86-93)
__global__ void k_penetration(int V, const ColliderSet* __restrict__ csp, const double* __restrict__ q,
                              EvalScalars* esc, SelfContact sc, double act) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const ColliderSet& cs = *csp;
  const double x[3] = {q[3 * v], q[3 * v + 1], q[3 * v + 2]};
  for (int j = 0; j < cs.n; ++j) {
    double n[3];
    if (gap_normal(cs, j, x, n) <= 0.0) { esc->penetrating = 1; esc->skip = 1; return; }
  }
  if (sc.enabled && sc.cand[v] >= 0) {
    double n[3];
    if (self_gap(sc, v, x, n) <= 0.0) { esc->penetrating = 1; esc->skip = 1; }
  }
}

void launch_penetration(dp_scene* s, const double* q, EvalScalars* esc) {
  if (contact_sources(s) == 0) return;
  k_penetration<<<grid_for(s->V, 256), 256, 0, s->stream>>>(s->V, s->d_colliders, q, esc, s->self, s->act);
  s->launches++;
}

// The penetration test of every line-search trial of one search at once
// (forward.py:218-219): bit k of esc->pen_mask = some vertex of
// q + 2^-k dq has a gap <= 0.  The trial point is formed exactly as
// k_axpy_to forms it (t * dq is exact for t = 2^-k), so each bit equals
// k_penetration's verdict on that trial.
__global__ void k_penetration_mask(int V, const ColliderSet* __restrict__ csp, const double* __restrict__ q,
                                   const double* __restrict__ dq, int nls, EvalScalars* esc, SelfContact sc) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned int m = 0;
  if (v < V) {
    const ColliderSet& cs = *csp;
    const double q0 = q[3 * v], q1 = q[3 * v + 1], q2 = q[3 * v + 2];
    const double d0 = dq[3 * v], d1 = dq[3 * v + 1], d2 = dq[3 * v + 2];
    double t = 1.0;
    for (int k = 0; k < nls; ++k, t *= 0.5) {
      const double x[3] = {q0 + t * d0, q1 + t * d1, q2 + t * d2};
      bool pen = false;
      for (int j = 0; j < cs.n && !pen; ++j) {
        double n[3];
        pen = gap_normal(cs, j, x, n) <= 0.0;
      }
      if (!pen && sc.enabled && sc.cand[v] >= 0) {
        double n[3];
        pen = self_gap(sc, v, x, n) <= 0.0;
      }
      if (pen) m |= 1u << k;
    }
  }
  m = __reduce_or_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m) atomicOr(&esc->pen_mask, m);
}

void launch_penetration_mask(dp_scene* s, const double* q, const double* dq, int nls, EvalScalars* esc) {
  if (contact_sources(s) == 0) return;
  k_penetration_mask<<<grid_for(s->V, 256), 256, 0, s->stream>>>(s->V, s->d_colliders, q, dq, nls < 32 ? nls : 32,
                                                                 esc, s->self);
  s->launches++;
}

// ---------------------------------------------------------------------------
// detection: count -> exclusive scan -> write (order: vertex, then collider)
// count + the block-local exclusive scan of the counts (the grid-level
// offsets come from k_scan_blocks; no library scan on the detection path)
constexpr int kDetNT = 256;
__device__ int detect_count_one(const ColliderSet* __restrict__ csp, const double* __restrict__ q, double act,
                                const SelfContact& sc, int v);
__global__ void __launch_bounds__(kDetNT) k_detect_count(int V, const ColliderSet* __restrict__ csp,
                                                         const double* __restrict__ q, double act,
                                                         int* __restrict__ count, int* __restrict__ local_off,
                                                         int* __restrict__ blk_sum, SelfContact sc) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  int c = 0;
  if (v < V) c = detect_count_one(csp, q, act, sc, v);
  if (v <= V) count[v] = (v < V) ? c : 0;
  // block exclusive scan (warp shuffles + one smem pass)
  __shared__ int ws[kDetNT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) ws[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int t = (lane < kDetNT / 32) ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kDetNT / 32) ws[lane] = t;   // inclusive over warps
  }
  __syncthreads();
  const int wpre = (wid > 0) ? ws[wid - 1] : 0;
  if (v <= V) local_off[v] = wpre + incl - c;
  if (threadIdx.x == kDetNT - 1) blk_sum[blockIdx.x] = ws[kDetNT / 32 - 1];
}

// exclusive scan of the per-block totals in one CTA; total -> esc->n_contacts
__global__ void __launch_bounds__(1024) k_scan_blocks(int nb, int* __restrict__ blk, EvalScalars* esc) {
  __shared__ int part[1024];
  const int t = threadIdx.x, nt = blockDim.x;
  const int per = (nb + nt - 1) / nt, lo = t * per, hi = min(nb, lo + per);
  int sum = 0;
  for (int i = lo; i < hi; ++i) sum += blk[i];
  part[t] = sum;
  __syncthreads();
  for (int off = 1; off < nt; off <<= 1) {
    const int y = (t >= off) ? part[t - off] : 0;
    __syncthreads();
    part[t] += y;
    __syncthreads();
  }
  int run = part[t] - sum;
  for (int i = lo; i < hi; ++i) {
    const int c = blk[i];
    blk[i] = run;
    run += c;
  }
  if (t == nt - 1) esc->n_contacts = part[nt - 1];
}

__device__ int detect_count_one(const ColliderSet* __restrict__ csp, const double* __restrict__ q, double act,
                                const SelfContact& sc, int v) {
  const ColliderSet& cs = *csp;
  const double x[3] = {q[3 * v], q[3 * v + 1], q[3 * v + 2]};
  int c = 0;
  for (int j = 0; j < cs.n; ++j) {
    double n[3];
    if (!(gap_normal(cs, j, x, n) > act)) ++c;
  }
  if (sc.enabled && sc.cand[v] >= 0) {
    double n[3];
    if (!(self_gap(sc, v, x, n) > act)) ++c;
  }
  return c;
}

__global__ void k_detect_write(int V, const ColliderSet* __restrict__ csp, const double* __restrict__ q, double act,
                               int* __restrict__ off, const int* __restrict__ count,
                               const int* __restrict__ blk_off, int* __restrict__ cvtx, int* __restrict__ ccol,
                               double* __restrict__ cframe, double* __restrict__ cdn, double* __restrict__ cmu,
                               EvalScalars* esc, SelfContact sc) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v > V) return;
  int o = off[v] + blk_off[v / kDetNT];   // block-local exclusive offset + the block's offset
  off[v] = o;
  if (v == V || count[v] == 0) return;
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
  if (sc.enabled && sc.cand[v] >= 0) {
    // self contact: collider index n_colliders, frame from the frozen
    // triangle plane's oriented normal
    double n[3], t1[3], t2[3];
    const double gap = self_gap(sc, v, x, n);
    if (!(gap > act)) {
      tangent_basis(n, t1, t2);
      cvtx[o] = v;
      ccol[o] = cs.n;
      double* fr = cframe + (size_t)o * 9;
      for (int i = 0; i < 3; ++i) { fr[i] = n[i]; fr[3 + i] = t1[i]; fr[6 + i] = t2[i]; }
      cdn[o] = dot3(n, x) - gap;
      cmu[o] = sc.mu;
    }
  }
}

int contact_scan_setup(dp_scene* s) {
  // per-block totals of the detection scan (one int per kDetNT vertices)
  const size_t bytes = sizeof(int) * ((size_t)(s->V + 1 + kDetNT - 1) / kDetNT + 1);
  if (bytes > s->scan_tmp_bytes) {
    if (s->scan_tmp) cudaFree(s->scan_tmp);
    DP_CUDA(cudaMalloc(&s->scan_tmp, bytes));
    s->scan_tmp_bytes = bytes;
  }
  return 0;
}

void launch_detect(dp_scene* s, const double* q) {
  const int V = s->V;
  if (contact_sources(s) == 0) {
    cudaMemsetAsync(&s->esc->n_contacts, 0, sizeof(int), s->stream);
    return;
  }
  const int nb = grid_for(V + 1, kDetNT);
  int* blk = static_cast<int*>(s->scan_tmp);
  k_detect_count<<<nb, kDetNT, 0, s->stream>>>(V, s->d_colliders, q, s->act, s->c_count, s->c_off, blk, s->self);
  k_scan_blocks<<<1, 1024, 0, s->stream>>>(nb, blk, s->esc);
  k_detect_write<<<nb, kDetNT, 0, s->stream>>>(V, s->d_colliders, q, s->act, s->c_off, s->c_count, blk, s->c_vertex,
                                               s->c_collider, s->c_frame, s->c_dn, s->c_mu, s->esc, s->self);
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
  if (contact_sources(s) == 0 && n_contacts <= 0) return;
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
