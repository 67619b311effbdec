// Aggregation multigrid preconditioner for the 3x3-block Newton / adjoint
// operators ("stronger preconditioners"; the
// reference offers sparse-inverse / Woodbury, linsolve.py:230-336, which the
// adjoint never calls).  B200-first design:
//
//  * setup (host, once per scene): greedy vertex aggregation of the block
//    graph, level by level, until <= kCoarseMax block rows; per level a
//    SELL-32 pattern, and a *Galerkin gather list* per coarse slot: the
//    fine SELL value addresses whose blocks sum into it (unsmoothed
//    aggregation, P = piecewise-constant 3x3 identity per aggregate, so
//    A_c = P^T A P is a pure block sum - no SpGEMM).
//  * per operator (every Newton iteration / adjoint step): one gather kernel
//    per level (deterministic, no atomics) + block-Jacobi inverses; the
//    coarsest operator is inverted densely in one CTA (Gauss-Jordan).
//  * apply (V-cycle): damped block-Jacobi pre/post smoothing, residual,
//    restriction (member gather), prolongation fused into the post-smoother's
//    SpMV gathers.  Symmetric for symmetric A (CG-safe).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "dp_common.cuh"
#include "dp_internal.h"

namespace cg = cooperative_groups;

#ifndef DP_SMOOTH_ASYNC
#define DP_SMOOTH_ASYNC 1   // fine-level smoother streams its slots through shared memory (cp.async)
#endif
#ifndef DP_SMOOTH_DEPTH
#define DP_SMOOTH_DEPTH 2
#endif
constexpr int kSmDepth = DP_SMOOTH_DEPTH;  // slots in flight per warp (fine level)
#ifndef DP_SMOOTH_DEPTHC
#define DP_SMOOTH_DEPTHC 2
#endif
constexpr int kSmDepthC = DP_SMOOTH_DEPTHC;  // slots in flight per warp (coarse levels, SPLIT = 8)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
#ifndef DP_SMOOTH_NT
#define DP_SMOOTH_NT 256   // CTA size of the fine-level smoother (one warp per slice)
#endif


namespace dp {

// fine-level smoother sweeps on an FP16 operator copy with per-block scales
// (26 instead of 40 bytes per block; the preconditioner only)
static const int g_smooth16 = getenv("DP_SMOOTH16") ? atoi(getenv("DP_SMOOTH16")) : 0;   // measured: no faster (latency-bound), off
// two coarsest levels in one cluster launch (k_mg_tail): C5 V-cycle tail 23 -> ~14 us
static const int g_mg_tail = getenv("DP_MG_TAIL") ? atoi(getenv("DP_MG_TAIL")) : 1;
static const int g_mg_agg2 = getenv("DP_MG_AGG2") ? atoi(getenv("DP_MG_AGG2")) : 0;
constexpr int kCoarseMax = 36;      // dense coarsest solve (<= 108 unknowns, shared memory)
constexpr int kDenseSmem = 108;
__global__ void k_mg_dense_invert(int N, const double* __restrict__ Ag, double* __restrict__ Ainv);
static int fused_grid_size(int device);

struct MGLevel {
  int n = 0, S = 0;
  int64_t NS = 0;
  int *slice_base = nullptr, *slice_width = nullptr, *col = nullptr, *diag_slot = nullptr;
  double *val = nullptr, *minv = nullptr;
  int *gal_ptr = nullptr, *gal = nullptr;      // coarse slot -> fine value addresses
  int *mem_ptr = nullptr, *mem = nullptr;      // coarse row -> fine rows
  int* agg = nullptr;                          // fine row -> coarse row (owned by the coarse level)
  int* slot_row = nullptr;                     // SELL slot -> block row
  int kmax = 0;                                // widest slice (slots per row)
  double *x = nullptr, *b = nullptr, *r = nullptr, *t = nullptr, *u = nullptr;
};

struct MG {
  std::vector<MGLevel> lv;   // lv[0] = fine level (aliases the scene's SELL arrays)
  double* dense = nullptr;   // coarsest dense operator (N x N), N = 3 n_coarsest
  double* dinv = nullptr;    // its inverse
  int N = 0;
  double omega = 0.8;
  double alpha = 1.5;        // coarse-correction scaling (over-correction for UA)
  double alpha_gm = 1.5;     // ... for the GMRES (non-symmetric / friction) solves
  double alpha_cg = 1.8;     // ... for the PCG solves (measured: C5 +8%; C1-C4 GMRES lose with 1.8)
  int nu = 1;
  int post = 1;               // post-smoothing sweeps on (1) / off (0, non-symmetric use only)
  int gamma = 1;              // coarse-grid corrections per visit below the fine level (2 = W-cycle)
  int coarse_sweeps = 4;      // >0: Jacobi sweeps at the coarsest level instead of the dense inverse
  int symmetric_needed = 0;  // set while a CG solve uses the V-cycle
  int fused = 1;              // coarse levels in one cooperative kernel (k_mg_coarse_fused)
  int prejac = 0;             // fine-level jacobi0 already applied by the caller
  // PCG fusion: the fine level's last post-smoothing sweep also forms
  // (r, z) and the CG beta (k_mg_smooth<..., DOT>) when dot_ks is set
  double* dot_partial = nullptr;
  unsigned int* dot_counter = nullptr;
  KrylovScalars* dot_ks = nullptr;
  int fused_grid = 0;
  size_t bytes = 0;
};

// ---------------------------------------------------------------------------
// host setup

struct HostPattern {
  int n = 0;
  std::vector<int> rowptr, col;
};

static void sell_layout(const HostPattern& P, std::vector<int>& slice_base, std::vector<int>& slice_width,
                        std::vector<int>& col, std::vector<int>& diag_slot, std::vector<int64_t>& slot_of) {
  const int n = P.n, S = (n + kSlice - 1) / kSlice;
  slice_base.assign(S + 1, 0);
  slice_width.assign(S, 0);
  for (int sl = 0; sl < S; ++sl) {
    int K = 0;
    for (int l = 0; l < kSlice; ++l) {
      const int row = sl * kSlice + l;
      if (row < n) K = std::max(K, P.rowptr[row + 1] - P.rowptr[row]);
    }
    slice_width[sl] = K;
    slice_base[sl + 1] = slice_base[sl] + K * kSlice;
  }
  col.assign(slice_base[S], 0);
  diag_slot.assign(n, 0);
  slot_of.assign(P.col.size(), 0);
  for (int i = 0; i < n; ++i) {
    const int sl = i / kSlice, l = i % kSlice;
    for (int k = P.rowptr[i]; k < P.rowptr[i + 1]; ++k) {
      const int64_t slot = slice_base[sl] + (int64_t)(k - P.rowptr[i]) * kSlice + l;
      col[slot] = P.col[k];
      slot_of[k] = slot;
      if (P.col[k] == i) diag_slot[i] = (int)slot;
    }
  }
}

// greedy aggregation (standard two-phase): returns #aggregates, agg[i]
static int aggregate(const HostPattern& P, std::vector<int>& agg) {
  const int n = P.n;
  agg.assign(n, -1);
  int na = 0;
  for (int i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    bool free_nbhd = true;
    for (int k = P.rowptr[i]; k < P.rowptr[i + 1]; ++k)
      if (agg[P.col[k]] >= 0) { free_nbhd = false; break; }
    if (!free_nbhd) continue;
    for (int k = P.rowptr[i]; k < P.rowptr[i + 1]; ++k) agg[P.col[k]] = na;
    agg[i] = na;
    ++na;
  }
  // phase 2: attach leftovers to the neighbouring aggregate they touch most
  std::vector<int> tmp = agg;
  for (int i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    int best = -1, bestc = 0;
    for (int k = P.rowptr[i]; k < P.rowptr[i + 1]; ++k) {
      const int a = agg[P.col[k]];
      if (a < 0) continue;
      int c = 0;
      for (int k2 = P.rowptr[i]; k2 < P.rowptr[i + 1]; ++k2) c += (agg[P.col[k2]] == a);
      if (c > bestc) { bestc = c; best = a; }
    }
    tmp[i] = best;
  }
  agg = tmp;
  for (int i = 0; i < n; ++i)
    if (agg[i] < 0) {
      agg[i] = na++;
      for (int k = P.rowptr[i]; k < P.rowptr[i + 1]; ++k)
        if (agg[P.col[k]] < 0) agg[P.col[k]] = agg[i];
    }
  return na;
}

template <class T>
static int up(MG* mg, T** p, const std::vector<T>& h) {
  const size_t n = std::max<size_t>(h.size(), 1);
  DP_CUDA(cudaMalloc((void**)p, n * sizeof(T)));
  mg->bytes += n * sizeof(T);
  if (!h.empty()) DP_CUDA(cudaMemcpy(*p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return 0;
}
template <class T>
static int al(MG* mg, T** p, size_t n) {
  n = std::max<size_t>(n, 1);
  DP_CUDA(cudaMalloc((void**)p, n * sizeof(T)));
  mg->bytes += n * sizeof(T);
  DP_CUDA(cudaMemset(*p, 0, n * sizeof(T)));
  return 0;
}

int mg_setup(dp_scene* s) {
  MG* mg = new MG();
  HostPattern fine;
  fine.n = s->V;
  fine.rowptr = s->h_rowptr;
  fine.col = s->h_colidx;
  // fine level aliases the scene's SELL storage
  MGLevel L0;
  L0.n = s->V;
  L0.S = s->S;
  L0.NS = s->NS;
  L0.slice_base = s->slice_base;
  L0.slice_width = s->slice_width;
  L0.col = s->col;
  L0.diag_slot = s->diag_slot;
  L0.minv = s->minv;
  int rc = 0;
  // mixed-precision preconditioner: the fine-level V-cycle reads FP32 copies
  // of the operator (written by k_assemble); the Krylov method itself runs on
  // the FP64 operator, so the solution accuracy is unaffected
  rc |= al(mg, &s->val32, (size_t)s->NS * kVal32PerSlot);
  rc |= al(mg, &s->minv32, (size_t)s->V * 9);
  if (g_smooth16 && s->S >= 4 * 148 && DP_VAL32_PACKED == 0) {
    rc |= al(mg, &s->val16, (size_t)s->NS * 9);
    rc |= al(mg, &s->sc16, (size_t)s->NS);
  }
  rc |= al(mg, &L0.x, (size_t)3 * s->V);
  rc |= al(mg, &L0.r, (size_t)3 * s->V);
  rc |= al(mg, &L0.t, (size_t)3 * s->V);
  rc |= al(mg, &L0.u, (size_t)3 * s->V);
  mg->lv.push_back(L0);
  // fine SELL addresses of every CSR block
  std::vector<int64_t> fine_addr(s->nnzb);
  for (int i = 0; i < s->V; ++i) {
    const int lane = i % kSlice;
    for (int k = s->h_rowptr[i]; k < s->h_rowptr[i + 1]; ++k) {
      const int64_t rel = k - s->h_rowptr[i];
      const int64_t base_s = s->h_block_slot[k] - rel * kSlice - lane;
      fine_addr[k] = base_s * 9 + rel * 9 * kSlice + lane;
    }
  }
  HostPattern cur = fine;
  // level 1 gathers from the FP32 fine copy (DP_VAL32_PACKED 2: slot * 8 +
  // tail, 1: slot * 12, else the FP64 layout's component-major addresses)
  std::vector<int64_t> cur_addr(s->nnzb);
  for (int64_t k = 0; k < s->nnzb; ++k)
    cur_addr[k] = DP_VAL32_PACKED == 2 ? s->h_block_slot[k] * 8
                  : DP_VAL32_PACKED   ? s->h_block_slot[k] * 12
                                      : fine_addr[k];
  int lev = 0;
  while (cur.n > kCoarseMax && !rc) {
    std::vector<int> agg;
    int na = aggregate(cur, agg);
    if (g_mg_agg2 && lev >= 1 && na > kCoarseMax) {
      // coarse levels: aggregate the aggregates once more (fewer, larger
      // coarse levels -> a shorter latency-bound coarse chain per V-cycle)
      HostPattern M;
      M.n = na;
      std::vector<std::vector<int>> mr(na);
      for (int i = 0; i < cur.n; ++i)
        for (int k = cur.rowptr[i]; k < cur.rowptr[i + 1]; ++k) mr[agg[i]].push_back(agg[cur.col[k]]);
      M.rowptr.assign(na + 1, 0);
      for (int I = 0; I < na; ++I) {
        auto& r = mr[I];
        std::sort(r.begin(), r.end());
        r.erase(std::unique(r.begin(), r.end()), r.end());
        M.rowptr[I + 1] = M.rowptr[I] + (int)r.size();
      }
      for (int I = 0; I < na; ++I) M.col.insert(M.col.end(), mr[I].begin(), mr[I].end());
      std::vector<int> agg2;
      const int na2 = aggregate(M, agg2);
      if (na2 >= 1 && na2 < na) {
        for (int i = 0; i < cur.n; ++i) agg[i] = agg2[agg[i]];
        na = na2;
      }
    }
    ++lev;
    if (na >= cur.n || na < 1 || (double)cur.n / na < 1.5) break;
    // coarse pattern
    HostPattern C;
    C.n = na;
    std::vector<std::vector<int>> rows(na);
    for (int i = 0; i < cur.n; ++i)
      for (int k = cur.rowptr[i]; k < cur.rowptr[i + 1]; ++k) rows[agg[i]].push_back(agg[cur.col[k]]);
    C.rowptr.assign(na + 1, 0);
    for (int I = 0; I < na; ++I) {
      auto& r = rows[I];
      std::sort(r.begin(), r.end());
      r.erase(std::unique(r.begin(), r.end()), r.end());
      C.rowptr[I + 1] = C.rowptr[I] + (int)r.size();
    }
    C.col.reserve(C.rowptr[na]);
    for (int I = 0; I < na; ++I) C.col.insert(C.col.end(), rows[I].begin(), rows[I].end());
    std::vector<int> sb, sw, cc, ds;
    std::vector<int64_t> slot_of;
    sell_layout(C, sb, sw, cc, ds, slot_of);
    const int64_t NS = sb.back();
    // Galerkin gather lists: coarse slot <- fine blocks (i,j) with agg(i)=I, agg(j)=J
    std::vector<int> gcount(NS + 1, 0);
    std::vector<int64_t> fslot(cur.col.size());
    for (int i = 0; i < cur.n; ++i) {
      const int I = agg[i];
      const int* rb = C.col.data() + C.rowptr[I];
      const int rl = C.rowptr[I + 1] - C.rowptr[I];
      for (int k = cur.rowptr[i]; k < cur.rowptr[i + 1]; ++k) {
        const int J = agg[cur.col[k]];
        const int kk = (int)(std::lower_bound(rb, rb + rl, J) - rb);
        const int64_t cs = slot_of[C.rowptr[I] + kk];
        fslot[k] = cs;
        gcount[cs + 1]++;
      }
    }
    for (int64_t t = 0; t < NS; ++t) gcount[t + 1] += gcount[t];
    std::vector<int> gal(gcount[NS]);
    {
      std::vector<int> fill(gcount.begin(), gcount.end() - 1);
      for (size_t k = 0; k < cur.col.size(); ++k) gal[fill[fslot[k]]++] = (int)cur_addr[k];
    }
    std::vector<int> mptr(na + 1, 0), mem(cur.n);
    for (int i = 0; i < cur.n; ++i) mptr[agg[i] + 1]++;
    for (int I = 0; I < na; ++I) mptr[I + 1] += mptr[I];
    {
      std::vector<int> fill(mptr.begin(), mptr.end() - 1);
      for (int i = 0; i < cur.n; ++i) mem[fill[agg[i]]++] = i;
    }
    MGLevel L;
    L.n = na;
    L.S = (na + kSlice - 1) / kSlice;
    L.NS = NS;
    rc |= up(mg, &L.slice_base, sb);
    rc |= up(mg, &L.slice_width, sw);
    L.kmax = sw.empty() ? 0 : *std::max_element(sw.begin(), sw.end());
    rc |= up(mg, &L.col, cc);
    rc |= up(mg, &L.diag_slot, ds);
    rc |= al(mg, &L.val, (size_t)NS * 9);
    rc |= al(mg, &L.minv, (size_t)na * 9);
    rc |= up(mg, &L.gal_ptr, gcount);
    rc |= up(mg, &L.gal, gal);
    rc |= up(mg, &L.mem_ptr, mptr);
    rc |= up(mg, &L.mem, mem);
    rc |= up(mg, &L.agg, agg);
    {
      std::vector<int> srow(NS);
      for (int64_t t = 0; t < NS; ++t) {
        const int64_t sl = std::upper_bound(sb.begin(), sb.end(), (int)t) - sb.begin() - 1;
        srow[t] = (int)(sl * kSlice + (t - sb[sl]) % kSlice);
      }
      rc |= up(mg, &L.slot_row, srow);
    }
    rc |= al(mg, &L.x, (size_t)3 * na);
    rc |= al(mg, &L.b, (size_t)3 * na);
    rc |= al(mg, &L.r, (size_t)3 * na);
    rc |= al(mg, &L.t, (size_t)3 * na);
    rc |= al(mg, &L.u, (size_t)3 * na);
    mg->lv.push_back(L);
    // next level's address list: coarse CSR block k -> its SELL value address
    std::vector<int64_t> caddr(C.col.size());
    for (int I = 0; I < na; ++I) {
      const int lane = I % kSlice;
      for (int k = C.rowptr[I]; k < C.rowptr[I + 1]; ++k) {
        const int64_t rel = k - C.rowptr[I];
        const int64_t base_s = slot_of[k] - rel * kSlice - lane;
        caddr[k] = base_s * 9 + rel * 9 * kSlice + lane;
      }
    }
    cur = C;
    cur_addr = caddr;
  }
  if (rc) { delete mg; return rc; }
  const MGLevel& Lc = mg->lv.back();
  mg->N = 3 * Lc.n;
  if (mg->lv.size() < 2 || mg->N > kDenseSmem) {
    // no useful hierarchy (tiny or unaggregatable graph): disable
    if (s->val32) { cudaFree(s->val32); s->val32 = nullptr; }
  if (s->val16) { cudaFree(s->val16); s->val16 = nullptr; }
  if (s->sc16) { cudaFree(s->sc16); s->sc16 = nullptr; }
    if (s->val16) { cudaFree(s->val16); s->val16 = nullptr; }
    if (s->sc16) { cudaFree(s->sc16); s->sc16 = nullptr; }
    if (s->minv32) { cudaFree(s->minv32); s->minv32 = nullptr; }
    delete mg;
    s->mg = nullptr;
    return 0;
  }
  cudaFuncSetAttribute(k_mg_dense_invert, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(2 * kDenseSmem * kDenseSmem * sizeof(double)));
  rc |= al(mg, &mg->dense, (size_t)mg->N * mg->N);
  rc |= al(mg, &mg->dinv, (size_t)mg->N * mg->N);
  if (rc) { delete mg; return rc; }
  if (getenv("DP_MG_OMEGA")) mg->omega = atof(getenv("DP_MG_OMEGA"));
  if (getenv("DP_MG_NU")) mg->nu = atoi(getenv("DP_MG_NU"));
  if (getenv("DP_MG_ALPHA")) mg->alpha = mg->alpha_gm = atof(getenv("DP_MG_ALPHA"));
  if (getenv("DP_MG_ALPHA_CG")) mg->alpha_cg = atof(getenv("DP_MG_ALPHA_CG"));
  if (getenv("DP_MG_POST")) mg->post = atoi(getenv("DP_MG_POST"));
  if (getenv("DP_MG_GAMMA")) mg->gamma = atoi(getenv("DP_MG_GAMMA"));
  if (getenv("DP_MG_CSWEEP")) mg->coarse_sweeps = atoi(getenv("DP_MG_CSWEEP"));
  mg->fused_grid = fused_grid_size(s->device);
  s->mg = mg;
  s->bytes += mg->bytes;
  return 0;
}

void mg_destroy(dp_scene* s) {
  MG* mg = s->mg;
  if (!mg) return;
  if (s->val32) { cudaFree(s->val32); s->val32 = nullptr; }
  if (s->val16) { cudaFree(s->val16); s->val16 = nullptr; }
  if (s->sc16) { cudaFree(s->sc16); s->sc16 = nullptr; }
  if (s->minv32) { cudaFree(s->minv32); s->minv32 = nullptr; }
  for (size_t l = 0; l < mg->lv.size(); ++l) {
    MGLevel& L = mg->lv[l];
    void* own[] = {L.x, L.r, L.t, L.u, L.b};
    for (void* p : own) if (p) cudaFree(p);
    if (l > 0) {
      void* p2[] = {L.slice_base, L.slice_width, L.col, L.diag_slot, L.val, L.minv, L.gal_ptr, L.gal,
                    L.mem_ptr, L.mem, L.agg, L.slot_row};
      for (void* p : p2) if (p) cudaFree(p);
    }
  }
  if (mg->dense) cudaFree(mg->dense);
  if (mg->dinv) cudaFree(mg->dinv);
  delete mg;
  s->mg = nullptr;
}

int mg_levels(const dp_scene* s) { return s->mg ? (int)s->mg->lv.size() : 0; }
int mg_level_rows(const dp_scene* s, int l) { return s->mg ? s->mg->lv[l].n : 0; }
void mg_set_params(dp_scene* s, double omega, int nu) {
  if (s->mg) { s->mg->omega = omega; s->mg->nu = nu; }
}

// ---------------------------------------------------------------------------
// kernels

__device__ __forceinline__ void inv3(const double a[9], double o[9]) {
  const double c00 = a[4] * a[8] - a[5] * a[7];
  const double c01 = a[5] * a[6] - a[3] * a[8];
  const double c02 = a[3] * a[7] - a[4] * a[6];
  const double det = a[0] * c00 + a[1] * c01 + a[2] * c02;
  const double id = 1.0 / det;
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

// The same product with an 8-lane group per coarse slot (4 slots per warp):
// most coarse slots gather a few dozen fine blocks, so the 9-value
// reduction over 8 lanes (3 shuffle rounds) replaces the 5-round warp tree
// that dominated the warp-per-slot kernel.  Component-major layouts only.
template <class TF>
__global__ void __launch_bounds__(256) k_mg_galerkin8(int n, const int* __restrict__ slice_base,
                                                      const int* __restrict__ diag_slot,
                                                      const int* __restrict__ gal_ptr, const int* __restrict__ gal,
                                                      const TF* __restrict__ valf, double* __restrict__ valc,
                                                      double* __restrict__ minv, const int* __restrict__ slot_row,
                                                      int64_t NS) {
  const int64_t slot = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int g = threadIdx.x & 7;
  const bool live = slot < NS;
  const int t0 = live ? gal_ptr[slot] : 0, t1 = live ? gal_ptr[slot + 1] : 0;
  double b[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int t = t0 + g; t < t1; t += 8) {
    const TF* src = valf + gal[t];
#pragma unroll
    for (int c = 0; c < 9; ++c) b[c] += (double)src[c * kSlice];
  }
#pragma unroll
  for (int c = 0; c < 9; ++c) {
    b[c] += __shfl_xor_sync(0xffffffffu, b[c], 4);
    b[c] += __shfl_xor_sync(0xffffffffu, b[c], 2);
    b[c] += __shfl_xor_sync(0xffffffffu, b[c], 1);
  }
  if (!live || t0 == t1) return;   // padding keeps the zero block from setup
  const int ln = (int)(slot % kSlice);
  double* dst = valc + (size_t)(slot - ln) * 9 + ln;
  // lanes 0..7 of the group write components g and g + 8
  double v = 0.0;
#pragma unroll
  for (int c = 0; c < 9; ++c) v = (g == c) ? b[c] : v;
  dst[g * kSlice] = v;
  if (g == 0) dst[8 * kSlice] = b[8];
  const int row = slot_row[slot];
  if (g == 0 && row < n && slot == diag_slot[row]) {
    double o[9];
    inv3(b, o);
#pragma unroll
    for (int c = 0; c < 9; ++c) minv[(size_t)c * n + row] = o[c];
  }
}

// coarse operator: val_c[slot] = sum of the fine blocks in its gather list
// (one warp per coarse slot, lanes over contributions); block-Jacobi inverse
// of the diagonal slots.
template <class TF, int CSTRIDE>
__global__ void __launch_bounds__(256) k_mg_galerkin(int n, int S, const int* __restrict__ slice_base,
                                                     const int* __restrict__ slice_width,
                                                     const int* __restrict__ diag_slot,
                                                     const int* __restrict__ gal_ptr, const int* __restrict__ gal,
                                                     const TF* __restrict__ valf, double* __restrict__ valc,
                                                     double* __restrict__ minv, const int* __restrict__ slot_row,
                                                     int64_t NS, const TF* __restrict__ tail) {
  const int64_t slot = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (slot >= NS) return;
  // SELL padding (no fine blocks): stays the zero block written at setup
  if (gal_ptr[slot] == gal_ptr[slot + 1]) return;
  double b[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int t = gal_ptr[slot] + lane; t < gal_ptr[slot + 1]; t += 32) {
    const TF* src = valf + gal[t];
    if (tail) {   // FP32 fine copy, 8 + 1 layout: gal[t] = 8 * fine slot
#pragma unroll
      for (int c = 0; c < 8; ++c) b[c] += (double)src[c];
      b[8] += (double)tail[gal[t] >> 3];
    } else {
#pragma unroll
      for (int c = 0; c < 9; ++c) b[c] += (double)src[c * CSTRIDE];
    }
  }
#pragma unroll
  for (int c = 0; c < 9; ++c) b[c] = warp_allsum(b[c]);
  // slot -> (slice, k, lane)
  const int row = slot_row[slot];
  const int sl = row / kSlice, ln = row % kSlice;
  const int base = slice_base[sl];
  const int k = (int)((slot - base - ln) / kSlice);
  if (lane < 9) {
    double v = 0.0;
#pragma unroll
    for (int c = 0; c < 9; ++c) v = (lane == c) ? b[c] : v;
    valc[(size_t)base * 9 + (k * 9 + lane) * kSlice + ln] = v;
  }
  if (lane == 0 && row < n && slot == diag_slot[row]) {
    double o[9];
    inv3(b, o);
#pragma unroll
    for (int c = 0; c < 9; ++c) minv[(size_t)c * n + row] = o[c];
  }
}

template <class TM>
__device__ __forceinline__ void mv_minv(const TM* __restrict__ minv, int n, int i, const double r[3], double u[3]) {
  u[0] = minv[0 * (size_t)n + i] * r[0] + minv[1 * (size_t)n + i] * r[1] + minv[2 * (size_t)n + i] * r[2];
  u[1] = minv[3 * (size_t)n + i] * r[0] + minv[4 * (size_t)n + i] * r[1] + minv[5 * (size_t)n + i] * r[2];
  u[2] = minv[6 * (size_t)n + i] * r[0] + minv[7 * (size_t)n + i] * r[1] + minv[8 * (size_t)n + i] * r[2];
}

// x = omega Minv b
__device__ __forceinline__ bool stopped(const int* stop) { return stop && *(volatile const int*)stop; }

template <class TM>
__global__ void k_mg_jacobi0(int n, const TM* __restrict__ minv, const double* __restrict__ b, double omega,
                             double* __restrict__ x, const int* stop) {
  if (stopped(stop)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double r[3] = {b[3 * i], b[3 * i + 1], b[3 * i + 2]};
  double u[3];
  mv_minv(minv, n, i, r, u);
  x[3 * i] = omega * u[0]; x[3 * i + 1] = omega * u[1]; x[3 * i + 2] = omega * u[2];
}

// out = xt + omega Minv (b - A xt), xt = x + P xc (xc/agg may be null)
// and optionally r_out = b - A xt (for the residual after the last pre-sweep)
// SPLIT = 1: one warp per SELL slice (fine level: plenty of slices).
// SPLIT = 8: one CTA per slice, warp w takes slots k = w, w+8, ... and the
// partial row sums meet in shared memory - the coarse levels have few slices
// but wide rows (a level-1 row couples ~27-100 aggregates), where a single
// warp per slice is a long dependent-latency chain.
// DOT (fine level, SPLIT = 1, with `out`): the PCG's (r, z) reduction fused
// into the epilogue - b is r, out is z; the last CTA folds the per-CTA
// partials in a fixed order and updates beta/gamma exactly as k_pcg_rz
template <class TV, int SPLIT, bool DOT = false, int BULK = 0>
__global__ void __launch_bounds__(256, 5) k_mg_smooth(int n, int S, const int* __restrict__ slice_base,
                                                   const int* __restrict__ slice_width, const int* __restrict__ col,
                                                   const TV* __restrict__ val, const TV* __restrict__ minv,
                                                   const double* __restrict__ b, const double* __restrict__ x,
                                                   const double* __restrict__ xc, const int* __restrict__ agg,
                                                   double omega, double* __restrict__ out, double* __restrict__ r_out,
                                                   const int* stop, double alpha, double* dot_partial = nullptr,
                                                   unsigned int* dot_counter = nullptr,
                                                   KrylovScalars* dot_ks = nullptr) {
  __shared__ double part[SPLIT > 1 ? SPLIT : 1][3][kSlice];
  if (stopped(stop)) return;   // uniform over the grid (set by an earlier kernel)
  const int lane = threadIdx.x & 31;
  const int wsub = (SPLIT > 1) ? (threadIdx.x >> 5) : 0;
  const int gw = (SPLIT > 1) ? blockIdx.x : (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double rz = 0.0;
  if (gw < S) {
  const int row = gw * kSlice + lane;
  const int base = slice_base[gw], K = slice_width[gw];
  const TV* vs = val + (size_t)base * 9 + lane;
  const int* cs = col + base + lane;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  double ex[3] = {0.0, 0.0, 0.0}, eb[3] = {0.0, 0.0, 0.0};   // x and b of the row, when staged (bulk path)
  TV em[9] = {};                                            // its Minv block, when staged
  bool staged = false;
#if DP_SMOOTH_ASYNC
  if constexpr (sizeof(TV) == 4 && SPLIT == 1 && DP_VAL32_PACKED == 0 && BULK > 0) {
    // the same ring filled by the TMA engine: one lane per warp issues two
    // bulk copies per slot (1,152 B of values + 128 B of columns) that
    // complete on the slot's mbarrier; same values, same order
    __shared__ __align__(128) float sv[DP_SMOOTH_NT / 32][BULK][9 * kSlice];
    __shared__ __align__(128) int sc[DP_SMOOTH_NT / 32][BULK][kSlice];
    __shared__ __align__(8) uint64_t mb[DP_SMOOTH_NT / 32][BULK];
    // the rows' own operands (x, b, Minv), fetched into shared memory while
    // the slots stream, so the epilogue does not wait a memory round trip
    __shared__ __align__(16) double sxb[DP_SMOOTH_NT / 32][2][3 * kSlice];
    __shared__ __align__(16) float smv[DP_SMOOTH_NT / 32][9][kSlice];
    const int w = threadIdx.x >> 5;
    const float* gv = reinterpret_cast<const float*>(val) + (size_t)base * 9;
    const int* gc = col + base;
    {
      const int row0 = gw * kSlice, nr = min(kSlice, n - row0);
      for (int t = lane; t < 3 * nr; t += 32) {
        cp_async8(&sxb[w][0][t], x + 3 * (size_t)row0 + t);
        cp_async8(&sxb[w][1][t], b + 3 * (size_t)row0 + t);
      }
      if (out && lane < nr) {
#pragma unroll
        for (int c = 0; c < 9; ++c) cp_async4(&smv[w][c][lane], minv + (size_t)c * n + row0 + lane);
      }
      cp_async_commit();
    }
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
      double m[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) m[c] = (double)vv[c * kSlice + lane];
      double x0 = __ldg(x + 3 * j), x1 = __ldg(x + 3 * j + 1), x2 = __ldg(x + 3 * j + 2);
      if (xc) {
        const int J = __ldg(agg + j);
        x0 += alpha * __ldg(xc + 3 * J); x1 += alpha * __ldg(xc + 3 * J + 1); x2 += alpha * __ldg(xc + 3 * J + 2);
      }
      a0 += m[0] * x0 + m[1] * x1 + m[2] * x2;
      a1 += m[3] * x0 + m[4] * x1 + m[5] * x2;
      a2 += m[6] * x0 + m[7] * x1 + m[8] * x2;
      __syncwarp();
      issue(k + BULK);
    }
    cp_async_wait<0>();
    __syncwarp();
    if (row < n) {
#pragma unroll
      for (int c = 0; c < 3; ++c) { ex[c] = sxb[w][0][3 * lane + c]; eb[c] = sxb[w][1][3 * lane + c]; }
      if (out) {
#pragma unroll
        for (int c = 0; c < 9; ++c) em[c] = smv[w][c][lane];
      }
      staged = true;
    }
  } else if constexpr (sizeof(TV) == 4 && SPLIT == 1 && DP_VAL32_PACKED == 0) {
    // fine level: the slice's slots stream through a per-warp shared-memory
    // ring, kSmDepth slots ahead, with cp.async (a slot is 1,152 contiguous
    // bytes of component-major FP32 values + 128 bytes of column indices), so
    // each warp keeps ~5 KB of loads in flight instead of one slot's worth.
    // Same values, same accumulation order as the direct loads below.
    __shared__ __align__(16) float sv[DP_SMOOTH_NT / 32][kSmDepth][9 * kSlice];
    __shared__ __align__(16) int sc[DP_SMOOTH_NT / 32][kSmDepth][kSlice];
    const int w = threadIdx.x >> 5;
    const float* gv = reinterpret_cast<const float*>(val) + (size_t)base * 9;
    const int* gc = col + base;
    auto issue = [&](int kk) {
      if (kk < K) {
        const float* src = gv + (size_t)kk * 9 * kSlice;
        float* dst = sv[w][kk % kSmDepth];
        for (int ch = lane; ch < 9 * kSlice / 4; ch += 32) cp_async16(dst + 4 * ch, src + 4 * ch);
        if (lane < kSlice / 4) cp_async16(&sc[w][kk % kSmDepth][4 * lane], gc + kk * kSlice + 4 * lane);
      }
      cp_async_commit();
    };
#pragma unroll
    for (int kk = 0; kk < kSmDepth; ++kk) issue(kk);
    for (int k = 0; k < K; ++k) {
      cp_async_wait<kSmDepth - 1>();
      __syncwarp();
      const float* vv = sv[w][k % kSmDepth];
      const int j = sc[w][k % kSmDepth][lane];
      double m[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) m[c] = (double)vv[c * kSlice + lane];
      double x0 = __ldg(x + 3 * j), x1 = __ldg(x + 3 * j + 1), x2 = __ldg(x + 3 * j + 2);
      if (xc) {
        const int J = __ldg(agg + j);
        x0 += alpha * __ldg(xc + 3 * J); x1 += alpha * __ldg(xc + 3 * J + 1); x2 += alpha * __ldg(xc + 3 * J + 2);
      }
      a0 += m[0] * x0 + m[1] * x1 + m[2] * x2;
      a1 += m[3] * x0 + m[4] * x1 + m[5] * x2;
      a2 += m[6] * x0 + m[7] * x1 + m[8] * x2;
      __syncwarp();
      issue(k + kSmDepth);
    }
    cp_async_wait<0>();
  } else if constexpr (sizeof(TV) == 8 && SPLIT == 8 && BULK > 0) {
    // coarse levels, the ring filled by TMA bulk copies (one lane per warp,
    // 2,304 + 128 B per slot, mbarrier completion); same values, same order
    __shared__ __align__(128) double sv[SPLIT][BULK][9 * kSlice];
    __shared__ __align__(128) int sc[SPLIT][BULK][kSlice];
    __shared__ __align__(8) uint64_t mb[SPLIT][BULK];
    const double* gv = reinterpret_cast<const double*>(val) + (size_t)base * 9;
    const int* gc = col + base;
    const int nk = (K > wsub) ? (K - wsub + SPLIT - 1) / SPLIT : 0;
    if (lane == 0) {
#pragma unroll
      for (int d = 0; d < BULK; ++d) mbar_init(&mb[wsub][d], 1);
      mbar_fence_init();
    }
    __syncwarp();
    auto issue = [&](int i) {
      if (i < nk && lane == 0) {
        const int kk = wsub + i * SPLIT;
        const int d = i % BULK;
        mbar_expect_tx(&mb[wsub][d], 9 * kSlice * 8 + kSlice * 4);
        bulk_g2s(sv[wsub][d], gv + (size_t)kk * 9 * kSlice, 9 * kSlice * 8, &mb[wsub][d]);
        bulk_g2s(sc[wsub][d], gc + (size_t)kk * kSlice, kSlice * 4, &mb[wsub][d]);
      }
    };
#pragma unroll
    for (int i = 0; i < BULK; ++i) issue(i);
    for (int i = 0; i < nk; ++i) {
      const int d = i % BULK;
      mbar_wait(&mb[wsub][d], (uint32_t)((i / BULK) & 1));
      const double* vv = sv[wsub][d];
      const int j = sc[wsub][d][lane];
      double m[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) m[c] = vv[c * kSlice + lane];
      double x0 = __ldg(x + 3 * j), x1 = __ldg(x + 3 * j + 1), x2 = __ldg(x + 3 * j + 2);
      if (xc) {
        const int J = __ldg(agg + j);
        x0 += alpha * __ldg(xc + 3 * J); x1 += alpha * __ldg(xc + 3 * J + 1); x2 += alpha * __ldg(xc + 3 * J + 2);
      }
      a0 += m[0] * x0 + m[1] * x1 + m[2] * x2;
      a1 += m[3] * x0 + m[4] * x1 + m[5] * x2;
      a2 += m[6] * x0 + m[7] * x1 + m[8] * x2;
      __syncwarp();
      issue(i + BULK);
    }
  } else if constexpr (sizeof(TV) == 8 && SPLIT == 8) {
    // coarse levels (L2-resident FP64): warp wsub's slots wsub, wsub + 8, ...
    // stream through a 2-deep per-warp shared-memory ring (2,304 + 128 bytes
    // per slot); same values, same order as the direct loads below
    __shared__ __align__(16) double sv[SPLIT][kSmDepthC][9 * kSlice];
    __shared__ __align__(16) int sc[SPLIT][kSmDepthC][kSlice];
    const double* gv = reinterpret_cast<const double*>(val) + (size_t)base * 9;
    const int* gc = col + base;
    const int nk = (K > wsub) ? (K - wsub + SPLIT - 1) / SPLIT : 0;
    auto issue = [&](int i) {
      if (i < nk) {
        const int kk = wsub + i * SPLIT;
        const double* src = gv + (size_t)kk * 9 * kSlice;
        double* dst = sv[wsub][i % kSmDepthC];
        for (int ch = lane; ch < 9 * kSlice / 2; ch += 32) cp_async16(dst + 2 * ch, src + 2 * ch);
        if (lane < kSlice / 4) cp_async16(&sc[wsub][i % kSmDepthC][4 * lane], gc + kk * kSlice + 4 * lane);
      }
      cp_async_commit();
    };
#pragma unroll
    for (int i = 0; i < kSmDepthC; ++i) issue(i);
    for (int i = 0; i < nk; ++i) {
      cp_async_wait<kSmDepthC - 1>();
      __syncwarp();
      const double* vv = sv[wsub][i % kSmDepthC];
      const int j = sc[wsub][i % kSmDepthC][lane];
      double m[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) m[c] = vv[c * kSlice + lane];
      double x0 = __ldg(x + 3 * j), x1 = __ldg(x + 3 * j + 1), x2 = __ldg(x + 3 * j + 2);
      if (xc) {
        const int J = __ldg(agg + j);
        x0 += alpha * __ldg(xc + 3 * J); x1 += alpha * __ldg(xc + 3 * J + 1); x2 += alpha * __ldg(xc + 3 * J + 2);
      }
      a0 += m[0] * x0 + m[1] * x1 + m[2] * x2;
      a1 += m[3] * x0 + m[4] * x1 + m[5] * x2;
      a2 += m[6] * x0 + m[7] * x1 + m[8] * x2;
      __syncwarp();
      issue(i + kSmDepthC);
    }
    cp_async_wait<0>();
  } else
#endif
  for (int k = wsub; k < K; k += SPLIT) {
    const int j = __ldg(cs + k * kSlice);
    double m[9];
    if (sizeof(TV) == 4 && DP_VAL32_PACKED == 2) {
      // 8 + 1 FP32 layout: one 256-bit load per block + the tail float
      const int slot = base + k * kSlice + lane;
      float f[8];
      ld256f(reinterpret_cast<const float*>(val) + (size_t)slot * 8, f);
#pragma unroll
      for (int c = 0; c < 8; ++c) m[c] = f[c];
      m[8] = __ldg(reinterpret_cast<const float*>(val) + (size_t)slice_base[S] * 8 + slot);
    } else if (sizeof(TV) == 4 && DP_VAL32_PACKED) {
      // packed FP32 fine level: 3 x 16-byte loads per block
      const float4* p4 = reinterpret_cast<const float4*>(val) + (size_t)(base + k * kSlice + lane) * 3;
      const float4 q0 = __ldg(p4), q1 = __ldg(p4 + 1), q2 = __ldg(p4 + 2);
      m[0] = q0.x; m[1] = q0.y; m[2] = q0.z; m[3] = q0.w;
      m[4] = q1.x; m[5] = q1.y; m[6] = q1.z; m[7] = q1.w; m[8] = q2.x;
    } else {
      const TV* v = vs + k * 9 * kSlice;
#pragma unroll
      for (int c = 0; c < 9; ++c) m[c] = (double)v[c * kSlice];
    }
    double x0 = __ldg(x + 3 * j), x1 = __ldg(x + 3 * j + 1), x2 = __ldg(x + 3 * j + 2);
    if (xc) {
      const int J = __ldg(agg + j);
      x0 += alpha * __ldg(xc + 3 * J); x1 += alpha * __ldg(xc + 3 * J + 1); x2 += alpha * __ldg(xc + 3 * J + 2);
    }
    a0 += m[0] * x0 + m[1] * x1 + m[2] * x2;
    a1 += m[3] * x0 + m[4] * x1 + m[5] * x2;
    a2 += m[6] * x0 + m[7] * x1 + m[8] * x2;
  }
  if (SPLIT > 1) {
    part[wsub][0][lane] = a0;
    part[wsub][1][lane] = a1;
    part[wsub][2][lane] = a2;
    __syncthreads();
    if (wsub != 0) return;
    a0 = a1 = a2 = 0.0;
#pragma unroll
    for (int w = 0; w < SPLIT; ++w) { a0 += part[w][0][lane]; a1 += part[w][1][lane]; a2 += part[w][2][lane]; }
  }
  if (row < n) {
    double xt[3], bb[3];
    if (staged) {
      xt[0] = ex[0]; xt[1] = ex[1]; xt[2] = ex[2];
      bb[0] = eb[0]; bb[1] = eb[1]; bb[2] = eb[2];
    } else {
      xt[0] = x[3 * row]; xt[1] = x[3 * row + 1]; xt[2] = x[3 * row + 2];
      bb[0] = b[3 * row]; bb[1] = b[3 * row + 1]; bb[2] = b[3 * row + 2];
    }
    if (xc) {
      const int I = agg[row];
      xt[0] += alpha * xc[3 * I]; xt[1] += alpha * xc[3 * I + 1]; xt[2] += alpha * xc[3 * I + 2];
    }
    const double rr[3] = {bb[0] - a0, bb[1] - a1, bb[2] - a2};
    if (r_out) { r_out[3 * row] = rr[0]; r_out[3 * row + 1] = rr[1]; r_out[3 * row + 2] = rr[2]; }
    if (out) {
      double u[3];
      if (staged) {
        u[0] = em[0] * rr[0] + em[1] * rr[1] + em[2] * rr[2];
        u[1] = em[3] * rr[0] + em[4] * rr[1] + em[5] * rr[2];
        u[2] = em[6] * rr[0] + em[7] * rr[1] + em[8] * rr[2];
      } else {
        mv_minv(minv, n, row, rr, u);
      }
      const double z0 = xt[0] + omega * u[0], z1 = xt[1] + omega * u[1], z2 = xt[2] + omega * u[2];
      out[3 * row] = z0;
      out[3 * row + 1] = z1;
      out[3 * row + 2] = z2;
      if (DOT) rz = bb[0] * z0 + bb[1] * z1 + bb[2] * z2;
    }
  }
  }   // gw < S
  if constexpr (DOT) {
    static_assert(SPLIT == 1, "fused (r, z) only on the one-warp-per-slice fine level");
    __shared__ double sh[32];
    __shared__ double o1[1];
    const double t = block_sum<DP_SMOOTH_NT>(rz, sh);
    if (threadIdx.x == 0) dot_partial[blockIdx.x] = t;
    if (last_block(dot_counter)) {
      fold_partials<DP_SMOOTH_NT, 1>(dot_partial, gridDim.x, o1, sh);
      if (threadIdx.x == 0) {
        const double g = o1[0];
        dot_ks->beta = (dot_ks->iters == 0) ? 0.0 : g / dot_ks->gamma;
        dot_ks->gamma = g;
        if (!(g > 0.0)) dot_ks->done = 2;     // preconditioner not SPD on this residual
        *dot_counter = 0;
      }
    }
  }
}


// Fine-level sweep on the FP16 operator copy (values scaled per block by
// sc16, dequantised to FP64 in registers): the same arithmetic as the FP32
// sweep otherwise, slots streamed through the per-warp cp.async ring
// (576 B values + 128 B scales + 128 B columns per slot).
template <bool DOT>
__global__ void __launch_bounds__(DP_SMOOTH_NT) k_mg_smooth16(int n, int S, const int* __restrict__ slice_base,
                                                            const int* __restrict__ slice_width,
                                                            const int* __restrict__ col,
                                                            const unsigned short* __restrict__ val16,
                                                            const float* __restrict__ sc16,
                                                            const float* __restrict__ minv, const double* __restrict__ b,
                                                            const double* __restrict__ x,
                                                            const double* __restrict__ xc,
                                                            const int* __restrict__ agg, double omega,
                                                            double* __restrict__ out, double* __restrict__ r_out,
                                                            const int* stop, double alpha, double* dot_partial,
                                                            unsigned int* dot_counter, KrylovScalars* dot_ks) {
  __shared__ __align__(16) unsigned short sv[DP_SMOOTH_NT / 32][kSmDepth][9 * kSlice];
  __shared__ __align__(16) float ss[DP_SMOOTH_NT / 32][kSmDepth][kSlice];
  __shared__ __align__(16) int sc[DP_SMOOTH_NT / 32][kSmDepth][kSlice];
  if (stopped(stop)) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double rz = 0.0;
  if (gw < S) {
    const int row = gw * kSlice + lane;
    const int base = slice_base[gw], K = slice_width[gw];
    const unsigned short* gv = val16 + (size_t)base * 9;
    const float* gs = sc16 + base;
    const int* gc = col + base;
    auto issue = [&](int kk) {
      if (kk < K) {
        const unsigned short* src = gv + (size_t)kk * 9 * kSlice;   // 576 B = 36 x 16 B
        unsigned short* dst = sv[w][kk % kSmDepth];
        for (int ch = lane; ch < 36; ch += 32) cp_async16(dst + 8 * ch, src + 8 * ch);
        if (lane < 8) cp_async16(&ss[w][kk % kSmDepth][4 * lane], gs + kk * kSlice + 4 * lane);
        else if (lane < 16) cp_async16(&sc[w][kk % kSmDepth][4 * (lane - 8)], gc + kk * kSlice + 4 * (lane - 8));
      }
      cp_async_commit();
    };
#pragma unroll
    for (int kk = 0; kk < kSmDepth; ++kk) issue(kk);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int k = 0; k < K; ++k) {
      cp_async_wait<kSmDepth - 1>();
      __syncwarp();
      const unsigned short* vv = sv[w][k % kSmDepth];
      const double scl = (double)ss[w][k % kSmDepth][lane];
      const int j = sc[w][k % kSmDepth][lane];
      double m[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) m[c] = (double)__half2float(__ushort_as_half(vv[c * kSlice + lane])) * scl;
      double x0 = __ldg(x + 3 * j), x1 = __ldg(x + 3 * j + 1), x2 = __ldg(x + 3 * j + 2);
      if (xc) {
        const int J = __ldg(agg + j);
        x0 += alpha * __ldg(xc + 3 * J); x1 += alpha * __ldg(xc + 3 * J + 1); x2 += alpha * __ldg(xc + 3 * J + 2);
      }
      a0 += m[0] * x0 + m[1] * x1 + m[2] * x2;
      a1 += m[3] * x0 + m[4] * x1 + m[5] * x2;
      a2 += m[6] * x0 + m[7] * x1 + m[8] * x2;
      __syncwarp();
      issue(k + kSmDepth);
    }
    cp_async_wait<0>();
    if (row < n) {
      double xt[3] = {x[3 * row], x[3 * row + 1], x[3 * row + 2]};
      if (xc) {
        const int I = agg[row];
        xt[0] += alpha * xc[3 * I]; xt[1] += alpha * xc[3 * I + 1]; xt[2] += alpha * xc[3 * I + 2];
      }
      const double bb[3] = {b[3 * row], b[3 * row + 1], b[3 * row + 2]};
      const double rr[3] = {bb[0] - a0, bb[1] - a1, bb[2] - a2};
      if (r_out) { r_out[3 * row] = rr[0]; r_out[3 * row + 1] = rr[1]; r_out[3 * row + 2] = rr[2]; }
      if (out) {
        double u[3];
        mv_minv(minv, n, row, rr, u);
        const double z0 = xt[0] + omega * u[0], z1 = xt[1] + omega * u[1], z2 = xt[2] + omega * u[2];
        out[3 * row] = z0;
        out[3 * row + 1] = z1;
        out[3 * row + 2] = z2;
        if (DOT) rz = bb[0] * z0 + bb[1] * z1 + bb[2] * z2;
      }
    }
  }
  if constexpr (DOT) {
    __shared__ double sh[32];
    __shared__ double o1[1];
    const double t = block_sum<DP_SMOOTH_NT>(rz, sh);
    if (threadIdx.x == 0) dot_partial[blockIdx.x] = t;
    if (last_block(dot_counter)) {
      fold_partials<DP_SMOOTH_NT, 1>(dot_partial, gridDim.x, o1, sh);
      if (threadIdx.x == 0) {
        const double g = o1[0];
        dot_ks->beta = (dot_ks->iters == 0) ? 0.0 : g / dot_ks->gamma;
        dot_ks->gamma = g;
        if (!(g > 0.0)) dot_ks->done = 2;
        *dot_counter = 0;
      }
    }
  }
}


// Fine-level FP32 sweep with the x gathers software-pipelined one slot ahead:
// a 3-deep cp.async ring; while slot k is accumulated, slot k+1's column
// indices (already in shared memory) feed the gathers of its x values, so
// the dependent x-gather latency of a slot overlaps the previous slot's
// arithmetic and ring wait instead of following it (the sweep is bound by
// that per-warp latency chain, not by bytes: the FP16 copy measured no
// faster).  Same values and accumulation order as k_mg_smooth<float,1>.
constexpr int kPfDepth = 3;
template <bool DOT>
__global__ void __launch_bounds__(DP_SMOOTH_NT) k_mg_smooth_pf(int n, int S, const int* __restrict__ slice_base,
                                                             const int* __restrict__ slice_width,
                                                             const int* __restrict__ col, const float* __restrict__ val,
                                                             const float* __restrict__ minv,
                                                             const double* __restrict__ b,
                                                             const double* __restrict__ x,
                                                             const double* __restrict__ xc,
                                                             const int* __restrict__ agg, double omega,
                                                             double* __restrict__ out, double* __restrict__ r_out,
                                                             const int* stop, double alpha, double* dot_partial,
                                                             unsigned int* dot_counter, KrylovScalars* dot_ks) {
  __shared__ __align__(16) float sv[DP_SMOOTH_NT / 32][kPfDepth][9 * kSlice];
  __shared__ __align__(16) int sc[DP_SMOOTH_NT / 32][kPfDepth][kSlice];
  if (stopped(stop)) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double rz = 0.0;
  if (gw < S) {
    const int row = gw * kSlice + lane;
    const int base = slice_base[gw], K = slice_width[gw];
    const float* gv = val + (size_t)base * 9;
    const int* gc = col + base;
    auto issue = [&](int kk) {
      if (kk < K) {
        const float* src = gv + (size_t)kk * 9 * kSlice;
        float* dst = sv[w][kk % kPfDepth];
        for (int ch = lane; ch < 9 * kSlice / 4; ch += 32) cp_async16(dst + 4 * ch, src + 4 * ch);
        if (lane < kSlice / 4) cp_async16(&sc[w][kk % kPfDepth][4 * lane], gc + kk * kSlice + 4 * lane);
      }
      cp_async_commit();
    };
    auto gather = [&](int kk, double xo[3]) {
      const int j = sc[w][kk % kPfDepth][lane];
      xo[0] = __ldg(x + 3 * j); xo[1] = __ldg(x + 3 * j + 1); xo[2] = __ldg(x + 3 * j + 2);
      if (xc) {
        const int J = __ldg(agg + j);
        xo[0] += alpha * __ldg(xc + 3 * J); xo[1] += alpha * __ldg(xc + 3 * J + 1);
        xo[2] += alpha * __ldg(xc + 3 * J + 2);
      }
    };
#pragma unroll
    for (int kk = 0; kk < kPfDepth; ++kk) issue(kk);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    double xcur[3] = {0.0, 0.0, 0.0};
    if (K > 0) {
      cp_async_wait<kPfDepth - 1>();   // slot 0 landed
      __syncwarp();
      gather(0, xcur);
    }
    for (int k = 0; k < K; ++k) {
      double xnext[3] = {0.0, 0.0, 0.0};
      if (k + 1 < K) {
        cp_async_wait<kPfDepth - 2>();   // slot k+1 landed
        __syncwarp();
        gather(k + 1, xnext);
      }
      const float* vv = sv[w][k % kPfDepth];
      double m[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) m[c] = (double)vv[c * kSlice + lane];
      a0 += m[0] * xcur[0] + m[1] * xcur[1] + m[2] * xcur[2];
      a1 += m[3] * xcur[0] + m[4] * xcur[1] + m[5] * xcur[2];
      a2 += m[6] * xcur[0] + m[7] * xcur[1] + m[8] * xcur[2];
      __syncwarp();
      issue(k + kPfDepth);   // reuses slot k's buffer (its columns and values are consumed)
      xcur[0] = xnext[0]; xcur[1] = xnext[1]; xcur[2] = xnext[2];
    }
    cp_async_wait<0>();
    if (row < n) {
      double xt[3] = {x[3 * row], x[3 * row + 1], x[3 * row + 2]};
      if (xc) {
        const int I = agg[row];
        xt[0] += alpha * xc[3 * I]; xt[1] += alpha * xc[3 * I + 1]; xt[2] += alpha * xc[3 * I + 2];
      }
      const double bb[3] = {b[3 * row], b[3 * row + 1], b[3 * row + 2]};
      const double rr[3] = {bb[0] - a0, bb[1] - a1, bb[2] - a2};
      if (r_out) { r_out[3 * row] = rr[0]; r_out[3 * row + 1] = rr[1]; r_out[3 * row + 2] = rr[2]; }
      if (out) {
        double u[3];
        mv_minv(minv, n, row, rr, u);
        const double z0 = xt[0] + omega * u[0], z1 = xt[1] + omega * u[1], z2 = xt[2] + omega * u[2];
        out[3 * row] = z0;
        out[3 * row + 1] = z1;
        out[3 * row + 2] = z2;
        if (DOT) rz = bb[0] * z0 + bb[1] * z1 + bb[2] * z2;
      }
    }
  }
  if constexpr (DOT) {
    __shared__ double sh[32];
    __shared__ double o1[1];
    const double t = block_sum<DP_SMOOTH_NT>(rz, sh);
    if (threadIdx.x == 0) dot_partial[blockIdx.x] = t;
    if (last_block(dot_counter)) {
      fold_partials<DP_SMOOTH_NT, 1>(dot_partial, gridDim.x, o1, sh);
      if (threadIdx.x == 0) {
        const double g = o1[0];
        dot_ks->beta = (dot_ks->iters == 0) ? 0.0 : g / dot_ks->gamma;
        dot_ks->gamma = g;
        if (!(g > 0.0)) dot_ks->done = 2;
        *dot_counter = 0;
      }
    }
  }
}

// fine sweep ring filled by TMA bulk copies (depth 2; 0 = per-lane cp.async ring): in situ 24.7 -> 23.6 us
static const int g_coarse_bulk = getenv("DP_COARSE_BULK") ? atoi(getenv("DP_COARSE_BULK")) : 1;
static const int g_gal8 = getenv("DP_GAL8") ? atoi(getenv("DP_GAL8")) : 1;
static const int g_smooth_bulk = getenv("DP_SMOOTH_BULK") ? atoi(getenv("DP_SMOOTH_BULK")) : 2;
static const int g_smooth_pf = getenv("DP_SMOOTH_PF") ? atoi(getenv("DP_SMOOTH_PF")) : 0;   // measured slower (25.6 vs 24.1 us in situ), off

// x = xa + alpha P xc
__global__ void k_mg_prolong(int n, const double* __restrict__ xa, const double* __restrict__ xc,
                             const int* __restrict__ agg, double alpha, double* __restrict__ x, const int* stop) {
  if (stopped(stop)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int I = agg[i];
#pragma unroll
  for (int c = 0; c < 3; ++c) x[3 * i + c] = xa[3 * i + c] + alpha * xc[3 * I + c];
}

// b_c[I] = sum over members of r_f (one warp per coarse row)
__global__ void k_mg_restrict(int nc, const int* __restrict__ mptr, const int* __restrict__ mem,
                              const double* __restrict__ rf, double* __restrict__ bc, const int* stop) {
  if (stopped(stop)) return;
  const int I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (I >= nc) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int t = mptr[I] + lane; t < mptr[I + 1]; t += 32) {
    const int i = mem[t];
    s0 += rf[3 * i]; s1 += rf[3 * i + 1]; s2 += rf[3 * i + 2];
  }
  s0 = warp_sum(s0); s1 = warp_sum(s1); s2 = warp_sum(s2);
  if (lane == 0) { bc[3 * I] = s0; bc[3 * I + 1] = s1; bc[3 * I + 2] = s2; }
}

// k_mg_restrict followed by k_mg_jacobi0 of the coarse level in one launch:
// b_c[I] = sum over members of r_f, x_c[I] = omega Minv_c b_c[I] (the same
// sums and the same products as the two kernels, bitwise identical)
template <class TM>
__global__ void k_mg_restrict_j0(int nc, const int* __restrict__ mptr, const int* __restrict__ mem,
                                 const double* __restrict__ rf, double* __restrict__ bc, const TM* __restrict__ minv,
                                 double omega, double* __restrict__ xc, const int* stop) {
  if (stopped(stop)) return;
  const int I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (I >= nc) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int t = mptr[I] + lane; t < mptr[I + 1]; t += 32) {
    const int i = mem[t];
    s0 += rf[3 * i]; s1 += rf[3 * i + 1]; s2 += rf[3 * i + 2];
  }
  s0 = warp_sum(s0); s1 = warp_sum(s1); s2 = warp_sum(s2);
  if (lane == 0) {
    bc[3 * I] = s0; bc[3 * I + 1] = s1; bc[3 * I + 2] = s2;
    const double r[3] = {s0, s1, s2};
    double u[3];
    mv_minv(minv, nc, I, r, u);
    xc[3 * I] = omega * u[0]; xc[3 * I + 1] = omega * u[1]; xc[3 * I + 2] = omega * u[2];
  }
}

// coarsest: scatter SELL blocks into a dense N x N row-major matrix
__global__ void k_mg_dense_build(int n, int S, const int* __restrict__ slice_base, const int* __restrict__ slice_width,
                                 const int* __restrict__ col, const double* __restrict__ val, double* __restrict__ A) {
  const int N = 3 * n;
  for (int t = threadIdx.x; t < N * N; t += blockDim.x) A[t] = 0.0;
  __syncthreads();
  for (int row = threadIdx.x; row < n; row += blockDim.x) {
    const int sl = row / kSlice, lane = row % kSlice;
    const int base = slice_base[sl], K = slice_width[sl];
    for (int k = 0; k < K; ++k) {
      const int j = col[base + k * kSlice + lane];
      const double* v = val + (size_t)base * 9 + (k * 9) * kSlice + lane;
      bool any = false;
#pragma unroll
      for (int c = 0; c < 9; ++c) any |= (v[c * kSlice] != 0.0);
      if (!any) continue;   // padding
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) A[(size_t)(3 * row + a) * N + 3 * j + c] += v[(a * 3 + c) * kSlice];
    }
  }
}

// Gauss-Jordan with partial pivoting in one CTA, matrices in shared memory
// (N <= kDenseSmem): Ainv = A^-1.  Rows are spread over warps, columns over
// lanes (no integer division in the elimination loop).
__global__ void __launch_bounds__(256) k_mg_dense_invert(int N, const double* __restrict__ Ag, double* __restrict__ Ainv) {
  extern __shared__ double smem[];
  double* A = smem;
  double* X = smem + N * N;
  __shared__ int piv;
  __shared__ double rowscale;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int t = threadIdx.x; t < N * N; t += blockDim.x) A[t] = Ag[t];
  for (int r = warp; r < N; r += nw)
    for (int c = lane; c < N; c += 32) X[r * N + c] = (r == c) ? 1.0 : 0.0;
  __syncthreads();
  for (int k = 0; k < N; ++k) {
    if (warp == 0) {
      double best = -1.0;
      int bi = k;
      for (int r = k + lane; r < N; r += 32) {
        const double v = fabs(A[r * N + k]);
        if (v > best) { best = v; bi = r; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, o);
        const int oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) { piv = bi; rowscale = 1.0 / A[bi * N + k]; }
    }
    __syncthreads();
    const int p = piv;
    const double id = rowscale;
    // swap rows k and p while scaling the new pivot row
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
      const double ak = A[k * N + c], ap = A[p * N + c];
      const double xk = X[k * N + c], xp = X[p * N + c];
      A[k * N + c] = ap * id;
      X[k * N + c] = xp * id;
      if (p != k) { A[p * N + c] = ak; X[p * N + c] = xk; }
    }
    __syncthreads();
    for (int r = warp; r < N; r += nw) {
      if (r == k) continue;
      const double f = A[r * N + k];
      if (f == 0.0) continue;
      for (int c = lane; c < N; c += 32) {
        if (c != k) A[r * N + c] -= f * A[k * N + c];
        X[r * N + c] -= f * X[k * N + c];
      }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < N; r += blockDim.x)
      if (r != k) A[r * N + k] = 0.0;
    __syncthreads();
  }
  for (int t = threadIdx.x; t < N * N; t += blockDim.x) Ainv[t] = X[t];
}

// coarsest level without a factorisation: nsweep damped block-Jacobi sweeps
// from zero in one CTA (a fixed symmetric polynomial in D^-1 A, so the
// V-cycle stays a fixed linear operator).  x is both iterate and output;
// y is scratch.
__global__ void __launch_bounds__(256) k_mg_coarse_jacobi(int n, int S, const int* __restrict__ slice_base,
                                                          const int* __restrict__ slice_width,
                                                          const int* __restrict__ col, const double* __restrict__ val,
                                                          const double* __restrict__ minv, double* b,
                                                          double* __restrict__ x, double* __restrict__ y, double omega,
                                                          int nsweep, const int* stop, const int* __restrict__ mptr,
                                                          const int* __restrict__ mem, const double* __restrict__ rf) {
  // one CTA; warp w handles slots k = w, w+8, ... of every slice, lanes = rows
  __shared__ double part[8][3][kSlice];
  if (stop && *(volatile const int*)stop) return;
  const int lane = threadIdx.x & 31, wsub = threadIdx.x >> 5;
  if (rf) {
    // the restriction b = R rf of k_mg_restrict (one warp per coarse row, same
    // order), done here instead of in a launch of its own
    for (int I = wsub; I < n; I += 8) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int t = mptr[I] + lane; t < mptr[I + 1]; t += 32) {
        const int i = mem[t];
        s0 += rf[3 * i]; s1 += rf[3 * i + 1]; s2 += rf[3 * i + 2];
      }
      s0 = warp_sum(s0); s1 = warp_sum(s1); s2 = warp_sum(s2);
      if (lane == 0) { b[3 * I] = s0; b[3 * I + 1] = s1; b[3 * I + 2] = s2; }
    }
    __syncthreads();
  }
  for (int row = threadIdx.x; row < n; row += blockDim.x) {
    double r[3] = {b[3 * row], b[3 * row + 1], b[3 * row + 2]}, u[3];
    mv_minv(minv, n, row, r, u);
#pragma unroll
    for (int c = 0; c < 3; ++c) x[3 * row + c] = omega * u[c];
  }
  __syncthreads();
  for (int it = 0; it < nsweep; ++it) {
    for (int sl = 0; sl < S; ++sl) {
      const int row = sl * kSlice + lane;
      const int base = slice_base[sl], K = slice_width[sl];
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (int k = wsub; k < K; k += 8) {
        const int j = col[base + k * kSlice + lane];
        const double* v = val + (size_t)base * 9 + (k * 9) * kSlice + lane;
        const double x0 = x[3 * j], x1 = x[3 * j + 1], x2 = x[3 * j + 2];
        a0 += v[0 * kSlice] * x0 + v[1 * kSlice] * x1 + v[2 * kSlice] * x2;
        a1 += v[3 * kSlice] * x0 + v[4 * kSlice] * x1 + v[5 * kSlice] * x2;
        a2 += v[6 * kSlice] * x0 + v[7 * kSlice] * x1 + v[8 * kSlice] * x2;
      }
      part[wsub][0][lane] = a0;
      part[wsub][1][lane] = a1;
      part[wsub][2][lane] = a2;
      __syncthreads();
      if (wsub == 0 && row < n) {
        a0 = a1 = a2 = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) { a0 += part[w][0][lane]; a1 += part[w][1][lane]; a2 += part[w][2][lane]; }
        double r[3] = {b[3 * row] - a0, b[3 * row + 1] - a1, b[3 * row + 2] - a2}, u[3];
        mv_minv(minv, n, row, r, u);
#pragma unroll
        for (int c = 0; c < 3; ++c) y[3 * row + c] = x[3 * row + c] + omega * u[c];
      }
      __syncthreads();
    }
    for (int t = threadIdx.x; t < 3 * n; t += blockDim.x) x[t] = y[t];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// All coarse levels of one V-cycle in ONE cooperative kernel.  Below the fine
// level every kernel of the V-cycle is latency-bound (level 1 at C5: 6,859
// block rows, 13 MB of values, L2-resident), so the nine launches of levels
// 1..3 (restrict+jacobi0, residual, restrict, ..., coarsest sweeps, post
// smoothers) become phases of one persistent grid separated by grid-wide
// barriers.  Every phase repeats the arithmetic of its stand-alone kernel
// term by term (same split of a slice over 8 warps, same partial order, same
// warp reductions), so the V-cycle output is bitwise identical to the
// multi-kernel path (checked by tests/test_gpu_scale.py::test_mg_fused_bitwise).

struct FusedLevel {
  int n, S;
  const int *slice_base, *slice_width, *col;
  const double *val, *minv;
  const int *mem_ptr, *mem;   // coarse row -> rows of the level above
  const int* agg;             // row of the level above -> coarse row
  double *x, *b, *r, *t;
};
constexpr int kMaxFusedLevels = 8;
struct FusedArgs {
  int L;                               // levels in the hierarchy (lv[0] unused: fine level)
  FusedLevel lv[kMaxFusedLevels];
  const double* r0;                    // fine-level residual
  double omega, alpha;
  int coarse_sweeps;
  const int* stop;
  unsigned long long* tstamp;          // DP_MG_FTIME: per-phase globaltimer stamps (CTA 0)
};

__device__ __forceinline__ void fused_stamp(const FusedArgs& A, int& ph) {
  if (A.tstamp && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    A.tstamp[ph] = t;
  }
  ++ph;
}

// b_l[I] = sum of r_{l-1} over the members of I; optionally t_l[I] = w Minv b_l[I]
__device__ __forceinline__ void fused_restrict_row(const FusedLevel& C, const double* rf, int I, int lane,
                                                   double omega, bool jac) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int t = C.mem_ptr[I] + lane; t < C.mem_ptr[I + 1]; t += 32) {
    const int i = C.mem[t];
    s0 += __ldcg(rf + 3 * i); s1 += __ldcg(rf + 3 * i + 1); s2 += __ldcg(rf + 3 * i + 2);
  }
  s0 = warp_sum(s0); s1 = warp_sum(s1); s2 = warp_sum(s2);
  if (lane == 0) {
    C.b[3 * I] = s0; C.b[3 * I + 1] = s1; C.b[3 * I + 2] = s2;
    if (jac) {
      const double r[3] = {s0, s1, s2};
      double u[3];
      mv_minv(C.minv, C.n, I, r, u);
      C.t[3 * I] = omega * u[0]; C.t[3 * I + 1] = omega * u[1]; C.t[3 * I + 2] = omega * u[2];
    }
  }
}

// k_mg_smooth<double, 8> for one slice (whole CTA); in-kernel data via __ldcg
__device__ __forceinline__ void fused_smooth_slice(const FusedLevel& L, int sl, const double* x, const double* xc,
                                                   const int* agg, double omega, double* out, double* r_out,
                                                   double alpha, double (*part)[3][kSlice]) {
  const int lane = threadIdx.x & 31, wsub = threadIdx.x >> 5;
  const int row = sl * kSlice + lane;
  const int base = L.slice_base[sl], K = L.slice_width[sl];
  const double* vs = L.val + (size_t)base * 9 + lane;
  const int* cs = L.col + base + lane;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int k = wsub; k < K; k += 8) {
    const int j = __ldg(cs + k * kSlice);
    double m[9];
    const double* v = vs + k * 9 * kSlice;
#pragma unroll
    for (int c = 0; c < 9; ++c) m[c] = (double)v[c * kSlice];
    double x0 = __ldcg(x + 3 * j), x1 = __ldcg(x + 3 * j + 1), x2 = __ldcg(x + 3 * j + 2);
    if (xc) {
      const int J = __ldg(agg + j);
      x0 += alpha * __ldcg(xc + 3 * J); x1 += alpha * __ldcg(xc + 3 * J + 1); x2 += alpha * __ldcg(xc + 3 * J + 2);
    }
    a0 += m[0] * x0 + m[1] * x1 + m[2] * x2;
    a1 += m[3] * x0 + m[4] * x1 + m[5] * x2;
    a2 += m[6] * x0 + m[7] * x1 + m[8] * x2;
  }
  part[wsub][0][lane] = a0;
  part[wsub][1][lane] = a1;
  part[wsub][2][lane] = a2;
  __syncthreads();
  if (wsub == 0 && row < L.n) {
    a0 = a1 = a2 = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) { a0 += part[w][0][lane]; a1 += part[w][1][lane]; a2 += part[w][2][lane]; }
    double xt[3] = {__ldcg(x + 3 * row), __ldcg(x + 3 * row + 1), __ldcg(x + 3 * row + 2)};
    if (xc) {
      const int I = agg[row];
      xt[0] += alpha * __ldcg(xc + 3 * I); xt[1] += alpha * __ldcg(xc + 3 * I + 1);
      xt[2] += alpha * __ldcg(xc + 3 * I + 2);
    }
    const double rr[3] = {__ldcg(L.b + 3 * row) - a0, __ldcg(L.b + 3 * row + 1) - a1,
                          __ldcg(L.b + 3 * row + 2) - a2};
    if (r_out) { r_out[3 * row] = rr[0]; r_out[3 * row + 1] = rr[1]; r_out[3 * row + 2] = rr[2]; }
    if (out) {
      double u[3];
      mv_minv(L.minv, L.n, row, rr, u);
      out[3 * row] = xt[0] + omega * u[0];
      out[3 * row + 1] = xt[1] + omega * u[1];
      out[3 * row + 2] = xt[2] + omega * u[2];
    }
  }
  __syncthreads();   // part[] is reused by the next slice
}

// k_mg_coarse_jacobi in the calling CTA, iterate and right-hand side in
// shared memory (the coarsest level has <= kCoarseMax rows); the arithmetic
// and its order are those of k_mg_coarse_jacobi.
__device__ __forceinline__ void fused_coarse_jacobi(const FusedLevel& C, double omega, int nsweep,
                                                    double (*part)[3][kSlice], double* xs, double* ys,
                                                    const double* bs) {
  const int lane = threadIdx.x & 31, wsub = threadIdx.x >> 5;
  const int n = C.n;
  for (int row = threadIdx.x; row < n; row += blockDim.x) {
    double r[3] = {bs[3 * row], bs[3 * row + 1], bs[3 * row + 2]}, u[3];
    mv_minv(C.minv, n, row, r, u);
#pragma unroll
    for (int c = 0; c < 3; ++c) xs[3 * row + c] = omega * u[c];
  }
  __syncthreads();
  for (int it = 0; it < nsweep; ++it) {
    for (int sl = 0; sl < C.S; ++sl) {
      const int row = sl * kSlice + lane;
      const int base = C.slice_base[sl], K = C.slice_width[sl];
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (int k = wsub; k < K; k += 8) {
        const int j = __ldg(C.col + base + k * kSlice + lane);
        const double* v = C.val + (size_t)base * 9 + (k * 9) * kSlice + lane;
        const double x0 = xs[3 * j], x1 = xs[3 * j + 1], x2 = xs[3 * j + 2];
        a0 += __ldg(v + 0 * kSlice) * x0 + __ldg(v + 1 * kSlice) * x1 + __ldg(v + 2 * kSlice) * x2;
        a1 += __ldg(v + 3 * kSlice) * x0 + __ldg(v + 4 * kSlice) * x1 + __ldg(v + 5 * kSlice) * x2;
        a2 += __ldg(v + 6 * kSlice) * x0 + __ldg(v + 7 * kSlice) * x1 + __ldg(v + 8 * kSlice) * x2;
      }
      part[wsub][0][lane] = a0;
      part[wsub][1][lane] = a1;
      part[wsub][2][lane] = a2;
      __syncthreads();
      if (wsub == 0 && row < n) {
        a0 = a1 = a2 = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) { a0 += part[w][0][lane]; a1 += part[w][1][lane]; a2 += part[w][2][lane]; }
        double r[3] = {bs[3 * row] - a0, bs[3 * row + 1] - a1, bs[3 * row + 2] - a2}, u[3];
        mv_minv(C.minv, n, row, r, u);
#pragma unroll
        for (int c = 0; c < 3; ++c) ys[3 * row + c] = xs[3 * row + c] + omega * u[c];
      }
      __syncthreads();
    }
    for (int t = threadIdx.x; t < 3 * n; t += blockDim.x) xs[t] = ys[t];
    __syncthreads();
  }
  for (int t = threadIdx.x; t < 3 * n; t += blockDim.x) C.x[t] = xs[t];
}

__global__ void __launch_bounds__(256) k_mg_coarse_fused(const __grid_constant__ FusedArgs A) {
  __shared__ double part[8][3][kSlice];
  if (A.stop && *(volatile const int*)A.stop) return;   // uniform over the grid
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * 8 + warp, nwarps = gridDim.x * 8;
  const int Lc = A.L - 1;
  int ph = 0;
  fused_stamp(A, ph);
  // descending: restrict + jacobi0, residual
  for (int l = 1; l < Lc; ++l) {
    const FusedLevel& C = A.lv[l];
    const double* rf = (l == 1) ? A.r0 : A.lv[l - 1].r;
    for (int I = gwarp; I < C.n; I += nwarps) fused_restrict_row(C, rf, I, lane, A.omega, true);
    fused_stamp(A, ph);
    grid.sync();
    fused_stamp(A, ph);
    for (int sl = blockIdx.x; sl < C.S; sl += gridDim.x)
      fused_smooth_slice(C, sl, C.t, nullptr, nullptr, A.omega, nullptr, C.r, 1.0, part);
    fused_stamp(A, ph);
    grid.sync();
    fused_stamp(A, ph);
  }
  // coarsest: restriction and the Jacobi sweeps in CTA 0
  if (blockIdx.x == 0) {
    __shared__ double xs[3 * kCoarseMax + 3], ys[3 * kCoarseMax + 3], bs[3 * kCoarseMax + 3];
    const FusedLevel& C = A.lv[Lc];
    const double* rf = (Lc == 1) ? A.r0 : A.lv[Lc - 1].r;
    for (int I = warp; I < C.n; I += 8) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int t = C.mem_ptr[I] + lane; t < C.mem_ptr[I + 1]; t += 32) {
        const int i = C.mem[t];
        s0 += __ldcg(rf + 3 * i); s1 += __ldcg(rf + 3 * i + 1); s2 += __ldcg(rf + 3 * i + 2);
      }
      s0 = warp_sum(s0); s1 = warp_sum(s1); s2 = warp_sum(s2);
      if (lane == 0) { bs[3 * I] = s0; bs[3 * I + 1] = s1; bs[3 * I + 2] = s2; }
    }
    __syncthreads();
    fused_coarse_jacobi(C, A.omega, A.coarse_sweeps, part, xs, ys, bs);
  }
  fused_stamp(A, ph);
  // ascending: post-smoothing with the coarse correction in its gathers
  for (int l = Lc - 1; l >= 1; --l) {
    grid.sync();
    fused_stamp(A, ph);
    const FusedLevel& C = A.lv[l];
    for (int sl = blockIdx.x; sl < C.S; sl += gridDim.x)
      fused_smooth_slice(C, sl, C.t, A.lv[l + 1].x, A.lv[l + 1].agg, A.omega, C.x, nullptr, A.alpha, part);
    fused_stamp(A, ph);
  }
}

// co-resident grid of the cooperative kernel: up to 2 CTAs per SM
static int fused_grid_size(int device) {
  int nsm = 0, per_sm = 0;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
  if (!coop) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mg_coarse_fused, 256, 0) != cudaSuccess) return 0;
  const int want = getenv("DP_MG_FGRID") ? atoi(getenv("DP_MG_FGRID")) : 2;
  return nsm * std::max(1, std::min(per_sm, want));
}

// x = Ainv b (dense, one row per warp)
__global__ void k_mg_dense_solve(int N, const double* __restrict__ Ainv, const double* __restrict__ b,
                                 double* __restrict__ x, const int* stop) {
  if (stopped(stop)) return;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= N) return;
  double acc = 0.0;
  for (int c = lane; c < N; c += 32) acc += Ainv[(size_t)w * N + c] * b[c];
  acc = warp_sum(acc);
  if (lane == 0) x[w] = acc;
}

// ---------------------------------------------------------------------------
// host drivers

// Galerkin hierarchy for a new fine operator `val` (fine minv already set)
void mg_assemble(dp_scene* s, const double* val) {
  MG* mg = s->mg;
  if (!mg) return;
  (void)val;   // the fine level is read from its FP32 copy (s->val32)
  const double* vf = nullptr;
  for (size_t l = 1; l < mg->lv.size(); ++l) {
    MGLevel& L = mg->lv[l];
    if (l == 1 && g_gal8 && DP_VAL32_PACKED == 0)
      k_mg_galerkin8<float><<<grid_for(L.NS * 8, 256), 256, 0, s->stream>>>(
          L.n, L.slice_base, L.diag_slot, L.gal_ptr, L.gal, s->val32, L.val, L.minv, L.slot_row, L.NS);
    else if (l == 1)
      k_mg_galerkin<float, DP_VAL32_PACKED ? 1 : kSlice><<<grid_for(L.NS * 32, 256), 256, 0, s->stream>>>(
          L.n, L.S, L.slice_base, L.slice_width, L.diag_slot, L.gal_ptr, L.gal, s->val32, L.val, L.minv, L.slot_row,
          L.NS, DP_VAL32_PACKED == 2 ? s->val32 + (size_t)s->NS * 8 : nullptr);
    else
      k_mg_galerkin<double, kSlice><<<grid_for(L.NS * 32, 256), 256, 0, s->stream>>>(
          L.n, L.S, L.slice_base, L.slice_width, L.diag_slot, L.gal_ptr, L.gal, vf, L.val, L.minv, L.slot_row, L.NS,
          (const double*)nullptr);
    vf = L.val;
    s->launches++;
  }
  const MGLevel& Lc = mg->lv.back();
  if (mg->coarse_sweeps > 0) return;   // coarsest handled by Jacobi sweeps (in-CTA / in the tail kernel)
  k_mg_dense_build<<<1, 1024, 0, s->stream>>>(Lc.n, Lc.S, Lc.slice_base, Lc.slice_width, Lc.col, Lc.val, mg->dense);
  k_mg_dense_invert<<<1, 256, (size_t)2 * mg->N * mg->N * sizeof(double), s->stream>>>(mg->N, mg->dense, mg->dinv);
  s->launches += 2;
}

// z = B r (one V-cycle), fine operator `val`.  r and z are 3V vectors (z != r).
template <class TV>
static void smooth(dp_scene* s, const MGLevel& L, const TV* val, const TV* minv, const double* b, const double* x,
                   const double* xc, const int* agg, double omega, double* out, double* r_out, const int* stop,
                   double alpha, bool dot = false) {
  MG* mg = s->mg;
  if (dot && mg->dot_ks && out && L.S < 4 * 148) {
    // fine level too small for the one-warp-per-slice kernel: the CTA-per-
    // slice sweep, then the PCG's (r, z) reduction in a launch of its own
    k_mg_smooth<TV, 8><<<L.S, 256, 0, s->stream>>>(L.n, L.S, L.slice_base, L.slice_width, L.col, val, minv, b, x,
                                                   xc, agg, omega, out, r_out, stop, alpha);
    s->launches++;
    launch_pcg_rz(s, b, out, mg->dot_partial, mg->dot_counter, mg->dot_ks);
    return;
  }
  const bool fine = (&L == &mg->lv[0]);
  if (fine) ktm_begin(s, KT_SMOOTH);
  if constexpr (sizeof(TV) == 4) {
    if (fine && g_smooth_pf && !s->val16 && L.S >= 4 * 148 && DP_VAL32_PACKED == 0) {
      const int nb = grid_for((int64_t)L.S * 32, DP_SMOOTH_NT);
      if (dot && mg->dot_ks && out)
        k_mg_smooth_pf<true><<<nb, DP_SMOOTH_NT, 0, s->stream>>>(L.n, L.S, L.slice_base, L.slice_width, L.col, val,
                                                                 minv, b, x, xc, agg, omega, out, r_out, stop, alpha,
                                                                 mg->dot_partial, mg->dot_counter, mg->dot_ks);
      else
        k_mg_smooth_pf<false><<<nb, DP_SMOOTH_NT, 0, s->stream>>>(L.n, L.S, L.slice_base, L.slice_width, L.col, val,
                                                                  minv, b, x, xc, agg, omega, out, r_out, stop, alpha,
                                                                  nullptr, nullptr, nullptr);
      ktm_end(s, KT_SMOOTH);
      s->launches++;
      return;
    }
    if (fine && s->val16 && L.S >= 4 * 148) {
      const int nb = grid_for((int64_t)L.S * 32, DP_SMOOTH_NT);
      if (dot && mg->dot_ks && out)
        k_mg_smooth16<true><<<nb, DP_SMOOTH_NT, 0, s->stream>>>(L.n, L.S, L.slice_base, L.slice_width, L.col,
                                                                s->val16, s->sc16, minv, b, x, xc, agg, omega, out,
                                                                r_out, stop, alpha, mg->dot_partial, mg->dot_counter,
                                                                mg->dot_ks);
      else
        k_mg_smooth16<false><<<nb, DP_SMOOTH_NT, 0, s->stream>>>(L.n, L.S, L.slice_base, L.slice_width, L.col,
                                                                 s->val16, s->sc16, minv, b, x, xc, agg, omega, out,
                                                                 r_out, stop, alpha, nullptr, nullptr, nullptr);
      ktm_end(s, KT_SMOOTH);
      s->launches++;
      return;
    }
  }
  if constexpr (sizeof(TV) == 4) {
    if (fine && g_smooth_bulk && L.S >= 4 * 148 && DP_VAL32_PACKED == 0) {
      const int nb = grid_for((int64_t)L.S * 32, DP_SMOOTH_NT);
#define DP_BULK_LAUNCH(DEPTH)                                                                                       \
  if (dot && mg->dot_ks && out)                                                                                     \
    k_mg_smooth<TV, 1, true, DEPTH><<<nb, DP_SMOOTH_NT, 0, s->stream>>>(L.n, L.S, L.slice_base, L.slice_width, L.col, \
                                                                     val, minv, b, x, xc, agg, omega, out, r_out,  \
                                                                     stop, alpha, mg->dot_partial, mg->dot_counter, \
                                                                     mg->dot_ks);                                   \
  else                                                                                                              \
    k_mg_smooth<TV, 1, false, DEPTH><<<nb, DP_SMOOTH_NT, 0, s->stream>>>(L.n, L.S, L.slice_base, L.slice_width,     \
                                                                      L.col, val, minv, b, x, xc, agg, omega, out, \
                                                                      r_out, stop, alpha);
      DP_BULK_LAUNCH(2)   // depth 3 / 4 measured no faster (and need > 48 KB of static shared memory)
#undef DP_BULK_LAUNCH
      ktm_end(s, KT_SMOOTH);
      s->launches++;
      return;
    }
  }
  if (dot && mg->dot_ks && out && L.S >= 4 * 148)
    k_mg_smooth<TV, 1, true><<<grid_for((int64_t)L.S * 32, DP_SMOOTH_NT), DP_SMOOTH_NT, 0, s->stream>>>(
        L.n, L.S, L.slice_base, L.slice_width, L.col, val, minv, b, x, xc, agg, omega, out, r_out, stop, alpha,
        mg->dot_partial, mg->dot_counter, mg->dot_ks);
  else if (L.S >= 4 * 148)
    k_mg_smooth<TV, 1><<<grid_for((int64_t)L.S * 32, DP_SMOOTH_NT), DP_SMOOTH_NT, 0, s->stream>>>(
        L.n, L.S, L.slice_base, L.slice_width, L.col, val, minv, b, x, xc, agg, omega, out, r_out, stop, alpha);
  else if (sizeof(TV) == 8 && g_coarse_bulk)
    k_mg_smooth<TV, 8, false, 2><<<L.S, 256, 0, s->stream>>>(L.n, L.S, L.slice_base, L.slice_width, L.col, val, minv,
                                                             b, x, xc, agg, omega, out, r_out, stop, alpha);
  else
    k_mg_smooth<TV, 8><<<L.S, 256, 0, s->stream>>>(L.n, L.S, L.slice_base, L.slice_width, L.col, val, minv, b, x,
                                                   xc, agg, omega, out, r_out, stop, alpha);
  if (fine) ktm_end(s, KT_SMOOTH);
  s->launches++;
}

template <class TV>
static void jacobi0(dp_scene* s, const MGLevel& L, const TV* minv, const double* b, double omega, double* x,
                    const int* stop) {
  k_mg_jacobi0<TV><<<grid_for(L.n, 256), 256, 0, s->stream>>>(L.n, minv, b, omega, x, stop);
  s->launches++;
}

template <class TV>
static void vcycle_level(dp_scene* s, int l, const TV* val, const TV* minv, const double* b, double* x,
                         const int* stop, bool pre_done = false);
static const int g_mg_rj0 = getenv("DP_MG_RJ0") ? atoi(getenv("DP_MG_RJ0")) : 1;


// ---------------------------------------------------------------------------
// The two coarsest levels of the V-cycle in ONE launch on a 16-CTA
// thread-block cluster (round 2).  Level a = L-2 (C5: 343 block rows, one
// SELL slice per CTA, one row per warp), level c = L-1 (27 rows, one slice).
// Replaces restrict+jacobi0 (a), residual sweep (a), restrict + the one-CTA
// Jacobi solve (c) and the post-sweep (a): four dependent launches that
// were pure latency (a few hundred KB, L2-resident).
// Each CTA stages its level-a slice and all of level c (values transposed
// to row-major [row][slot][9] so a warp's lanes, one per slot, hit distinct
// banks) in shared memory with cp.async while phase 1 gathers the fine
// residual; the level-a iterate / rhs / residual never leave shared memory:
// other CTAs read them through distributed shared memory (DSMEM) after a
// cluster barrier.  Level c is solved redundantly by every CTA, which saves
// a barrier.  Same operators, smoother and coarse sweeps as the per-level
// kernels (summation order differs: warp trees instead of slot order).
constexpr int kTailCTAs = 16;   // non-portable cluster size (sm_100 allows 16)
constexpr int kTailNT = 1024;   // 32 warps = one level-a slice per CTA
constexpr int kTailMaxC = 32;   // level c: one slice
constexpr int kTailKW = 16;     // warps splitting a level-c row's slots in the coarse sweeps

struct TailArgs {
  // level a (L-2)
  int na;
  const int *sb_a, *sw_a, *col_a;
  const double *val_a, *minv_a;
  const int *mptr_a, *mem_a;      // level-a row -> rows of the level above (rf)
  double* x_a;                    // output
  // level c (L-1)
  int nc;
  const int *sw_c, *col_c;
  const double *val_c, *minv_c;
  const int *mptr_c, *mem_c;      // level-c row -> level-a rows
  const int* agg_c;               // level-a row -> level-c row
  const double* rf;               // residual of the level above level a
  double omega, alpha;
  int sweeps, ka, kc;             // coarse sweeps; shared-memory slot capacity of a / c
  const int* stop;
};

// phase timestamps of CTA 0 (diagnostics: build with -DDP_MG_TAIL_TIMING=1
// and run with DP_MG_TAIL_DBG=1 DP_GRAPHS=0)
#ifndef DP_MG_TAIL_TIMING
#define DP_MG_TAIL_TIMING 0
#endif
__device__ unsigned long long g_tail_clk[12], g_tail_cyc[12];
__device__ __forceinline__ void tail_mark(int k) {
  if (DP_MG_TAIL_TIMING && threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tail_clk[k] = t;
    g_tail_cyc[k] = clock64();
  }
}

// one SELL slice (base, width K) -> row-major shared copies sv[(li K + k) 9 + e], sc[li K + k]
__device__ __forceinline__ void tail_stage_slice(const double* __restrict__ val, const int* __restrict__ col, int base,
                                                 int K, double* sv, int* sc) {
  for (int g = threadIdx.x; g < K * 9 * kSlice; g += blockDim.x) {
    const int li = g % kSlice, ke = g / kSlice, k = ke / 9, e = ke - 9 * k;
    cp_async8(sv + (li * K + k) * 9 + e, val + (size_t)base * 9 + g);
  }
  for (int g = threadIdx.x; g < K * kSlice; g += blockDim.x) {
    const int li = g % kSlice, k = g / kSlice;
    cp_async4(sc + li * K + k, col + base + g);
  }
}

__global__ void __launch_bounds__(kTailNT) k_mg_tail(const __grid_constant__ TailArgs A) {
  extern __shared__ __align__(16) double tsm[];
  if (stopped(A.stop)) return;   // uniform (set by an earlier kernel)
  cg::cluster_group cl = cg::this_cluster();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rank = (int)cl.block_rank();
  const double om = A.omega;
  // shared layout
  double* sv_a = tsm;                                  // [32][ka][9]
  double* sv_c = sv_a + (size_t)kSlice * A.ka * 9;     // [32][kc][9]
  double* sm_a = sv_c + (size_t)kSlice * A.kc * 9;     // minv, [9][32]
  double* sm_c = sm_a + 9 * kSlice;
  double* sxa = sm_c + 9 * kSlice;                     // level-a pre-smoothed iterate (own slice)
  double* sba = sxa + 3 * kSlice;                      // level-a rhs
  double* sra = sba + 3 * kSlice;                      // level-a residual
  double* xs = sra + 3 * kSlice;                       // level-c iterate
  double* ys = xs + 3 * kTailMaxC;
  double* bs = ys + 3 * kTailMaxC;
  double* spc = bs + 3 * kTailMaxC;                    // this slice's part of the level-c rhs
  double* spart = spc + 3 * kTailMaxC;                 // [kTailKW][3][32] partial row sums
  int* sc_a = (int*)(spart + kTailKW * 3 * kSlice);    // [32][ka]
  int* sc_c = sc_a + kSlice * A.ka;                    // [32][kc]
  int* sagg = sc_c + kSlice * A.kc;                    // agg_c
  const int I = rank * kSlice + w;                     // this warp's level-a row
  const bool own = I < A.na;
  const int Ka = rank * kSlice < A.na ? A.sw_a[rank] : 0;
  const int Kc = A.sw_c[0];
  tail_mark(0);
  // prefetch (async) everything phases 2-4 read
  if (rank * kSlice < A.na) tail_stage_slice(A.val_a, A.col_a, A.sb_a[rank], Ka, sv_a, sc_a);
  tail_stage_slice(A.val_c, A.col_c, 0, Kc, sv_c, sc_c);
  for (int g = threadIdx.x; g < 9 * kSlice; g += blockDim.x) {
    const int e = g / kSlice, li = g % kSlice;
    if (rank * kSlice + li < A.na) cp_async8(sm_a + g, A.minv_a + (size_t)e * A.na + rank * kSlice + li);
    if (li < A.nc) cp_async8(sm_c + g, A.minv_c + (size_t)e * A.nc + li);
  }
  for (int g = threadIdx.x; g < A.na; g += blockDim.x) cp_async4(sagg + g, A.agg_c + g);
  asm volatile("cp.async.commit_group;" ::: "memory");
  // phase 1: restriction to level a (gather of the fine residual) and its
  // first Jacobi sweep from zero
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  if (own) {
    for (int t = A.mptr_a[I] + lane; t < A.mptr_a[I + 1]; t += 32) {
      const int i = A.mem_a[t];
      s0 += A.rf[3 * i]; s1 += A.rf[3 * i + 1]; s2 += A.rf[3 * i + 2];
    }
    s0 = warp_sum(s0); s1 = warp_sum(s1); s2 = warp_sum(s2);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (own && lane == 0) {
    sba[3 * w] = s0; sba[3 * w + 1] = s1; sba[3 * w + 2] = s2;
    const double r[3] = {s0, s1, s2};
    double u[3];
    mv_minv(sm_a, kSlice, w, r, u);
    sxa[3 * w] = om * u[0]; sxa[3 * w + 1] = om * u[1]; sxa[3 * w + 2] = om * u[2];
  }
  tail_mark(1);
  cl.sync();
  tail_mark(2);
  // phase 2: residual of level a after the pre-sweep (x of other slices via DSMEM)
  if (own) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int k = lane; k < Ka; k += 32) {
      const int j = sc_a[w * Ka + k];
      const double* v = sv_a + (w * Ka + k) * 9;
      const double* xr = cl.map_shared_rank(sxa, j / kSlice) + 3 * (j % kSlice);
      const double x0 = xr[0], x1 = xr[1], x2 = xr[2];
      a0 += v[0] * x0 + v[1] * x1 + v[2] * x2;
      a1 += v[3] * x0 + v[4] * x1 + v[5] * x2;
      a2 += v[6] * x0 + v[7] * x1 + v[8] * x2;
    }
    a0 = warp_sum(a0); a1 = warp_sum(a1); a2 = warp_sum(a2);
    if (lane == 0) {
      sra[3 * w] = sba[3 * w] - a0; sra[3 * w + 1] = sba[3 * w + 1] - a1; sra[3 * w + 2] = sba[3 * w + 2] - a2;
    }
  }
  __syncthreads();
  // this slice's contribution to the level-c restriction (rows in order)
  if (w == 0 && lane < A.nc) {
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    const int nr = min(kSlice, A.na - rank * kSlice);
    for (int li = 0; li < nr; ++li)
      if (sagg[rank * kSlice + li] == lane) { t0 += sra[3 * li]; t1 += sra[3 * li + 1]; t2 += sra[3 * li + 2]; }
    spc[3 * lane] = t0; spc[3 * lane + 1] = t1; spc[3 * lane + 2] = t2;
  }
  tail_mark(3);
  cl.sync();
  tail_mark(4);
  // phase 3 (every CTA): restriction to level c = sum over the cluster's
  // CTAs of their per-slice partial sums (DSMEM, fixed CTA order), and
  // k_mg_coarse_jacobi's iteration x = w Minv b, then `sweeps` times
  // x <- x + w Minv (b - A x)
  if (w == 0 && lane < A.nc) {
    double t0 = 0.0, t1 = 0.0, t2 = 0.0, p[3 * kTailCTAs];
#pragma unroll
    for (int q = 0; q < kTailCTAs; ++q) {   // all loads in flight, then the ordered sum
      const double* pr = cl.map_shared_rank(spc, q) + 3 * lane;
      p[3 * q] = pr[0]; p[3 * q + 1] = pr[1]; p[3 * q + 2] = pr[2];
    }
#pragma unroll
    for (int q = 0; q < kTailCTAs; ++q) { t0 += p[3 * q]; t1 += p[3 * q + 1]; t2 += p[3 * q + 2]; }
    bs[3 * lane] = t0; bs[3 * lane + 1] = t1; bs[3 * lane + 2] = t2;
    const double r[3] = {t0, t1, t2};
    double u[3];
    mv_minv(sm_c, kSlice, lane, r, u);
    xs[3 * lane] = om * u[0]; xs[3 * lane + 1] = om * u[1]; xs[3 * lane + 2] = om * u[2];
  }
  __syncthreads();
  tail_mark(7);
  const double* xcs = xs;
  // sweeps: lane = level-c row, warps split the row's slots (partial sums
  // in shared memory), ping-pong iterates: two block barriers per sweep
  {
    double* xc = xs;
    double* yc = ys;
    for (int it = 0; it < A.sweeps; ++it) {
      if (w < kTailKW) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        if (lane < A.nc) {
          for (int k = w; k < Kc; k += kTailKW) {
            const int j = sc_c[lane * Kc + k];
            const double* v = sv_c + (lane * Kc + k) * 9;
            const double x0 = xc[3 * j], x1 = xc[3 * j + 1], x2 = xc[3 * j + 2];
            a0 += v[0] * x0 + v[1] * x1 + v[2] * x2;
            a1 += v[3] * x0 + v[4] * x1 + v[5] * x2;
            a2 += v[6] * x0 + v[7] * x1 + v[8] * x2;
          }
        }
        spart[(w * 3 + 0) * kSlice + lane] = a0;
        spart[(w * 3 + 1) * kSlice + lane] = a1;
        spart[(w * 3 + 2) * kSlice + lane] = a2;
      }
      __syncthreads();
      if (w == 0 && lane < A.nc) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
        for (int q = 0; q < kTailKW; ++q) {
          a0 += spart[(q * 3 + 0) * kSlice + lane];
          a1 += spart[(q * 3 + 1) * kSlice + lane];
          a2 += spart[(q * 3 + 2) * kSlice + lane];
        }
        const double r[3] = {bs[3 * lane] - a0, bs[3 * lane + 1] - a1, bs[3 * lane + 2] - a2};
        double u[3];
        mv_minv(sm_c, kSlice, lane, r, u);
#pragma unroll
        for (int c = 0; c < 3; ++c) yc[3 * lane + c] = xc[3 * lane + c] + om * u[c];
      }
      __syncthreads();
      double* t = xc; xc = yc; yc = t;
    }
    xcs = xc;
  }
  tail_mark(5);
  // phase 4: post-sweep of level a with the coarse correction in its gathers
  const double* xcr = xcs;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  if (own) {
    for (int k = lane; k < Ka; k += 32) {
      const int j = sc_a[w * Ka + k];
      const double* v = sv_a + (w * Ka + k) * 9;
      const double* xr = cl.map_shared_rank(sxa, j / kSlice) + 3 * (j % kSlice);
      const int J = sagg[j];
      const double x0 = xr[0] + A.alpha * xcr[3 * J], x1 = xr[1] + A.alpha * xcr[3 * J + 1],
                   x2 = xr[2] + A.alpha * xcr[3 * J + 2];
      a0 += v[0] * x0 + v[1] * x1 + v[2] * x2;
      a1 += v[3] * x0 + v[4] * x1 + v[5] * x2;
      a2 += v[6] * x0 + v[7] * x1 + v[8] * x2;
    }
    a0 = warp_sum(a0); a1 = warp_sum(a1); a2 = warp_sum(a2);
  }
  cl.barrier_arrive();   // last remote (DSMEM) read done; the wait below keeps our shared memory alive for the others
  if (own && lane == 0) {
    const int J = sagg[I];
    const double a[3] = {a0, a1, a2};
    double xt[3], r[3], u[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      xt[c] = sxa[3 * w + c] + A.alpha * xcr[3 * J + c];
      r[c] = sba[3 * w + c] - a[c];
    }
    mv_minv(sm_a, kSlice, w, r, u);
#pragma unroll
    for (int c = 0; c < 3; ++c) A.x_a[3 * I + c] = xt[c] + om * u[c];
  }
  tail_mark(6);
  cl.barrier_wait();
}

static size_t tail_smem_bytes(int na, int nc, int ka, int kc) {
  return sizeof(double) * ((size_t)kSlice * (ka + kc) * 9 + 2 * 9 * kSlice + 3 * 3 * kSlice + 4 * 3 * kTailMaxC +
                            kTailKW * 3 * kSlice) +
         sizeof(int) * ((size_t)kSlice * (ka + kc) + (size_t)na);
}

// the cluster size the device launches k_mg_tail with (0: none)
static int tail_cluster(size_t smem) {
  static int ok = -1;
  static size_t ok_smem = 0;
  if (ok >= 0 && ok_smem >= smem) return ok;
  cudaFuncSetAttribute(k_mg_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_mg_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kTailCTAs);
  cfg.blockDim = dim3(kTailNT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kTailCTAs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_mg_tail, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  ok = n > 0 ? kTailCTAs : 0;
  ok_smem = smem;
  return ok;
}

static int g_tail_failed = 0;   // a cluster launch was refused: per-level V-cycle from then on

// usable for the level pair (l, l+1) = (L-2, L-1)
static bool tail_usable(const MG* mg, int la) {
  const int L = (int)mg->lv.size();
  if (!(g_mg_tail && !g_tail_failed && L >= 2 && la == L - 2 && la >= 1 && mg->nu == 1 && mg->gamma == 1 && mg->coarse_sweeps > 0 &&
        (mg->post == 1 || mg->symmetric_needed)))
    return false;
  const MGLevel &a = mg->lv[L - 2], &c = mg->lv[L - 1];
  if (c.n > kTailMaxC || a.n > kSlice * kTailCTAs) return false;
  const size_t smem = tail_smem_bytes(a.n, c.n, a.kmax, c.kmax);
  return smem <= 200 * 1024 && tail_cluster(smem) > 0;
}

// false: the launch was refused (the caller runs the per-level kernels)
static bool launch_tail(dp_scene* s, const double* rf, const int* stop) {
  MG* mg = s->mg;
  const int L = (int)mg->lv.size();
  MGLevel& a = mg->lv[L - 2];
  MGLevel& c = mg->lv[L - 1];
  TailArgs A;
  A.na = a.n; A.sb_a = a.slice_base; A.sw_a = a.slice_width; A.col_a = a.col; A.val_a = a.val; A.minv_a = a.minv;
  A.mptr_a = a.mem_ptr; A.mem_a = a.mem; A.x_a = a.x;
  A.nc = c.n; A.sw_c = c.slice_width; A.col_c = c.col; A.val_c = c.val; A.minv_c = c.minv;
  A.mptr_c = c.mem_ptr; A.mem_c = c.mem; A.agg_c = c.agg;
  A.rf = rf; A.omega = mg->omega; A.alpha = mg->alpha; A.sweeps = mg->coarse_sweeps; A.stop = stop;
  A.ka = a.kmax; A.kc = c.kmax;
  const size_t smem = tail_smem_bytes(a.n, c.n, a.kmax, c.kmax);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kTailCTAs);
  cfg.blockDim = dim3(kTailNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kTailCTAs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, k_mg_tail, A) != cudaSuccess) {
    cudaGetLastError();
    g_tail_failed = 1;
    return false;
  }
  s->launches++;
  if (DP_MG_TAIL_TIMING && getenv("DP_MG_TAIL_DBG")) {
    static double acc[9];
    static long cnt = 0;
    unsigned long long t[12];
    host_sync(s);
    cudaMemcpyFromSymbol(t, g_tail_clk, sizeof(t));
    unsigned long long cy[12];
    cudaMemcpyFromSymbol(cy, g_tail_cyc, sizeof(cy));
    static double cacc[8];
    for (int k = 1; k < 7; ++k) cacc[k] += (double)(cy[k] - cy[k - 1]);
    cacc[7] += (double)(cy[7] - cy[4]);
    if (t[6] > t[0]) {
      for (int k = 1; k < 7; ++k) acc[k] += (double)(t[k] - t[k - 1]);
      acc[7] += (double)(t[7] - t[4]);
      if (++cnt % 200 == 0)
        fprintf(stderr, "tail phases ns: p1 %.0f sync %.0f p2 %.0f sync %.0f p3 %.0f p4 %.0f restrict_c %.0f (n=%ld) "
                "nc %d na %d ka %d kc %d smem %zu\n",
                acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, acc[5] / cnt, acc[6] / cnt, acc[7] / cnt,
                cnt, A.nc, A.na, A.ka, A.kc, smem);
      if (cnt % 200 == 0)
        fprintf(stderr, "tail phases cycles: p1 %.0f sync %.0f p2 %.0f sync %.0f p3 %.0f p4 %.0f restrict_c %.0f\n",
                cacc[1] / cnt, cacc[2] / cnt, cacc[3] / cnt, cacc[4] / cnt, cacc[5] / cnt, cacc[6] / cnt, cacc[7] / cnt);
    }
  }
  return true;
}

static const int g_mg_fused_env = getenv("DP_MG_FUSED") ? atoi(getenv("DP_MG_FUSED")) : 0;

static bool fused_usable(const MG* mg) {
  return g_mg_fused_env && mg->fused && mg->fused_grid > 0 && mg->nu == 1 && mg->post == 1 && mg->gamma == 1 &&
         mg->coarse_sweeps > 0 && mg->lv.size() >= 2 && mg->lv.size() <= (size_t)kMaxFusedLevels &&
         mg->lv.back().n <= kCoarseMax;
}

// levels 1..L-1 of the V-cycle for the fine residual r0 -> lv[1].x
static void launch_coarse_fused(dp_scene* s, const double* r0, const int* stop) {
  MG* mg = s->mg;
  FusedArgs a;
  a.L = (int)mg->lv.size();
  for (int l = 1; l < a.L; ++l) {
    const MGLevel& L = mg->lv[l];
    FusedLevel& f = a.lv[l];
    f.n = L.n; f.S = L.S;
    f.slice_base = L.slice_base; f.slice_width = L.slice_width; f.col = L.col;
    f.val = L.val; f.minv = L.minv;
    f.mem_ptr = L.mem_ptr; f.mem = L.mem; f.agg = L.agg;
    f.x = L.x; f.b = L.b; f.r = L.r; f.t = L.t;
  }
  a.r0 = r0;
  a.omega = mg->omega;
  a.alpha = mg->alpha;
  a.coarse_sweeps = mg->coarse_sweeps;
  a.stop = stop;
  a.tstamp = nullptr;
  static const int ftime = getenv("DP_MG_FTIME") ? atoi(getenv("DP_MG_FTIME")) : 0;
  static unsigned long long* dts = nullptr;
  static long calls = 0;
  if (ftime) {
    // diagnostics only: phase stamps of one call in 64, printed on the host
    if (!dts) cudaMalloc(&dts, 64 * sizeof(unsigned long long));
    if (calls % 64 == 63) {
      unsigned long long h[64];
      host_sync(s);
      cudaMemcpy(h, dts, sizeof(h), cudaMemcpyDeviceToHost);
      fprintf(stderr, "[mg-fused] L=%d phases(us):", a.L);
      for (int i = 1; i < 32 && h[i]; ++i) fprintf(stderr, " %.2f", (h[i] - h[i - 1]) * 1e-3);
      fprintf(stderr, "\n");
    }
    if (calls % 64 == 62) {
      cudaMemsetAsync(dts, 0, 64 * sizeof(unsigned long long), s->stream);
      a.tstamp = dts;
    }
    ++calls;
  }
  void* args[] = {&a};
  cudaLaunchCooperativeKernel((const void*)k_mg_coarse_fused, dim3(mg->fused_grid), dim3(256), args, 0, s->stream);
  s->launches++;
}

static void vcycle(dp_scene* s, int l, const double* b, double* x, const int* stop) {
  MG* mg = s->mg;
  if (l == (int)mg->lv.size() - 1) {
    if (mg->coarse_sweeps > 0) {
      const MGLevel& Lc = mg->lv[l];
      k_mg_coarse_jacobi<<<1, 256, 0, s->stream>>>(Lc.n, Lc.S, Lc.slice_base, Lc.slice_width, Lc.col, Lc.val, Lc.minv,
                                                   const_cast<double*>(b), x, Lc.t, mg->omega, mg->coarse_sweeps, stop,
                                                   nullptr, nullptr, nullptr);
    } else {
      k_mg_dense_solve<<<grid_for((int64_t)mg->N * 32, 256), 256, 0, s->stream>>>(mg->N, mg->dinv, b, x, stop);
    }
    s->launches++;
    return;
  }
  if (l == 0) vcycle_level<float>(s, 0, s->val32, s->minv32, b, x, stop);
  else vcycle_level<double>(s, l, mg->lv[l].val, mg->lv[l].minv, b, x, stop);
}

template <class TV>
static void vcycle_level(dp_scene* s, int l, const TV* val, const TV* minv, const double* b, double* x,
                         const int* stop, bool pre_done) {
  MG* mg = s->mg;
  MGLevel& L = mg->lv[l];
  MGLevel& C = mg->lv[l + 1];
  const double om = mg->omega;
  // pre-smoothing from zero: x = w Minv b, then nu-1 sweeps; last pass also gives r
  double* xa = L.t;   // work buffers never alias the output x
  double* xb = L.u;
  // the fine-level first sweep from zero may already be done by the caller
  // (k_gm_prec fuses it into the basis-vector pass): mg_apply(..., prejac)
  if (!pre_done && !(l == 0 && mg->prejac)) jacobi0<TV>(s, L, minv, b, om, xa, stop);
  for (int it = 1; it < mg->nu; ++it) {
    smooth<TV>(s, L, val, minv, b, xa, nullptr, nullptr, om, xb, nullptr, stop, 1.0);
    std::swap(xa, xb);
  }
  // coarse-grid corrections: one at the fine level (V-cycle), `gamma` at the
  // coarse levels (gamma = 2: W-cycle below the fine level, cheap there)
  const int ncorr = (l == 0) ? 1 : mg->gamma;
  for (int g = 0; g < ncorr; ++g) {
    smooth<TV>(s, L, val, minv, b, xa, nullptr, nullptr, om, nullptr, L.r, stop, 1.0);
    if (l == 0 && fused_usable(mg)) {
      launch_coarse_fused(s, L.r, stop);   // restriction to level 1 is its first phase
    } else if (tail_usable(mg, l + 1) && launch_tail(s, L.r, stop)) {
      // levels l+1 and l+2 in one cluster launch -> C.x (a refused launch
      // falls through to the per-level kernels below)
    } else if (g_mg_rj0 && l + 1 == (int)mg->lv.size() - 1 && mg->coarse_sweeps > 0) {
      // coarsest level: the restriction is the first phase of its one-CTA solve
      k_mg_coarse_jacobi<<<1, 256, 0, s->stream>>>(C.n, C.S, C.slice_base, C.slice_width, C.col, C.val, C.minv, C.b,
                                                   C.x, C.t, om, mg->coarse_sweeps, stop, C.mem_ptr, C.mem, L.r);
      s->launches++;
    } else if (g_mg_rj0 && l + 1 < (int)mg->lv.size() - 1) {
      // restriction and the coarse level's first Jacobi sweep from zero in one launch
      k_mg_restrict_j0<double><<<grid_for((int64_t)C.n * 32, 256), 256, 0, s->stream>>>(
          C.n, C.mem_ptr, C.mem, L.r, C.b, C.minv, om, C.t, stop);
      s->launches++;
      vcycle_level<double>(s, l + 1, C.val, C.minv, C.b, C.x, stop, true);
    } else {
      k_mg_restrict<<<grid_for((int64_t)C.n * 32, 256), 256, 0, s->stream>>>(C.n, C.mem_ptr, C.mem, L.r, C.b, stop);
      s->launches++;
      vcycle(s, l + 1, C.b, C.x, stop);
    }
    const bool last = (g == ncorr - 1);
    if (mg->post == 0 && !mg->symmetric_needed && last) {
      // V(nu,0): x = x_pre + alpha P x_c (no post-smoothing SpMV)
      k_mg_prolong<<<grid_for(L.n, 256), 256, 0, s->stream>>>(L.n, xa, C.x, C.agg, mg->alpha, x, stop);
      s->launches++;
      return;
    }
    // post-smoothing; the first sweep applies the coarse correction in its gathers
    for (int it = 0; it < mg->nu; ++it) {
      double* dst = (last && it == mg->nu - 1) ? x : xb;
      smooth<TV>(s, L, val, minv, b, xa, it == 0 ? C.x : nullptr, it == 0 ? C.agg : nullptr, om, dst, nullptr, stop,
                 mg->alpha, l == 0 && dst == x);
      if (dst == xb) std::swap(xa, xb);
    }
  }
}

// PCG fusion (pcg_mg_solve): the fine level's final post-smoothing sweep of
// every V-cycle forms (r, z) and the CG beta; nullptr ks switches it off
void mg_set_pcg_dot(dp_scene* s, double* partial, unsigned int* counter, KrylovScalars* ks) {
  if (!s->mg) return;
  s->mg->dot_partial = partial;
  s->mg->dot_counter = counter;
  s->mg->dot_ks = ks;
}

void mg_set_symmetric(dp_scene* s, int on) {
  if (s->mg) {
    s->mg->symmetric_needed = on;
    s->mg->alpha = on ? s->mg->alpha_cg : s->mg->alpha_gm;
  }
}

// one fine-level damped block-Jacobi sweep out = x + w Minv32 (b - A32 x)
// (the V-cycle's dominant kernel) `reps` times, for the bench roofline
int mg_bench_fine_smooth(dp_scene* s, const double* x, const double* b, double* out, int reps) {
  MG* mg = s->mg;
  if (!mg || !s->val32) return 1;
  const MGLevel& L = mg->lv[0];
  for (int r = 0; r < reps; ++r)
    smooth<float>(s, L, s->val32, s->minv32, b, x, nullptr, nullptr, mg->omega, out, nullptr, nullptr, 1.0);
  return 0;
}

void mg_fine_jacobi0_target(dp_scene* s, const float** minv32, double** xa, double* omega) {
  *minv32 = s->minv32;
  *xa = s->mg->lv[0].t;
  *omega = s->mg->omega;
}

void mg_apply_prejac(dp_scene* s, const double* val, const double* r, double* z, const int* stop) {
  s->mg->prejac = 1;
  mg_apply(s, val, r, z, stop);
  s->mg->prejac = 0;
}

void mg_apply(dp_scene* s, const double* val, const double* r, double* z, const int* stop) {
  (void)val;   // the V-cycle uses the operator assembled by the last mg_assemble
  vcycle(s, 0, r, z, stop);
}

}  // namespace dp
