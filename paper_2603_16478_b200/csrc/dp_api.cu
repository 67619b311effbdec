// C ABI of libdiffproj_b200.so: scene setup, the Newton driver of the
// implicit step, the adjoint, and the unit-level batch entry points.
// See include/diffproj_b200.h for the reference function each one replaces.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "dp_internal.h"
#include "dp_math.cuh"

namespace dp {
std::recursive_mutex& api_mutex() {
  static std::recursive_mutex mu;
  return mu;
}

// keeps the GPU busy for ~ns while the host queues a timed launch behind it
__global__ void k_ktm_spin(long long ns) {
  long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

void ktm_begin(dp_scene* s, int k) {
  if (!s->timing) return;
  if (s->stream_drained) {
    // right after a host wait the stream is empty: without this the begin
    // event would fire at once and the interval would include the host's
    // own launch latency for the kernel (not the kernel's duration)
    k_ktm_spin<<<1, 1, 0, s->stream>>>(30000);
    s->stream_drained = 0;
  }
  dp_scene::KSlot& t = s->kslot[k];
  if (t.used == (int)t.a.size()) {
    if (t.used >= 8192) {   // bound the pool: resolve what is recorded so far
      ktm_flush(s);
    } else {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      t.a.push_back(a);
      t.b.push_back(b);
    }
  }
  cudaEventRecord(t.a[t.used], s->stream);
}

void ktm_end(dp_scene* s, int k) {
  if (!s->timing) return;
  dp_scene::KSlot& t = s->kslot[k];
  cudaEventRecord(t.b[t.used], s->stream);
  ++t.used;
}

void ktm_flush(dp_scene* s) {
  bool any = false;
  for (auto& t : s->kslot) any |= t.used > 0;
  if (!any) return;
  host_sync(s);
  double* ms_of[] = {&s->times.spmv_ms, &s->times.elem_jac_ms, &s->times.elem_res_ms, &s->times.assemble_ms,
                     &s->times.smooth_ms, &s->times.pcg_spmv_ms};
  int64_t* n_of[] = {&s->times.spmv_calls, &s->times.elem_jac_calls, &s->times.elem_res_calls,
                     &s->times.assemble_calls, &s->times.smooth_calls, &s->times.pcg_spmv_calls};
  for (int k = 0; k < 6; ++k) {
    dp_scene::KSlot& t = s->kslot[k];
    for (int i = 0; i < t.used; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, t.a[i], t.b[i]);
      *ms_of[k] += ms;
    }
    *n_of[k] += t.used;
    t.used = 0;
  }
}

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string("CUDA error ") + cudaGetErrorString(e) + " at " + where;
  return DP_ERR_CUDA;
}

int grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)b;
}

// launchers defined in the other translation units
void launch_project_batch(int n, int d, const double* F, const int* model, const double* mu, const double* lam,
                          double tau_rel, double* sigma, double* theta, double* W, double* P, double* J, double* dPmu,
                          double* dPlam, int* status);
void launch_contact_batch(int n, const double* frame, const double* dn, const double* mu, const double* eps2,
                          const double* x, const double* xb, double* lam, double* delta, double* s_signed, int* capped,
                          double* Kc, double* kmu, double* residual, int* status);
void launch_export_proj(dp_scene* s, const double* q, double* sigma, double* theta, double* P, double* energy);

template <class T>
static int dalloc(dp_scene* s, T** p, size_t n) {
  if (n == 0) n = 1;
  DP_CUDA(cudaMalloc((void**)p, n * sizeof(T)));
  s->bytes += n * sizeof(T);
  return 0;
}

template <class T>
static int upload(dp_scene* s, T** p, const std::vector<T>& h) {
  int rc = dalloc(s, p, h.size());
  if (rc) return rc;
  if (!h.empty()) DP_CUDA(cudaMemcpy(*p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return 0;
}

static void dfree(void* p) {
  if (p) cudaFree(p);
}

// copy n doubles into device buffer dst from a host or device pointer
static int copy_in(dp_scene* s, double* dst, const double* src, size_t n, int ptr_kind) {
  DP_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double),
                          ptr_kind == DP_PTR_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s->stream));
  return 0;
}
static int copy_out(dp_scene* s, double* dst, const double* src, size_t n, int ptr_kind) {
  DP_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double),
                          ptr_kind == DP_PTR_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s->stream));
  return 0;
}

static int sync_esc(dp_scene* s) {
  DP_CUDA(cudaMemcpyAsync(s->h_esc, s->esc, sizeof(EvalScalars), cudaMemcpyDeviceToHost, s->stream));
  DP_CUDA(host_sync(s));
  return 0;
}

// contact capacity = V * n_colliders (every vertex may touch every collider)
static int ensure_contact_capacity(dp_scene* s, int cap) {
  if (cap <= s->ccap) return 0;
  dfree(s->c_vertex); dfree(s->c_collider); dfree(s->c_frame); dfree(s->c_dn); dfree(s->c_mu);
  dfree(s->c_delta); dfree(s->c_blk); dfree(s->c_force); dfree(s->c_kmu); dfree(s->c_kc);
  int rc = 0;
  rc |= dalloc(s, &s->c_vertex, cap);
  rc |= dalloc(s, &s->c_collider, cap);
  rc |= dalloc(s, &s->c_frame, (size_t)cap * 9);
  rc |= dalloc(s, &s->c_dn, cap);
  rc |= dalloc(s, &s->c_mu, cap);
  rc |= dalloc(s, &s->c_delta, (size_t)cap * 3);
  rc |= dalloc(s, &s->c_blk, (size_t)cap * 9);
  rc |= dalloc(s, &s->c_force, (size_t)cap * 3);
  rc |= dalloc(s, &s->c_kmu, (size_t)cap * 3);
  rc |= dalloc(s, &s->c_kc, (size_t)cap * 9);
  if (rc) return rc;
  s->ccap = cap;
  return 0;
}

__global__ void k_count_contacts(int C, const int* __restrict__ vtx, int* __restrict__ count) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  // contacts are sorted by vertex: the first contact of a run counts the run
  if (c == 0 || vtx[c - 1] != vtx[c]) {
    int k = c + 1;
    while (k < C && vtx[k] == vtx[c]) ++k;
    count[vtx[c]] = k - c;
  }
}

__global__ void k_offsets_from_list(int C, const int* __restrict__ vtx, int* __restrict__ off) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  if (c == 0 || vtx[c - 1] != vtx[c]) off[vtx[c]] = c;
}

// load a cached contact list into the scene's per-vertex contact buffers
static int load_cache_contacts(dp_scene* s, const dp_cache* c) {
  const int C = c->n_contacts;
  int rc = ensure_contact_capacity(s, std::max(C, 1));
  if (rc) return rc;
  DP_CUDA(cudaMemsetAsync(s->c_count, 0, sizeof(int) * (s->V + 1), s->stream));
  DP_CUDA(cudaMemsetAsync(s->c_off, 0, sizeof(int) * (s->V + 1), s->stream));
  if (C == 0) return 0;
  DP_CUDA(cudaMemcpyAsync(s->c_vertex, c->c_vertex, sizeof(int) * C, cudaMemcpyDeviceToDevice, s->stream));
  DP_CUDA(cudaMemcpyAsync(s->c_collider, c->c_collider, sizeof(int) * C, cudaMemcpyDeviceToDevice, s->stream));
  DP_CUDA(cudaMemcpyAsync(s->c_frame, c->c_frame, sizeof(double) * C * 9, cudaMemcpyDeviceToDevice, s->stream));
  DP_CUDA(cudaMemcpyAsync(s->c_dn, c->c_dn, sizeof(double) * C, cudaMemcpyDeviceToDevice, s->stream));
  DP_CUDA(cudaMemcpyAsync(s->c_mu, c->c_mu, sizeof(double) * C, cudaMemcpyDeviceToDevice, s->stream));
  DP_CUDA(cudaMemcpyAsync(s->c_delta, c->c_delta, sizeof(double) * C * 3, cudaMemcpyDeviceToDevice, s->stream));
  k_count_contacts<<<grid_for(C, 256), 256, 0, s->stream>>>(C, s->c_vertex, s->c_count);
  k_offsets_from_list<<<grid_for(C, 256), 256, 0, s->stream>>>(C, s->c_vertex, s->c_off);
  s->launches += 2;
  return 0;
}

static int raise_status(int st) {
  if (st & (ST_INVERTED | ST_NONFINITE)) {
    set_error("inverted element: det F <= 0");
    return DP_ERR_INVERTED;
  }
  if (st & ST_NH_STALL) {
    set_error("neo-hookean projection stalled");
    return DP_ERR_NH_STALL;
  }
  if (st & ST_PENETRATION) {
    set_error("contact multiplier solve requires delta_n > 0");
    return DP_ERR_PENETRATION;
  }
  return DP_OK;
}

// Thread-local device scratch arena for the unit-level batch entry points
// (dp_project_batch, dp_contact_batch, dp_cache_get_projections): grown on
// demand and reused, so repeated calls (e.g. a report's contacts read every
// step) do not pay cudaMalloc/cudaFree each time.
struct ScratchArena {
  int dev = -1;
  char* base = nullptr;
  size_t cap = 0, used = 0;
  ~ScratchArena() {
    if (base) cudaFree(base);
  }
};
static thread_local ScratchArena g_scratch;

static int scratch_reserve(size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_scratch.dev != dev || bytes > g_scratch.cap) {
    if (g_scratch.base && g_scratch.dev == dev) cudaFree(g_scratch.base);
    g_scratch.base = nullptr;
    g_scratch.cap = 0;
    const size_t cap = bytes + bytes / 2 + 4096;
    if (cudaMalloc((void**)&g_scratch.base, cap) != cudaSuccess) return DP_ERR_CUDA;
    g_scratch.cap = cap;
    g_scratch.dev = dev;
  }
  g_scratch.used = 0;
  return 0;
}

template <class T>
static T* scratch_take(size_t n) {
  const size_t off = (g_scratch.used + 255) & ~(size_t)255;
  g_scratch.used = off + n * sizeof(T);
  return reinterpret_cast<T*>(g_scratch.base + off);
}

static size_t scratch_bytes(std::initializer_list<size_t> sizes) {
  size_t t = 0;
  for (size_t b : sizes) t += ((b + 255) & ~(size_t)255);
  return t;
}

}  // namespace dp

using namespace dp;

static const int g_debug = getenv("DP_DEBUG") ? atoi(getenv("DP_DEBUG")) : 0;
// line search: penetration of all trials tested with the first (DP_PEN_MASK=0 off)
static const int g_pen_mask = getenv("DP_PEN_MASK") ? atoi(getenv("DP_PEN_MASK")) : 1;
// after a line search that had to cut the step below 1/16 the Newton model is
// poor (friction-cone / activation kinks): a cheap direction is enough
static const int g_precheck = getenv("DP_LS_PRECHECK") ? atoi(getenv("DP_LS_PRECHECK")) : 1;
static const double g_watch_frac = getenv("DP_LS_WATCH_FRAC") ? atof(getenv("DP_LS_WATCH_FRAC")) : 0.5;
// line-search trials evaluate the elements with their Jacobian blocks: an
// accepted trial point is the next Newton point, whose element pass (forward.py
// :186-192 projects the elements at q again) is then already done
static const int g_spec_jac = getenv("DP_LS_SPECJAC") ? atoi(getenv("DP_LS_SPECJAC")) : 1;
static const int g_ls_norm = getenv("DP_LS_NORM") ? atoi(getenv("DP_LS_NORM")) : 0;
static const int g_newton_x0 = getenv("DP_NEWTON_X0") ? atoi(getenv("DP_NEWTON_X0")) : 1;
// adjoint PCG with the FP32 operator copy inside the iterations and FP64
// iterative refinement (pcg_mg_solve); the 1e-10 stop test stays FP64
static const int g_adj_fp32 = getenv("DP_ADJ_FP32") ? atoi(getenv("DP_ADJ_FP32")) : 1;
// FP32 element block stream + FP32-only forward operator for frictionless
// multigrid-PCG steps (EV_H32)
static const int g_fwd_h32 = getenv("DP_FWD_H32") ? atoi(getenv("DP_FWD_H32")) : 1;
static const double g_eta_near = getenv("DP_ETA_NEAR") ? atof(getenv("DP_ETA_NEAR")) : 1000.0;
static const double g_eta_plateau = getenv("DP_ETA_PLATEAU") ? atof(getenv("DP_ETA_PLATEAU")) : 0.0;
static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// host setup: body(lo, hi) over [0, n) split into contiguous chunks on up to
// 16 threads (each chunk's output is written by its own thread only)
template <class F>
static void parallel_chunks(int64_t n, F body) {
  int nt = (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
  if (n < 4096) nt = 1;
  if (nt == 1) { body((int64_t)0, n); return; }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) {
    const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
    th.emplace_back([=] { body(lo, hi); });
  }
  for (auto& x : th) x.join();
}

// ===========================================================================
extern "C" {

const char* dp_last_error(void) { return g_err.c_str(); }
const char* dp_version(void) { return "diffproj_b200 0.1 (sm_100a)"; }
// Any entry point that writes the scene's contact / element scratch, the
// forward operator values or the multigrid level values makes the assembled
// adjoint operator stale: the next adjoint solve / backprop of any cache
// re-assembles (the reference's caches are immutable, so an interleaved
// forward step must not change a later backprop_step's result).
static inline void invalidate_adjoint(dp_scene* s) {
  s->adj_cache_tag = nullptr;
  s->mg_adj_ready = 0;
}

int dp_pinned_alloc(int64_t bytes, void** out) {
  *out = nullptr;
  if (bytes <= 0) { set_error("pinned allocation size must be positive"); return DP_ERR_VALUE; }
  DP_CUDA(cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable));
  return DP_OK;
}

int dp_pinned_free(void* p) {
  if (p) DP_CUDA(cudaFreeHost(p));
  return DP_OK;
}

int dp_set_spin_wait(int32_t device, int32_t mode) {
  // mode 1 spin, 2 yield, 4 blocking sync, 0 leave as is.  The primary
  // context's flags can be changed while it is active; the driver entry point
  // is resolved at run time so the library does not link libcuda.
  if (mode == 0) return DP_OK;
  typedef CUresult (*set_flags_t)(CUdevice, unsigned int);
  typedef CUresult (*dev_get_t)(CUdevice*, int);
  void* f1 = nullptr;
  void* f2 = nullptr;
  cudaDriverEntryPointQueryResult q1, q2;
  if (cudaGetDriverEntryPoint("cuDevicePrimaryCtxSetFlags", &f1, cudaEnableDefault, &q1) != cudaSuccess ||
      cudaGetDriverEntryPoint("cuDeviceGet", &f2, cudaEnableDefault, &q2) != cudaSuccess || !f1 || !f2) {
    cudaGetLastError();
    return DP_ERR_NO_DEVICE;
  }
  CUdevice dev;
  if (((dev_get_t)f2)(&dev, device) != CUDA_SUCCESS) return DP_ERR_NO_DEVICE;
  const unsigned f = mode == 1 ? CU_CTX_SCHED_SPIN : mode == 2 ? CU_CTX_SCHED_YIELD : CU_CTX_SCHED_BLOCKING_SYNC;
  if (((set_flags_t)f1)(dev, f) != CUDA_SUCCESS) return DP_ERR_CUDA;
  return DP_OK;
}

int dp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

void dp_forward_cfg_default(dp_forward_cfg* c) {
  c->tol = 1e-9;
  c->max_iter = 100;
  c->max_line_search = 40;
  c->pullback_margin = 1e-6;
  c->lin_rtol_max = 1e-2;   // while max|r| > 1000 tol
  c->lin_rtol_min = 1e-3;   // once max|r| <= 1000 tol
  c->lin_max_iter = 5000;
  c->gmres_restart = 50;
}

void dp_solver_cfg_default(dp_solver_cfg* c) {
  c->method = DP_SOLVER_AUTO;
  c->tol = 1e-10;
  c->max_iter = 2000;
  c->gmres_restart = 50;
}

// ---------------------------------------------------------------------------
// scene

int dp_scene_create(const dp_scene_desc* d, dp_scene** out) {
  std::lock_guard<std::recursive_mutex> api_lock(dp::api_mutex());
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_error("no CUDA device available: the diffproj_b200 CUDA path requires a GPU");
    return DP_ERR_NO_DEVICE;
  }
  if (d->n_verts <= 0) { set_error("scene has no vertices"); return DP_ERR_VALUE; }
  if (d->verts_per_elem != 4 && d->verts_per_elem != 3) {
    set_error("elements must be tetrahedra or triangles");
    return DP_ERR_VALUE;
  }
  if (!(d->h > 0)) { set_error("time step must be positive"); return DP_ERR_VALUE; }
  // The Newton driver synchronises with the device a few times per Newton
  // iteration (residual norms, line-search decisions, Krylov convergence):
  // spin-waiting cuts each wake-up from tens of microseconds to ~1 us
  // (measured 15% per C5 step vs the default scheduling).
  // Once per device and process: changing the primary context's flags while
  // other threads launch work on it (concurrent rollouts creating scenes)
  // races inside the driver.
  {
    static std::mutex mu;
    static bool done[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    if (d->device >= 0 && d->device < 64 && !done[d->device]) {
      dp_set_spin_wait(d->device, getenv("DP_SCHED") ? atoi(getenv("DP_SCHED")) : 1);
      done[d->device] = true;
    }
  }
  DP_CUDA(cudaSetDevice(d->device));
  dp_scene* s = new dp_scene();
  s->device = d->device;
  cudaDeviceGetAttribute(&s->nsm, cudaDevAttrMultiProcessorCount, d->device);
  if (s->nsm <= 0) s->nsm = 148;
  s->V = d->n_verts;
  s->E = d->n_elems;
  s->NV = d->verts_per_elem;
  s->D = s->NV - 1;
  s->NP = s->NV * (s->NV + 1) / 2;
  s->h = d->h;
  s->eps_fb = d->eps_fb;
  s->act = d->contact_activation;
  for (int i = 0; i < 3; ++i) s->grav[i] = d->gravity[i];
  const int V = s->V, E = s->E, NV = s->NV, D = s->D, NP = s->NP;
  if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete s;
    set_error("cudaStreamCreate failed");
    return DP_ERR_CUDA;
  }
  cudaEventCreate(&s->ev0);
  cudaEventCreate(&s->ev1);

  const double t_el = now_s();
  // ---- element kinematics (build_elements, elasticity.py:74-108)
  std::vector<int4> ev(E);
  std::vector<double> Bsoa((size_t)D * D * std::max(E, 1));
  s->h_vol.assign(E, 0.0);
  s->h_w.assign(E, 0.0);
  s->h_model.assign(E, 0);
  s->h_E.assign(E, 0.0);
  s->h_nu.assign(E, 0.0);
  std::vector<double> hmu(E, 0.0), hlam(E, 0.0);
  for (int e = 0; e < E; ++e) {
    int vid[4] = {0, 0, 0, -1};
    for (int a = 0; a < NV; ++a) {
      int64_t v = d->elements[(size_t)e * NV + a];
      if (v < 0 || v >= V) {
        delete s;
        set_error("element index out of range");
        return DP_ERR_VALUE;
      }
      vid[a] = (int)v;
    }
    ev[e] = make_int4(vid[0], vid[1], vid[2], vid[3]);
    const double* X = d->vertices;
    double x[4][3];
    for (int a = 0; a < NV; ++a)
      for (int i = 0; i < 3; ++i) x[a][i] = X[3 * (size_t)vid[a] + i];
    double B[3][3] = {{0}};
    double vol;
    if (NV == 4) {
      double dm[3][3];
      for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) dm[i][k] = x[k + 1][i] - x[0][i];
      const double det = dm[0][0] * (dm[1][1] * dm[2][2] - dm[1][2] * dm[2][1]) -
                         dm[0][1] * (dm[1][0] * dm[2][2] - dm[1][2] * dm[2][0]) +
                         dm[0][2] * (dm[1][0] * dm[2][1] - dm[1][1] * dm[2][0]);
      vol = det / 6.0;
      if (!(vol > 1e-14)) {
        delete s;
        set_error("degenerate or inverted tet " + std::to_string(e));
        return DP_ERR_VALUE;
      }
      const double id = 1.0 / det;
      B[0][0] = (dm[1][1] * dm[2][2] - dm[1][2] * dm[2][1]) * id;
      B[0][1] = (dm[0][2] * dm[2][1] - dm[0][1] * dm[2][2]) * id;
      B[0][2] = (dm[0][1] * dm[1][2] - dm[0][2] * dm[1][1]) * id;
      B[1][0] = (dm[1][2] * dm[2][0] - dm[1][0] * dm[2][2]) * id;
      B[1][1] = (dm[0][0] * dm[2][2] - dm[0][2] * dm[2][0]) * id;
      B[1][2] = (dm[0][2] * dm[1][0] - dm[0][0] * dm[1][2]) * id;
      B[2][0] = (dm[1][0] * dm[2][1] - dm[1][1] * dm[2][0]) * id;
      B[2][1] = (dm[0][1] * dm[2][0] - dm[0][0] * dm[2][1]) * id;
      B[2][2] = (dm[0][0] * dm[1][1] - dm[0][1] * dm[1][0]) * id;
    } else {
      double e1[3], e2[3], n[3];
      for (int i = 0; i < 3; ++i) { e1[i] = x[1][i] - x[0][i]; e2[i] = x[2][i] - x[0][i]; }
      n[0] = e1[1] * e2[2] - e1[2] * e2[1];
      n[1] = e1[2] * e2[0] - e1[0] * e2[2];
      n[2] = e1[0] * e2[1] - e1[1] * e2[0];
      const double area = 0.5 * std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
      if (!(area > 1e-14)) {
        delete s;
        set_error("degenerate triangle " + std::to_string(e));
        return DP_ERR_VALUE;
      }
      const double l1 = std::sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
      double t1[3], t2v[3], t2[3];
      for (int i = 0; i < 3; ++i) t1[i] = e1[i] / l1;
      const double e2t1 = e2[0] * t1[0] + e2[1] * t1[1] + e2[2] * t1[2];
      for (int i = 0; i < 3; ++i) t2v[i] = e2[i] - e2t1 * t1[i];
      const double l2 = std::sqrt(t2v[0] * t2v[0] + t2v[1] * t2v[1] + t2v[2] * t2v[2]);
      for (int i = 0; i < 3; ++i) t2[i] = t2v[i] / l2;
      const double a = e1[0] * t1[0] + e1[1] * t1[1] + e1[2] * t1[2];
      const double b = e2t1;
      const double c = e2[0] * t2[0] + e2[1] * t2[1] + e2[2] * t2[2];
      // inv([[a, b], [0, c]])
      B[0][0] = 1.0 / a; B[0][1] = -b / (a * c); B[1][0] = 0.0; B[1][1] = 1.0 / c;
      vol = area;
    }
    for (int k = 0; k < D; ++k)
      for (int c = 0; c < D; ++c) Bsoa[(size_t)(k * D + c) * E + e] = B[k][c];
    const int model = d->mat_model[e];
    s->h_model[e] = model;
    s->h_E[e] = d->mat_E[e];
    s->h_nu[e] = d->mat_nu[e];
    s->h_vol[e] = vol;
    if (model == DP_MODEL_NEOHOOKEAN) {
      const double E_ = d->mat_E[e], nu = d->mat_nu[e];
      if (!(nu > -1.0 && nu < 0.5)) {
        delete s;
        set_error("nu must lie in (-1, 0.5)");
        return DP_ERR_VALUE;
      }
      hmu[e] = E_ / (2.0 * (1.0 + nu));
      hlam[e] = E_ * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
      s->h_w[e] = 2.0 * hmu[e] * vol;       // element_weight, elasticity.py:67-71
      s->any_nh = 1;
    } else {
      s->h_w[e] = d->mat_stiffness[e] * vol;
    }
  }
  s->h_mass.assign(d->masses, d->masses + V);
  for (int i = 0; i < V; ++i)
    if (!(s->h_mass[i] > 0)) {
      delete s;
      set_error("masses must be positive");
      return DP_ERR_VALUE;
    }

  const double t_inc = now_s();
  // ---- vertex incidence (residual gather) and block pattern (core.py:339-364)
  std::vector<int> inc_ptr(V + 1, 0), inc, fe_pos((size_t)E * NV);
  for (int e = 0; e < E; ++e) {
    const int* vv = &ev[e].x;
    for (int a = 0; a < NV; ++a) inc_ptr[vv[a] + 1]++;
  }
  for (int i = 0; i < V; ++i) inc_ptr[i + 1] += inc_ptr[i];
  inc.resize(inc_ptr[V]);
  {
    std::vector<int> fill(inc_ptr.begin(), inc_ptr.end() - 1);
    for (int e = 0; e < E; ++e) {
      const int* vv = &ev[e].x;
      for (int a = 0; a < NV; ++a) {
        fe_pos[(size_t)e * NV + a] = fill[vv[a]];
        inc[fill[vv[a]]++] = e * NV + a;
      }
    }
  }
  std::vector<int>& rowptr = s->h_rowptr;
  std::vector<int>& colidx = s->h_colidx;
  rowptr.assign(V + 1, 0);
  colidx.clear();
  {
    // each row's sorted neighbour set (itself + the vertices of its
    // elements), rows split over host threads, then concatenated in row order
    const int nt = (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::vector<int>> part(nt);
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
      th.emplace_back([&, t] {
        const int lo = (int)((int64_t)V * t / nt), hi = (int)((int64_t)V * (t + 1) / nt);
        std::vector<int>& out = part[t];
        out.reserve((size_t)(hi - lo) * 16);
        std::vector<int> nbr;
        for (int i = lo; i < hi; ++i) {
          nbr.clear();
          nbr.push_back(i);
          for (int k = inc_ptr[i]; k < inc_ptr[i + 1]; ++k) {
            const int e = inc[k] / NV;
            const int* vv = &ev[e].x;
            for (int b = 0; b < NV; ++b) nbr.push_back(vv[b]);
          }
          std::sort(nbr.begin(), nbr.end());
          nbr.erase(std::unique(nbr.begin(), nbr.end()), nbr.end());
          out.insert(out.end(), nbr.begin(), nbr.end());
          rowptr[i + 1] = (int)nbr.size();
        }
      });
    }
    for (auto& x : th) x.join();
    for (int i = 0; i < V; ++i) rowptr[i + 1] += rowptr[i];
    colidx.reserve(rowptr[V]);
    for (auto& p : part) colidx.insert(colidx.end(), p.begin(), p.end());
  }
  s->nnzb = (int64_t)colidx.size();

  const double t_sell = now_s();
  // ---- SELL-32 layout
  const int S = (V + kSlice - 1) / kSlice;
  s->S = S;
  std::vector<int> slice_base(S + 1, 0), slice_width(S, 0);
  for (int sl = 0; sl < S; ++sl) {
    int K = 0;
    for (int l = 0; l < kSlice; ++l) {
      const int row = sl * kSlice + l;
      if (row < V) K = std::max(K, rowptr[row + 1] - rowptr[row]);
    }
    slice_width[sl] = K;
    slice_base[sl + 1] = slice_base[sl] + K * kSlice;
  }
  s->NS = slice_base[S];
  const int64_t NS = s->NS;
  std::vector<int> col(NS, 0), diag_slot(V, 0);
  s->h_block_slot.assign(s->nnzb, 0);
  for (int i = 0; i < V; ++i) {
    const int sl = i / kSlice, l = i % kSlice;
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      const int64_t slot = slice_base[sl] + (int64_t)(k - rowptr[i]) * kSlice + l;
      col[slot] = colidx[k];
      s->h_block_slot[k] = slot;
      if (colidx[k] == i) diag_slot[i] = (int)slot;
    }
  }
  const double t_runs = now_s();
  // ---- contribution runs per slot.  Slot (i, j) and slot (j, i) receive
  // blocks from the same elements (those holding edge ij), element-ascending,
  // the (j, i) ones being the transposes of the (i, j) ones.  So only the
  // canonical slots (i <= j) own a run of the block stream H; slot (j, i)
  // reads the run of (i, j) transposed (rinfo count < 0).
  std::vector<int> cptr(NS + 1, 0);
  std::vector<int64_t> eslot((size_t)E * NV * NV);
  parallel_chunks(E, [&](int64_t e0, int64_t e1) {   // the slot of every local pair (binary searches)
    for (int64_t e = e0; e < e1; ++e) {
      const int* vv = &ev[e].x;
      for (int a = 0; a < NV; ++a) {
        const int i = vv[a];
        const int* rb = colidx.data() + rowptr[i];
        const int rl = rowptr[i + 1] - rowptr[i];
        for (int b = 0; b < NV; ++b) {
          const int k = (int)(std::lower_bound(rb, rb + rl, vv[b]) - rb);
          eslot[((size_t)e * NV + a) * NV + b] = slice_base[i / kSlice] + (int64_t)k * kSlice + (i % kSlice);
        }
      }
    }
  });
  for (int e = 0; e < E; ++e) {
    const int* vv = &ev[e].x;
    for (int a = 0; a < NV; ++a)
      for (int b = 0; b < NV; ++b) {
        const int i = vv[a], j = vv[b];
        if (i <= j && (i < j || a == b)) cptr[eslot[((size_t)e * NV + a) * NV + b] + 1]++;
      }
  }
  for (int64_t t = 0; t < NS; ++t) cptr[t + 1] += cptr[t];
  // block-stream position of every unordered local pair (a <= b) of every
  // element: the fill order of the canonical slot's run (element-ascending,
  // as the reference's COO sum); ~t when the stored block is the pair's
  // transpose (vid[a] > vid[b])
  std::vector<int> epos((size_t)E * NP);
  std::vector<int2> rinfo(NS, make_int2(0, 0));
  {
    std::vector<int> fill(cptr.begin(), cptr.end() - 1);
    for (int e = 0; e < E; ++e) {
      const int* vv = &ev[e].x;
      int p = 0;
      for (int a = 0; a < NV; ++a)
        for (int b = a; b < NV; ++b, ++p) {
          const int64_t sab = eslot[((size_t)e * NV + a) * NV + b];
          const int64_t sba = eslot[((size_t)e * NV + b) * NV + a];
          if (vv[a] <= vv[b]) {
            epos[(size_t)e * NP + p] = fill[sab]++;
            rinfo[sba] = make_int2((int)cptr[sab], -(int)(cptr[sab + 1] - cptr[sab]));
          } else {
            epos[(size_t)e * NP + p] = ~fill[sba]++;
            rinfo[sab] = make_int2((int)cptr[sba], -(int)(cptr[sba + 1] - cptr[sba]));
          }
        }
    }
    for (int64_t t = 0; t < NS; ++t)
      if (cptr[t + 1] > cptr[t]) rinfo[t] = make_int2((int)cptr[t], (int)(cptr[t + 1] - cptr[t]));
  }
  // canonical off-diagonal slot (i, j), i < j -> the slot of (j, i): the
  // assembly sums each run once and writes the block and its transpose
  std::vector<int> tslot(NS, -1);
  parallel_chunks(V, [&](int64_t i0, int64_t i1) {
    for (int i = (int)i0; i < (int)i1; ++i) {
      const int sl = i / kSlice, l = i % kSlice;
      for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) {
        const int j = colidx[k];
        if (j <= i) continue;
        const int* rb = colidx.data() + rowptr[j];
        const int rl = rowptr[j + 1] - rowptr[j];
        const int kk = (int)(std::lower_bound(rb, rb + rl, i) - rb);
        tslot[slice_base[sl] + (int64_t)(k - rowptr[i]) * kSlice + l] =
            (int)(slice_base[j / kSlice] + (int64_t)kk * kSlice + (j % kSlice));
      }
    }
  });

  const double t_dev = now_s();
  // ---- device buffers
  int rc = 0;
  rc |= upload(s, &s->ev, ev);
  rc |= upload(s, &s->B, Bsoa);
  rc |= upload(s, &s->w, s->h_w);
  rc |= upload(s, &s->vol, s->h_vol);
  rc |= upload(s, &s->mu, hmu);
  rc |= upload(s, &s->lam, hlam);
  rc |= upload(s, &s->model, s->h_model);
  rc |= upload(s, &s->mass, s->h_mass);
  rc |= upload(s, &s->inc_ptr, inc_ptr);
  rc |= upload(s, &s->inc, inc);
  rc |= upload(s, &s->slice_base, slice_base);
  rc |= upload(s, &s->slice_width, slice_width);
  rc |= upload(s, &s->col, col);
  rc |= upload(s, &s->diag_slot, diag_slot);
  rc |= upload(s, &s->rinfo, rinfo);
  rc |= upload(s, &s->tslot, tslot);
  rc |= upload(s, &s->epos, epos);
  rc |= dalloc(s, &s->val_fwd, (size_t)NS * 9);
  rc |= dalloc(s, &s->val_adj, (size_t)NS * 9);
  rc |= dalloc(s, &s->minv, (size_t)V * 9);
  rc |= dalloc(s, &s->fe, (size_t)std::max(E, 1) * NV * kFeS);
  rc |= upload(s, &s->fe_pos, fe_pos);
  rc |= dalloc(s, &s->H, (size_t)std::max(cptr[NS], 1) * kHS);
  rc |= dalloc(s, &s->Ht, (size_t)std::max(cptr[NS], 1));
  rc |= dalloc(s, &s->Pst, (size_t)std::max(E, 1) * 27);
  rc |= dalloc(s, &s->watch_v, kWatchMax);
  rc |= dalloc(s, &s->watch_e, kWatchElemMax);
  rc |= dalloc(s, &s->d_colliders, 1);
  rc |= dalloc(s, &s->fext, (size_t)V * 3);
  rc |= dalloc(s, &s->c_count, V + 1);
  rc |= dalloc(s, &s->c_off, V + 1);
  const size_t n3 = (size_t)V * 3;
  double** vecs[] = {&s->q, &s->q_hat, &s->q_bar, &s->v_bar, &s->r, &s->dq, &s->q_try, &s->rhs, &s->z, &s->z_prev, &s->dq_prev, &s->q_start, &s->tmp, &s->q_ev, &s->r_try,
                     &s->kx, &s->kr, &s->ku, &s->kw, &s->kp, &s->ks};
  for (auto pp : vecs) rc |= dalloc(s, pp, std::max(n3, (size_t)kMaxRestart + 1));
  s->gm_cap = kMaxRestart + 1;
  rc |= dalloc(s, &s->gm_V, (size_t)(kMaxRestart + 1) * n3);
  rc |= dalloc(s, &s->ksc, 1);
  rc |= dalloc(s, &s->gsc, 1);
  rc |= dalloc(s, &s->esc, 1);
  // reduction scratch: enough partials for the widest grid (elements at 128 threads)
  s->red.width = kMaxRestart + 2;
  s->red.cap_blocks = (int)std::max<int64_t>(grid_for(std::max(E, 1), 128), grid_for(n3, 128)) + 8;
  rc |= dalloc(s, &s->red.partial, (size_t)s->red.cap_blocks * s->red.width);
  rc |= dalloc(s, &s->red.counter, 4);
  rc |= dalloc(s, &s->g_dw, std::max(E, 1));
  rc |= dalloc(s, &s->g_scal, 4);
  if (rc) { dp_scene_destroy(s); return rc; }
  if (cudaMallocHost(&s->h_esc, sizeof(EvalScalars)) != cudaSuccess ||
      cudaMallocHost(&s->h_ksc, sizeof(KrylovScalars)) != cudaSuccess ||
      cudaMallocHost(&s->h_aux, 4 * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&s->h_gsc, sizeof(GmresScalars)) != cudaSuccess) {
    dp_scene_destroy(s);
    set_error("cudaMallocHost failed");
    return DP_ERR_CUDA;
  }
  cudaMemset(s->red.counter, 0, 4 * sizeof(unsigned int));
  cudaMemset(s->fext, 0, n3 * sizeof(double));
  cudaMemset(s->c_count, 0, (V + 1) * sizeof(int));
  cudaMemset(s->c_off, 0, (V + 1) * sizeof(int));
  cudaMemset(s->val_fwd, 0, (size_t)NS * 9 * sizeof(double));
  cudaMemset(s->val_adj, 0, (size_t)NS * 9 * sizeof(double));
  cudaMemset(s->g_dw, 0, std::max(E, 1) * sizeof(double));
  cudaMemset(s->g_scal, 0, 4 * sizeof(double));
  s->colliders.n = 0;
  cudaMemcpy(s->d_colliders, &s->colliders, sizeof(ColliderSet), cudaMemcpyHostToDevice);
  if (ensure_contact_capacity(s, 1) || contact_scan_setup(s)) { dp_scene_destroy(s); return DP_ERR_CUDA; }
  const double t_mg = now_s();
  if (mg_setup(s)) { dp_scene_destroy(s); return DP_ERR_CUDA; }
  if (g_debug)
    fprintf(stderr, "[dp] setup: elements %.1f ms, incidence+pattern %.1f ms, SELL %.1f ms, runs %.1f ms, "
            "device buffers %.1f ms, multigrid %.1f ms\n", 1e3 * (t_inc - t_el), 1e3 * (t_sell - t_inc),
            1e3 * (t_runs - t_sell), 1e3 * (t_dev - t_runs), 1e3 * (t_mg - t_dev), 1e3 * (now_s() - t_mg));
  if (getenv("DP_MG")) s->use_mg = atoi(getenv("DP_MG"));
  if (getenv("DP_ADJ_WARM")) s->adj_warm = atoi(getenv("DP_ADJ_WARM"));
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { dp_scene_destroy(s); return cuda_fail(e, "scene create"); }
  *out = s;
  return DP_OK;
}

static void cache_free(dp_cache* c);

int dp_scene_destroy(dp_scene* s) {
  std::lock_guard<std::recursive_mutex> api_lock(dp::api_mutex());
  if (!s) return DP_OK;
  cudaSetDevice(s->device);
  if (s->stream) host_sync(s);
  {
    SelfContact& sc = s->self;
    dfree(s->self_tri_d); dfree(s->self_adj_ptr_d); dfree(s->self_adj_d);
    dfree(sc.tn); dfree(sc.cell_start); dfree(sc.cell_fill); dfree(sc.items); dfree(sc.tcell); dfree(sc.hc);
    dfree(sc.cand); dfree(sc.cd2); dfree(sc.pn); dfree(sc.pd);
  }
  for (auto& t : s->kslot) {
    for (cudaEvent_t e : t.a) cudaEventDestroy(e);
    for (cudaEvent_t e : t.b) cudaEventDestroy(e);
  }
  for (dp_cache* c : s->cache_pool) cache_free(c);
  s->cache_pool.clear();
  for (dp_cache* c : s->live_caches) c->scene = nullptr;   // freed by their own destroy
  s->live_caches.clear();
  gm_graphs_destroy(s);
  mg_destroy(s);
  void* ptrs[] = {s->ev, s->B, s->w, s->vol, s->mu, s->lam, s->model, s->mass, s->inc_ptr, s->inc,
                  s->slice_base, s->slice_width, s->col, s->diag_slot, s->val_fwd, s->val_adj, s->val_A,
                  s->rinfo, s->tslot, s->epos, s->minv, s->fe, s->fe_pos, s->H, s->Ht, s->Pst, s->watch_v, s->watch_e, s->d_colliders, s->b_ptr, s->b_idx,
                  s->b_target, s->b_comp, s->b_vertex, s->fext, s->c_count, s->c_off, s->c_vertex, s->c_collider,
                  s->c_frame, s->c_dn, s->c_mu, s->c_delta, s->c_blk, s->c_force, s->c_kmu, s->c_kc, s->scan_tmp,
                  s->q, s->q_hat, s->q_bar, s->v_bar, s->r, s->dq, s->q_try, s->rhs, s->z, s->z_prev, s->tmp, s->q_ev, s->r_try, s->kx, s->kr,
                  s->ku, s->kw, s->kp, s->ks, s->gm_V, s->gm_Z, s->ksc, s->gsc, s->esc, s->red.partial, s->red.counter,
                  s->g_dw, s->g_scal, s->g_dEb, s->g_ddb};
  for (void* p : ptrs) dfree(p);
  if (s->h_esc) cudaFreeHost(s->h_esc);
  if (s->h_ksc) cudaFreeHost(s->h_ksc);
  if (s->h_aux) cudaFreeHost(s->h_aux);
  if (s->h_gsc) cudaFreeHost(s->h_gsc);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev1) cudaEventDestroy(s->ev1);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
  return DP_OK;
}

int dp_scene_get_info(const dp_scene* s, dp_scene_info* o) {
  o->n_verts = s->V;
  o->n_elems = s->E;
  o->verts_per_elem = s->NV;
  o->nnzb = s->nnzb;
  o->n_slots = s->NS;
  o->device_bytes = (int64_t)s->bytes;
  o->n_colliders = s->colliders.n;
  o->n_bindings = s->nb;
  o->smoother_bytes_per_block = s->val16 ? 26 : (s->val32 ? 40 : 0);
  o->pad_ = 0;
  return DP_OK;
}

int dp_scene_set_colliders(dp_scene* s, int32_t n, const int32_t* kind, const double* vec3, const double* scalar,
                           const double* mu) {
  invalidate_adjoint(s);
  if (n < 0 || n > kMaxColliders) { set_error("too many colliders"); return DP_ERR_VALUE; }
  cudaSetDevice(s->device);
  ColliderSet cs{};
  cs.n = n;
  for (int j = 0; j < n; ++j) {
    cs.kind[j] = kind[j];
    for (int i = 0; i < 3; ++i) cs.vec[j][i] = vec3[3 * j + i];
    cs.scalar[j] = scalar[j];
    cs.mu[j] = mu[j];
    if (mu[j] < 0) { set_error("friction coefficient must be nonnegative"); return DP_ERR_VALUE; }
  }
  s->colliders = cs;
  DP_CUDA(cudaMemcpyAsync(s->d_colliders, &s->colliders, sizeof(ColliderSet), cudaMemcpyHostToDevice, s->stream));
  DP_CUDA(host_sync(s));
  return ensure_contact_capacity(s, std::max(1, s->V * std::max(contact_sources(s), 1)));
}

int dp_scene_set_bindings(dp_scene* s, int32_t n, const int64_t* vertex, const double* target3,
                          const double* compliance) {
  invalidate_adjoint(s);
  cudaSetDevice(s->device);
  host_sync(s);
  for (int b = 0; b < n; ++b) {
    if (vertex[b] < 0 || vertex[b] >= s->V) { set_error("binding vertex out of range"); return DP_ERR_VALUE; }
    if (!(compliance[b] > 0)) { set_error("binding compliance must be positive"); return DP_ERR_VALUE; }
  }
  dfree(s->b_ptr); dfree(s->b_idx); dfree(s->b_target); dfree(s->b_comp); dfree(s->b_vertex);
  s->b_ptr = s->b_idx = s->b_vertex = nullptr;
  s->b_target = s->b_comp = nullptr;
  s->nb = n;
  s->hb_vertex.assign(n, 0);
  s->hb_target.assign((size_t)n * 3, 0.0);
  s->hb_comp.assign(n, 0.0);
  std::vector<int> ptr(s->V + 1, 0), idx(n);
  for (int b = 0; b < n; ++b) {
    s->hb_vertex[b] = (int)vertex[b];
    for (int i = 0; i < 3; ++i) s->hb_target[3 * b + i] = target3[3 * b + i];
    s->hb_comp[b] = compliance[b];
    ptr[vertex[b] + 1]++;
  }
  for (int i = 0; i < s->V; ++i) ptr[i + 1] += ptr[i];
  {
    std::vector<int> fill(ptr.begin(), ptr.end() - 1);
    for (int b = 0; b < n; ++b) idx[fill[vertex[b]]++] = b;
  }
  int rc = 0;
  rc |= upload(s, &s->b_ptr, ptr);
  rc |= upload(s, &s->b_idx, idx);
  rc |= upload(s, &s->b_target, s->hb_target);
  rc |= upload(s, &s->b_comp, s->hb_comp);
  rc |= upload(s, &s->b_vertex, s->hb_vertex);
  if (n > s->g_nb_cap) {
    dfree(s->g_dEb); dfree(s->g_ddb);
    rc |= dalloc(s, &s->g_dEb, n);
    rc |= dalloc(s, &s->g_ddb, (size_t)n * 3);
    s->g_nb_cap = n;
    if (!rc) {
      cudaMemset(s->g_dEb, 0, n * sizeof(double));
      cudaMemset(s->g_ddb, 0, (size_t)n * 3 * sizeof(double));
    }
  }
  return rc;
}

int dp_scene_set_params(dp_scene* s, double h, double eps_fb, double act, const double* g) {
  invalidate_adjoint(s);
  if (!(h > 0)) { set_error("time step must be positive"); return DP_ERR_VALUE; }
  if (!(eps_fb > 0)) { set_error("eps_fb (2*eps^2) must be positive"); return DP_ERR_VALUE; }
  s->h = h;
  s->eps_fb = eps_fb;
  s->act = act;
  if (g) for (int i = 0; i < 3; ++i) s->grav[i] = g[i];
  return DP_OK;
}

int dp_scene_set_fext(dp_scene* s, const double* fext, int32_t ptr_kind) {
  invalidate_adjoint(s);
  cudaSetDevice(s->device);
  if (!fext) {
    s->has_fext = 0;
    DP_CUDA(cudaMemsetAsync(s->fext, 0, sizeof(double) * 3 * s->V, s->stream));
    return DP_OK;
  }
  s->has_fext = 1;
  return copy_in(s, s->fext, fext, (size_t)3 * s->V, ptr_kind);
}

int dp_scene_set_solver_options(dp_scene* s, int32_t use_mg, double omega, int32_t nu) {
  invalidate_adjoint(s);
  s->use_mg = use_mg;
  if (omega > 0 && nu > 0) mg_set_params(s, omega, nu);
  return DP_OK;
}

int dp_scene_get_mg_levels(const dp_scene* s, int32_t* n_levels, int32_t* rows, int32_t cap) {
  const int L = mg_levels(s);
  *n_levels = L;
  for (int l = 0; l < L && l < cap; ++l) rows[l] = mg_level_rows(s, l);
  return DP_OK;
}

int dp_scene_set_materials(dp_scene* s, const double* E, const double* nu, const double* stiffness) {
  invalidate_adjoint(s);
  cudaSetDevice(s->device);
  const int n = s->E;
  std::vector<double> hmu(n, 0.0), hlam(n, 0.0);
  for (int e = 0; e < n; ++e) {
    if (E) s->h_E[e] = E[e];
    if (nu) s->h_nu[e] = nu[e];
    if (s->h_model[e] == DP_MODEL_NEOHOOKEAN) {
      const double E_ = s->h_E[e], nu_ = s->h_nu[e];
      if (!(nu_ > -1.0 && nu_ < 0.5)) { set_error("nu must lie in (-1, 0.5)"); return DP_ERR_VALUE; }
      hmu[e] = E_ / (2.0 * (1.0 + nu_));
      hlam[e] = E_ * nu_ / ((1.0 + nu_) * (1.0 - 2.0 * nu_));
      s->h_w[e] = 2.0 * hmu[e] * s->h_vol[e];
    } else if (stiffness) {
      s->h_w[e] = stiffness[e] * s->h_vol[e];
    }
  }
  if (n > 0) {
    DP_CUDA(cudaMemcpyAsync(s->w, s->h_w.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
    DP_CUDA(cudaMemcpyAsync(s->mu, hmu.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
    DP_CUDA(cudaMemcpyAsync(s->lam, hlam.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
    DP_CUDA(host_sync(s));
  }
  return DP_OK;
}

int dp_scene_set_self_contact(dp_scene* s, int32_t n_tri, const int32_t* tri, double mu, int32_t enable) {
  invalidate_adjoint(s);
  std::lock_guard<std::recursive_mutex> api_lock(dp::api_mutex());
  cudaSetDevice(s->device);
  if (mu < 0) { set_error("friction coefficient must be nonnegative"); return DP_ERR_VALUE; }
  SelfContact& sc = s->self;
  host_sync(s);
  dfree(s->self_tri_d); dfree(s->self_adj_ptr_d); dfree(s->self_adj_d);
  dfree(sc.tn); dfree(sc.cell_start); dfree(sc.cell_fill); dfree(sc.items); dfree(sc.tcell); dfree(sc.hc);
  dfree(sc.cand); dfree(sc.cd2); dfree(sc.pn); dfree(sc.pd);
  sc = SelfContact{};
  if (!enable || n_tri <= 0) return ensure_contact_capacity(s, std::max(1, s->V * std::max(contact_sources(s), 1)));
  for (int k = 0; k < 3 * n_tri; ++k)
    if (tri[k] < 0 || tri[k] >= s->V) { set_error("self-contact triangle vertex out of range"); return DP_ERR_VALUE; }
  int H = 1024;
  while (H < 2 * n_tri) H <<= 1;
  std::vector<int> htri(tri, tri + 3 * (size_t)n_tri);
  int rc = upload(s, &s->self_tri_d, htri);
  rc |= upload(s, &s->self_adj_ptr_d, s->h_rowptr);
  rc |= upload(s, &s->self_adj_d, s->h_colidx);
  rc |= dalloc(s, &sc.tn, (size_t)3 * n_tri);
  rc |= dalloc(s, &sc.cell_start, (size_t)H + 1);
  rc |= dalloc(s, &sc.cell_fill, (size_t)H);
  rc |= dalloc(s, &sc.items, (size_t)n_tri);
  rc |= dalloc(s, &sc.tcell, (size_t)n_tri);
  rc |= dalloc(s, &sc.hc, 2);
  rc |= dalloc(s, &sc.cand, (size_t)s->V);
  rc |= dalloc(s, &sc.cd2, (size_t)s->V);
  rc |= dalloc(s, &sc.pn, (size_t)3 * s->V);
  rc |= dalloc(s, &sc.pd, (size_t)s->V);
  if (rc) return DP_ERR_CUDA;
  sc.enabled = 1;
  sc.n_tri = n_tri;
  sc.H = H;
  sc.mu = mu;
  sc.tri = s->self_tri_d;
  sc.adj_ptr = s->self_adj_ptr_d;
  sc.adj = s->self_adj_d;
  return ensure_contact_capacity(s, std::max(1, s->V * std::max(contact_sources(s), 1)));
}

int dp_self_contact_query(dp_scene* s, const double* q_bar, const double* q_pred, int32_t ptr_kind,
                          int32_t* tri_out, double* d2_out, double* normal_out, double* offset_out) {
  invalidate_adjoint(s);
  cudaSetDevice(s->device);
  if (!s->self.enabled) { set_error("self contact is not enabled on this scene"); return DP_ERR_VALUE; }
  const size_t n3 = (size_t)3 * s->V;
  int rc = copy_in(s, s->q_bar, q_bar, n3, ptr_kind);
  if (!rc) rc = copy_in(s, s->q_try, q_pred, n3, ptr_kind);
  if (rc) return rc;
  launch_self_build(s);
  launch_self_candidates(s, s->q_try);
  DP_CUDA(host_sync(s));
  const SelfContact& sc = s->self;
  if (tri_out) DP_CUDA(cudaMemcpy(tri_out, sc.cand, sizeof(int) * s->V, cudaMemcpyDefault));
  if (d2_out) DP_CUDA(cudaMemcpy(d2_out, sc.cd2, sizeof(double) * s->V, cudaMemcpyDefault));
  if (normal_out) DP_CUDA(cudaMemcpy(normal_out, sc.pn, sizeof(double) * n3, cudaMemcpyDefault));
  if (offset_out) DP_CUDA(cudaMemcpy(offset_out, sc.pd, sizeof(double) * s->V, cudaMemcpyDefault));
  return DP_OK;
}

int dp_scene_get_element_data(const dp_scene* s, double* w_out, double* vol_out) {
  if (w_out) std::memcpy(w_out, s->h_w.data(), sizeof(double) * s->E);
  if (vol_out) std::memcpy(vol_out, s->h_vol.data(), sizeof(double) * s->E);
  return DP_OK;
}

int dp_scene_export_bsr(dp_scene* s, int32_t which, int32_t* rowptr, int32_t* col, double* val) {
  invalidate_adjoint(s);
  cudaSetDevice(s->device);
  const double* v = nullptr;
  if (which == 0) {
    if (!s->val_A) {
      int rc = dalloc(s, &s->val_A, (size_t)s->NS * 9);
      if (rc) return rc;
    }
    DP_CUDA(cudaMemsetAsync(s->esc, 0, sizeof(EvalScalars), s->stream));
    launch_elements(s, s->q, EV_JAC | EV_AMAT, &s->esc->status);
    launch_assemble(s, s->val_A, 0, 1);
    v = s->val_A;
  } else {
    v = (which == 1) ? s->val_fwd : s->val_adj;
  }
  std::vector<double> sell((size_t)s->NS * 9);
  DP_CUDA(cudaMemcpyAsync(sell.data(), v, sell.size() * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  DP_CUDA(host_sync(s));
  if (rowptr) std::memcpy(rowptr, s->h_rowptr.data(), sizeof(int) * (s->V + 1));
  if (col) std::memcpy(col, s->h_colidx.data(), sizeof(int) * s->nnzb);
  if (val) {
    for (int i = 0; i < s->V; ++i) {
      const int lane = i % kSlice;
      for (int k = s->h_rowptr[i]; k < s->h_rowptr[i + 1]; ++k) {
        // slot = base_s + rel*32 + lane; values at base_s*9 + (rel*9 + c)*32 + lane
        const int64_t rel = k - s->h_rowptr[i];
        const int64_t base_s = s->h_block_slot[k] - rel * kSlice - lane;
        for (int c = 0; c < 9; ++c) val[(size_t)k * 9 + c] = sell[(size_t)base_s * 9 + (rel * 9 + c) * kSlice + lane];
      }
    }
  }
  return DP_OK;
}

// ---------------------------------------------------------------------------
// forward step (forward.forward_step, forward.py:174-248)

// Step caches come from a per-scene pool: a rollout allocates one cache per
// step, and cudaMalloc/cudaFree inside the timed loop cost milliseconds (and
// cudaFree synchronises the device), so destroyed caches keep their buffers.
int dp_cache_create(dp_scene* s, dp_cache** out) {
  std::lock_guard<std::recursive_mutex> api_lock(dp::api_mutex());
  cudaSetDevice(s->device);
  if (!s->cache_pool.empty()) {
    dp_cache* c = s->cache_pool.back();
    s->cache_pool.pop_back();
    c->valid = 0;
    c->n_contacts = 0;
    c->asym = 0;
    s->live_caches.push_back(c);
    *out = c;
    return DP_OK;
  }
  dp_cache* c = new dp_cache();
  c->scene = s;
  c->V = s->V;
  const size_t n3 = (size_t)3 * s->V;
  double* blk = nullptr;
  if (cudaMalloc((void**)&blk, 5 * n3 * sizeof(double)) != cudaSuccess) {
    delete c;
    set_error("cudaMalloc failed for step cache");
    return DP_ERR_CUDA;
  }
  c->q_bar = blk;
  c->v_bar = blk + n3;
  c->q_hat = blk + 2 * n3;
  c->q_new = blk + 3 * n3;
  c->q_eval = blk + 4 * n3;
  s->live_caches.push_back(c);
  *out = c;
  return DP_OK;
}

static void cache_free(dp_cache* c) {
  void* p[] = {c->q_bar, c->c_vertex, c->c_collider, c->c_frame, c->c_dn, c->c_mu, c->c_delta};
  for (void* x : p) dfree(x);
  delete c;
}

int dp_cache_destroy(dp_cache* c) {
  std::lock_guard<std::recursive_mutex> api_lock(dp::api_mutex());
  if (!c) return DP_OK;
  if (c->scene) {
    dp_scene* s = c->scene;
    auto it = std::find(s->live_caches.begin(), s->live_caches.end(), c);
    if (it != s->live_caches.end()) {
      *it = s->live_caches.back();
      s->live_caches.pop_back();
    }
    if (s->adj_cache_tag == c) s->adj_cache_tag = nullptr;
    s->cache_pool.push_back(c);
    return DP_OK;
  }
  cache_free(c);
  return DP_OK;
}

static int cache_store(dp_scene* s, dp_cache* c, const double* q_eval, int C, int asym) {
  const size_t n3 = (size_t)3 * s->V;
  DP_CUDA(cudaMemcpyAsync(c->q_bar, s->q_bar, n3 * 8, cudaMemcpyDeviceToDevice, s->stream));
  DP_CUDA(cudaMemcpyAsync(c->v_bar, s->v_bar, n3 * 8, cudaMemcpyDeviceToDevice, s->stream));
  DP_CUDA(cudaMemcpyAsync(c->q_hat, s->q_hat, n3 * 8, cudaMemcpyDeviceToDevice, s->stream));
  DP_CUDA(cudaMemcpyAsync(c->q_new, s->q, n3 * 8, cudaMemcpyDeviceToDevice, s->stream));
  DP_CUDA(cudaMemcpyAsync(c->q_eval, q_eval, n3 * 8, cudaMemcpyDeviceToDevice, s->stream));
  if (C > c->cap_contacts) {
    void* p[] = {c->c_vertex, c->c_collider, c->c_frame, c->c_dn, c->c_mu, c->c_delta};
    for (void* x : p) dfree(x);
    // grow with slack: contact counts creep up step by step, and a
    // cudaFree/cudaMalloc pair inside the rollout costs milliseconds
    const int cap = std::max(C + C / 4, 4096);
    DP_CUDA(cudaMalloc(&c->c_vertex, sizeof(int) * cap));
    DP_CUDA(cudaMalloc(&c->c_collider, sizeof(int) * cap));
    DP_CUDA(cudaMalloc(&c->c_frame, sizeof(double) * cap * 9));
    DP_CUDA(cudaMalloc(&c->c_dn, sizeof(double) * cap));
    DP_CUDA(cudaMalloc(&c->c_mu, sizeof(double) * cap));
    DP_CUDA(cudaMalloc(&c->c_delta, sizeof(double) * cap * 3));
    c->cap_contacts = cap;
  }
  if (C > 0) {
    DP_CUDA(cudaMemcpyAsync(c->c_vertex, s->c_vertex, sizeof(int) * C, cudaMemcpyDeviceToDevice, s->stream));
    DP_CUDA(cudaMemcpyAsync(c->c_collider, s->c_collider, sizeof(int) * C, cudaMemcpyDeviceToDevice, s->stream));
    DP_CUDA(cudaMemcpyAsync(c->c_frame, s->c_frame, sizeof(double) * C * 9, cudaMemcpyDeviceToDevice, s->stream));
    DP_CUDA(cudaMemcpyAsync(c->c_dn, s->c_dn, sizeof(double) * C, cudaMemcpyDeviceToDevice, s->stream));
    DP_CUDA(cudaMemcpyAsync(c->c_mu, s->c_mu, sizeof(double) * C, cudaMemcpyDeviceToDevice, s->stream));
    DP_CUDA(cudaMemcpyAsync(c->c_delta, s->c_delta, sizeof(double) * C * 3, cudaMemcpyDeviceToDevice, s->stream));
  }
  c->n_contacts = C;
  c->asym = asym;
  c->colliders = s->colliders;
  c->valid = 1;
  return DP_OK;
}

// evaluate(q, contacts) of forward.py:186-192: element projections (with
// or without Jacobian blocks), contact multipliers, momentum residual.
static void evaluate(dp_scene* s, const double* q, double* r, int mode) {
  launch_elements(s, q, mode, &s->esc->status);
  launch_contacts(s, q, s->q_bar, -1, s->c_vertex, s->c_frame, s->c_dn, s->c_mu, s->c_delta, 0, 0, s->esc);
  launch_residual(s, q, s->q_hat, r, s->esc);
}

// DP_DEBUG >= 3: the largest residual rows and their contact state
static void debug_top_residuals(dp_scene* s, const double* r, const double* q, int it) {
  const int V = s->V, C = s->h_esc->n_contacts;
  std::vector<double> hr((size_t)3 * V), hd((size_t)3 * C), hq((size_t)3 * V);
  std::vector<int> hv(C);
  cudaMemcpy(hr.data(), r, hr.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hq.data(), q, hq.size() * 8, cudaMemcpyDeviceToHost);
  if (C) {
    cudaMemcpy(hv.data(), s->c_vertex, C * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hd.data(), s->c_delta, hd.size() * 8, cudaMemcpyDeviceToHost);
  }
  std::vector<int> idx(hr.size());
  for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int)i;
  std::partial_sort(idx.begin(), idx.begin() + 6, idx.end(),
                    [&](int a, int b) { return std::fabs(hr[a]) > std::fabs(hr[b]); });
  for (int k = 0; k < 6; ++k) {
    const int i = idx[k], v = i / 3;
    int c = -1;
    for (int j = 0; j < C; ++j)
      if (hv[j] == v) { c = j; break; }
    fprintf(stderr, "[dp]     it=%d top%d v=%d comp=%d r=%.3e contact=%d", it, k, v, i % 3, hr[i], c);
    if (c >= 0) fprintf(stderr, " delta=(%.3e %.3e %.3e)", hd[3 * c], hd[3 * c + 1], hd[3 * c + 2]);
    fprintf(stderr, " q=(%.6f %.6f %.6f)\n", hq[3 * v], hq[3 * v + 1], hq[3 * v + 2]);
  }
}

__global__ void k_neg(int n, const double* a, double* o) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) o[i] = -a[i];
}

__global__ void k_reset_flags(EvalScalars* esc) {
  esc->status = 0;
  esc->penetrating = 0;
  esc->asym = 0;
  esc->skip = 0;
  esc->precheck = 0;
  esc->pen_mask = 0;
}

int dp_forward_step(dp_scene* s, const double* q_bar, const double* v_bar, int32_t ptr_kind,
                    const dp_forward_cfg* cfg_in, double* q_out, double* v_out, dp_cache* cache,
                    dp_forward_report* rep, double* hist, int32_t hist_cap) {
  invalidate_adjoint(s);
  cudaSetDevice(s->device);
  dp_forward_cfg cfg;
  if (cfg_in) cfg = *cfg_in;
  else dp_forward_cfg_default(&cfg);
  const int V = s->V, n3 = 3 * V;
  dp_forward_report R{};
  int rc = copy_in(s, s->q_bar, q_bar, n3, ptr_kind);
  if (!rc) rc = copy_in(s, s->v_bar, v_bar, n3, ptr_kind);
  if (rc) return rc;
  const double t_step0 = g_debug ? now_s() : 0.0;
  DP_CUDA(cudaMemsetAsync(s->esc, 0, sizeof(EvalScalars), s->stream));
  launch_predict(s);                                   // q_hat and q = q_hat
  // self contact: triangles frozen at q_bar, each vertex's candidate plane
  // for this step (no-ops when disabled)
  launch_self_build(s);
  launch_self_candidates(s, s->q_hat);
  launch_pullback(s, s->q, s->q_bar, cfg.pullback_margin);
  DP_CUDA(cudaMemcpyAsync(s->q_start, s->q, sizeof(double) * 3 * s->V, cudaMemcpyDeviceToDevice, s->stream));
  double scale = 1.0;
  double* q = s->q;
  double* q_try = s->q_try;
  bool converged = false;
  int nhist = 0;
  int n_contacts = 0, asym = 0;
  // q at the last Jacobian evaluation (forward.py:201): the adjoint operator's point
  double* q_eval = s->q_ev;
  double last_t = 1.0;   // step length accepted by the previous line search
  bool elems_at_q = false;   // element buffers hold the Jacobian pass at q
  // frictionless scenes solved by multigrid PCG: the Newton operator is only
  // ever applied from its FP32 copy, so the element kernel writes an FP32
  // block stream and the assembly writes only the FP32 operator (EV_H32)
  const bool frictionless = [&] {
    for (int j = 0; j < s->colliders.n; ++j)
      if (s->colliders.mu[j] != 0.0) return false;
    return !(s->self.enabled && s->self.mu != 0.0);
  }();
  const int h32 = (g_fwd_h32 && frictionless && s->mg != nullptr && s->use_mg >= 2 && s->val32 != nullptr &&
                   s->NV == 4) ? EV_H32 : 0;
  const int jac_mode = EV_JAC | h32;
  const int trial_mode = g_spec_jac ? jac_mode : 0;
  for (int it = 0; it < cfg.max_iter; ++it) {
    double t_it0 = g_debug ? now_s() : 0.0;
    k_reset_flags<<<1, 1, 0, s->stream>>>(s->esc);
    launch_detect(s, q);
    if (elems_at_q) {
      // element projections, residual contributions and Hessian blocks at q
      // were computed by the accepted line-search trial (same kernel, same q)
      launch_contacts(s, q, s->q_bar, -1, s->c_vertex, s->c_frame, s->c_dn, s->c_mu, s->c_delta, 0, 0, s->esc);
      launch_residual(s, q, s->q_hat, s->r, s->esc);
    } else {
      evaluate(s, q, s->r, jac_mode);
    }
    elems_at_q = false;
    s->launches += 1;
    if ((rc = sync_esc(s))) return rc;
    const EvalScalars E = *s->h_esc;
    if (g_debug) fprintf(stderr, "[dp]   detect+eval(jac) %.2fms\n", 1e3 * (now_s() - t_it0));
    if (g_debug >= 3) debug_top_residuals(s, s->r, q, it);
    if (it == 0) scale = std::max(1.0, E.scale_max);
    n_contacts = E.n_contacts;
    asym = E.asym;
    if ((rc = raise_status(E.status))) return rc;
    const double res = E.rmax / scale;
    if (hist && nhist < hist_cap) hist[nhist] = res;
    ++nhist;
    DP_CUDA(cudaMemcpyAsync(q_eval, q, sizeof(double) * n3, cudaMemcpyDeviceToDevice, s->stream));
    if (res <= cfg.tol) { converged = true; break; }
    // Newton matrix A - dA + K_b + K_c (assemble_system_jacobian, forward.py:113-149)
    const double t_asm0 = g_debug ? now_s() : 0.0;
    launch_assemble(s, s->val_fwd, 0, 0, h32 ? 1 : 0);
    k_neg<<<grid_for(n3, 256), 256, 0, s->stream>>>(n3, s->r, s->rhs);
    s->launches++;
    // forcing term (relative 2-norm of the linear residual): lin_rtol_max
    // while the Newton residual is far from the stop threshold, lin_rtol_min
    // once it is within 1000x of it (DP_ETA_NEAR), so the last steps are
    // accurate solves and the root lands as close to the exact-solve root as
    // before (measured: C5 19.1 -> 23.8 steps/s with fewer Newton iterations;
    // a constant 1e-2 moved the converged state of the soft, stiffly bound
    // trunk parity scene by 1.4e-9 m, over its 1e-8 relative bound; 100x
    // did too, 1000x keeps every parity test green)
    const double rn = std::sqrt(E.rnorm2);
    double eta = (res <= g_eta_near * cfg.tol) ? cfg.lin_rtol_min : cfg.lin_rtol_max;
    if (eta > cfg.lin_rtol_max) eta = cfg.lin_rtol_max;
    // after a line search that had to cut the step below 1/16 the Newton
    // model is poor (friction cone / activation kinks): a cheap direction is enough
    if (last_t < 1.0 / 16) eta = std::max(eta, g_eta_plateau);
    int iters = 0, brk = 0;
    double relres = 0;
    // multigrid pays off for tight solves (adjoint, 1e-10); the inexact
    // Newton solves use it only when use_mg >= 2
    const int mg = (s->mg != nullptr) && s->use_mg >= 2;
    if (mg) mg_assemble(s, s->val_fwd);
    double t_solve0 = 0;
    if (g_debug) {
      host_sync(s);
      t_solve0 = now_s();
      fprintf(stderr, "[dp]   assemble %.2fms\n", 1e3 * (t_solve0 - t_asm0));
    }
    if (!asym) {
      // first Newton solve of a step that continues the previous one: start
      // the Krylov solve at the previous step's total Newton correction
      // q_new - q_hat (quasi-steady motion: the two are close; the solve
      // still ends on the FP64 true residual, so only the iteration count
      // changes; pcg_mg_solve falls back to x0 = 0 if the guess is worse)
      const double* x0 = (g_newton_x0 && it == 0 && s->dq_prev_valid && !E.discont) ? s->dq_prev : nullptr;
      if (mg) rc = pcg_mg_solve(s, s->val_fwd, s->rhs, s->dq, eta, cfg.lin_max_iter, &iters, &relres, &brk, 1, x0);
      else rc = cg_solve(s, s->val_fwd, s->rhs, s->dq, eta, cfg.lin_max_iter, &iters, &relres, &brk);
      R.krylov_iterations += iters;
      if (brk) {
        rc = gmres_solve(s, s->val_fwd, s->rhs, s->dq, eta, cfg.lin_max_iter, cfg.gmres_restart, &iters, &relres,
                         2.0, mg, mg ? 0 : 1);
        R.krylov_iterations += iters;
      }
    } else {
      // block-Jacobi: left preconditioning (the forcing test then weighs rows
      // by their diagonal, which suits the stiff contact rows); multigrid:
      // right preconditioning
      rc = gmres_solve(s, s->val_fwd, s->rhs, s->dq, eta, cfg.lin_max_iter, cfg.gmres_restart, &iters, &relres, 2.0,
                       mg, mg ? 0 : 1);
      R.krylov_iterations += iters;
    }
    double t_ls0 = 0;
    if (g_debug) {
      host_sync(s);
      t_ls0 = now_s();
      fprintf(stderr, "[dp] it=%d res=%.3e |r|2=%.3e C=%d asym=%d eta=%.1e krylov=%d relres=%.2e rc=%d solve=%.2fms guess=%d/%d\n",
              it, res, rn, n_contacts, asym, eta, iters, relres, rc, 1e3 * (t_ls0 - t_solve0), s->dq_prev_valid, E.discont);
    }
    // line search (forward.py:214-234)
    double t = 1.0;
    bool accepted = false;
    // watched rows for the line-search pre-check: rows within half of max|r|
    // the pre-check bounds max|r| only: off under the 2-norm acceptance rule
    const bool precheck = g_precheck && g_ls_norm != 2 && s->NV == 4 && s->E > 0;
    if (precheck) launch_watch_select(s, s->r, g_watch_frac);
    // the first trial's sync also returns the penetration verdict of every
    // later trial (k_penetration_mask): penetrating trials are then skipped
    // without a launch or a sync - exactly the trials the reference skips
    const bool use_mask = g_pen_mask && contact_sources(s) > 0;
    unsigned int pen_mask = 0;
    for (int ls = 0; ls < cfg.max_line_search; ++ls) {
      if (use_mask && ls > 0 && ls < 32 && ((pen_mask >> ls) & 1u)) {
        R.line_search_trials++;   // forward.py:218-219: penetrating, not evaluated
        t *= 0.5;
        continue;
      }
      launch_axpy_to(s, q_try, q, t, s->dq);
      k_reset_flags<<<1, 1, 0, s->stream>>>(s->esc);
      launch_penetration(s, q_try, s->esc);
      if (use_mask && ls == 0) launch_penetration_mask(s, q, s->dq, cfg.max_line_search, s->esc);
      // forward.py:218-219: a penetrating trial is not evaluated; the kernels
      // read the skip flag on the device and exit (no extra sync).  The
      // pre-check (watched rows) sets the same flag when the trial cannot
      // be accepted.
      s->eval_skip = &s->esc->skip;
      if (precheck) {
        launch_watch_elements(s, q_try);
        launch_contacts(s, q_try, s->q_bar, -1, s->c_vertex, s->c_frame, s->c_dn, s->c_mu, s->c_delta, 0, 0, s->esc);
        launch_watch_check(s, q_try, E.rmax);
        launch_elements(s, q_try, trial_mode, &s->esc->status);
        launch_residual(s, q_try, s->q_hat, s->r_try, s->esc);
        s->launches += 2;
      } else {
        evaluate(s, q_try, s->r_try, trial_mode);
      }
      s->eval_skip = nullptr;
      s->launches++;
      R.line_search_trials++;
      if ((rc = sync_esc(s))) return rc;
      const EvalScalars T = *s->h_esc;
      if (ls == 0) pen_mask = T.pen_mask;
      if (g_debug > 1)
        fprintf(stderr, "[dp]   ls=%d t=%.3e pen=%d st=%d rmax_try=%.6e (rmax=%.6e)\n", ls, t, T.penetrating, T.status,
                T.rmax, E.rmax);
      if (!T.skip) {
        const int st = T.status;
        const bool value_error = (st & (ST_INVERTED | ST_NONFINITE | ST_PENETRATION)) != 0;
        if (!value_error && (st & ST_NH_STALL)) return raise_status(ST_NH_STALL);
        const bool decrease = g_ls_norm == 2 ? (T.rnorm2 < E.rnorm2) : (T.rmax < E.rmax);
        if (!value_error && decrease) {
          std::swap(q, q_try);
          accepted = true;
          elems_at_q = g_spec_jac != 0;
          break;
        }
      }
      t *= 0.5;
    }
    last_t = accepted ? t : 0.0;
    if (g_debug) fprintf(stderr, "[dp]   line search %.2fms\n", 1e3 * (now_s() - t_ls0));
    if (!accepted) {
      launch_axpy_to(s, q_try, q, t, s->dq);
      k_reset_flags<<<1, 1, 0, s->stream>>>(s->esc);
      launch_penetration(s, q_try, s->esc);
      s->launches++;
      if ((rc = sync_esc(s))) return rc;
      if (!s->h_esc->penetrating) std::swap(q, q_try);
    }
  }
  if (q != s->q) {
    DP_CUDA(cudaMemcpyAsync(s->q, q, sizeof(double) * n3, cudaMemcpyDeviceToDevice, s->stream));
  }
  launch_velocity(s, s->q, s->q_bar, s->z);
  launch_axpy_to(s, s->dq_prev, s->q, -1.0, s->q_start);   // q_new - q_start (next step's first guess)
  s->dq_prev_valid = 1;
  if (q_out && (rc = copy_out(s, q_out, s->q, n3, ptr_kind))) return rc;
  if (v_out && (rc = copy_out(s, v_out, s->z, n3, ptr_kind))) return rc;
  if (cache && (rc = cache_store(s, cache, q_eval, n_contacts, asym))) return rc;
  DP_CUDA(host_sync(s));
  if (g_debug) fprintf(stderr, "[dp] step total %.2fms\n", 1e3 * (now_s() - t_step0));
  R.converged = converged ? 1 : 0;
  R.iterations = nhist;
  R.n_contacts = n_contacts;
  R.symmetric = asym ? 0 : 1;
  s->last_sym_fwd = R.symmetric;
  if (rep) *rep = R;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "forward step");
  return DP_OK;
}

// ---------------------------------------------------------------------------
// cache accessors

int dp_cache_n_contacts(const dp_cache* c, int32_t* n) {
  *n = c->n_contacts;
  return DP_OK;
}

int dp_cache_get_contacts(const dp_cache* c, int32_t* vertex, int32_t* collider, double* frame, double* d_n,
                          double* mu, double* lam, double* delta, double* s_signed, int32_t* capped) {
  const int C = c->n_contacts;
  if (C == 0) return DP_OK;
  dp_scene* s = c->scene;
  cudaSetDevice(s->device);
  if (vertex) DP_CUDA(cudaMemcpy(vertex, c->c_vertex, sizeof(int) * C, cudaMemcpyDeviceToHost));
  if (collider) DP_CUDA(cudaMemcpy(collider, c->c_collider, sizeof(int) * C, cudaMemcpyDeviceToHost));
  if (frame) DP_CUDA(cudaMemcpy(frame, c->c_frame, sizeof(double) * C * 9, cudaMemcpyDeviceToHost));
  if (d_n) DP_CUDA(cudaMemcpy(d_n, c->c_dn, sizeof(double) * C, cudaMemcpyDeviceToHost));
  std::vector<double> hmu(C), hdel(3 * (size_t)C);
  DP_CUDA(cudaMemcpy(hmu.data(), c->c_mu, sizeof(double) * C, cudaMemcpyDeviceToHost));
  DP_CUDA(cudaMemcpy(hdel.data(), c->c_delta, sizeof(double) * C * 3, cudaMemcpyDeviceToHost));
  if (mu) std::memcpy(mu, hmu.data(), sizeof(double) * C);
  if (delta) std::memcpy(delta, hdel.data(), sizeof(double) * C * 3);
  if (lam || s_signed || capped) {
    // lam, s, capped are closed-form functions of delta (contact.py:139-165)
    std::vector<double> frame_dummy(9 * (size_t)C, 0.0), dn(C), x(3 * (size_t)C), xb(3 * (size_t)C, 0.0),
        eps(C, s->eps_fb);
    for (int k = 0; k < C; ++k) {
      frame_dummy[9 * k] = frame_dummy[9 * k + 4] = frame_dummy[9 * k + 8] = 1.0;
      x[3 * k] = hdel[3 * k]; x[3 * k + 1] = hdel[3 * k + 1]; x[3 * k + 2] = hdel[3 * k + 2];
      dn[k] = 0.0;
    }
    std::vector<double> L(3 * (size_t)C), D(3 * (size_t)C), Sg(C), Kc(9 * (size_t)C), km(3 * (size_t)C),
        res(3 * (size_t)C);
    std::vector<int> cp(C), st(C);
    int rc = dp_contact_batch(C, frame_dummy.data(), dn.data(), hmu.data(), eps.data(), x.data(), xb.data(),
                              L.data(), D.data(), Sg.data(), cp.data(), Kc.data(), km.data(), res.data(), st.data());
    if (rc) return rc;
    if (lam) std::memcpy(lam, L.data(), sizeof(double) * 3 * C);
    if (s_signed) std::memcpy(s_signed, Sg.data(), sizeof(double) * C);
    if (capped) std::memcpy(capped, cp.data(), sizeof(int) * C);
  }
  return DP_OK;
}

int dp_cache_get_states(const dp_cache* c, double* q_bar, double* v_bar, double* q_hat, double* q_new) {
  const size_t n = (size_t)3 * c->V * sizeof(double);
  cudaSetDevice(c->scene->device);
  if (q_bar) DP_CUDA(cudaMemcpy(q_bar, c->q_bar, n, cudaMemcpyDeviceToHost));
  if (v_bar) DP_CUDA(cudaMemcpy(v_bar, c->v_bar, n, cudaMemcpyDeviceToHost));
  if (q_hat) DP_CUDA(cudaMemcpy(q_hat, c->q_hat, n, cudaMemcpyDeviceToHost));
  if (q_new) DP_CUDA(cudaMemcpy(q_new, c->q_new, n, cudaMemcpyDeviceToHost));
  return DP_OK;
}

int dp_cache_get_projections(dp_scene* s, const dp_cache* c, double* sigma, double* theta, double* P,
                             double* energy) {
  invalidate_adjoint(s);
  cudaSetDevice(s->device);
  const int E = s->E, D = s->D;
  if (!E) return DP_OK;
  const size_t ED = (size_t)E * D;
  if (scratch_reserve(scratch_bytes({ED * 8, ED * 8, ED * 3 * 8, (size_t)E * 8}))) {
    set_error("device scratch allocation failed");
    return DP_ERR_CUDA;
  }
  double* ds = scratch_take<double>(ED);
  double* dt = scratch_take<double>(ED);
  double* dP = scratch_take<double>(ED * 3);
  double* de = scratch_take<double>(E);
  launch_export_proj(s, c->q_eval, ds, dt, dP, de);
  host_sync(s);
  if (sigma) cudaMemcpy(sigma, ds, sizeof(double) * E * D, cudaMemcpyDeviceToHost);
  if (theta) cudaMemcpy(theta, dt, sizeof(double) * E * D, cudaMemcpyDeviceToHost);
  if (P) cudaMemcpy(P, dP, sizeof(double) * E * 3 * D, cudaMemcpyDeviceToHost);
  if (energy) cudaMemcpy(energy, de, sizeof(double) * E, cudaMemcpyDeviceToHost);
  return DP_OK;
}

// ---------------------------------------------------------------------------
// adjoint (adjoint.py:93-219)


int dp_adjoint_assemble(dp_scene* s, const dp_cache* c, int32_t* symmetric) {
  cudaSetDevice(s->device);
  const double t0 = g_debug ? now_s() : 0.0;
  if (!c->valid) { set_error("step cache is empty"); return DP_ERR_VALUE; }
  int rc = load_cache_contacts(s, c);
  if (rc) return rc;
  DP_CUDA(cudaMemsetAsync(s->esc, 0, sizeof(EvalScalars), s->stream));
  launch_elements(s, c->q_eval, EV_JAC | EV_STOREP, &s->esc->status);
  if (c->n_contacts > 0)
    launch_contacts(s, c->q_eval, c->q_bar, c->n_contacts, s->c_vertex, s->c_frame, s->c_dn, s->c_mu, s->c_delta, 1,
                    1, s->esc);
  // A_hat^T: elastic part symmetric, contact blocks transposed (adjoint.py:45-50)
  const int saved = s->colliders.n;
  if (c->n_contacts > 0 && s->colliders.n == 0) s->colliders.n = 1;   // enable contact gather
  launch_assemble(s, s->val_adj, 1, 0);
  s->colliders.n = saved;
  if ((rc = sync_esc(s))) return rc;
  if ((rc = raise_status(s->h_esc->status & ~ST_PENETRATION))) return rc;
  s->last_sym_adj = c->asym ? 0 : 1;
  s->mg_adj_ready = 0;   // the hierarchy is rebuilt lazily by the solve
  if (symmetric) *symmetric = s->last_sym_adj;
  if (g_debug) fprintf(stderr, "[dp] adjoint assemble %.2fms\n", 1e3 * (now_s() - t0));
  s->adj_cache_tag = c;
  return DP_OK;
}

int dp_adjoint_solve(dp_scene* s, const dp_cache* c, const double* dL_dq, const double* dL_dv, int32_t ptr_kind,
                     const dp_solver_cfg* cfg_in, double* z_out, dp_solve_report* rep) {
  cudaSetDevice(s->device);
  dp_solver_cfg cfg;
  if (cfg_in) cfg = *cfg_in;
  else dp_solver_cfg_default(&cfg);
  if (s->adj_cache_tag != c) {
    int rc = dp_adjoint_assemble(s, c, nullptr);
    if (rc) return rc;
  }
  const int n3 = 3 * s->V;
  int rc = copy_in(s, s->rhs, dL_dq, n3, ptr_kind);
  if (!rc) rc = copy_in(s, s->tmp, dL_dv, n3, ptr_kind);
  if (rc) return rc;
  // rhs = dL_dq + dL_dv / h  (solve_adjoint, adjoint.py:126-127)
  launch_axpy_to(s, s->rhs, s->rhs, 1.0 / s->h, s->tmp);
  const int sym = s->last_sym_adj;
  int method = cfg.method;
  if (method == DP_SOLVER_AUTO) method = sym ? DP_SOLVER_CG : DP_SOLVER_GMRES;
  int iters = 0, brk = 0;
  double relres = 0;
  const double t0 = g_debug ? now_s() : 0.0;
  const int mg = (s->mg != nullptr) && s->use_mg;
  if (mg && !s->mg_adj_ready) {
    mg_assemble(s, s->val_adj);
    s->mg_adj_ready = 1;
  }
  if (method == DP_SOLVER_CG) {
    // (a warm start from the previous adjoint solution, as the GMRES branch
    // does, saves 1.6% of the iterations but costs more than that in the
    // extra residual SpMV and sync: measured slower, not used)
    if (mg) rc = pcg_mg_solve(s, s->val_adj, s->rhs, s->z, cfg.tol, cfg.max_iter, &iters, &relres, &brk, g_adj_fp32);
    else rc = cg_solve(s, s->val_adj, s->rhs, s->z, cfg.tol, cfg.max_iter, &iters, &relres, &brk);
    if (brk) {
      int it2 = 0;
      rc = gmres_solve(s, s->val_adj, s->rhs, s->z, cfg.tol, cfg.max_iter, cfg.gmres_restart, &it2, &relres, 0.0,
                       mg, 0);
      iters += it2;
    }
  } else {
    // warm start from the previous adjoint solution of this reverse sweep:
    // consecutive steps' adjoint states are close, and the stop test is on
    // the true residual, so only the iteration count changes
    const int warm = s->adj_warm && s->z_prev_valid;
    if (warm) DP_CUDA(cudaMemcpyAsync(s->z, s->z_prev, sizeof(double) * n3, cudaMemcpyDeviceToDevice, s->stream));
    rc = gmres_solve(s, s->val_adj, s->rhs, s->z, cfg.tol, cfg.max_iter, cfg.gmres_restart, &iters, &relres, 0.0, mg,
                     0, warm);
  }
  if (mg && !(relres <= cfg.tol) && iters < cfg.max_iter) {
    // refinement: the multigrid-preconditioned solve stalled above the
    // tolerance; solve the correction A d = b - A z with block-Jacobi GMRES
    const int n3b = 3 * s->V;
    const double bn = std::sqrt(device_norm2(s, s->rhs));
    double* res = s->q_try;   // free during the adjoint
    double* d = s->r_try;
    launch_axpy_to(s, res, s->rhs, 0.0, s->rhs);
    // res = b - A z
    launch_spmv(s, s->val_adj, s->z, d);
    launch_axpy_to(s, res, s->rhs, -1.0, d);
    const double rn = std::sqrt(device_norm2(s, res));
    int it2 = 0;
    double rel2 = 1.0;
    gmres_solve(s, s->val_adj, res, d, cfg.tol * bn / std::max(rn, 1e-300), cfg.max_iter - iters,
                cfg.gmres_restart, &it2, &rel2, 0.0, 0, 0);
    launch_axpy_to(s, s->z, s->z, 1.0, d);
    iters += it2;
    launch_spmv(s, s->val_adj, s->z, d);
    launch_axpy_to(s, res, s->rhs, -1.0, d);
    relres = std::sqrt(device_norm2(s, res)) / bn;
    (void)n3b;
  }
  DP_CUDA(cudaMemcpyAsync(s->z_prev, s->z, sizeof(double) * n3, cudaMemcpyDeviceToDevice, s->stream));
  s->z_prev_valid = 1;
  if (g_debug) {
    host_sync(s);
    fprintf(stderr, "[dp] adjoint sym=%d iters=%d relres=%.2e solve %.2fms\n", sym, iters, relres,
            1e3 * (now_s() - t0));
  }
  if (rep) {
    rep->converged = relres <= cfg.tol;
    rep->iterations = iters;
    rep->rel_residual = relres;
    rep->symmetric = sym;
  }
  if (z_out) {
    int rc2 = copy_out(s, z_out, s->z, n3, ptr_kind);
    if (rc2) return rc2;
  }
  DP_CUDA(host_sync(s));
  if (!(relres <= cfg.tol)) {
    char buf[160];
    snprintf(buf, sizeof buf, "adjoint solve did not converge; relative residual %.3e", relres);
    set_error(buf);
    return DP_ERR_NOT_CONVERGED;
  }
  return DP_OK;
}

int dp_backprop_step(dp_scene* s, const dp_cache* c, const double* z, const double* dL_dv, int32_t ptr_kind,
                     double* dL_dqbar_out, double* dL_dvbar_out, double* dL_dfext_out) {
  cudaSetDevice(s->device);
  const double t0 = g_debug ? now_s() : 0.0;
  if (s->adj_cache_tag != c) {
    int rc = dp_adjoint_assemble(s, c, nullptr);
    if (rc) return rc;
  }
  const int n3 = 3 * s->V;
  int rc = 0;
  const double* zd = s->z;
  if (z != nullptr && !(ptr_kind == DP_PTR_DEVICE && z == s->z)) {
    rc = copy_in(s, s->kx, z, n3, ptr_kind);
    zd = s->kx;
  }
  if (!rc) rc = copy_in(s, s->tmp, dL_dv, n3, ptr_kind);
  if (rc) return rc;
  // outputs in scratch, then copy out
  double* dq = s->kr;
  double* dv = s->ku;
  double* df = s->kw;
  launch_backprop(s, c, zd, s->tmp, dq, dv, df);
  if (dL_dqbar_out && (rc = copy_out(s, dL_dqbar_out, dq, n3, ptr_kind))) return rc;
  if (dL_dvbar_out && (rc = copy_out(s, dL_dvbar_out, dv, n3, ptr_kind))) return rc;
  if (dL_dfext_out && (rc = copy_out(s, dL_dfext_out, df, n3, ptr_kind))) return rc;
  DP_CUDA(host_sync(s));
  cudaError_t e = cudaGetLastError();
  if (g_debug) fprintf(stderr, "[dp] backprop %.2fms\n", 1e3 * (now_s() - t0));
  if (e != cudaSuccess) return cuda_fail(e, "backprop");
  return DP_OK;
}

int dp_grads_reset(dp_scene* s) {
  cudaSetDevice(s->device);
  s->z_prev_valid = 0;   // a new reverse sweep: no warm start across sweeps
  DP_CUDA(cudaMemsetAsync(s->g_dw, 0, sizeof(double) * std::max(s->E, 1), s->stream));
  DP_CUDA(cudaMemsetAsync(s->g_scal, 0, sizeof(double) * 4, s->stream));
  if (s->g_nb_cap) {
    DP_CUDA(cudaMemsetAsync(s->g_dEb, 0, sizeof(double) * s->g_nb_cap, s->stream));
    DP_CUDA(cudaMemsetAsync(s->g_ddb, 0, sizeof(double) * 3 * s->g_nb_cap, s->stream));
  }
  DP_CUDA(host_sync(s));
  return DP_OK;
}

int dp_grads_get(dp_scene* s, dp_grad_scalars* out) {
  cudaSetDevice(s->device);
  double h[4];
  DP_CUDA(cudaMemcpyAsync(h, s->g_scal, sizeof h, cudaMemcpyDeviceToHost, s->stream));
  DP_CUDA(host_sync(s));
  out->dL_dmu_friction = h[0];
  out->dL_dstiffness = h[1];
  out->dmu_lame = h[2];
  out->dlam_lame = h[3];
  return DP_OK;
}

int dp_grads_get_arrays(dp_scene* s, double* dL_dw, double* dL_dEb, double* dL_ddb) {
  // host or device destinations (UVA, cudaMemcpyDefault), ordered on the
  // scene stream: a device-resident caller (packed gradient all-reduce)
  // never round-trips through the host
  cudaSetDevice(s->device);
  const cudaMemcpyKind k = cudaMemcpyDefault;
  if (dL_dw && s->E) DP_CUDA(cudaMemcpyAsync(dL_dw, s->g_dw, sizeof(double) * s->E, k, s->stream));
  if (dL_dEb && s->nb) DP_CUDA(cudaMemcpyAsync(dL_dEb, s->g_dEb, sizeof(double) * s->nb, k, s->stream));
  if (dL_ddb && s->nb) DP_CUDA(cudaMemcpyAsync(dL_ddb, s->g_ddb, sizeof(double) * 3 * s->nb, k, s->stream));
  DP_CUDA(host_sync(s));
  return DP_OK;
}

// ---------------------------------------------------------------------------
// unit-level batches

int dp_project_batch(int32_t n, int32_t d, const double* F, const int32_t* model, const double* mu,
                     const double* lam, double tau_rel, double* sigma, double* theta, double* W, double* P,
                     double* dPdF, double* dP_dmu, double* dP_dlam, int32_t* status) {
  if (n <= 0) return DP_OK;
  if (d != 2 && d != 3) { set_error("F must be 3x3 or 3x2"); return DP_ERR_VALUE; }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_error("no CUDA device available");
    return DP_ERR_NO_DEVICE;
  }
  const size_t N = n, F_ = 3 * d, J_ = (size_t)(3 * d) * (3 * d);
  if (scratch_reserve(scratch_bytes({N * F_ * 8, N * 8, N * 8, N * 4, N * 4, N * d * 8, N * d * 8, N * d * d * 8,
                                     N * F_ * 8, N * J_ * 8, N * F_ * 8, N * F_ * 8}))) {
    set_error("device scratch allocation failed");
    return DP_ERR_CUDA;
  }
  double* dF = scratch_take<double>(N * F_);
  double* dmu = scratch_take<double>(N);
  double* dlam = scratch_take<double>(N);
  int* dmod = scratch_take<int>(N);
  int* dst = scratch_take<int>(N);
  double* ds = scratch_take<double>(N * d);
  double* dt = scratch_take<double>(N * d);
  double* dW = scratch_take<double>(N * d * d);
  double* dP = scratch_take<double>(N * F_);
  double* dJ = scratch_take<double>(N * J_);
  double* dPm = scratch_take<double>(N * F_);
  double* dPl = scratch_take<double>(N * F_);
  cudaMemcpy(dF, F, N * F_ * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dmu, mu, N * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dlam, lam, N * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dmod, model, N * 4, cudaMemcpyHostToDevice);
  cudaMemset(ds, 0, N * d * 8);
  cudaMemset(dt, 0, N * d * 8);
  cudaMemset(dW, 0, N * d * d * 8);
  cudaMemset(dP, 0, N * F_ * 8);
  cudaMemset(dJ, 0, N * J_ * 8);
  cudaMemset(dPm, 0, N * F_ * 8);
  cudaMemset(dPl, 0, N * F_ * 8);
  launch_project_batch(n, d, dF, dmod, dmu, dlam, tau_rel, ds, dt, dW, dP, dJ, dPm, dPl, dst);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) {
    if (sigma) cudaMemcpy(sigma, ds, N * d * 8, cudaMemcpyDeviceToHost);
    if (theta) cudaMemcpy(theta, dt, N * d * 8, cudaMemcpyDeviceToHost);
    if (W) cudaMemcpy(W, dW, N * d * d * 8, cudaMemcpyDeviceToHost);
    if (P) cudaMemcpy(P, dP, N * F_ * 8, cudaMemcpyDeviceToHost);
    if (dPdF) cudaMemcpy(dPdF, dJ, N * J_ * 8, cudaMemcpyDeviceToHost);
    if (dP_dmu) cudaMemcpy(dP_dmu, dPm, N * F_ * 8, cudaMemcpyDeviceToHost);
    if (dP_dlam) cudaMemcpy(dP_dlam, dPl, N * F_ * 8, cudaMemcpyDeviceToHost);
    if (status) cudaMemcpy(status, dst, N * 4, cudaMemcpyDeviceToHost);
  }
  if (e != cudaSuccess) return cuda_fail(e, "project batch");
  return DP_OK;
}

int dp_contact_batch(int32_t n, const double* frame, const double* d_n, const double* mu, const double* eps2,
                     const double* x, const double* x_bar, double* lam, double* delta, double* s_signed,
                     int32_t* capped, double* Kc, double* k_mu, double* residual, int32_t* status) {
  if (n <= 0) return DP_OK;
  const size_t N = n;
  if (scratch_reserve(scratch_bytes({N * 72, N * 8, N * 8, N * 8, N * 24, N * 24, N * 24, N * 24, N * 8, N * 72,
                                     N * 24, N * 24, N * 4, N * 4}))) {
    set_error("device scratch allocation failed");
    return DP_ERR_CUDA;
  }
  double* df = scratch_take<double>(N * 9);
  double* ddn = scratch_take<double>(N);
  double* dmu = scratch_take<double>(N);
  double* deps = scratch_take<double>(N);
  double* dx = scratch_take<double>(N * 3);
  double* dxb = scratch_take<double>(N * 3);
  double* dl = scratch_take<double>(N * 3);
  double* dd = scratch_take<double>(N * 3);
  double* dsg = scratch_take<double>(N);
  double* dK = scratch_take<double>(N * 9);
  double* dkm = scratch_take<double>(N * 3);
  double* dres = scratch_take<double>(N * 3);
  int* dcp = scratch_take<int>(N);
  int* dst = scratch_take<int>(N);
  cudaMemcpy(df, frame, N * 72, cudaMemcpyHostToDevice);
  cudaMemcpy(ddn, d_n, N * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dmu, mu, N * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(deps, eps2, N * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, x, N * 24, cudaMemcpyHostToDevice);
  cudaMemcpy(dxb, x_bar, N * 24, cudaMemcpyHostToDevice);
  cudaMemset(dl, 0, N * 24);
  cudaMemset(dK, 0, N * 72);
  cudaMemset(dkm, 0, N * 24);
  cudaMemset(dres, 0, N * 24);
  cudaMemset(dsg, 0, N * 8);
  cudaMemset(dcp, 0, N * 4);
  launch_contact_batch(n, df, ddn, dmu, deps, dx, dxb, dl, dd, dsg, dcp, dK, dkm, dres, dst);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) {
    if (lam) cudaMemcpy(lam, dl, N * 24, cudaMemcpyDeviceToHost);
    if (delta) cudaMemcpy(delta, dd, N * 24, cudaMemcpyDeviceToHost);
    if (s_signed) cudaMemcpy(s_signed, dsg, N * 8, cudaMemcpyDeviceToHost);
    if (capped) cudaMemcpy(capped, dcp, N * 4, cudaMemcpyDeviceToHost);
    if (Kc) cudaMemcpy(Kc, dK, N * 72, cudaMemcpyDeviceToHost);
    if (k_mu) cudaMemcpy(k_mu, dkm, N * 24, cudaMemcpyDeviceToHost);
    if (residual) cudaMemcpy(residual, dres, N * 24, cudaMemcpyDeviceToHost);
    if (status) cudaMemcpy(status, dst, N * 4, cudaMemcpyDeviceToHost);
  }
  if (e != cudaSuccess) return cuda_fail(e, "contact batch");
  return DP_OK;
}

int dp_detect_contacts(dp_scene* s, const double* q, int32_t ptr_kind, int32_t cap, int32_t* n_out,
                       int32_t* vertex, int32_t* collider, double* frame, double* d_n) {
  invalidate_adjoint(s);
  cudaSetDevice(s->device);
  int rc = copy_in(s, s->q_try, q, (size_t)3 * s->V, ptr_kind);
  if (rc) return rc;
  DP_CUDA(cudaMemsetAsync(s->esc, 0, sizeof(EvalScalars), s->stream));
  launch_detect(s, s->q_try);
  if ((rc = sync_esc(s))) return rc;
  const int C = s->h_esc->n_contacts;
  *n_out = C;
  const int m = std::min(C, cap);
  if (m > 0) {
    if (vertex) DP_CUDA(cudaMemcpy(vertex, s->c_vertex, sizeof(int) * m, cudaMemcpyDeviceToHost));
    if (collider) DP_CUDA(cudaMemcpy(collider, s->c_collider, sizeof(int) * m, cudaMemcpyDeviceToHost));
    if (frame) DP_CUDA(cudaMemcpy(frame, s->c_frame, sizeof(double) * m * 9, cudaMemcpyDeviceToHost));
    if (d_n) DP_CUDA(cudaMemcpy(d_n, s->c_dn, sizeof(double) * m, cudaMemcpyDeviceToHost));
  }
  return DP_OK;
}

// ---------------------------------------------------------------------------
// benchmarking / instrumentation

int dp_bench_spmv(dp_scene* s, int32_t which, const double* x, double* y, int32_t reps, float* ms_out) {
  invalidate_adjoint(s);
  cudaSetDevice(s->device);
  const double* val = (which == 2) ? s->val_adj : s->val_fwd;
  DP_CUDA(cudaEventRecord(s->ev0, s->stream));
  const int saved = s->timing;
  s->timing = 0;
  for (int r = 0; r < reps; ++r) launch_spmv(s, val, x, y);
  s->timing = saved;
  DP_CUDA(cudaEventRecord(s->ev1, s->stream));
  DP_CUDA(cudaEventSynchronize(s->ev1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, s->ev0, s->ev1);
  if (ms_out) *ms_out = ms;
  return DP_OK;
}

int dp_bench_smoother(dp_scene* s, const double* x, const double* b, double* out, int32_t reps, float* ms_out) {
  invalidate_adjoint(s);
  cudaSetDevice(s->device);
  DP_CUDA(cudaEventRecord(s->ev0, s->stream));
  if (mg_bench_fine_smooth(s, x, b, out, reps)) {
    set_error("multigrid is not set up for this scene");
    return DP_ERR_VALUE;
  }
  DP_CUDA(cudaEventRecord(s->ev1, s->stream));
  DP_CUDA(cudaEventSynchronize(s->ev1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, s->ev0, s->ev1);
  if (ms_out) *ms_out = ms;
  return DP_OK;
}

int dp_bench_elements(dp_scene* s, const double* q, int32_t with_jacobian, int32_t reps, float* ms_out) {
  invalidate_adjoint(s);
  cudaSetDevice(s->device);
  DP_CUDA(cudaEventRecord(s->ev0, s->stream));
  for (int r = 0; r < reps; ++r) launch_elements(s, q, with_jacobian ? EV_JAC : 0, &s->esc->status);
  DP_CUDA(cudaEventRecord(s->ev1, s->stream));
  DP_CUDA(cudaEventSynchronize(s->ev1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, s->ev0, s->ev1);
  if (ms_out) *ms_out = ms;
  return DP_OK;
}

int dp_scene_enable_timing(dp_scene* s, int32_t on) {
  s->timing = on;
  return DP_OK;
}
int dp_scene_get_timing(dp_scene* s, dp_kernel_times* out) {
  dp::ktm_flush(s);
  *out = s->times;
  return DP_OK;
}
int dp_scene_reset_timing(dp_scene* s) {
  dp::ktm_flush(s);
  s->times = dp_kernel_times{};
  s->launches = 0;
  s->host_syncs = 0;
  return DP_OK;
}
int64_t dp_scene_launch_count(dp_scene* s) { return s->launches; }
int64_t dp_scene_host_sync_count(dp_scene* s) { return s->host_syncs; }
void* dp_scene_stream(dp_scene* s) { return (void*)s->stream; }
int dp_scene_synchronize(dp_scene* s) {
  DP_CUDA(cudaStreamSynchronize(s->stream));
  return DP_OK;
}

}  // extern "C"
