// Internal declarations shared by the CUDA translation units of
// libdiffproj_b200.so.  Not part of the ABI (see include/diffproj_b200.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <mutex>
#include <vector>

#include "../../include/diffproj_b200.h"

namespace dp {
struct MG;

constexpr int kSlice = 32;          // SELL slice height (rows per warp)
constexpr int kMaxColliders = 64;

// Status word written by kernels (bit-or of ST_* codes, dp_math.cuh).
// Reduction scalars of the Newton loop live in one struct so one D2H copy
// returns everything the host needs per evaluation.
struct EvalScalars {
  double rmax;          // max |r|
  double rnorm2;        // |r|_2^2
  double scale_max;     // max |m * q_hat|  (forward.py:169-171)
  int status;           // OR of element / contact status bits
  int penetrating;      // any gap <= 0 (forward.py:86-93)
  int n_contacts;
  int asym;             // any active contact with mu != 0
  int skip;             // line-search trial needs no full evaluation (penetrating or pre-check rejected)
  int precheck;         // pre-check rejected the trial (a watched row already >= max|r|)
  int n_watch;          // watched rows (pre-check), capped at kWatchMax
  int n_watch_elem;     // element entries of the watched rows, capped at kWatchElemMax
  int discont;          // q_bar differs from the previous step's output (not a rollout continuation)
  unsigned int pen_mask;   // bit k: the line-search trial q + 2^-k dq penetrates (k_penetration_mask)
};
constexpr int kWatchMax = 256;
constexpr int kWatchElemMax = 256 * 32;

// Krylov scalars (device resident; the host only polls `done`).
struct KrylovScalars {
  double alpha, beta, gamma, delta, rho;   // CG recurrences
  double bnorm2, tol2;                      // |b|^2, (tol*|b|)^2
  int done;                                 // 1 converged, 2 breakdown
  int iters;
  int maxit;                                // PCG graph loop: stop after this many iterations
  int pad_i;
  double pad[2];
};

// GMRES restart cap: the default cycle is 50; solves that stagnate escalate
// to longer cycles (indefinite Newton matrices of compressed cloth).
// FP32 fine-level operator copy: 2 = slot-major first 8 floats of a block
// (32 B: one 256-bit load per lane, 1 KB contiguous per warp) + the 9th float
// in a tail array after them (val32[8 NS + slot]); 1 = slot-major, 12 floats
// per slot (three float4 loads per block); 0 = component-major like the FP64
// values (nine coalesced 128 B loads per warp and block)
#ifndef DP_VAL32_PACKED
#define DP_VAL32_PACKED 0
#endif
constexpr int kVal32PerSlot = DP_VAL32_PACKED == 1 ? 12 : 9;

// element Hessian blocks in the slot-ordered stream (canonical slots i <= j
// only): the first 8 doubles of a block in H (64 B, 32-byte aligned: two full
// sectors), the 9th in Ht; one block per (element, a <= b) pair, laid out in
// the canonical slots' run order so the assembly streams them
constexpr int kHS = 8;
// element residual contributions: one 32-byte entry (3 doubles + pad) per
// (element, vertex), laid out in the vertices' incidence order
constexpr int kFeS = 4;

constexpr int kMaxRestart = 200;
struct GmresScalars {
  double wn2_before;                            // |w|^2 before orthogonalisation
  double hn;                                    // H[j+1, j] before rotation
  double beta;                                  // |M^-1 r0|
  double nmb;                                   // |M^-1 b|
  double thr;                                   // stop when |g[j+1]| <= thr
  double est;                                   // |g[j+1]| / nmb
  double reorth_thr;                            // re-orthogonalise when |w|^2 < thr |w_before|^2
  int done;                                     // 1 inner stop, 2 lucky breakdown
  int reorth;
  int used;                                     // columns finished in this cycle
  int j;                                        // current column (device-driven loop)
  int m;                                        // restart length of this cycle
  int maxit;                                    // iteration budget of this cycle
  int active;                                   // 0 once j == m or the budget is spent
  int pad;
  double cs[kMaxRestart], sn[kMaxRestart], g[kMaxRestart + 1];
  double coef[kMaxRestart + 1];                 // coefficients of the current pass
  double H[kMaxRestart * (kMaxRestart + 1)];   // column j at H[j*(kMaxRestart+1) + i]; keep last
};

struct ColliderSet {
  int n;
  int kind[kMaxColliders];
  double vec[kMaxColliders][3];
  double scalar[kMaxColliders];
  double mu[kMaxColliders];
};

// Self-contact (the reference has none): vertices against
// the mesh's own surface triangles, FROZEN at the step's start positions
// q_bar (a lagged obstacle, re-read every step like the analytic colliders,
// contact.py:125-127).  Once per step every vertex v picks its candidate: the
// nearest non-adjacent surface triangle (closest-point distance at q_bar, ties
// to the lower index) within R_v = activation + |q_hat_v - q_bar_v| (the
// predicted motion).  For the rest of the step that triangle's plane,
// oriented to the side v was on at q_bar, is v's half-space collider (index
// n_colliders): detection (gap <= activation), pullback and the penetration
// test are the reference's HalfSpace rules (forward.py:63-93,
// contact.py:115-136), and every downstream kernel (condensation, blocks,
// adjoint) is unchanged.  An infinite plane per vertex also catches a vertex
// that would cross its triangle in one Newton step.  Broad phase: a uniform-
// grid spatial hash of the triangle centroids, rebuilt on the device each
// step (cell = activation + the largest centroid radius).
struct SelfContact {
  int enabled = 0;
  int n_tri = 0;
  int H = 0;                       // hash table size (power of two)
  double mu = 0.0;
  const int* tri = nullptr;        // 3 n_tri vertex ids
  const int* adj_ptr = nullptr;    // vertex graph CSR (the block pattern: 1-ring incl. the vertex)
  const int* adj = nullptr;
  double* tn = nullptr;            // unit triangle normals at q_bar (3 n_tri)
  int* cell_start = nullptr;       // H + 1
  int* cell_fill = nullptr;        // H (counts, then fill cursors)
  int* items = nullptr;            // n_tri triangle ids bucketed by cell hash
  int* tcell = nullptr;            // n_tri: hash of each triangle's centroid cell
  double* hc = nullptr;            // device scalars: cell size, radius scratch
  int* cand = nullptr;             // per vertex: candidate triangle of this step (-1: none)
  double* cd2 = nullptr;           // per vertex: its closest-point distance^2 at q_bar
  double* pn = nullptr;            // per vertex: oriented plane normal (3V)
  double* pd = nullptr;            // per vertex: plane offset n . a
  const double* qb = nullptr;      // positions the structure was built from (the scene's q_bar)
};

// reduction scratch: partial sums per block + a completion counter
struct Reduce {
  double* partial = nullptr;     // [nblocks * width]
  unsigned int* counter = nullptr;
  int cap_blocks = 0;
  int width = 0;
};

template <class T>
struct DArr {
  T* p = nullptr;
  size_t n = 0;
};

}  // namespace dp

struct dp_cache {
  dp_scene* scene = nullptr;
  int V = 0;
  int valid = 0;
  double *q_bar = nullptr, *v_bar = nullptr, *q_hat = nullptr, *q_new = nullptr, *q_eval = nullptr;
  // contact records of the final evaluation
  int n_contacts = 0;
  int cap_contacts = 0;
  int* c_vertex = nullptr;
  int* c_collider = nullptr;
  double* c_frame = nullptr;   // C*9
  double* c_dn = nullptr;
  double* c_mu = nullptr;
  double* c_delta = nullptr;   // C*3 (lam/s/capped/Kc are functions of delta)
  int asym = 0;
  // colliders / bindings used by the step (bindings are needed by backprop)
  dp::ColliderSet colliders;
};

struct dp_scene {
  int device = 0;
  int nsm = 148;                  // SMs of the device (grid sizing)
  cudaStream_t stream = nullptr;
  int V = 0, E = 0, NV = 4, D = 3, NP = 10;
  double h = 0.01, eps_fb = 1e-6, act = 1e-3, grav[3] = {0, 0, -9.8};
  int64_t nnzb = 0;
  int64_t NS = 0;            // SELL slots
  int S = 0;                 // slices
  size_t bytes = 0;

  // host mirrors
  std::vector<double> h_vol, h_w, h_mass;
  std::vector<int> h_model;
  std::vector<double> h_E, h_nu;
  std::vector<int> h_rowptr, h_colidx;   // CSR block pattern
  std::vector<int64_t> h_block_slot;     // CSR block -> SELL slot
  std::vector<int> h_orig;               // element order on device -> original index (identity)

  // device element data (SoA)
  int4* ev = nullptr;
  double* B = nullptr;       // [9][E] (tets) or [4][E] (tris)
  double *w = nullptr, *vol = nullptr, *mu = nullptr, *lam = nullptr;
  int* model = nullptr;
  int any_nh = 0;

  // per-vertex
  double* mass = nullptr;
  int *inc_ptr = nullptr, *inc = nullptr;

  // SELL-32 BSR
  int *slice_base = nullptr, *slice_width = nullptr, *col = nullptr, *diag_slot = nullptr;
  int *row_slot_ptr = nullptr;     // unused padding helper
  double* val_fwd = nullptr;       // forward Newton matrix
  double* val_adj = nullptr;       // adjoint operator (transposed contact blocks)
  double* val_A = nullptr;         // constant A (lazy, export only)
  int2* rinfo = nullptr;           // slot -> {start, count} of its run of H (count < 0: read transposed)
  int* tslot = nullptr;            // canonical slot (i < j) -> slot of (j, i); -1 otherwise
  int* epos = nullptr;             // E*NP: (element, a <= b) -> position in H (~pos: stored transposed)
  double* minv = nullptr;          // block-Jacobi inverses [9][V]
  float* val32 = nullptr;          // FP32 copy of the last assembled operator (multigrid fine level)
  // FP16 copy for the fine-level smoother sweeps: component-major like val32,
  // each slot's 9 values scaled by its block max |a| (sc16[slot], FP32)
  unsigned short* val16 = nullptr;
  float* sc16 = nullptr;
  const double* val32_src = nullptr;   // operator val32 was last written from
  int val64_valid = 1;                 // 0: the last assembly wrote only the FP32 copy (EV_H32 forward)
  float* minv32 = nullptr;         // FP32 block-Jacobi inverses (multigrid smoother)

  // element outputs
  double* fe = nullptr;            // E*NV entries of kFeS doubles, incidence order (fe_pos)
  int* fe_pos = nullptr;           // E*NV: (element, a) -> entry of fe
  double* H = nullptr;             // block stream, E*NP blocks of kHS doubles (canonical-slot order)
  double* Ht = nullptr;            // 9th double of every block of H
  double* Pst = nullptr;           // E*27 (P, dP/dmu, dP/dlam) for backprop

  // colliders / bindings / fext
  dp::ColliderSet colliders;
  dp::ColliderSet* d_colliders = nullptr;
  int nb = 0;
  std::vector<int> hb_vertex;
  std::vector<double> hb_target, hb_comp;
  int *b_ptr = nullptr, *b_idx = nullptr;   // per-vertex CSR of binding ids
  double *b_target = nullptr, *b_comp = nullptr;
  int* b_vertex = nullptr;
  double* fext = nullptr;   // 3V, zero when unset
  int has_fext = 0;

  // contacts (capacity V * n_colliders)
  int ccap = 0;
  dp::SelfContact self;             // self-contact (disabled unless dp_scene_set_self_contact)
  int* self_tri_d = nullptr;        // owned device storage behind `self`
  int* self_adj_ptr_d = nullptr;
  int* self_adj_d = nullptr;
  int *c_count = nullptr, *c_off = nullptr, *c_vertex = nullptr, *c_collider = nullptr;
  double *c_frame = nullptr, *c_dn = nullptr, *c_mu = nullptr, *c_delta = nullptr;
  double *c_blk = nullptr, *c_force = nullptr, *c_kmu = nullptr, *c_kc = nullptr;
  void* scan_tmp = nullptr;
  size_t scan_tmp_bytes = 0;

  // vectors (3V each)
  double *q = nullptr, *q_hat = nullptr, *q_bar = nullptr, *v_bar = nullptr, *r = nullptr, *dq = nullptr;
  double *q_try = nullptr, *rhs = nullptr, *z = nullptr, *tmp = nullptr, *q_ev = nullptr, *r_try = nullptr;
  const int* eval_skip = nullptr;   // device flag: element/contact/residual kernels exit when set (penetrating trial)
  int* watch_v = nullptr;           // line-search pre-check: watched rows and the elements incident to them
  int* watch_e = nullptr;
  double* z_prev = nullptr;   // last adjoint solution of the current reverse sweep (warm start)
  double* dq_prev = nullptr;  // q_new - q_start of the previous forward step (first Newton solve's initial guess)
  double* q_start = nullptr;  // the Newton start point (pulled-back q_hat) of the current step
  int dq_prev_valid = 0;
  int z_prev_valid = 0;
  int adj_warm = 1;
  // Krylov workspace
  double *kx = nullptr, *kr = nullptr, *ku = nullptr, *kw = nullptr, *kp = nullptr, *ks = nullptr;
  double* gm_V = nullptr;          // (restart+1) * 3V basis
  double* gm_Z = nullptr;          // preconditioned basis M v_j (right multigrid GMRES, allocated on first use)
  int gm_cap = 0;
  dp::KrylovScalars* ksc = nullptr;
  dp::GmresScalars* gsc = nullptr;
  dp::EvalScalars* esc = nullptr;
  dp::EvalScalars* h_esc = nullptr;     // pinned
  dp::KrylovScalars* h_ksc = nullptr;   // pinned
  double* h_aux = nullptr;               // pinned: values read back with a later sync (|b|^2 of a solve)
  dp::GmresScalars* h_gsc = nullptr;    // pinned
  dp::Reduce red;

  // gradient accumulators
  double* g_dw = nullptr;       // E
  double* g_scal = nullptr;     // [mu_fric, stiffness, dmu_lame, dlam_lame]
  double* g_dEb = nullptr;      // nb
  double* g_ddb = nullptr;      // nb*3
  int g_nb_cap = 0;

  // timing
  int timing = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  dp_kernel_times times{};
  // event pairs per instrumented kernel (KT_*), resolved in ktm_flush
  struct KSlot {
    std::vector<cudaEvent_t> a, b;
    int used = 0;
  } kslot[8];
  int64_t launches = 0;
  int64_t host_syncs = 0;         // host waits on the scene stream (host_sync)
  int stream_drained = 1;         // the host just waited on the stream (ktm_begin: GPU idle)

  // last assembled operator: symmetric flag
  int last_sym_fwd = 1, last_sym_adj = 1;

  // multigrid preconditioner (dp_mg.cu); nullptr = block-Jacobi only
  dp::MG* mg = nullptr;
  int use_mg = 2;
  int mg_adj_ready = 0;
  const dp_cache* adj_cache_tag = nullptr;   // cache whose A_hat^T is assembled

  std::vector<dp_cache*> cache_pool;   // recycled step caches
  std::vector<dp_cache*> live_caches;  // handed out, not yet destroyed
  std::vector<std::pair<uint64_t, void*>> gm_graphs;   // instantiated GMRES cycle graphs
};

namespace dp {

// error helpers -------------------------------------------------------------
void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
#define DP_CUDA(call)                                         \
  do {                                                        \
    cudaError_t _e = (call);                                  \
    if (_e != cudaSuccess) return dp::cuda_fail(_e, #call);   \
  } while (0)

int grid_for(int64_t n, int threads);

// launchers (dp_kernels.cu) -----------------------------------------------
// element evaluation: mode bit 1 = jacobian blocks, bit 2 = store P/dP for
// backprop, bit 4 = zero jacobian (A-matrix assembly).
enum { EV_JAC = 1, EV_STOREP = 2, EV_AMAT = 4, EV_LIST = 8, EV_H32 = 16 };
void launch_elements(dp_scene* s, const double* q, int mode, int* status);
// residual gather r = M(q - q_hat) + sum_e f_e - h^2 J_b^T lam_b + contact forces; max|r| into esc
void launch_residual(dp_scene* s, const double* q, const double* q_hat, double* r, dp::EvalScalars* esc);
// line-search pre-check (dp_kernels.cu)
void launch_watch_select(dp_scene* s, const double* r, double frac);
void launch_watch_elements(dp_scene* s, const double* q);
void launch_watch_check(dp_scene* s, const double* q, double rmax_prev);
// BSR gather: val = M + sum_e H_e + K_b + (K_c or K_c^T); plus block-Jacobi inverses
void launch_assemble(dp_scene* s, double* val, int transpose_contacts, int amat, int h32 = 0);
void launch_spmv(dp_scene* s, const double* val, const double* x, double* y);
// Krylov
int cg_solve(dp_scene* s, const double* val, const double* b, double* x, double rtol, int max_iter,
             int* iters, double* relres, int* breakdown);
int gmres_solve(dp_scene* s, const double* val, const double* b, double* x, double rtol, int max_iter,
                int restart, int* iters, double* relres, double min_cycle_gain = 0.0, int use_mg = 0,
                int left = 1, int use_x0 = 0);
int pcg_mg_solve(dp_scene* s, const double* val, const double* b, double* x, double rtol, int max_iter, int* iters,
                 double* relres, int* breakdown, int fp32, const double* x0 = nullptr);
double device_norm2(dp_scene* s, const double* x);   // sum of squares, synchronous
// vector ops
void launch_axpy_to(dp_scene* s, double* out, const double* a, double t, const double* b);   // out = a + t*b
void launch_predict(dp_scene* s);   // q_hat, q (pre-pullback copy), scale
void launch_velocity(dp_scene* s, const double* q, const double* q_bar, double* v);
void launch_reset_eval(dp_scene* s, dp::EvalScalars* esc);
// backprop
void launch_backprop(dp_scene* s, const dp_cache* c, const double* z, const double* dL_dv,
                     double* dqbar, double* dvbar, double* dfext);

// launchers (dp_contact.cu) ------------------------------------------------
void launch_pullback(dp_scene* s, double* q, const double* q_bar, double margin);
void launch_penetration(dp_scene* s, const double* q, dp::EvalScalars* esc);
void launch_penetration_mask(dp_scene* s, const double* q, const double* dq, int nls, dp::EvalScalars* esc);
void launch_detect(dp_scene* s, const double* q);   // fills contact records + esc->n_contacts
// per-contact condensation; writes c_delta, c_blk (h^2 fr^T Kc fr, or ^T if
// transpose), c_force; status/asym bits into esc
void launch_contacts(dp_scene* s, const double* q, const double* q_bar, int n_contacts,
                     const int* vtx, const double* frame, const double* dn, const double* mu,
                     double* delta_out, int from_delta, int transpose, dp::EvalScalars* esc);
int contact_scan_setup(dp_scene* s);

// multigrid (dp_mg.cu)
int mg_setup(dp_scene* s);
void mg_destroy(dp_scene* s);
void mg_assemble(dp_scene* s, const double* val);
void mg_apply(dp_scene* s, const double* val, const double* r, double* z, const int* stop);
// the V-cycle with its fine-level first Jacobi sweep (x = omega Minv32 r into
// the level-0 work vector) already done by the caller
void mg_apply_prejac(dp_scene* s, const double* val, const double* r, double* z, const int* stop);
void mg_fine_jacobi0_target(dp_scene* s, const float** minv32, double** xa, double* omega);
int mg_bench_fine_smooth(dp_scene* s, const double* x, const double* b, double* out, int reps);
int mg_levels(const dp_scene* s);
int mg_level_rows(const dp_scene* s, int l);
void mg_set_params(dp_scene* s, double omega, int nu);
void mg_set_symmetric(dp_scene* s, int on);
void mg_set_pcg_dot(dp_scene* s, double* partial, unsigned int* counter, KrylovScalars* ks);
void launch_self_build(dp_scene* s);
void launch_self_candidates(dp_scene* s, const double* q_pred);
void launch_pcg_rz(dp_scene* s, const double* r, const double* z, double* partial, unsigned int* counter,
                   KrylovScalars* ks);
void gm_graphs_destroy(dp_scene* s);
// Process-wide lock around the calls that allocate / free device memory or
// capture CUDA graphs (scene and cache create/destroy, GMRES graph capture):
// concurrent rollouts on host threads otherwise interleave allocations with
// another thread's capture (observed: intermittent host crash in the
// concurrent-rollout test).  Steps themselves never take it.
std::recursive_mutex& api_mutex();
// analytic colliders + the self-contact "collider" (index n_colliders)
inline int contact_sources(const dp_scene* s) { return s->colliders.n + (s->self.enabled ? 1 : 0); }
// kernel timing (dp_scene_enable_timing): event pair around one launch
enum { KT_SPMV = 0, KT_ELEM_JAC = 1, KT_ELEM_RES = 2, KT_ASSEMBLE = 3, KT_SMOOTH = 4, KT_PCG_SPMV = 5 };
void ktm_begin(dp_scene* s, int slot);
void ktm_end(dp_scene* s, int slot);
void ktm_flush(dp_scene* s);

// every host wait on a scene's stream goes through here (counted: the
// Newton / line-search loop's round trips, dp_scene_host_sync_count)
inline cudaError_t host_sync(dp_scene* s) {
  ++s->host_syncs;
  s->stream_drained = 1;
  return cudaStreamSynchronize(s->stream);
}

}  // namespace dp
