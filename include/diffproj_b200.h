/*
 * diffproj_b200 — C ABI of the B200-native implicit step + adjoint.
 *
 * A drop-in for the hot path of the reference package `diffproj`
 * (arXiv 2603.16478, /root/reference/pkg/src/diffproj).  The reference is
 * pure Python, so it has no FFI of its own; every entry point below replaces
 * one Python function of the reference (cited per function) and is bound from
 * Python with ctypes by `paper_2603_16478_b200/_lib.py`.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch or C++ types cross the ABI;
 *   - FP64 everywhere; positions/velocities are flat xyz-interleaved arrays of
 *     length 3*n_verts, exactly the reference layout (core.py:31-33);
 *   - `ptr_kind` = DP_PTR_DEVICE (pointers are CUDA device memory on the
 *     scene's device) or DP_PTR_HOST (host memory; the library copies);
 *   - every function returns a dp_status; on error dp_last_error() returns a
 *     message matching the reference exception text where one exists.
 */
#ifndef DIFFPROJ_B200_H
#define DIFFPROJ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DP_OK = 0,
  DP_ERR_VALUE = 1,          /* ValueError: bad input / degenerate element   */
  DP_ERR_INVERTED = 2,       /* ValueError: det F <= 0 (elasticity.py:148)   */
  DP_ERR_PENETRATION = 3,    /* ValueError: delta_n <= 0 (contact.py:149)    */
  DP_ERR_NH_STALL = 4,       /* RuntimeError: NH projection (elasticity.py:222) */
  DP_ERR_NOT_CONVERGED = 5,  /* RuntimeError: adjoint solve (adjoint.py:134) */
  DP_ERR_BREAKDOWN = 6,      /* RuntimeError: CG breakdown (linsolve.py:89)  */
  DP_ERR_CUDA = 7,
  DP_ERR_NO_DEVICE = 8
} dp_status;

enum { DP_PTR_DEVICE = 0, DP_PTR_HOST = 1 };
enum { DP_MODEL_ARAP = 0, DP_MODEL_NEOHOOKEAN = 1 };
enum { DP_COLLIDER_HALFSPACE = 0, DP_COLLIDER_SPHERE = 1 };
enum { DP_SOLVER_AUTO = 0, DP_SOLVER_CG = 1, DP_SOLVER_GMRES = 2 };

typedef struct dp_scene dp_scene;   /* device-resident scene + system matrix   */
typedef struct dp_cache dp_cache;   /* device-resident StepCache (forward.py:47) */

/* Scene description (core.Scene fields, core.py:146-165). */
typedef struct {
  int32_t n_verts;
  int32_t n_elems;
  int32_t verts_per_elem;        /* 4 = tetrahedra, 3 = triangles             */
  int32_t device;                /* CUDA device ordinal                       */
  const double* vertices;        /* host (n_verts,3) rest positions           */
  const int64_t* elements;       /* host (n_elems,verts_per_elem)             */
  const double* masses;          /* host (n_verts) lumped masses              */
  const int32_t* mat_model;      /* host (n_elems) DP_MODEL_*                 */
  const double* mat_E;           /* host (n_elems) Young's modulus            */
  const double* mat_nu;          /* host (n_elems) Poisson ratio              */
  const double* mat_stiffness;   /* host (n_elems) ARAP stiffness             */
  double gravity[3];
  double h;
  double eps_fb;                 /* 2 eps^2                                   */
  double contact_activation;
} dp_scene_desc;

typedef struct {
  int32_t n_verts, n_elems, verts_per_elem;
  int64_t nnzb;                  /* 3x3 blocks in the BSR pattern of A        */
  int64_t n_slots;               /* blocks incl. SELL-32 padding              */
  int64_t device_bytes;          /* bytes of device memory owned              */
  int32_t n_colliders, n_bindings;
  int32_t smoother_bytes_per_block; /* fine-level V-cycle operator copy: 40 = FP32 values + column,
                                       26 = FP16 values + per-block FP32 scale + column, 0 = none */
  int32_t pad_;
} dp_scene_info;

/* ForwardConfig (forward.py:29-34) + Krylov controls of the inexact Newton. */
typedef struct {
  double tol;                    /* 1e-9   */
  int32_t max_iter;              /* 100    */
  int32_t max_line_search;       /* 40     */
  double pullback_margin;        /* 1e-6   */
  double lin_rtol_max;           /* Newton linear-solve rtol while the residual
                                    is > 1000 tol (1e-2)                     */
  double lin_rtol_min;           /* ... and once within 1000 tol (1e-3)      */
  int32_t lin_max_iter;          /* per Newton linear solve                   */
  int32_t gmres_restart;         /* 50                                        */
} dp_forward_cfg;

typedef struct {
  int32_t converged;
  int32_t iterations;            /* len(residual_history) (forward.py:235)    */
  int32_t n_contacts;            /* contacts of the final evaluation          */
  int32_t krylov_iterations;     /* total inner iterations of the step        */
  int32_t line_search_trials;
  int32_t symmetric;             /* all contact mu == 0                       */
} dp_forward_report;

/* SolverConfig (linsolve.py:21-33) for the adjoint solve. */
typedef struct {
  int32_t method;                /* DP_SOLVER_AUTO: CG iff symmetric (adjoint.py:128-133) */
  double tol;                    /* 1e-10 relative true residual              */
  int32_t max_iter;              /* 2000                                      */
  int32_t gmres_restart;         /* 50                                        */
} dp_solver_cfg;

typedef struct {
  int32_t converged;
  int32_t iterations;
  double rel_residual;           /* recomputed true residual                  */
  int32_t symmetric;
} dp_solve_report;

/* Scalar parameter gradients accumulated on device (GradientReport,
 * adjoint.py:70-90).  Per-element dL_dw and per-binding arrays are read with
 * dp_grads_get_arrays. */
typedef struct {
  double dL_dmu_friction;
  double dL_dstiffness;
  double dmu_lame;               /* sum over NH elements, before the E,nu chain */
  double dlam_lame;
} dp_grad_scalars;

/* ---- library -------------------------------------------------------------- */
const char* dp_last_error(void);
const char* dp_version(void);
int dp_device_count(void);
/* host wait policy for device synchronisation on `device`: 1 spin (default
 * at scene creation), 2 yield, 4 blocking sync, 0 unchanged */
/* Page-locked host memory for the public API's per-step output arrays
 * (cudaHostAlloc, portable).  The Python side carves arrays out of these
 * slabs and recycles them; they are not returned before process exit. */
int dp_pinned_alloc(int64_t bytes, void** out);
int dp_pinned_free(void* p);
int dp_set_spin_wait(int32_t device, int32_t mode);

/* ---- scene (core.assemble_system_matrix, core.py:379-389; build_elements,
 *      elasticity.py:74-108; build_block_pattern, core.py:339-364) ---------- */
int dp_scene_create(const dp_scene_desc* desc, dp_scene** out);
int dp_scene_destroy(dp_scene* s);
int dp_scene_get_info(const dp_scene* s, dp_scene_info* out);
/* colliders are re-read every step (contact.py:125-127) */
int dp_scene_set_colliders(dp_scene* s, int32_t n, const int32_t* kind,
                           const double* vec3, const double* scalar, const double* mu);
/* bindings (core.BindingSpec, core.py:70-90) */
int dp_scene_set_bindings(dp_scene* s, int32_t n, const int64_t* vertex,
                          const double* target3, const double* compliance);
/* step parameters read every step (Scene.h, eps_fb, contact_activation,
 * gravity; core.py:155-165).  gravity3 may be NULL (unchanged). */
int dp_scene_set_params(dp_scene* s, double h, double eps_fb, double contact_activation,
                        const double* gravity3);
/* per-dof fext (core.Scene.fext); NULL clears it.  ptr_kind as above. */
int dp_scene_set_fext(dp_scene* s, const double* fext, int32_t ptr_kind);
/* Krylov preconditioner: 0 -> 3x3 block-Jacobi everywhere; 1 (default) ->
 * aggregation-multigrid V-cycle (damped block-Jacobi smoothing, weight
 * omega, nu sweeps) for the adjoint solves, block-Jacobi for the inexact
 * Newton solves; 2 -> multigrid for both.  omega <= 0 or nu <= 0 keeps the
 * current smoother. */
int dp_scene_set_solver_options(dp_scene* s, int32_t use_mg, double omega, int32_t nu);
/* Replace the per-element material parameters in place (host arrays of
 * n_elems values in the original element order; NULL keeps a field): the
 * element weights w, Lame mu, lambda are recomputed exactly as at scene
 * creation (elasticity.py:67-71, 327-333) and uploaded; the pattern, element
 * kinematics and multigrid hierarchy are kept.  Used by the batched
 * identification loop (ident.fd_gradient) to evaluate parameter candidates
 * on pooled device scenes instead of rebuilding one per rollout. */
int dp_scene_set_materials(dp_scene* s, const double* E, const double* nu, const double* stiffness);
/* Self-contact (no reference implementation): vertices
 * against the scene's own surface triangles (tri: 3 n_tri vertex ids; the
 * caller passes the boundary faces of a tet mesh or every cloth triangle),
 * frozen at each step's q_bar.  Per step every vertex picks its candidate,
 * the nearest non-adjacent triangle within activation + |q_hat - q_bar| of
 * its q_bar position, and that triangle's plane (oriented to the vertex's
 * q_bar side) is its half-space collider for the step, index n_colliders
 * (HalfSpace detection / pullback / penetration rules).  Broad phase: a
 * per-step device spatial hash of triangle centroids.  enable = 0 turns it
 * off. */
int dp_scene_set_self_contact(dp_scene* s, int32_t n_tri, const int32_t* tri, double mu, int32_t enable);
/* Query for parity tests: build the hash at q_bar and the candidates for the
 * predicted positions q_pred; per vertex the candidate triangle (-1: none),
 * its squared closest-point distance at q_bar (-1: none), the oriented plane
 * normal (3 per vertex) and offset (gap(x) = n . x - offset).  Outputs are
 * host or device pointers (UVA); overwrites the scene's q_bar. */
int dp_self_contact_query(dp_scene* s, const double* q_bar, const double* q_pred, int32_t ptr_kind,
                          int32_t* tri_out, double* d2_out, double* normal_out, double* offset_out);
/* multigrid hierarchy: number of levels and block rows per level (<= cap) */
int dp_scene_get_mg_levels(const dp_scene* s, int32_t* n_levels, int32_t* rows, int32_t cap);
/* per-element element weights w_e and host copies of vol (elasticity.py:67-71) */
int dp_scene_get_element_data(const dp_scene* s, double* w_out, double* vol_out);
/* BSR pattern of A: rowptr (V+1), col (nnzb) and values (nnzb*9, row-major
 * 3x3 blocks) of A = M + h^2 sum w G^T G (which = 0), the last Newton matrix
 * of the forward solve (which = 1), or the last adjoint operator A_hat^T
 * (which = 2).  Host pointers. */
int dp_scene_export_bsr(dp_scene* s, int32_t which, int32_t* rowptr, int32_t* col, double* val);

/* ---- forward (forward.forward_step, forward.py:174-248) ------------------- */
void dp_forward_cfg_default(dp_forward_cfg* cfg);
int dp_forward_step(dp_scene* s, const double* q_bar, const double* v_bar, int32_t ptr_kind,
                    const dp_forward_cfg* cfg, double* q_out, double* v_out,
                    dp_cache* cache, dp_forward_report* report,
                    double* residual_history, int32_t history_cap);

/* ---- step cache (forward.StepCache, forward.py:47-60) --------------------- */
int dp_cache_create(dp_scene* s, dp_cache** out);
int dp_cache_destroy(dp_cache* c);
int dp_cache_n_contacts(const dp_cache* c, int32_t* n);
/* contact records of the cached step, detection order (contact.py:115-136):
 * vertex, collider, frame (C,3,3 rows n,t1,t2), d_n, mu, lam (C,3),
 * delta (C,3), s_signed, cone_capped.  Host pointers; any may be NULL. */
int dp_cache_get_contacts(const dp_cache* c, int32_t* vertex, int32_t* collider, double* frame,
                          double* d_n, double* mu, double* lam, double* delta, double* s_signed,
                          int32_t* capped);
/* q_bar, v_bar, q_hat, q_new of the cached step (host pointers, may be NULL) */
int dp_cache_get_states(const dp_cache* c, double* q_bar, double* v_bar, double* q_hat, double* q_new);
/* per-element projection outputs at the cached state (ElementCache,
 * elasticity.py:353-362): sigma (E,d), theta (E,d), P (E,3,d) column-stacked,
 * energy density (E).  Host pointers, may be NULL. */
int dp_cache_get_projections(dp_scene* s, const dp_cache* c, double* sigma, double* theta,
                             double* P, double* energy);

/* ---- adjoint (adjoint.py:93-219) ----------------------------------------- */
void dp_solver_cfg_default(dp_solver_cfg* cfg);
/* assemble_adjoint_operator (adjoint.py:93-120): builds A_hat^T on device */
int dp_adjoint_assemble(dp_scene* s, const dp_cache* c, int32_t* symmetric);
/* solve_adjoint (adjoint.py:123-139): A_hat^T z = dL_dq + dL_dv / h */
int dp_adjoint_solve(dp_scene* s, const dp_cache* c, const double* dL_dq, const double* dL_dv,
                     int32_t ptr_kind, const dp_solver_cfg* cfg, double* z_out,
                     dp_solve_report* report);
/* backprop_step (adjoint.py:154-219): state gradients for the previous step
 * and per-step control gradient; parameter gradients accumulate on device. */
int dp_backprop_step(dp_scene* s, const dp_cache* c, const double* z, const double* dL_dv,
                     int32_t ptr_kind, double* dL_dqbar_out, double* dL_dvbar_out,
                     double* dL_dfext_out);
int dp_grads_reset(dp_scene* s);
int dp_grads_get(dp_scene* s, dp_grad_scalars* out);
/* dL_dw (E, original element order), dL_dEb (B), dL_ddb (B,3); host or device
 * pointers (UVA), each may be NULL; returns after the copies completed */
int dp_grads_get_arrays(dp_scene* s, double* dL_dw, double* dL_dEb, double* dL_ddb);

/* ---- batched per-item kernels (unit-level parity with the reference) ----- */
/* project_element + proj_jacobian + dP_dlame over a batch of deformation
 * gradients F (n, 3, d) column-major per item (elasticity.py:137-324).
 * Outputs (host): sigma (n,d), theta (n,d), W (n,d,d), P (n,3,d),
 * dPdF (n,3d,3d), dP_dmu (n,3,d), dP_dlam (n,3,d), status (n). */
int dp_project_batch(int32_t n, int32_t d, const double* F, const int32_t* model,
                     const double* mu, const double* lam, double tau_rel,
                     double* sigma, double* theta, double* W, double* P, double* dPdF,
                     double* dP_dmu, double* dP_dlam, int32_t* status);
/* solve_multipliers + contact_block + contact_residual over a batch of
 * contacts (contact.py:139-248).  frame (n,3,3), x/x_bar (n,3). */
int dp_contact_batch(int32_t n, const double* frame, const double* d_n, const double* mu,
                     const double* eps2, const double* x, const double* x_bar,
                     double* lam, double* delta, double* s_signed, int32_t* capped,
                     double* Kc, double* k_mu, double* residual, int32_t* status);
/* detect_contacts (contact.py:115-136) at positions q (host, 3V): returns the
 * count in *n_out and fills vertex/collider/frame/d_n up to cap. */
int dp_detect_contacts(dp_scene* s, const double* q, int32_t ptr_kind, int32_t cap,
                       int32_t* n_out, int32_t* vertex, int32_t* collider, double* frame,
                       double* d_n);

/* ---- raw device kernels for benchmarking ------------------------------- */
/* y = A_hat x with the last assembled operator (which = 1 forward, 2 adjoint);
 * device pointers; returns after enqueueing `reps` launches on the scene
 * stream and (if ms_out) the CUDA-event time of all reps. */
int dp_bench_spmv(dp_scene* s, int32_t which, const double* x, double* y, int32_t reps,
                  float* ms_out);
/* Element kernel (projection + residual contributions, with the Jacobian
 * blocks when with_jacobian) at the device state q, `reps` launches on the
 * scene stream; CUDA-event time of all reps in ms_out.  Overwrites the
 * scene's element scratch (call between steps, not inside one). */
int dp_bench_elements(dp_scene* s, const double* q, int32_t with_jacobian, int32_t reps, float* ms_out);
/* One fine-level V-cycle smoothing sweep out = x + omega Minv (b - A x) with
 * the FP32 copy of the last assembled operator (the V-cycle's dominant
 * kernel), `reps` times; device pointers; CUDA-event time in ms_out. */
int dp_bench_smoother(dp_scene* s, const double* x, const double* b, double* out, int32_t reps, float* ms_out);
/* Kernel timing of the instrumented kernels since the last reset: total ms
 * and launch count per kernel, from CUDA event pairs recorded around each
 * launch on the scene stream while timing is enabled (no host
 * synchronisation per launch; the events are resolved by
 * dp_scene_get_timing).  smooth = the fine-level V-cycle sweep
 * (k_mg_smooth on level 0), pcg_spmv = the PCG's fused p-update + SpMV. */
typedef struct {
  double spmv_ms;  int64_t spmv_calls;
  double elem_jac_ms; int64_t elem_jac_calls;
  double elem_res_ms; int64_t elem_res_calls;
  double assemble_ms; int64_t assemble_calls;
  double smooth_ms; int64_t smooth_calls;
  double pcg_spmv_ms; int64_t pcg_spmv_calls;
} dp_kernel_times;
int dp_scene_enable_timing(dp_scene* s, int32_t on);
int dp_scene_get_timing(dp_scene* s, dp_kernel_times* out);
int dp_scene_reset_timing(dp_scene* s);
/* number of kernel launches issued by the library on this scene since reset */
int64_t dp_scene_launch_count(dp_scene* s);
/* Host waits on the scene's stream issued by the library since the last
 * dp_scene_reset_timing (Newton and line-search decisions, Krylov stop tests,
 * step ends); for the bench's host-sync-per-step figure.  New in round 2. */
int64_t dp_scene_host_sync_count(dp_scene* s);
/* CUDA stream (cudaStream_t) of the scene, for callers that interleave work */
void* dp_scene_stream(dp_scene* s);
int dp_scene_synchronize(dp_scene* s);

#ifdef __cplusplus
}
#endif
#endif /* DIFFPROJ_B200_H */
