/*
 * curvopt_b200 -- C ABI of the B200-native curvature-matvec hot path.
 *
 * Drop-in boundary for the reference package `curvopt` 0.1.0 (paths relative to
 * /root/reference/pkg/src/curvopt).  The reference has no FFI; its seams are
 * Python callables, and each entry point below replaces one of them:
 *
 *   cv_linearize          models.py:337-396 (linearize) + curvature.py:87-131 (make_snapshot)
 *   cv_matvec             curvature.py:109-110 (GGN closure) / models.py:287-307 (Linearization.hvp)
 *   cv_jvp / cv_vjp       models.py:243-255 / models.py:274-285
 *   cv_cg_solve           solvers.py:60-143 (_cg_core, cg_solve)
 *   cv_hutchinson         telemetry.py:91-110 (hutchinson_diag / hutchinson_trace)
 *   cv_power_iter         telemetry.py:113-126 (power_iter_top_eig)
 *   cv_rademacher         numeric.py:124-128,157-162 (Rng._raw, rademacher)
 *   cv_diag_ema           control.py:70-77 + method.py:404-409
 *   cv_loss_at            curvature.py:82-84 (Snapshot.loss_at) -> models.py:399-408
 *   cv_rho_terms          control.py:94-96 (g.u and u.Hu of compute_rho)
 *   cv_row_rhs            curvature.py:112-119 (RowOps seeds / rhs)
 *   cv_row_gram           models.py:309-334 (output_gram) via curvature.py:62-65
 *   cv_row_solve_cholesky solvers.py:146-161
 *   cv_backproject        curvature.py:53-60 (scaled_row_transpose)
 *   cv_row_solve_cg       solvers.py:164-174 (row_solve_cg) via method.py:270-282
 *   cv_dense_*            solvers.py:146-174 on a caller-owned Gram
 *   cv_apply_update       method.py:345-357 (chain of scale links + w + update + norms)
 *   cv_chain_apply        transforms.py:148-199 (chain_apply, every link kind) + method.py:345-357
 *   cv_gnb_diag           telemetry.py:129-160 (gnb_diag, sampled-label GGN diagonal)
 *
 * Conventions
 *   - Every pointer argument is a DEVICE pointer owned by the caller, unless its
 *     comment says "host".  Vectors are fp32, scalar results are fp64 (device).
 *   - Parameter vectors use the reference flat layout (models.py:87-93): per layer
 *     W[fan_in][fan_out] row-major, then b[fan_out].
 *   - All work is enqueued on the context stream (cv_ctx_set_stream); nothing in
 *     this API synchronises the host except cv_row_solve_cholesky's PD check flag
 *     reads (documented there) and cv_ctx_create/destroy.
 *   - Return 0 on success; CV_E_* otherwise, with a message in cv_last_error().
 *     CV_E_CONTRACT mirrors the reference's ContractError (same message text where
 *     the reference has one); CV_E_NOT_PD mirrors solvers.py:157-160.
 *   - World > 1: the batch is sharded (b_local rows per rank, b_global overall);
 *     gradients, losses and every curvature product are NCCL all-reduced inside
 *     the library, so all returned vectors/scalars are replicated and global.
 */
#ifndef CURVOPT_B200_H
#define CURVOPT_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define CV_API __attribute__((visibility("default")))
#else
#define CV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cv_ctx cv_ctx;
typedef struct cv_snap cv_snap;

enum {
  CV_OK = 0,
  CV_E_CONTRACT = 1,  /* ContractError */
  CV_E_NOT_PD = 2,    /* row system not positive definite */
  CV_E_CUDA = 3,
  CV_E_NCCL = 4,
  CV_E_UNSUPPORTED = 5
};

enum { CV_ACT_RELU = 0, CV_ACT_TANH = 1 };
enum { CV_LOSS_MSE = 0, CV_LOSS_CE = 1 };
enum { CV_KIND_GGN = 0, CV_KIND_HESSIAN = 1 };
enum { CV_ENGINE_AUTO = 0, CV_ENGINE_SIMT = 1, CV_ENGINE_TC = 2 };

/* CG solve statistics written to device memory (solvers.py:36-42). */
typedef struct cv_cg_stats {
  double relres;        /* final_relative_residual */
  double bnorm;         /* ||g|| */
  int32_t iterations;
  int32_t converged;    /* 0/1 */
  int32_t neg_curv;     /* 0/1 */
  int32_t gv_count;     /* curvature products applied */
  int32_t done;         /* internal */
  int32_t x0_nonzero;   /* internal */
  int32_t pad[2];
} cv_cg_stats;

/* ---- context ------------------------------------------------------------ */
/* nccl_id: host pointer to a 128-byte ncclUniqueId.  world > 1 with nccl_id == NULL
 * creates a context whose collectives go through an external communicator that the
 * caller installs with cv_ctx_set_comm before the first call. */
CV_API int cv_ctx_create(int device, int world, int rank, const void* nccl_id, cv_ctx** out);

/* External communicator (instead of NCCL): called on the host, in enqueue order, for
 * every collective of the context: in-place sum all-reduce of `count` elements of
 * `dtype` (CV_DTYPE_*) at device pointer `buf`, ordered on `stream` (the work enqueued
 * before it must be complete when the data is read; the result must be visible to work
 * enqueued on `stream` afterwards -- a host-staged implementation synchronises the
 * stream and copies back before returning).  Return 0 on success.  Lets a host runtime
 * plug in its own transport (e.g. a gloo process group, several ranks on one GPU). */
enum { CV_DTYPE_F32 = 0, CV_DTYPE_F64 = 1 };
typedef int (*cv_comm_fn)(void* user, int dtype, void* buf, int64_t count, void* stream);
CV_API int cv_ctx_set_comm(cv_ctx* ctx, cv_comm_fn fn, void* user);
CV_API int cv_ctx_destroy(cv_ctx* ctx);
CV_API int cv_ctx_set_stream(cv_ctx* ctx, void* cuda_stream);
CV_API int cv_ctx_set_engine(cv_ctx* ctx, int engine);   /* CV_ENGINE_*: GEMM engine selection */
CV_API const char* cv_last_error(const cv_ctx* ctx);
/* CUDA-graph capture support: between begin and end every device buffer the library
 * allocates (snapshots, solver scratch, split-K partials) comes from a fresh arena that
 * the caller then owns with the captured graph (replays write into it, so it must not be
 * shared with other work); cv_arena_free releases it once the graph is destroyed. */
CV_API int cv_ctx_capture_begin(cv_ctx* ctx);
CV_API int cv_ctx_capture_end(cv_ctx* ctx, void** arena_out);
CV_API int cv_arena_free(cv_ctx* ctx, void* arena);
CV_API int cv_nccl_unique_id(void* out128);               /* host buffer of 128 bytes */
CV_API const char* cv_version(void);
CV_API int64_t cv_kernel_launches(const cv_ctx* ctx);     /* kernels enqueued so far (instrumentation) */

/* ---- snapshot (one linearization) --------------------------------------- */
/* dims: host array of n_layers+1 ints.  y: int64[b_local] class ids (CE) or
 * float[b_local*c] targets (MSE).  loss_out: device double; grad_out: device
 * float[d] (may be NULL).  The snapshot keeps copies of everything it needs. */
CV_API int cv_linearize(cv_ctx* ctx, int n_layers, const int* dims, int act, int loss,
                 const float* w, const float* X, const void* y, int b_local, int b_global,
                 cv_snap** snap, double* loss_out, float* grad_out);
CV_API int cv_snap_free(cv_snap* snap);
CV_API int64_t cv_snap_dim(const cv_snap* snap);
CV_API int cv_snap_outputs(cv_snap* snap, float* out /* b_local*c logits */);
/* hidden activation a_layer (1 <= layer < n_layers), b_local x dims[layer], fp32 */
CV_API int cv_snap_activation(cv_snap* snap, int layer, float* out);

/* ---- curvature products ------------------------------------------------- */
CV_API int cv_matvec(cv_snap* snap, int kind, const float* v, float* out);
CV_API int cv_jvp(cv_snap* snap, const float* v, float* out_bc);
CV_API int cv_vjp(cv_snap* snap, const float* U_bc, float* out);

/* ---- solver --------------------------------------------------------------- */
/* precond, x0 nullable.  lam/tol/floor are host doubles. */
CV_API int cv_cg_solve(cv_snap* snap, int kind, const float* g, double lam, double tol, int maxiter,
                int stabilise_every, const float* precond, double floor, const float* x0,
                float* x, cv_cg_stats* stats);

/* ---- estimators / control ----------------------------------------------- */
CV_API int cv_rademacher(cv_ctx* ctx, uint64_t seed, uint64_t counter, int64_t n, float* out);
/* Probes consume counter .. counter + n_probes*d (host keeps the Rng counter). */
CV_API int cv_hutchinson(cv_snap* snap, int kind, uint64_t seed, uint64_t counter, int n_probes,
                  float* diag_out /*nullable*/, double* trace_out /*nullable*/);
CV_API int cv_power_iter(cv_snap* snap, int kind, uint64_t seed, uint64_t counter, int iters,
                  double* eig_out);
/* mode 0: diag = max(beta*diag + (1-beta)*est, 0); mode 1: diag = max(est, 0). */
CV_API int cv_diag_ema(cv_ctx* ctx, float* diag, const float* est, double beta, int64_t d, int mode,
                double* mean_out /*nullable*/);
CV_API int cv_loss_at(cv_snap* snap, const float* w_next, double* loss_out);
CV_API int cv_rho_terms(cv_snap* snap, int kind, const float* g, const float* u,
                 double* g_dot_u, double* u_H_u);
/* update = coef * direction; w_next = w + update; scal[0]=||update||, scal[1]=#nonfinite
 * (direction, update, w_next), scal[2]=||direction||^2 (device doubles). */
CV_API int cv_apply_update(cv_ctx* ctx, const float* w, const float* direction, double coef, int64_t d,
                    float* update, float* w_next, double* scal);
/* scal[0] = ||x||^2, scal[1] = #nonfinite(x) (device doubles). */
CV_API int cv_norm_check(cv_ctx* ctx, const float* x, int64_t d, double* scal);

/* One link of a post-direction transform chain (transforms.py:22-99).  Host-side
 * scalars are pre-evaluated by the caller (schedules at step t, Adam bias
 * corrections at the link's step count), so the device never sees t:
 *   CV_LINK_SCALE                 p[0] = value (scale, or scale_by_schedule's value at t)
 *   CV_LINK_TRACE_MOMENTUM        p[0] = beta;          state_in[0] = trace, state_out[0] = new trace
 *   CV_LINK_ADD_DECAYED_WEIGHTS   p[0] = weight_decay   (reads w)
 *   CV_LINK_CLIP_GLOBAL_NORM      p[0] = max_norm       (global ||x|| reduced on the device)
 *   CV_LINK_SCALE_BY_ADAM         p[0..6] = b1, 1-b1, b2, 1-b2, eps, 1/(1-b1^t), 1/(1-b2^t);
 *                                 state_in/out[0] = m, [1] = v
 *   CV_LINK_SOPHIA_CLIP           p[0] = gamma, p[1] = eps (reads precond_diag)
 * State outputs are fresh buffers (the caller keeps the old state for an aborted step). */
enum {
  CV_LINK_SCALE = 0,
  CV_LINK_TRACE_MOMENTUM = 1,
  CV_LINK_ADD_DECAYED_WEIGHTS = 2,
  CV_LINK_SCALE_BY_ADAM = 3,
  CV_LINK_SOPHIA_CLIP = 4,
  CV_LINK_CLIP_GLOBAL_NORM = 5
};
typedef struct cv_link {
  int32_t kind;
  int32_t pad;
  double p[7];
  const float* state_in[2];
  float* state_out[2];
} cv_link;

/* update = chain(direction); w_next = w + update; scal as cv_apply_update.
 * links: host array of n_links; precond_diag nullable unless a sophia_clip link is present. */
CV_API int cv_chain_apply(cv_ctx* ctx, int n_links, const cv_link* links, const float* direction, const float* w,
                          const float* precond_diag, int64_t d, float* update, float* w_next, double* scal);

/* GNB diagonal over n_samples label draws; draw r uses the uniforms counter + r*b_global + 1
 * + row_offset + i for local row i (Rng.uniform(b_global), rows of this rank's shard). */
CV_API int cv_gnb_diag(cv_snap* snap, uint64_t seed, uint64_t counter, int n_samples, int64_t row_offset,
                       float* diag_out);

/* ---- engine unit test ----------------------------------------------------- */
/* out[M x N] (ld ldo) = A B with A, B given as fp32 (split inside): A(m,k) =
 * a[m*lda + k] if a_kmajor else a[k*lda + m]; B(k,n) = b[k*ldb + n] if !b_kmajor
 * else b[n*ldb + k].  engine: CV_ENGINE_SIMT or CV_ENGINE_TC (strict). */
CV_API int cv_gemm_test(cv_ctx* ctx, int engine, int M, int N, int K, const float* a, int64_t lda, int a_kmajor,
                        const float* b, int64_t ldb, int b_kmajor, float* out, int64_t ldo);

/* Diagnostic: average time (ms) of one tensor-core GEMM of the given shape on
 * resident random operands; mode 0 = fp32 store epilogue, 1 = split + ReLU-mask
 * epilogue (the JVP / backward epilogue).  Tuning aid, not on any product path. */
CV_API int cv_gemm_bench(cv_ctx* ctx, int M, int N, int K, int a_kmajor, int b_kmajor, int mode, int iters,
                         float* ms_out);

/* Test: two-segment tensor-core GEMM out = A.B + A.(s2 B), A M x K and B N x K
 * (K-major, K % 8 == 0): the segments' scale exponents differ by ~log2(s2),
 * exercising the accumulator rescaling between K segments. */
CV_API int cv_gemm_test_seg2(cv_ctx* ctx, int M, int N, int K, const float* a, const float* b, float s2, float* out);

/* ---- row lane ------------------------------------------------------------- */
CV_API int64_t cv_row_dim(const cv_snap* snap);                        /* m = b * c */
CV_API int cv_row_rhs(cv_snap* snap, float* rhs_out /* m */);
CV_API int cv_row_gram(cv_snap* snap, float* gram_out /* m*m, nullable: keep on device */);
CV_API int cv_row_solve_cholesky(cv_snap* snap, double mu, const float* rhs, float* v_out);
CV_API int cv_backproject(cv_snap* snap, const float* v_row, float* out);
/* Distributed row lane (solvers.py:146-161 across the ranks of ctx): the
 * same solve as cv_row_solve_cholesky with the Gram never held whole by one rank --
 * block-cyclic 1024-row panels, SYRK strips, right-looking Cholesky with broadcast
 * panels, distributed triangular solves and fp64 refinement.  `snap` is a whole-batch
 * snapshot built on a world-1 context of the same device (every rank gathers the batch);
 * rhs, v_out are the whole m-vectors, replicated.  Collective over ctx's ranks. */
CV_API int cv_row_solve_cholesky_dist(cv_ctx* ctx, cv_snap* snap, double mu, const float* rhs, float* v_out);
/* Row-space CG across the ranks of ctx (solvers.py:164-174): the cv_row_solve_cg loop with
 * replicated fp64 vectors, each Gram product from the ranks' block-cyclic Gram strips plus
 * one m-vector all-reduce.  Same snapshot / vector conventions as the Cholesky above. */
CV_API int cv_row_solve_cg_dist(cv_ctx* ctx, cv_snap* snap, double mu, const float* rhs, double tol, int maxiter,
                                int stabilise_every, const float* x0, float* v_out, cv_cg_stats* stats);
/* Row-space CG on (Gram + mu I) v = rhs with the snapshot's Gram (solvers.py:164-174,
 * method.py:270-282: row_solve_cg(lambda u: gram @ u, rhs, mu, cfg, x0)); the same
 * device-resident loop as cv_cg_solve, products are dense Gram GEMVs.  x0 nullable. */
CV_API int cv_row_solve_cg(cv_snap* snap, double mu, const float* rhs, double tol, int maxiter, int stabilise_every,
                           const float* x0, float* v_out, cv_cg_stats* stats);
/* The same two solves on a caller-owned dense symmetric Gram (m x m fp32, full storage,
 * device): solvers.py:146-161 row_solve_cholesky(gram, rhs, mu) and row_solve_cg with
 * gram_matvec = gram @ u.  Not positive definite -> CV_E_NOT_PD (the ContractError text). */
CV_API int cv_dense_cholesky_solve(cv_ctx* ctx, const float* gram, int64_t m, double mu, const float* rhs,
                                   float* v_out);
CV_API int cv_dense_cg_solve(cv_ctx* ctx, const float* gram, int64_t m, double mu, const float* rhs, double tol,
                             int maxiter, int stabilise_every, const float* x0, float* v_out, cv_cg_stats* stats);

#ifdef __cplusplus
}
#endif
#endif
