// extern "C" entry points (include/curvopt_b200.h).
#include <stdio.h>
#include <string.h>

#include <stdexcept>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace cv {
void nccl_unique_id(void* out);
void nccl_init(cv_ctx* ctx, const void* id_bytes);
void nccl_destroy(cv_ctx* ctx);
// row.cu
void row_rhs(cv_ctx* ctx, cv_snap* s, float* rhs);
void row_gram(cv_ctx* ctx, cv_snap* s, float* gram_out);
int row_solve_cholesky(cv_ctx* ctx, cv_snap* s, double mu, const float* rhs, float* v);
void row_backproject(cv_ctx* ctx, cv_snap* s, const float* v, float* out);
const float* row_gram_dev(cv_ctx* ctx, cv_snap* s);
}  // namespace cv

using namespace cv;

struct CvError : std::runtime_error {
  int code;
  CvError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CV_TRY(ctxp)                                   \
  cv_ctx* _ctx = (ctxp);                               \
  if (!_ctx) return CV_E_CONTRACT;                     \
  try {                                                \
    cudaSetDevice(_ctx->device);
#define CV_CATCH                                       \
    check_launch(_ctx);                                \
    return CV_OK;                                      \
  } catch (const CvError& e) {                         \
    _ctx->err = e.what();                              \
    return e.code;                                     \
  } catch (const std::invalid_argument& e) {           \
    _ctx->err = e.what();                              \
    return CV_E_CONTRACT;                              \
  } catch (const std::exception& e) {                  \
    _ctx->err = e.what();                              \
    return strstr(e.what(), "NCCL") ? CV_E_NCCL : CV_E_CUDA; \
  }

static void contract(bool ok, const char* msg) {
  if (!ok) throw CvError(CV_E_CONTRACT, msg);
}

extern "C" {

const char* cv_version(void) { return "curvopt_b200 0.2.0 (sm_100a, tcgen05 scaled 3xFP16 + SIMT fp32)"; }

int cv_nccl_unique_id(void* out128) {
  try {
    nccl_unique_id(out128);
    return CV_OK;
  } catch (...) {
    return CV_E_NCCL;
  }
}

int cv_ctx_create(int device, int world, int rank, const void* nccl_id, cv_ctx** out) {
  if (!out || world < 1 || rank < 0 || rank >= world) return CV_E_CONTRACT;
  cv_ctx* c = new cv_ctx();
  c->device = device;
  c->world = world;
  c->rank = rank;
  *out = c;
  CV_TRY(c)
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (sms > 0) c->sm_count = sms;
  c->red_ws = (double*)c->pool.get(sizeof(double) * kRedBlocks * 8);
  c->scal_ws = (double*)c->pool.get(sizeof(double) * 64);
  c->amax_ws = (float*)c->pool.get(sizeof(float) * (2 * kAmaxWsFloats + kOffTabMax));  // split.cu SP_NB x SP_MAXL, mr; k_cg_fused
  c->amax_counter = (unsigned*)c->pool.get(sizeof(unsigned) * 64);
  cudaMemsetAsync(c->amax_counter, 0, sizeof(unsigned) * 64, c->stream);
  if (const char* e = getenv("CURVOPT_SHARD_CG")) c->shard_cg = atoi(e) != 0;  // test hook (default: by size)
  if (world > 1) {
    if (nccl_id) nccl_init(c, nccl_id);  // else: cv_ctx_set_comm installs the communicator
  } else if (getenv("CURVOPT_FORCE_NCCL")) {
    // single-rank communicator: exercises the NCCL path of every product on one GPU
    char id[128];
    nccl_unique_id(id);
    nccl_init(c, id);
  }
  CV_CATCH
}

int cv_ctx_set_comm(cv_ctx* ctx, cv_comm_fn fn, void* user) {
  CV_TRY(ctx)
  contract(_ctx->world > 1, "an external communicator needs world > 1");
  contract(_ctx->nccl == nullptr, "the context already owns an NCCL communicator");
  _ctx->comm_fn = fn;
  _ctx->comm_user = user;
  CV_CATCH
}

int cv_ctx_destroy(cv_ctx* ctx) {
  if (!ctx) return CV_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  try { nccl_destroy(ctx); } catch (...) {}
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
    cudaEventDestroy(ctx->ev_fork);
    cudaEventDestroy(ctx->ev_join);
  }
  if (ctx->side2) {
    cudaStreamSynchronize(ctx->side2);
    cudaStreamDestroy(ctx->side2);
    cudaEventDestroy(ctx->ev_fork2);
    cudaEventDestroy(ctx->ev_join2);
  }
  if (ctx->comm) {
    cudaStreamSynchronize(ctx->comm);
    cudaStreamDestroy(ctx->comm);
  }
  for (cudaEvent_t e : ctx->comm_ev) cudaEventDestroy(e);
  ctx->pool.release_all();
  delete ctx;
  return CV_OK;
}

int cv_ctx_set_stream(cv_ctx* ctx, void* stream) {
  if (!ctx) return CV_E_CONTRACT;
  ctx->stream = (cudaStream_t)stream;
  return CV_OK;
}

int cv_ctx_set_engine(cv_ctx* ctx, int engine) {
  if (!ctx || engine < 0 || engine > 2) return CV_E_CONTRACT;
  ctx->engine = engine;
  return CV_OK;
}

const char* cv_last_error(const cv_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int cv_ctx_capture_begin(cv_ctx* ctx) {
  CV_TRY(ctx)
  contract(_ctx->pool.redirected() == nullptr, "a graph capture is already open on this context");
  _ctx->pool.redirect(new Pool());
  CV_CATCH
}

int cv_ctx_capture_end(cv_ctx* ctx, void** arena_out) {
  if (!ctx || !arena_out) return CV_E_CONTRACT;
  Pool* a = ctx->pool.redirected();
  ctx->pool.redirect(nullptr);
  *arena_out = a;
  return a ? CV_OK : CV_E_CONTRACT;
}

int cv_arena_free(cv_ctx* ctx, void* arena) {
  if (!ctx) return CV_E_CONTRACT;
  cudaSetDevice(ctx->device);
  delete static_cast<Pool*>(arena);  // (after the graph that wrote into it is gone)
  return CV_OK;
}

int64_t cv_kernel_launches(const cv_ctx* ctx) { return ctx ? ctx->launches : -1; }

// ---------------------------------------------------------------------------
static float* alloc_f(cv_snap* s, int64_t n) {
  float* p = (float*)s->ctx->pool.get(sizeof(float) * (size_t)(n > 0 ? n : 1));
  s->owned.push_back(p);
  return p;
}

static __half* alloc_h(cv_snap* s, int64_t n) {
  __half* p = (__half*)s->ctx->pool.get(sizeof(__half) * (size_t)(n > 0 ? n : 1));
  s->owned.push_back(p);
  return p;
}

static SplitBuf alloc_split(cv_snap* s, int rows, int n, Scale* sc) {
  SplitBuf b;
  b.ld = ld_for(n);
  b.hi = alloc_h(s, (int64_t)rows * b.ld);
  b.lo = alloc_h(s, (int64_t)rows * b.ld);
  b.sc = sc;
  return b;
}

int cv_linearize(cv_ctx* ctx, int n_layers, const int* dims, int act, int loss, const float* w, const float* X,
                 const void* y, int b_local, int b_global, cv_snap** snap, double* loss_out, float* grad_out) {
  CV_TRY(ctx)
  contract(snap && dims && w && X && y && loss_out, "null argument");
  contract(n_layers >= 1, "model needs at least one layer");
  contract(b_local >= 1 && b_global >= b_local, "batch inputs must be a (b, input_dim) matrix with b >= 1");
  contract(act == CV_ACT_RELU || act == CV_ACT_TANH, "unknown activation");
  contract(loss == CV_LOSS_MSE || loss == CV_LOSS_CE, "unknown loss kind");
  for (int i = 0; i <= n_layers; ++i) contract(dims[i] >= 1, "layer widths must be >= 1");
  const int c = dims[n_layers];
  if (loss == CV_LOSS_CE) contract(c >= 2, "ce loss requires output_dim >= 2");
  if (c > 32) throw CvError(CV_E_UNSUPPORTED, "output_dim > 32 is not supported by the skinny output kernels");

  cv_snap* s = new cv_snap();
  s->ctx = ctx;
  s->L = n_layers;
  s->dims.assign(dims, dims + n_layers + 1);
  s->act = act;
  s->loss = loss;
  s->bl = b_local;
  s->bg = b_global;
  s->c = c;
  int64_t off = 0;
  for (int l = 0; l < n_layers; ++l) {
    s->off.push_back(off);
    off += (int64_t)(dims[l] + 1) * dims[l + 1];
  }
  s->d = off;
  const int L = n_layers, b = b_local;
  try {
    // Scale slots: w[L] v[L] acts[L] G[L-1] P[L-1] gout | per product: da[L-1] gs[L-1] U U2 dz[L-1] | scratch[8]
    const int H = L - 1;
    s->n_scales = 3 * L + 2 * H + 1 + (3 * H + 2) + 8;
    s->scales = (Scale*)ctx->pool.get(sizeof(Scale) * s->n_scales);
    s->owned.push_back(s->scales);
    Scale* p = s->scales;
    s->w_sc = p; p += L;
    s->v_sc = p; p += L;
    Scale* acts_sc = p; p += L;
    Scale* G_sc = p; p += H;
    Scale* P_sc = p; p += H;
    s->gout_sc = p; p += 1;
    s->prod_sc = p;
    Scale* da_sc = p; p += H;
    Scale* gs_sc = p; p += H;
    s->U_sc = p; p += 1;
    s->U2_sc = p; p += 1;
    Scale* dz_sc = p; p += H;
    s->n_prod = (int)(p - s->prod_sc);
    s->scratch_sc = p; p += 8;
    cudaMemsetAsync(s->scales, 0, sizeof(Scale) * s->n_scales, ctx->stream);

    s->w_hi = alloc_h(s, s->d);
    s->w_lo = alloc_h(s, s->d);
    s->v_hi = alloc_h(s, s->d);
    s->v_lo = alloc_h(s, s->d);
    for (int l = 0; l < L; ++l) s->acts.push_back(alloc_split(s, b, dims[l], acts_sc + l));
    // the weight and input splits go to the GPU before the remaining allocations: that host
    // work no longer leaves the device idle at the start of every step
    split_flat(ctx, w, s->d, s->off, s->w_hi, s->w_lo, s->w_sc, nullptr, 0, nullptr);
    split_rows(ctx, X, dims[0], b, dims[0], s->acts[0], 1);
    s->bits_buf.assign(L, nullptr);
    if (act == CV_ACT_RELU && ctx->engine != CV_ENGINE_SIMT)
      for (int l = 1; l < L; ++l) {
        const int64_t ldw = ((dims[l] + 15) / 16 + 7) / 8 * 8;
        s->bits_buf[l] = (uint16_t*)ctx->pool.get(sizeof(uint16_t) * (size_t)b * ldw);
        s->owned.push_back(s->bits_buf[l]);
      }
    s->logits = alloc_f(s, (int64_t)b * c);
    s->probs = alloc_f(s, (int64_t)b * c);
    s->gout = alloc_f(s, (int64_t)b * c);
    s->U = alloc_f(s, (int64_t)b * c);
    s->U2 = alloc_f(s, (int64_t)b * c);
    if (loss == CV_LOSS_CE) {
      s->y_i = (int64_t*)ctx->pool.get(sizeof(int64_t) * b);
      s->owned.push_back(s->y_i);
      cudaMemcpyAsync(s->y_i, y, sizeof(int64_t) * b, cudaMemcpyDeviceToDevice, ctx->stream);
    } else {
      s->y_f = alloc_f(s, (int64_t)b * c);
      cudaMemcpyAsync(s->y_f, y, sizeof(float) * b * c, cudaMemcpyDeviceToDevice, ctx->stream);
    }
    for (int l = 0; l + 1 < L; ++l) {
      const int n = dims[l + 1];
      s->G.push_back(alloc_split(s, b, n, G_sc + l));
      s->da.push_back(alloc_split(s, b, n, da_sc + l));
      s->gs.push_back(alloc_split(s, b, n, gs_sc + l));
      s->P.push_back(act == CV_ACT_TANH ? alloc_f(s, (int64_t)b * ld_for(n)) : nullptr);
      s->dz.push_back(act == CV_ACT_TANH ? alloc_f(s, (int64_t)b * ld_for(n)) : nullptr);
      s->P_sc.push_back(P_sc + l);
      s->dz_sc.push_back(dz_sc + l);
    }
    // skinny weight-gradient partials: up to 2*SMs column blocks x (n+1) x c
    int64_t need = 0;
    const int mrows = dims[L - 1] + 1;
    need = (int64_t)(2 * ctx->sm_count + 1) * mrows * c;
    s->skinny_ws_elems = need;
    s->skinny_ws = alloc_f(s, need);
    // output layer on the tensor-core engine when the shapes allow TMA operands
    s->cp = c;
    s->tc_out = ctx->engine != CV_ENGINE_SIMT && c >= 8 && b >= 128 && dims[L - 1] >= 64;
    if (s->tc_out) {
      s->cp = c <= 16 ? 16 : 32;
      s->ldw = ((int64_t)dims[L - 1] + 1 + 7) / 8 * 8;
      s->ldb = ((int64_t)b + 7) / 8 * 8;
      s->wl_hi = alloc_h(s, s->cp * s->ldw);
      s->wl_lo = alloc_h(s, s->cp * s->ldw);
      s->vl_hi = alloc_h(s, s->cp * s->ldw);
      s->vl_lo = alloc_h(s, s->cp * s->ldw);
      s->U_hi = alloc_h(s, s->cp * s->ldb);
      s->U_lo = alloc_h(s, s->cp * s->ldb);
      s->gout_hi = alloc_h(s, s->cp * s->ldb);
      s->gout_lo = alloc_h(s, s->cp * s->ldb);
    }
    if (L >= 2 && c <= 16 && ctx->engine != CV_ENGINE_SIMT) {
      s->wl_f32 = alloc_f(s, (int64_t)(dims[L - 1] + 1) * c);
      s->head_groups_max = 2 * ((dims[L - 1] + 63) / 64);  // narrowest head tile: 64 columns
      s->head_part = alloc_f(s, (int64_t)s->head_groups_max * b * c);
    }
  } catch (...) {
    for (void* p : s->owned) ctx->pool.put(p);
    delete s;
    throw;
  }
  if (s->wl_f32)
    cudaMemcpyAsync(s->wl_f32, w + s->off[L - 1], sizeof(float) * (size_t)(dims[L - 1] + 1) * c,
                    cudaMemcpyDeviceToDevice, ctx->stream);
  if (s->tc_out) pad_last_weights(ctx, s);
  for (int l = 0; l + 1 < L; ++l) set_col_value(ctx, s->da[l], b, dims[l + 1], 0.f);
  mlp_linearize(ctx, s, loss_out, grad_out);
  *snap = s;
  CV_CATCH
}

int cv_snap_free(cv_snap* s) {
  if (!s) return CV_OK;
  for (void* p : s->owned) s->ctx->pool.put(p);
  delete s;
  return CV_OK;
}

int64_t cv_snap_dim(const cv_snap* s) { return s ? s->d : -1; }

int cv_snap_outputs(cv_snap* s, float* out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  cudaMemcpyAsync(out, s->logits, sizeof(float) * s->bl * s->c, cudaMemcpyDeviceToDevice, _ctx->stream);
  CV_CATCH
}

int cv_snap_activation(cv_snap* s, int layer, float* out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  contract(layer >= 1 && layer < s->L, "activation layer out of range");
  gather_rows(_ctx, s->acts[layer], s->bl, s->dims[layer], out);
  CV_CATCH
}

int cv_matvec(cv_snap* s, int kind, const float* v, float* out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  contract(kind == CV_KIND_GGN || kind == CV_KIND_HESSIAN, "unknown curvature kind");
  matvec_fn(kind)(_ctx, s, v, out, nullptr);
  CV_CATCH
}

int cv_jvp(cv_snap* s, const float* v, float* out_bc) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  mlp_jvp(_ctx, s, v, out_bc);
  CV_CATCH
}

int cv_vjp(cv_snap* s, const float* U, float* out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  mlp_vjp(_ctx, s, U, out);
  CV_CATCH
}

int cv_cg_solve(cv_snap* s, int kind, const float* g, double lam, double tol, int maxiter, int stabilise_every,
                const float* precond, double floor, const float* x0, float* x, cv_cg_stats* stats) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  contract(tol > 0, "cg tol must be positive");
  contract(maxiter >= 1, "cg maxiter must be >= 1");
  contract(g && x && stats, "null argument");
  cg_solve(_ctx, s, kind, g, lam, tol, maxiter, stabilise_every, precond, floor, x0, x, stats);
  CV_CATCH
}

int cv_rademacher(cv_ctx* ctx, uint64_t seed, uint64_t counter, int64_t n, float* out) {
  CV_TRY(ctx)
  contract(n >= 1, "rademacher requires n >= 1");
  rademacher(_ctx, seed, counter, n, out);
  CV_CATCH
}

int cv_hutchinson(cv_snap* s, int kind, uint64_t seed, uint64_t counter, int n_probes, float* diag_out,
                  double* trace_out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  contract(n_probes >= 1, "hutchinson_diag requires n_probes >= 1");
  hutchinson(_ctx, s, kind, seed, counter, n_probes, diag_out, trace_out);
  CV_CATCH
}

int cv_power_iter(cv_snap* s, int kind, uint64_t seed, uint64_t counter, int iters, double* eig_out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  contract(iters >= 1, "power_iter_top_eig requires iters >= 1");
  power_iter(_ctx, s, kind, seed, counter, iters, eig_out);
  CV_CATCH
}

int cv_diag_ema(cv_ctx* ctx, float* diag, const float* est, double beta, int64_t d, int mode, double* mean_out) {
  CV_TRY(ctx)
  diag_ema(_ctx, diag, est, beta, d, mode, mean_out);
  CV_CATCH
}

int cv_loss_at(cv_snap* s, const float* w_next, double* loss_out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  mlp_loss_at(_ctx, s, w_next, loss_out);
  CV_CATCH
}

int cv_rho_terms(cv_snap* s, int kind, const float* g, const float* u, double* g_dot_u, double* u_H_u) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  dot_into(_ctx, g, u, s->d, g_dot_u);
  float* hu = s->cg_ap;
  if (!hu) {
    hu = (float*)_ctx->pool.get(sizeof(float) * s->d);
    s->owned.push_back(hu);
    s->cg_ap = hu;
  }
  matvec_fn(kind)(_ctx, s, u, hu, nullptr);
  dot_into(_ctx, hu, u, s->d, u_H_u);
  CV_CATCH
}

int cv_apply_update(cv_ctx* ctx, const float* w, const float* direction, double coef, int64_t d, float* update,
                    float* w_next, double* scal) {
  CV_TRY(ctx)
  apply_update(_ctx, w, direction, coef, d, update, w_next, scal);
  CV_CATCH
}

int cv_norm_check(cv_ctx* ctx, const float* x, int64_t d, double* scal) {
  CV_TRY(ctx)
  norm_check(_ctx, x, d, scal);
  CV_CATCH
}

int cv_chain_apply(cv_ctx* ctx, int n_links, const cv_link* links, const float* direction, const float* w,
                   const float* precond_diag, int64_t d, float* update, float* w_next, double* scal) {
  CV_TRY(ctx)
  contract(n_links >= 0 && (n_links == 0 || links), "chain links missing");
  contract(direction && w && update && w_next && scal && d >= 1, "chain_apply needs direction, w and outputs");
  chain_apply(_ctx, n_links, links, direction, w, precond_diag, d, update, w_next, scal);
  CV_CATCH
}

int cv_gnb_diag(cv_snap* s, uint64_t seed, uint64_t counter, int n_samples, int64_t row_offset, float* diag_out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  contract(diag_out != nullptr, "gnb_diag needs an output");
  gnb_diag(_ctx, s, seed, counter, n_samples, row_offset, diag_out);
  CV_CATCH
}

int cv_gemm_test(cv_ctx* ctx, int engine, int M, int N, int K, const float* a, int64_t lda, int a_kmajor,
                 const float* b, int64_t ldb, int b_kmajor, float* out, int64_t ldo) {
  CV_TRY(ctx)
  // a: M x K (K-major, ld lda) or K x M (M-major); b: K x N (N-major, ld ldb) or N x K (K-major)
  const int ar = a_kmajor ? M : K, ac = a_kmajor ? K : M;
  const int br = b_kmajor ? N : K, bc = b_kmajor ? K : N;
  const int64_t na = (int64_t)ar * lda, nb = (int64_t)br * ldb;
  __half* buf = (__half*)_ctx->pool.get(sizeof(__half) * (size_t)(2 * na + 2 * nb) + 64);
  Scale* sc = (Scale*)_ctx->pool.get(sizeof(Scale) * 2);
  __half *ahi = buf, *alo = buf + na, *bhi = buf + 2 * na, *blo = buf + 2 * na + nb;
  split_mat(_ctx, a, lda, ar, ac, ahi, alo, lda, 0, sc, 0, nullptr);
  split_mat(_ctx, b, ldb, br, bc, bhi, blo, ldb, 0, sc + 1, 0, nullptr);
  GemmArgs g;
  g.M = M;
  g.N = N;
  g.nseg = 1;
  Operand A, B;
  A.hi = ahi; A.lo = alo; A.sc = sc;
  B.hi = bhi; B.lo = blo; B.sc = sc + 1;
  if (a_kmajor) { A.si = lda; A.sj = 1; } else { A.si = 1; A.sj = lda; }
  if (b_kmajor) { B.si = 1; B.sj = ldb; } else { B.si = ldb; B.sj = 1; }
  g.seg[0].A = A;
  g.seg[0].B = B;
  g.seg[0].K = K;
  g.epi.mode = EPI_STORE;
  g.epi.out = out;
  g.epi.ld = ldo;
  if (engine == CV_ENGINE_TC) {
    contract(gemm_tc_supported(g), "shape/alignment not supported by the tensor-core engine");
    gemm_tc(_ctx, g);
  } else {
    gemm_simt(_ctx, g);
  }
  _ctx->pool.put(sc);
  _ctx->pool.put(buf);
  CV_CATCH
}

int64_t cv_row_dim(const cv_snap* s) { return s ? (int64_t)s->bl * s->c : -1; }

int cv_row_rhs(cv_snap* s, float* rhs_out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  row_rhs(_ctx, s, rhs_out);
  CV_CATCH
}

int cv_row_gram(cv_snap* s, float* gram_out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  contract(_ctx->world == 1, "row lane is single-GPU (replicas only)");
  row_gram(_ctx, s, gram_out);
  CV_CATCH
}

int cv_row_solve_cholesky(cv_snap* s, double mu, const float* rhs, float* v_out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  contract(_ctx->world == 1, "row lane is single-GPU (replicas only)");
  if (row_solve_cholesky(_ctx, s, mu, rhs, v_out) != 0)
    throw CvError(CV_E_NOT_PD, "row system is not positive definite; mu too small or gram invalid");
  CV_CATCH
}

int cv_row_solve_cholesky_dist(cv_ctx* ctx, cv_snap* s, double mu, const float* rhs, float* v_out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(ctx)
  contract(s->ctx->device == _ctx->device, "snapshot and context are on different devices");
  contract(s->ctx->world == 1, "the distributed row lane takes a whole-batch (replicated) snapshot");
  if (s->ctx->stream != _ctx->stream) {  // the snapshot's work first
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, s->ctx->stream);
    cudaStreamWaitEvent(_ctx->stream, e, 0);
    cudaEventDestroy(e);
  }
  if (dist_row_cholesky(_ctx, s, mu, rhs, v_out) != 0)
    throw CvError(CV_E_NOT_PD, "row system is not positive definite; mu too small or gram invalid");
  CV_CATCH
}

int cv_row_solve_cg_dist(cv_ctx* ctx, cv_snap* s, double mu, const float* rhs, double tol, int maxiter,
                         int stabilise_every, const float* x0, float* v_out, cv_cg_stats* stats) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(ctx)
  contract(s->ctx->device == _ctx->device, "snapshot and context are on different devices");
  contract(s->ctx->world == 1, "the distributed row lane takes a whole-batch (replicated) snapshot");
  contract(tol > 0 && maxiter >= 1, "cg tol must be positive and maxiter >= 1");
  if (s->ctx->stream != _ctx->stream) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, s->ctx->stream);
    cudaStreamWaitEvent(_ctx->stream, e, 0);
    cudaEventDestroy(e);
  }
  dist_row_cg(_ctx, s, mu, rhs, tol, maxiter, stabilise_every, x0, v_out, stats);
  CV_CATCH
}

int cv_row_solve_cg(cv_snap* s, double mu, const float* rhs, double tol, int maxiter, int stabilise_every,
                    const float* x0, float* v_out, cv_cg_stats* stats) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  contract(_ctx->world == 1, "row lane is single-GPU (replicas only)");
  contract(tol > 0 && maxiter >= 1, "cg tol must be positive and maxiter >= 1");
  const float* G = row_gram_dev(_ctx, s);
  dense_cg_solve(_ctx, G, (int64_t)s->bl * s->c, rhs, mu, tol, maxiter, stabilise_every, x0, v_out, stats);
  CV_CATCH
}

int cv_dense_cholesky_solve(cv_ctx* ctx, const float* gram, int64_t m, double mu, const float* rhs, float* v_out) {
  CV_TRY(ctx)
  contract(m >= 1 && gram && rhs && v_out, "gram must be a square matrix");
  if (dense_cholesky(_ctx, gram, m, mu, rhs, v_out) != 0)
    throw CvError(CV_E_NOT_PD, "row system is not positive definite; mu too small or gram invalid");
  CV_CATCH
}

int cv_dense_cg_solve(cv_ctx* ctx, const float* gram, int64_t m, double mu, const float* rhs, double tol, int maxiter,
                      int stabilise_every, const float* x0, float* v_out, cv_cg_stats* stats) {
  CV_TRY(ctx)
  contract(m >= 1 && gram && rhs && v_out && stats, "gram must be a square matrix");
  contract(tol > 0 && maxiter >= 1, "cg tol must be positive and maxiter >= 1");
  dense_cg_solve(_ctx, gram, m, rhs, mu, tol, maxiter, stabilise_every, x0, v_out, stats);
  CV_CATCH
}

int cv_backproject(cv_snap* s, const float* v_row, float* out) {
  if (!s) return CV_E_CONTRACT;
  CV_TRY(s->ctx)
  row_backproject(_ctx, s, v_row, out);
  CV_CATCH
}

}  // extern "C"
