// Internal (non-ABI) structures of curvopt_b200.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <functional>
#include <map>
#include <string>
#include <vector>

#include "../../include/curvopt_b200.h"

namespace cv {

struct Scale;  // common.cuh: {int e; float amax;}

// ---------------------------------------------------------------------------
// Logical operand views.  X(i, j) = (hi[i*si + j*sj] + lo[i*si + j*sj]) * 2^-sc->e
// (scaled fp16 split, common.cuh), or plain fp32 f32[i*si + j*sj] (SIMT only).
// ---------------------------------------------------------------------------
struct Operand {
  const __half* hi = nullptr;
  const __half* lo = nullptr;
  int64_t si = 0, sj = 0;
  const Scale* sc = nullptr;
  const float* f32 = nullptr;   // plain fp32 operand (hi/lo unused)
};

struct GemmSeg {
  Operand A;  // M x K
  Operand B;  // K x N
  int K = 0;
};

enum EpiMode : int {
  EPI_STORE = 0,       // out[m*ld+n] = acc                      (weight gradients)
  EPI_SPLIT_ACT = 1,   // a = act(acc) -> split(out_hi/out_lo)   (forward hidden layers)
  EPI_SPLIT_MASK = 2,  // v = acc * act'(mask) -> split          (tangents, backward)
  EPI_HVP = 3,         // v = acc*sp + P*spp*dz (tanh) -> split   (HVP backward)
  EPI_GRAM = 4,        // out (+)= acc * SA[m/k, n/k]             (row-space Gram, models.py:323-333)
  EPI_ACCUM = 5,       // out += alpha * acc                      (Cholesky trailing update)
};

// Rigorous bound on |accumulator| used to pick a split output's exponent:
// sum_t k[t] * (*x[t]) * (*y[t]), the x / y being amax slots of the inputs.
struct AccBound {
  int n = 0;
  float k[4] = {0.f, 0.f, 0.f, 0.f};
  const float* x[4] = {nullptr, nullptr, nullptr, nullptr};
  const float* y[4] = {nullptr, nullptr, nullptr, nullptr};
};

struct Epilogue {
  int mode = EPI_STORE;
  int act = 0;                   // CV_ACT_*
  float* out = nullptr;          // fp32 output (EPI_STORE / GRAM / ACCUM)
  __half* out_hi = nullptr;      // split outputs
  __half* out_lo = nullptr;
  Scale* out_sc = nullptr;       // exponent written by the producer, amax accumulated
  int out_unit = 0;              // the output carries a ones column: its scale covers 1.0
  AccBound bound;                // bound on |acc| (split outputs)
  int64_t ld = 0;
  const __half* mask_hi = nullptr;  // stored activation a (split) at [m, n] for act'
  const __half* mask_lo = nullptr;
  const Scale* mask_sc = nullptr;
  int64_t mask_ld = 0;
  float* raw = nullptr;          // optional: pre-mask value (fp32), ld raw_ld
  int64_t raw_ld = 0;
  float* raw_amax = nullptr;     // optional: max |raw|
  const float* P = nullptr;      // EPI_HVP tanh: pre-mask G W^T from linearize
  int64_t P_ld = 0;
  const float* P_amax = nullptr;
  const float* dz = nullptr;     // EPI_HVP tanh: pre-mask tangent from the JVP
  int64_t dz_ld = 0;
  const float* dz_amax = nullptr;
  int mask_div = 1;              // mask row = m / mask_div (row lane: k rows per example)
  const float* sa = nullptr;     // EPI_GRAM: b x b activation Gram, ld sa_ld
  int64_t sa_ld = 0;
  int kdiv = 1;                  // EPI_GRAM: rows per example
  int64_t row0 = 0;              // EPI_GRAM: Gram row of the output's row 0 (row strips)
  int first = 0;                 // EPI_GRAM: overwrite instead of accumulate
  float alpha = 1.f;             // EPI_ACCUM
  // Fused output-layer JVP ("head", EPI_SPLIT_MASK on the last hidden layer only):
  // each epilogue thread accumulates, over its row m and its column half,
  //   head_part[g][m][:hc] = sum_n a(m, n) Vh[n, :] + t(m, n) Wh[n, :]
  // with a = the stored activation (mask operand), t = the masked tangent; a
  // fixed-order reduction over the groups g adds the bias row (models.py:243-255).
  const float* head_w = nullptr;   // N x hc fp32 (output layer W rows)
  const float* head_v = nullptr;   // N x hc fp32 (the product's V rows)
  float* head_part = nullptr;      // [groups][M][hc]
  int head_c = 0;
  int head_only = 0;               // skip the split tangent store (GGN: the head is its only consumer)
  // ReLU mask as packed bits (SplitBuf::bits): consumers read 2 bytes per 16 columns
  // instead of the 32-byte fp16 row; producers (EPI_SPLIT_ACT) write them
  const uint16_t* mask_bits = nullptr;
  int64_t mbits_ld = 0;
  uint16_t* bits_out = nullptr;
  int64_t bits_out_ld = 0;
};

// the row index lower_only compares against (GemmArgs / TcArgs)
template <class Args>
__host__ __device__ inline int lo_row(const Args& a, int m) {
  return a.cyc_nb ? m + (m / a.cyc_nb) * a.cyc_skip : m;
}

struct GemmArgs {
  int M = 0, N = 0;
  int nseg = 1;
  GemmSeg seg[2];
  Epilogue epi;
  const int* skip = nullptr;     // device flag: kernel returns immediately when != 0
  int lower_only = 0;            // > 0: only the lower part n <= m + (lower_only - 1) (diagonal offset)
  // lower_only on block-cyclic rows (the distributed row lane: a rank's panels of cyc_nb
  // rows are every world-th panel of the matrix): row m counts as m + (m / cyc_nb) * cyc_skip
  int cyc_nb = 0, cyc_skip = 0;
  cudaStream_t stream = nullptr; // nullptr: the context stream
  int max_ctas = 0;              // > 0: cap on the persistent grid (SM share when co-scheduled)
  int unsplit = 0;               // plan without split-K (the fused output head needs whole tiles)
};

struct SplitBuf {
  __half* hi = nullptr;
  __half* lo = nullptr;
  int64_t ld = 0;
  Scale* sc = nullptr;
  // ReLU activations: packed sign bits (bit k of word j of row m = hi[m, 16 j + k] > 0),
  // written by the forward epilogue; nullptr when not available (consumers read hi)
  uint16_t* bits = nullptr;
  int64_t bits_ld = 0;  // words per row (multiple of 8)
};

// Caching device allocator: exact-size free lists, never returns memory to the
// driver until the context dies (allocation on the step path must be free).
class Pool {
 public:
  void* get(size_t bytes);
  void put(void* p);
  void release_all();
  bool owns(void* p) const { return live_.count(p) != 0; }
  // While a CUDA graph is captured, allocations come from a separate arena the graph
  // owns: its replays write into those blocks, which must never be handed to other work.
  void redirect(Pool* arena) { redirect_ = arena; }
  Pool* redirected() const { return redirect_; }
  ~Pool() { release_all(); }

 private:
  std::map<void*, size_t> live_;
  std::multimap<size_t, void*> free_;
  Pool* redirect_ = nullptr;
};

}  // namespace cv

struct cv_ctx {
  int device = 0, world = 1, rank = 0;
  cudaStream_t stream = nullptr;
  int engine = CV_ENGINE_AUTO;
  int sm_count = 148;
  std::string err;
  cv::Pool pool;
  void* nccl = nullptr;          // ncclComm_t
  cv_comm_fn comm_fn = nullptr;  // external communicator (cv_ctx_set_comm), used instead of NCCL
  void* comm_user = nullptr;
  cudaStream_t comm = nullptr;   // NCCL stream of the per-layer (bucketed) gradient all-reduces
  std::vector<cudaEvent_t> comm_ev;
  double* red_ws = nullptr;      // reduction partials: kRedBlocks * 8 doubles
  double* scal_ws = nullptr;     // scratch scalars (64 doubles)
  float* amax_ws = nullptr;      // split.cu: per-block maxima (4 x 148 x 16 floats)
  unsigned* amax_counter = nullptr;  // split.cu: last-block counter (returns to 0 after each pass)
  int64_t launches = 0;
  cudaStream_t side = nullptr;   // second stream for co-scheduled independent GEMMs
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::vector<void*> deferred;   // side-stream scratch, returned to the pool after the join
  cudaStream_t side2 = nullptr;  // third stream: the output layer's weight gradient beside the pair
  cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;
  std::vector<void*> deferred2;  // side2 scratch, returned after side_join
  bool side_live = false, side2_live = false;  // forked and not yet joined
  int shard_cg = -1;             // CG vector sharding across ranks: -1 by size, 0 never, 1 always
  int64_t shard_chunk = 0;       // while a sharded CG's product runs: owner chunk of the reduction
};

struct cv_snap {
  cv_ctx* ctx = nullptr;
  int L = 0;
  std::vector<int> dims;
  std::vector<int64_t> off;       // flat offset of layer l's [W; b] block
  int64_t d = 0;
  int act = 0, loss = 0;
  int bl = 0, bg = 0;             // local / global batch
  int c = 0;
  // Scale slots (device, one array; common.cuh).  Linearization slots are zeroed
  // by cv_linearize, the per-product block [prod_sc, prod_sc + n_prod) by the
  // split of every product input.
  cv::Scale* scales = nullptr;
  int n_scales = 0;
  cv::Scale* w_sc = nullptr;      // [L] linearization weights, per layer block
  cv::Scale* v_sc = nullptr;      // [L] product input, per layer block
  cv::Scale* gout_sc = nullptr;   // G[L-1] (fp32 amax) and its split
  cv::Scale* U_sc = nullptr;      // product cotangent U (fp32 amax) and its split
  cv::Scale* U2_sc = nullptr;     // U2 amax
  cv::Scale* prod_sc = nullptr;   // start of the per-product block
  int n_prod = 0;
  int v_ready = 0;                // next product input: 1 scales published by its producer, 2 split written
  cv::Scale* scratch_sc = nullptr;  // [8] row lane / tests
  // weights of the linearization point, split, flat layout
  __half* w_hi = nullptr;
  __half* w_lo = nullptr;
  // augmented activations: acts[0] = [X | 1], acts[l] = [a_l | 1]; b x ld(n_l)
  std::vector<cv::SplitBuf> acts;
  std::vector<uint16_t*> bits_buf;  // [L] packed ReLU bits of acts[l] (l >= 1), see SplitBuf::bits
  int64_t bits_ld_max = 0;
  // loss state
  float* logits = nullptr;        // b x c
  float* probs = nullptr;         // b x c (ce)
  float* gout = nullptr;          // G[L-1] = out_grad / b_global, b x c fp32
  float* y_f = nullptr;           // mse targets copy
  int64_t* y_i = nullptr;         // ce labels copy
  // G[l] for hidden layers (l < L-1): b x ld(n_{l+1}); P[l] = G[l+1] W^T pre-mask (tanh)
  std::vector<cv::SplitBuf> G;
  std::vector<float*> P;
  std::vector<cv::Scale*> P_sc;   // amax of P[l]
  // per-product scratch
  __half* v_hi = nullptr;         // split of the product input (d)
  __half* v_lo = nullptr;
  std::vector<cv::SplitBuf> da;   // tangents of acts[l+1], zero column at n
  std::vector<float*> dz;         // pre-mask tangents (tanh HVP)
  std::vector<cv::Scale*> dz_sc;  // amax of dz[l]
  std::vector<cv::SplitBuf> gs;   // backward scratch (ping-pong size L-1)
  float* U = nullptr;             // b x c cotangent
  float* U2 = nullptr;            // b x c (backprojection cotangent)
  float* skinny_ws = nullptr;     // partial sums for skinny weight-gradient kernels
  int64_t skinny_ws_elems = 0;
  // tensor-core output layer (tc_out): the c-wide operands stored transposed and
  // padded (c -> cp rows, K contiguous, 16-byte rows) so TMA reads them K-major:
  // last-layer [W; b]^T (wl, ld ldw), per-product [V; Vb]^T (vl), cotangents U^T and
  // G[L-1]^T (ld ldb).  cp == c when the SIMT skinny kernels are used.
  int tc_out = 0, cp = 0;
  int64_t ldw = 0, ldb = 0;
  __half* wl_hi = nullptr; __half* wl_lo = nullptr;
  __half* vl_hi = nullptr; __half* vl_lo = nullptr;
  __half* U_hi = nullptr; __half* U_lo = nullptr;
  __half* gout_hi = nullptr; __half* gout_lo = nullptr;
  // fused output-layer head (EPI head_*): fp32 copy of the last layer's [W; b] block
  // ((n+1) x c) and the per-group partials of the output tangent
  float* wl_f32 = nullptr;
  float* head_part = nullptr;
  int head_groups_max = 0;
  // row lane (lazily built)
  float* seeds = nullptr;         // b x c x c  (H_z^{1/2})
  float* pinv = nullptr;          // b x c x c
  float* rhs = nullptr;           // m
  float* gram = nullptr;          // m x m
  float* chol = nullptr;          // m x m, Cholesky factor of gram + mu I (lower)
  float* dinv = nullptr;          // inverses of the 64-wide diagonal blocks of chol
  float* winv = nullptr;          // inverses of the 512-wide diagonal (panel) blocks of chol
  int row_state = 0;              // bit0 seeds built, bit1 gram (lower) built, bit2 gram mirrored
  // solver scratch (lazily allocated, d each)
  float* cg_r = nullptr; float* cg_p = nullptr; float* cg_ap = nullptr;
  float* tmp_d = nullptr; float* tmp_d2 = nullptr;
  std::vector<void*> owned;
};

// ---- internal launch helpers (defined in the .cu files) ----
namespace cv {
int64_t ld_for(int n);
void gemm_simt(cv_ctx* ctx, const GemmArgs& a);
bool gemm_tc_supported(const GemmArgs& a);
void gemm_tc(cv_ctx* ctx, const GemmArgs& a);
void gemm(cv_ctx* ctx, const GemmArgs& a);  // engine dispatch
// two independent GEMMs at once: a on the context stream, b on the side stream,
// the SMs split between them by estimated time; returns when both are enqueued
// (the context stream waits for b)
cudaStream_t gemm_pair(cv_ctx* ctx, GemmArgs a, GemmArgs b);  // returns the stream b ran on
double gemm_tc_estimate(const cv_ctx* ctx, const GemmArgs& g, int ctas);  // relative time on `ctas` SMs
cudaStream_t side_fork(cv_ctx* ctx);  // side stream ordered after the context stream's current work
cudaStream_t side2_fork(cv_ctx* ctx); // third stream, same ordering; joined by side_join
void side_join(cv_ctx* ctx);          // context stream waits for the side streams
// Enqueue on another stream for a scope: restores the context stream on exit, and on an
// exception also joins the side streams so no forked work is left unjoined.
struct StreamSwap {
  cv_ctx* c;
  cudaStream_t prev;
  int exc;
  StreamSwap(cv_ctx* ctx, cudaStream_t s);
  ~StreamSwap();
  StreamSwap(const StreamSwap&) = delete;
  StreamSwap& operator=(const StreamSwap&) = delete;
};
int gemm_tc_partial(cv_ctx* ctx, const GemmArgs& g, float** partial);  // N <= 32, raw split-K partials
// 0: no fused output-layer head; *via_reduce = 1: plan split-K (unsplit = 0) and the head
// is formed in the split-K reduction
int gemm_tc_head_groups(const cv_ctx* ctx, const GemmArgs& g, int* via_reduce = nullptr);
bool gemm_tc_tma_split(const cv_ctx* ctx, const GemmArgs& g);           // runs the TMA split epilogue (bits producer)

// runtime.cu
inline bool distributed(const cv_ctx* ctx) { return ctx->nccl != nullptr || ctx->comm_fn != nullptr; }
void allreduce_f32(cv_ctx* ctx, float* buf, int64_t n);
void allreduce_f64(cv_ctx* ctx, double* buf, int64_t n);
void reduce_to_owners(cv_ctx* ctx, float* buf, int64_t b0, int64_t b1, int64_t chunk, cudaStream_t st);
void allgather_f32(cv_ctx* ctx, float* buf, int64_t chunk);
void broadcast(cv_ctx* ctx, void* buf, int64_t n, int dtype, int root);
void comm_group(cv_ctx* ctx, bool begin);
int dist_row_cholesky(cv_ctx* ctx, cv_snap* s, double mu, const float* rhs, float* v_out);
void dist_row_cg(cv_ctx* ctx, cv_snap* s, double mu, const float* rhs, double tol, int maxiter, int stab,
                 const float* x0, float* v_out, cv_cg_stats* stats);
void dense_cg_run(cv_ctx* ctx, int64_t m, const std::function<void(const double*, double*, const int*)>& A,
                  const float* rhs, double mu, double tol, int maxiter, int stab, const float* x0, float* xout,
                  cv_cg_stats* stats);
// Per-layer ("bucketed") all-reduce of a flat parameter-space vector being produced
// layer by layer: ready(l, st) is called once layer l's block is final on stream st;
// with NCCL its all-reduce starts at once on the comm stream, overlapping the GEMMs
// still running for the lower layers; finish() orders the context stream after all
// of them.  With an external communicator the whole vector is reduced in finish().
struct LayerAllreduce {
  cv_ctx* ctx;
  float* out;
  const std::vector<int64_t>* off;
  int64_t d;
  int pending = 0;
  LayerAllreduce(cv_ctx* c, float* o, const std::vector<int64_t>& offs, int64_t dd) : ctx(c), out(o), off(&offs), d(dd) {}
  void ready(int l, cudaStream_t st);
  void finish();
};
void check_launch(cv_ctx* ctx);

// per-layer offset table of a flat parameter-space vector (kernel argument)
constexpr int kOffTabMax = 16;
struct OffTab {
  int64_t off[kOffTabMax + 1];
  int L;
};
inline OffTab make_off_tab(const std::vector<int64_t>& off, int64_t d) {
  OffTab t;
  t.L = (int)off.size();
  for (int l = 0; l < t.L; ++l) t.off[l] = off[l];
  t.off[t.L] = d;
  return t;
}
constexpr int kAmaxWsFloats = 4 * 148 * kOffTabMax;  // amax_ws block maxima; kOffTabMax floats follow,
                                                      // then k_cg_fused's second block-maxima table

// split.cu: scaled fp16 splits with exact amax (two passes)
void amax_into(cv_ctx* ctx, const float* x, int64_t n, Scale* slot);  // slot->amax = max|x|
void split_flat(cv_ctx* ctx, const float* x, int64_t d, const std::vector<int64_t>& off, __half* hi, __half* lo,
                Scale* sc, Scale* zero_sc, int n_zero, const int* skip);
void split_flat_apply(cv_ctx* ctx, const float* x, int64_t d, const std::vector<int64_t>& off, __half* hi,
                      __half* lo, const Scale* sc, const int* skip);
// p = M^-1 r + beta p with the per-layer amax of p published into sc (false: not fused, L > 16)
bool cg_pnext_amax(cv_ctx* ctx, const float* r, const float* pre, float lam, float floor_, const double* beta,
                   const int* done, float* p, int64_t d, const std::vector<int64_t>& off, Scale* sc, Scale* zero_sc,
                   int n_zero);
void split_rows(cv_ctx* ctx, const float* src, int64_t lds, int rows, int cols, const SplitBuf& dst, int ones);
void split_mat(cv_ctx* ctx, const float* src, int64_t lds, int rows, int cols, __half* hi, __half* lo, int64_t ldd,
               int trans, Scale* sc, int amax_ready, const int* skip, int pad_cols = 0);
void set_col_value(cv_ctx* ctx, const SplitBuf& b, int rows, int col, float v);
void gather_rows(cv_ctx* ctx, const SplitBuf& b, int rows, int cols, float* out);  // out = hi + lo

// mlp.cu
void mlp_linearize(cv_ctx* ctx, cv_snap* s, double* loss_out, float* grad_out);
void pad_last_weights(cv_ctx* ctx, cv_snap* s);
void mlp_ggn(cv_ctx* ctx, cv_snap* s, const float* v, float* out, const int* skip);
void mlp_hvp(cv_ctx* ctx, cv_snap* s, const float* v, float* out, const int* skip);
void mlp_jvp(cv_ctx* ctx, cv_snap* s, const float* v, float* out_bc);
void mlp_vjp(cv_ctx* ctx, cv_snap* s, const float* U, float* out);
void mlp_loss_at(cv_ctx* ctx, cv_snap* s, const float* w, double* loss_out);

using MatvecFn = void (*)(cv_ctx*, cv_snap*, const float*, float*, const int*);
inline MatvecFn matvec_fn(int kind) { return kind == CV_KIND_HESSIAN ? mlp_hvp : mlp_ggn; }

// vec.cu
void scale_scalar(cv_ctx* ctx, double* x, double s);
void cg_solve(cv_ctx* ctx, cv_snap* s, int kind, const float* g, double lam, double tol, int maxiter,
              int stab, const float* precond, double floor, const float* x0, float* x, cv_cg_stats* stats);
void dense_cg_solve(cv_ctx* ctx, const float* gram, int64_t m, const float* rhs, double mu, double tol, int maxiter,
                    int stab, const float* x0, float* x, cv_cg_stats* stats);
void rademacher(cv_ctx* ctx, uint64_t seed, uint64_t counter, int64_t n, float* out);
void hutchinson(cv_ctx* ctx, cv_snap* s, int kind, uint64_t seed, uint64_t counter, int n_probes, float* diag,
                double* trace);
void power_iter(cv_ctx* ctx, cv_snap* s, int kind, uint64_t seed, uint64_t counter, int iters, double* eig);
void diag_ema(cv_ctx* ctx, float* diag, const float* est, double beta, int64_t d, int mode, double* mean);
void dot_into(cv_ctx* ctx, const float* a, const float* b, int64_t n, double* out);
void apply_update(cv_ctx* ctx, const float* w, const float* dir, double coef, int64_t d, float* upd,
                  float* wn, double* scal);
void norm_check(cv_ctx* ctx, const float* x, int64_t d, double* scal);

// row.cu
int dense_cholesky(cv_ctx* ctx, const float* gram, int64_t m, double mu, const float* rhs, float* v_out);

// chain.cu
void chain_apply(cv_ctx* ctx, int n_links, const cv_link* links, const float* dir, const float* w, const float* pre,
                 int64_t d, float* upd, float* wn, double* scal);
void gnb_diag(cv_ctx* ctx, cv_snap* s, uint64_t seed, uint64_t counter, int n_samples, int64_t row_offset,
              float* diag);
}  // namespace cv
