// MLP linearization and curvature products on device.
//
// Notation (augmented form): A_l = [a_l | 1] (b x ld, ones column at n_l) and the
// parameter block of layer l, [W_l ; b_l], is the (n_l+1) x n_{l+1} row-major slice
// of the flat vector (models.py:87-93).  Hence
//   forward   z_l   = A_l [W_l; b_l]                      (models.py:346-357)
//   jvp       dz_l  = A_l [V_l; Vb_l] + da_{l-1} W_l      (models.py:243-255)
//   vjp       [gW;gb]_l = A_l^T G_l                       (models.py:274-285)
//   hvp       [gW;gb]_l = A_l^T dG + [da_{l-1}|0]^T G_l   (models.py:287-307)
// so biases never need their own epilogue and the bias gradient is the extra row.
//
// Every GEMM operand is a scaled fp16 pair (common.cuh).  Split outputs take their
// exponent from a bound on |acc| built from the inputs' amax slots (AccBound):
// for a segment with reduction depth K, |sum_k A_mk B_kn| <= K amax(A) amax(B).
#include "common.cuh"
#include "internal.h"
#include "epilogue.cuh"
#include "skinny.cuh"

namespace cv {

// leading dimension of a b x (n + 1) split activation: 16-byte rows for TMA
int64_t ld_for(int n) { return ((int64_t)n + 1 + 7) / 8 * 8; }

static int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

static const float* am(const Scale* sc) { return &sc->amax; }

static void bound_add(AccBound& b, float k, const Scale* x, const Scale* y) {
  b.k[b.n] = k;
  b.x[b.n] = am(x);
  b.y[b.n] = am(y);
  ++b.n;
}

// ---------------------------------------------------------------------------
// Loss rows: softmax-CE / MSE value, probabilities and G[L-1] = out_grad / b
// (models.py:358-383).  Per-block fp64 partial sums of the per-example loss.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_loss_rows(const float* __restrict__ logits, int rows, int c, int loss,
                                                   const int64_t* __restrict__ yi, const float* __restrict__ yf,
                                                   float* probs, float* gout, float inv_b, double* partial,
                                                   int write_state, float* gout_amax) {
  CV_PDL_ENTRY();
  double part[1] = {0.0};
  float amax = 0.f;
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < rows; m += gridDim.x * blockDim.x) {
    const float* z = logits + (int64_t)m * c;
    if (loss == CV_LOSS_CE) {
      double mx = z[0];
      for (int j = 1; j < c; ++j) mx = fmax(mx, (double)z[j]);
      double se = 0.0;
      for (int j = 0; j < c; ++j) se += exp((double)z[j] - mx);
      const int64_t y = yi[m];
      part[0] += log(se) - ((double)z[y] - mx);
      if (write_state) {
        for (int j = 0; j < c; ++j) {
          const double p = exp((double)z[j] - mx) / se;
          probs[(int64_t)m * c + j] = (float)p;
          const float g = (float)((p - (j == y ? 1.0 : 0.0)) * inv_b);
          gout[(int64_t)m * c + j] = g;
          amax = fmaxf(amax, fabsf(g));
        }
      }
    } else {
      double s = 0.0;
      for (int j = 0; j < c; ++j) {
        const double r = (double)z[j] - (double)yf[(int64_t)m * c + j];
        s += r * r;
        if (write_state) {
          const float g = (float)(r * inv_b);
          gout[(int64_t)m * c + j] = g;
          amax = fmaxf(amax, fabsf(g));
        }
      }
      part[0] += 0.5 * s;
    }
  }
  amax = warp_max_f(amax);
  if ((threadIdx.x & 31) == 0 && write_state) atomic_amax(gout_amax, amax);
  block_sum<1>(part);
  if (threadIdx.x == 0) partial[blockIdx.x] = part[0];
}

// Sum nblk partials in fixed order, scale, store to *out (device double).
__global__ void k_finalize_sum(const double* partial, int nblk, double scale, double* out) {
  CV_PDL_ENTRY();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nblk; ++i) s += partial[i];
    *out = s * scale;
  }
}

// ---------------------------------------------------------------------------
// Tensor-core output layer helpers (tc_out)
// ---------------------------------------------------------------------------
// (rows x c, ld c) split block -> transposed, padded (cp x ldo) split, same exponent
__global__ void k_pad_t(const __half* hi, const __half* lo, int rows, int c, int cp, int64_t ldo, __half* ohi,
                        __half* olo, const int* skip) {
  CV_PDL_ENTRY();
  if (skip_if(skip)) return;
  const int64_t total = (int64_t)cp * rows;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / rows, r = i - j * rows;
    __half h = __float2half_rn(0.f), l = h;
    if (j < c) {
      h = hi[r * c + j];
      l = lo[r * c + j];
    }
    ohi[j * ldo + r] = h;
    olo[j * ldo + r] = l;
  }
}

// out-layer JVP: sum the split-K / head-group partials of z = J v per row (+ the
// bias row), then either store the logits tangent (POST_LOGITS) or
// U = H_z(z) * scale (models.py:199-204).  A block owns 128 rows: the partial
// slabs [z][rows][c] are read coalesced (each thread sums fixed element positions
// over z in fixed order), then rows are finished from shared memory.
template <int CM>
__global__ void __launch_bounds__(128) k_out_reduce(const float* part, int splits, int rows, int c, int post, int loss,
                                                    const float* probs, float scale, float* out, float* out_amax,
                                                    const int* skip, const float* bias) {
  constexpr int RB = 32;             // rows per block
  constexpr int PT = RB * CM / 128;  // element positions per thread
  constexpr int SB = 8;              // slabs in flight
  __shared__ float tile[RB * CM];
  const int m0 = blockIdx.x * RB;
  const int nrows = min(RB, rows - m0);
  const int nel = nrows * c;
  // bias and probabilities come from the linearization / the product input: loaded before
  // the wait for the partials' producer
  float acc[PT];
#pragma unroll
  for (int u = 0; u < PT; ++u) {
    const int e = threadIdx.x + 128 * u;
    acc[u] = (bias && e < nel) ? bias[e % c] : 0.f;
  }
  const int r = threadIdx.x, m = m0 + r;
  float pr[CM];
  const bool hz_ce = post == 1 && loss == CV_LOSS_CE;
#pragma unroll
  for (int j = 0; j < CM; ++j) pr[j] = (hz_ce && r < nrows && j < c) ? probs[(int64_t)m * c + j] : 0.f;
  CV_PDL_ENTRY();
  if (skip_if(skip)) return;
  // SB slabs' loads in flight before their (fixed-order) adds
  int z = 0;
  for (; z + SB <= splits; z += SB) {
    float x[SB][PT];
#pragma unroll
    for (int i = 0; i < SB; ++i) {
      const float* p = part + ((int64_t)(z + i) * rows + m0) * c;
#pragma unroll
      for (int u = 0; u < PT; ++u) {
        const int e = threadIdx.x + 128 * u;
        x[i][u] = e < nel ? p[e] : 0.f;
      }
    }
#pragma unroll
    for (int i = 0; i < SB; ++i)
#pragma unroll
      for (int u = 0; u < PT; ++u) acc[u] += x[i][u];
  }
  for (; z < splits; ++z) {
    const float* p = part + ((int64_t)z * rows + m0) * c;
#pragma unroll
    for (int u = 0; u < PT; ++u) {
      const int e = threadIdx.x + 128 * u;
      if (e < nel) acc[u] += p[e];
    }
  }
#pragma unroll
  for (int u = 0; u < PT; ++u) {
    const int e = threadIdx.x + 128 * u;
    if (e < nel) tile[e] = acc[u];
  }
  __syncthreads();
  float amax = 0.f;
  if (r < nrows) {
    float t[CM];
#pragma unroll
    for (int j = 0; j < CM; ++j) t[j] = j < c ? tile[r * c + j] : 0.f;
    if (post == 1) {
      if (loss == CV_LOSS_CE) {
        const float* p = pr;
        float pt = 0.f;
#pragma unroll
        for (int j = 0; j < CM; ++j)
          if (j < c) pt = fmaf(p[j], t[j], pt);
#pragma unroll
        for (int j = 0; j < CM; ++j)
          if (j < c) t[j] = (p[j] * t[j] - p[j] * pt) * scale;
      } else {
#pragma unroll
        for (int j = 0; j < CM; ++j) t[j] *= scale;
      }
    }
#pragma unroll
    for (int j = 0; j < CM; ++j)
      if (j < c) {
        tile[r * c + j] = t[j];
        amax = fmaxf(amax, fabsf(t[j]));
      }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nel; e += 128) out[(int64_t)m0 * c + e] = tile[e];  // coalesced
  amax = warp_max_f(amax);
  if ((threadIdx.x & 31) == 0 && out_amax) atomic_amax(out_amax, amax);
}

// ---------------------------------------------------------------------------
// Host orchestration
// ---------------------------------------------------------------------------
static Operand mk_op(const __half* hi, const __half* lo, int64_t si, int64_t sj, const Scale* sc) {
  Operand o;
  o.hi = hi;
  o.lo = lo;
  o.si = si;
  o.sj = sj;
  o.sc = sc;
  return o;
}
static Operand op_rows(const SplitBuf& b) { return mk_op(b.hi, b.lo, b.ld, 1, b.sc); }   // X(m,k)=buf[m,k]
static Operand op_trans(const SplitBuf& b) { return mk_op(b.hi, b.lo, 1, b.ld, b.sc); }  // X(m,k)=buf[k,m]
// layer block [W; b] (rows x nout, row-major): B(k, n) = W[k, n]  /  B(k, n) = W[n, k]
static Operand op_wblock(const __half* hi, const __half* lo, int nout, const Scale* sc) {
  return mk_op(hi, lo, nout, 1, sc);
}
static Operand op_wT(const __half* hi, const __half* lo, int nout, const Scale* sc) { return mk_op(hi, lo, 1, nout, sc); }

static void split_epi(Epilogue& e, const SplitBuf& out) {
  e.out_hi = out.hi;
  e.out_lo = out.lo;
  e.ld = out.ld;
  e.out_sc = out.sc;
}
static void mask_epi(Epilogue& e, const SplitBuf& a) {
  e.mask_hi = a.hi;
  e.mask_lo = a.lo;
  e.mask_ld = a.ld;
  e.mask_sc = a.sc;
  e.mask_bits = a.bits;
  e.mbits_ld = a.bits_ld;
}

// last-layer block of a split flat vector -> transposed padded split (tc_out)
static void pad_last(cv_ctx* ctx, cv_snap* s, const __half* hi, const __half* lo, __half* ohi, __half* olo,
                     const int* skip) {
  const int l = s->L - 1;
  const int rows = s->dims[l] + 1;
  launch_k(ctx->stream, k_pad_t, grid_for((int64_t)rows * s->cp), 256, 0, hi + s->off[l], lo + s->off[l], rows, s->c, s->cp,
                                                                     s->ldw, ohi, olo, skip);
  ctx->launches++;
}

void pad_last_weights(cv_ctx* ctx, cv_snap* s) { pad_last(ctx, s, s->w_hi, s->w_lo, s->wl_hi, s->wl_lo, nullptr); }

// The transposed split (cp x ldb) of a b x c cotangent whose amax slot is valid:
// G[L-1] keeps its resident split, anything else is split into U_hi / U_lo.
static const Scale* cot_split(cv_ctx* ctx, cv_snap* s, const float* U, Scale* usc, const __half** hi,
                              const __half** lo, const int* skip) {
  if (U == s->gout) {
    *hi = s->gout_hi;
    *lo = s->gout_lo;
    return s->gout_sc;
  }
  split_mat(ctx, U, s->c, s->bl, s->c, s->U_hi, s->U_lo, s->ldb, 1, usc, 1, skip);
  *hi = s->U_hi;
  *lo = s->U_lo;
  return usc;
}

// bits: packed ReLU sign-bit buffer of `out` (linearization only); returns whether the
// GEMM's epilogue wrote it
// head_groups: when non-null and this is the last hidden layer, the output layer's
// logits are accumulated in the GEMM's epilogue (partials in s->head_part; the count is
// returned, 0 when the GEMM cannot carry the head)
bool mlp_forward_layer(cv_ctx* ctx, cv_snap* s, int l, const SplitBuf& in, const __half* whi, const __half* wlo,
                       const Scale* wsc, const SplitBuf& out, uint16_t* bits = nullptr, int* head_groups = nullptr,
                       const float* head_wf = nullptr) {
  GemmArgs g;
  g.M = s->bl;
  g.N = s->dims[l + 1];
  g.nseg = 1;
  g.seg[0] = GemmSeg{op_rows(in), op_wblock(whi + s->off[l], wlo + s->off[l], s->dims[l + 1], wsc + l), s->dims[l] + 1};
  g.epi.mode = EPI_SPLIT_ACT;
  g.epi.act = s->act;
  split_epi(g.epi, out);
  g.epi.out_unit = 1;
  bound_add(g.epi.bound, (float)(s->dims[l] + 1), in.sc, wsc + l);
  if (head_groups) {
    *head_groups = 0;
    if (s->head_part && head_wf && l == s->L - 2) {
      g.epi.head_w = head_wf;
      g.epi.head_v = head_wf;  // unused by the forward head (zero activation tangent)
      g.epi.head_c = s->c;
      g.epi.head_part = s->head_part;
      g.unsplit = 1;
      const int gr = gemm_tc_head_groups(ctx, g);
      if (gr > 0 && gr <= s->head_groups_max) {
        *head_groups = gr;
      } else {
        g.epi.head_w = g.epi.head_v = nullptr;
        g.epi.head_part = nullptr;
        g.epi.head_c = 0;
        g.unsplit = 0;
      }
    }
  }
  bool wrote = false;
  if (bits && s->act == CV_ACT_RELU && gemm_tc_tma_split(ctx, g)) {
    g.epi.bits_out = bits;
    g.epi.bits_out_ld = ((s->dims[l + 1] + 15) / 16 + 7) / 8 * 8;
    wrote = true;
  }
  const bool tma_epi = gemm_tc_tma_split(ctx, g);  // that epilogue also writes the ones column
  gemm(ctx, g);
  // the ones column of the next layer's augmented input (covered by the scale)
  if (!tma_epi) set_col_value(ctx, out, s->bl, s->dims[l + 1], 1.f);
  return wrote;
}

// logits = A_{L-1} [W; b]  (skinny)
void mlp_output_layer(cv_ctx* ctx, cv_snap* s, const SplitBuf& in, const __half* whi, const __half* wlo,
                      const Scale* wsc, float* logits) {
  const int l = s->L - 1;
  if (s->tc_out) {
    const __half *bh = s->wl_hi, *bl = s->wl_lo;
    if (whi != s->w_hi) {  // another parameter point (loss_at): pad its last block
      pad_last(ctx, s, whi, wlo, s->vl_hi, s->vl_lo, nullptr);
      bh = s->vl_hi;
      bl = s->vl_lo;
    }
    GemmArgs g;
    g.M = s->bl;
    g.N = s->c;
    g.nseg = 1;
    g.seg[0] = GemmSeg{op_rows(in), mk_op(bh, bl, 1, s->ldw, wsc + l), s->dims[l] + 1};
    g.epi.mode = EPI_STORE;
    g.epi.out = logits;
    g.epi.ld = s->c;
    gemm(ctx, g);
    return;
  }
  SkinnyRowsArgs a{};
  a.rows = s->bl;
  a.c = s->c;
  a.nseg = 1;
  a.seg[0] = SkinnySeg{in.hi, in.lo, in.ld, in.sc, whi + s->off[l], wlo + s->off[l], s->c, wsc + l, s->dims[l] + 1};
  a.post = POST_LOGITS;
  a.loss = s->loss;
  a.out = logits;
  skinny_rows(ctx, a);
}

void mlp_loss(cv_ctx* ctx, cv_snap* s, const float* logits, int write_state, double* loss_out);

// G_prev = (U W_l^T) * act'(a_l) for the output layer (l = L-1), skinny K = c.
static void skinny_backward(cv_ctx* ctx, cv_snap* s, const float* U, Scale* usc, const __half* whi, const __half* wlo,
                            const Scale* wsc, const SplitBuf& out, float* raw, Scale* raw_sc, const int* skip) {
  const int l = s->L - 1;
  SkinnyDxArgs a{};
  a.rows = s->bl;
  a.n = s->dims[l];
  a.c = s->c;
  a.nseg = 1;
  a.U[0] = U;
  a.w_hi[0] = whi + s->off[l];
  a.w_lo[0] = wlo + s->off[l];
  a.w_sc[0] = wsc + l;
  a.epi.mode = EPI_SPLIT_MASK;
  a.epi.act = s->act;
  split_epi(a.epi, out);
  mask_epi(a.epi, s->acts[l]);
  a.epi.raw = raw;
  a.epi.raw_ld = out.ld;
  a.epi.raw_amax = raw_sc ? &raw_sc->amax : nullptr;
  bound_add(a.epi.bound, (float)s->c, usc, wsc + l);
  a.skip = skip;
  skinny_dx(ctx, a);
}

// G_prev = (G_l W_l^T) * act'(a_l), hidden layer l >= 1
static GemmArgs hidden_backward_args(cv_snap* s, int l, const SplitBuf& Gl, const __half* whi, const __half* wlo,
                                     const Scale* wsc, const SplitBuf& out, float* raw, Scale* raw_sc,
                                     const int* skip) {
  GemmArgs g;
  g.M = s->bl;
  g.N = s->dims[l];
  g.nseg = 1;
  g.seg[0] = GemmSeg{op_rows(Gl), op_wT(whi + s->off[l], wlo + s->off[l], s->dims[l + 1], wsc + l), s->dims[l + 1]};
  g.epi.mode = EPI_SPLIT_MASK;
  g.epi.act = s->act;
  split_epi(g.epi, out);
  mask_epi(g.epi, s->acts[l]);
  g.epi.raw = raw;
  g.epi.raw_ld = out.ld;
  g.epi.raw_amax = raw_sc ? &raw_sc->amax : nullptr;
  bound_add(g.epi.bound, (float)s->dims[l + 1], Gl.sc, wsc + l);
  g.skip = skip;
  return g;
}

// [gW; gb]_l = A_l^T G (+ A2^T G2), written into out + off[l] (hidden layers); the
// ones column of A_l makes the bias gradient the GEMM's last row.
static GemmArgs weight_grad_args(cv_snap* s, int l, const SplitBuf& G1, const SplitBuf* A2, const SplitBuf* G2,
                                 float* out, const int* skip) {
  GemmArgs g;
  g.M = s->dims[l] + 1;
  g.N = s->dims[l + 1];
  g.nseg = A2 ? 2 : 1;
  g.seg[0] = GemmSeg{op_trans(s->acts[l]), mk_op(G1.hi, G1.lo, G1.ld, 1, G1.sc), s->bl};
  if (A2) g.seg[1] = GemmSeg{op_trans(*A2), mk_op(G2->hi, G2->lo, G2->ld, 1, G2->sc), s->bl};
  g.epi.mode = EPI_STORE;
  g.epi.out = out + s->off[l];
  g.epi.ld = s->dims[l + 1];
  g.skip = skip;
  return g;
}

// last layer: [gW; gb] = A^T U (+ A2^T U2); returns the stream the result is final on
static cudaStream_t skinny_weight_grad(cv_ctx* ctx, cv_snap* s, const float* U, Scale* usc, const SplitBuf* A2,
                               const float* U2, Scale* u2sc, float* out, const int* skip, bool side = false) {
  const int l = s->L - 1;
  if (s->tc_out) {
    // beside the output-layer backward: the cotangent split and the GEMM both go to the
    // second side stream (the caller joins it) on 128 CTAs (measured best at C3)
    constexpr int side_ctas = 128;
    const bool on_side = side && ctx->engine != CV_ENGINE_SIMT;
    StreamSwap swap(ctx, on_side ? side2_fork(ctx) : ctx->stream);
    const cudaStream_t used = ctx->stream;
    const __half *uh, *ul, *u2h = nullptr, *u2l = nullptr;
    const Scale* uc = cot_split(ctx, s, U, usc, &uh, &ul, skip);
    const Scale* u2c = nullptr;
    if (A2) u2c = cot_split(ctx, s, U2, u2sc, &u2h, &u2l, skip);
    GemmArgs g;
    g.M = s->dims[l] + 1;
    g.N = s->c;
    g.nseg = A2 ? 2 : 1;
    g.seg[0] = GemmSeg{op_trans(s->acts[l]), mk_op(uh, ul, 1, s->ldb, uc), s->bl};
    if (A2) g.seg[1] = GemmSeg{op_trans(*A2), mk_op(u2h, u2l, 1, s->ldb, u2c), s->bl};
    g.epi.mode = EPI_STORE;
    g.epi.out = out + s->off[l];
    g.epi.ld = s->c;
    g.skip = skip;
    if (on_side && gemm_tc_supported(g)) {
      g.stream = ctx->stream;
      g.max_ctas = side_ctas;
    }
    gemm(ctx, g);
    return used;
  }
  SkinnyDwArgs a{};
  a.rows = s->bl;
  a.M = s->dims[l] + 1;
  a.c = s->c;
  a.nseg = A2 ? 2 : 1;
  a.a_hi[0] = s->acts[l].hi; a.a_lo[0] = s->acts[l].lo; a.lda[0] = s->acts[l].ld; a.a_sc[0] = s->acts[l].sc;
  a.U[0] = U;
  if (A2) { a.a_hi[1] = A2->hi; a.a_lo[1] = A2->lo; a.lda[1] = A2->ld; a.a_sc[1] = A2->sc; a.U[1] = U2; }
  a.out = out + s->off[l];
  a.skip = skip;
  skinny_dw(ctx, a, s->skinny_ws, s->skinny_ws_elems);
  return ctx->stream;
}


// Full linearization (models.py:337-396): acts, loss, probs, G, grad.
void mlp_linearize(cv_ctx* ctx, cv_snap* s, double* loss_out, float* grad_out) {
  const int L = s->L;
  int head_groups = 0;
  for (int l = 0; l < L - 1; ++l) {
    SplitBuf& o = s->acts[l + 1];
    const bool wrote = mlp_forward_layer(ctx, s, l, s->acts[l], s->w_hi, s->w_lo, s->w_sc, o, s->bits_buf[l + 1],
                                         &head_groups, s->wl_f32);
    o.bits = wrote ? s->bits_buf[l + 1] : nullptr;
    o.bits_ld = wrote ? ((s->dims[l + 1] + 15) / 16 + 7) / 8 * 8 : 0;
  }
  if (head_groups > 0) {
    // logits = sum of the head partials + the bias row, in fixed order (models.py:357)
    const float* bias = s->wl_f32 + (int64_t)s->dims[L - 1] * s->c;
    launch_k(ctx->stream, k_out_reduce<16>, (s->bl + 31) / 32, 128, 0, (const float*)s->head_part, head_groups, s->bl,
             s->c, 0, s->loss, (const float*)s->probs, 1.f, s->logits, (float*)nullptr, (const int*)nullptr, bias);
    ctx->launches++;
  } else {
    mlp_output_layer(ctx, s, s->acts[L - 1], s->w_hi, s->w_lo, s->w_sc, s->logits);
  }
  mlp_loss(ctx, s, s->logits, 1, loss_out);
  // primal backward: G[l-1] = (G[l] W_l^T) * sp[l-1]   (models.py:378-381), with the
  // weight gradient of layer l co-scheduled beside the backward GEMM of layer l
  const bool tanh_ = s->act == CV_ACT_TANH;
  LayerAllreduce ar(ctx, grad_out, s->off, s->d);
  if (grad_out)
    ar.ready(L - 1, skinny_weight_grad(ctx, s, s->gout, s->gout_sc, nullptr, nullptr, nullptr, grad_out, nullptr));
  if (L >= 2) {
    skinny_backward(ctx, s, s->gout, s->gout_sc, s->w_hi, s->w_lo, s->w_sc, s->G[L - 2],
                    tanh_ ? s->P[L - 2] : nullptr, tanh_ ? s->P_sc[L - 2] : nullptr, nullptr);
    for (int l = L - 2; l >= 1; --l) {
      const GemmArgs dx = hidden_backward_args(s, l, s->G[l], s->w_hi, s->w_lo, s->w_sc, s->G[l - 1],
                                               tanh_ ? s->P[l - 1] : nullptr, tanh_ ? s->P_sc[l - 1] : nullptr,
                                               nullptr);
      if (grad_out) {
        ar.ready(l, gemm_pair(ctx, dx, weight_grad_args(s, l, s->G[l], nullptr, nullptr, grad_out, nullptr)));
      } else {
        gemm(ctx, dx);
      }
    }
    if (grad_out) {
      gemm(ctx, weight_grad_args(s, 0, s->G[0], nullptr, nullptr, grad_out, nullptr));
      ar.ready(0, ctx->stream);
    }
    side_join(ctx);
  }
  if (grad_out) ar.finish();
}

// split of a product input v into v_hi / v_lo (per-layer exponents); also
// zeroes this product's amax slots
static void split_input(cv_ctx* ctx, cv_snap* s, const float* v, const int* skip) {
  if (s->v_ready == 2) {  // the split itself was written by its producer (Rademacher probes)
    s->v_ready = 0;
    return;
  }
  if (s->v_ready) {  // scales already published (and slots zeroed) by the fused CG update
    split_flat_apply(ctx, v, s->d, s->off, s->v_hi, s->v_lo, s->v_sc, skip);
    s->v_ready = 0;
    return;
  }
  split_flat(ctx, v, s->d, s->off, s->v_hi, s->v_lo, s->v_sc, s->prod_sc, s->n_prod, skip);
}

// JVP through the hidden layers: da[l] = act'(a_{l+1}) * (A_l V_l + da[l-1] W_l).
// With v (the fp32 product input) the last hidden GEMM also carries the output
// layer's JVP in its epilogue (Epilogue::head_*): returns the number of partial
// groups it leaves in s->head_part (0: not fused, jvp_out runs the output layer).
// head_only: da[L-2] has no other consumer (GGN / JVP) and is not stored.
static int jvp_hidden(cv_ctx* ctx, cv_snap* s, bool keep_dz, const int* skip, const float* v = nullptr,
                      bool head_only = false) {
  int groups = 0;
  for (int l = 0; l < s->L - 1; ++l) {
    GemmArgs g;
    g.M = s->bl;
    g.N = s->dims[l + 1];
    g.seg[0] = GemmSeg{op_rows(s->acts[l]),
                       op_wblock(s->v_hi + s->off[l], s->v_lo + s->off[l], s->dims[l + 1], s->v_sc + l),
                       s->dims[l] + 1};
    g.nseg = 1;
    bound_add(g.epi.bound, (float)(s->dims[l] + 1), s->acts[l].sc, s->v_sc + l);
    if (l > 0) {
      g.seg[1] = GemmSeg{op_rows(s->da[l - 1]),
                         op_wblock(s->w_hi + s->off[l], s->w_lo + s->off[l], s->dims[l + 1], s->w_sc + l), s->dims[l]};
      g.nseg = 2;
      bound_add(g.epi.bound, (float)s->dims[l], s->da[l - 1].sc, s->w_sc + l);
    }
    g.epi.mode = EPI_SPLIT_MASK;
    g.epi.act = s->act;
    split_epi(g.epi, s->da[l]);
    mask_epi(g.epi, s->acts[l + 1]);
    g.epi.raw = keep_dz ? s->dz[l] : nullptr;
    g.epi.raw_ld = s->da[l].ld;
    g.epi.raw_amax = keep_dz ? &s->dz_sc[l]->amax : nullptr;
    g.skip = skip;
    if (v && s->head_part && l == s->L - 2) {
      g.epi.head_w = s->wl_f32;
      g.epi.head_v = v + s->off[l + 1];
      g.epi.head_c = s->c;
      g.epi.head_part = s->head_part;
      g.epi.head_only = head_only;
      g.unsplit = 1;  // the head needs whole tiles (or a split-K head reduction, below)
      int via_reduce = 0;
      groups = gemm_tc_head_groups(ctx, g, &via_reduce);
      if (via_reduce) g.unsplit = 0;
      if (groups <= 0 || groups > s->head_groups_max) {
        groups = 0;
        g.epi.head_part = nullptr;
        g.epi.head_only = 0;
        g.unsplit = 0;
      }
    }
    gemm(ctx, g);
  }
  return groups;
}

// Output tangent with fused H_z: U = H_z(J v) * scale (post HZ) or raw J v (logits).
static void jvp_out(cv_ctx* ctx, cv_snap* s, int post, float scale, float* out, float* out_amax, const int* skip,
                    int head_groups = 0, const float* v = nullptr) {
  const int l = s->L - 1;
  if (head_groups > 0) {
    // the last hidden GEMM left per-group partials of z = J v: add the bias row
    // [Vb]_{L-1} and reduce in fixed order (+ H_z)
    const float* bias = v + s->off[l] + (int64_t)s->dims[l] * s->c;
    launch_k(ctx->stream, k_out_reduce<16>, (s->bl + 31) / 32, 128, 0, (const float*)s->head_part, head_groups, s->bl,
             s->c, post == POST_HZ ? 1 : 0, s->loss, (const float*)s->probs, scale, out, out_amax, skip, bias);
    ctx->launches++;
    return;
  }
  if (s->tc_out) {
    pad_last(ctx, s, s->v_hi, s->v_lo, s->vl_hi, s->vl_lo, skip);
    GemmArgs g;
    g.M = s->bl;
    g.N = s->c;
    g.nseg = 1;
    g.seg[0] = GemmSeg{op_rows(s->acts[l]), mk_op(s->vl_hi, s->vl_lo, 1, s->ldw, s->v_sc + l), s->dims[l] + 1};
    if (l > 0) {
      g.seg[1] = GemmSeg{op_rows(s->da[l - 1]), mk_op(s->wl_hi, s->wl_lo, 1, s->ldw, s->w_sc + l), s->dims[l]};
      g.nseg = 2;
    }
    g.skip = skip;
    float* part = nullptr;
    const int splits = gemm_tc_partial(ctx, g, &part);
    const bool hz = post == POST_HZ;
    if (s->c <= 16)
      launch_k(ctx->stream, k_out_reduce<16>, (s->bl + 31) / 32, 128, 0, part, splits, s->bl, s->c, hz, s->loss, s->probs,
                                                                    scale, out, out_amax, skip, (const float*)nullptr);
    else
      launch_k(ctx->stream, k_out_reduce<32>, (s->bl + 31) / 32, 128, 0, part, splits, s->bl, s->c, hz, s->loss, s->probs,
                                                                    scale, out, out_amax, skip, (const float*)nullptr);
    ctx->launches++;
    ctx->pool.put(part);
    return;
  }
  SkinnyRowsArgs a{};
  a.rows = s->bl;
  a.c = s->c;
  a.seg[0] = SkinnySeg{s->acts[l].hi, s->acts[l].lo, s->acts[l].ld, s->acts[l].sc, s->v_hi + s->off[l],
                       s->v_lo + s->off[l], s->c, s->v_sc + l, s->dims[l] + 1};
  a.nseg = 1;
  if (l > 0) {
    a.seg[1] = SkinnySeg{s->da[l - 1].hi, s->da[l - 1].lo, s->da[l - 1].ld, s->da[l - 1].sc, s->w_hi + s->off[l],
                         s->w_lo + s->off[l], s->c, s->w_sc + l, s->dims[l]};
    a.nseg = 2;
  }
  a.post = post;
  a.loss = s->loss;
  a.probs = s->probs;
  a.scale = scale;
  a.out = out;
  a.out_amax = out_amax;
  a.skip = skip;
  skinny_rows(ctx, a);
}

// sum_i J_i^T U_i (no 1/b) into out (models.py:274-285); usc->amax = max|U|.
// The per-layer gradient blocks are all-reduced as they become final (LayerAllreduce).
static void vjp_from(cv_ctx* ctx, cv_snap* s, const float* U, Scale* usc, float* out, const int* skip) {
  const int L = s->L;
  LayerAllreduce ar(ctx, out, s->off, s->d);
  ar.ready(L - 1, skinny_weight_grad(ctx, s, U, usc, nullptr, nullptr, nullptr, out, skip, true));
  if (L >= 2) {
    skinny_backward(ctx, s, U, usc, s->w_hi, s->w_lo, s->w_sc, s->gs[L - 2], nullptr, nullptr, skip);
    for (int l = L - 2; l >= 0; --l) {
      const GemmArgs dw = weight_grad_args(s, l, s->gs[l], nullptr, nullptr, out, skip);
      if (l > 0) {
        ar.ready(l, gemm_pair(ctx, hidden_backward_args(s, l, s->gs[l], s->w_hi, s->w_lo, s->w_sc, s->gs[l - 1], nullptr,
                                                        nullptr, skip),
                              dw));
      } else {
        gemm(ctx, dw);
        ar.ready(0, ctx->stream);
      }
    }
  }
  side_join(ctx);
  ar.finish();
}

// GGN product (1/b) J^T H_z J v (curvature.py:109-110).
void mlp_ggn(cv_ctx* ctx, cv_snap* s, const float* v, float* out, const int* skip) {
  split_input(ctx, s, v, skip);
  const int hg = jvp_hidden(ctx, s, false, skip, v, true);
  jvp_out(ctx, s, POST_HZ, 1.0f / (float)s->bg, s->U, &s->U_sc->amax, skip, hg, v);
  vjp_from(ctx, s, s->U, s->U_sc, out, skip);
}

void mlp_jvp(cv_ctx* ctx, cv_snap* s, const float* v, float* out_bc) {
  split_input(ctx, s, v, nullptr);
  const int hg = jvp_hidden(ctx, s, false, nullptr, v, true);
  jvp_out(ctx, s, POST_LOGITS, 1.f, out_bc, nullptr, nullptr, hg, v);
}

void mlp_vjp(cv_ctx* ctx, cv_snap* s, const float* U, float* out) {
  cudaMemsetAsync(s->prod_sc, 0, sizeof(Scale) * s->n_prod, ctx->stream);
  amax_into(ctx, U, (int64_t)s->bl * s->c, s->U_sc);
  vjp_from(ctx, s, U, s->U_sc, out, nullptr);
}

// HVP backward epilogue for the layer below l: (dG W^T + G V^T) * sp [+ tanh P spp dz]
static void hvp_epi(cv_snap* s, Epilogue& e, int l) {
  e.mode = EPI_HVP;
  e.act = s->act;
  split_epi(e, s->gs[l - 1]);
  mask_epi(e, s->acts[l]);
  if (s->act == CV_ACT_TANH) {
    e.P = s->P[l - 1];
    e.P_ld = s->gs[l - 1].ld;
    e.P_amax = &s->P_sc[l - 1]->amax;
    e.dz = s->dz[l - 1];
    e.dz_ld = s->da[l - 1].ld;
    e.dz_amax = &s->dz_sc[l - 1]->amax;
  }
}

// Exact Hessian-vector product (models.py:287-307), forward-over-reverse.
void mlp_hvp(cv_ctx* ctx, cv_snap* s, const float* v, float* out, const int* skip) {
  const int L = s->L;
  const bool tanh_ = s->act == CV_ACT_TANH;
  split_input(ctx, s, v, skip);
  const int hg = jvp_hidden(ctx, s, tanh_, skip, v, false);
  // dG_{L-1} = H_z dz_{L-1} / b
  jvp_out(ctx, s, POST_HZ, 1.0f / (float)s->bg, s->U, &s->U_sc->amax, skip, hg, v);
  // last layer: [gW; gb] = A^T dG + [da|0]^T G_{L-1}
  LayerAllreduce ar(ctx, out, s->off, s->d);
  ar.ready(L - 1, skinny_weight_grad(ctx, s, s->U, s->U_sc, L >= 2 ? &s->da[L - 2] : nullptr, s->gout, s->gout_sc,
                                     out, skip));
  if (L >= 2) {
    // dG_{L-2} = (dG W^T + G_{L-1} V^T) * sp + [tanh] P * spp * dz
    const int l = L - 1;
    {
      SkinnyDxArgs a{};
      a.rows = s->bl;
      a.n = s->dims[l];
      a.c = s->c;
      a.nseg = 2;
      a.U[0] = s->U;
      a.w_hi[0] = s->w_hi + s->off[l];
      a.w_lo[0] = s->w_lo + s->off[l];
      a.w_sc[0] = s->w_sc + l;
      a.U[1] = s->gout;
      a.w_hi[1] = s->v_hi + s->off[l];
      a.w_lo[1] = s->v_lo + s->off[l];
      a.w_sc[1] = s->v_sc + l;
      hvp_epi(s, a.epi, l);
      bound_add(a.epi.bound, (float)s->c, s->U_sc, s->w_sc + l);
      bound_add(a.epi.bound, (float)s->c, s->gout_sc, s->v_sc + l);
      a.skip = skip;
      skinny_dx(ctx, a);
    }
    for (int h = L - 2; h >= 0; --h) {
      const GemmArgs dw = weight_grad_args(s, h, s->gs[h], h > 0 ? &s->da[h - 1] : nullptr, h > 0 ? &s->G[h] : nullptr,
                                           out, skip);
      if (h > 0) {
        GemmArgs g;
        g.M = s->bl;
        g.N = s->dims[h];
        g.nseg = 2;
        g.seg[0] = GemmSeg{op_rows(s->gs[h]),
                           op_wT(s->w_hi + s->off[h], s->w_lo + s->off[h], s->dims[h + 1], s->w_sc + h),
                           s->dims[h + 1]};
        g.seg[1] = GemmSeg{op_rows(s->G[h]),
                           op_wT(s->v_hi + s->off[h], s->v_lo + s->off[h], s->dims[h + 1], s->v_sc + h),
                           s->dims[h + 1]};
        hvp_epi(s, g.epi, h);
        bound_add(g.epi.bound, (float)s->dims[h + 1], s->gs[h].sc, s->w_sc + h);
        bound_add(g.epi.bound, (float)s->dims[h + 1], s->G[h].sc, s->v_sc + h);
        g.skip = skip;
        ar.ready(h, gemm_pair(ctx, g, dw));
      } else {
        gemm(ctx, dw);
        ar.ready(0, ctx->stream);
      }
    }
  }
  side_join(ctx);
  ar.finish();
}

void mlp_loss(cv_ctx* ctx, cv_snap* s, const float* logits, int write_state, double* loss_out) {
  const int nblk = 64;
  launch_k(ctx->stream, k_loss_rows, nblk, 256, 0, logits, s->bl, s->c, s->loss, s->y_i, s->y_f, s->probs, s->gout,
                                             1.0f / (float)s->bg, ctx->red_ws, write_state, &s->gout_sc->amax);
  if (write_state && s->tc_out)
    split_mat(ctx, s->gout, s->c, s->bl, s->c, s->gout_hi, s->gout_lo, s->ldb, 1, s->gout_sc, 1, nullptr);
  const double scale = 1.0 / (double)s->bg;
  launch_k(ctx->stream, k_finalize_sum, 1, 32, 0, ctx->red_ws, nblk, distributed(ctx) ? 1.0 : scale, loss_out);
  ctx->launches += 2;
  if (distributed(ctx)) {
    allreduce_f64(ctx, loss_out, 1);
    scale_scalar(ctx, loss_out, scale);
  }
}

// Loss at another parameter point on the snapshot batch (curvature.py:82-84).
void mlp_loss_at(cv_ctx* ctx, cv_snap* s, const float* w, double* loss_out) {
  // split w into the product scratch (v_hi / v_lo) and run a forward pass on the
  // backward scratch buffers (gs[]) -- no product is in flight concurrently.  The
  // logits take the same path as the linearization's (fused head or output GEMM), so
  // loss_before and loss_after share their rounding and rho's difference stays exact.
  split_input(ctx, s, w, nullptr);
  const int L = s->L;
  const SplitBuf* in = &s->acts[0];
  int head_groups = 0;
  const float* wl = w + s->off[L - 1];
  for (int l = 0; l < L - 1; ++l) {
    mlp_forward_layer(ctx, s, l, *in, s->v_hi, s->v_lo, s->v_sc, s->gs[l], nullptr, &head_groups, wl);
    in = &s->gs[l];
  }
  if (head_groups > 0) {
    const float* bias = wl + (int64_t)s->dims[L - 1] * s->c;
    launch_k(ctx->stream, k_out_reduce<16>, (s->bl + 31) / 32, 128, 0, (const float*)s->head_part, head_groups, s->bl,
             s->c, 0, s->loss, (const float*)s->probs, 1.f, s->U, (float*)nullptr, (const int*)nullptr, bias);
    ctx->launches++;
  } else {
    mlp_output_layer(ctx, s, *in, s->v_hi, s->v_lo, s->v_sc, s->U);
  }
  mlp_loss(ctx, s, s->U, 0, loss_out);
}

}  // namespace cv
