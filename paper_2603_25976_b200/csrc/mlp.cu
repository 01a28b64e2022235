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
#include "common.cuh"
#include "internal.h"
#include "epilogue.cuh"
#include "skinny.cuh"

namespace cv {

int64_t ld_for(int n) { return ((int64_t)n + 1 + 3) / 4 * 4; }

// ---------------------------------------------------------------------------
// elementwise helpers
// ---------------------------------------------------------------------------
__global__ void k_split_vec(const float* __restrict__ x, float* __restrict__ hi, float* __restrict__ lo,
                            int64_t n, const int* skip) {
  if (skip_if(skip)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float h, l;
    split2(x[i], h, l);
    hi[i] = h;
    lo[i] = l;
  }
}

// dst[r, 0:cols] = split(src[r, 0:cols]); dst[r, cols] = (1, 0) when ones.
__global__ void k_split_rows(const float* __restrict__ src, int64_t lds, int rows, int cols,
                             float* __restrict__ hi, float* __restrict__ lo, int64_t ldd, int ones) {
  const int64_t total = (int64_t)rows * (cols + 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (cols + 1);
    const int c = (int)(i - r * (cols + 1));
    if (c == cols) {
      if (ones) { hi[r * ldd + c] = 1.f; lo[r * ldd + c] = 0.f; }
      continue;
    }
    float h, l;
    split2(src[r * lds + c], h, l);
    hi[r * ldd + c] = h;
    lo[r * ldd + c] = l;
  }
}

__global__ void k_set_col(float* hi, float* lo, int64_t ld, int rows, int col, float v) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    hi[(int64_t)r * ld + col] = v;
    lo[(int64_t)r * ld + col] = 0.f;
  }
}

static int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

void split_vec(cv_ctx* ctx, const float* x, float* hi, float* lo, int64_t n, const int* skip) {
  k_split_vec<<<grid_for(n), 256, 0, ctx->stream>>>(x, hi, lo, n, skip);
  ctx->launches++;
}

// ---------------------------------------------------------------------------
// Loss rows: softmax-CE / MSE value, probabilities and G[L-1] = out_grad / b
// (models.py:358-383).  Per-block fp64 partial sums of the per-example loss.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_loss_rows(const float* __restrict__ logits, int rows, int c, int loss,
                                                   const int64_t* __restrict__ yi, const float* __restrict__ yf,
                                                   float* probs, float* gout, float inv_b, double* partial,
                                                   int write_state) {
  double part[1] = {0.0};
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
          gout[(int64_t)m * c + j] = (float)((p - (j == y ? 1.0 : 0.0)) * inv_b);
        }
      }
    } else {
      double s = 0.0;
      for (int j = 0; j < c; ++j) {
        const double r = (double)z[j] - (double)yf[(int64_t)m * c + j];
        s += r * r;
        if (write_state) gout[(int64_t)m * c + j] = (float)(r * inv_b);
      }
      part[0] += 0.5 * s;
    }
  }
  block_sum<1>(part);
  if (threadIdx.x == 0) partial[blockIdx.x] = part[0];
}

// Sum nblk partials in fixed order, scale, store to *out (device double).
__global__ void k_finalize_sum(const double* partial, int nblk, double scale, double* out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nblk; ++i) s += partial[i];
    *out = s * scale;
  }
}

// ---------------------------------------------------------------------------
// Tensor-core output layer helpers (tc_out): padded split copies of the c-wide
// operands and the row-wise post-processing of the JVP partials.
// ---------------------------------------------------------------------------
// rows x c (ld ld_src) -> rows x cp split, zero padded; from (hi, lo) or from plain fp32
__global__ void k_pad_split(const float* hi, const float* lo, const float* plain, int64_t ld_src, int rows, int c,
                            int cp, float* ohi, float* olo, const int* skip) {
  if (skip_if(skip)) return;
  const int64_t total = (int64_t)rows * cp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cp;
    const int j = (int)(i - r * cp);
    float h = 0.f, l = 0.f;
    if (j < c) {
      if (plain) split2(plain[r * ld_src + j], h, l);
      else { h = hi[r * ld_src + j]; l = lo[r * ld_src + j]; }
    }
    ohi[i] = h;
    olo[i] = l;
  }
}

// out-layer JVP: sum the split-K partials of z = J v per row, then either store
// the logits tangent (POST_LOGITS) or U = H_z(z) * scale (models.py:199-204)
template <int CM>
__global__ void k_out_reduce(const float* part, int splits, int rows, int c, int post, int loss, const float* probs,
                             float scale, float* out_plain, float* ohi, float* olo, int cp, const int* skip) {
  if (skip_if(skip)) return;
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= rows) return;
  float t[CM];
#pragma unroll
  for (int j = 0; j < CM; ++j) t[j] = 0.f;
  for (int z = 0; z < splits; ++z) {
    const float* p = part + ((int64_t)z * rows + m) * c;
#pragma unroll
    for (int j = 0; j < CM; ++j)
      if (j < c) t[j] += p[j];
  }
  if (post == 1) {
    if (loss == CV_LOSS_CE) {
      const float* p = probs + (int64_t)m * c;
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
  if (out_plain)
#pragma unroll
    for (int j = 0; j < CM; ++j)
      if (j < c) out_plain[(int64_t)m * c + j] = t[j];
  if (ohi)
#pragma unroll
    for (int j = 0; j < CM; ++j)
      if (j < cp) {
        float h = 0.f, l = 0.f;
        if (j < c) split2(t[j], h, l);
        ohi[(int64_t)m * cp + j] = h;
        olo[(int64_t)m * cp + j] = l;
      }
}

// ---------------------------------------------------------------------------
// Host orchestration
// ---------------------------------------------------------------------------
static void launch_skinny_rows(cv_ctx* ctx, const SkinnyRowsArgs& a) { skinny_rows(ctx, a); }
static void launch_skinny_dx(cv_ctx* ctx, const SkinnyDxArgs& a) { skinny_dx(ctx, a); }
static void launch_skinny_dw(cv_ctx* ctx, cv_snap* s, SkinnyDwArgs a) { skinny_dw(ctx, a, s->skinny_ws, s->skinny_ws_elems); }

// Operand views --------------------------------------------------------------
static Operand op_rows(const SplitBuf& b) { return Operand{b.hi, b.lo, b.ld, 1}; }          // X(m,k)=buf[m,k]
static Operand op_trans(const SplitBuf& b) { return Operand{b.hi, b.lo, 1, b.ld}; }         // X(m,k)=buf[k,m]
static Operand op_wblock(const float* hi, const float* lo, int nout) { return Operand{hi, lo, nout, 1}; }
static Operand op_wT(const float* hi, const float* lo, int nout) { return Operand{hi, lo, 1, nout}; }

// last-layer block of a split flat vector -> padded split copy (tc_out)
static void pad_last(cv_ctx* ctx, cv_snap* s, const float* hi, const float* lo, float* ohi, float* olo,
                     const int* skip) {
  const int l = s->L - 1;
  const int rows = s->dims[l] + 1;
  k_pad_split<<<grid_for((int64_t)rows * s->cp), 256, 0, ctx->stream>>>(hi + s->off[l], lo + s->off[l], nullptr, s->c,
                                                                         rows, s->c, s->cp, ohi, olo, skip);
  ctx->launches++;
}

void pad_last_weights(cv_ctx* ctx, cv_snap* s) { pad_last(ctx, s, s->w_hi, s->w_lo, s->wl_hi, s->wl_lo, nullptr); }

// the split (ld cp) form of a b x c cotangent: U / G[L-1] map to their resident
// splits, any other (plain, ld c) matrix is split into U_hi / U_lo
static void cot_split(cv_ctx* ctx, cv_snap* s, const float* U, const float** hi, const float** lo, const int* skip) {
  if (U == s->gout) { *hi = s->gout_hi; *lo = s->gout_lo; return; }
  if (U != s->U) {
    k_pad_split<<<grid_for((int64_t)s->bl * s->cp), 256, 0, ctx->stream>>>(nullptr, nullptr, U, s->c, s->bl, s->c,
                                                                           s->cp, s->U_hi, s->U_lo, skip);
    ctx->launches++;
  }
  *hi = s->U_hi;
  *lo = s->U_lo;
}

void mlp_forward_layer(cv_ctx* ctx, cv_snap* s, int l, const SplitBuf& in, const float* whi, const float* wlo,
                       const SplitBuf& out) {
  GemmArgs g;
  g.M = s->bl;
  g.N = s->dims[l + 1];
  g.nseg = 1;
  g.seg[0] = GemmSeg{op_rows(in), op_wblock(whi + s->off[l], wlo + s->off[l], s->dims[l + 1]), s->dims[l] + 1};
  g.epi.mode = EPI_SPLIT_ACT;
  g.epi.act = s->act;
  g.epi.out_hi = out.hi;
  g.epi.out_lo = out.lo;
  g.epi.ld = out.ld;
  gemm(ctx, g);
}

// logits = A_{L-1} [W; b]  (skinny)
void mlp_output_layer(cv_ctx* ctx, cv_snap* s, const SplitBuf& in, const float* whi, const float* wlo,
                      float* logits) {
  const int l = s->L - 1;
  if (s->tc_out) {
    const float *bh = s->wl_hi, *bl = s->wl_lo;
    if (whi != s->w_hi) {  // another parameter point (loss_at): pad its last block
      pad_last(ctx, s, whi, wlo, s->vl_hi, s->vl_lo, nullptr);
      bh = s->vl_hi;
      bl = s->vl_lo;
    }
    GemmArgs g;
    g.M = s->bl;
    g.N = s->c;
    g.nseg = 1;
    g.seg[0] = GemmSeg{op_rows(in), Operand{bh, bl, s->cp, 1}, s->dims[l] + 1};
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
  a.seg[0] = SkinnySeg{in.hi, in.lo, in.ld, whi + s->off[l], wlo + s->off[l], s->c, s->dims[l] + 1};
  a.post = POST_LOGITS;
  a.loss = s->loss;
  a.out = logits;
  launch_skinny_rows(ctx, a);
}

// Loss value (+ optionally probs / G[L-1]) from logits; *loss_out = global mean.
void mlp_loss(cv_ctx* ctx, cv_snap* s, const float* logits, int write_state, double* loss_out);

// G_prev = (U W_l^T) * act'(a_l) for the output layer (l = L-1), skinny K = c.
static void skinny_backward(cv_ctx* ctx, cv_snap* s, const float* U, const float* whi, const float* wlo,
                            const SplitBuf& out, float* raw, const int* skip) {
  const int l = s->L - 1;
  if (s->tc_out && s->tc_dx) {
    const float *uh, *ul;
    cot_split(ctx, s, U, &uh, &ul, skip);
    GemmArgs g;
    g.M = s->bl;
    g.N = s->dims[l];
    g.nseg = 1;
    g.seg[0] = GemmSeg{Operand{uh, ul, s->cp, 1}, Operand{s->wl_hi, s->wl_lo, 1, s->cp}, s->c};
    g.epi.mode = EPI_SPLIT_MASK;
    g.epi.act = s->act;
    g.epi.out_hi = out.hi;
    g.epi.out_lo = out.lo;
    g.epi.ld = out.ld;
    g.epi.mask_hi = s->acts[l].hi;
    g.epi.mask_lo = s->acts[l].lo;
    g.epi.mask_ld = s->acts[l].ld;
    g.epi.raw = raw;
    g.epi.raw_ld = out.ld;
    g.skip = skip;
    gemm(ctx, g);
    return;
  }
  SkinnyDxArgs a{};
  a.rows = s->bl;
  a.n = s->dims[l];
  a.c = s->c;
  a.nseg = 1;
  a.U[0] = U;
  a.w_hi[0] = whi + s->off[l];
  a.w_lo[0] = wlo + s->off[l];
  a.epi.mode = EPI_SPLIT_MASK;
  a.epi.act = s->act;
  a.epi.out_hi = out.hi;
  a.epi.out_lo = out.lo;
  a.epi.ld = out.ld;
  a.epi.mask_hi = s->acts[l].hi;
  a.epi.mask_lo = s->acts[l].lo;
  a.epi.mask_ld = s->acts[l].ld;
  a.epi.raw = raw;
  a.epi.raw_ld = out.ld;
  a.skip = skip;
  launch_skinny_dx(ctx, a);
}

// G_prev = (G_l W_l^T) * act'(a_l), hidden layer l >= 1
static void hidden_backward(cv_ctx* ctx, cv_snap* s, int l, const SplitBuf& Gl, const float* whi,
                            const float* wlo, const SplitBuf& out, float* raw, const int* skip) {
  GemmArgs g;
  g.M = s->bl;
  g.N = s->dims[l];
  g.nseg = 1;
  g.seg[0] = GemmSeg{op_rows(Gl), op_wT(whi + s->off[l], wlo + s->off[l], s->dims[l + 1]), s->dims[l + 1]};
  g.epi.mode = EPI_SPLIT_MASK;
  g.epi.act = s->act;
  g.epi.out_hi = out.hi;
  g.epi.out_lo = out.lo;
  g.epi.ld = out.ld;
  g.epi.mask_hi = s->acts[l].hi;
  g.epi.mask_lo = s->acts[l].lo;
  g.epi.mask_ld = s->acts[l].ld;
  g.epi.raw = raw;
  g.epi.raw_ld = out.ld;
  g.skip = skip;
  gemm(ctx, g);
}

// [gW; gb]_l = A_l^T G (+ A2^T G2), written into out + off[l] (hidden layers).
static void weight_grad(cv_ctx* ctx, cv_snap* s, int l, const SplitBuf& G1, const SplitBuf* A2,
                        const SplitBuf* G2, float* out, const int* skip) {
  GemmArgs g;
  g.M = s->dims[l] + 1;
  g.N = s->dims[l + 1];
  g.nseg = A2 ? 2 : 1;
  g.seg[0] = GemmSeg{op_trans(s->acts[l]), Operand{G1.hi, G1.lo, G1.ld, 1}, s->bl};
  if (A2) g.seg[1] = GemmSeg{op_trans(*A2), Operand{G2->hi, G2->lo, G2->ld, 1}, s->bl};
  g.epi.mode = EPI_STORE;
  g.epi.out = out + s->off[l];
  g.epi.ld = s->dims[l + 1];
  g.skip = skip;
  gemm(ctx, g);
}

static void skinny_weight_grad(cv_ctx* ctx, cv_snap* s, const float* U, const SplitBuf* A2, const float* U2,
                               float* out, const int* skip) {
  const int l = s->L - 1;
  if (s->tc_out) {
    const float *uh, *ul, *u2h = nullptr, *u2l = nullptr;
    cot_split(ctx, s, U, &uh, &ul, skip);
    if (A2) cot_split(ctx, s, U2, &u2h, &u2l, skip);
    GemmArgs g;
    g.M = s->dims[l] + 1;
    g.N = s->c;
    g.nseg = A2 ? 2 : 1;
    g.seg[0] = GemmSeg{op_trans(s->acts[l]), Operand{uh, ul, s->cp, 1}, s->bl};
    if (A2) g.seg[1] = GemmSeg{op_trans(*A2), Operand{u2h, u2l, s->cp, 1}, s->bl};
    g.epi.mode = EPI_STORE;
    g.epi.out = out + s->off[l];
    g.epi.ld = s->c;
    g.skip = skip;
    gemm(ctx, g);
    return;
  }
  SkinnyDwArgs a{};
  a.rows = s->bl;
  a.M = s->dims[l] + 1;
  a.c = s->c;
  a.nseg = A2 ? 2 : 1;
  a.a_hi[0] = s->acts[l].hi; a.a_lo[0] = s->acts[l].lo; a.lda[0] = s->acts[l].ld; a.U[0] = U;
  if (A2) { a.a_hi[1] = A2->hi; a.a_lo[1] = A2->lo; a.lda[1] = A2->ld; a.U[1] = U2; }
  a.out = out + s->off[l];
  a.skip = skip;
  launch_skinny_dw(ctx, s, a);
}


// Full linearization (models.py:337-396): acts, loss, probs, G, grad.
void mlp_linearize(cv_ctx* ctx, cv_snap* s, double* loss_out, float* grad_out) {
  const int L = s->L;
  for (int l = 0; l < L - 1; ++l) mlp_forward_layer(ctx, s, l, s->acts[l], s->w_hi, s->w_lo, s->acts[l + 1]);
  mlp_output_layer(ctx, s, s->acts[L - 1], s->w_hi, s->w_lo, s->logits);
  mlp_loss(ctx, s, s->logits, 1, loss_out);
  // primal backward: G[l-1] = (G[l] W_l^T) * sp[l-1]   (models.py:378-381)
  if (L >= 2) {
    skinny_backward(ctx, s, s->gout, s->w_hi, s->w_lo, s->G[L - 2], s->act == CV_ACT_TANH ? s->P[L - 2] : nullptr,
                    nullptr);
    for (int l = L - 2; l >= 1; --l)
      hidden_backward(ctx, s, l, s->G[l], s->w_hi, s->w_lo, s->G[l - 1],
                      s->act == CV_ACT_TANH ? s->P[l - 1] : nullptr, nullptr);
  }
  if (grad_out) {
    skinny_weight_grad(ctx, s, s->gout, nullptr, nullptr, grad_out, nullptr);
    for (int l = L - 2; l >= 0; --l) weight_grad(ctx, s, l, s->G[l], nullptr, nullptr, grad_out, nullptr);
    if (ctx->nccl) allreduce_f32(ctx, grad_out, s->d);
  }
}

// JVP through the hidden layers: da[l] = act'(a_{l+1}) * (A_l V_l + da[l-1] W_l).
static void jvp_hidden(cv_ctx* ctx, cv_snap* s, const float* vhi, const float* vlo, bool keep_dz,
                       const int* skip) {
  for (int l = 0; l < s->L - 1; ++l) {
    GemmArgs g;
    g.M = s->bl;
    g.N = s->dims[l + 1];
    g.seg[0] = GemmSeg{op_rows(s->acts[l]), op_wblock(vhi + s->off[l], vlo + s->off[l], s->dims[l + 1]),
                       s->dims[l] + 1};
    g.nseg = 1;
    if (l > 0) {
      g.seg[1] = GemmSeg{op_rows(s->da[l - 1]), op_wblock(s->w_hi + s->off[l], s->w_lo + s->off[l], s->dims[l + 1]),
                         s->dims[l]};
      g.nseg = 2;
    }
    g.epi.mode = EPI_SPLIT_MASK;
    g.epi.act = s->act;
    g.epi.out_hi = s->da[l].hi;
    g.epi.out_lo = s->da[l].lo;
    g.epi.ld = s->da[l].ld;
    g.epi.mask_hi = s->acts[l + 1].hi;
    g.epi.mask_lo = s->acts[l + 1].lo;
    g.epi.mask_ld = s->acts[l + 1].ld;
    g.epi.raw = keep_dz ? s->dz[l] : nullptr;
    g.epi.raw_ld = s->da[l].ld;
    g.skip = skip;
    gemm(ctx, g);
  }
}

// Output tangent with fused H_z: U = H_z(J v) * scale (post HZ) or raw J v (logits).
static void jvp_out(cv_ctx* ctx, cv_snap* s, const float* vhi, const float* vlo, int post, float scale,
                    float* out, const int* skip) {
  const int l = s->L - 1;
  if (s->tc_out) {
    pad_last(ctx, s, vhi, vlo, s->vl_hi, s->vl_lo, skip);
    GemmArgs g;
    g.M = s->bl;
    g.N = s->c;
    g.nseg = 1;
    g.seg[0] = GemmSeg{op_rows(s->acts[l]), Operand{s->vl_hi, s->vl_lo, s->cp, 1}, s->dims[l] + 1};
    if (l > 0) {
      g.seg[1] = GemmSeg{op_rows(s->da[l - 1]), Operand{s->wl_hi, s->wl_lo, s->cp, 1}, s->dims[l]};
      g.nseg = 2;
    }
    g.skip = skip;
    float* part = nullptr;
    const int splits = gemm_tc_partial(ctx, g, &part);
    const bool hz = post == POST_HZ;
    if (s->c <= 16)
      k_out_reduce<16><<<(s->bl + 127) / 128, 128, 0, ctx->stream>>>(part, splits, s->bl, s->c, hz, s->loss, s->probs,
                                                                    scale, out, hz ? s->U_hi : nullptr,
                                                                    hz ? s->U_lo : nullptr, s->cp, skip);
    else
      k_out_reduce<32><<<(s->bl + 127) / 128, 128, 0, ctx->stream>>>(part, splits, s->bl, s->c, hz, s->loss, s->probs,
                                                                    scale, out, hz ? s->U_hi : nullptr,
                                                                    hz ? s->U_lo : nullptr, s->cp, skip);
    ctx->launches++;
    ctx->pool.put(part);
    return;
  }
  SkinnyRowsArgs a{};
  a.rows = s->bl;
  a.c = s->c;
  a.seg[0] = SkinnySeg{s->acts[l].hi, s->acts[l].lo, s->acts[l].ld, vhi + s->off[l], vlo + s->off[l], s->c,
                       s->dims[l] + 1};
  a.nseg = 1;
  if (l > 0) {
    a.seg[1] = SkinnySeg{s->da[l - 1].hi, s->da[l - 1].lo, s->da[l - 1].ld, s->w_hi + s->off[l], s->w_lo + s->off[l],
                         s->c, s->dims[l]};
    a.nseg = 2;
  }
  a.post = post;
  a.loss = s->loss;
  a.probs = s->probs;
  a.scale = scale;
  a.out = out;
  a.skip = skip;
  launch_skinny_rows(ctx, a);
}

// sum_i J_i^T U_i (no 1/b) into out (models.py:274-285).
static void vjp_from(cv_ctx* ctx, cv_snap* s, const float* U, float* out, const int* skip) {
  const int L = s->L;
  skinny_weight_grad(ctx, s, U, nullptr, nullptr, out, skip);
  if (L >= 2) {
    int cur = 0;
    skinny_backward(ctx, s, U, s->w_hi, s->w_lo, s->gs[L - 2], nullptr, skip);
    (void)cur;
    for (int l = L - 2; l >= 0; --l) {
      weight_grad(ctx, s, l, s->gs[l], nullptr, nullptr, out, skip);
      if (l > 0) hidden_backward(ctx, s, l, s->gs[l], s->w_hi, s->w_lo, s->gs[l - 1], nullptr, skip);
    }
  }
}

// GGN product (1/b) J^T H_z J v (curvature.py:109-110); v given split.
void mlp_ggn(cv_ctx* ctx, cv_snap* s, const float* vhi, const float* vlo, float* out, const int* skip) {
  jvp_hidden(ctx, s, vhi, vlo, false, skip);
  jvp_out(ctx, s, vhi, vlo, POST_HZ, 1.0f / (float)s->bg, s->U, skip);
  vjp_from(ctx, s, s->U, out, skip);
  if (ctx->nccl) allreduce_f32(ctx, out, s->d);
}

void mlp_jvp(cv_ctx* ctx, cv_snap* s, const float* vhi, const float* vlo, float* out_bc) {
  jvp_hidden(ctx, s, vhi, vlo, false, nullptr);
  jvp_out(ctx, s, vhi, vlo, POST_LOGITS, 1.f, out_bc, nullptr);
}

void mlp_vjp(cv_ctx* ctx, cv_snap* s, const float* U, float* out) {
  vjp_from(ctx, s, U, out, nullptr);
  if (ctx->nccl) allreduce_f32(ctx, out, s->d);
}

// Exact Hessian-vector product (models.py:287-307), forward-over-reverse.
void mlp_hvp(cv_ctx* ctx, cv_snap* s, const float* vhi, const float* vlo, float* out, const int* skip) {
  const int L = s->L;
  const bool tanh_ = s->act == CV_ACT_TANH;
  jvp_hidden(ctx, s, vhi, vlo, tanh_, skip);
  // dG_{L-1} = H_z dz_{L-1} / b
  jvp_out(ctx, s, vhi, vlo, POST_HZ, 1.0f / (float)s->bg, s->U, skip);
  // last layer: [gW; gb] = A^T dG + [da|0]^T G_{L-1}
  skinny_weight_grad(ctx, s, s->U, L >= 2 ? &s->da[L - 2] : nullptr, s->gout, out, skip);
  if (L >= 2) {
    // dG_{L-2} = (dG W^T + G_{L-1} V^T) * sp + [tanh] P * spp * dz
    const int l = L - 1;
    if (s->tc_out && s->tc_dx) {
      // vl holds this product's padded last block (written by jvp_out)
      GemmArgs g;
      g.M = s->bl;
      g.N = s->dims[l];
      g.nseg = 2;
      g.seg[0] = GemmSeg{Operand{s->U_hi, s->U_lo, s->cp, 1}, Operand{s->wl_hi, s->wl_lo, 1, s->cp}, s->c};
      g.seg[1] = GemmSeg{Operand{s->gout_hi, s->gout_lo, s->cp, 1}, Operand{s->vl_hi, s->vl_lo, 1, s->cp}, s->c};
      g.epi.mode = EPI_HVP;
      g.epi.act = s->act;
      g.epi.out_hi = s->gs[l - 1].hi;
      g.epi.out_lo = s->gs[l - 1].lo;
      g.epi.ld = s->gs[l - 1].ld;
      g.epi.mask_hi = s->acts[l].hi;
      g.epi.mask_lo = s->acts[l].lo;
      g.epi.mask_ld = s->acts[l].ld;
      if (tanh_) {
        g.epi.P = s->P[l - 1];
        g.epi.P_ld = s->gs[l - 1].ld;
        g.epi.dz = s->dz[l - 1];
        g.epi.dz_ld = s->da[l - 1].ld;
      }
      g.skip = skip;
      gemm(ctx, g);
    }
    SkinnyDxArgs a{};
    a.rows = s->bl;
    a.n = s->dims[l];
    a.c = s->c;
    a.nseg = 2;
    a.U[0] = s->U;
    a.w_hi[0] = s->w_hi + s->off[l];
    a.w_lo[0] = s->w_lo + s->off[l];
    a.U[1] = s->gout;
    a.w_hi[1] = vhi + s->off[l];
    a.w_lo[1] = vlo + s->off[l];
    a.epi.mode = EPI_HVP;
    a.epi.act = s->act;
    a.epi.out_hi = s->gs[l - 1].hi;
    a.epi.out_lo = s->gs[l - 1].lo;
    a.epi.ld = s->gs[l - 1].ld;
    a.epi.mask_hi = s->acts[l].hi;
    a.epi.mask_lo = s->acts[l].lo;
    a.epi.mask_ld = s->acts[l].ld;
    if (tanh_) {
      a.epi.P = s->P[l - 1];
      a.epi.P_ld = s->gs[l - 1].ld;
      a.epi.dz = s->dz[l - 1];
      a.epi.dz_ld = s->da[l - 1].ld;
    }
    a.skip = skip;
    if (!(s->tc_out && s->tc_dx)) launch_skinny_dx(ctx, a);
    for (int h = L - 2; h >= 0; --h) {
      weight_grad(ctx, s, h, s->gs[h], h > 0 ? &s->da[h - 1] : nullptr, h > 0 ? &s->G[h] : nullptr, out, skip);
      if (h > 0) {
        GemmArgs g;
        g.M = s->bl;
        g.N = s->dims[h];
        g.nseg = 2;
        g.seg[0] = GemmSeg{op_rows(s->gs[h]), op_wT(s->w_hi + s->off[h], s->w_lo + s->off[h], s->dims[h + 1]),
                           s->dims[h + 1]};
        g.seg[1] = GemmSeg{op_rows(s->G[h]), op_wT(vhi + s->off[h], vlo + s->off[h], s->dims[h + 1]),
                           s->dims[h + 1]};
        g.epi.mode = EPI_HVP;
        g.epi.act = s->act;
        g.epi.out_hi = s->gs[h - 1].hi;
        g.epi.out_lo = s->gs[h - 1].lo;
        g.epi.ld = s->gs[h - 1].ld;
        g.epi.mask_hi = s->acts[h].hi;
        g.epi.mask_lo = s->acts[h].lo;
        g.epi.mask_ld = s->acts[h].ld;
        if (tanh_) {
          g.epi.P = s->P[h - 1];
          g.epi.P_ld = s->gs[h - 1].ld;
          g.epi.dz = s->dz[h - 1];
          g.epi.dz_ld = s->da[h - 1].ld;
        }
        g.skip = skip;
        gemm(ctx, g);
      }
    }
  }
  if (ctx->nccl) allreduce_f32(ctx, out, s->d);
}

void mlp_loss(cv_ctx* ctx, cv_snap* s, const float* logits, int write_state, double* loss_out) {
  const int nblk = 64;
  k_loss_rows<<<nblk, 256, 0, ctx->stream>>>(logits, s->bl, s->c, s->loss, s->y_i, s->y_f, s->probs, s->gout,
                                             1.0f / (float)s->bg, ctx->red_ws, write_state);
  if (write_state && s->tc_out) {
    k_pad_split<<<grid_for((int64_t)s->bl * s->cp), 256, 0, ctx->stream>>>(nullptr, nullptr, s->gout, s->c, s->bl,
                                                                           s->c, s->cp, s->gout_hi, s->gout_lo,
                                                                           nullptr);
    ctx->launches++;
  }
  const double scale = 1.0 / (double)s->bg;
  k_finalize_sum<<<1, 32, 0, ctx->stream>>>(ctx->red_ws, nblk, ctx->nccl ? 1.0 : scale, loss_out);
  ctx->launches += 2;
  if (ctx->nccl) {
    allreduce_f64(ctx, loss_out, 1);
    scale_scalar(ctx, loss_out, scale);
  }
}

// Loss at another parameter point on the snapshot batch (curvature.py:82-84).
void mlp_loss_at(cv_ctx* ctx, cv_snap* s, const float* w, double* loss_out) {
  // split w into the product scratch (v_hi / v_lo) and run a forward pass on the
  // tangent scratch buffers (da[]) -- no product is in flight concurrently.
  split_vec(ctx, w, s->v_hi, s->v_lo, s->d, nullptr);
  const int L = s->L;
  const SplitBuf* in = &s->acts[0];
  for (int l = 0; l < L - 1; ++l) {
    mlp_forward_layer(ctx, s, l, *in, s->v_hi, s->v_lo, s->gs[l]);
    // gs[l] needs the ones column for the next layer's bias
    k_set_col<<<grid_for(s->bl), 256, 0, ctx->stream>>>(s->gs[l].hi, s->gs[l].lo, s->gs[l].ld, s->bl,
                                                          s->dims[l + 1], 1.f);
    ctx->launches++;
    in = &s->gs[l];
  }
  mlp_output_layer(ctx, s, *in, s->v_hi, s->v_lo, s->U);
  mlp_loss(ctx, s, s->U, 0, loss_out);
}

void set_col_value(cv_ctx* ctx, const SplitBuf& b, int rows, int col, float v) {
  k_set_col<<<grid_for(rows), 256, 0, ctx->stream>>>(b.hi, b.lo, b.ld, rows, col, v);
  ctx->launches++;
}

void set_ones_col(cv_ctx* ctx, const SplitBuf& b, int rows, int col) { set_col_value(ctx, b, rows, col, 1.f); }

__global__ void k_gather_rows(const float* hi, const float* lo, int64_t ld, int rows, int cols, float* out) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    out[i] = hi[r * ld + c] + lo[r * ld + c];
  }
}

void gather_rows(cv_ctx* ctx, const SplitBuf& b, int rows, int cols, float* out) {
  k_gather_rows<<<grid_for((int64_t)rows * cols), 256, 0, ctx->stream>>>(b.hi, b.lo, b.ld, rows, cols, out);
  ctx->launches++;
}

void split_rows(cv_ctx* ctx, const float* src, int64_t lds, int rows, int cols, const SplitBuf& dst, int ones) {
  k_split_rows<<<grid_for((int64_t)rows * (cols + 1)), 256, 0, ctx->stream>>>(src, lds, rows, cols, dst.hi, dst.lo,
                                                                               dst.ld, ones);
  ctx->launches++;
}

}  // namespace cv
