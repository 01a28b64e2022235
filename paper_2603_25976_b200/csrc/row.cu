// Row-space lane: per-example H_z roots, Gram of the seeded Jacobian rows,
// blocked Cholesky of (Gram + mu I), triangular solves and backprojection.
//   seeds / rhs        curvature.py:112-119, models.py:206-239
//   Gram               models.py:309-334 (layer-wise, the m x d row matrix never exists)
//   Cholesky + solve   solvers.py:146-161 (LAPACK potrf/potrs in the reference)
//   backprojection     curvature.py:53-60
#include "common.cuh"
#include "internal.h"

#include <stdexcept>
#include <type_traits>
#include <vector>

namespace cv {

constexpr int CH_NB = 64;  // Cholesky block size

// ---------------------------------------------------------------------------
// Per-example symmetric eigen-decomposition of H_z = diag(p) - p p^T (c x c) by
// cyclic Jacobi in fp64, one thread per example; then the root and pseudo-inverse
// root with the reference's floor (1e-10 * max(lambda_max, 0)).  MSE: identity.
// ---------------------------------------------------------------------------
template <int CM>
__global__ void k_hz_roots(const float* logits, const int64_t* yi, const float* yf, int b, int c, int loss,
                           float* seeds, float* pinv, float* rhs) {
  CV_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b) return;
  const size_t cc = (size_t)c * c;
  if (loss == CV_LOSS_MSE) {
    for (int a = 0; a < c; ++a) {
      for (int j = 0; j < c; ++j) {
        seeds[i * cc + a * c + j] = a == j ? 1.f : 0.f;
        pinv[i * cc + a * c + j] = a == j ? 1.f : 0.f;
      }
      rhs[(size_t)i * c + a] = (float)((double)logits[(size_t)i * c + a] - (double)yf[(size_t)i * c + a]);
    }
    return;
  }
  // softmax in fp64 from the logits (models.py:371-377)
  double H[CM][CM], Q[CM][CM], p[CM];
  bool finite = true;
  double mx = logits[(size_t)i * c];
  for (int a = 1; a < c; ++a) mx = fmax(mx, (double)logits[(size_t)i * c + a]);
  double se = 0.0;
  for (int a = 0; a < c; ++a) {
    p[a] = exp((double)logits[(size_t)i * c + a] - mx);
    se += p[a];
  }
  for (int a = 0; a < c; ++a) {
    p[a] /= se;
    finite = finite && isfinite(p[a]);
  }
  if (!finite) {
    for (size_t e = 0; e < cc; ++e) { seeds[i * cc + e] = NAN; pinv[i * cc + e] = NAN; }
    for (int a = 0; a < c; ++a) rhs[(size_t)i * c + a] = NAN;
    return;
  }
  for (int a = 0; a < c; ++a)
    for (int j = 0; j < c; ++j) {
      H[a][j] = (a == j ? p[a] : 0.0) - p[a] * p[j];
      Q[a][j] = a == j ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int a = 0; a < c; ++a)
      for (int j = 0; j < c; ++j) {
        tot += H[a][j] * H[a][j];
        if (a != j) off += H[a][j] * H[a][j];
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int pp = 0; pp < c - 1; ++pp)
      for (int q = pp + 1; q < c; ++q) {
        const double apq = H[pp][q];
        if (fabs(apq) < 1e-300) continue;
        const double theta = (H[q][q] - H[pp][pp]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < c; ++k) {  // H <- J^T H J
          const double hkp = H[k][pp], hkq = H[k][q];
          H[k][pp] = cs * hkp - sn * hkq;
          H[k][q] = sn * hkp + cs * hkq;
        }
        for (int k = 0; k < c; ++k) {
          const double hpk = H[pp][k], hqk = H[q][k];
          H[pp][k] = cs * hpk - sn * hqk;
          H[q][k] = sn * hpk + cs * hqk;
        }
        for (int k = 0; k < c; ++k) {  // Q <- Q J
          const double qkp = Q[k][pp], qkq = Q[k][q];
          Q[k][pp] = cs * qkp - sn * qkq;
          Q[k][q] = sn * qkp + cs * qkq;
        }
      }
  }
  double lmax = -1e300;
  for (int a = 0; a < c; ++a) lmax = fmax(lmax, H[a][a]);
  const double floor_ = 1e-10 * fmax(lmax, 0.0);
  double r[CM], ri[CM];
  for (int a = 0; a < c; ++a) {
    const bool keep = H[a][a] > floor_;
    r[a] = keep ? sqrt(fmax(H[a][a], 0.0)) : 0.0;
    ri[a] = keep ? 1.0 / r[a] : 0.0;
  }
  double og[CM];
  for (int a = 0; a < c; ++a) og[a] = p[a] - (a == yi[i] ? 1.0 : 0.0);
  for (int a = 0; a < c; ++a) {
    double acc_rhs = 0.0;
    for (int j = 0; j < c; ++j) {
      double s = 0.0, si = 0.0;
      for (int k = 0; k < c; ++k) {
        s += Q[a][k] * r[k] * Q[j][k];
        si += Q[a][k] * ri[k] * Q[j][k];
      }
      seeds[i * cc + a * c + j] = (float)s;
      pinv[i * cc + a * c + j] = (float)si;
      acc_rhs += si * og[j];
    }
    rhs[(size_t)i * c + a] = (float)acc_rhs;
  }
}

// cot[i, a] = sum_j seeds[i, a, j] u[i, j]  (curvature.py:58-59)
__global__ void k_seed_apply(const float* seeds, const float* u, int b, int c, float* out) {
  CV_PDL_ENTRY();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)b * c) return;
  const int64_t i = e / c;
  const int a = (int)(e - i * c);
  float s = 0.f;
  for (int j = 0; j < c; ++j) s = fmaf(seeds[(i * c + a) * c + j], u[i * c + j], s);
  out[e] = s;
}

static float* snap_alloc(cv_snap* s, int64_t n) {
  float* p = (float*)s->ctx->pool.get(sizeof(float) * (size_t)n);
  s->owned.push_back(p);
  return p;
}

static void ensure_seeds(cv_ctx* ctx, cv_snap* s) {
  if (s->row_state & 1) return;
  const int b = s->bl, c = s->c;
  s->seeds = snap_alloc(s, (int64_t)b * c * c);
  s->pinv = snap_alloc(s, (int64_t)b * c * c);
  s->rhs = snap_alloc(s, (int64_t)b * c);
  if (c <= 16)
    launch_k(ctx->stream, k_hz_roots<16>, (b + 63) / 64, 64, 0, s->logits, s->y_i, s->y_f, b, c, s->loss, s->seeds,
                                                          s->pinv, s->rhs);
  else
    launch_k(ctx->stream, k_hz_roots<32>, (b + 31) / 32, 32, 0, s->logits, s->y_i, s->y_f, b, c, s->loss, s->seeds,
                                                          s->pinv, s->rhs);
  ctx->launches++;
  s->row_state |= 1;
}

void row_rhs(cv_ctx* ctx, cv_snap* s, float* rhs) {
  ensure_seeds(ctx, s);
  cudaMemcpyAsync(rhs, s->rhs, sizeof(float) * s->bl * s->c, cudaMemcpyDeviceToDevice, ctx->stream);
}

static Operand sop(const SplitBuf& b, bool trans) {
  Operand o;
  o.hi = b.hi;
  o.lo = b.lo;
  o.si = trans ? 1 : b.ld;
  o.sj = trans ? b.ld : 1;
  o.sc = b.sc;
  return o;
}

__global__ void __launch_bounds__(256) k_sym_mirror(float* G, int64_t m);

// A block of Gram rows [r0, r0 + rows), columns 0 .. r0 + rows - 1 (lower part and the
// diagonal block), stored at out with leading dimension ld: the distributed row lane's
// block-cyclic row panels.
struct GramStrip {
  int64_t r0;
  int rows;
  float* out;
  int64_t ld;
};

// Gram = sum_l (D_l D_l^T) o kron(A_l A_l^T, 1 1^T): into s->gram (whole, mirrored), or
// into the given row strips only (the D chain and A_l A_l^T are formed whole either way).
static void gram_build(cv_ctx* ctx, cv_snap* s, const std::vector<GramStrip>* strips);

// Lower triangle (+ the diagonal tiles) of the snapshot Gram: all the Cholesky path reads.
static void ensure_gram(cv_ctx* ctx, cv_snap* s) {
  if (s->row_state & 2) return;
  gram_build(ctx, s, nullptr);
  s->row_state |= 2;
}
// The whole symmetric Gram (the upper half mirrored): the caller's copy and row CG's GEMV.
static void ensure_gram_full(cv_ctx* ctx, cv_snap* s) {
  ensure_gram(ctx, s);
  if (s->row_state & 4) return;
  const int64_t m = (int64_t)s->bl * s->c;
  const int nt = (int)((m + 31) / 32);
  launch_k(ctx->stream, k_sym_mirror, dim3(nt, nt), 256, 0, s->gram, m);
  ctx->launches++;
  s->row_state |= 4;
}

static void gram_build(cv_ctx* ctx, cv_snap* s, const std::vector<GramStrip>* strips) {
  ensure_seeds(ctx, s);
  const int b = s->bl, c = s->c, L = s->L;
  const int64_t m = (int64_t)b * c;
  if (!strips && !s->gram) s->gram = snap_alloc(s, m * m);
  float* sa = snap_alloc(s, (int64_t)b * b);
  // D ping-pong buffers sized for the widest layer
  int wmax = c;
  for (int l = 1; l < L; ++l) wmax = wmax > s->dims[l] ? wmax : s->dims[l];
  const int64_t ldD = ld_for(wmax);
  SplitBuf D[2];
  for (int k = 0; k < 2; ++k) {
    D[k].hi = (__half*)snap_alloc(s, (m * ldD + 1) / 2);
    D[k].lo = (__half*)snap_alloc(s, (m * ldD + 1) / 2);
    D[k].ld = ldD;
    D[k].sc = s->scratch_sc + k;
  }
  // D0 rows (i, a) = seeds[i, a, :]  (exact amax, two passes)
  // (zero columns c..15: the output layer's Gram term runs on the tensor engine with K = 16)
  split_mat(ctx, s->seeds, c, (int)m, c, D[0].hi, D[0].lo, ldD, 0, D[0].sc, 0, nullptr, ldD >= 16 ? 16 : 0);
  int cur = 0;
  for (int l = L - 1; l >= 0; --l) {
    const int nout = s->dims[l + 1];
    // SA = A_l A_l^T  (A augmented with the ones column: +1 covers the bias)
    GemmArgs g;
    g.M = b;
    g.N = b;
    g.nseg = 1;
    g.seg[0] = GemmSeg{sop(s->acts[l], false), sop(s->acts[l], true), s->dims[l] + 1};
    g.epi.mode = EPI_STORE;
    g.epi.out = sa;
    g.epi.ld = b;
    gemm(ctx, g);
    // gram (+)= (D D^T) o kron(SA, 1 1^T)
    GemmArgs h;
    h.M = (int)m;
    h.N = (int)m;
    h.nseg = 1;
    h.seg[0] = GemmSeg{sop(D[cur], false), sop(D[cur], true), (l == L - 1 && nout < 16 && ldD >= 16) ? 16 : nout};
    h.epi.mode = EPI_GRAM;
    h.epi.out = s->gram;
    h.epi.ld = m;
    h.epi.sa = sa;
    h.epi.sa_ld = b;
    h.epi.kdiv = c;
    h.epi.first = l == L - 1;
    h.lower_only = 1;  // SYRK: lower tiles only, mirrored below
    if (!strips) {
      gemm(ctx, h);
    } else {
      for (const GramStrip& g : *strips) {  // rows [r0, r0 + rows) against rows [0, r0 + rows)
        GemmArgs hs = h;
        hs.M = g.rows;
        hs.N = (int)(g.r0 + g.rows);
        hs.seg[0].A.hi += g.r0 * ldD;
        hs.seg[0].A.lo += g.r0 * ldD;
        hs.epi.out = g.out;
        hs.epi.ld = g.ld;
        hs.epi.row0 = g.r0;
        hs.lower_only = (int)g.r0 + 1;
        gemm(ctx, hs);
      }
    }
    if (l > 0) {
      // D <- (D W_l^T) * act'(a_l) broadcast over the k rows of each example
      cudaMemsetAsync(D[cur ^ 1].sc, 0, sizeof(Scale), ctx->stream);
      GemmArgs q;
      q.M = (int)m;
      q.N = s->dims[l];
      q.nseg = 1;
      Operand wt;
      wt.hi = s->w_hi + s->off[l];
      wt.lo = s->w_lo + s->off[l];
      wt.si = 1;
      wt.sj = nout;
      wt.sc = s->w_sc + l;
      int kq = nout;
      if (l == L - 1 && s->tc_out && nout < 16 && ldD >= 16) {
        // the output layer (K = c < 16): its transposed, zero-padded copy [W; b]^T (cp rows)
        // with D's zero columns c..15 gives the tensor engine a K = 16 slab
        wt.hi = s->wl_hi;
        wt.lo = s->wl_lo;
        wt.si = s->ldw;
        wt.sj = 1;
        kq = 16;
      }
      q.seg[0] = GemmSeg{sop(D[cur], false), wt, kq};
      q.epi.mode = EPI_SPLIT_MASK;
      q.epi.act = s->act;
      q.epi.out_hi = D[cur ^ 1].hi;
      q.epi.out_lo = D[cur ^ 1].lo;
      q.epi.out_sc = D[cur ^ 1].sc;
      q.epi.ld = ldD;
      q.epi.mask_hi = s->acts[l].hi;
      q.epi.mask_lo = s->acts[l].lo;
      q.epi.mask_sc = s->acts[l].sc;
      q.epi.mask_ld = s->acts[l].ld;
      q.epi.mask_div = c;
      q.epi.bound.n = 1;
      q.epi.bound.k[0] = (float)nout;
      q.epi.bound.x[0] = &D[cur].sc->amax;
      q.epi.bound.y[0] = &(s->w_sc + l)->amax;
      gemm(ctx, q);
      cur ^= 1;
    }
  }
}

const float* row_gram_dev(cv_ctx* ctx, cv_snap* s) {
  ensure_gram_full(ctx, s);
  return s->gram;
}

void row_gram(cv_ctx* ctx, cv_snap* s, float* gram_out) {
  ensure_gram_full(ctx, s);
  const int64_t m = (int64_t)s->bl * s->c;
  if (gram_out) cudaMemcpyAsync(gram_out, s->gram, sizeof(float) * m * m, cudaMemcpyDeviceToDevice, ctx->stream);
}

// ---------------------------------------------------------------------------
// Blocked right-looking Cholesky, lower, in place on chol = gram + mu I.
// ---------------------------------------------------------------------------
// dst = src + mu I on the lower triangle only (the factorization and the
// triangular solves never read above the diagonal): 32 x 32 tiles, tiles strictly
// above the diagonal skip; 128-bit rows when m % 4 == 0.
__global__ void __launch_bounds__(256) k_copy_lower_add_diag(const float* src, float* dst, int64_t m, float mu) {
  CV_PDL_ENTRY();
  const int64_t ti = blockIdx.y, tj = blockIdx.x;
  if (tj > ti) return;
  const int64_t i0 = ti * 32, j0 = tj * 32;
  const int c4 = threadIdx.x & 7, r8 = threadIdx.x >> 3;
  for (int rr = r8; rr < 32; rr += 32) {
    const int64_t i = i0 + rr;
    if (i >= m) break;
    const int64_t j = j0 + 4 * c4;
    if ((m & 3) == 0 && j + 3 < m) {
      float4 v = *reinterpret_cast<const float4*>(src + i * m + j);
      if (i >= j && i <= j + 3) (&v.x)[i - j] += mu;
      *reinterpret_cast<float4*>(dst + i * m + j) = v;
    } else {
      for (int q = 0; q < 4 && j + q < m; ++q) dst[i * m + j + q] = src[i * m + j + q] + (i == j + q ? mu : 0.f);
    }
  }
}

// G[j, i] = G[i, j] for i > j: the Gram is built as a SYRK (lower tiles only) and
// mirrored once, so consumers that stream whole rows (refinement residual, row-space
// CG products, cv_row_gram) see the full symmetric matrix.
__global__ void __launch_bounds__(256) k_sym_mirror(float* G, int64_t m) {
  CV_PDL_ENTRY();
  const int64_t ti = blockIdx.y, tj = blockIdx.x;  // destination tile (upper: tj >= ti)
  if (tj < ti) return;
  __shared__ float t[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  // source: rows tj*32.., cols ti*32.. (lower)
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = tj * 32 + r, j = ti * 32 + tx;
    if (i < m && j < m) t[r][tx] = G[i * m + j];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = ti * 32 + r, j = tj * 32 + tx;
    if (i < m && j < m && j > i) G[i * m + j] = t[tx][r];  // (diagonal tiles: their upper half only)
  }
}


// ---------------------------------------------------------------------------
// Diagonal (panel) block factorization.  The nbo x nbo diagonal block of a panel
// (nbo <= 512) is factored by 64-row tiles: one launch per tile column j, whose CTAs
// own the lower tiles (r, c), j < c <= r: CTA (r, c) forms L_rj = A_rj Dinv_j^T and
// L_cj (64^3 SIMT micro-GEMMs from shared memory), applies A_rc -= L_rj L_cj^T in
// place, and the CTA of the next diagonal tile (j+1, j+1) factors it at once
// (potrf64).  Column j is only read during launch j, so CTAs never race; L goes to a
// separate nbo x nbo block (Lblk) read by k_trtri_panel.  8 dependent launches per
// 512-wide panel.
// ---------------------------------------------------------------------------
constexpr int PS_LD = CH_NB + 1;  // padded shared row (floats)

struct Potrf64Smem {
  float colb[2][CH_NB];         // column k of the elimination (row k of X), double buffered
  float dg[CH_NB];              // pivots
  float Lsc[CH_NB][CH_NB + 1];  // Lsc[k][i] = L_ik / L_ii (i > k)
  int bad;
};

// Cholesky of a 64 x 64 SPD block held as 4 x 4 fp32 tiles by a 256-thread CTA
// (thread (ty, tx) = (tid / 16, tid % 16) owns tile (ty, tx); the lower tiles are
// used).  Step k applies a_ij -= a_ik a_jk / a_kk to the owned values with j > k,
// reading column k (final after step k-1) from a double-buffered shared row that the
// owners of column k+1 refill right after their own update: one barrier per column;
// the scaling by 1/sqrt(a_kk) is applied once at the end.  X = L^-1 is formed the
// same way (row k of X final at step k).  fp32 (the fp64 iterative refinement of the
// solve absorbs the factor's rounding).  Rows/cols >= nb must hold the identity.
CV_DEV void potrf64(float (&a)[4][4], int ty, int tx, int nb, float* Lout, int64_t ldl, float* Xout,
                    Potrf64Smem& sm, int* flag) {
  const bool own = ty >= tx;
  if (threadIdx.x == 0) sm.bad = 0;
  // column k lives in tile column k / 4, its column k % 4
  auto pub_col = [&](int kb, auto kk_) {
    constexpr int kk = decltype(kk_)::value;
    if (!own || tx != kb) return;
    float* cb = sm.colb[(4 * kb + kk) & 1];
#pragma unroll
    for (int r = 0; r < 4; ++r) cb[4 * ty + r] = a[r][kk];
  };
  auto elim = [&](int kb, auto kk_) {
    constexpr int kk = decltype(kk_)::value;
    const int k = 4 * kb + kk;
    const float* cb = sm.colb[k & 1];
    float piv = cb[k];
    if (!(piv > 0.f) || !isfinite(piv)) piv = 1.f;  // (flagged below by the pivot's owner)
    if (threadIdx.x == 0) sm.dg[k] = cb[k];
    if (!own || tx < kb) return;
    const float rp = 1.f / piv;
    float ci[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) ci[r] = cb[4 * ty + r];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (tx == kb && c <= kk) continue;
      const float sj = cb[4 * tx + c] * rp;
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r][c] = fmaf(-ci[r], sj, a[r][c]);
    }
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  using I3 = std::integral_constant<int, 3>;
  pub_col(0, I0{});
  __syncthreads();
  for (int kb = 0; kb < 16; ++kb) {
    elim(kb, I0{}); pub_col(kb, I1{}); __syncthreads();
    elim(kb, I1{}); pub_col(kb, I2{}); __syncthreads();
    elim(kb, I2{}); pub_col(kb, I3{}); __syncthreads();
    elim(kb, I3{}); if (kb + 1 < 16) pub_col(kb + 1, I0{}); __syncthreads();
  }
  // L_ij = a_ij / sqrt(d_j) (i > j), L_jj = sqrt(d_j); Lsc[k][i] = L_ik / L_ii
  float rs[4], rsi[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float d = sm.dg[4 * tx + q];
    if (!(d > 0.f) || !isfinite(d)) {
      if (ty == tx) sm.bad = 1;
      d = 1.f;
    }
    rs[q] = rsqrtf(d);
    float di = sm.dg[4 * ty + q];
    if (!(di > 0.f) || !isfinite(di)) di = 1.f;
    rsi[q] = rsqrtf(di);
  }
  float l[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const bool dgl = ty == tx && r == c;
      l[r][c] = (ty == tx && c > r) ? 0.f : (dgl ? 1.f / rs[c] : a[r][c] * rs[c]);
      if (own && (ty > tx || r > c)) sm.Lsc[4 * tx + c][4 * ty + r] = l[r][c] * rsi[r];
    }
  // X = L^-1: x[i][c] = delta_ic / L_ii, then x[i][c] -= (L_ik / L_ii) X[k][c] for k < i
  float x[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) x[r][c] = (ty == tx && r == c) ? rsi[r] : 0.f;
  __syncthreads();
  auto pub_row = [&](int kb, auto kk_) {
    constexpr int kk = decltype(kk_)::value;
    if (!own || ty != kb) return;
    float* rb = sm.colb[(4 * kb + kk) & 1];
#pragma unroll
    for (int c = 0; c < 4; ++c) rb[4 * tx + c] = x[kk][c];
  };
  auto inv_step = [&](int kb, auto kk_) {
    constexpr int kk = decltype(kk_)::value;
    const int k = 4 * kb + kk;
    if (!own || ty < kb || tx > kb) return;  // X[k][c] = 0 for c > k
    const float* rb = sm.colb[k & 1];
    float xk[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) xk[c] = rb[4 * tx + c];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (ty == kb && r <= kk) continue;
      const float lk = sm.Lsc[k][4 * ty + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) x[r][c] = fmaf(-lk, xk[c], x[r][c]);
    }
  };
  for (int kb = 0; kb < 16; ++kb) {
    pub_row(kb, I0{}); __syncthreads(); inv_step(kb, I0{});
    pub_row(kb, I1{}); __syncthreads(); inv_step(kb, I1{});
    pub_row(kb, I2{}); __syncthreads(); inv_step(kb, I2{});
    pub_row(kb, I3{}); __syncthreads(); inv_step(kb, I3{});
  }
  if (own) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = 4 * ty + r, j = 4 * tx + c;
        if (i >= nb || j >= nb) continue;
        if (j <= i) {
          Xout[i * nb + j] = x[r][c];
          Lout[(int64_t)i * ldl + j] = l[r][c];
          if (j != i) Xout[j * nb + i] = 0.f;
        }
      }
  }
  __syncthreads();
  if (threadIdx.x == 0 && sm.bad) *flag = 1;
}

// 64 x 64 tile (rows < rows_valid, cols < cols_valid, zero elsewhere) -> shared (ld PS_LD)
CV_DEV void load_tile(float* dst, const float* src, int64_t ld, int rows_valid, int cols_valid) {
  for (int e = threadIdx.x; e < CH_NB * CH_NB; e += blockDim.x) {
    const int i = e >> 6, j = e & 63;
    dst[i * PS_LD + j] = (i < rows_valid && j < cols_valid) ? src[(int64_t)i * ld + j] : 0.f;
  }
}
// acc[r][c] (+)= sign * sum_k X[4ty+r][k] Y[4tx+c][k]   (X, Y in shared memory, ld PS_LD)
CV_DEV void mm_xyt(const float* X, const float* Y, int ty, int tx, float (&acc)[4][4], float sign) {
#pragma unroll 4
  for (int k = 0; k < CH_NB; ++k) {
    float xr[4], yr[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      xr[q] = X[(4 * ty + q) * PS_LD + k];
      yr[q] = Y[(4 * tx + q) * PS_LD + k];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(sign * xr[r], yr[c], acc[r][c]);
  }
}

// First diagonal tile of a panel: factor A[p0.., p0..] (64 x 64, nb valid).
__global__ void __launch_bounds__(256) k_potrf_diag(const float* A, int64_t lda, int nb, float* Lblk, int64_t ldl,
                                                    float* dinv_blk, int* flag) {
  CV_PDL_ENTRY();
  __shared__ Potrf64Smem sm;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  float a[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = 4 * ty + r, j = 4 * tx + c;
      a[r][c] = (i < nb && j < nb) ? A[(int64_t)i * lda + j] : (i == j ? 1.f : 0.f);
    }
  potrf64(a, ty, tx, nb, Lblk, ldl, dinv_blk, sm, flag);
}

// Launch j of a panel's diagonal-block factorization (see above).  blockIdx.x
// enumerates the lower tiles (r, c), j < c <= r < nsub.
__global__ void __launch_bounds__(256) k_panel_step(float* A, int64_t lda, int nbo, int j, float* Lblk,
                                                    float* dinv, int* flag) {
  CV_PDL_ENTRY();
  extern __shared__ __align__(16) unsigned char psm[];
  float* D = reinterpret_cast<float*>(psm);              // Dinv_j
  float* T = D + CH_NB * PS_LD;                          // A_rj / A_cj staging
  float* LR = T + CH_NB * PS_LD;
  float* LC = LR + CH_NB * PS_LD;
  Potrf64Smem& sm = *reinterpret_cast<Potrf64Smem*>(LC + CH_NB * PS_LD);
  int e = blockIdx.x, r = j + 1;
  while (e >= r - j) { e -= r - j; ++r; }
  const int c = j + 1 + e;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  auto bsize = [&](int b) { return nbo - CH_NB * b < CH_NB ? nbo - CH_NB * b : CH_NB; };
  const int nbj = bsize(j), nbr = bsize(r), nbc = bsize(c);
  {
    const float* Dj = dinv + (int64_t)j * CH_NB * CH_NB;
    for (int q = threadIdx.x; q < CH_NB * CH_NB; q += blockDim.x) {
      const int i = q >> 6, k = q & 63;
      D[i * PS_LD + k] = (i < nbj && k < nbj) ? Dj[i * nbj + k] : 0.f;
    }
  }
  // L_rj = A_rj Dinv_j^T
  load_tile(T, A + (int64_t)CH_NB * r * lda + CH_NB * j, lda, nbr, nbj);
  __syncthreads();
  float acc[4][4] = {};
  mm_xyt(T, D, ty, tx, acc, 1.f);
#pragma unroll
  for (int rr = 0; rr < 4; ++rr)
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) LR[(4 * ty + rr) * PS_LD + 4 * tx + cc] = acc[rr][cc];
  if (c == j + 1) {  // one writer per L tile of column j
#pragma unroll
    for (int rr = 0; rr < 4; ++rr)
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int i = 4 * ty + rr, k = 4 * tx + cc;
        if (i < nbr && k < nbj) Lblk[(int64_t)(CH_NB * r + i) * nbo + CH_NB * j + k] = acc[rr][cc];
      }
  }
  const float* LCp = LR;
  if (c != r) {
    __syncthreads();  // T reused
    load_tile(T, A + (int64_t)CH_NB * c * lda + CH_NB * j, lda, nbc, nbj);
    __syncthreads();
    float acc2[4][4] = {};
    mm_xyt(T, D, ty, tx, acc2, 1.f);
#pragma unroll
    for (int rr = 0; rr < 4; ++rr)
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) LC[(4 * ty + rr) * PS_LD + 4 * tx + cc] = acc2[rr][cc];
    LCp = LC;
  }
  __syncthreads();
  // A_rc -= L_rj L_cj^T
  float* Arc = A + (int64_t)CH_NB * r * lda + CH_NB * c;
  float u[4][4];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr)
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const int i = 4 * ty + rr, k = 4 * tx + cc;
      u[rr][cc] = (i < nbr && k < nbc) ? Arc[(int64_t)i * lda + k] : 0.f;
    }
  mm_xyt(LR, LCp, ty, tx, u, -1.f);
  if (r == c && r == j + 1) {
    float a[4][4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr)
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int i = 4 * ty + rr, k = 4 * tx + cc;
        a[rr][cc] = (i < nbr && k < nbr) ? u[rr][cc] : (i == k ? 1.f : 0.f);
      }
    potrf64(a, ty, tx, nbr, Lblk + (int64_t)CH_NB * r * nbo + CH_NB * r, nbo, dinv + (int64_t)r * CH_NB * CH_NB, sm,
            flag);
  } else {
#pragma unroll
    for (int rr = 0; rr < 4; ++rr)
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int i = 4 * ty + rr, k = 4 * tx + cc;
        if (i < nbr && k < nbc) Arc[(int64_t)i * lda + k] = u[rr][cc];
      }
  }
}
constexpr int PS_SMEM = 4 * CH_NB * PS_LD * 4 + (int)sizeof(Potrf64Smem);

// W = L11^-1 for the nbo x nbo diagonal block of a panel (nbo <= TT_MAX), from the
// factored block (lower, in A at (p0, p0)) and the inverses of its 64-blocks (dinv):
// block forward substitution  X_jj = Dinv_j,  X_ij = -Dinv_i sum_{k=j}^{i-1} L_ik X_kj.
// Columns of the inverse are independent: each CTA owns TT_C columns (all inside one
// 64-block j) and walks the block rows i > j with its column strip in shared memory.
// W is row-major nbo x nbo, zero above the diagonal.
constexpr int TT_C = 4;
constexpr int TT_MAX = 1024;
// the (ib, kb) tiles a column strip walks, in order: L[ib][jb..ib-1], then Dinv_ib
struct TtTile {
  const float* p;
  int64_t ld;
  int rows, cols;
};
__global__ void __launch_bounds__(256) k_trtri_panel(const float* A, int64_t lda, const float* dinv, int p0, int nbo,
                                                     float* W, float* Wt) {
  CV_PDL_ENTRY();
  __shared__ float X[TT_MAX][TT_C];
  __shared__ __align__(16) float Lt[CH_NB][CH_NB + 4];
  __shared__ float S[CH_NB][TT_C];
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * TT_C;
  const int jb = c0 / CH_NB;
  const int nsub = (nbo + CH_NB - 1) / CH_NB;
  auto bsize = [&](int b) { return nbo - CH_NB * b < CH_NB ? nbo - CH_NB * b : CH_NB; };
  const int nbj = bsize(jb);
  const float* Dj = dinv + (int64_t)((p0 + CH_NB * jb) / CH_NB) * CH_NB * CH_NB;
  for (int e = tid; e < CH_NB * TT_C; e += blockDim.x) {
    const int r = e / TT_C, cc = e % TT_C, c = c0 + cc - CH_NB * jb;
    X[CH_NB * jb + r][cc] = (r < nbj && c < nbj && c <= r) ? Dj[r * nbj + c] : 0.f;
  }
  // tile t of the walk: for ib = jb+1.., kb = jb..ib-1 (L tiles) then the Dinv_ib tile
  auto tile_of = [&](int ib, int kb) {
    TtTile t;
    const int nbi = bsize(ib);
    if (kb < ib) {
      t.p = A + (int64_t)(p0 + CH_NB * ib) * lda + p0 + CH_NB * kb;
      t.ld = lda;
      t.rows = nbi;
      t.cols = CH_NB;
    } else {
      t.p = dinv + (int64_t)((p0 + CH_NB * ib) / CH_NB) * CH_NB * CH_NB;
      t.ld = nbi;
      t.rows = nbi;
      t.cols = nbi;
    }
    return t;
  };
  // register-staged prefetch of the next tile (4 x 16 bytes per thread, 128-bit when aligned)
  float4 pre[4];
  auto fetch = [&](const TtTile& t) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + u * 256;  // float4 index in the 64 x 64 tile
      const int rr = e / 16, c4 = (e % 16) * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (rr < t.rows) {
        const float* src = t.p + (int64_t)rr * t.ld + c4;
        if (c4 + 3 < t.cols && ((uintptr_t)src & 15) == 0) v = *reinterpret_cast<const float4*>(src);
        else {
          if (c4 < t.cols) v.x = src[0];
          if (c4 + 1 < t.cols) v.y = src[1];
          if (c4 + 2 < t.cols) v.z = src[2];
          if (c4 + 3 < t.cols) v.w = src[3];
        }
      }
      pre[u] = v;
    }
  };
  auto commit = [&]() {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + u * 256;
      *reinterpret_cast<float4*>(&Lt[e / 16][(e % 16) * 4]) = pre[u];
    }
  };
  int ib = jb + 1, kb = jb;
  if (ib < nsub) fetch(tile_of(ib, kb));
  __syncthreads();
  const int r = tid / 4, cq = (tid % 4) * (TT_C / 4);  // 64 rows x 4 column pairs
  float acc[TT_C / 4] = {};
  while (ib < nsub) {
    commit();
    __syncthreads();
    // next tile in flight while this one is used
    int nib = ib, nkb = kb + 1;
    if (nkb > ib) { nib = ib + 1; nkb = jb; }
    if (nib < nsub) fetch(tile_of(nib, nkb));
    const int nbi = bsize(ib);
    if (kb < ib) {
#pragma unroll 8
      for (int kk = 0; kk < CH_NB; ++kk) {
        const float l = Lt[r][kk];
#pragma unroll
        for (int u = 0; u < TT_C / 4; ++u) acc[u] = fmaf(l, X[CH_NB * kb + kk][cq + u], acc[u]);
      }
      __syncthreads();
      if (kb + 1 == ib) {  // S = sum_k L_ik X_kj complete
#pragma unroll
        for (int u = 0; u < TT_C / 4; ++u) {
          S[r][cq + u] = acc[u];
          acc[u] = 0.f;
        }
      }
    } else {
      // X_ib = -Dinv_ib S
      float o[TT_C / 4] = {};
      for (int kk = 0; kk <= r && kk < nbi; ++kk) {
        const float dk = Lt[r][kk];
#pragma unroll
        for (int u = 0; u < TT_C / 4; ++u) o[u] = fmaf(dk, S[kk][cq + u], o[u]);
      }
#pragma unroll
      for (int u = 0; u < TT_C / 4; ++u) X[CH_NB * ib + r][cq + u] = r < nbi ? -o[u] : 0.f;
      __syncthreads();
    }
    ib = nib;
    kb = nkb;
  }
  __syncthreads();
  for (int e = tid; e < nbo * TT_C; e += blockDim.x) {
    const int rr = e / TT_C, cc = e % TT_C, c = c0 + cc;
    if (c < nbo) W[(int64_t)rr * nbo + c] = rr < CH_NB * jb ? 0.f : X[rr][cc];
  }
  // and W^T (row c = column c of W, contiguous): the backward solve reads it by rows
  for (int e = tid; e < nbo * TT_C; e += blockDim.x) {
    const int cc = e / nbo, rr = e % nbo, c = c0 + cc;
    if (c < nbo) Wt[(int64_t)c * nbo + rr] = rr < CH_NB * jb ? 0.f : X[rr][cc];
  }
}

// Triangular solves with the panel inverses W_p = L_pp^-1 (k_trtri_panel, kept per
// panel): forward  y_p = W_p r_p,  r_below -= L21_p y_p;  backward  x_p = W_p^T (y_p -
// L21_p^T x_below).  Every step is a GEMV spread over many CTAs (fp32 matrix, fp64
// vectors), so a solve is ~5 short launches per 512-column panel.
__global__ void k_trsv_fwd_update(const float* A, int64_t lda, int64_t m, int j0, int nb, const double* y, double* r) {
  CV_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t row = j0 + nb + (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= m) return;
  double s = 0.0;
  const float* Ar = A + row * lda + j0;
  if ((nb & 127) == 0 && !(((uintptr_t)Ar) & 15)) {
    // 128-bit loads, all of a lane's loads independent (nb / 128 in flight)
#pragma unroll 4
    for (int k = lane * 4; k < nb; k += 128) {
      const float4 a = *reinterpret_cast<const float4*>(Ar + k);
      s += (double)a.x * y[j0 + k] + (double)a.y * y[j0 + k + 1] + (double)a.z * y[j0 + k + 2] +
           (double)a.w * y[j0 + k + 3];
    }
  } else {
    for (int k = lane; k < nb; k += 32) s += (double)Ar[k] * y[j0 + k];
  }
  s = warp_sum(s);
  if (lane == 0) r[row] -= s;
}
// backward: s_blk = L[j0+nb:, blk]^T v[j0+nb:]; v_blk = Dinv^T (y_blk - s_blk)
__global__ void k_trsv_bwd_gather(const float* A, int64_t lda, int64_t m, int j0, int nb, const double* v,
                                  double* partial, int rows_per_block) {
  CV_PDL_ENTRY();
  // partial[blockIdx.x * nb + k] = sum over this block's rows of A[row, j0+k] v[row]
  const int k = threadIdx.x;
  if (k >= nb) return;
  const int64_t r0 = j0 + nb + (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = r0 + rows_per_block < m ? r0 + rows_per_block : m;
  // 8 independent accumulators: 8 row loads in flight per thread
  double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int64_t row = r0;
  for (; row + 8 <= r1; row += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] += (double)A[(row + u) * lda + j0 + k] * v[row + u];
  }
  for (; row < r1; ++row) acc[0] += (double)A[row * lda + j0 + k] * v[row];
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += acc[u];
  partial[blockIdx.x * nb + k] = s;
}
// y[p0 + i] = sum_{j <= i} W[i, j] r[p0 + j]   (one warp per row of the lower W_p)
__global__ void __launch_bounds__(256) k_tri_wgemv(const float* W, int nbo, int p0, const double* r, double* y) {
  CV_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= nbo) return;
  double s = 0.0;
  const float* w = W + (int64_t)i * nbo;
  if ((nbo & 3) == 0) {  // 128-bit rows (W is stored with explicit zeros above the diagonal)
    for (int j = lane * 4; j <= i; j += 128) {
      const float4 q = *reinterpret_cast<const float4*>(w + j);
      const double* rr = r + p0 + j;
      s += (double)q.x * rr[0] + (double)q.y * rr[1] + (double)q.z * rr[2] + (double)q.w * rr[3];
    }
  } else {
    for (int j = lane; j <= i; j += 32) s += (double)w[j] * r[p0 + j];
  }
  s = warp_sum(s);
  if (lane == 0) y[p0 + i] = s;
}
// t_i = y[p0 + i] - sum_b partial[b][i] (fixed order): 32 rows i per CTA, its 8 warps
// stride over the partial blocks b and reduce in shared memory
__global__ void __launch_bounds__(256) k_tri_bwd_reduce(const double* y, const double* partial, int nparts, int nbo,
                                                        int p0, double* t) {
  CV_PDL_ENTRY();
  __shared__ double red[8][32];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (i < nbo)
    for (int b = wp; b < nparts; b += 8) s += partial[(int64_t)b * nbo + i];
  red[wp][lane] = s;
  __syncthreads();
  if (wp == 0 && i < nbo) {
    double a = 0.0;
    for (int w = 0; w < 8; ++w) a += red[w][lane];
    t[i] = y[p0 + i] - a;
  }
}
// x[p0 + j] = sum_{i >= j} W[i, j] t_i = sum_{i >= j} Wt[j, i] t_i: one warp per row of W^T
__global__ void __launch_bounds__(256) k_tri_wtgemv(const float* Wt, int nbo, int p0, const double* t, double* x) {
  CV_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (j >= nbo) return;
  double s = 0.0;
  const float* w = Wt + (int64_t)j * nbo;
  if ((nbo & 3) == 0) {  // 128-bit rows from the aligned start (W^T has zeros left of the diagonal)
    for (int i = (j & ~3) + lane * 4; i < nbo; i += 128) {
      const float4 q = *reinterpret_cast<const float4*>(w + i);
      s += (double)q.x * t[i] + (double)q.y * t[i + 1] + (double)q.z * t[i + 2] + (double)q.w * t[i + 3];
    }
  } else {
    for (int i = j + lane; i < nbo; i += 32) s += (double)w[i] * t[i];
  }
  s = warp_sum(s);
  if (lane == 0) x[p0 + j] = s;
}

// out[i] += sign * sum_{j < len_i} A[i, j] x[j], len_i = ncols (diag_off < 0) or
// diag_off + i + 1 (the lower part of a Gram strip row); one 256-thread block per row,
// 128-bit loads, two accumulators per thread, fixed-order block reduction
__global__ void __launch_bounds__(256) k_row_dot(const float* A, int64_t lda, int64_t ncols, int64_t diag_off,
                                                 const double* x, double sign, double* out, const int* skip) {
  CV_PDL_ENTRY();
  if (skip && *skip) return;
  const int i = blockIdx.x;
  const float* a = A + (int64_t)i * lda;
  const int64_t len = diag_off < 0 ? ncols : diag_off + i + 1;
  const bool vec = ((lda & 3) == 0) && !((uintptr_t)A & 15);
  const int64_t n4 = vec ? (len & ~(int64_t)3) : 0;
  double s0 = 0.0, s1 = 0.0;
  int64_t j = (int64_t)threadIdx.x * 4;
  for (; j + 1024 < n4; j += 2048) {
    const float4 p = *reinterpret_cast<const float4*>(a + j);
    const float4 q = *reinterpret_cast<const float4*>(a + j + 1024);
    s0 += (double)p.x * x[j] + (double)p.y * x[j + 1] + (double)p.z * x[j + 2] + (double)p.w * x[j + 3];
    s1 += (double)q.x * x[j + 1024] + (double)q.y * x[j + 1025] + (double)q.z * x[j + 1026] + (double)q.w * x[j + 1027];
  }
  for (; j < n4; j += 1024) {
    const float4 p = *reinterpret_cast<const float4*>(a + j);
    s0 += (double)p.x * x[j] + (double)p.y * x[j + 1] + (double)p.z * x[j + 2] + (double)p.w * x[j + 3];
  }
  for (int64_t t = n4 + threadIdx.x; t < len; t += 256) s1 += (double)a[t] * x[t];
  double v[1] = {s0 + s1};
  block_sum<1>(v);
  if (threadIdx.x == 0) out[i] += sign * v[0];
}
// Column sums in row slices: part[y][j] = sum over rows i of slice y (i >= j - r0 + 1
// when strict) of A[i, j] x[i], for j < ncols; k_col_reduce adds the slices in order.
constexpr int CD_SLICES = 32;
__global__ void __launch_bounds__(256) k_col_dot_part(const float* A, int64_t lda, int rows, int64_t ncols,
                                                      int64_t r0, int strict, const double* x, double* part,
                                                      const int* skip) {
  CV_PDL_ENTRY();
  if (skip && *skip) return;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  const int per = (rows + gridDim.y - 1) / gridDim.y;
  int i0 = blockIdx.y * per;
  const int i1 = min(rows, i0 + per);
  if (strict && j - r0 + 1 > i0) i0 = (int)(j - r0 + 1 < (int64_t)i1 ? j - r0 + 1 : (int64_t)i1);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int i = i0;
  for (; i + 4 <= i1; i += 4)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] += (double)A[(int64_t)(i + u) * lda + j] * x[i + u];
  for (; i < i1; ++i) acc[0] += (double)A[(int64_t)i * lda + j] * x[i];
  part[(int64_t)blockIdx.y * ncols + j] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
}
__global__ void k_col_reduce(const double* part, int slices, int64_t ncols, double* z, const int* skip) {
  CV_PDL_ENTRY();
  if (skip && *skip) return;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < ncols; j += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int y = 0; y < slices; ++y) s += part[(int64_t)y * ncols + j];
    z[j] += s;
  }
}
__global__ void k_sub_d(const double* y, const double* z, int n, double* t) {
  CV_PDL_ENTRY();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) t[i] = y[i] - z[i];
}
// r = rhs - (u + mu v)
__global__ void k_res_from(const float* rhs, const double* u, const double* v, double mu, int64_t m, double* r) {
  CV_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = (double)rhs[i] - (u[i] + mu * v[i]);
}
__global__ void k_flag_d(const int* flag, double* out) {
  CV_PDL_ENTRY();
  *out = *flag ? 1.0 : 0.0;
}

// z[j] += sum_i A[i, j] x[i] over a row block of a strip layout (ld m); strict: only
// the strictly-lower part (rows with r0 + i > j).  part: CD_SLICES x ncols doubles.
static void col_dot(cv_ctx* ctx, const float* A, int64_t m, int rows, int64_t ncols, int64_t r0, int strict,
                    const double* x, double* z, double* part, const int* skip) {
  const int slices = std::min(CD_SLICES, std::max(1, rows / 32));
  launch_k(ctx->stream, k_col_dot_part, dim3((unsigned)((ncols + 255) / 256), (unsigned)slices), 256, 0, A, m, rows,
           ncols, r0, strict, x, part, skip);
  launch_k(ctx->stream, k_col_reduce, (int)std::min<int64_t>(1024, (ncols + 255) / 256), 256, 0, (const double*)part,
           slices, ncols, z, skip);
  ctx->launches += 2;
}

__global__ void k_axpy_d(const double* x, double* y, int64_t n) {
  CV_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) y[i] += x[i];
}

__global__ void k_f2d(const float* x, double* y, int64_t n) {
  CV_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) y[i] = x[i];
}
__global__ void k_d2f(const double* x, float* y, int64_t n) {
  CV_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) y[i] = (float)x[i];
}

// (Gram + mu I) v = rhs for a dense symmetric m x m fp32 Gram (full storage) on the
// device (solvers.py:146-161).  Workspace: chol (m x m, lower factor) and dinv
// (inverses of the 64-blocks).  Returns 1 if the system is not positive definite.
//
// Two-level right-looking blocked Cholesky.  Each 512-column panel:
//  (1) its 512 x 512 diagonal block is factored with the register-resident fp64
//      64-block kernel (k_potrf_diag) and SIMT TRSM / updates confined to the block;
//  (2) W = L11^-1 (k_trtri_panel);
//  (3) the panel below the block, L21 = A21 W^T, is one tensor-core GEMM;
//  (4) the trailing update A22 -= L21 L21^T (lower tiles) is one tensor-core GEMM.
// All but O(m^2 x 512) of the m^3/3 flops run on the tensor engine (3xFP16 split
// operands); fp64 triangular solves and two steps of fp64 iterative refinement
// against the fp32 Gram absorb the split's rounding (cf. the 1e-6 lane-equivalence
// bound, tests/test_solvers.py:216-236).  The SIMT engine (CV_ENGINE_SIMT) or a
// system of one panel factors everything with exact-fp32 SIMT kernels.
int dense_cholesky_solve(cv_ctx* ctx, const float* gram, int64_t m, double mu, const float* rhs, float* v_out,
                         float* chol, float* dinv, float* winv, Scale* scr_sc) {
  cudaStream_t st = ctx->stream;
  {
    const int nt = (int)((m + 31) / 32);
    launch_k(st, k_copy_lower_add_diag, dim3(nt, nt), 256, 0, gram, chol, m, (float)mu);
  }
  int* flag = (int*)(ctx->scal_ws + 32);
  cudaMemsetAsync(flag, 0, sizeof(int), st);
  ctx->launches++;
  constexpr int NBO = TT_MAX;  // panel width (a multiple of CH_NB)
  const bool tc = m > NBO;     // (the GEMMs follow the context's engine selection)
  float* winvT = winv + ((m + NBO - 1) / NBO) * (int64_t)NBO * NBO;  // second half: the W^T of each panel
  __half *l21h = nullptr, *l21l = nullptr, *wh = nullptr, *wl = nullptr;
  if (tc) {
    l21h = (__half*)ctx->pool.get(sizeof(__half) * (size_t)(m - NBO) * NBO);
    l21l = (__half*)ctx->pool.get(sizeof(__half) * (size_t)(m - NBO) * NBO);
    wh = (__half*)ctx->pool.get(sizeof(__half) * (size_t)NBO * NBO);
    wl = (__half*)ctx->pool.get(sizeof(__half) * (size_t)NBO * NBO);
  }
  Scale* l21sc = scr_sc;
  Scale* wsc = scr_sc + 1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_panel_step, cudaFuncAttributeMaxDynamicSharedMemorySize, PS_SMEM);
    attr = true;
  }
  float* Lblk = (float*)ctx->pool.get(sizeof(float) * (size_t)NBO * NBO);
  // (1)+(2) the diagonal block of the panel at p0 (first tile, then one launch per tile
  // column) and W = L11^-1 (kept: the triangular solves multiply by it), on stream `ds`
  auto diag = [&](int64_t p0, cudaStream_t ds) {
    const int nbo = (int)((m - p0) < NBO ? (m - p0) : NBO);
    const int nsub = (nbo + CH_NB - 1) / CH_NB;
    float* Ad = chol + p0 * m + p0;
    float* dp = dinv + (p0 / CH_NB) * (int64_t)CH_NB * CH_NB;
    launch_k(ds, k_potrf_diag, 1, 256, 0, (const float*)Ad, m, nbo < CH_NB ? nbo : CH_NB, Lblk, (int64_t)nbo, dp,
             flag);
    for (int j = 0; j + 1 < nsub; ++j) {
      const int tiles = (nsub - j - 1) * (nsub - j) / 2;
      launch_k(ds, k_panel_step, tiles, 256, PS_SMEM, Ad, m, nbo, j, Lblk, dp, flag);
    }
    launch_k(ds, k_trtri_panel, (nbo + TT_C - 1) / TT_C, 256, 0, (const float*)Lblk, (int64_t)nbo, (const float*)dp,
             0, nbo, winv + (p0 / NBO) * (int64_t)NBO * NBO, winvT + (p0 / NBO) * (int64_t)NBO * NBO);
    ctx->launches += nsub + 1;
  };
  // Look-ahead: once L21 of panel p is known, the diagonal block of panel p+1 is updated
  // first (a small GEMM), then factored on a side stream while the rest of panel p's
  // trailing update runs on the other SMs -- the latency-bound diagonal work hides under
  // the tensor-core update instead of following it.
  constexpr int kReserveSMs = 16;
  diag(0, st);
  for (int64_t p0 = 0; p0 < m; p0 += NBO) {
    const int nbo = (int)((m - p0) < NBO ? (m - p0) : NBO);
    const int rest2 = (int)(m - p0 - nbo);
    if (rest2 <= 0) break;
    float* W = winv + (p0 / NBO) * (int64_t)NBO * NBO;
    // (3) L21 = A21 W^T on the tensor cores (A21 split first; the GEMM writes fp32 L21 in place)
    float* A21 = chol + (p0 + nbo) * m + p0;
    split_mat(ctx, A21, m, rest2, nbo, l21h, l21l, nbo, 0, l21sc, 0, nullptr);
    split_mat(ctx, W, nbo, nbo, nbo, wh, wl, nbo, 0, wsc, 0, nullptr);
    {
      Operand A, B;
      A.hi = l21h; A.lo = l21l; A.sc = l21sc; A.si = nbo; A.sj = 1;  // A(i, k) = A21[i, k]
      B.hi = wh; B.lo = wl; B.sc = wsc; B.si = 1; B.sj = nbo;        // B(k, j) = W[j, k]
      GemmArgs t;
      t.M = rest2;
      t.N = nbo;
      t.nseg = 1;
      t.seg[0] = GemmSeg{A, B, nbo};
      t.epi.mode = EPI_STORE;
      t.epi.out = A21;
      t.epi.ld = m;
      gemm(ctx, t);
    }
    // (4) trailing update A22 -= L21 L21^T (lower) on the tensor cores, in two parts
    split_mat(ctx, A21, m, rest2, nbo, l21h, l21l, nbo, 0, l21sc, 0, nullptr);
    const int64_t nx = p0 + nbo;  // the next panel
    const int nb1 = rest2 < NBO ? rest2 : NBO;
    auto update = [&](int64_t r0, int rows, int cols, int offset, int max_ctas) {
      Operand A, B;
      A.hi = l21h + (r0 - nx) * nbo; A.lo = l21l + (r0 - nx) * nbo; A.sc = l21sc; A.si = nbo; A.sj = 1;
      B.hi = l21h; B.lo = l21l; B.sc = l21sc; B.si = 1; B.sj = nbo;  // B(k, j) = L21[j, k]
      GemmArgs u;
      u.M = rows;
      u.N = cols;
      u.nseg = 1;
      u.seg[0] = GemmSeg{A, B, nbo};
      u.epi.mode = EPI_ACCUM;
      u.epi.alpha = -1.f;
      u.epi.out = chol + r0 * m + nx;
      u.epi.ld = m;
      u.lower_only = offset + 1;  // lower part relative to the diagonal `offset` columns right
      u.max_ctas = max_ctas;
      gemm(ctx, u);
    };
    // (4a) the next panel's diagonal block
    update(nx, nb1, nb1, 0, 0);
    // look ahead while the rest of the update is long enough that overlapping it with the
    // diagonal work (~0.7 ms on the reserved SMs) beats giving it every SM (measured at C4:
    // threshold 1.0 ms -> 126.9 ms/step, 0.3 ms -> 123.9, 0 -> 124.2)
    const double rows = (double)(rest2 - nb1), upd_ms = rows * ((double)rest2 - 0.5 * rows) * 2.0 * nbo / 4.5e11;
    if (rest2 > nb1 && upd_ms > 0.3 && ctx->sm_count > 4 * kReserveSMs) {
      // (4b) its factorization beside (4c) the rest of the update: rows below it, columns
      // from it on (the lower part relative to the shifted diagonal)
      cudaStream_t side = side_fork(ctx);
      diag(nx, side);
      update(nx + nb1, rest2 - nb1, rest2, nb1, ctx->sm_count - kReserveSMs);
      side_join(ctx);
    } else {
      if (rest2 > nb1) update(nx + nb1, rest2 - nb1, rest2, nb1, 0);
      diag(nx, st);
    }
  }
  ctx->pool.put(Lblk);
  if (tc) {
    ctx->pool.put(l21h);
    ctx->pool.put(l21l);
    ctx->pool.put(wh);
    ctx->pool.put(wl);
  }
  int hflag = 0;
  cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  if (hflag) return 1;
  // fp64 triangular solves, then iterative refinement against the fp32 Gram:
  // v <- v + (L L^T)^-1 (rhs - (Gram + mu I) v), residual accumulated in fp64
  double* r = (double*)ctx->pool.get(sizeof(double) * m * 5);
  double* y = r + m;
  double* v = r + 2 * m;
  double* dv = r + 3 * m;
  double* zz = r + 4 * m;
  double* cpart = (double*)ctx->pool.get(sizeof(double) * (size_t)(CD_SLICES * m));
  const int64_t nparts_max = 2 * ctx->sm_count;
  double* part = (double*)ctx->pool.get(sizeof(double) * (size_t)(nparts_max + 1) * NBO);
  double* tvec = part + nparts_max * NBO;
  const int npan = (int)((m + NBO - 1) / NBO);
  auto tri_solve = [&](double* x) {  // r -> x = (L L^T)^-1 r   (r is consumed)
    for (int pi = 0; pi < npan; ++pi) {
      const int p0 = pi * NBO;
      const int nbp = (int)((m - p0) < NBO ? (m - p0) : NBO);
      const float* W = winv + (int64_t)pi * NBO * NBO;
      launch_k(st, k_tri_wgemv, (nbp + 7) / 8, 256, 0, W, nbp, p0, (const double*)r, y);
      const int64_t rest = m - p0 - nbp;
      if (rest > 0) launch_k(st, k_trsv_fwd_update, (int)((rest + 7) / 8), 256, 0, chol, m, m, p0, nbp, y, r);
      ctx->launches += rest > 0 ? 2 : 1;
    }
    for (int pi = npan - 1; pi >= 0; --pi) {
      const int p0 = pi * NBO;
      const int nbp = (int)((m - p0) < NBO ? (m - p0) : NBO);
      const int64_t rest = m - p0 - nbp;
      int nparts = 0;
      if (rest > 0) {
        int64_t rpb = (rest + nparts_max - 1) / nparts_max;
        if (rpb < 32) rpb = 32;
        nparts = (int)((rest + rpb - 1) / rpb);
        launch_k(st, k_trsv_bwd_gather, nparts, NBO, 0, chol, m, m, p0, nbp, (const double*)x, part, (int)rpb);
        ctx->launches++;
      }
      launch_k(st, k_tri_bwd_reduce, (nbp + 31) / 32, 256, 0, (const double*)y, (const double*)part, nparts, nbp, p0,
               tvec);
      launch_k(st, k_tri_wtgemv, (nbp + 7) / 8, 256, 0, winvT + (int64_t)pi * NBO * NBO, nbp, p0,
               (const double*)tvec, x);
      ctx->launches += 2;
    }
  };
  launch_k(st, k_f2d, 256, 256, 0, rhs, r, m);
  tri_solve(v);
  for (int it = 0; it < 2; ++it) {
    // r = rhs - (Gram + mu I) v from the lower triangle only (row parts j <= i, then the
    // transposed strictly-lower parts): the Gram's upper half is never read
    cudaMemsetAsync(zz, 0, sizeof(double) * m, st);
    launch_k(st, k_row_dot, (int)m, 256, 0, gram, m, (int64_t)0, (int64_t)0, (const double*)v, 1.0, zz,
             (const int*)nullptr);
    ctx->launches++;
    col_dot(ctx, gram, m, (int)m, m, 0, 1, v, zz, cpart, nullptr);
    launch_k(st, k_res_from, 256, 256, 0, rhs, (const double*)zz, (const double*)v, mu, m, r);
    tri_solve(dv);
    launch_k(st, k_axpy_d, 256, 256, 0, dv, v, m);
    ctx->launches += 2;
  }
  launch_k(st, k_d2f, 256, 256, 0, v, v_out, m);
  ctx->launches += 2;
  ctx->pool.put(cpart);
  ctx->pool.put(part);
  ctx->pool.put(r);
  return 0;
}

int row_solve_cholesky(cv_ctx* ctx, cv_snap* s, double mu, const float* rhs, float* v_out) {
  ensure_gram(ctx, s);
  const int64_t m = (int64_t)s->bl * s->c;
  if (!s->chol) s->chol = snap_alloc(s, m * m);
  const int nblk = (int)((m + CH_NB - 1) / CH_NB);
  if (!s->dinv) s->dinv = snap_alloc(s, (int64_t)nblk * CH_NB * CH_NB);
  const int64_t npan = (m + TT_MAX - 1) / TT_MAX;
  if (!s->winv) s->winv = snap_alloc(s, 2 * npan * TT_MAX * TT_MAX);  // W and W^T per panel
  return dense_cholesky_solve(ctx, s->gram, m, mu, rhs, v_out, s->chol, s->dinv, s->winv, s->scratch_sc + 2);
}

int dense_cholesky(cv_ctx* ctx, const float* gram, int64_t m, double mu, const float* rhs, float* v_out) {
  float* chol = (float*)ctx->pool.get(sizeof(float) * (size_t)(m * m));
  const int64_t nblk = (m + CH_NB - 1) / CH_NB;
  float* dinv = (float*)ctx->pool.get(sizeof(float) * (size_t)(nblk * CH_NB * CH_NB));
  Scale* sc = (Scale*)ctx->pool.get(sizeof(Scale) * 4);
  const int64_t npan = (m + TT_MAX - 1) / TT_MAX;
  float* winv = (float*)ctx->pool.get(sizeof(float) * (size_t)(2 * npan * TT_MAX * TT_MAX));  // W and W^T
  int rc = 1;
  try {
    rc = dense_cholesky_solve(ctx, gram, m, mu, rhs, v_out, chol, dinv, winv, sc);
  } catch (...) {
    ctx->pool.put(winv); ctx->pool.put(sc); ctx->pool.put(dinv); ctx->pool.put(chol);
    throw;
  }
  ctx->pool.put(winv);
  ctx->pool.put(sc);
  ctx->pool.put(dinv);
  ctx->pool.put(chol);
  return rc;
}

void row_backproject(cv_ctx* ctx, cv_snap* s, const float* v, float* out) {
  ensure_seeds(ctx, s);
  const int64_t m = (int64_t)s->bl * s->c;
  launch_k(ctx->stream, k_seed_apply, (int)((m + 255) / 256), 256, 0, s->seeds, v, s->bl, s->c, s->U2);
  ctx->launches++;
  mlp_vjp(ctx, s, s->U2, out);
}

// ---------------------------------------------------------------------------
// Distributed row lane: (Gram + mu I) v = rhs across the ranks of the
// context, the Gram never held whole by any rank.  The m rows are cut into panels of
// NBO = 1024 rows dealt block-cyclically (panel p on rank p mod world), so every rank
// holds ~m/world rows of the lower triangle and the factorization's work stays
// balanced as the trailing matrix shrinks.  The snapshot `s` holds the whole batch on
// every rank (the caller gathers it): the D chain and A_l A_l^T are formed whole, the
// Gram SYRK only for the rank's row panels (gram_build with strips).
//
// Right-looking factorization, step k (panel column k):
//  - the owner of panel k factors its diagonal block and forms W_k = L_kk^-1 (the
//    single-GPU kernels: k_potrf_diag, k_panel_step, k_trtri_panel); W_k and W_k^T are
//    broadcast (the triangular solves of every rank use them);
//  - each rank forms L_ik = A_ik W_k^T for its panels i > k (one tensor-core GEMM over
//    its contiguous local rows) and the panels are broadcast by their owners into a
//    buffer in global row order (one NCCL group);
//  - each rank applies A_ij -= L_ik L_jk^T to its panels i > k (lower part, red.add
//    epilogue), the owner of panel k+1 first, whose diagonal block is then factored on a
//    side stream while the rest of the update runs (look-ahead).
// Triangular solves with replicated fp64 vectors: forward, the owner of panel k forms
// y_k = W_k (r_k - L_k,<k y_<k) and broadcasts it; backward, every rank accumulates
// L_i,<i^T x_i of its own panels, the k-block of those sums is all-reduced, and every
// rank forms x_k = W_k^T (y_k - s_k) itself.  Two steps of fp64 refinement use the
// rank's Gram strips (row part + transposed strictly-lower part, all-reduced).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_strip_lower_add_diag(const float* src, float* dst, int rows, int64_t r0,
                                                              int64_t ld, float mu) {
  CV_PDL_ENTRY();
  const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  if (j0 > r0 + i0 + 31) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int rr = ty; rr < 32; rr += 8) {
    const int64_t i = i0 + rr, j = j0 + tx;
    if (i >= rows || j > r0 + i) continue;
    const float v = src[i * ld + j];
    dst[i * ld + j] = j == r0 + i ? v + mu : v;
  }
}
// The rank's Gram row strips (block-cyclic 1024-row panels), built from the snapshot.
static std::vector<GramStrip> build_strips(cv_ctx* ctx, cv_snap* s, float* gram) {
  constexpr int NBO = TT_MAX;
  const int W = ctx->world, R = ctx->rank;
  const int64_t m = (int64_t)s->bl * s->c;
  const int np = (int)((m + NBO - 1) / NBO);
  std::vector<GramStrip> strips;
  int64_t lr = 0;
  for (int p = R; p < np; p += W) {
    const int rows = (int)std::min<int64_t>(NBO, m - (int64_t)p * NBO);
    strips.push_back(GramStrip{(int64_t)p * NBO, rows, gram + lr * m, m});
    lr += rows;
  }
  if (!strips.empty()) gram_build(ctx, s, &strips);
  else ensure_seeds(ctx, s);
  return strips;
}
static int64_t strip_rows(const cv_ctx* ctx, int64_t m) {
  constexpr int NBO = TT_MAX;
  const int np = (int)((m + NBO - 1) / NBO);
  int64_t lr = 0;
  for (int p = ctx->rank; p < np; p += ctx->world) lr += std::min<int64_t>(NBO, m - (int64_t)p * NBO);
  return lr;
}
// z = Gram v, summed over the ranks' strips (row parts + transposed strictly-lower parts)
static void strips_gv(cv_ctx* ctx, const std::vector<GramStrip>& strips, int64_t m, const double* v, double* z,
                      double* part, const int* skip) {
  cudaMemsetAsync(z, 0, sizeof(double) * m, ctx->stream);
  for (const GramStrip& g : strips) {
    launch_k(ctx->stream, k_row_dot, g.rows, 256, 0, (const float*)g.out, m, (int64_t)0, g.r0, v, 1.0, z + g.r0,
             skip);
    ctx->launches++;
    col_dot(ctx, g.out, m, g.rows, g.r0 + g.rows, g.r0, 1, v + g.r0, z, part, skip);
  }
  allreduce_f64(ctx, z, m);
}

// Row-space CG (solvers.py:164-174) across the ranks: the dense CG loop (replicated fp64
// m-vectors and decisions) with the Gram product from the rank's strips + an m-vector
// all-reduce per product.
void dist_row_cg(cv_ctx* ctx, cv_snap* s, double mu, const float* rhs, double tol, int maxiter, int stab,
                 const float* x0, float* v_out, cv_cg_stats* stats) {
  const int64_t m = (int64_t)s->bl * s->c;
  float* gram = (float*)ctx->pool.get(sizeof(float) * (size_t)std::max<int64_t>(1, strip_rows(ctx, m) * m));
  double* part = (double*)ctx->pool.get(sizeof(double) * (size_t)(CD_SLICES * m));
  try {
    const std::vector<GramStrip> strips = build_strips(ctx, s, gram);
    dense_cg_run(ctx, m, [&](const double* in, double* out, const int* skip) {
      strips_gv(ctx, strips, m, in, out, part, skip);
    }, rhs, mu, tol, maxiter, stab, x0, v_out, stats);
  } catch (...) {
    ctx->pool.put(part);
    ctx->pool.put(gram);
    throw;
  }
  ctx->pool.put(part);
  ctx->pool.put(gram);
}

int dist_row_cholesky(cv_ctx* ctx, cv_snap* s, double mu, const float* rhs, float* v_out) {
  constexpr int NBO = TT_MAX;
  const int W = ctx->world, R = ctx->rank;
  const int64_t m = (int64_t)s->bl * s->c;
  const int np = (int)((m + NBO - 1) / NBO);
  cudaStream_t st = ctx->stream;
  auto owner = [&](int p) { return p % W; };
  auto mine = [&](int p) { return p % W == R; };
  auto prow = [&](int p) { return (int)std::min<int64_t>(NBO, m - (int64_t)p * NBO); };
  auto lrow = [&](int p) { return (int64_t)(p / W) * NBO; };  // local row of my panel p
  int64_t lrows = 0;
  for (int p = R; p < np; p += W) lrows += prow(p);
  Pool& pool = ctx->pool;
  std::vector<void*> bufs;
  auto get = [&](size_t bytes) {
    void* q = pool.get(bytes ? bytes : 16);
    bufs.push_back(q);
    return q;
  };
  int rc = 0;
  try {
    float* gram = (float*)get(sizeof(float) * (size_t)(lrows * m));
    float* chol = (float*)get(sizeof(float) * (size_t)(lrows * m));
    float* dinv = (float*)get(sizeof(float) * (size_t)(((m + CH_NB - 1) / CH_NB) * CH_NB * CH_NB));
    float* winv = (float*)get(sizeof(float) * (size_t)(2 * (int64_t)np * NBO * NBO));
    float* winvT = winv + (int64_t)np * NBO * NBO;
    float* gbuf = (float*)get(sizeof(float) * (size_t)(m * NBO));
    __half* gh = (__half*)get(sizeof(__half) * (size_t)(m * NBO));
    __half* gl = (__half*)get(sizeof(__half) * (size_t)(m * NBO));
    __half* ah = (__half*)get(sizeof(__half) * (size_t)(lrows * NBO));
    __half* al = (__half*)get(sizeof(__half) * (size_t)(lrows * NBO));
    __half* wh = (__half*)get(sizeof(__half) * (size_t)NBO * NBO);
    __half* wl = (__half*)get(sizeof(__half) * (size_t)NBO * NBO);
    float* Lblk = (float*)get(sizeof(float) * (size_t)NBO * NBO);
    Scale* sc = (Scale*)get(sizeof(Scale) * 4);
    double* vecs = (double*)get(sizeof(double) * (size_t)(6 * m + 8));
    // Gram strips of my panels, then chol = their lower part + mu I
    const std::vector<GramStrip> strips = build_strips(ctx, s, gram);
    for (const GramStrip& g : strips) {
      launch_k(st, k_strip_lower_add_diag, dim3((unsigned)((m + 31) / 32), (unsigned)((g.rows + 31) / 32)), 256, 0,
               (const float*)g.out, chol + (g.out - gram), g.rows, g.r0, m, (float)mu);
      ctx->launches++;
    }
    int* flag = (int*)(ctx->scal_ws + 32);
    cudaMemsetAsync(flag, 0, sizeof(int), st);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_panel_step, cudaFuncAttributeMaxDynamicSharedMemorySize, PS_SMEM);
      attr = true;
    }
    // my diagonal block of panel k: factor, 64-block inverses, W_k and W_k^T
    auto diag = [&](int k, cudaStream_t ds) {
      const int nbo = prow(k);
      const int nsub = (nbo + CH_NB - 1) / CH_NB;
      const int64_t p0 = (int64_t)k * NBO;
      float* Ad = chol + lrow(k) * m + p0;
      float* dp = dinv + (p0 / CH_NB) * (int64_t)CH_NB * CH_NB;
      launch_k(ds, k_potrf_diag, 1, 256, 0, (const float*)Ad, m, nbo < CH_NB ? nbo : CH_NB, Lblk, (int64_t)nbo, dp,
               flag);
      for (int j = 0; j + 1 < nsub; ++j) {
        const int tiles = (nsub - j - 1) * (nsub - j) / 2;
        launch_k(ds, k_panel_step, tiles, 256, PS_SMEM, Ad, m, nbo, j, Lblk, dp, flag);
      }
      launch_k(ds, k_trtri_panel, (nbo + TT_C - 1) / TT_C, 256, 0, (const float*)Lblk, (int64_t)nbo,
               (const float*)dp, 0, nbo, winv + (int64_t)k * NBO * NBO, winvT + (int64_t)k * NBO * NBO);
      ctx->launches += nsub + 1;
    };
    constexpr int kReserveSMs = 16;
    int ahead = -1;  // panel whose diagonal block the previous step already factored
    for (int k = 0; k < np; ++k) {
      const int64_t p0 = (int64_t)k * NBO;
      const int nbk = prow(k);
      if (mine(k) && ahead != k) diag(k, st);
      comm_group(ctx, true);
      broadcast(ctx, winv + (int64_t)k * NBO * NBO, (int64_t)nbk * nbk, CV_DTYPE_F32, owner(k));
      broadcast(ctx, winvT + (int64_t)k * NBO * NBO, (int64_t)nbk * nbk, CV_DTYPE_F32, owner(k));
      comm_group(ctx, false);
      const int64_t rest = m - p0 - nbk;
      if (rest <= 0) break;
      // L_ik = A_ik W_k^T for my panels i > k (contiguous local rows), in place
      int pf = k + 1;
      while (pf < np && !mine(pf)) ++pf;
      if (pf < np) {
        const int64_t rowsA = lrows - lrow(pf);
        float* A21 = chol + lrow(pf) * m + p0;
        const float* Wk = winv + (int64_t)k * NBO * NBO;
        split_mat(ctx, A21, m, (int)rowsA, nbk, ah, al, nbk, 0, sc, 0, nullptr);
        split_mat(ctx, Wk, nbk, nbk, nbk, wh, wl, nbk, 0, sc + 1, 0, nullptr);
        Operand A, B;
        A.hi = ah; A.lo = al; A.sc = sc; A.si = nbk; A.sj = 1;
        B.hi = wh; B.lo = wl; B.sc = sc + 1; B.si = 1; B.sj = nbk;  // B(k, j) = W[j, k]
        GemmArgs t;
        t.M = (int)rowsA;
        t.N = nbk;
        t.nseg = 1;
        t.seg[0] = GemmSeg{A, B, nbk};
        t.epi.mode = EPI_STORE;
        t.epi.out = A21;
        t.epi.ld = m;
        gemm(ctx, t);
        for (int p = pf; p < np; p += W)  // into the global-order panel column
          cudaMemcpy2DAsync(gbuf + (int64_t)(p - k - 1) * NBO * nbk, sizeof(float) * nbk, chol + lrow(p) * m + p0,
                            sizeof(float) * m, sizeof(float) * nbk, prow(p), cudaMemcpyDeviceToDevice, st);
        // my rows of the panel column, split: the A operand of my trailing update
        split_mat(ctx, A21, m, (int)rowsA, nbk, ah, al, nbk, 0, sc + 3, 0, nullptr);
      }
      comm_group(ctx, true);
      for (int p = k + 1; p < np; ++p)
        broadcast(ctx, gbuf + (int64_t)(p - k - 1) * NBO * nbk, (int64_t)prow(p) * nbk, CV_DTYPE_F32, owner(p));
      comm_group(ctx, false);
      if (pf >= np) continue;  // no trailing rows here
      // the trailing update of my panels from the (replicated) panel column
      split_mat(ctx, gbuf, nbk, (int)rest, nbk, gh, gl, nbk, 0, sc + 2, 0, nullptr);
      // A_ij -= L_ik L_jk^T for my panels i >= p_start (contiguous local rows) and j <= i:
      // one GEMM, the block-cyclic lower predicate (cyc_nb / cyc_skip) skipping the tiles
      // right of each panel's diagonal
      auto update = [&](int p_start, int p_count, int max_ctas) {
        const int64_t lr0 = lrow(p_start) - lrow(pf);
        int64_t rows = 0;
        for (int p = p_start, c = 0; p < np && c < p_count; p += W, ++c) rows += prow(p);
        Operand A, B;
        A.hi = ah + lr0 * nbk; A.lo = al + lr0 * nbk; A.sc = sc + 3; A.si = nbk; A.sj = 1;
        B.hi = gh; B.lo = gl; B.sc = sc + 2; B.si = 1; B.sj = nbk;  // B(k, j) = L[j, k]
        GemmArgs u;
        u.M = (int)rows;
        u.N = (int)std::min<int64_t>(rest, (int64_t)(p_start - k - 1 + (int64_t)(p_count - 1) * W) * NBO +
                                               prow(std::min(np - 1, p_start + (p_count - 1) * W)));
        u.nseg = 1;
        u.seg[0] = GemmSeg{A, B, nbk};
        u.epi.mode = EPI_ACCUM;
        u.epi.alpha = -1.f;
        u.epi.out = chol + lrow(p_start) * m + p0 + nbk;
        u.epi.ld = m;
        u.lower_only = (p_start - k - 1) * NBO + 1;
        u.cyc_nb = NBO;
        u.cyc_skip = (W - 1) * NBO;
        u.max_ctas = max_ctas;
        gemm(ctx, u);
      };
      const int nmine = (int)((np - 1 - pf) / W) + 1;  // my panels from pf on
      if (pf == k + 1) {  // I own the next panel: its diagonal block first, then its factorization beside the rest
        update(pf, 1, 0);
        if (nmine > 1 && ctx->sm_count > 4 * kReserveSMs) {
          cudaStream_t side = side_fork(ctx);
          diag(pf, side);
          ahead = pf;
          update(pf + W, nmine - 1, ctx->sm_count - kReserveSMs);
          side_join(ctx);
        } else if (nmine > 1) {
          update(pf + W, nmine - 1, 0);
        }
      } else {
        update(pf, nmine, 0);
      }
    }
    // not positive definite anywhere -> everywhere
    double* fl = vecs + 6 * m;
    launch_k(st, k_flag_d, 1, 1, 0, (const int*)flag, fl);
    allreduce_f64(ctx, fl, 1);
    double hflag = 0.0;
    cudaMemcpyAsync(&hflag, fl, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (hflag != 0.0) {
      rc = 1;
    } else {
      double *r = vecs, *y = vecs + m, *v = vecs + 2 * m, *dv = vecs + 3 * m, *z = vecs + 4 * m, *t = vecs + 5 * m;
      double* part = (double*)get(sizeof(double) * (size_t)(CD_SLICES * m));
      auto tri_solve = [&](double* x) {  // r -> x = (L L^T)^-1 r, r consumed
        for (int k = 0; k < np; ++k) {
          const int64_t p0 = (int64_t)k * NBO;
          const int nbk = prow(k);
          if (mine(k)) {
            if (k > 0)
              launch_k(st, k_row_dot, nbk, 256, 0, (const float*)(chol + lrow(k) * m), m, p0, (int64_t)-1,
                       (const double*)y, -1.0, r + p0, (const int*)nullptr);
            launch_k(st, k_tri_wgemv, (nbk + 7) / 8, 256, 0, (const float*)(winv + (int64_t)k * NBO * NBO), nbk,
                     (int)p0, (const double*)r, y);
            ctx->launches += 2;
          }
          broadcast(ctx, y + p0, nbk, CV_DTYPE_F64, owner(k));
        }
        cudaMemsetAsync(z, 0, sizeof(double) * m, st);
        for (int k = np - 1; k >= 0; --k) {
          const int64_t p0 = (int64_t)k * NBO;
          const int nbk = prow(k);
          allreduce_f64(ctx, z + p0, nbk);
          launch_k(st, k_sub_d, (nbk + 255) / 256, 256, 0, (const double*)(y + p0), (const double*)(z + p0), nbk, t);
          launch_k(st, k_tri_wtgemv, (nbk + 7) / 8, 256, 0, (const float*)(winvT + (int64_t)k * NBO * NBO), nbk,
                   (int)p0, (const double*)t, x);
          ctx->launches += 2;
          if (mine(k) && k > 0) col_dot(ctx, chol + lrow(k) * m, m, nbk, p0, 0, 0, x + p0, z, part, nullptr);
        }
      };
      launch_k(st, k_f2d, 256, 256, 0, rhs, r, m);
      tri_solve(v);
      for (int it = 0; it < 2; ++it) {
        strips_gv(ctx, strips, m, v, z, part, nullptr);  // z = Gram v
        launch_k(st, k_res_from, 256, 256, 0, rhs, (const double*)z, (const double*)v, mu, m, r);
        tri_solve(dv);
        launch_k(st, k_axpy_d, 256, 256, 0, (const double*)dv, v, m);
        ctx->launches += 2;
      }
      launch_k(st, k_d2f, 256, 256, 0, (const double*)v, v_out, m);
      ctx->launches += 2;
    }
  } catch (...) {
    for (void* q : bufs) pool.put(q);
    throw;
  }
  for (void* q : bufs) pool.put(q);
  return rc;
}

}  // namespace cv
