// Row-space lane: per-example H_z roots, Gram of the seeded Jacobian rows,
// blocked Cholesky of (Gram + mu I), triangular solves and backprojection.
//   seeds / rhs        curvature.py:112-119, models.py:206-239
//   Gram               models.py:309-334 (layer-wise, the m x d row matrix never exists)
//   Cholesky + solve   solvers.py:146-161 (LAPACK potrf/potrs in the reference)
//   backprojection     curvature.py:53-60
#include "common.cuh"
#include "internal.h"

#include <stdexcept>
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

static Operand f32op(const float* p, int64_t si, int64_t sj) {
  Operand o;
  o.f32 = p;
  o.si = si;
  o.sj = sj;
  return o;
}

static void ensure_gram(cv_ctx* ctx, cv_snap* s) {
  if (s->row_state & 2) return;
  ensure_seeds(ctx, s);
  const int b = s->bl, c = s->c, L = s->L;
  const int64_t m = (int64_t)b * c;
  if (!s->gram) s->gram = snap_alloc(s, m * m);
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
    gemm(ctx, h);
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
      q.seg[0] = GemmSeg{sop(D[cur], false), wt, nout};
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
  s->row_state |= 2;
}

void row_gram(cv_ctx* ctx, cv_snap* s, float* gram_out) {
  ensure_gram(ctx, s);
  const int64_t m = (int64_t)s->bl * s->c;
  if (gram_out) cudaMemcpyAsync(gram_out, s->gram, sizeof(float) * m * m, cudaMemcpyDeviceToDevice, ctx->stream);
}

// ---------------------------------------------------------------------------
// Blocked right-looking Cholesky, lower, in place on chol = gram + mu I.
// ---------------------------------------------------------------------------
__global__ void k_copy_add_diag(const float* src, float* dst, int64_t m, float mu) {
  CV_PDL_ENTRY();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * m; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / m, j = e - i * m;
    dst[e] = src[e] + (i == j ? mu : 0.f);
  }
}

// Factor the nb x nb diagonal block at j0 in fp64 shared memory, write L11 back
// and its inverse (fp32) into dinv[blk]; flag <- 1 if not positive definite.
__global__ void __launch_bounds__(256) k_potrf_diag(float* A, int64_t lda, int j0, int nb, float* dinv_blk,
                                                    int* flag) {
  CV_PDL_ENTRY();
  __shared__ double T[CH_NB][CH_NB + 1];
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    T[i][j] = j <= i ? (double)A[(int64_t)(j0 + i) * lda + j0 + j] : 0.0;
  }
  __syncthreads();
  for (int k = 0; k < nb; ++k) {
    if (tid == 0) {
      const double dkk = T[k][k];
      if (!(dkk > 0.0) || !isfinite(dkk)) { bad = 1; T[k][k] = 1.0; }
      else T[k][k] = sqrt(dkk);
    }
    __syncthreads();
    const double dk = T[k][k];
    for (int i = k + 1 + tid; i < nb; i += blockDim.x) T[i][k] /= dk;
    __syncthreads();
    for (int e = tid; e < (nb - k - 1) * (nb - k - 1); e += blockDim.x) {
      const int i = k + 1 + e / (nb - k - 1), j = k + 1 + e % (nb - k - 1);
      if (j <= i) T[i][j] -= T[i][k] * T[j][k];
    }
    __syncthreads();
  }
  // inverse of the lower-triangular factor, one column per thread
  // (column j of the inverse lives in dinv_blk[:, j]; only its own thread touches it)
  for (int j = tid; j < nb; j += blockDim.x) {
    double xc[CH_NB];
    for (int i = 0; i < nb; ++i) {
      if (i < j) { xc[i] = 0.0; dinv_blk[i * nb + j] = 0.f; continue; }
      double s = i == j ? 1.0 : 0.0;
      for (int k = j; k < i; ++k) s -= T[i][k] * xc[k];
      xc[i] = s / T[i][i];
      dinv_blk[i * nb + j] = (float)xc[i];
    }
  }
  __syncthreads();
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    if (j <= i) A[(int64_t)(j0 + i) * lda + j0 + j] = (float)T[i][j];
  }
  if (tid == 0 && bad) *flag = 1;
}

// forward substitution, one diagonal block: y_blk = Dinv (r_blk) ; then
// r[j0+nb:] -= L[j0+nb:, blk] y_blk    (r, y in fp64)
__global__ void k_trsv_fwd_diag(const float* dinv, int nb, int j0, double* r, double* y) {
  CV_PDL_ENTRY();
  __shared__ double rb[CH_NB];
  const int t = threadIdx.x;
  if (t < nb) rb[t] = r[j0 + t];
  __syncthreads();
  if (t < nb) {
    double s = 0.0;
    for (int k = 0; k <= t; ++k) s += (double)dinv[t * nb + k] * rb[k];
    y[j0 + t] = s;
  }
}
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
__global__ void k_trsv_bwd_diag(const float* dinv, int nb, int j0, const double* y, const double* partial,
                                int nparts, double* v) {
  CV_PDL_ENTRY();
  __shared__ double rb[CH_NB];
  const int t = threadIdx.x;
  if (t < nb) {
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += partial[p * nb + t];
    rb[t] = y[j0 + t] - s;
  }
  __syncthreads();
  if (t < nb) {
    double s = 0.0;
    for (int k = t; k < nb; ++k) s += (double)dinv[k * nb + t] * rb[k];  // Dinv^T
    v[j0 + t] = s;
  }
}
// Panel forms of the two substitutions (TS_NB = 512 columns = 8 diagonal 64-blocks per
// launch): one CTA walks the panel's 64-blocks with their precomputed inverses (fp64
// right-hand sides in shared memory), so a triangular solve is 2 x m/512 dependent
// launches instead of 4 x m/64.
constexpr int TS_NB = 512;

// forward: y[j0 : j0+nbp] from r (the panel rows of r are consumed in smem)
__global__ void __launch_bounds__(TS_NB) k_trsv_fwd_panel(const float* A, int64_t lda, const float* dinv, int j0,
                                                          int nbp, const double* r, double* y) {
  CV_PDL_ENTRY();
  __shared__ double rb[TS_NB];
  __shared__ double yb[CH_NB];
  const int t = threadIdx.x;
  if (t < nbp) rb[t] = r[j0 + t];
  __syncthreads();
  for (int s0 = 0; s0 < nbp; s0 += CH_NB) {
    const int nb = nbp - s0 < CH_NB ? nbp - s0 : CH_NB;
    const float* D = dinv + (int64_t)((j0 + s0) / CH_NB) * CH_NB * CH_NB;
    if (t < nb) {
      double acc = 0.0;
      for (int k = 0; k <= t; ++k) acc += (double)D[t * nb + k] * rb[s0 + k];
      yb[t] = acc;
      y[j0 + s0 + t] = acc;
    }
    __syncthreads();
    // later rows of the panel: rb[i] -= L[i, s0 : s0+nb] yb
    const int i = s0 + nb + t;
    if (i < nbp) {
      const float* Li = A + (int64_t)(j0 + i) * lda + j0 + s0;
      double acc = 0.0;
      for (int k = 0; k < nb; ++k) acc += (double)Li[k] * yb[k];
      rb[i] -= acc;
    }
    __syncthreads();
  }
}

// backward: v[j0 : j0+nbp] from y and the gathered partials L[below, panel]^T v[below]
__global__ void __launch_bounds__(TS_NB) k_trsv_bwd_panel(const float* A, int64_t lda, const float* dinv, int j0,
                                                          int nbp, const double* y, const double* partial, int nparts,
                                                          double* v) {
  CV_PDL_ENTRY();
  __shared__ double rb[TS_NB];
  __shared__ double xb[TS_NB];
  __shared__ double red[8][CH_NB];
  const int t = threadIdx.x;
  if (t < nbp) {
    double acc = 0.0;
    for (int p = 0; p < nparts; ++p) acc += partial[(int64_t)p * nbp + t];
    rb[t] = y[j0 + t] - acc;
  }
  __syncthreads();
  const int nsub = (nbp + CH_NB - 1) / CH_NB;
  for (int sb = nsub - 1; sb >= 0; --sb) {
    const int s0 = sb * CH_NB;
    const int nb = nbp - s0 < CH_NB ? nbp - s0 : CH_NB;
    // rb[s0 + k] -= sum over the panel's later rows i of L[i, s0 + k] x[i]  (8 row groups)
    const int k = t & (CH_NB - 1), grp = t / CH_NB;
    double acc = 0.0;
    if (k < nb)
      for (int i = s0 + nb + grp; i < nbp; i += 8) acc += (double)A[(int64_t)(j0 + i) * lda + j0 + s0 + k] * xb[i];
    red[grp][k] = acc;
    __syncthreads();
    if (t < nb) {
      double s = rb[s0 + t];
      for (int g2 = 0; g2 < 8; ++g2) s -= red[g2][t];
      rb[s0 + t] = s;
    }
    __syncthreads();
    const float* D = dinv + (int64_t)((j0 + s0) / CH_NB) * CH_NB * CH_NB;
    if (t < nb) {
      double s = 0.0;
      for (int kk = t; kk < nb; ++kk) s += (double)D[kk * nb + t] * rb[s0 + kk];  // Dinv^T
      xb[s0 + t] = s;
      v[j0 + s0 + t] = s;
    }
    __syncthreads();
  }
}

// r = rhs - (G + mu I) v, one warp per row, fp64 accumulation (refinement residual)
__global__ void k_row_residual(const float* G, int64_t m, float mu, const float* rhs, const double* v, double* r) {
  CV_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= m) return;
  const float* g = G + row * m;
  const bool vec = (m & 3) == 0;
  double s = 0.0;
  for (int64_t k = lane * 4; k < m; k += 128) {
    if (vec && k + 3 < m) {
      const float4 q = *reinterpret_cast<const float4*>(g + k);
      s += (double)q.x * v[k] + (double)q.y * v[k + 1] + (double)q.z * v[k + 2] + (double)q.w * v[k + 3];
    } else {
      for (int64_t t = k; t < k + 4 && t < m; ++t) s += (double)g[t] * v[t];
    }
  }
  s = warp_sum(s);
  if (lane == 0) r[row] = (double)rhs[row] - (s + (double)mu * v[row]);
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

int row_solve_cholesky(cv_ctx* ctx, cv_snap* s, double mu, const float* rhs, float* v_out) {
  ensure_gram(ctx, s);
  const int64_t m = (int64_t)s->bl * s->c;
  if (!s->chol) s->chol = snap_alloc(s, m * m);
  const int nblk = (int)((m + CH_NB - 1) / CH_NB);
  if (!s->dinv) s->dinv = snap_alloc(s, (int64_t)nblk * CH_NB * CH_NB);
  cudaStream_t st = ctx->stream;
  launch_k(st, k_copy_add_diag, 4096, 256, 0, s->gram, s->chol, m, (float)mu);
  int* flag = (int*)(ctx->scal_ws + 32);
  cudaMemsetAsync(flag, 0, sizeof(int), st);
  ctx->launches++;
  // Two-level right-looking blocked Cholesky: panels of CH_NBO columns are factored
  // with the 64-wide fp64 diagonal kernel, a SIMT triangular solve and SIMT updates
  // confined to the panel; the trailing matrix update A22 -= L21 L21^T of each panel
  // (all but O(m^2 CH_NBO) of the m^3/3 flops) runs on the tensor-core engine with L21
  // as a scaled fp16 pair.  The fp64 iterative refinement below absorbs the split's
  // rounding (cf. the 1e-6 lane-equivalence bound, tests/test_solvers.py:216-236).
  constexpr int NBO = 512;  // panel width (a multiple of CH_NB)
  const bool tc = ctx->engine != CV_ENGINE_SIMT && m > NBO;
  __half* l21h = nullptr;
  __half* l21l = nullptr;
  if (tc) {
    l21h = (__half*)ctx->pool.get(sizeof(__half) * (size_t)(m - NBO) * NBO);
    l21l = (__half*)ctx->pool.get(sizeof(__half) * (size_t)(m - NBO) * NBO);
  }
  Scale* l21sc = s->scratch_sc + 2;
  for (int64_t p0 = 0; p0 < m; p0 += NBO) {
    const int nbo = (int)((m - p0) < NBO ? (m - p0) : NBO);
    const int64_t pend = tc ? p0 + nbo : m;  // columns the in-panel updates cover
    for (int64_t j0 = p0; j0 < p0 + nbo; j0 += CH_NB) {
      const int bi = (int)(j0 / CH_NB);
      const int nb = (int)((m - j0) < CH_NB ? (m - j0) : CH_NB);
      float* dblk = s->dinv + (int64_t)bi * CH_NB * CH_NB;
      launch_k(st, k_potrf_diag, 1, 256, 0, s->chol, m, (int)j0, nb, dblk, flag);
      ctx->launches++;
      const int rest = (int)(m - j0 - nb);
      if (rest <= 0) continue;
      float* A21 = s->chol + (int64_t)(j0 + nb) * m + j0;
      // A21 <- A21 * L11^-T
      GemmArgs p;
      p.M = rest;
      p.N = nb;
      p.nseg = 1;
      p.seg[0] = GemmSeg{f32op(A21, m, 1), f32op(dblk, 1, nb), nb};
      p.epi.mode = EPI_STORE;
      p.epi.out = A21;
      p.epi.ld = m;
      gemm_simt(ctx, p);  // in place: one N tile per CTA row block
      // A22 -= A21 A21^T, columns [j0+nb, pend) (lower part)
      const int ncols = (int)(pend - j0 - nb);
      if (ncols <= 0) continue;
      GemmArgs u;
      u.M = rest;
      u.N = ncols;
      u.nseg = 1;
      u.seg[0] = GemmSeg{f32op(A21, m, 1), f32op(A21, 1, m), nb};
      u.epi.mode = EPI_ACCUM;
      u.epi.alpha = -1.f;
      u.epi.out = s->chol + (int64_t)(j0 + nb) * m + (j0 + nb);
      u.epi.ld = m;
      u.lower_only = 1;
      gemm_simt(ctx, u);
    }
    const int rest2 = (int)(m - p0 - nbo);
    if (!tc || rest2 <= 0) continue;
    // trailing update of the whole remaining matrix on the tensor cores
    split_mat(ctx, s->chol + (p0 + nbo) * m + p0, m, rest2, nbo, l21h, l21l, nbo, 0, l21sc, 0, nullptr);
    Operand A, B;
    A.hi = l21h; A.lo = l21l; A.sc = l21sc; A.si = nbo; A.sj = 1;  // A(i, k) = L21[i, k]
    B.hi = l21h; B.lo = l21l; B.sc = l21sc; B.si = 1; B.sj = nbo;  // B(k, j) = L21[j, k]
    GemmArgs u;
    u.M = rest2;
    u.N = rest2;
    u.nseg = 1;
    u.seg[0] = GemmSeg{A, B, nbo};
    u.epi.mode = EPI_ACCUM;
    u.epi.alpha = -1.f;
    u.epi.out = s->chol + (p0 + nbo) * m + (p0 + nbo);
    u.epi.ld = m;
    u.lower_only = 1;
    gemm(ctx, u);
  }
  if (tc) {
    ctx->pool.put(l21h);
    ctx->pool.put(l21l);
  }
  int hflag = 0;
  cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  if (hflag) return 1;
  // fp64 triangular solves, then iterative refinement against the fp32 Gram:
  // v <- v + (L L^T)^-1 (rhs - (Gram + mu I) v), residual accumulated in fp64
  double* r = (double*)ctx->pool.get(sizeof(double) * m * 4);
  double* y = r + m;
  double* v = r + 2 * m;
  double* dv = r + 3 * m;
  const int rpb = 64;
  const int nparts_max = (int)((m + rpb - 1) / rpb);
  double* part = (double*)ctx->pool.get(sizeof(double) * (size_t)nparts_max * TS_NB);
  auto tri_solve = [&](double* x) {  // r -> x = (L L^T)^-1 r   (r is consumed)
    const int npan = (int)((m + TS_NB - 1) / TS_NB);
    for (int pi = 0; pi < npan; ++pi) {
      const int j0 = pi * TS_NB;
      const int nbp = (int)((m - j0) < TS_NB ? (m - j0) : TS_NB);
      launch_k(st, k_trsv_fwd_panel, 1, TS_NB, 0, (const float*)s->chol, m, (const float*)s->dinv, j0, nbp,
               (const double*)r, y);
      const int64_t rest = m - j0 - nbp;
      if (rest > 0) launch_k(st, k_trsv_fwd_update, (int)((rest + 7) / 8), 256, 0, s->chol, m, m, j0, nbp, y, r);
    }
    for (int pi = npan - 1; pi >= 0; --pi) {
      const int j0 = pi * TS_NB;
      const int nbp = (int)((m - j0) < TS_NB ? (m - j0) : TS_NB);
      const int64_t rest = m - j0 - nbp;
      const int nparts = (int)((rest + rpb - 1) / rpb);
      if (nparts > 0) launch_k(st, k_trsv_bwd_gather, nparts, TS_NB, 0, s->chol, m, m, j0, nbp, x, part, rpb);
      launch_k(st, k_trsv_bwd_panel, 1, TS_NB, 0, (const float*)s->chol, m, (const float*)s->dinv, j0, nbp,
               (const double*)y, (const double*)part, nparts, x);
    }
    ctx->launches += 4 * npan;
  };
  launch_k(st, k_f2d, 256, 256, 0, rhs, r, m);
  tri_solve(v);
  for (int it = 0; it < 2; ++it) {
    launch_k(st, k_row_residual, (int)((m + 7) / 8), 256, 0, s->gram, m, (float)mu, rhs, v, r);
    tri_solve(dv);
    launch_k(st, k_axpy_d, 256, 256, 0, dv, v, m);
    ctx->launches += 2;
  }
  launch_k(st, k_d2f, 256, 256, 0, v, v_out, m);
  ctx->launches += 2;
  ctx->pool.put(part);
  ctx->pool.put(r);
  return 0;
}

void row_backproject(cv_ctx* ctx, cv_snap* s, const float* v, float* out) {
  ensure_seeds(ctx, s);
  const int64_t m = (int64_t)s->bl * s->c;
  launch_k(ctx->stream, k_seed_apply, (int)((m + 255) / 256), 256, 0, s->seeds, v, s->bl, s->c, s->U2);
  ctx->launches++;
  mlp_vjp(ctx, s, s->U2, out);
}

}  // namespace cv
