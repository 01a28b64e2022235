// Scaled fp16 splits (common.cuh) of fp32 inputs, with the exact amax.
//
// Each split is two launches: an amax pass whose last block to finish reduces
// the per-block maxima and publishes {e, amax} into the tensor's Scale slot
// (max is order independent, so the result is deterministic), then the split
// pass.  Used for everything whose scale cannot come from a GEMM bound: the
// product inputs (CG directions, probes, loss_at points), the input batch, the
// weights, and the c-wide cotangents of the output layer.
#include "common.cuh"
#include "internal.h"

namespace cv {

constexpr int SP_NB = 4 * 148, SP_NT = 256, SP_MAXL = kOffTabMax;  // grid: 16 B x 151K threads in flight per stream

CV_DEV float block_max(float v, float* sh) {
  v = warp_max_f(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float r = 0.f;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.f;
    r = warp_max_f(r);
  }
  return r;  // valid in thread 0
}

// last block of the grid? (after every block wrote its partials)
CV_DEV bool last_block(unsigned* counter) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  return last;
}

// block maxima -> part; the grid's last block reduces them and publishes sc[l]
// (and zeroes the zero_sc block of Scale slots).
CV_DEV void flat_amax_finish(const OffTab& t, int* smax, float* sh, float* part, unsigned* counter, Scale* sc,
                             Scale* zero_sc, int n_zero) {
  __syncthreads();
  if (threadIdx.x < t.L) part[blockIdx.x * SP_MAXL + threadIdx.x] = __int_as_float(smax[threadIdx.x]);
  if (!last_block(counter)) return;
  for (int l2 = 0; l2 < t.L; ++l2) {
    float mm = 0.f;
    for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) mm = fmaxf(mm, __ldcg(part + b * SP_MAXL + l2));
    mm = block_max(mm, sh);
    if (threadIdx.x == 0) {
      sc[l2].amax = mm;
      sc[l2].e = exp_for_bound(mm);
    }
  }
  for (int i = threadIdx.x; i < n_zero; i += blockDim.x) {
    zero_sc[i].e = 0;
    zero_sc[i].amax = 0.f;
  }
  if (threadIdx.x == 0) *counter = 0;
}

// per-layer amax of a flat vector; the last block publishes sc[l] and zeroes zero_sc.
// One grid-stride pass of 128-bit loads; a thread's indices only increase, so it
// tracks its current layer and folds the running max into shared memory when the
// layer changes (at most L times).
__global__ void __launch_bounds__(SP_NT) k_flat_amax(const float* __restrict__ x, OffTab t, float* part,
                                                     unsigned* counter, Scale* sc, Scale* zero_sc, int n_zero,
                                                     const int* skip) {
  CV_PDL_ENTRY();
  if (skip_if(skip)) return;
  __shared__ float sh[SP_NT / 32];
  __shared__ int smax[SP_MAXL];
  if (threadIdx.x < SP_MAXL) smax[threadIdx.x] = 0;
  __syncthreads();
  const int64_t d = t.off[t.L], base = t.off[0];
  const int64_t n = d - base;
  const int64_t lead = ((base + 3) & ~(int64_t)3) - base;  // elements before the first 16-byte boundary
  int l = 0;
  float m = 0.f;
  auto take = [&](int64_t i, float v) {
    if (i >= t.off[l + 1]) {
      atomicMax(&smax[l], __float_as_int(m));
      m = 0.f;
      while (i >= t.off[l + 1]) ++l;
    }
    m = fmaxf(m, fabsf(v));
  };
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = base + tid; i < base + (lead < n ? lead : n); i += nth) take(i, x[i]);
  const int64_t q0 = (base + lead) / 4, q1 = (base + n) / 4;
  int64_t q = q0 + tid;
  // four 16-byte loads in flight per thread (one left HBM at half its bandwidth)
  for (; q + 3 * nth < q1; q += 4 * nth) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const float4*>(x + 4 * (q + u * nth));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = 4 * (q + u * nth);
      take(i, v[u].x);
      take(i + 1, v[u].y);
      take(i + 2, v[u].z);
      take(i + 3, v[u].w);
    }
  }
  for (; q < q1; q += nth) {
    const float4 v = *reinterpret_cast<const float4*>(x + 4 * q);
    take(4 * q, v.x);
    take(4 * q + 1, v.y);
    take(4 * q + 2, v.z);
    take(4 * q + 3, v.w);
  }
  for (int64_t i = (q1 * 4 > base + lead ? q1 * 4 : base + lead) + tid; i < d; i += nth) take(i, x[i]);
  atomicMax(&smax[l], __float_as_int(m));
  flat_amax_finish(t, smax, sh, part, counter, sc, zero_sc, n_zero);
}

// CG direction update fused with the per-layer amax of the next product input:
// p = M^-1 r + beta p (solvers.py:111-112), then the last block publishes the
// scales (the product's split pass follows without its own amax pass).
__global__ void __launch_bounds__(SP_NT) k_cg_pnext_amax(const float* __restrict__ r, const float* __restrict__ pre,
                                                         float lam, float floor_, const double* beta_p,
                                                         const int* done, float* __restrict__ p, OffTab t,
                                                         float* part, unsigned* counter, Scale* sc, Scale* zero_sc,
                                                         int n_zero) {
  CV_PDL_ENTRY();
  if (*(volatile const int*)done) return;
  __shared__ float sh[SP_NT / 32];
  __shared__ int smax[SP_MAXL];
  if (threadIdx.x < SP_MAXL) smax[threadIdx.x] = 0;
  __syncthreads();
  const float beta = (float)*beta_p;
  const int64_t d = t.off[t.L];
  int l = 0;
  float m = 0.f;
  auto take = [&](int64_t i, float v) {
    if (i >= t.off[l + 1]) {
      atomicMax(&smax[l], __float_as_int(m));
      m = 0.f;
      while (i >= t.off[l + 1]) ++l;
    }
    m = fmaxf(m, fabsf(v));
  };
  auto minv = [&](int64_t i) { return pre ? 1.f / (fmaxf(pre[i], floor_) + lam) : 1.f; };
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t nq = d >> 2;
  const bool pre4 = pre && !((uintptr_t)pre & 15);
  for (int64_t q = tid; q < nq; q += nth) {
    const int64_t i = 4 * q;
    const float4 r4 = *reinterpret_cast<const float4*>(r + i);
    float4 p4 = *reinterpret_cast<const float4*>(p + i);
    float4 m4 = make_float4(1.f, 1.f, 1.f, 1.f);
    if (pre4) {
      m4 = *reinterpret_cast<const float4*>(pre + i);
      m4.x = 1.f / (fmaxf(m4.x, floor_) + lam);
      m4.y = 1.f / (fmaxf(m4.y, floor_) + lam);
      m4.z = 1.f / (fmaxf(m4.z, floor_) + lam);
      m4.w = 1.f / (fmaxf(m4.w, floor_) + lam);
    } else if (pre) {
      m4 = make_float4(minv(i), minv(i + 1), minv(i + 2), minv(i + 3));
    }
    p4.x = m4.x * r4.x + beta * p4.x;
    p4.y = m4.y * r4.y + beta * p4.y;
    p4.z = m4.z * r4.z + beta * p4.z;
    p4.w = m4.w * r4.w + beta * p4.w;
    *reinterpret_cast<float4*>(p + i) = p4;
    take(i, p4.x);
    take(i + 1, p4.y);
    take(i + 2, p4.z);
    take(i + 3, p4.w);
  }
  for (int64_t i = 4 * nq + tid; i < d; i += nth) {
    const float v = minv(i) * r[i] + beta * p[i];
    p[i] = v;
    take(i, v);
  }
  atomicMax(&smax[l], __float_as_int(m));
  flat_amax_finish(t, smax, sh, part, counter, sc, zero_sc, n_zero);
}


__global__ void __launch_bounds__(SP_NT) k_flat_split(const float* __restrict__ x, OffTab t, const Scale* sc,
                                                      __half* __restrict__ hi, __half* __restrict__ lo,
                                                      const int* skip) {
  CV_PDL_ENTRY();
  if (skip_if(skip)) return;
  for (int l = 0; l < t.L; ++l) {
    const float s = pow2f(sc[l].e);
    const int64_t b = t.off[l], e = t.off[l + 1];
    int64_t b8 = (b + 7) & ~(int64_t)7;  // 8-aligned body (16-byte half stores)
    if (b8 > e) b8 = e;
    const int64_t e8 = b8 + ((e - b8) & ~(int64_t)7);
    for (int64_t i = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (b8 < e ? b8 : e);
         i += (int64_t)gridDim.x * blockDim.x)
      split16(x[i], s, hi[i], lo[i]);
    for (int64_t q = b8 / 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < e8 / 8;
         q += (int64_t)gridDim.x * blockDim.x) {
      const float4 a = *reinterpret_cast<const float4*>(x + 8 * q);
      const float4 c = *reinterpret_cast<const float4*>(x + 8 * q + 4);
      union { uint4 u; __half h[8]; } H, Lo;
      const float v[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) split16(v[k], s, H.h[k], Lo.h[k]);
      *reinterpret_cast<uint4*>(hi + 8 * q) = H.u;
      *reinterpret_cast<uint4*>(lo + 8 * q) = Lo.u;
    }
    for (int64_t i = (e8 > b8 ? e8 : b8) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e;
         i += (int64_t)gridDim.x * blockDim.x)
      if (i >= b8) split16(x[i], s, hi[i], lo[i]);
  }
}

static unsigned* counter_of(cv_ctx* ctx) { return ctx->amax_counter; }
static float* part_of(cv_ctx* ctx) { return ctx->amax_ws; }

void split_flat(cv_ctx* ctx, const float* x, int64_t d, const std::vector<int64_t>& off, __half* hi, __half* lo,
                Scale* sc, Scale* zero_sc, int n_zero, const int* skip) {
  const int L = (int)off.size();
  for (int l0 = 0; l0 < L; l0 += SP_MAXL) {
    OffTab t;
    t.L = L - l0 < SP_MAXL ? L - l0 : SP_MAXL;
    for (int l = 0; l <= t.L; ++l) t.off[l] = l0 + l < L ? off[l0 + l] : d;
    const bool last = l0 + t.L >= L;
    launch_k(ctx->stream, k_flat_amax, SP_NB, SP_NT, 0, x, t, part_of(ctx), counter_of(ctx), sc + l0,
                                                  last ? zero_sc : nullptr, last ? n_zero : 0, skip);
    launch_k(ctx->stream, k_flat_split, SP_NB, SP_NT, 0, x, t, sc + l0, hi, lo, skip);
    ctx->launches += 2;
  }
}

static OffTab off_tab(const std::vector<int64_t>& off, int64_t d) { return make_off_tab(off, d); }

// split pass only (the scales were published by a fused producer)
void split_flat_apply(cv_ctx* ctx, const float* x, int64_t d, const std::vector<int64_t>& off, __half* hi,
                      __half* lo, const Scale* sc, const int* skip) {
  launch_k(ctx->stream, k_flat_split, SP_NB, SP_NT, 0, x, off_tab(off, d), sc, hi, lo, skip);
  ctx->launches++;
}

bool cg_pnext_amax(cv_ctx* ctx, const float* r, const float* pre, float lam, float floor_, const double* beta,
                   const int* done, float* p, int64_t d, const std::vector<int64_t>& off, Scale* sc, Scale* zero_sc,
                   int n_zero) {
  if ((int)off.size() > SP_MAXL) return false;
  launch_k(ctx->stream, k_cg_pnext_amax, SP_NB, SP_NT, 0, r, pre, lam, floor_, beta, done, p, off_tab(off, d), part_of(ctx),
                                                    counter_of(ctx), sc, zero_sc, n_zero);
  ctx->launches++;
  return true;
}


// ---------------------------------------------------------------------------
// 2-D splits: [rows x cols] fp32 (ld lds) -> split (ld ldd), optionally
// transposed (dst[j, i]) and with a ones column at `cols` (augmented activations)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SP_NT) k_mat_amax(const float* __restrict__ x, int64_t lds, int rows, int cols,
                                                    float floor_, float* part, unsigned* counter, Scale* sc,
                                                    const int* skip) {
  CV_PDL_ENTRY();
  if (skip_if(skip)) return;
  __shared__ float sh[SP_NT / 32];
  // one warp per row, lanes over columns (128-bit when the rows are aligned)
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (lds & 3) == 0 && ((uintptr_t)x & 15) == 0;
  float m = 0.f;
  if (rows == 1) {  // flat vector: all threads over the columns
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t nq = vec ? cols / 4 : 0;
    for (int64_t q = tid; q < nq; q += nth) {
      const float4 v = *reinterpret_cast<const float4*>(x + 4 * q);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    for (int64_t i = 4 * nq + tid; i < cols; i += nth) m = fmaxf(m, fabsf(x[i]));
  } else {
    for (int64_t r = warp; r < rows; r += nwarps) {
      const float* row = x + r * lds;
      int c0 = 0;
      if (vec)
        for (; c0 + 128 <= cols; c0 += 128) {
          const float4 v = *reinterpret_cast<const float4*>(row + c0 + 4 * lane);
          m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        }
      for (int c = c0 + lane; c < cols; c += 32) m = fmaxf(m, fabsf(row[c]));
    }
  }
  m = block_max(m, sh);
  if (threadIdx.x == 0) part[blockIdx.x * SP_MAXL] = m;
  if (!last_block(counter)) return;
  m = 0.f;
  for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) m = fmaxf(m, __ldcg(part + b * SP_MAXL));
  m = block_max(m, sh);
  if (threadIdx.x == 0) {
    m = fmaxf(m, floor_);
    sc->amax = m;
    sc->e = exp_for_bound(m);
    *counter = 0;
  }
}

__global__ void __launch_bounds__(SP_NT) k_mat_split(const float* __restrict__ x, int64_t lds, int rows, int cols,
                                                     int out_rows, int out_cols, int trans, int ones,
                                                     Scale* sc, int from_amax, __half* __restrict__ hi,
                                                     __half* __restrict__ lo, int64_t ldd, const int* skip) {
  CV_PDL_ENTRY();
  if (skip_if(skip)) return;
  // from_amax: the producer accumulated max|x| in sc->amax; derive (and publish) e here
  const int e = from_amax ? exp_for_bound(sc->amax) : sc->e;
  if (from_amax && blockIdx.x == 0 && threadIdx.x == 0) sc->e = e;
  const float s = pow2f(e);
  if (trans) {  // few long destination rows (c-wide cotangents): flat over elements
    const int64_t total = (int64_t)out_rows * out_cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = i / out_cols, c = i - r * out_cols;
      const float v = (c < rows && r < cols) ? x[c * lds + r] : 0.f;
      split16(v, s, hi[r * ldd + c], lo[r * ldd + c]);
    }
    return;
  }
  // destination rows r (one warp each), lanes over columns c
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < out_rows; r += nwarps) {
    for (int64_t c = lane; c < out_cols; c += 32) {
      float v = 0.f;
      if (r < rows && c < cols) v = x[r * lds + c];
      else if (ones && r < rows && c == cols) v = 1.f;
      split16(v, s, hi[r * ldd + c], lo[r * ldd + c]);
    }
  }
}

static int grid_for(int64_t n) {
  int64_t g = (n + SP_NT - 1) / SP_NT;
  return (int)(g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g));
}

void amax_into(cv_ctx* ctx, const float* x, int64_t n, Scale* slot) {
  launch_k(ctx->stream, k_mat_amax, SP_NB, SP_NT, 0, x, n, 1, (int)n, 0.f, part_of(ctx), counter_of(ctx), slot, nullptr);
  ctx->launches++;
}

void split_rows(cv_ctx* ctx, const float* src, int64_t lds, int rows, int cols, const SplitBuf& dst, int ones) {
  launch_k(ctx->stream, k_mat_amax, SP_NB, SP_NT, 0, src, lds, rows, cols, ones ? 1.f : 0.f, part_of(ctx),
                                               counter_of(ctx), dst.sc, nullptr);
  const int oc = ones ? cols + 1 : cols;
  launch_k(ctx->stream, k_mat_split, grid_for((int64_t)rows * oc), SP_NT, 0, src, lds, rows, cols, rows, oc, 0, ones, dst.sc,
                                                                      0, dst.hi, dst.lo, dst.ld, nullptr);
  ctx->launches += 2;
}

// src rows x cols -> (trans ? cols_pad x ldd : rows x ldd) split; amax_ready: sc->amax
// already holds max|src| (accumulated by the producer)
void split_mat(cv_ctx* ctx, const float* src, int64_t lds, int rows, int cols, __half* hi, __half* lo, int64_t ldd,
               int trans, Scale* sc, int amax_ready, const int* skip, int pad_cols) {
  if (!amax_ready) {
    launch_k(ctx->stream, k_mat_amax, SP_NB, SP_NT, 0, src, lds, rows, cols, 0.f, part_of(ctx), counter_of(ctx), sc, skip);
    ctx->launches++;
  }
  const int orows = trans ? (int)((cols + 15) / 16 * 16) : rows;
  const int ocols = trans ? rows : (pad_cols > cols ? pad_cols : cols);  // zero columns up to pad_cols
  launch_k(ctx->stream, k_mat_split, grid_for((int64_t)orows * ocols), SP_NT, 0, src, lds, rows, cols, orows, ocols, trans, 0,
                                                                          sc, amax_ready, hi, lo, ldd, skip);
  ctx->launches++;
}

// column `col` of a split buffer := v (scaled by the buffer's exponent); amax covers |v|
__global__ void k_set_col(__half* hi, __half* lo, int64_t ld, int rows, int col, float v, Scale* sc) {
  CV_PDL_ENTRY();
  const float s = pow2f(sc->e);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
    split16(v, s, hi[(int64_t)r * ld + col], lo[(int64_t)r * ld + col]);
  if (blockIdx.x == 0 && threadIdx.x == 0) atomic_amax(&sc->amax, fabsf(v));
}

void set_col_value(cv_ctx* ctx, const SplitBuf& b, int rows, int col, float v) {
  launch_k(ctx->stream, k_set_col, grid_for(rows), SP_NT, 0, b.hi, b.lo, b.ld, rows, col, v, b.sc);
  ctx->launches++;
}

__global__ void k_gather_rows(const __half* hi, const __half* lo, int64_t ld, int rows, int cols, const Scale* sc,
                              float* out) {
  CV_PDL_ENTRY();
  const float inv = pow2f(-sc->e);
  const int64_t total = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    out[i] = join16(hi[r * ld + c], lo[r * ld + c], inv);
  }
}

void gather_rows(cv_ctx* ctx, const SplitBuf& b, int rows, int cols, float* out) {
  launch_k(ctx->stream, k_gather_rows, grid_for((int64_t)rows * cols), SP_NT, 0, b.hi, b.lo, b.ld, rows, cols, b.sc, out);
  ctx->launches++;
}

}  // namespace cv
