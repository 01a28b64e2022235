// Device-resident CG/PCG, SplitMix64 probes, Hutchinson estimators, EMA and the
// step-tail vector kernels.  Every d-length pass is a grid-stride loop over a fixed
// grid (kRedBlocks x 256) whose fp64 block partials are summed in a fixed order,
// so all scalars are bitwise reproducible run to run.
#include "common.cuh"
#include "internal.h"
#include "vecutil.cuh"
#include "epilogue.cuh"

#include <algorithm>
#include <float.h>
#include <functional>
#include <stdlib.h>

#include <type_traits>

namespace cv {

__global__ void k_rademacher(uint64_t seed, uint64_t counter, int64_t n, float scale, float* out) {
  CV_PDL_ENTRY();
  vec_for(n, al16p(out), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    Vf<W> o;
#pragma unroll
    for (int j = 0; j < W; ++j) o.v[j] = rad(seed, counter, i + j) * scale;
    stv<W>(out + i, o);
  });
}

void rademacher(cv_ctx* ctx, uint64_t seed, uint64_t counter, int64_t n, float* out) {
  launch_k(ctx->stream, k_rademacher, NB, NT, 0, seed, counter, n, 1.f, out);
  ctx->launches++;
}

// ---------------------------------------------------------------------------
// small scalar utilities
// ---------------------------------------------------------------------------
__global__ void k_scale_scalar(double* x, double s) {
  CV_PDL_ENTRY(); *x *= s; }
void scale_scalar(cv_ctx* ctx, double* x, double s) {
  launch_k(ctx->stream, k_scale_scalar, 1, 1, 0, x, s);
  ctx->launches++;
}

__global__ void k_dot(const float* a, const float* b, int64_t n, double* ws) {
  CV_PDL_ENTRY();
  double t[1] = {0.0};
  vec_for(n, al16p(a, b), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    const Vf<W> x = ldv<W>(a + i), y = ldv<W>(b + i);
#pragma unroll
    for (int j = 0; j < W; ++j) t[0] += (double)x.v[j] * (double)y.v[j];
  });
  write_partials<1>(ws, t);
}
__global__ void k_dot_final(const double* ws, double* out) {
  CV_PDL_ENTRY();
  double t[1];
  sum_partials<1>(ws, t);
  if (threadIdx.x == 0) *out = t[0];
}
void dot_into(cv_ctx* ctx, const float* a, const float* b, int64_t n, double* out) {
  launch_k(ctx->stream, k_dot, NB, NT, 0, a, b, n, ctx->red_ws);
  launch_k(ctx->stream, k_dot_final, 1, NT, 0, ctx->red_ws, out);
  ctx->launches += 2;
}

// update = coef*dir; w_next = w + update; scal = [||update||, #nonfinite, ||dir||^2]
// (method.py:345-357; the all-`scale` chain collapses to one coefficient)
__global__ void k_apply_update(const float* w, const float* dir, float coef, int64_t d, float* upd, float* wn,
                               double* ws) {
  CV_PDL_ENTRY();
  double t[3] = {0.0, 0.0, 0.0};
  vec_for(d, al16p(w, dir, upd, wn), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    const Vf<W> dv = ldv<W>(dir + i), wv = ldv<W>(w + i);
    Vf<W> uv, xv;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const float di = dv.v[j];
      const float u = di * coef;
      const float x = wv.v[j] + u;
      uv.v[j] = u;
      xv.v[j] = x;
      t[0] += (double)u * u;
      t[1] += (!isfinite(di) || !isfinite(u) || !isfinite(x)) ? 1.0 : 0.0;
      t[2] += (double)di * di;
    }
    stv<W>(upd + i, uv);
    stv<W>(wn + i, xv);
  });
  write_partials<3>(ws, t);
}
__global__ void k_apply_update_final(const double* ws, double* scal) {
  CV_PDL_ENTRY();
  double t[3];
  sum_partials<3>(ws, t);
  if (threadIdx.x == 0) { scal[0] = sqrt(t[0]); scal[1] = t[1]; scal[2] = t[2]; }
}
void apply_update(cv_ctx* ctx, const float* w, const float* dir, double coef, int64_t d, float* upd, float* wn,
                  double* scal) {
  launch_k(ctx->stream, k_apply_update, NB, NT, 0, w, dir, (float)coef, d, upd, wn, ctx->red_ws);
  launch_k(ctx->stream, k_apply_update_final, 1, NT, 0, ctx->red_ws, scal);
  ctx->launches += 2;
}

__global__ void k_norm_check(const float* x, int64_t d, double* ws) {
  CV_PDL_ENTRY();
  double t[2] = {0.0, 0.0};
  vec_for(d, al16p(x), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    const Vf<W> xv = ldv<W>(x + i);
#pragma unroll
    for (int j = 0; j < W; ++j) {
      t[0] += (double)xv.v[j] * xv.v[j];
      t[1] += isfinite(xv.v[j]) ? 0.0 : 1.0;
    }
  });
  write_partials<2>(ws, t);
}
__global__ void k_norm_check_final(const double* ws, double* scal) {
  CV_PDL_ENTRY();
  double t[2];
  sum_partials<2>(ws, t);
  if (threadIdx.x == 0) { scal[0] = t[0]; scal[1] = t[1]; }
}
void norm_check(cv_ctx* ctx, const float* x, int64_t d, double* scal) {
  launch_k(ctx->stream, k_norm_check, NB, NT, 0, x, d, ctx->red_ws);
  launch_k(ctx->stream, k_norm_check_final, 1, NT, 0, ctx->red_ws, scal);
  ctx->launches += 2;
}

// diag EMA (control.py:70-77) / floored store (method.py:407-408) + mean (method.py:409)
__global__ void k_diag_ema(float* diag, const float* est, float beta, int64_t d, int mode, double* ws) {
  CV_PDL_ENTRY();
  double t[1] = {0.0};
  vec_for(d, al16p(diag, est), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    const Vf<W> ev = ldv<W>(est + i);
    Vf<W> dv = ldv<W>(diag + i);
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const float e = ev.v[j];
      const float v = mode == 0 ? fmaxf(beta * dv.v[j] + (1.f - beta) * e, 0.f) : fmaxf(e, 0.f);
      dv.v[j] = v;
      t[0] += v;
    }
    stv<W>(diag + i, dv);
  });
  write_partials<1>(ws, t);
}
__global__ void k_mean_final(const double* ws, double inv_n, double* out) {
  CV_PDL_ENTRY();
  double t[1];
  sum_partials<1>(ws, t);
  if (threadIdx.x == 0) *out = t[0] * inv_n;
}
void diag_ema(cv_ctx* ctx, float* diag, const float* est, double beta, int64_t d, int mode, double* mean) {
  launch_k(ctx->stream, k_diag_ema, NB, NT, 0, diag, est, (float)beta, d, mode, ctx->red_ws);
  ctx->launches++;
  if (mean) {
    launch_k(ctx->stream, k_mean_final, 1, NT, 0, ctx->red_ws, 1.0 / (double)d, mean);
    ctx->launches++;
  }
}

// ---------------------------------------------------------------------------
// Hutchinson (telemetry.py:91-110): z regenerated from (seed, counter) in the
// accumulation pass instead of being re-read.
// ---------------------------------------------------------------------------
// A Rademacher probe (numeric.py:157-162) written straight as the product input's split:
// z_i = +-1 is exact in the fp16 pair (hi = z 2^e, lo = 0, e = exp_for_bound(1), every
// layer block's amax = 1: what the amax + split passes of an fp32 z would produce,
// bit for bit); the signs are kept as packed bits for the accumulation pass, and fp32
// values only for the output-layer block (the fused head and the bias row read those).
// One thread per 32-element word.
__global__ void k_rad_split(uint64_t seed, uint64_t counter, int64_t d, int64_t last_off, __half* hi, __half* lo,
                            uint32_t* bits, float* zf, Scale* v_sc, int L, Scale* zero_sc, int n_zero) {
  CV_PDL_ENTRY();
  const int e = exp_for_bound(1.f);
  if (blockIdx.x == 0) {
    if (threadIdx.x < L) { v_sc[threadIdx.x].e = e; v_sc[threadIdx.x].amax = 1.f; }
    if (threadIdx.x < n_zero) { zero_sc[threadIdx.x].e = 0; zero_sc[threadIdx.x].amax = 0.f; }
  }
  const __half hp = __float2half_rn(pow2f(e)), hn = __float2half_rn(-pow2f(e)), hz = __float2half_rn(0.f);
  const int64_t words = (d + 31) / 32;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = 32 * w;
    uint32_t wd = 0;
    if (i0 + 32 <= d && !(i0 & 7)) {
      H8 h[4], z8;
#pragma unroll
      for (int j = 0; j < 8; ++j) z8.h[j] = hz;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool pos = (splitmix(seed, counter + 1 + (uint64_t)(i0 + j)) >> 63) != 0;
        wd |= (pos ? 1u : 0u) << j;
        h[j >> 3].h[j & 7] = pos ? hp : hn;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        *reinterpret_cast<uint4*>(hi + i0 + 8 * q) = h[q].u;
        *reinterpret_cast<uint4*>(lo + i0 + 8 * q) = z8.u;
      }
    } else {
      for (int j = 0; j < 32 && i0 + j < d; ++j) {
        const bool pos = (splitmix(seed, counter + 1 + (uint64_t)(i0 + j)) >> 63) != 0;
        wd |= (pos ? 1u : 0u) << j;
        hi[i0 + j] = pos ? hp : hn;
        lo[i0 + j] = hz;
      }
    }
    bits[w] = wd;
    if (i0 + 32 > last_off)
      for (int j = 0; j < 32 && i0 + j < d; ++j)
        if (i0 + j >= last_off) zf[i0 + j] = ((wd >> j) & 1u) ? 1.f : -1.f;
  }
}

// diag (+)= z * Hz / n with z from the probe's packed signs; partial sums of z.Hz
__global__ void k_hutch_acc_bits(const uint32_t* bits, const float* hz, int64_t d, float* diag, int first, int last,
                                 float inv_n, double* ws) {
  CV_PDL_ENTRY();
  double t[1] = {0.0};
  vec_for(d, al16p(hz, diag), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    const Vf<W> hv = ldv<W>(hz + i);
    Vf<W> dv;
    if (diag && !first) dv = ldv<W>(diag + i);
    // (W = 4 groups start at multiples of 4: their signs sit in one word)
    const uint32_t wd = __ldg(bits + (i >> 5)) >> (i & 31);
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const float zh = ((wd >> j) & 1u) ? hv.v[j] : -hv.v[j];
      t[0] += (double)zh;
      float a = first ? zh : dv.v[j] + zh;
      if (last) a *= inv_n;
      dv.v[j] = a;
    }
    if (diag) stv<W>(diag + i, dv);
  });
  write_partials<1>(ws, t);
}

__global__ void k_trace_final(const double* ws, double inv_n, double* out, int first) {
  CV_PDL_ENTRY();
  double t[1];
  sum_partials<1>(ws, t);
  if (threadIdx.x == 0) *out = (first ? 0.0 : *out) + t[0] * inv_n;
}

static float* snap_tmp(cv_snap* s, float** slot) {
  if (!*slot) {
    *slot = (float*)s->ctx->pool.get(sizeof(float) * s->d);
    s->owned.push_back(*slot);
  }
  return *slot;
}

void hutchinson(cv_ctx* ctx, cv_snap* s, int kind, uint64_t seed, uint64_t counter, int n_probes, float* diag,
                double* trace) {
  float* hz = snap_tmp(s, &s->tmp_d);
  float* z = snap_tmp(s, &s->tmp_d2);
  uint32_t* zbits = (uint32_t*)ctx->pool.get(sizeof(uint32_t) * (size_t)((s->d + 31) / 32));
  MatvecFn mv = matvec_fn(kind);
  const int64_t words = (s->d + 31) / 32;
  const int rgrid = (int)(words / NT + 1 < 8 * (int64_t)ctx->sm_count ? words / NT + 1 : 8 * (int64_t)ctx->sm_count);
  for (int j = 0; j < n_probes; ++j) {
    const uint64_t ctr = counter + (uint64_t)j * (uint64_t)s->d;
    // the probe goes straight into the product input's split (no fp32 probe pass)
    launch_k(ctx->stream, k_rad_split, rgrid, NT, 0, seed, ctr, s->d, s->off[s->L - 1], s->v_hi, s->v_lo, zbits, z,
             s->v_sc, s->L, s->prod_sc, s->n_prod);
    ctx->launches++;
    s->v_ready = 2;
    mv(ctx, s, z, hz, nullptr);
    launch_k(ctx->stream, k_hutch_acc_bits, NB, NT, 0, (const uint32_t*)zbits, (const float*)hz, s->d, diag, j == 0,
             j == n_probes - 1, 1.f / (float)n_probes, ctx->red_ws);
    ctx->launches++;
    if (trace) {
      launch_k(ctx->stream, k_trace_final, 1, NT, 0, ctx->red_ws, 1.0 / (double)n_probes, trace, j == 0);
      ctx->launches++;
    }
  }
  ctx->pool.put(zbits);  // stream-ordered reuse
}

// ---------------------------------------------------------------------------
// Power iteration (telemetry.py:113-126)
// ---------------------------------------------------------------------------
struct PiDev { double ray, result; int done; };

__global__ void k_pi_init(PiDev* st) {
  CV_PDL_ENTRY(); st->ray = 0.0; st->result = 0.0; st->done = 0; }
__global__ void k_pi_reduce(const float* v, const float* hv, int64_t d, double* ws, const int* skip) {
  CV_PDL_ENTRY();
  if (skip_if(skip)) return;
  double t[2] = {0.0, 0.0};
  vec_for(d, al16p(v, hv), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    const Vf<W> a = ldv<W>(v + i), h = ldv<W>(hv + i);
#pragma unroll
    for (int j = 0; j < W; ++j) {
      t[0] += (double)a.v[j] * h.v[j];
      t[1] += (double)h.v[j] * h.v[j];
    }
  });
  write_partials<2>(ws, t);
}
__global__ void k_pi_final(const double* ws, PiDev* st, double* norm_out) {
  CV_PDL_ENTRY();
  if (st->done) return;
  double t[2];
  sum_partials<2>(ws, t);
  if (threadIdx.x == 0) {
    const double nrm = sqrt(t[1]);
    st->ray = t[0];
    if (nrm == 0.0) { st->result = 0.0; st->done = 1; }
    else st->result = t[0];
    *norm_out = nrm;
  }
}
__global__ void k_pi_next(const float* hv, const double* nrm, int64_t d, float* v, const int* skip) {
  CV_PDL_ENTRY();
  if (skip_if(skip)) return;
  const double nr = *nrm;
  vec_for(d, al16p(hv, v), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    Vf<W> a = ldv<W>(hv + i);
#pragma unroll
    for (int j = 0; j < W; ++j) a.v[j] = (float)((double)a.v[j] / nr);
    stv<W>(v + i, a);
  });
}
__global__ void k_pi_out(const PiDev* st, double* out) {
  CV_PDL_ENTRY(); *out = st->result; }

void power_iter(cv_ctx* ctx, cv_snap* s, int kind, uint64_t seed, uint64_t counter, int iters, double* eig) {
  float* v = snap_tmp(s, &s->tmp_d);
  float* hv = snap_tmp(s, &s->tmp_d2);
  PiDev* st = (PiDev*)ctx->scal_ws;
  double* nrm = ctx->scal_ws + 4;
  launch_k(ctx->stream, k_pi_init, 1, 1, 0, st);
  const float scale = (float)(1.0 / sqrt((double)s->d));
  launch_k(ctx->stream, k_rademacher, NB, NT, 0, seed, counter, s->d, scale, v);
  ctx->launches += 2;
  MatvecFn mv = matvec_fn(kind);
  for (int it = 0; it < iters; ++it) {
    mv(ctx, s, v, hv, &st->done);
    launch_k(ctx->stream, k_pi_reduce, NB, NT, 0, v, hv, s->d, ctx->red_ws, &st->done);
    launch_k(ctx->stream, k_pi_final, 1, NT, 0, ctx->red_ws, st, nrm);
    launch_k(ctx->stream, k_pi_next, NB, NT, 0, hv, nrm, s->d, v, &st->done);
    ctx->launches += 3;
  }
  launch_k(ctx->stream, k_pi_out, 1, 1, 0, st, eig);
  ctx->launches++;
}

// ---------------------------------------------------------------------------
// (P)CG, device resident (solvers.py:60-114).  Control decisions are taken by
// single-block "final" kernels that also write the predicate read by every later
// kernel of the solve, so the host enqueues the whole loop without reading back.
// ---------------------------------------------------------------------------
struct CgDev {
  double bnorm, rz, alpha, rr, relres;
  int done, x0nz, gv_skip, iters, conv, neg, gv;
};

__global__ void k_cg_init(const float* g, const float* x0, int64_t d, double* ws) {
  CV_PDL_ENTRY();
  double t[2] = {0.0, 0.0};
  vec_for(d, al16p(g, x0), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    const Vf<W> gv = ldv<W>(g + i);
    Vf<W> xv;
    if (x0) xv = ldv<W>(x0 + i);
#pragma unroll
    for (int j = 0; j < W; ++j) {
      t[0] += (double)gv.v[j] * gv.v[j];
      if (x0) t[1] += xv.v[j] != 0.f ? 1.0 : 0.0;
    }
  });
  write_partials<2>(ws, t);
}
// The control decisions, from the totals of a reduction (one thread).  The
// replicated loop takes them in the last block of the reducing kernel; the sharded
// loop after the all-reduce of the per-rank totals.
CV_DEV void init_decide(double gg, double nz, CgDev* st) {
  st->bnorm = sqrt(gg);
  st->x0nz = nz > 0.0;
  st->rz = st->alpha = st->rr = 0.0;
  st->relres = 0.0;
  st->iters = 0; st->conv = 0; st->neg = 0; st->gv = 0;
  st->done = st->bnorm == 0.0;
  if (st->done) { st->conv = 1; st->x0nz = 0; }
  st->gv_skip = st->done || !st->x0nz;
}
CV_DEV void r0_decide(double rr, CgDev* st, double tol) {
  if (st->x0nz) st->gv++;
  st->relres = sqrt(rr) / st->bnorm;
  if (st->relres <= tol) { st->done = 1; st->conv = 1; st->iters = 0; }
  st->gv_skip = st->done;
}
CV_DEV void pap_decide(double pap, double mx, double nonfinite, CgDev* st, int k, int stab) {
  st->gv++;
  if (!isfinite(pap)) { st->done = 1; st->iters = k; st->conv = 0; }
  else if (pap <= 0.0) { st->done = 1; st->iters = k; st->conv = 0; st->neg = 1; }
  else {
    const double alpha = st->rz / pap;
    const bool step_ok = isfinite(alpha) && nonfinite == 0.0 && fabs((double)(float)alpha) * mx < (double)FLT_MAX;
    if (!step_ok) { st->done = 1; st->iters = k; st->conv = 0; }
    st->alpha = alpha;
  }
  st->gv_skip = st->done || !stab;
}
CV_DEV void r_decide(double rr, double rz_new, CgDev* st, int k, int maxiter, int stab, double tol) {
  if (stab) st->gv++;
  const double relres = sqrt(rr) / st->bnorm;
  st->relres = relres;
  if (!isfinite(relres)) { st->done = 1; st->iters = k; st->conv = 0; }
  else if (relres <= tol) { st->done = 1; st->iters = k; st->conv = 1; }
  else {
    st->alpha = rz_new / st->rz;  // beta, consumed by k_cg_pnext
    st->rz = rz_new;
    if (k == maxiter) { st->done = 1; st->iters = maxiter; st->conv = 0; }
  }
  st->gv_skip = st->done;
}

__global__ void k_cg_init_final(const double* ws, CgDev* st) {
  CV_PDL_ENTRY();
  double t[2];
  sum_partials<2>(ws, t);
  if (threadIdx.x == 0) init_decide(t[0], t[1], st);
}
// x = x0 (if any nonzero entry) else 0
__global__ void k_cg_setup_x(const float* x0, const CgDev* st, int64_t d, float* x) {
  CV_PDL_ENTRY();
  const bool use = st->x0nz;
  vec_for(d, al16p(x0, x), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    Vf<W> a;
    if (use) a = ldv<W>(x0 + i);
    else
#pragma unroll
      for (int j = 0; j < W; ++j) a.v[j] = 0.f;
    stv<W>(x + i, a);
  });
}
// r = g - (Ax + lam x) (warm) or g; partial ||r||^2
__global__ void k_cg_r0(const float* g, const float* ax, const float* x, float lam, const CgDev* st, int64_t d,
                        float* r, double* ws) {
  CV_PDL_ENTRY();
  if (st->done) return;
  const bool warm = st->x0nz;
  double t[1] = {0.0};
  vec_for(d, al16p(g, ax, x, r), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    Vf<W> v = ldv<W>(g + i);
    if (warm) {
      const Vf<W> av = ldv<W>(ax + i), xv = ldv<W>(x + i);
#pragma unroll
      for (int j = 0; j < W; ++j) v.v[j] = v.v[j] - (av.v[j] + lam * xv.v[j]);
    }
#pragma unroll
    for (int j = 0; j < W; ++j) t[0] += (double)v.v[j] * v.v[j];
    stv<W>(r + i, v);
  });
  write_partials<1>(ws, t);
}
__global__ void k_cg_r0_final(const double* ws, CgDev* st, double tol) {
  CV_PDL_ENTRY();
  if (st->done) return;
  double t[1];
  sum_partials<1>(ws, t);
  if (threadIdx.x == 0) r0_decide(t[0], st, tol);
}
// p = z = M^-1 r; rz = r.z
__global__ void k_cg_p0(const float* r, const float* pre, float lam, float floor_, const CgDev* st, int64_t d,
                        float* p, double* ws) {
  CV_PDL_ENTRY();
  if (st->done) return;
  double t[1] = {0.0};
  vec_for(d, al16p(r, pre, p), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    const Vf<W> rv = ldv<W>(r + i);
    Vf<W> mv, z;
    if (pre) mv = ldv<W>(pre + i);
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const float mi = pre ? 1.f / (fmaxf(mv.v[j], floor_) + lam) : 1.f;
      z.v[j] = mi * rv.v[j];
      t[0] += (double)rv.v[j] * z.v[j];
    }
    stv<W>(p + i, z);
  });
  write_partials<1>(ws, t);
}
__global__ void k_cg_p0_final(const double* ws, CgDev* st) {
  CV_PDL_ENTRY();
  if (st->done) return;
  double t[1];
  sum_partials<1>(ws, t);
  if (threadIdx.x == 0) st->rz = t[0];
}
CV_DEV void pap_final_body(const double* ws, CgDev* st, int k, int stab);
CV_DEV void r_final_body(const double* ws, CgDev* st, int k, int maxiter, int stab, double tol);

// Ap = Gv(p) + lam p (in place); partials p.Ap, max|p|, #nonfinite(p); the last
// block turns them into alpha and the termination flags (solvers.py:90-105)
__global__ void k_cg_pap(float* ap, const float* p, float lam, CgDev* st, int64_t d, double* ws, unsigned* ctr, int k,
                         int stab) {
  CV_PDL_ENTRY();
  if (st->done) return;
  double t[3] = {0.0, 0.0, 0.0};
  auto body = [&](float pi, float& a) {
    a += lam * pi;
    t[0] += (double)pi * a;
    t[2] += isfinite(pi) ? 0.0 : 1.0;
    t[1] = fmax(t[1], (double)fabsf(pi));
  };
  const int64_t nq = d >> 2;  // 128-bit body (vectors are 256-byte aligned pool buffers)
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    const float4 p4 = ld4g(p + 4 * q);
    float4 a4 = ld4g(ap + 4 * q);
    body(p4.x, a4.x); body(p4.y, a4.y); body(p4.z, a4.z); body(p4.w, a4.w);
    *reinterpret_cast<float4*>(ap + 4 * q) = a4;
  }
  for (int64_t i = 4 * nq + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
    float a = ap[i];
    body(p[i], a);
    ap[i] = a;
  }
  // max is not a sum: reduce it separately through the same shared buffer
  double mx = t[1];
  t[1] = 0.0;
  write_partials<3>(ws, t);
  __shared__ double smx[NT / 32];
  mx = warp_max_d(mx);
  if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < NT / 32; ++w) m = fmax(m, smx[w]);
    ws[blockIdx.x * 8 + 1] = m;
  }
  if (ctr && grid_last(ctr)) pap_final_body(ws, st, k, stab);
}
CV_DEV void pap_final_body(const double* ws, CgDev* st, int k, int stab) {
  double t[3];
  // sums of slots 0 and 2; max of slot 1
  double s0 = 0.0, s2 = 0.0, mx = 0.0;
  for (int b = threadIdx.x; b < NB; b += NT) {
    s0 += __ldcg(ws + b * 8 + 0);
    s2 += __ldcg(ws + b * 8 + 2);
    mx = fmax(mx, __ldcg(ws + b * 8 + 1));
  }
  t[0] = s0; t[1] = 0.0; t[2] = s2;
  block_sum<3>(t);
  __shared__ double smx[NT / 32];
  mx = warp_max_d(mx);
  if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < NT / 32; ++w) mx = fmax(mx, smx[w]);
    pap_decide(t[0], mx, t[2], st, k, stab);
  }
}
// plain iteration: x += a p; r -= a Ap; partials ||r||^2, r.M^-1 r
__global__ void k_cg_update(float* x, float* r, const float* p, const float* ap, const float* pre, float lam,
                            float floor_, CgDev* st, int64_t d, double* ws, unsigned* ctr, int k, int maxiter,
                            double tol) {
  CV_PDL_ENTRY();
  if (st->done) return;
  const float a = (float)st->alpha;
  double t[2] = {0.0, 0.0};
  auto body = [&](int64_t i, float& xi, float& ri, float pi, float api) {
    xi += a * pi;
    ri -= a * api;
    const float z = minv_of(pre, i, lam, floor_) * ri;
    t[0] += (double)ri * ri;
    t[1] += (double)ri * z;
  };
  const int64_t nq = d >> 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = 4 * q;
    float4 x4 = ld4g(x + i), r4 = ld4g(r + i);
    const float4 p4 = ld4g(p + i), a4 = ld4g(ap + i);
    body(i, x4.x, r4.x, p4.x, a4.x); body(i + 1, x4.y, r4.y, p4.y, a4.y);
    body(i + 2, x4.z, r4.z, p4.z, a4.z); body(i + 3, x4.w, r4.w, p4.w, a4.w);
    *reinterpret_cast<float4*>(x + i) = x4;
    *reinterpret_cast<float4*>(r + i) = r4;
  }
  for (int64_t i = 4 * nq + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
    float xi = x[i], ri = r[i];
    body(i, xi, ri, p[i], ap[i]);
    x[i] = xi;
    r[i] = ri;
  }
  write_partials<2>(ws, t);
  if (ctr && grid_last(ctr)) r_final_body(ws, st, k, maxiter, 0, tol);
}
// stabilising iteration: x += a p (the explicit residual product follows)
__global__ void k_cg_xupdate(float* x, const float* p, const CgDev* st, int64_t d) {
  CV_PDL_ENTRY();
  if (st->done) return;
  const float a = (float)st->alpha;
  vec_for(d, al16p(x, p), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    Vf<W> xv = ldv<W>(x + i);
    const Vf<W> pv = ldv<W>(p + i);
#pragma unroll
    for (int j = 0; j < W; ++j) xv.v[j] += a * pv.v[j];
    stv<W>(x + i, xv);
  });
}
// r = g - (Ax + lam x); partials ||r||^2, r.M^-1 r
__global__ void k_cg_rstab(const float* g, const float* ax, const float* x, float* r, const float* pre, float lam,
                           float floor_, CgDev* st, int64_t d, double* ws, unsigned* ctr, int k, int maxiter,
                           double tol) {
  CV_PDL_ENTRY();
  if (st->done) return;
  double t[2] = {0.0, 0.0};
  vec_for(d, al16p(g, ax, x, r) && al16p(pre), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    const Vf<W> gv = ldv<W>(g + i), av = ldv<W>(ax + i), xv = ldv<W>(x + i);
    Vf<W> mv, rv;
    if (pre) mv = ldv<W>(pre + i);
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const float ri = gv.v[j] - (av.v[j] + lam * xv.v[j]);
      rv.v[j] = ri;
      const float mi = pre ? 1.f / (fmaxf(mv.v[j], floor_) + lam) : 1.f;
      t[0] += (double)ri * ri;
      t[1] += (double)ri * (mi * ri);
    }
    stv<W>(r + i, rv);
  });
  write_partials<2>(ws, t);
  if (ctr && grid_last(ctr)) r_final_body(ws, st, k, maxiter, 1, tol);
}
CV_DEV void r_final_body(const double* ws, CgDev* st, int k, int maxiter, int stab, double tol) {
  double t[2] = {0.0, 0.0};
  for (int b = threadIdx.x; b < NB; b += NT) {
    t[0] += __ldcg(ws + b * 8 + 0);
    t[1] += __ldcg(ws + b * 8 + 1);
  }
  block_sum<2>(t);
  if (threadIdx.x == 0) r_decide(t[0], t[1], st, k, maxiter, stab, tol);
}
// p = M^-1 r + beta p
__global__ void k_cg_pnext(const float* r, const float* pre, float lam, float floor_, const CgDev* st, int64_t d,
                           float* p) {
  CV_PDL_ENTRY();
  if (st->done) return;
  const float beta = (float)st->alpha;
  const int64_t nq = d >> 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = 4 * q;
    const float4 r4 = ld4g(r + i);
    float4 p4 = ld4g(p + i);
    p4.x = minv_of(pre, i, lam, floor_) * r4.x + beta * p4.x;
    p4.y = minv_of(pre, i + 1, lam, floor_) * r4.y + beta * p4.y;
    p4.z = minv_of(pre, i + 2, lam, floor_) * r4.z + beta * p4.z;
    p4.w = minv_of(pre, i + 3, lam, floor_) * r4.w + beta * p4.w;
    *reinterpret_cast<float4*>(p + i) = p4;
  }
  for (int64_t i = 4 * nq + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = minv_of(pre, i, lam, floor_) * r[i] + beta * p[i];
}
// ---------------------------------------------------------------------------
// One plain (non-stabilising) (P)CG iteration after its product, in ONE launch
// (solvers.py:90-113): pap -> alpha -> x, r update -> beta -> next direction ->
// its per-layer scales -> the next product's input split.  The dependent
// reductions are separated by two grid barriers instead of four kernel boundaries;
// the grid is the reduction grid (NB blocks x NT threads, 4 per SM, co-resident by
// cooperative launch) and each thread keeps its <= CGF_MAXQ 16-byte groups of p and
// Ap (then z) in shared memory across the barriers, so the pass reads p, Ap, x, r, M
// and writes x, r, p and the split once: 9 d-vectors instead of the 16 of the four
// separate kernels, and no per-kernel launch / last-block tails.  The reductions are
// the separate kernels' (fixed-order fp64 block partials summed by the barrier's
// last block, which also takes the control decision); every block then reads the
// decided scalars.
// ---------------------------------------------------------------------------
constexpr int CGF_MAXQ = 4;
struct CgFusedArgs {
  float* x;
  float* r;
  float* p;
  const float* ap;
  const float* pre;
  float lam, floor_;
  CgDev* st;
  int64_t d;
  double* ws;
  unsigned* bar;  // [0] arrivals, [32] generation (separate 128-byte lines)
  int k, maxiter;
  double tol;
  OffTab t;
  float* part;   // NB x kOffTabMax block maxima of |z| per layer
  float* part2;  // NB x kOffTabMax block maxima of |p| per layer
  Scale* sc;
  Scale* zero_sc;
  int n_zero;
  __half* hi;
  __half* lo;
};

// Grid barrier whose last arriving block runs fin() (all its threads: the
// fixed-order reduction and the control decision) before it releases the others;
// then thread 0 of every block runs post() (the decided scalars into shared memory:
// one L2 request per block, not per warp).  The arrival counter and the generation
// word sit on separate 128-byte lines; release/acquire at gpu scope (the block's
// writes before the bar.sync are visible to every block after the barrier).  A
// bounded spin: a grid that is not co-resident traps instead of hanging the device.
template <typename F, typename G>
CV_DEV void grid_sync_last(unsigned* bar, F&& fin, G&& post) {
  __shared__ unsigned s_last;
  unsigned* genp = bar + 32;
  unsigned g = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(genp) : "memory");
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    s_last = old == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    fin();
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(genp) : "memory");
    }
  } else if (threadIdx.x == 0) {
    unsigned spins = 0, now;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(now) : "l"(genp) : "memory");
      if (++spins > (1u << 26)) __trap();
    } while (now == g);
  }
  if (threadIdx.x == 0) post();
  __syncthreads();
}

// Fixed-order sums of the NV partials at slots [off, off + NV) of every block (as
// sum_partials), all loads issued before the adds; result valid in thread 0.
template <int NV>
CV_DEV void sum_slots(const double* ws, int off, double (&t)[NV]) {
  constexpr int U = (NB + NT - 1) / NT;
  double v[U][NV];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int b = threadIdx.x + u * NT;
#pragma unroll
    for (int j = 0; j < NV; ++j) v[u][j] = b < NB ? __ldcg(ws + b * 8 + off + j) : 0.0;
  }
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    t[j] = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) t[j] += v[u][j];
  }
  block_sum<NV>(t);
}
CV_DEV double max_slot(const double* ws, int off) {
  constexpr int U = (NB + NT - 1) / NT;
  double m = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int b = threadIdx.x + u * NT;
    if (b < NB) m = fmax(m, __ldcg(ws + b * 8 + off));
  }
  __shared__ double smx[NT / 32];
  m = warp_max_d(m);
  if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; ++w) m = fmax(m, smx[w]);
  __syncthreads();
  return m;  // valid in thread 0
}

// Running per-layer max of a thread's increasing indices, folded into shared
// memory when the layer changes (at most L times per thread).
struct LayerMax {
  const OffTab& T;
  int* smax;
  int l = 0;
  float m = 0.f;
  CV_DEV void take4(int64_t i, const float4& v) {
    if (i + 3 < T.off[l + 1]) {  // the whole group in the current layer (the common case)
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      return;
    }
    take(i, v.x); take(i + 1, v.y); take(i + 2, v.z); take(i + 3, v.w);
  }
  CV_DEV void take(int64_t i, float v) {
    if (i >= T.off[l + 1]) {
      atomicMax(&smax[l], __float_as_int(m));
      m = 0.f;
      while (i >= T.off[l + 1]) ++l;
    }
    m = fmaxf(m, fabsf(v));
  }
  CV_DEV void flush() { atomicMax(&smax[l], __float_as_int(m)); }
};

// red_ws slots of the fused iteration (8 per block): 0-2 pap (p.Ap, max|p|,
// #nonfinite), 3-4 residual (||r||^2, r.z) -- disjoint, so a fast block's residual
// partials never overwrite pap partials a slow block is still reducing.
// STAB: the stabilising iteration's first half (solvers.py:97-101 with k % stabilise_every
// == 0): after the pap phase, x += alpha p with x's exact per-layer max, then x's split --
// the input of the explicit-residual product (k_cg_pap + k_cg_xupdate + that product's
// amax and split passes, bitwise: the same exponents as its exact-amax split).
template <int NQ, bool STAB = false>
__global__ void __launch_bounds__(NT, 4) k_cg_fused(CgFusedArgs a) {
  CV_PDL_ENTRY();
  __shared__ int s_done;
  __shared__ float s_val;  // alpha after the pap decision, beta after the residual decision
  __shared__ float sscale[kOffTabMax];
  __shared__ int smax[kOffTabMax], smaxp[kOffTabMax];
  // this thread's groups of p and Ap (then z) across the barriers: shared memory
  // (32 KB per block at NQ = 4), so the registers carry the loads in flight
  __shared__ float4 sP[NQ][NT], sA[NQ][NT];
  const OffTab& T = a.t;
  volatile CgDev* vst = a.st;
  if (threadIdx.x == 0) s_done = vst->done;  // nothing writes the flag before the first barrier
  if (threadIdx.x < kOffTabMax) smax[threadIdx.x] = smaxp[threadIdx.x] = 0;
  __syncthreads();
  if (s_done) return;
  auto read_decision = [&] {
    s_done = vst->done;
    s_val = (float)vst->alpha;
  };
  const int64_t tid = blockIdx.x * (int64_t)NT + threadIdx.x, nth = (int64_t)gridDim.x * NT;
  const int64_t nq = a.d >> 2;
  const int64_t it = 4 * nq + tid;  // scalar tail element of this thread (d % 4 threads)
  const bool has_t = it < a.d;
  const int tx = threadIdx.x;
  float pt = 0.f, at = 0.f;
  const float lam = a.lam;
  const float* __restrict__ gp = a.p;
  const float* __restrict__ gap = a.ap;
  const float* __restrict__ gpre = a.pre;
  float* __restrict__ gx = a.x;
  float* __restrict__ gr = a.r;

  // (1) Ap += lam p; partials p.Ap, max|p|, #nonfinite(p)  (k_cg_pap)
  {
    double t[3] = {0.0, 0.0, 0.0};
    double mx = 0.0;
    auto body = [&](float pi, float& ai) {
      ai += lam * pi;
      t[0] += (double)pi * ai;
      t[2] += isfinite(pi) ? 0.0 : 1.0;
      mx = fmax(mx, (double)fabsf(pi));
    };
    float4 P[NQ], A[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int64_t q = tid + j * nth;
      if (q < nq) {
        P[j] = ld4g(gp + 4 * q);
        A[j] = ld4g(gap + 4 * q);
      }
    }
    LayerMax lmp{T, smaxp};
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int64_t q = tid + j * nth;
      if (q < nq) {
        body(P[j].x, A[j].x); body(P[j].y, A[j].y); body(P[j].z, A[j].z); body(P[j].w, A[j].w);
        sP[j][tx] = P[j];
        sA[j][tx] = A[j];
        lmp.take4(4 * q, P[j]);
      }
    }
    if (has_t) {
      pt = gp[it];
      at = gap[it];
      body(pt, at);
      lmp.take(it, pt);
    }
    lmp.flush();
    t[1] = 0.0;
    write_partials<3>(a.ws, t);  // (its barriers also publish smaxp)
    if (threadIdx.x < T.L) a.part2[blockIdx.x * kOffTabMax + threadIdx.x] = __int_as_float(smaxp[threadIdx.x]);
    __shared__ double smx[NT / 32];
    mx = warp_max_d(mx);
    if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int w = 0; w < NT / 32; ++w) m = fmax(m, smx[w]);
      a.ws[blockIdx.x * 8 + 1] = m;
    }
    grid_sync_last(
        a.bar,
        [&] {
          double u[3];
          sum_slots<3>(a.ws, 0, u);
          const double pmax = max_slot(a.ws, 1);
          if (threadIdx.x == 0) pap_decide(u[0], pmax, u[2], a.st, a.k, STAB ? 1 : 0);
        },
        read_decision);
  }
  if (s_done) return;
  if constexpr (STAB) {
    // x += alpha p (k_cg_xupdate) and x's exact per-layer max
    const float al = s_val;
    float4 XV[NQ];
    float xt = 0.f;
    {
      LayerMax lm{T, smax};
      float4 X[NQ];
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        const int64_t q = tid + j * nth;
        if (q < nq) X[j] = ld4g(gx + 4 * q);
      }
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        const int64_t q = tid + j * nth;
        if (q < nq) {
          const float4 Pj = sP[j][tx];
          X[j].x += al * Pj.x; X[j].y += al * Pj.y; X[j].z += al * Pj.z; X[j].w += al * Pj.w;
          *reinterpret_cast<float4*>(gx + 4 * q) = X[j];
          lm.take4(4 * q, X[j]);
          XV[j] = X[j];
        }
      }
      if (has_t) {
        xt = gx[it] + al * pt;
        gx[it] = xt;
        lm.take(it, xt);
      }
      lm.flush();
      __syncthreads();
      if (threadIdx.x < T.L) a.part[blockIdx.x * kOffTabMax + threadIdx.x] = __int_as_float(smax[threadIdx.x]);
      __shared__ float shx[kOffTabMax][NT / 32];
      grid_sync_last(
          a.bar,
          [&] {
            for (int l2 = 0; l2 < T.L; ++l2) {
              float mm = 0.f;
#pragma unroll
              for (int v = 0; v < (NB + NT - 1) / NT; ++v) {
                const int b = threadIdx.x + v * NT;
                if (b < NB) mm = fmaxf(mm, __ldcg(a.part + b * kOffTabMax + l2));
              }
              mm = warp_max_f(mm);
              if ((threadIdx.x & 31) == 0) shx[l2][threadIdx.x >> 5] = mm;
            }
            __syncthreads();
            if (threadIdx.x == 0)
              for (int l2 = 0; l2 < T.L; ++l2) {
                float mx = 0.f;
                for (int w = 0; w < NT / 32; ++w) mx = fmaxf(mx, shx[l2][w]);
                a.sc[l2].amax = mx;
                a.sc[l2].e = exp_for_bound(mx);
              }
            for (int i = threadIdx.x; i < a.n_zero; i += NT) {
              a.zero_sc[i].e = 0;
              a.zero_sc[i].amax = 0.f;
            }
          },
          [&] {
            for (int l2 = 0; l2 < T.L; ++l2) sscale[l2] = pow2f(((volatile Scale*)a.sc)[l2].e);
          });
    }
    // x's split: the explicit-residual product's input
    int l = 0;
    auto scale_at = [&](int64_t i) {
      while (i >= T.off[l + 1]) ++l;
      return sscale[l];
    };
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int64_t q = tid + j * nth;
      if (q < nq) {
        const int64_t i = 4 * q;
        union { uint2 u; __half h[4]; } H, L;
        split16(XV[j].x, scale_at(i), H.h[0], L.h[0]);
        split16(XV[j].y, scale_at(i + 1), H.h[1], L.h[1]);
        split16(XV[j].z, scale_at(i + 2), H.h[2], L.h[2]);
        split16(XV[j].w, scale_at(i + 3), H.h[3], L.h[3]);
        *reinterpret_cast<uint2*>(a.hi + i) = H.u;
        *reinterpret_cast<uint2*>(a.lo + i) = L.u;
      }
    }
    if (has_t) split16(xt, scale_at(it), a.hi[it], a.lo[it]);
    return;
  }

  // (2) x += alpha p; r -= alpha Ap; z = M^-1 r; partials ||r||^2, r.z  (k_cg_update)
  //     and the per-layer max|z|: with the current direction's per-layer max|p_l|
  //     (phase 1), B_l = max|z_l| + |beta| max|p_l| bounds the next direction, so its
  //     split exponent is known at this barrier (no third reduction; the exponent is
  //     the exact-amax one or one binade below it; the bound is rebuilt from exact
  //     maxima every iteration, so it never compounds).
  {
    const float al = s_val;
    double t[2] = {0.0, 0.0};
    LayerMax lm{T, smax};
    auto minv = [&](float m) { return 1.f / (fmaxf(m, a.floor_) + lam); };
    auto body = [&](float& xi, float& ri, float pi, float& ai, float mi) {
      xi += al * pi;
      ri -= al * ai;
      const float z = mi * ri;
      t[0] += (double)ri * ri;
      t[1] += (double)ri * z;
      ai = z;
    };
    float4 X[NQ], R[NQ], M[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int64_t q = tid + j * nth;
      if (q < nq) {
        X[j] = ld4g(gx + 4 * q);
        R[j] = ld4g(gr + 4 * q);
        M[j] = gpre ? ld4g(gpre + 4 * q) : make_float4(1.f, 1.f, 1.f, 1.f);
      }
    }
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int64_t q = tid + j * nth;
      if (q < nq) {
        const int64_t i = 4 * q;
        const float4 Pj = sP[j][tx];
        float4 Aj = sA[j][tx], Mj = M[j];
        if (gpre) Mj = make_float4(minv(Mj.x), minv(Mj.y), minv(Mj.z), minv(Mj.w));
        body(X[j].x, R[j].x, Pj.x, Aj.x, Mj.x); body(X[j].y, R[j].y, Pj.y, Aj.y, Mj.y);
        body(X[j].z, R[j].z, Pj.z, Aj.z, Mj.z); body(X[j].w, R[j].w, Pj.w, Aj.w, Mj.w);
        *reinterpret_cast<float4*>(gx + i) = X[j];
        *reinterpret_cast<float4*>(gr + i) = R[j];
        sA[j][tx] = Aj;
        lm.take4(i, Aj);
      }
    }
    if (has_t) {
      float xi = gx[it], ri = gr[it];
      body(xi, ri, pt, at, gpre ? minv(gpre[it]) : 1.f);
      gx[it] = xi;
      gr[it] = ri;
      lm.take(it, at);
    }
    lm.flush();
    block_sum<2>(t);  // (its barriers also publish smax)
    if (threadIdx.x == 0) {
      a.ws[blockIdx.x * 8 + 3] = t[0];
      a.ws[blockIdx.x * 8 + 4] = t[1];
    }
    if (threadIdx.x < T.L) a.part[blockIdx.x * kOffTabMax + threadIdx.x] = __int_as_float(smax[threadIdx.x]);
    __shared__ float sh[kOffTabMax][NT / 32], shp[kOffTabMax][NT / 32];
    grid_sync_last(
        a.bar,
        [&] {
          double tot[2];
          sum_slots<2>(a.ws, 3, tot);
          // per-layer max|z| over the blocks (order free)
          for (int l2 = 0; l2 < T.L; ++l2) {
            float mm = 0.f, mp = 0.f;
#pragma unroll
            for (int u = 0; u < (NB + NT - 1) / NT; ++u) {
              const int b = threadIdx.x + u * NT;
              if (b < NB) {
                mm = fmaxf(mm, __ldcg(a.part + b * kOffTabMax + l2));
                mp = fmaxf(mp, __ldcg(a.part2 + b * kOffTabMax + l2));
              }
            }
            mm = warp_max_f(mm);
            mp = warp_max_f(mp);
            if ((threadIdx.x & 31) == 0) {
              sh[l2][threadIdx.x >> 5] = mm;
              shp[l2][threadIdx.x >> 5] = mp;
            }
          }
          __syncthreads();
          if (threadIdx.x == 0) {
            r_decide(tot[0], tot[1], a.st, a.k, a.maxiter, 0, a.tol);
            if (!a.st->done) {
              const float beta = fabsf((float)a.st->alpha);
              for (int l2 = 0; l2 < T.L; ++l2) {
                float mz = 0.f, mp = 0.f;
                for (int w = 0; w < NT / 32; ++w) {
                  mz = fmaxf(mz, sh[l2][w]);
                  mp = fmaxf(mp, shp[l2][w]);
                }
                const float B = mz + beta * mp;
                a.sc[l2].amax = B;
                a.sc[l2].e = exp_for_bound(B);
              }
            }
          }
          __syncthreads();
          if (!a.st->done)
            for (int i = threadIdx.x; i < a.n_zero; i += NT) {
              a.zero_sc[i].e = 0;
              a.zero_sc[i].amax = 0.f;
            }
        },
        [&] {
          read_decision();
          if (!s_done)
            for (int l2 = 0; l2 < T.L; ++l2) sscale[l2] = pow2f(((volatile Scale*)a.sc)[l2].e);
        });
  }
  if (s_done) return;  // converged, failed, or k == maxiter: the direction is never used

  // (3) p = z + beta p (solvers.py:111-112) and the next product's input split
  {
    const float beta = s_val;
    int l = 0;
    auto scale_at = [&](int64_t i) {
      while (i >= T.off[l + 1]) ++l;
      return sscale[l];
    };
    float* __restrict__ wp = a.p;
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int64_t q = tid + j * nth;
      if (q < nq) {
        const int64_t i = 4 * q;
        float4 Pj = sP[j][tx];
        const float4 Zj = sA[j][tx];
        Pj.x = Zj.x + beta * Pj.x;
        Pj.y = Zj.y + beta * Pj.y;
        Pj.z = Zj.z + beta * Pj.z;
        Pj.w = Zj.w + beta * Pj.w;
        *reinterpret_cast<float4*>(wp + i) = Pj;
        union { uint2 u; __half h[4]; } H, L;
        if (i + 3 < T.off[l + 1] && i >= T.off[l]) {
          const float sc4 = sscale[l];
          split16(Pj.x, sc4, H.h[0], L.h[0]);
          split16(Pj.y, sc4, H.h[1], L.h[1]);
          split16(Pj.z, sc4, H.h[2], L.h[2]);
          split16(Pj.w, sc4, H.h[3], L.h[3]);
        } else {
          split16(Pj.x, scale_at(i), H.h[0], L.h[0]);
          split16(Pj.y, scale_at(i + 1), H.h[1], L.h[1]);
          split16(Pj.z, scale_at(i + 2), H.h[2], L.h[2]);
          split16(Pj.w, scale_at(i + 3), H.h[3], L.h[3]);
        }
        *reinterpret_cast<uint2*>(a.hi + i) = H.u;
        *reinterpret_cast<uint2*>(a.lo + i) = L.u;
      }
    }
    if (has_t) {
      pt = at + beta * pt;
      wp[it] = pt;
      split16(pt, scale_at(it), a.hi[it], a.lo[it]);
    }
  }
}

// The start of a (P)CG run after the warm-start product, in one launch
// (solvers.py:76-84): r = g - (Ax + lam x) (or g), ||r||^2 -> the r0 decision ->
// p = z = M^-1 r, r.z and the exact per-layer max|p| -> p's scales -> the first
// product's input split.  The same reductions as k_cg_r0 / k_cg_p0 (bitwise: same
// thread mapping and summation order) and the same exact-amax split as the product's
// own split pass, so the iterates equal the per-kernel start's.  red_ws slots 5, 6.
template <int NQ>
__global__ void __launch_bounds__(NT, 4) k_cg_start(CgFusedArgs a, const float* __restrict__ g) {
  CV_PDL_ENTRY();
  __shared__ int s_done, s_warm;
  __shared__ float sscale[kOffTabMax];
  __shared__ int smax[kOffTabMax];
  __shared__ float4 sR[NQ][NT];
  const OffTab& T = a.t;
  volatile CgDev* vst = a.st;
  if (threadIdx.x == 0) {
    s_done = vst->done;
    s_warm = vst->x0nz;
  }
  if (threadIdx.x < kOffTabMax) smax[threadIdx.x] = 0;
  __syncthreads();
  if (s_done) return;
  const bool warm = s_warm;
  const int64_t tid = blockIdx.x * (int64_t)NT + threadIdx.x, nth = (int64_t)gridDim.x * NT;
  const int64_t nq = a.d >> 2;
  const int64_t it = 4 * nq + tid;
  const bool has_t = it < a.d;
  const int tx = threadIdx.x;
  const float lam = a.lam;
  float rt = 0.f;

  // (1) r0 (k_cg_r0)
  {
    double t[1] = {0.0};
    float4 G[NQ], AX[NQ], X[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int64_t q = tid + j * nth;
      if (q < nq) {
        G[j] = ld4g(g + 4 * q);
        if (warm) {
          AX[j] = ld4g(a.ap + 4 * q);
          X[j] = ld4g(a.x + 4 * q);
        }
      }
    }
    auto body = [&](float& v, float av, float xv) {
      if (warm) v = v - (av + lam * xv);
      t[0] += (double)v * v;
    };
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int64_t q = tid + j * nth;
      if (q < nq) {
        float4 v = G[j];
        body(v.x, AX[j].x, X[j].x); body(v.y, AX[j].y, X[j].y); body(v.z, AX[j].z, X[j].z); body(v.w, AX[j].w, X[j].w);
        *reinterpret_cast<float4*>(a.r + 4 * q) = v;
        sR[j][tx] = v;
      }
    }
    if (has_t) {
      rt = g[it];
      body(rt, warm ? a.ap[it] : 0.f, warm ? a.x[it] : 0.f);
      a.r[it] = rt;
    }
    block_sum<1>(t);
    if (threadIdx.x == 0) a.ws[blockIdx.x * 8 + 5] = t[0];
    grid_sync_last(
        a.bar,
        [&] {
          double u[1];
          sum_slots<1>(a.ws, 5, u);
          if (threadIdx.x == 0) r0_decide(u[0], a.st, a.tol);
        },
        [&] { s_done = vst->done; });
  }
  if (s_done) return;

  // (2) p = z = M^-1 r; r.z; exact per-layer max|p|  (k_cg_p0 + the product's amax pass)
  {
    double t[1] = {0.0};
    LayerMax lm{T, smax};
    auto minv = [&](float m) { return a.pre ? 1.f / (fmaxf(m, a.floor_) + lam) : 1.f; };
    float4 M[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int64_t q = tid + j * nth;
      if (q < nq) M[j] = a.pre ? ld4g(a.pre + 4 * q) : make_float4(1.f, 1.f, 1.f, 1.f);
    }
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int64_t q = tid + j * nth;
      if (q < nq) {
        const float4 rv = sR[j][tx];
        float4 z;
        z.x = minv(M[j].x) * rv.x; z.y = minv(M[j].y) * rv.y; z.z = minv(M[j].z) * rv.z; z.w = minv(M[j].w) * rv.w;
        t[0] += (double)rv.x * z.x; t[0] += (double)rv.y * z.y; t[0] += (double)rv.z * z.z; t[0] += (double)rv.w * z.w;
        *reinterpret_cast<float4*>(a.p + 4 * q) = z;
        sR[j][tx] = z;
        lm.take4(4 * q, z);
      }
    }
    if (has_t) {
      const float z = minv(a.pre ? a.pre[it] : 1.f) * rt;
      t[0] += (double)rt * z;
      rt = z;
      a.p[it] = z;
      lm.take(it, z);
    }
    lm.flush();
    block_sum<1>(t);  // (its barriers also publish smax)
    if (threadIdx.x == 0) a.ws[blockIdx.x * 8 + 6] = t[0];
    if (threadIdx.x < T.L) a.part[blockIdx.x * kOffTabMax + threadIdx.x] = __int_as_float(smax[threadIdx.x]);
    __shared__ float sh[kOffTabMax][NT / 32];
    grid_sync_last(
        a.bar,
        [&] {
          double u[1];
          sum_slots<1>(a.ws, 6, u);
          for (int l2 = 0; l2 < T.L; ++l2) {
            float mm = 0.f;
#pragma unroll
            for (int v = 0; v < (NB + NT - 1) / NT; ++v) {
              const int b = threadIdx.x + v * NT;
              if (b < NB) mm = fmaxf(mm, __ldcg(a.part + b * kOffTabMax + l2));
            }
            mm = warp_max_f(mm);
            if ((threadIdx.x & 31) == 0) sh[l2][threadIdx.x >> 5] = mm;
          }
          __syncthreads();
          if (threadIdx.x == 0) {
            a.st->rz = u[0];
            for (int l2 = 0; l2 < T.L; ++l2) {
              float mz = 0.f;
              for (int w = 0; w < NT / 32; ++w) mz = fmaxf(mz, sh[l2][w]);
              a.sc[l2].amax = mz;
              a.sc[l2].e = exp_for_bound(mz);
            }
          }
          for (int i = threadIdx.x; i < a.n_zero; i += NT) {
            a.zero_sc[i].e = 0;
            a.zero_sc[i].amax = 0.f;
          }
        },
        [&] {
          for (int l2 = 0; l2 < T.L; ++l2) sscale[l2] = pow2f(((volatile Scale*)a.sc)[l2].e);
        });
  }

  // (3) the first product's input split
  {
    int l = 0;
    auto scale_at = [&](int64_t i) {
      while (i >= T.off[l + 1]) ++l;
      return sscale[l];
    };
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int64_t q = tid + j * nth;
      if (q < nq) {
        const int64_t i = 4 * q;
        const float4 Pj = sR[j][tx];
        union { uint2 u; __half h[4]; } H, L;
        split16(Pj.x, scale_at(i), H.h[0], L.h[0]);
        split16(Pj.y, scale_at(i + 1), H.h[1], L.h[1]);
        split16(Pj.z, scale_at(i + 2), H.h[2], L.h[2]);
        split16(Pj.w, scale_at(i + 3), H.h[3], L.h[3]);
        *reinterpret_cast<uint2*>(a.hi + i) = H.u;
        *reinterpret_cast<uint2*>(a.lo + i) = L.u;
      }
    }
    if (has_t) split16(rt, scale_at(it), a.hi[it], a.lo[it]);
  }
}

// The fused iteration applies when every thread's share fits its registers and the
// 16-byte / 8-byte vector accesses are aligned.
static int cg_fused_nq(int64_t d, const OffTab& t, const void* x, const void* r, const void* p, const void* ap,
                       const void* pre, const void* hi, const void* lo) {
  if (t.L < 1 || t.L > kOffTabMax || t.off[0] != 0) return 0;
  if (((uintptr_t)x | (uintptr_t)r | (uintptr_t)p | (uintptr_t)ap | (uintptr_t)pre) & 15) return 0;
  if (((uintptr_t)hi | (uintptr_t)lo) & 7) return 0;
  const int64_t nth = (int64_t)NB * NT;
  const int64_t nq = (d >> 2) + nth - 1;
  const int64_t q = nq / nth;
  return q >= 1 && q <= CGF_MAXQ ? (int)q : (d > 0 && d < 4 ? 1 : 0);
}

static bool cg_fused_enabled() {
  static const int on = !(getenv("CURVOPT_CG_FUSED") && getenv("CURVOPT_CG_FUSED")[0] == '0');
  return on;
}

// The grid must be co-resident (cooperative launch): NB blocks on this device's
// SMs at the kernel's occupancy (4 per SM on a full B200; a smaller partition, e.g.
// a MIG slice, keeps the per-kernel passes).
static int occupancy_of(const void* k) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NT, 0) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 0;
  }
  return per_sm;
}
template <int NQ>
static bool cg_fused_fits_nq(int sms) {
  const int per_sm = std::min({occupancy_of((const void*)k_cg_fused<NQ>), occupancy_of((const void*)k_cg_fused<NQ, true>),
                               occupancy_of((const void*)k_cg_start<NQ>)});
  return per_sm * sms >= NB;
}
static bool cg_fused_fits(int nq) {
  constexpr int kMaxDev = 64;
  static int fits[kMaxDev][CGF_MAXQ + 1];  // per device: 0 unknown, 1 fits, 2 does not
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) return false;
  int& f = fits[dev][nq];
  if (f == 0) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const bool ok = nq == 1 ? cg_fused_fits_nq<1>(sms) : nq == 2 ? cg_fused_fits_nq<2>(sms)
                  : nq == 3 ? cg_fused_fits_nq<3>(sms) : cg_fused_fits_nq<4>(sms);
    f = ok ? 1 : 2;
  }
  return f == 1;
}

static void launch_cg_start(cudaStream_t st, int nq, const CgFusedArgs& a, const float* g) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(NB);
  cfg.blockDim = dim3(NT);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  switch (nq) {
    case 1: cudaLaunchKernelEx(&cfg, k_cg_start<1>, a, g); break;
    case 2: cudaLaunchKernelEx(&cfg, k_cg_start<2>, a, g); break;
    case 3: cudaLaunchKernelEx(&cfg, k_cg_start<3>, a, g); break;
    default: cudaLaunchKernelEx(&cfg, k_cg_start<4>, a, g); break;
  }
}

static void launch_cg_fused(cudaStream_t st, int nq, const CgFusedArgs& a, bool stab = false) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(NB);
  cfg.blockDim = dim3(NT);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (stab) switch (nq) {
      case 1: cudaLaunchKernelEx(&cfg, k_cg_fused<1, true>, a); break;
      case 2: cudaLaunchKernelEx(&cfg, k_cg_fused<2, true>, a); break;
      case 3: cudaLaunchKernelEx(&cfg, k_cg_fused<3, true>, a); break;
      default: cudaLaunchKernelEx(&cfg, k_cg_fused<4, true>, a); break;
    }
  else switch (nq) {
      case 1: cudaLaunchKernelEx(&cfg, k_cg_fused<1>, a); break;
      case 2: cudaLaunchKernelEx(&cfg, k_cg_fused<2>, a); break;
      case 3: cudaLaunchKernelEx(&cfg, k_cg_fused<3>, a); break;
      default: cudaLaunchKernelEx(&cfg, k_cg_fused<4>, a); break;
    }
}

__global__ void k_cg_finish(const CgDev* st, cv_cg_stats* out) {
  CV_PDL_ENTRY();
  out->relres = st->relres;
  out->bnorm = st->bnorm;
  out->iterations = st->iters;
  out->converged = st->conv;
  out->neg_curv = st->neg;
  out->gv_count = st->gv;
  out->done = st->done;
  out->x0_nonzero = st->x0nz;
}

// Sharded loop: reductions end in per-rank totals, all-reduced, then decided.
template <int NV>
__global__ void k_cgs_total(const double* ws, double* tot) {
  CV_PDL_ENTRY();
  double t[NV];
  sum_partials<NV>(ws, t);
  if (threadIdx.x == 0)
#pragma unroll
    for (int v = 0; v < NV; ++v) tot[v] = t[v];
}
// p.Ap and #nonfinite summed; max|p| into this rank's slot (the sum-only all-reduce
// then carries every rank's maximum)
__global__ void k_cgs_pap_total(const double* ws, double* tot, int rank, int world) {
  CV_PDL_ENTRY();
  double t[3] = {0.0, 0.0, 0.0}, mx = 0.0;
  for (int b = threadIdx.x; b < NB; b += NT) {
    t[0] += ws[b * 8 + 0];
    t[2] += ws[b * 8 + 2];
    mx = fmax(mx, ws[b * 8 + 1]);
  }
  block_sum<3>(t);
  __shared__ double smx[NT / 32];
  mx = warp_max_d(mx);
  if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < NT / 32; ++w) mx = fmax(mx, smx[w]);
    tot[0] = t[0];
    tot[1] = t[2];
    for (int j = 0; j < world; ++j) tot[2 + j] = j == rank ? mx : 0.0;
  }
}
enum { CGS_INIT, CGS_R0, CGS_P0, CGS_PAP, CGS_R };
__global__ void k_cgs_decide(const double* tot, CgDev* st, int what, int k, int maxiter, int stab, double tol,
                             int world) {
  CV_PDL_ENTRY();
  if (what == CGS_INIT) return init_decide(tot[0], tot[1], st);
  if (st->done) return;
  if (what == CGS_R0) r0_decide(tot[0], st, tol);
  else if (what == CGS_P0) st->rz = tot[0];
  else if (what == CGS_PAP) {
    double mx = 0.0;
    for (int j = 0; j < world; ++j) mx = fmax(mx, tot[2 + j]);
    pap_decide(tot[0], mx, tot[1], st, k, stab);
  } else r_decide(tot[0], tot[1], st, k, maxiter, stab, tol);
}

// The operator of a parameter-space CG run: a snapshot's curvature product (the
// direction update also publishes the next product's input scales).
struct CgOperator {
  int64_t d = 0;
  cv_snap* s = nullptr;
  MatvecFn mv = nullptr;
  void apply(cv_ctx* ctx, const float* in, float* out, const int* skip) const { mv(ctx, s, in, out, skip); }
};

static void cg_run(cv_ctx* ctx, const CgOperator& op, const float* g, double lam, double tol, int maxiter, int stab,
                   const float* precond, double floor, const float* x0, float* x, cv_cg_stats* stats, float* r,
                   float* p, float* ap);
static void cg_run_sharded(cv_ctx* ctx, const CgOperator& op, const float* g, double lam, double tol, int maxiter,
                           int stab, const float* precond, double floor, const float* x0, float* x,
                           cv_cg_stats* stats);

// Shard the CG vectors across ranks once the replicated vector passes (13 x 4 d bytes
// per iteration, ~0.15 ms at d = 8M) outweigh the sharded loop's extra launches and
// scalar all-reduces (~30-40 us per iteration): C5 (d = 63M) shards, C3 (d = 1.9M)
// stays replicated.
constexpr int64_t kShardMinD = int64_t(1) << 23;
static bool cg_sharded(const cv_ctx* ctx, int64_t d) {
  if (!distributed(ctx) || ctx->shard_cg == 0) return false;
  return ctx->shard_cg == 1 || (ctx->world > 1 && d >= kShardMinD);
}

void cg_solve(cv_ctx* ctx, cv_snap* s, int kind, const float* g, double lam, double tol, int maxiter, int stab,
              const float* precond, double floor, const float* x0, float* x, cv_cg_stats* stats) {
  CgOperator op;
  op.d = s->d;
  op.s = s;
  op.mv = matvec_fn(kind);
  if (cg_sharded(ctx, s->d)) return cg_run_sharded(ctx, op, g, lam, tol, maxiter, stab, precond, floor, x0, x, stats);
  cg_run(ctx, op, g, lam, tol, maxiter, stab, precond, floor, x0, x, stats, snap_tmp(s, &s->cg_r),
         snap_tmp(s, &s->cg_p), snap_tmp(s, &s->cg_ap));
}

// ---------------------------------------------------------------------------
// Row-space CG on a dense Gram (solvers.py:164-174 with gram_matvec = gram @ u):
// the same control flow and device-resident scalars as the parameter-space loop
// (CgDev, pap_final_body, r_final_body), with the m-length vectors kept in fp64.
// m = b*c is small (40,960 at C4), and the row systems are solved to few digits in
// maxiter iterations, where fp32 residual recurrences drift from the f64 reference
// by ~1e-4 (residual cancellation against |Gram| ~ 50x |rhs|); fp64 vectors track it.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_gram_gemv_d(const float* G, const double* x, int64_t m, double* y,
                                                     const int* skip) {
  CV_PDL_ENTRY();
  if (skip && *skip) return;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); row < m; row += nwarps) {
    const float* g = G + row * m;
    double s = 0.0;
    if ((m & 3) == 0) {
      for (int64_t k = lane * 4; k < m; k += 128) {
        const float4 q = __ldcs(reinterpret_cast<const float4*>(g + k));
        s += (double)q.x * x[k] + (double)q.y * x[k + 1] + (double)q.z * x[k + 2] + (double)q.w * x[k + 3];
      }
    } else {
      for (int64_t k = lane; k < m; k += 32) s += (double)g[k] * x[k];
    }
    s = warp_sum(s);
    if (lane == 0) y[row] = s;
  }
}
#define DCG_FOR(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)
__global__ void k_dcg_setup(const float* g, const float* x0, const CgDev* st, int64_t m, double* b, double* x) {
  CV_PDL_ENTRY();
  DCG_FOR(i, m) {
    b[i] = g[i];
    x[i] = st->x0nz ? (double)x0[i] : 0.0;
  }
}
// r = b - (Ax + lam x) (warm) or b; partial ||r||^2
__global__ void k_dcg_r0(const double* b, const double* ax, const double* x, double lam, const CgDev* st, int64_t m,
                         double* r, double* ws) {
  CV_PDL_ENTRY();
  if (st->done) return;
  double t[1] = {0.0};
  DCG_FOR(i, m) {
    const double v = st->x0nz ? b[i] - (ax[i] + lam * x[i]) : b[i];
    r[i] = v;
    t[0] += v * v;
  }
  write_partials<1>(ws, t);
}
__global__ void k_dcg_p0(const double* r, const CgDev* st, int64_t m, double* p, double* ws) {
  CV_PDL_ENTRY();
  if (st->done) return;
  double t[1] = {0.0};
  DCG_FOR(i, m) {
    p[i] = r[i];
    t[0] += r[i] * r[i];
  }
  write_partials<1>(ws, t);
}
__global__ void k_dcg_pap(double* ap, const double* p, double lam, CgDev* st, int64_t m, double* ws, unsigned* ctr,
                          int k, int stab) {
  CV_PDL_ENTRY();
  if (st->done) return;
  double t[3] = {0.0, 0.0, 0.0};
  double mx = 0.0;
  DCG_FOR(i, m) {
    const double a = ap[i] + lam * p[i];
    ap[i] = a;
    t[0] += p[i] * a;
    t[2] += isfinite(p[i]) ? 0.0 : 1.0;
    mx = fmax(mx, fabs(p[i]));
  }
  write_partials<3>(ws, t);
  __shared__ double smx[NT / 32];
  mx = warp_max_d(mx);
  if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double q = 0.0;
    for (int w = 0; w < NT / 32; ++w) q = fmax(q, smx[w]);
    ws[blockIdx.x * 8 + 1] = q;
  }
  if (ctr && grid_last(ctr)) pap_final_body(ws, st, k, stab);
}
__global__ void k_dcg_update(double* x, double* r, const double* p, const double* ap, CgDev* st, int64_t m, double* ws,
                             unsigned* ctr, int k, int maxiter, double tol) {
  CV_PDL_ENTRY();
  if (st->done) return;
  const double a = st->alpha;
  double t[2] = {0.0, 0.0};
  DCG_FOR(i, m) {
    x[i] += a * p[i];
    const double ri = r[i] - a * ap[i];
    r[i] = ri;
    t[0] += ri * ri;
    t[1] += ri * ri;
  }
  write_partials<2>(ws, t);
  if (ctr && grid_last(ctr)) r_final_body(ws, st, k, maxiter, 0, tol);
}
__global__ void k_dcg_xupdate(double* x, const double* p, const CgDev* st, int64_t m) {
  CV_PDL_ENTRY();
  if (st->done) return;
  const double a = st->alpha;
  DCG_FOR(i, m) x[i] += a * p[i];
}
__global__ void k_dcg_rstab(const double* b, const double* ax, const double* x, double* r, double lam, CgDev* st,
                            int64_t m, double* ws, unsigned* ctr, int k, int maxiter, double tol) {
  CV_PDL_ENTRY();
  if (st->done) return;
  double t[2] = {0.0, 0.0};
  DCG_FOR(i, m) {
    const double ri = b[i] - (ax[i] + lam * x[i]);
    r[i] = ri;
    t[0] += ri * ri;
    t[1] += ri * ri;
  }
  write_partials<2>(ws, t);
  if (ctr && grid_last(ctr)) r_final_body(ws, st, k, maxiter, 1, tol);
}
__global__ void k_dcg_pnext(const double* r, const CgDev* st, int64_t m, double* p) {
  CV_PDL_ENTRY();
  if (st->done) return;
  const double beta = st->alpha;
  DCG_FOR(i, m) p[i] = r[i] + beta * p[i];
}
__global__ void k_dcg_out(const double* x, int64_t m, float* out) {
  CV_PDL_ENTRY();
  DCG_FOR(i, m) out[i] = (float)x[i];
}

void dense_cg_solve(cv_ctx* ctx, const float* gram, int64_t m, const float* rhs, double mu, double tol, int maxiter,
                    int stab, const float* x0, float* xout, cv_cg_stats* stats) {
  const int64_t gb = (m + 7) / 8;
  const int ggrid = (int)(gb < 16 * (int64_t)ctx->sm_count ? gb : 16 * (int64_t)ctx->sm_count);
  dense_cg_run(ctx, m, [&](const double* in, double* out, const int* skip) {
    launch_k(ctx->stream, k_gram_gemv_d, ggrid, 256, 0, gram, in, m, out, skip);
    ctx->launches++;
  }, rhs, mu, tol, maxiter, stab, x0, xout, stats);
}

// The row-space CG loop on any Gram product A(in, out, skip) = Gram . in (fp64 vectors;
// the damping mu is added by the loop).
void dense_cg_run(cv_ctx* ctx, int64_t m, const std::function<void(const double*, double*, const int*)>& A,
                  const float* rhs, double mu, double tol, int maxiter, int stab, const float* x0, float* xout,
                  cv_cg_stats* stats) {
  CgDev* st = (CgDev*)(ctx->scal_ws + 8);
  double* ws = ctx->red_ws;
  cudaStream_t sm = ctx->stream;
  unsigned* ctr = ctx->amax_counter + 1;
  const int64_t ms = (m + 31) / 32 * 32;
  double* buf = (double*)ctx->pool.get(sizeof(double) * (size_t)(5 * ms));
  double *b = buf, *x = buf + ms, *r = buf + 2 * ms, *p = buf + 3 * ms, *ap = buf + 4 * ms;
  launch_k(sm, k_cg_init, NB, NT, 0, rhs, x0, m, ws);
  launch_k(sm, k_cg_init_final, 1, NT, 0, (const double*)ws, st);
  launch_k(sm, k_dcg_setup, NB, NT, 0, rhs, x0, (const CgDev*)st, m, b, x);
  ctx->launches += 3;
  if (x0) A(x, ap, &st->gv_skip);
  launch_k(sm, k_dcg_r0, NB, NT, 0, (const double*)b, (const double*)ap, (const double*)x, mu, (const CgDev*)st, m, r,
           ws);
  launch_k(sm, k_cg_r0_final, 1, NT, 0, (const double*)ws, st, tol);
  launch_k(sm, k_dcg_p0, NB, NT, 0, (const double*)r, (const CgDev*)st, m, p, ws);
  launch_k(sm, k_cg_p0_final, 1, NT, 0, (const double*)ws, st);
  ctx->launches += 4;
  for (int k = 1; k <= maxiter; ++k) {
    const int is_stab = (stab > 0 && k % stab == 0) ? 1 : 0;
    A(p, ap, &st->done);
    launch_k(sm, k_dcg_pap, NB, NT, 0, ap, (const double*)p, mu, st, m, ws, ctr, k, is_stab);
    ctx->launches++;
    if (is_stab) {
      launch_k(sm, k_dcg_xupdate, NB, NT, 0, x, (const double*)p, (const CgDev*)st, m);
      A(x, ap, &st->gv_skip);
      launch_k(sm, k_dcg_rstab, NB, NT, 0, (const double*)b, (const double*)ap, (const double*)x, r, mu, st, m, ws,
               ctr, k, maxiter, tol);
      ctx->launches += 2;
    } else {
      launch_k(sm, k_dcg_update, NB, NT, 0, x, r, (const double*)p, (const double*)ap, st, m, ws, ctr, k, maxiter,
               tol);
      ctx->launches++;
    }
    if (k == maxiter) break;
    launch_k(sm, k_dcg_pnext, NB, NT, 0, (const double*)r, (const CgDev*)st, m, p);
    ctx->launches++;
  }
  launch_k(sm, k_dcg_out, NB, NT, 0, (const double*)x, m, xout);
  launch_k(sm, k_cg_finish, 1, 1, 0, (const CgDev*)st, stats);
  ctx->launches += 2;
  ctx->pool.put(buf);  // stream-ordered reuse
}

static void cg_run(cv_ctx* ctx, const CgOperator& op, const float* g, double lam, double tol, int maxiter, int stab,
                   const float* precond, double floor, const float* x0, float* x, cv_cg_stats* stats, float* r,
                   float* p, float* ap) {
  const int64_t d = op.d;
  cv_snap* s = op.s;
  CgDev* st = (CgDev*)(ctx->scal_ws + 8);
  double* ws = ctx->red_ws;
  cudaStream_t sm = ctx->stream;
  const float flam = (float)lam, ffl = (float)floor;

  launch_k(sm, k_cg_init, NB, NT, 0, g, x0, d, ws);
  launch_k(sm, k_cg_init_final, 1, NT, 0, ws, st);
  ctx->launches += 2;
  if (x0) {
    launch_k(sm, k_cg_setup_x, NB, NT, 0, x0, st, d, x);
    ctx->launches++;
    op.apply(ctx, x, ap, &st->gv_skip);
  } else {
    cudaMemsetAsync(x, 0, sizeof(float) * d, sm);
  }
  unsigned* ctr = ctx->amax_counter + 1;
  CgFusedArgs fa{};
  int fq = 0;
  if (s && (int)s->off.size() <= kOffTabMax && cg_fused_enabled()) {
    fa = CgFusedArgs{x, r, p, ap, precond, flam, ffl, st, d, ws, ctx->amax_counter + 16, 0, maxiter, tol,
                     make_off_tab(s->off, d), ctx->amax_ws, ctx->amax_ws + kAmaxWsFloats + kOffTabMax, s->v_sc,
                     s->prod_sc, s->n_prod, s->v_hi, s->v_lo};
    fq = cg_fused_nq(d, fa.t, x, r, p, ap, precond, s->v_hi, s->v_lo);
    if (fq && (((uintptr_t)g & 15) || !cg_fused_fits(fq))) fq = 0;
  }
  if (fq) {  // r0, p0, p0's scales and split in one launch
    launch_cg_start(sm, fq, fa, g);
    ctx->launches++;
    s->v_ready = 2;
  } else {
    launch_k(sm, k_cg_r0, NB, NT, 0, g, ap, x, flam, st, d, r, ws);
    launch_k(sm, k_cg_r0_final, 1, NT, 0, ws, st, tol);
    launch_k(sm, k_cg_p0, NB, NT, 0, r, precond, flam, ffl, st, d, p, ws);
    launch_k(sm, k_cg_p0_final, 1, NT, 0, ws, st);
    ctx->launches += 4;
  }
  for (int k = 1; k <= maxiter; ++k) {
    const int is_stab = (stab > 0 && k % stab == 0) ? 1 : 0;
    op.apply(ctx, p, ap, &st->done);
    if (!is_stab && fq) {  // pap, update, direction, scales and split in one launch
      fa.k = k;
      launch_cg_fused(sm, fq, fa);
      ctx->launches++;
      if (k == maxiter) break;
      s->v_ready = 2;
      continue;
    }
    if (is_stab && fq) {  // pap, x update and x's split in one launch
      fa.k = k;
      launch_cg_fused(sm, fq, fa, true);
      ctx->launches++;
      s->v_ready = 2;
    } else {
      launch_k(sm, k_cg_pap, NB, NT, 0, ap, p, flam, st, d, ws, ctr, k, is_stab);
      ctx->launches++;
    }
    if (is_stab) {
      if (!fq) {
        launch_k(sm, k_cg_xupdate, NB, NT, 0, x, p, st, d);
        ctx->launches++;
      }
      op.apply(ctx, x, ap, &st->gv_skip);
      launch_k(sm, k_cg_rstab, NB, NT, 0, g, ap, x, r, precond, flam, ffl, st, d, ws, ctr, k, maxiter, tol);
    } else {
      launch_k(sm, k_cg_update, NB, NT, 0, x, r, p, ap, precond, flam, ffl, st, d, ws, ctr, k, maxiter, tol);
    }
    ctx->launches++;
    if (k == maxiter) break;  // the direction of a last iteration is never used
    // p <- M^-1 r + beta p, fused with the next product's input scales
    if (s && cg_pnext_amax(ctx, r, precond, flam, ffl, &st->alpha, &st->done, p, d, s->off, s->v_sc, s->prod_sc,
                           s->n_prod)) {
      s->v_ready = 1;
    } else {
      launch_k(sm, k_cg_pnext, NB, NT, 0, r, precond, flam, ffl, st, d, p);
      ctx->launches++;
    }
  }
  launch_k(sm, k_cg_finish, 1, 1, 0, st, stats);
  ctx->launches++;
}

// Data-parallel CG with sharded vectors (world ranks, batch-sharded products).  Rank r
// owns [r*chunk, (r+1)*chunk) of x, r, p and Ap: the summed product is reduced only onto
// its owners (reduce_to_owners, per layer as the weight gradients finish), the update,
// residual and direction passes run on d/world elements, each reduction is a few-double
// all-reduce of per-rank totals followed by the replicated decision, and p (and x before
// a stabilising product, and at the end) is all-gathered for the next product.  Same
// recurrence and decisions as cg_run (solvers.py:60-114); only the summation order of
// the dot products differs.
static void cg_run_sharded(cv_ctx* ctx, const CgOperator& op, const float* g, double lam, double tol, int maxiter,
                           int stab, const float* precond, double floor, const float* x0, float* x,
                           cv_cg_stats* stats) {
  const int64_t d = op.d;
  const int W = ctx->world, R = ctx->rank;
  const int64_t chunk = ((d + W - 1) / W + 63) / 64 * 64;  // 256-byte aligned shards
  const int64_t lo = std::min(d, (int64_t)R * chunk);
  const int64_t n = std::max<int64_t>(0, std::min(d, lo + chunk) - lo);
  const int64_t dp = chunk * W;
  CgDev* st = (CgDev*)(ctx->scal_ws + 8);
  double* ws = ctx->red_ws;
  cudaStream_t sm = ctx->stream;
  const float flam = (float)lam, ffl = (float)floor;
  float* buf = (float*)ctx->pool.get(sizeof(float) * 4 * dp);
  double* tot = (double*)ctx->pool.get(sizeof(double) * (8 + W));
  float *xs = buf, *r = buf + dp, *p = buf + 2 * dp, *ap = buf + 3 * dp;
  cudaMemsetAsync(buf, 0, sizeof(float) * 4 * dp, sm);  // padding beyond d stays finite
  const float* gl = g + lo;
  const float* pre = precond ? precond + lo : nullptr;
  float *xl = xs + lo, *rl = r + lo, *pl = p + lo, *apl = ap + lo;

  auto decide = [&](int what, int nv, int k, int is_stab) {
    allreduce_f64(ctx, tot, nv);
    launch_k(sm, k_cgs_decide, 1, 1, 0, (const double*)tot, st, what, k, maxiter, is_stab, tol, W);
    ctx->launches += 2;
  };
  auto product = [&](const float* in, const int* skip) {
    ctx->shard_chunk = chunk;
    try {
      op.apply(ctx, in, ap, skip);
    } catch (...) {
      ctx->shard_chunk = 0;
      throw;
    }
    ctx->shard_chunk = 0;
  };

  launch_k(sm, k_cg_init, NB, NT, 0, gl, x0 ? x0 + lo : nullptr, n, ws);
  launch_k(sm, k_cgs_total<2>, 1, NT, 0, (const double*)ws, tot);
  decide(CGS_INIT, 2, 0, 0);
  if (x0) {
    launch_k(sm, k_cg_setup_x, NB, NT, 0, x0, (const CgDev*)st, d, xs);  // whole x: the product's input
    ctx->launches++;
    product(xs, &st->gv_skip);
  }
  launch_k(sm, k_cg_r0, NB, NT, 0, gl, (const float*)apl, (const float*)xl, flam, (const CgDev*)st, n, rl, ws);
  launch_k(sm, k_cgs_total<1>, 1, NT, 0, (const double*)ws, tot);
  decide(CGS_R0, 1, 0, 0);
  launch_k(sm, k_cg_p0, NB, NT, 0, (const float*)rl, pre, flam, ffl, (const CgDev*)st, n, pl, ws);
  launch_k(sm, k_cgs_total<1>, 1, NT, 0, (const double*)ws, tot);
  decide(CGS_P0, 1, 0, 0);
  allgather_f32(ctx, p, chunk);
  ctx->launches += 6;
  for (int k = 1; k <= maxiter; ++k) {
    const int is_stab = (stab > 0 && k % stab == 0) ? 1 : 0;
    product(p, &st->done);
    launch_k(sm, k_cg_pap, NB, NT, 0, apl, (const float*)pl, flam, st, n, ws, (unsigned*)nullptr, k, is_stab);
    launch_k(sm, k_cgs_pap_total, 1, NT, 0, (const double*)ws, tot, R, W);
    decide(CGS_PAP, 2 + W, k, is_stab);
    if (is_stab) {
      launch_k(sm, k_cg_xupdate, NB, NT, 0, xl, (const float*)pl, (const CgDev*)st, n);
      allgather_f32(ctx, xs, chunk);
      product(xs, &st->gv_skip);
      launch_k(sm, k_cg_rstab, NB, NT, 0, gl, (const float*)apl, (const float*)xl, rl, pre, flam, ffl, st, n, ws,
               (unsigned*)nullptr, k, maxiter, tol);
    } else {
      launch_k(sm, k_cg_update, NB, NT, 0, xl, rl, (const float*)pl, (const float*)apl, pre, flam, ffl, st, n, ws,
               (unsigned*)nullptr, k, maxiter, tol);
    }
    launch_k(sm, k_cgs_total<2>, 1, NT, 0, (const double*)ws, tot);
    decide(CGS_R, 2, k, is_stab);
    ctx->launches += 4 + is_stab;
    if (k == maxiter) break;
    launch_k(sm, k_cg_pnext, NB, NT, 0, (const float*)rl, pre, flam, ffl, (const CgDev*)st, n, pl);
    allgather_f32(ctx, p, chunk);
    ctx->launches++;
  }
  allgather_f32(ctx, xs, chunk);
  cudaMemcpyAsync(x, xs, sizeof(float) * d, cudaMemcpyDeviceToDevice, sm);
  launch_k(sm, k_cg_finish, 1, 1, 0, (const CgDev*)st, stats);
  ctx->launches++;
  ctx->pool.put(buf);
  ctx->pool.put(tot);
}

}  // namespace cv
