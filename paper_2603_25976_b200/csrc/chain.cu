// Device transform chain (transforms.py:148-199) and the step tail (method.py:345-357),
// plus the sampled-label GNB diagonal estimator (telemetry.py:129-160).
//
// A chain is applied element-wise in ONE pass per clip_global_norm-delimited segment:
// every link but clip_global_norm is element-local, so a segment's kernel reads the
// direction (or the previous segment's output), the link states and w once, applies
// the links in order in registers and writes the new link states.  A segment that
// ends at a clip link also reduces ||x||^2 (fixed-order fp64 partials) and its last
// block turns it into the clip factor the next segment multiplies in; the last
// segment writes update = x and w_next = w + x and reduces the step's norms and
// non-finite counts.  No host synchronisation.
#include "common.cuh"
#include "internal.h"
#include "vecutil.cuh"

#include <math.h>

#include <stdexcept>
#include <string>

namespace cv {

struct DevLink {
  int kind;
  float p[7];
  const float* in0;
  const float* in1;
  float* out0;
  float* out1;
};

constexpr int kSegMax = 8;
struct Seg {
  int n;
  DevLink l[kSegMax];
};

// the segment's links on W consecutive elements starting at i (x in registers)
template <int W>
CV_DEV void chain_links(const Seg& sg, Vf<W>& x, int64_t i, const float* w, const float* pre) {
#pragma unroll 1
  for (int k = 0; k < sg.n; ++k) {
    const DevLink& L = sg.l[k];
    switch (L.kind) {
      case CV_LINK_SCALE:
#pragma unroll
        for (int j = 0; j < W; ++j) x.v[j] *= L.p[0];
        break;
      case CV_LINK_TRACE_MOMENTUM: {  // m = beta trace + x; x = m
        const Vf<W> t = ldv<W>(L.in0 + i);
#pragma unroll
        for (int j = 0; j < W; ++j) x.v[j] = fmaf(L.p[0], t.v[j], x.v[j]);
        stv<W>(L.out0 + i, x);
        break;
      }
      case CV_LINK_ADD_DECAYED_WEIGHTS: {
        const Vf<W> wv = ldv<W>(w + i);
#pragma unroll
        for (int j = 0; j < W; ++j) x.v[j] = fmaf(L.p[0], wv.v[j], x.v[j]);
        break;
      }
      case CV_LINK_SCALE_BY_ADAM: {
        // m = b1 m + (1-b1) x; v = b2 v + (1-b2) x^2; x = m/(1-b1^t) / (sqrt(v/(1-b2^t)) + eps)
        const Vf<W> m0 = ldv<W>(L.in0 + i), v0 = ldv<W>(L.in1 + i);
        Vf<W> m, v;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          m.v[j] = L.p[0] * m0.v[j] + L.p[1] * x.v[j];
          v.v[j] = L.p[2] * v0.v[j] + L.p[3] * (x.v[j] * x.v[j]);
          x.v[j] = (m.v[j] * L.p[5]) / (sqrtf(v.v[j] * L.p[6]) + L.p[4]);
        }
        stv<W>(L.out0 + i, m);
        stv<W>(L.out1 + i, v);
        break;
      }
      case CV_LINK_SOPHIA_CLIP: {  // x = clip(x / max(gamma diag, eps), -1, 1)
        const Vf<W> dv = ldv<W>(pre + i);
#pragma unroll
        for (int j = 0; j < W; ++j) x.v[j] = fminf(fmaxf(x.v[j] / fmaxf(L.p[0] * dv.v[j], L.p[1]), -1.f), 1.f);
        break;
      }
      default:
        break;
    }
  }
}

// One segment.  src = direction (first segment) or the previous segment's output,
// scaled by the previous clip factor *fac_in.  Not last: dst = the segment output,
// the last block writes the clip factor of max_norm into *fac_out.  Last: dst =
// update, wn = w + update, scal[0] = ||update||.  scal[1] accumulates the non-finite
// count of (direction, update, w_next), scal[2] = ||direction||^2 (first segment).
__global__ void k_chain_seg(const Seg sg, const float* src, const double* fac_in, const float* w, const float* pre,
                            int64_t d, int first, int last, int al, float* dst, float* wn, float max_norm,
                            double* fac_out, double* scal, double* ws, unsigned* ctr) {
  CV_PDL_ENTRY();
  const float fac = fac_in ? (float)*fac_in : 1.f;
  double t[3] = {0.0, 0.0, 0.0};
  vec_for(d, al != 0, [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    Vf<W> x = ldv<W>(src + i);
    if (first) {
#pragma unroll
      for (int j = 0; j < W; ++j) {
        t[1] += isfinite(x.v[j]) ? 0.0 : 1.0;
        t[2] += (double)x.v[j] * x.v[j];
      }
    }
#pragma unroll
    for (int j = 0; j < W; ++j) x.v[j] *= fac;
    chain_links<W>(sg, x, i, w, pre);
    stv<W>(dst + i, x);
    if (last) {
      const Vf<W> wv = ldv<W>(w + i);
      Vf<W> nx;
#pragma unroll
      for (int j = 0; j < W; ++j) {
        nx.v[j] = wv.v[j] + x.v[j];
        t[1] += (isfinite(x.v[j]) && isfinite(nx.v[j])) ? 0.0 : 1.0;
      }
      stv<W>(wn + i, nx);
    }
#pragma unroll
    for (int j = 0; j < W; ++j) t[0] += (double)x.v[j] * x.v[j];
  });
  write_partials<3>(ws, t);
  if (grid_last(ctr)) {
    double s[3];
    sum_partials<3>(ws, s);
    if (threadIdx.x == 0) {
      const double nrm = sqrt(s[0]);
      if (first) {
        scal[1] = s[1];
        scal[2] = s[2];
      } else {
        scal[1] += s[1];
      }
      if (last) {
        scal[0] = nrm;
      } else {
        // transforms.py:176-180: scale only when the norm exceeds max_norm (NaN: no scaling)
        *fac_out = (nrm > (double)max_norm && nrm > 0.0) ? (double)max_norm / nrm : 1.0;
      }
    }
  }
}

void chain_apply(cv_ctx* ctx, int n_links, const cv_link* links, const float* dir, const float* w, const float* pre,
                 int64_t d, float* upd, float* wn, double* scal) {
  // split at clip links: segments [s0, clip) ... each non-last segment ends at a clip
  std::vector<Seg> segs(1);
  std::vector<float> clips;
  segs[0].n = 0;
  bool al = (((uintptr_t)dir | (uintptr_t)w | (uintptr_t)upd | (uintptr_t)wn | (uintptr_t)pre) & 15) == 0;
  for (int k = 0; k < n_links; ++k) {
    const cv_link& L = links[k];
    if (L.kind == CV_LINK_CLIP_GLOBAL_NORM) {
      clips.push_back((float)L.p[0]);
      segs.emplace_back();
      segs.back().n = 0;
      continue;
    }
    if (L.kind < CV_LINK_SCALE || L.kind > CV_LINK_SOPHIA_CLIP)
      throw std::invalid_argument("unknown transform link kind " + std::to_string(L.kind));
    Seg& sg = segs.back();
    if (sg.n >= kSegMax) throw std::invalid_argument("too many links between clip_global_norm links");
    DevLink& D = sg.l[sg.n++];
    D.kind = L.kind;
    for (int q = 0; q < 7; ++q) D.p[q] = (float)L.p[q];
    D.in0 = L.state_in[0];
    D.in1 = L.state_in[1];
    D.out0 = L.state_out[0];
    D.out1 = L.state_out[1];
    if (L.kind == CV_LINK_TRACE_MOMENTUM && (!D.in0 || !D.out0))
      throw std::invalid_argument("trace_momentum needs its trace state");
    if (L.kind == CV_LINK_SCALE_BY_ADAM && (!D.in0 || !D.in1 || !D.out0 || !D.out1))
      throw std::invalid_argument("scale_by_adam needs its moment states");
    if (L.kind == CV_LINK_SOPHIA_CLIP && !pre)
      throw std::invalid_argument("sophia_clip requires a preconditioner diagonal");
    if (L.kind == CV_LINK_ADD_DECAYED_WEIGHTS && !w) throw std::invalid_argument("add_decayed_weights needs w");
    al = al && ((((uintptr_t)D.in0 | (uintptr_t)D.in1 | (uintptr_t)D.out0 | (uintptr_t)D.out1) & 15) == 0);
  }
  const int ns = (int)segs.size();
  float* tmp = ns > 1 ? (float*)ctx->pool.get(sizeof(float) * (size_t)d) : nullptr;
  double* fac = ctx->scal_ws + 40;  // clip factors, ping-pong
  unsigned* ctr = ctx->amax_counter + 2;
  const float* src = dir;
  for (int q = 0; q < ns; ++q) {
    const bool last = q == ns - 1;
    const double* fin = q > 0 ? fac + ((q - 1) & 1) : nullptr;
    double* fout = last ? nullptr : fac + (q & 1);
    float* dst = last ? upd : tmp;
    launch_k(ctx->stream, k_chain_seg, kRedBlocks, kRedThreads, 0, segs[q], src, fin, w, pre, d, q == 0 ? 1 : 0,
             last ? 1 : 0, al ? 1 : 0, dst, wn, last ? 0.f : clips[q], fout, scal, ctx->red_ws, ctr);
    ctx->launches++;
    src = tmp;
  }
  if (tmp) ctx->pool.put(tmp);
}

// ---------------------------------------------------------------------------
// GNB diagonal (telemetry.py:129-160): per round, labels sampled from the softmax
// by inverse CDF against the reference's uniform stream, cotangent (p - onehot)/b,
// one VJP, acc += b * g^2.  Uniform j of a round is draw counter + 1 + j of
// Rng.uniform(b_global) (numeric.py:130-132); a rank's rows start at row_offset.
// ---------------------------------------------------------------------------
__global__ void k_gnb_cot(const float* probs, int b, int c, uint64_t seed, uint64_t counter, int64_t row_offset,
                          float inv_b, float* U) {
  CV_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b) return;
  const uint64_t raw = splitmix(seed, counter + 1 + (uint64_t)(row_offset + i));
  const double u = (double)(raw >> 11) * 0x1p-53;
  const float* p = probs + (int64_t)i * c;
  double cum = 0.0;
  int label = 0;
  for (int j = 0; j < c; ++j) {
    cum += (double)p[j];
    label += u > cum ? 1 : 0;
  }
  if (label > c - 1) label = c - 1;
  for (int j = 0; j < c; ++j) U[(int64_t)i * c + j] = (p[j] - (j == label ? 1.f : 0.f)) * inv_b;
}

__global__ void k_gnb_acc(const float* g, int64_t d, float scale, int first, float* acc) {
  CV_PDL_ENTRY();
  vec_for(d, al16p(g, acc), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    const Vf<W> gv = ldv<W>(g + i);
    Vf<W> a;
    if (!first) a = ldv<W>(acc + i);
#pragma unroll
    for (int j = 0; j < W; ++j) a.v[j] = (first ? 0.f : a.v[j]) + scale * (gv.v[j] * gv.v[j]);
    stv<W>(acc + i, a);
  });
}

__global__ void k_scale_vec(float* x, int64_t d, float s) {
  CV_PDL_ENTRY();
  vec_for(d, al16p(x), [&](auto W_, int64_t i) {
    constexpr int W = decltype(W_)::value;
    Vf<W> v = ldv<W>(x + i);
#pragma unroll
    for (int j = 0; j < W; ++j) v.v[j] *= s;
    stv<W>(x + i, v);
  });
}

void gnb_diag(cv_ctx* ctx, cv_snap* s, uint64_t seed, uint64_t counter, int n_samples, int64_t row_offset,
              float* diag) {
  if (s->loss != CV_LOSS_CE) throw std::invalid_argument("gnb_diag requires a cross-entropy batch");
  if (n_samples < 1) throw std::invalid_argument("gnb_diag requires n_samples >= 1");
  if (row_offset < 0 || row_offset + s->bl > s->bg) throw std::invalid_argument("gnb_diag: row range outside the batch");
  float* gh = (float*)ctx->pool.get(sizeof(float) * (size_t)s->d);
  for (int r = 0; r < n_samples; ++r) {
    launch_k(ctx->stream, k_gnb_cot, (s->bl + 127) / 128, 128, 0, (const float*)s->probs, s->bl, s->c, seed,
             counter + (uint64_t)r * (uint64_t)s->bg, row_offset, 1.f / (float)s->bg, s->U2);
    ctx->launches++;
    mlp_vjp(ctx, s, s->U2, gh);  // the global gradient for the sampled labels (all-reduced for world > 1)
    launch_k(ctx->stream, k_gnb_acc, kRedBlocks, kRedThreads, 0, (const float*)gh, s->d, (float)s->bg, r == 0 ? 1 : 0,
             diag);
    ctx->launches++;
  }
  if (n_samples > 1) {
    launch_k(ctx->stream, k_scale_vec, kRedBlocks, kRedThreads, 0, diag, s->d, 1.f / (float)n_samples);
    ctx->launches++;
  }
  ctx->pool.put(gh);
}

}  // namespace cv
