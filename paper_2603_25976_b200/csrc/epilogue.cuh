// Element-wise epilogue shared by the SIMT, skinny and tensor-core GEMMs.
//
// Split outputs (activations, tangents, cotangents) are written as scaled fp16
// pairs (common.cuh).  Their exponent comes from a rigorous bound on |acc| built
// from the inputs' amax slots (AccBound), known before the kernel starts; every
// thread derives the same exponent in epi_prepare, one thread publishes it, and
// the producer accumulates the true amax of what it wrote for its consumers.
#pragma once
#include "common.cuh"
#include "internal.h"

namespace cv {

CV_DEV float ld_op(const Operand& o, float inv, int64_t i, int64_t j) {
  const int64_t idx = i * o.si + j * o.sj;
  if (o.f32) return o.f32[idx];
  return join16(o.hi[idx], o.lo[idx], inv);
}

CV_DEV float op_inv(const Operand& o) { return (o.f32 || !o.sc) ? 1.f : pow2f(-o.sc->e); }

// per-kernel constants of an epilogue
struct EpiRt {
  float out_s = 1.f;      // 2^e of the split output
  float mask_inv = 1.f;   // 2^-e of the stored activation
  int out_e = 0;
  int split = 0;
};

CV_DEV bool epi_is_split(int mode) { return mode == EPI_SPLIT_ACT || mode == EPI_SPLIT_MASK || mode == EPI_HVP; }

CV_DEV EpiRt epi_prepare(const Epilogue& e) {
  EpiRt r;
  if (e.mask_sc) r.mask_inv = pow2f(-e.mask_sc->e);
  r.split = epi_is_split(e.mode);
  if (r.split) {
    float B = 0.f;
    for (int t = 0; t < e.bound.n; ++t) B += e.bound.k[t] * *e.bound.x[t] * *e.bound.y[t];
    B *= 1.0009765625f;  // fp32 rounding of the accumulation itself
    if (e.mode == EPI_SPLIT_ACT && e.act == CV_ACT_TANH) B = fminf(B, 1.f);
    if (e.mode == EPI_HVP && e.act == CV_ACT_TANH && e.P_amax && e.dz_amax)
      B += 0.77f * *e.P_amax * *e.dz_amax;  // |2a(1-a^2)| <= 4/(3 sqrt 3)
    if (e.out_unit) B = fmaxf(B, 1.f);
    r.out_e = exp_for_bound(B);
    r.out_s = pow2f(r.out_e);
  }
  return r;
}

// one thread of the kernel that applies the epilogue records the output exponent
CV_DEV void epi_publish(const Epilogue& e, const EpiRt& r) {
  if (r.split && e.out_sc) e.out_sc->e = r.out_e;
}

CV_DEV float mask_val(const Epilogue& e, const EpiRt& rt, int64_t mi) {
  if (e.act == CV_ACT_RELU) return __half2float(e.mask_hi[mi]);  // sign only: hi > 0 <=> a > 0
  return join16(e.mask_hi[mi], e.mask_lo[mi], rt.mask_inv);
}

// Epilogue for one output element (m, n) with accumulator v; amax/ramax collect
// max |written split value| and max |raw| for the caller's atomic publication.
// out += v without returning the old value (L2-side reduction; FTZ: subnormal sums flush)
CV_DEV void red_add_v4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
CV_DEV void red_add_f32(float* p, float v) { asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory"); }

CV_DEV void epi_apply(const Epilogue& e, const EpiRt& rt, int m, int n, float v, float& amax, float& ramax) {
  switch (e.mode) {
    case EPI_STORE:
      e.out[(int64_t)m * e.ld + n] = v;
      return;
    case EPI_SPLIT_ACT: {
      const float a = e.act == CV_ACT_RELU ? relu_f(v) : tanhf(v);
      split16(a, rt.out_s, e.out_hi[(int64_t)m * e.ld + n], e.out_lo[(int64_t)m * e.ld + n]);
      amax = fmaxf(amax, fabsf(a));
      return;
    }
    case EPI_SPLIT_MASK:
    case EPI_HVP: {
      if (e.raw) {
        e.raw[(int64_t)m * e.raw_ld + n] = v;
        ramax = fmaxf(ramax, fabsf(v));
      }
      const int64_t mi = (int64_t)(m / e.mask_div) * e.mask_ld + n;
      const float a = mask_val(e, rt, mi);
      const float sp = act_deriv(e.act, a);
      float r = v * sp;
      if (e.mode == EPI_HVP && e.act == CV_ACT_TANH) {
        // (G W^T) * spp * dz with spp = -2 a sp  (models.py:192-197, 305-306)
        r += e.P[(int64_t)m * e.P_ld + n] * (-2.f * a * sp) * e.dz[(int64_t)m * e.dz_ld + n];
      }
      split16(r, rt.out_s, e.out_hi[(int64_t)m * e.ld + n], e.out_lo[(int64_t)m * e.ld + n]);
      amax = fmaxf(amax, fabsf(r));
      return;
    }
    case EPI_GRAM: {
      const float sa = e.sa[(int64_t)((m + e.row0) / e.kdiv) * e.sa_ld + n / e.kdiv];
      float* o = e.out + (int64_t)m * e.ld + n;
      if (e.first) *o = v * sa;
      else red_add_f32(o, v * sa);
      return;
    }
    case EPI_ACCUM: {
      red_add_f32(e.out + (int64_t)m * e.ld + n, e.alpha * v);
      return;
    }
  }
}

CV_DEV bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }
CV_DEV bool al8(const void* p) { return ((uintptr_t)p & 7) == 0; }

// 8 halves <-> 16 bytes
union H8 {
  uint4 u;
  __half h[8];
};
union H4 {
  uint2 u;
  __half h[4];
};

CV_DEV void split16x8(const float* x, float s, __half* hi, __half* lo) {
  H8 a, b;
#pragma unroll
  for (int t = 0; t < 8; ++t) split16(x[t], s, a.h[t], b.h[t]);
  *reinterpret_cast<uint4*>(hi) = a.u;
  *reinterpret_cast<uint4*>(lo) = b.u;
}

// NC (multiple of 8) consecutive columns [nb, nb+NC) of row m with 128-bit accesses.
// Returns false (nothing written) when the row segment is not 16-byte aligned; the
// caller then falls back to the per-element path.
template <int NC>
CV_DEV bool epi_applyV(const Epilogue& e, const EpiRt& rt, int m, int nb, const float (&v)[NC], float& amax,
                       float& ramax) {
  static_assert(NC % 8 == 0, "vector epilogue works on 8-column groups");
  const int64_t o = (int64_t)m * e.ld + nb;
  switch (e.mode) {
    case EPI_STORE: {
      float* out = e.out + o;
      if (!al16(out)) return false;
#pragma unroll
      for (int j = 0; j < NC; j += 4) *reinterpret_cast<float4*>(out + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      return true;
    }
    case EPI_SPLIT_ACT: {
      __half* oh = e.out_hi + o;
      __half* ol = e.out_lo + o;
      if (!al16(oh) || !al16(ol)) return false;
#pragma unroll
      for (int j = 0; j < NC; j += 8) {
        float a[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          a[t] = e.act == CV_ACT_RELU ? relu_f(v[j + t]) : tanhf(v[j + t]);
          amax = fmaxf(amax, fabsf(a[t]));
        }
        split16x8(a, rt.out_s, oh + j, ol + j);
      }
      return true;
    }
    case EPI_SPLIT_MASK:
    case EPI_HVP: {
      const bool tanh_ = e.act == CV_ACT_TANH;
      const bool hvp_t = e.mode == EPI_HVP && tanh_;
      __half* oh = e.out_hi + o;
      __half* ol = e.out_lo + o;
      const int64_t mo = (int64_t)(m / e.mask_div) * e.mask_ld + nb;
      const __half* mh = e.mask_hi + mo;
      const __half* ml = e.mask_lo + mo;
      float* raw = e.raw ? e.raw + (int64_t)m * e.raw_ld + nb : nullptr;
      const float* P = hvp_t ? e.P + (int64_t)m * e.P_ld + nb : nullptr;
      const float* dz = hvp_t ? e.dz + (int64_t)m * e.dz_ld + nb : nullptr;
      if (!al16(oh) || !al16(ol) || !al16(mh) || (tanh_ && !al16(ml)) || (raw && !al16(raw)) ||
          (hvp_t && (!al16(P) || !al16(dz))))
        return false;
#pragma unroll
      for (int j = 0; j < NC; j += 8) {
        H8 h8;
        h8.u = *reinterpret_cast<const uint4*>(mh + j);
        float a[8];
        if (tanh_) {
          H8 l8;
          l8.u = *reinterpret_cast<const uint4*>(ml + j);
#pragma unroll
          for (int t = 0; t < 8; ++t) a[t] = (__half2float(h8.h[t]) + __half2float(l8.h[t])) * rt.mask_inv;
        } else {
#pragma unroll
          for (int t = 0; t < 8; ++t) a[t] = __half2float(h8.h[t]);
        }
        if (raw) {
          *reinterpret_cast<float4*>(raw + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          *reinterpret_cast<float4*>(raw + j + 4) = make_float4(v[j + 4], v[j + 5], v[j + 6], v[j + 7]);
#pragma unroll
          for (int t = 0; t < 8; ++t) ramax = fmaxf(ramax, fabsf(v[j + t]));
        }
        float r[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) r[t] = v[j + t] * act_deriv(e.act, a[t]);
        if (hvp_t) {
#pragma unroll
          for (int t = 0; t < 8; ++t) r[t] += P[j + t] * (-2.f * a[t] * act_deriv(e.act, a[t])) * dz[j + t];
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) amax = fmaxf(amax, fabsf(r[t]));
        split16x8(r, rt.out_s, oh + j, ol + j);
      }
      return true;
    }
    case EPI_GRAM: {
      float* out = e.out + o;
      const float* sa = e.sa + (int64_t)((m + e.row0) / e.kdiv) * e.sa_ld;
      if (!al16(out)) return false;
#pragma unroll
      // all loads of the row segment first (the stores alias them: issued in one batch
      // the read latency is paid once per chunk, not once per 16 bytes)
      // accumulation: one fire-and-forget vector reduction per 16 bytes (the L2 does the
      // read-modify-write; each element gets exactly one add per GEMM, so the result is
      // the same rounding as load + add + store, without the read round trip in the SM)
      // the example of column nb + j: one division per chunk, then a running (q, r) --
      // a division per element made the epilogue of the K = 16 output-layer term the
      // bottleneck of that GEMM
      int q = nb / e.kdiv, r = nb - q * e.kdiv;
      float f[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        f[j] = v[j] * sa[q];
        if (++r == e.kdiv) {
          r = 0;
          ++q;
        }
      }
#pragma unroll
      for (int j = 0; j < NC; j += 4) {
        const float4 c = make_float4(f[j], f[j + 1], f[j + 2], f[j + 3]);
        if (e.first) *reinterpret_cast<float4*>(out + j) = c;
        else red_add_v4(out + j, c);
      }
      return true;
    }
    case EPI_ACCUM: {
      float* out = e.out + o;
      if (!al16(out)) return false;
#pragma unroll
      for (int j = 0; j < NC; j += 4)
        red_add_v4(out + j, make_float4(e.alpha * v[j], e.alpha * v[j + 1], e.alpha * v[j + 2], e.alpha * v[j + 3]));
      return true;
    }
  }
  return false;
}

// Publish a warp's running maxima (all 32 lanes must call).
CV_DEV void epi_flush_amax(const Epilogue& e, float& amax, float& ramax) {
  if (!e.out_sc && !e.raw_amax) return;  // (uniform) nothing to publish: no warp reduction
  const float a = warp_max_f(amax), r = warp_max_f(ramax);
  if ((threadIdx.x & 31) == 0) {
    if (e.out_sc && a > 0.f) atomic_amax(&e.out_sc->amax, a);
    if (e.raw_amax && r > 0.f) atomic_amax(e.raw_amax, r);
  }
  amax = 0.f;
  ramax = 0.f;
}

}  // namespace cv
