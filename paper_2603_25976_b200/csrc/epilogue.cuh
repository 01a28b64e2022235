// Element-wise epilogue shared by the SIMT, skinny and tensor-core GEMMs.
#pragma once
#include "common.cuh"
#include "internal.h"

namespace cv {

CV_DEV float ld_op(const Operand& o, int64_t i, int64_t j) {
  const int64_t idx = i * o.si + j * o.sj;
  float v = o.hi[idx];
  if (o.lo) v += o.lo[idx];
  return v;
}

// Epilogue for one output element (m, n) with accumulator v.
CV_DEV void epi_apply(const Epilogue& e, int m, int n, float v) {
  switch (e.mode) {
    case EPI_STORE:
      e.out[(int64_t)m * e.ld + n] = v;
      return;
    case EPI_SPLIT_ACT: {
      float a = e.act == CV_ACT_RELU ? relu_f(v) : tanhf(v);
      float h, l;
      split2(a, h, l);
      e.out_hi[(int64_t)m * e.ld + n] = h;
      e.out_lo[(int64_t)m * e.ld + n] = l;
      return;
    }
    case EPI_SPLIT_MASK:
    case EPI_HVP: {
      if (e.raw) e.raw[(int64_t)m * e.raw_ld + n] = v;
      const int64_t mi = (int64_t)(m / e.mask_div) * e.mask_ld + n;
      float a = e.mask_hi[mi];
      if (e.act == CV_ACT_TANH) a += e.mask_lo[mi];
      const float sp = act_deriv(e.act, a);
      float r = v * sp;
      if (e.mode == EPI_HVP && e.act == CV_ACT_TANH) {
        // (G W^T) * spp * dz with spp = -2 a sp  (models.py:192-197, 305-306)
        r += e.P[(int64_t)m * e.P_ld + n] * (-2.f * a * sp) * e.dz[(int64_t)m * e.dz_ld + n];
      }
      float h, l;
      split2(r, h, l);
      e.out_hi[(int64_t)m * e.ld + n] = h;
      e.out_lo[(int64_t)m * e.ld + n] = l;
      return;
    }
    case EPI_GRAM: {
      const float sa = e.sa[(int64_t)(m / e.kdiv) * e.sa_ld + n / e.kdiv];
      float* o = e.out + (int64_t)m * e.ld + n;
      *o = e.first ? v * sa : *o + v * sa;
      return;
    }
    case EPI_ACCUM: {
      float* o = e.out + (int64_t)m * e.ld + n;
      *o += e.alpha * v;
      return;
    }
  }
}

CV_DEV bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// NC (multiple of 4) consecutive columns [nb, nb+NC) of row m with 128-bit accesses.
// Returns false (nothing written) when the row segment is not 16-byte aligned; the
// caller then falls back to the per-element path.
template <int NC>
CV_DEV bool epi_applyV(const Epilogue& e, int m, int nb, const float (&v)[NC]) {
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
      float* oh = e.out_hi + o;
      float* ol = e.out_lo + o;
      if (!al16(oh) || !al16(ol)) return false;
#pragma unroll
      for (int j = 0; j < NC; j += 4) {
        float h[4], l[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) split2(e.act == CV_ACT_RELU ? relu_f(v[j + t]) : tanhf(v[j + t]), h[t], l[t]);
        *reinterpret_cast<float4*>(oh + j) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(ol + j) = make_float4(l[0], l[1], l[2], l[3]);
      }
      return true;
    }
    case EPI_SPLIT_MASK:
    case EPI_HVP: {
      const bool tanh_ = e.act == CV_ACT_TANH;
      const bool hvp_t = e.mode == EPI_HVP && tanh_;
      float* oh = e.out_hi + o;
      float* ol = e.out_lo + o;
      const int64_t mo = (int64_t)(m / e.mask_div) * e.mask_ld + nb;
      const float* mh = e.mask_hi + mo;
      const float* ml = e.mask_lo + mo;
      float* raw = e.raw ? e.raw + (int64_t)m * e.raw_ld + nb : nullptr;
      const float* P = hvp_t ? e.P + (int64_t)m * e.P_ld + nb : nullptr;
      const float* dz = hvp_t ? e.dz + (int64_t)m * e.dz_ld + nb : nullptr;
      if (!al16(oh) || !al16(ol) || !al16(mh) || (tanh_ && !al16(ml)) || (raw && !al16(raw)) ||
          (hvp_t && (!al16(P) || !al16(dz))))
        return false;
#pragma unroll
      for (int j = 0; j < NC; j += 4) {
        const float4 a4 = *reinterpret_cast<const float4*>(mh + j);
        float a[4] = {a4.x, a4.y, a4.z, a4.w};
        if (tanh_) {
          const float4 l4 = *reinterpret_cast<const float4*>(ml + j);
          a[0] += l4.x; a[1] += l4.y; a[2] += l4.z; a[3] += l4.w;
        }
        if (raw) *reinterpret_cast<float4*>(raw + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        float r[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) r[t] = v[j + t] * act_deriv(e.act, a[t]);
        if (hvp_t) {
          const float4 p4 = *reinterpret_cast<const float4*>(P + j);
          const float4 z4 = *reinterpret_cast<const float4*>(dz + j);
          const float pp[4] = {p4.x, p4.y, p4.z, p4.w}, zz[4] = {z4.x, z4.y, z4.z, z4.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) r[t] += pp[t] * (-2.f * a[t] * act_deriv(e.act, a[t])) * zz[t];
        }
        float h[4], l[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) split2(r[t], h[t], l[t]);
        *reinterpret_cast<float4*>(oh + j) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(ol + j) = make_float4(l[0], l[1], l[2], l[3]);
      }
      return true;
    }
    case EPI_GRAM: {
      float* out = e.out + o;
      const float* sa = e.sa + (int64_t)(m / e.kdiv) * e.sa_ld;
      if (!al16(out)) return false;
#pragma unroll
      for (int j = 0; j < NC; j += 4) {
        float4 cur = e.first ? make_float4(0.f, 0.f, 0.f, 0.f) : *reinterpret_cast<float4*>(out + j);
        cur.x += v[j] * sa[(nb + j) / e.kdiv];
        cur.y += v[j + 1] * sa[(nb + j + 1) / e.kdiv];
        cur.z += v[j + 2] * sa[(nb + j + 2) / e.kdiv];
        cur.w += v[j + 3] * sa[(nb + j + 3) / e.kdiv];
        *reinterpret_cast<float4*>(out + j) = cur;
      }
      return true;
    }
    case EPI_ACCUM: {
      float* out = e.out + o;
      if (!al16(out)) return false;
#pragma unroll
      for (int j = 0; j < NC; j += 4) {
        float4 cur = *reinterpret_cast<float4*>(out + j);
        cur.x += e.alpha * v[j];
        cur.y += e.alpha * v[j + 1];
        cur.z += e.alpha * v[j + 2];
        cur.w += e.alpha * v[j + 3];
        *reinterpret_cast<float4*>(out + j) = cur;
      }
      return true;
    }
  }
  return false;
}

CV_DEV bool epi_apply32(const Epilogue& e, int m, int nb, const float (&v)[32]) { return epi_applyV<32>(e, m, nb, v); }

}  // namespace cv
