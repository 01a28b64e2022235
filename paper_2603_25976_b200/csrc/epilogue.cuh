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

}  // namespace cv
