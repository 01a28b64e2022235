// Shared device/host helpers for the curvopt_b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#define CV_DEV __device__ __forceinline__

namespace cv {

constexpr int kRedBlocks = 592;    // 4 x 148 SMs; fixed => deterministic reductions
constexpr int kRedThreads = 256;

// Round-to-nearest (ties away) fp32 -> tf32, returned as an fp32 bit pattern with
// the low 13 mantissa bits cleared.  The tensor core consumes exactly these bits.
CV_DEV float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// x ~= hi + lo, both exact tf32 values (|x - hi - lo| <= 2^-22 |x|).  lo is rounded
// to nearest here rather than left with 13 significant bits: the tensor core
// truncates operand bits beyond tf32, which biases every 3xTF32 product toward
// zero (measured -8e-7 relative, amplified ~20x by the per-example cancellation
// in the weight gradients).
CV_DEV void split2(float x, float& hi, float& lo) {
  hi = tf32_rna(x);
  lo = tf32_rna(x - hi);
}

CV_DEV float relu_f(float x) { return x > 0.f ? x : 0.f; }

// Activation derivative from the stored activation value a = act(z)
// (relu: z > 0  <=>  a > 0, models.py:351-353; tanh: 1 - a^2, models.py:355-356).
CV_DEV float act_deriv(int act, float a) { return act == 0 ? (a > 0.f ? 1.f : 0.f) : 1.f - a * a; }

template <typename T>
CV_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

CV_DEV double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum of NV doubles (blockDim.x == kRedThreads). Result valid in thread 0.
template <int NV>
CV_DEV void block_sum(double (&v)[NV]) {
  __shared__ double sh[NV][kRedThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double t = warp_sum(v[i]);
    if (lane == 0) sh[i][w] = t;
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double t = lane < kRedThreads / 32 ? sh[i][lane] : 0.0;
      v[i] = warp_sum(t);
    }
  }
  __syncthreads();
}

CV_DEV bool skip_if(const int* flag) { return flag != nullptr && *(volatile const int*)flag != 0; }

}  // namespace cv
