// Shared device/host helpers for the curvopt_b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <stdlib.h>
#include <cuda_fp16.h>

#define CV_DEV __device__ __forceinline__

// Programmatic dependent launch: every kernel is launched with programmatic
// stream serialization (launch_k) and starts by waiting for its predecessor grid
// (full completion + memory flush, so RAW/WAR hazards are as with plain stream
// order) and then allowing its own successor to be scheduled.  The successor's
// launch and prologue thus overlap this kernel's tail instead of following it.
#define CV_PDL_ENTRY()                                        \
  do {                                                        \
    asm volatile("griddepcontrol.wait;" ::: "memory");        \
    asm volatile("griddepcontrol.launch_dependents;" :::);    \
  } while (0)

namespace cv {

inline int pdl_enabled() {
  static const int on = !(getenv("CURVOPT_PDL") && getenv("CURVOPT_PDL")[0] == '0');
  return on;
}

template <typename... KArgs, typename... Args>
inline void launch_k(cudaStream_t st, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

constexpr int kRedBlocks = 592;    // 4 x 148 SMs; fixed => deterministic reductions
constexpr int kRedThreads = 256;

// ---------------------------------------------------------------------------
// Scaled fp16 split ("3xFP16"): a tensor X is stored as two fp16 planes with one
// power-of-two exponent e per tensor,
//     X ~= (hi + lo) * 2^-e,   hi = rn(X 2^e),  lo = rn(X 2^e - hi),
// which carries 22 significant bits (|X - (hi+lo)2^-e| <= 2^-22 |X| for entries
// whose scaled magnitude is >= 2^-3; smaller entries keep an absolute error of
// 2^-25 in scaled units).  e is chosen from a rigorous bound B >= max|X| so that
// B 2^e <= 2^14: no overflow is possible and the scaled range keeps 14 binades of
// headroom above fp16's subnormal floor.  The tensor core consumes the fp16
// planes at twice the TF32 rate (hi.hi + hi.lo + lo.hi, fp32 accumulation).
// ---------------------------------------------------------------------------
struct Scale {
  int e;        // X = (hi + lo) * 2^-e
  float amax;   // max |X| of the stored tensor (true scale), maintained by its producer
};

// 2^e as a float for |e| <= 126
CV_DEV float pow2f(int e) { return __int_as_float((127 + e) << 23); }

// largest e with B * 2^e <= 2^14; 0 for zero / non-finite bounds (then the data
// itself is zero or non-finite and the scale is irrelevant)
CV_DEV int exp_for_bound(float B) {
  if (!(B > 0.f) || !(B < 3.0e38f)) return 0;
  int x;
  frexpf(B, &x);  // B = f 2^x, f in [0.5, 1)  =>  B < 2^x
  int e = 14 - x;
  return e < -100 ? -100 : (e > 100 ? 100 : e);
}

CV_DEV void split16(float x, float s, __half& hi, __half& lo) {
  const float xs = x * s;
  hi = __float2half_rn(xs);
  lo = __float2half_rn(xs - __half2float(hi));
}

CV_DEV float join16(__half hi, __half lo, float inv) { return (__half2float(hi) + __half2float(lo)) * inv; }

// max|x| of non-negative float bit patterns via integer atomicMax (exact, order free)
CV_DEV void atomic_amax(float* slot, float v) {
  if (slot && v > 0.f) atomicMax(reinterpret_cast<int*>(slot), __float_as_int(v));
  else if (slot && !(v == v)) atomicMax(reinterpret_cast<int*>(slot), 0x7fc00000);  // NaN poisons the bound
}

CV_DEV float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
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
