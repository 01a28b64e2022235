// Shared helpers of the d-length vector kernels (vec.cu, chain.cu): fixed-grid
// grid-stride loops with 128-bit bodies, fixed-order fp64 block partials, the
// last-block pattern and the SplitMix64 stream.
#pragma once
#include <type_traits>

#include "common.cuh"

namespace cv {

constexpr int NB = kRedBlocks, NT = kRedThreads;
#define GRID_STRIDE(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); \
                               i += (int64_t)gridDim.x * blockDim.x)

// Sum the NV partials of every block (ws[blk*8 + v]); result valid in thread 0.
template <int NV>
CV_DEV void sum_partials(const double* ws, double (&t)[NV]) {
#pragma unroll
  for (int v = 0; v < NV; ++v) t[v] = 0.0;
  for (int b = threadIdx.x; b < NB; b += NT)
#pragma unroll
    for (int v = 0; v < NV; ++v) t[v] += ws[b * 8 + v];
  block_sum<NV>(t);
}

template <int NV>
CV_DEV void write_partials(double* ws, double (&t)[NV]) {
  block_sum<NV>(t);
  if (threadIdx.x == 0)
#pragma unroll
    for (int v = 0; v < NV; ++v) ws[blockIdx.x * 8 + v] = t[v];
}

CV_DEV float4 ld4g(const float* p) { return *reinterpret_cast<const float4*>(p); }

// W consecutive floats (W = 4: one 128-bit access) -- the vector kernels below are
// written once as body(W, i) and run on 4-element groups plus a scalar tail, so
// every thread keeps 16 bytes per stream in flight (what HBM needs at this grid).
template <int W>
struct Vf {
  float v[W];
};
template <int W>
CV_DEV Vf<W> ldv(const float* p) {
  Vf<W> r;
  if constexpr (W == 4) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
  } else {
    r.v[0] = *p;
  }
  return r;
}
template <int W>
CV_DEV void stv(float* p, const Vf<W>& r) {
  if constexpr (W == 4) *reinterpret_cast<float4*>(p) = make_float4(r.v[0], r.v[1], r.v[2], r.v[3]);
  else *p = r.v[0];
}
using W4 = std::integral_constant<int, 4>;
using W1 = std::integral_constant<int, 1>;
CV_DEV bool al16p(const void* a, const void* b = nullptr, const void* c = nullptr, const void* d = nullptr) {
  return (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c | (uintptr_t)d) & 15) == 0;
}
// grid-stride over 4-element groups (when `al`), then the scalar tail
template <typename F>
CV_DEV void vec_for(int64_t n, bool al, F&& body) {
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
  const int64_t nq = al ? (n >> 2) : 0;
  for (int64_t q = t0; q < nq; q += st) body(W4{}, 4 * q);
  for (int64_t i = 4 * nq + t0; i < n; i += st) body(W1{}, i);
}

CV_DEV float minv_of(const float* pre, int64_t i, float lam, float floor_) {
  return pre ? 1.f / (fmaxf(pre[i], floor_) + lam) : 1.f;
}

// grid's last block? (after every block wrote its partials; counter returns to 0)
CV_DEV bool grid_last(unsigned* ctr) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) *ctr = 0;
  return last;
}

// ---------------------------------------------------------------------------
// SplitMix64 (numeric.py:95-104, 124-128, 157-162)
// ---------------------------------------------------------------------------
CV_DEV uint64_t splitmix(uint64_t seed, uint64_t idx) {
  uint64_t x = seed + 0x9E3779B97F4A7C15ull * idx;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// element i (0-based) of rademacher(Rng(seed, counter), n): index counter + 1 + i
CV_DEV float rad(uint64_t seed, uint64_t counter, int64_t i) {
  return (splitmix(seed, counter + 1 + (uint64_t)i) >> 63) ? 1.f : -1.f;
}

}  // namespace cv
