// Generic SIMT fp32 GEMM with the curvature epilogues, plus the skinny
// (output-layer, N = c <= 32) kernels.  The SIMT GEMM is the exact-fp32 path for
// shapes the tcgen05 engine does not take (unaligned widths, tiny test nets) and
// the cross-check for the tensor-core engine; the skinny kernels carry the
// softmax-CE loss Hessian (models.py:199-204) fused into the last-layer tangent.
#include "common.cuh"
#include "internal.h"
#include "epilogue.cuh"

namespace cv {

constexpr int SB_M = 64, SB_N = 64, SB_K = 16;

__global__ void __launch_bounds__(256) k_gemm_simt(GemmArgs a) {
  CV_PDL_ENTRY();
  if (skip_if(a.skip)) return;
  if (a.lower_only && (int)(blockIdx.x * SB_N) > lo_row(a, (int)(blockIdx.y * SB_M + SB_M - 1)) + a.lower_only - 1)
    return;
  __shared__ __align__(16) float As[SB_K][SB_M + 4];
  __shared__ __align__(16) float Bs[SB_K][SB_N + 4];
  const int tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;
  const int m0 = blockIdx.y * SB_M, n0 = blockIdx.x * SB_N;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int s = 0; s < a.nseg; ++s) {
    const GemmSeg& g = a.seg[s];
    const float ainv = op_inv(g.A), binv = op_inv(g.B);
    const bool a_kc = g.A.sj == 1;  // K contiguous in A
    const bool b_nc = g.B.sj == 1;  // N contiguous in B
    for (int k0 = 0; k0 < g.K; k0 += SB_K) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int e = tid + r * 256;
        int mm, kk;
        if (a_kc) { mm = e >> 4; kk = e & 15; } else { kk = e >> 6; mm = e & 63; }
        const int gm = m0 + mm, gk = k0 + kk;
        As[kk][mm] = (gm < a.M && gk < g.K) ? ld_op(g.A, ainv, gm, gk) : 0.f;
        int nn;
        if (b_nc) { kk = e >> 6; nn = e & 63; } else { nn = e >> 4; kk = e & 15; }
        const int gn = n0 + nn, gk2 = k0 + kk;
        Bs[kk][nn] = (gn < a.N && gk2 < g.K) ? ld_op(g.B, binv, gk2, gn) : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < SB_K; ++kk) {
        const float4 av = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
        const float4 bv = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
        const float ar[4] = {av.x, av.y, av.z, av.w};
        const float br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ar[i], br[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
  const EpiRt rt = epi_prepare(a.epi);
  if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) epi_publish(a.epi, rt);
  float amax = 0.f, ramax = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < a.N && (!a.lower_only || n <= lo_row(a, m) + a.lower_only - 1))
        epi_apply(a.epi, rt, m, n, acc[i][j], amax, ramax);
    }
  }
  epi_flush_amax(a.epi, amax, ramax);
}

void gemm_simt(cv_ctx* ctx, const GemmArgs& a) {
  if (a.M <= 0 || a.N <= 0) return;
  dim3 grid((a.N + SB_N - 1) / SB_N, (a.M + SB_M - 1) / SB_M);
  launch_k(a.stream ? a.stream : ctx->stream, k_gemm_simt, grid, 256, 0, a);
  ctx->launches++;
}

}  // namespace cv
