// Output-layer kernels (c = output width <= 32).  All three are HBM-bound streams
// over one b x n activation/tangent matrix, so they are written for bandwidth:
// 128-bit loads/stores, the tiny c-wide operand staged in shared memory, several
// rows or columns per thread in flight, deterministic fixed-order reductions.
//   skinny_rows : last-layer JVP + fused H_z (models.py:243-255, 199-204)
//   skinny_dw   : last-layer [gW; gb] = A^T U (models.py:280-281)
//   skinny_dx   : G = (U W^T) * act'(a) (models.py:282-284, 378-381)
#include "common.cuh"
#include "epilogue.cuh"
#include "internal.h"
#include "skinny.cuh"

namespace cv {

CV_DEV float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// ---------------------------------------------------------------------------
// rows: one warp per RPW rows, lanes stride K in float4 steps, B^T chunk in smem
// ---------------------------------------------------------------------------
template <int CM, int RPW>
__global__ void __launch_bounds__(256) k_rows(SkinnyRowsArgs a) {
  if (skip_if(a.skip)) return;
  constexpr int RK = 8192 / CM;  // K chunk: 32 KB of B^T
  __shared__ __align__(16) float Bt[CM][RK];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int m0 = (blockIdx.x * 8 + w) * RPW;
  float acc[RPW][CM];
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int j = 0; j < CM; ++j) acc[r][j] = 0.f;
  for (int s = 0; s < a.nseg; ++s) {
    const SkinnySeg g = a.seg[s];
    for (int k0 = 0; k0 < g.K; k0 += RK) {
      const int kmax = min(RK, g.K - k0);
      __syncthreads();
      for (int e = threadIdx.x; e < RK * CM; e += 256) {
        const int kk = e % RK, j = e / RK;
        float v = 0.f;
        if (kk < kmax && j < a.c) {
          const int64_t idx = (int64_t)(k0 + kk) * g.ldb + j;
          v = g.b_hi[idx] + g.b_lo[idx];
        }
        Bt[j][kk] = v;
      }
      __syncthreads();
      for (int kk = lane * 4; kk < kmax; kk += 128) {
        float av[RPW][4];
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
          const int m = m0 + r;
          if (m < a.rows) {
            const float* ph = g.a_hi + (int64_t)m * g.lda + k0 + kk;
            const float* pl = g.a_lo + (int64_t)m * g.lda + k0 + kk;
            if (kk + 3 < kmax) {
              const float4 h = ld4(ph), l = ld4(pl);
              av[r][0] = h.x + l.x; av[r][1] = h.y + l.y; av[r][2] = h.z + l.z; av[r][3] = h.w + l.w;
            } else {
#pragma unroll
              for (int t = 0; t < 4; ++t) av[r][t] = kk + t < kmax ? ph[t] + pl[t] : 0.f;
            }
          } else {
#pragma unroll
            for (int t = 0; t < 4; ++t) av[r][t] = 0.f;
          }
        }
#pragma unroll
        for (int j = 0; j < CM; ++j) {
          const float4 b4 = *reinterpret_cast<const float4*>(&Bt[j][kk]);
#pragma unroll
          for (int r = 0; r < RPW; ++r)
            acc[r][j] = fmaf(av[r][0], b4.x, fmaf(av[r][1], b4.y, fmaf(av[r][2], b4.z, fmaf(av[r][3], b4.w, acc[r][j]))));
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
#pragma unroll
    for (int j = 0; j < CM; ++j) acc[r][j] = warp_sum(acc[r][j]);
    const int m = m0 + r;
    if (m >= a.rows) continue;
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < CM; ++j)
      if (j == lane) t = acc[r][j];
    if (a.post == POST_LOGITS || a.loss == CV_LOSS_MSE) {
      if (lane < a.c) a.out[(int64_t)m * a.c + lane] = a.post == POST_LOGITS ? t : t * a.scale;
    } else {
      // H_z T = p*T - p*(p.T)  (softmax-CE, per example)
      const float* p = a.probs + (int64_t)m * a.c;
      float pt = 0.f;
#pragma unroll
      for (int j = 0; j < CM; ++j)
        if (j < a.c) pt = fmaf(p[j], acc[r][j], pt);
      if (lane < a.c) {
        const float pj = p[lane];
        a.out[(int64_t)m * a.c + lane] = (pj * t - pj * pt) * a.scale;
      }
    }
  }
}

void skinny_rows(cv_ctx* ctx, const SkinnyRowsArgs& a) {
  if (a.c <= 16) {
    constexpr int RPW = 4;
    k_rows<16, RPW><<<(a.rows + 8 * RPW - 1) / (8 * RPW), 256, 0, ctx->stream>>>(a);
  } else {
    constexpr int RPW = 2;
    k_rows<32, RPW><<<(a.rows + 8 * RPW - 1) / (8 * RPW), 256, 0, ctx->stream>>>(a);
  }
  ctx->launches++;
}

// ---------------------------------------------------------------------------
// dx: block = 32 rows x NT columns; thread = 4 adjacent columns x 8 rows; W^T tile
// and U rows in smem; 128-bit fused epilogue
// ---------------------------------------------------------------------------
template <int CM, int NT>
__global__ void __launch_bounds__(256) k_dx(SkinnyDxArgs a) {
  if (skip_if(a.skip)) return;
  constexpr int RB = 32;
  constexpr int QPR = NT / 4;             // column quads per block row
  constexpr int RSTEP = 256 / QPR;        // row groups
  __shared__ __align__(16) float Wt[2][CM][NT];
  __shared__ float Us[2][RB][CM];
  const int n0 = blockIdx.x * NT, m0 = blockIdx.y * RB;
  for (int e = threadIdx.x; e < 2 * CM * NT; e += 256) {
    const int s = e / (CM * NT), rem = e % (CM * NT), j = rem / NT, nn = rem % NT;
    float v = 0.f;
    if (s < a.nseg && j < a.c && n0 + nn < a.n) {
      const int64_t idx = (int64_t)(n0 + nn) * a.c + j;
      v = a.w_hi[s][idx] + a.w_lo[s][idx];
    }
    Wt[s][j][nn] = v;
  }
  for (int e = threadIdx.x; e < 2 * RB * CM; e += 256) {
    const int s = e / (RB * CM), rem = e % (RB * CM), r = rem / CM, j = rem % CM;
    float v = 0.f;
    if (s < a.nseg && m0 + r < a.rows && j < a.c) v = a.U[s][(int64_t)(m0 + r) * a.c + j];
    Us[s][r][j] = v;
  }
  __syncthreads();
  const int q = threadIdx.x % QPR, rg = threadIdx.x / QPR;
  const int nb = n0 + 4 * q;
  if (nb >= a.n) return;
  for (int r = rg; r < RB; r += RSTEP) {
    const int m = m0 + r;
    if (m >= a.rows) break;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (s >= a.nseg) break;
#pragma unroll
      for (int j = 0; j < CM; ++j) {
        const float u = Us[s][r][j];
        const float4 w4 = *reinterpret_cast<const float4*>(&Wt[s][j][4 * q]);
        v[0] = fmaf(u, w4.x, v[0]);
        v[1] = fmaf(u, w4.y, v[1]);
        v[2] = fmaf(u, w4.z, v[2]);
        v[3] = fmaf(u, w4.w, v[3]);
      }
    }
    if (!(nb + 4 <= a.n && epi_applyV<4>(a.epi, m, nb, v))) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (nb + t < a.n) epi_apply(a.epi, m, nb + t, v[t]);
    }
  }
}

void skinny_dx(cv_ctx* ctx, const SkinnyDxArgs& a) {
  if (a.c <= 16) {
    dim3 grid((a.n + 255) / 256, (a.rows + 31) / 32);
    k_dx<16, 256><<<grid, 256, 0, ctx->stream>>>(a);
  } else {
    dim3 grid((a.n + 127) / 128, (a.rows + 31) / 32);
    k_dx<32, 128><<<grid, 256, 0, ctx->stream>>>(a);
  }
  ctx->launches++;
}

// ---------------------------------------------------------------------------
// dw: block = 128 threads x 4 columns; grid.y splits the batch rows; U tile in
// smem; fp32 partials reduced in fixed order by a second kernel
// ---------------------------------------------------------------------------
template <int CM>
__global__ void __launch_bounds__(128) k_dw_partial(SkinnyDwArgs a) {
  if (skip_if(a.skip)) return;
  constexpr int KT = 64;
  __shared__ float Us[KT][CM];
  const int m = blockIdx.x * 512 + threadIdx.x * 4;
  const int chunk = (a.rows + a.ksplit - 1) / a.ksplit;
  const int kb = blockIdx.y * chunk, ke = min(a.rows, kb + chunk);
  float acc[4][CM];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int j = 0; j < CM; ++j) acc[t][j] = 0.f;
  const bool full = m + 3 < a.M;
  for (int s = 0; s < a.nseg; ++s) {
    const float* ah = a.a_hi[s];
    const float* al = a.a_lo[s];
    const int64_t lda = a.lda[s];
    for (int k0 = kb; k0 < ke; k0 += KT) {
      const int kn = min(KT, ke - k0);
      __syncthreads();
      for (int e = threadIdx.x; e < KT * CM; e += 128) {
        const int kk = e / CM, j = e % CM;
        Us[kk][j] = (kk < kn && j < a.c) ? a.U[s][(int64_t)(k0 + kk) * a.c + j] : 0.f;
      }
      __syncthreads();
      if (m >= a.M) continue;
#pragma unroll 4
      for (int kk = 0; kk < kn; ++kk) {
        const int64_t o = (int64_t)(k0 + kk) * lda + m;
        float x[4];
        if (full) {
          const float4 h = ld4(ah + o), l = ld4(al + o);
          x[0] = h.x + l.x; x[1] = h.y + l.y; x[2] = h.z + l.z; x[3] = h.w + l.w;
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t) x[t] = m + t < a.M ? ah[o + t] + al[o + t] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < CM; ++j) {
          const float u = Us[kk][j];
#pragma unroll
          for (int t = 0; t < 4; ++t) acc[t][j] = fmaf(x[t], u, acc[t][j]);
        }
      }
    }
  }
  if (m >= a.M) return;
  for (int t = 0; t < 4; ++t) {
    if (m + t >= a.M) break;
    float* dst = a.partial + ((int64_t)blockIdx.y * a.M + m + t) * a.c;
#pragma unroll
    for (int j = 0; j < CM; ++j)
      if (j < a.c) dst[j] = acc[t][j];
  }
}

__global__ void k_dw_final(SkinnyDwArgs a) {
  if (skip_if(a.skip)) return;
  const int64_t total = (int64_t)a.M * a.c;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int ks = 0; ks < a.ksplit; ++ks) s += a.partial[(int64_t)ks * total + i];
    a.out[i] = s;
  }
}

void skinny_dw(cv_ctx* ctx, SkinnyDwArgs a, float* ws, int64_t ws_elems) {
  const int mblocks = (a.M + 511) / 512;
  int ks = (4 * ctx->sm_count + mblocks - 1) / mblocks;
  const int max_by_rows = (a.rows + 63) / 64;
  if (ks > max_by_rows) ks = max_by_rows;
  while (ks > 1 && (int64_t)ks * a.M * a.c > ws_elems) --ks;
  if (ks < 1) ks = 1;
  a.ksplit = ks;
  a.partial = ws;
  dim3 grid(mblocks, ks);
  if (a.c <= 16) k_dw_partial<16><<<grid, 128, 0, ctx->stream>>>(a);
  else k_dw_partial<32><<<grid, 128, 0, ctx->stream>>>(a);
  const int64_t total = (int64_t)a.M * a.c;
  k_dw_final<<<(int)((total + 255) / 256), 256, 0, ctx->stream>>>(a);
  ctx->launches += 2;
}

}  // namespace cv
