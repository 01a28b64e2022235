// Output-layer kernels (c = output width <= 32).  All three are HBM-bound streams
// over one b x n activation/tangent matrix, so they are written for bandwidth:
// wide loads/stores, the tiny c-wide operand staged in shared memory or
// registers, several rows or columns per thread in flight, deterministic
// fixed-order reductions.  Activations arrive as scaled fp16 pairs (common.cuh).
//   skinny_rows : last-layer JVP + fused H_z (models.py:243-255, 199-204)
//   skinny_dw   : last-layer [gW; gb] = A^T U (models.py:280-281)
//   skinny_dx   : G = (U W^T) * act'(a) (models.py:282-284, 378-381)
#include <type_traits>

#include "common.cuh"
#include "epilogue.cuh"
#include "internal.h"
#include "skinny.cuh"

namespace cv {


// 4 consecutive split elements (8-byte aligned) -> fp32
CV_DEV void ld_join4(const __half* hi, const __half* lo, float inv, float (&x)[4]) {
  H4 a, b;
  a.u = *reinterpret_cast<const uint2*>(hi);
  b.u = *reinterpret_cast<const uint2*>(lo);
#pragma unroll
  for (int t = 0; t < 4; ++t) x[t] = (__half2float(a.h[t]) + __half2float(b.h[t])) * inv;
}

// ---------------------------------------------------------------------------
// rows: one warp per RPW rows, lanes stride K in 4-element steps, B^T chunk in smem
// ---------------------------------------------------------------------------
template <int CM, int RPW>
__global__ void __launch_bounds__(256) k_rows(SkinnyRowsArgs a) {
  CV_PDL_ENTRY();
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
    const float ainv = pow2f(-g.a_sc->e), binv = pow2f(-g.b_sc->e);
    for (int k0 = 0; k0 < g.K; k0 += RK) {
      const int kmax = min(RK, g.K - k0);
      __syncthreads();
      for (int e = threadIdx.x; e < RK * CM; e += 256) {
        const int kk = e % RK, j = e / RK;
        float v = 0.f;
        if (kk < kmax && j < a.c) {
          const int64_t idx = (int64_t)(k0 + kk) * g.ldb + j;
          v = join16(g.b_hi[idx], g.b_lo[idx], binv);
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
            const __half* ph = g.a_hi + (int64_t)m * g.lda + k0 + kk;
            const __half* pl = g.a_lo + (int64_t)m * g.lda + k0 + kk;
            if (kk + 3 < kmax && al8(ph) && al8(pl)) {
              ld_join4(ph, pl, ainv, av[r]);
            } else {
#pragma unroll
              for (int t = 0; t < 4; ++t) av[r][t] = kk + t < kmax ? join16(ph[t], pl[t], ainv) : 0.f;
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
  float amax = 0.f;
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
    float o;
    if (a.post == POST_LOGITS || a.loss == CV_LOSS_MSE) {
      o = a.post == POST_LOGITS ? t : t * a.scale;
    } else {
      // H_z T = p*T - p*(p.T)  (softmax-CE, per example)
      const float* p = a.probs + (int64_t)m * a.c;
      float pt = 0.f;
#pragma unroll
      for (int j = 0; j < CM; ++j)
        if (j < a.c) pt = fmaf(p[j], acc[r][j], pt);
      const float pj = lane < a.c ? p[lane] : 0.f;
      o = (pj * t - pj * pt) * a.scale;
    }
    if (lane < a.c) {
      a.out[(int64_t)m * a.c + lane] = o;
      amax = fmaxf(amax, fabsf(o));
    }
  }
  amax = warp_max_f(amax);
  if (lane == 0 && a.out_amax) atomic_amax(a.out_amax, amax);
}

template <int CM, int RPW>
static void launch_rows(cv_ctx* ctx, const SkinnyRowsArgs& a) {
  launch_k(ctx->stream, k_rows<CM, RPW>, (a.rows + 8 * RPW - 1) / (8 * RPW), 256, 0, a);
}

void skinny_rows(cv_ctx* ctx, const SkinnyRowsArgs& a) {
  // one row per warp unless that already gives >= 2 blocks per SM (small batches:
  // every row in flight at once)
  const bool many = (a.rows + 7) / 8 >= 2 * ctx->sm_count;
  if (a.c == 1) many ? launch_rows<1, 4>(ctx, a) : launch_rows<1, 1>(ctx, a);
  else if (a.c <= 4) many ? launch_rows<4, 4>(ctx, a) : launch_rows<4, 1>(ctx, a);
  else if (a.c <= 16) many ? launch_rows<16, 4>(ctx, a) : launch_rows<16, 1>(ctx, a);
  else many ? launch_rows<32, 2>(ctx, a) : launch_rows<32, 1>(ctx, a);
  ctx->launches++;
}

// ---------------------------------------------------------------------------
// dx: thread = 4 adjacent columns with their W^T entries held in registers; a
// warp covers 128 contiguous columns of a row (coalesced accesses); the block
// walks 32-row tiles (U rows staged in smem) and issues the R activation loads of
// a row group before any of its stores.
// ---------------------------------------------------------------------------
template <int C, int NSEG, bool TANH>
__global__ void __launch_bounds__(128) k_dx(SkinnyDxArgs a) {
  CV_PDL_ENTRY();
  if (skip_if(a.skip)) return;
  constexpr int RT = 32;   // rows per tile
  constexpr int R = 8;     // rows per thread in flight
  __shared__ __align__(16) float Us[NSEG][RT][C];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = blockIdx.x * 128 + lane * 4;
  const bool colok = nb < a.n;
  float w[NSEG][C][4];
#pragma unroll
  for (int s = 0; s < NSEG; ++s) {
    const float winv = pow2f(-a.w_sc[s]->e);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const bool ok = nb + t < a.n;
      const int64_t base = (int64_t)(nb + t) * a.c;
#pragma unroll
      for (int j = 0; j < C; ++j)
        w[s][j][t] = (ok && j < a.c) ? join16(a.w_hi[s][base + j], a.w_lo[s][base + j], winv) : 0.f;
    }
  }
  const Epilogue& e = a.epi;
  const EpiRt rt = epi_prepare(e);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) epi_publish(e, rt);
  const bool fast = (e.mode == EPI_SPLIT_MASK || (e.mode == EPI_HVP && !TANH)) && e.mask_div == 1 &&
                    al8(e.out_hi) && al8(e.out_lo) && al8(e.mask_hi) && (!TANH || al8(e.mask_lo)) &&
                    (e.ld & 3) == 0 && (e.mask_ld & 3) == 0 && (!e.raw || (al16(e.raw) && (e.raw_ld & 3) == 0));
  const bool full = nb + 4 <= a.n;
  const int tiles = (a.rows + RT - 1) / RT;
  float amax = 0.f, ramax = 0.f;
  for (int tile = blockIdx.y; tile < tiles; tile += gridDim.y) {
    const int m0 = tile * RT;
    __syncthreads();
    for (int i = threadIdx.x; i < NSEG * RT * C; i += 128) {
      const int s = i / (RT * C), rem = i % (RT * C), r = rem / C, j = rem % C;
      Us[s][r][j] = (m0 + r < a.rows && j < a.c) ? a.U[s][(int64_t)(m0 + r) * a.c + j] : 0.f;
    }
    __syncthreads();
    if (!colok) continue;
    uint2 mh[R], ml[TANH ? R : 1];
    if (fast) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int m = m0 + warp + 4 * i;
        if (m < a.rows && full) {
          const int64_t mo = (int64_t)m * e.mask_ld + nb;
          mh[i] = *reinterpret_cast<const uint2*>(e.mask_hi + mo);
          if constexpr (TANH) ml[i] = *reinterpret_cast<const uint2*>(e.mask_lo + mo);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = warp + 4 * i, m = m0 + r;
      if (m >= a.rows) break;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int s = 0; s < NSEG; ++s)
#pragma unroll
        for (int j = 0; j < C; ++j) {
          const float u = Us[s][r][j];
          v[0] = fmaf(u, w[s][j][0], v[0]);
          v[1] = fmaf(u, w[s][j][1], v[1]);
          v[2] = fmaf(u, w[s][j][2], v[2]);
          v[3] = fmaf(u, w[s][j][3], v[3]);
        }
      if (fast && full) {
        H4 hh;
        hh.u = mh[i];
        float av[4];
        if constexpr (TANH) {
          H4 ll;
          ll.u = ml[i];
#pragma unroll
          for (int t = 0; t < 4; ++t) av[t] = (__half2float(hh.h[t]) + __half2float(ll.h[t])) * rt.mask_inv;
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t) av[t] = __half2float(hh.h[t]);
        }
        if (e.raw) {
          *reinterpret_cast<float4*>(e.raw + (int64_t)m * e.raw_ld + nb) = make_float4(v[0], v[1], v[2], v[3]);
#pragma unroll
          for (int t = 0; t < 4; ++t) ramax = fmaxf(ramax, fabsf(v[t]));
        }
        H4 oh, ol;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float x = v[t] * act_deriv(TANH ? CV_ACT_TANH : CV_ACT_RELU, av[t]);
          amax = fmaxf(amax, fabsf(x));
          split16(x, rt.out_s, oh.h[t], ol.h[t]);
        }
        const int64_t o = (int64_t)m * e.ld + nb;
        *reinterpret_cast<uint2*>(e.out_hi + o) = oh.u;
        *reinterpret_cast<uint2*>(e.out_lo + o) = ol.u;
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (nb + t < a.n) epi_apply(e, rt, m, nb + t, v[t], amax, ramax);
      }
    }
  }
  epi_flush_amax(e, amax, ramax);
}

// dx, streaming variant for the hot case (one segment, ReLU mask, c <= 10, n <= 1024,
// 16-byte rows): a thread owns 4 adjacent columns with their W entries in
// registers, n/4 threads span a row, and each block streams a contiguous range of
// rows: the block's U rows are staged in shared memory once (one barrier), the
// 64-bit mask loads of DXW_R rows are in flight ahead of their use, the split
// output leaves as two 64-bit stores per row.
constexpr int DXW_R = 8;
constexpr int DXW_C = 10;
// two resident 256-thread blocks per SM (a three-block bound spills: measured slower)

// d = a * b + c on two fp32 lanes (sm_100 FFMA2)
CV_DEV float2 ffma2_dx(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
// RPP: rows per pass (256 / (n / 4)) when known at compile time (n = 1024: 1), else 0.
// Everything row-invariant (parameters, base pointers, the mask bit offset) is hoisted
// out of the row loop, U rows are staged at a fixed stride of DXW_C (zero-padded) so a
// row's coefficients are five 64-bit shared loads, and the split runs on half2 pairs
// (same rounding as split16).
template <int RPP, bool BITS>
__global__ void __launch_bounds__(256, 2) k_dx_wide(SkinnyDxArgs a, int rows_per_block) {
  const int tpr = a.n >> 2;                     // threads per row (<= 256)
  const int rpp = RPP > 0 ? RPP : 256 / tpr;    // rows per pass
  const int rl = threadIdx.x / tpr, col = (threadIdx.x - rl * tpr) * 4;
  float2 w01[DXW_C], w23[DXW_C];
  {
    const float winv = pow2f(-a.w_sc[0]->e);
    float w[4][DXW_C];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t base = (int64_t)(col + q) * a.c;
#pragma unroll
      for (int j = 0; j < DXW_C; ++j)
        w[q][j] = j < a.c ? join16(a.w_hi[0][base + j], a.w_lo[0][base + j], winv) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < DXW_C; ++j) {
      w01[j] = make_float2(w[0][j], w[1][j]);
      w23[j] = make_float2(w[2][j], w[3][j]);
    }
  }
  // the weights (and their scale) are the linearization's: loaded before the wait, so
  // they overlap the predecessor's tail
  CV_PDL_ENTRY();
  if (skip_if(a.skip)) return;
  const Epilogue& e = a.epi;
  const EpiRt rt = epi_prepare(e);
  if (blockIdx.x == 0 && threadIdx.x == 0) epi_publish(e, rt);
  float amax = 0.f;
  const int r_begin = blockIdx.x * rows_per_block;
  const int r_end = min(a.rows, r_begin + rows_per_block);
  constexpr bool bits = BITS;
  // the block's mask rows are one contiguous range: pull it toward L2 in bulk first
  if (threadIdx.x < 8 && r_end > r_begin && !bits) {
    const char* mb = reinterpret_cast<const char*>(e.mask_hi + (int64_t)r_begin * e.mask_ld);
    const int64_t bytes = ((int64_t)(r_end - r_begin) * e.mask_ld * 2) & ~(int64_t)15;
    const int64_t chunk = ((bytes / 8) + 15) & ~(int64_t)15;
    const int64_t o = chunk * threadIdx.x;
    const int64_t len = o >= bytes ? 0 : (bytes - o < chunk ? bytes - o : chunk);
    if (len > 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(mb + o), "r"((unsigned)len) : "memory");
  }
  // row-invariant addressing: 2-byte elements in both mask forms (packed-bit words, mask halves)
  const int64_t mrow = 2 * (bits ? e.mbits_ld : e.mask_ld);
  const char* mbase = bits ? reinterpret_cast<const char*>(e.mask_bits + (col >> 4))
                           : reinterpret_cast<const char*>(e.mask_hi + col);
  const int bsh = col & 15;
  const int64_t ld = e.ld;
  __half* const ohb = e.out_hi + col;
  __half* const olb = e.out_lo + col;
  const float out_s = rt.out_s;
  // mask loads of a batch of DXW_R rows (double buffered: batch b+1 is in flight while b is computed)
  using MaskT = typename std::conditional<BITS, uint32_t, uint2>::type;
  auto load_batch = [&](int r0, MaskT (&mk)[DXW_R]) {
    const char* p = mbase + (int64_t)r0 * mrow;
#pragma unroll
    for (int i = 0; i < DXW_R; ++i) {
      mk[i] = MaskT{};
      if (rl < rpp && r0 + i * rpp < r_end) {
        const char* q = p + (int64_t)i * rpp * mrow;
        if constexpr (BITS) mk[i] = __ldg(reinterpret_cast<const uint16_t*>(q));  // shifted at use
        else mk[i] = __ldg(reinterpret_cast<const uint2*>(q));
      }
    }
  };
  MaskT mcur[DXW_R], mnext[DXW_R];
  load_batch(r_begin + rl, mcur);
  // the block's U rows (contiguous) staged once at stride DXW_C: every later U read is a
  // 64-bit smem broadcast
  extern __shared__ __align__(16) float Us[];
  {
    const int nr = r_end - r_begin, c = a.c;
    const float* Ug = a.U[0] + (int64_t)r_begin * c;
    for (int i = threadIdx.x; i < nr * DXW_C; i += blockDim.x) {
      const int rr = i / DXW_C, j = i - rr * DXW_C;
      Us[i] = j < c ? Ug[rr * c + j] : 0.f;
    }
  }
  __syncthreads();
  if (rl >= rpp) return;
  const int64_t ostep = (int64_t)rpp * ld;
  for (int r0 = r_begin + rl; r0 < r_end; r0 += rpp * DXW_R) {
    if (r0 + rpp * DXW_R < r_end) load_batch(r0 + rpp * DXW_R, mnext);
    const float* ub = Us + (r0 - r_begin) * DXW_C;
    __half* oh = ohb + (int64_t)r0 * ld;
    __half* ol = olb + (int64_t)r0 * ld;
    const int cnt = (r_end - r0 + rpp - 1) / rpp;
    auto row = [&](int i) {
      const float2* u2 = reinterpret_cast<const float2*>(ub + i * rpp * DXW_C);
      // column pairs on FFMA2
      float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
      for (int jj = 0; jj < DXW_C / 2; ++jj) {
        const float2 uu = u2[jj];
        const float2 ux = make_float2(uu.x, uu.x), uy = make_float2(uu.y, uu.y);
        acc0 = ffma2_dx(ux, w01[2 * jj], acc0);
        acc1 = ffma2_dx(ux, w23[2 * jj], acc1);
        acc0 = ffma2_dx(uy, w01[2 * jj + 1], acc0);
        acc1 = ffma2_dx(uy, w23[2 * jj + 1], acc1);
      }
      float x[4];
      if constexpr (BITS) {
        const uint32_t wd = mcur[i] >> bsh;
        x[0] = (wd & 1u) ? acc0.x : 0.f;
        x[1] = (wd & 2u) ? acc0.y : 0.f;
        x[2] = (wd & 4u) ? acc1.x : 0.f;
        x[3] = (wd & 8u) ? acc1.y : 0.f;
      } else {
        H4 hm;
        hm.u = mcur[i];
        x[0] = __half2float(hm.h[0]) > 0.f ? acc0.x : 0.f;
        x[1] = __half2float(hm.h[1]) > 0.f ? acc0.y : 0.f;
        x[2] = __half2float(hm.h[2]) > 0.f ? acc1.x : 0.f;
        x[3] = __half2float(hm.h[3]) > 0.f ? acc1.y : 0.f;
      }
      amax = fmaxf(amax, fmaxf(fmaxf(fabsf(x[0]), fabsf(x[1])), fmaxf(fabsf(x[2]), fabsf(x[3]))));
      // split16 on pairs: hi = rn(x s), lo = rn(x s - hi)
      const float s0 = x[0] * out_s, s1 = x[1] * out_s, s2 = x[2] * out_s, s3 = x[3] * out_s;
      const __half2 h01 = __floats2half2_rn(s0, s1), h23 = __floats2half2_rn(s2, s3);
      const float2 b01 = __half22float2(h01), b23 = __half22float2(h23);
      const __half2 l01 = __floats2half2_rn(s0 - b01.x, s1 - b01.y), l23 = __floats2half2_rn(s2 - b23.x, s3 - b23.y);
      uint2 hv, lv;
      hv.x = *reinterpret_cast<const uint32_t*>(&h01);
      hv.y = *reinterpret_cast<const uint32_t*>(&h23);
      lv.x = *reinterpret_cast<const uint32_t*>(&l01);
      lv.y = *reinterpret_cast<const uint32_t*>(&l23);
      *reinterpret_cast<uint2*>(oh + i * ostep) = hv;
      *reinterpret_cast<uint2*>(ol + i * ostep) = lv;
    };
    if (cnt >= DXW_R) {  // full batch: rows unrolled without predicates (cross-row ILP)
#pragma unroll
      for (int i = 0; i < DXW_R; ++i) row(i);
    } else {
#pragma unroll
      for (int i = 0; i < DXW_R; ++i)
        if (i < cnt) row(i);
    }
#pragma unroll
    for (int i = 0; i < DXW_R; ++i) mcur[i] = mnext[i];
  }
  float ramax = 0.f;
  epi_flush_amax(e, amax, ramax);
}

static bool dx_wide_ok(const SkinnyDxArgs& a) {
  const Epilogue& e = a.epi;
  return a.nseg == 1 && a.c <= DXW_C && (a.n & 7) == 0 && a.n <= 1024 && a.n >= 64 &&
         e.mode == EPI_SPLIT_MASK && e.act == CV_ACT_RELU && !e.raw && e.mask_div == 1 && (e.ld & 7) == 0 &&
         (e.mask_ld & 7) == 0 && !(((uintptr_t)e.out_hi | (uintptr_t)e.out_lo | (uintptr_t)e.mask_hi) & 15);
}

template <int C, int NSEG>
static void launch_dx(cv_ctx* ctx, const SkinnyDxArgs& a) {
  const int gx = (a.n + 127) / 128;
  const int tiles = (a.rows + 31) / 32;
  int gy = (ctx->sm_count * 4 + gx - 1) / gx;  // ~4 resident 128-thread blocks per SM
  if (gy > tiles) gy = tiles;
  if (a.epi.act == CV_ACT_TANH) launch_k(ctx->stream, k_dx<C, NSEG, true>, dim3(gx, gy), 128, 0, a);
  else launch_k(ctx->stream, k_dx<C, NSEG, false>, dim3(gx, gy), 128, 0, a);
}

void skinny_dx(cv_ctx* ctx, const SkinnyDxArgs& a) {
  if (dx_wide_ok(a)) {
    const SkinnyDxArgs& b = a;
    // contiguous row ranges, 2 resident 256-thread blocks per SM
    const int blocks = 2 * ctx->sm_count;
    const int rpb = (a.rows + blocks - 1) / blocks;
    const size_t smem = sizeof(float) * (size_t)rpb * DXW_C;
    const int grid = (a.rows + rpb - 1) / rpb;
    const bool bt = b.epi.mask_bits != nullptr;
    if (a.n == 1024) bt ? launch_k(ctx->stream, k_dx_wide<1, true>, grid, 256, smem, b, rpb)
                        : launch_k(ctx->stream, k_dx_wide<1, false>, grid, 256, smem, b, rpb);
    else bt ? launch_k(ctx->stream, k_dx_wide<0, true>, grid, 256, smem, b, rpb)
            : launch_k(ctx->stream, k_dx_wide<0, false>, grid, 256, smem, b, rpb);
    ctx->launches++;
    return;
  }
  const bool two = a.nseg > 1;
  if (a.c == 1) two ? launch_dx<1, 2>(ctx, a) : launch_dx<1, 1>(ctx, a);  // scalar regression output
  else if (a.c <= 4) two ? launch_dx<4, 2>(ctx, a) : launch_dx<4, 1>(ctx, a);
  else if (a.c == 10) two ? launch_dx<10, 2>(ctx, a) : launch_dx<10, 1>(ctx, a);
  else if (a.c <= 16) two ? launch_dx<16, 2>(ctx, a) : launch_dx<16, 1>(ctx, a);
  else two ? launch_dx<32, 2>(ctx, a) : launch_dx<32, 1>(ctx, a);
  ctx->launches++;
}

// ---------------------------------------------------------------------------
// dw: block = 128 threads x 4 columns; grid.y splits the batch rows; U tile in
// smem; fp32 partials reduced in fixed order by a second kernel
// ---------------------------------------------------------------------------
template <int CM>
__global__ void __launch_bounds__(128) k_dw_partial(SkinnyDwArgs a) {
  CV_PDL_ENTRY();
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
    const __half* ah = a.a_hi[s];
    const __half* al = a.a_lo[s];
    const int64_t lda = a.lda[s];
    const float inv = pow2f(-a.a_sc[s]->e);
    const bool vec = full && (lda & 3) == 0 && al8(ah) && al8(al);
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
        if (vec) {
          ld_join4(ah + o, al + o, inv, x);
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t) x[t] = m + t < a.M ? join16(ah[o + t], al[o + t], inv) : 0.f;
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
  CV_PDL_ENTRY();
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
  const int max_by_rows = (a.rows + 15) / 16;  // >= 16 rows per block: small batches still fill the SMs
  if (ks > max_by_rows) ks = max_by_rows;
  while (ks > 1 && (int64_t)ks * a.M * a.c > ws_elems) --ks;
  if (ks < 1) ks = 1;
  a.ksplit = ks;
  a.partial = ws;
  dim3 grid(mblocks, ks);
  if (a.c == 1) launch_k(ctx->stream, k_dw_partial<1>, grid, 128, 0, a);
  else if (a.c <= 4) launch_k(ctx->stream, k_dw_partial<4>, grid, 128, 0, a);
  else if (a.c <= 16) launch_k(ctx->stream, k_dw_partial<16>, grid, 128, 0, a);
  else launch_k(ctx->stream, k_dw_partial<32>, grid, 128, 0, a);
  const int64_t total = (int64_t)a.M * a.c;
  launch_k(ctx->stream, k_dw_final, (int)((total + 255) / 256), 256, 0, a);
  ctx->launches += 2;
}

}  // namespace cv
