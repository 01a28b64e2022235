// tcgen05 / TMA split-precision (3xFP16, scaled) GEMM engine for sm_100a.
//
//   D[M x N] = sum_seg A_seg[M x K] . B_seg[K x N]        (fp32 accumulate in TMEM)
//   with X = (X_hi + X_lo) 2^-e_X (scaled fp16 pairs, common.cuh):
//   D = 2^-(eA+eB) (A_hi.B_hi + A_hi.B_lo + A_lo.B_hi)    (3 tcgen05.mma kind::f16)
//
// Operands are the split buffers of internal.h (row-major, leading dim ld), each
// either K-major (K contiguous) or MN-major (M/N contiguous); both are native
// tcgen05 operand majors for 16-bit types, so no transposed copies exist anywhere.
//
// Two K segments (A1.B1 + A2.B2, e.g. the JVP's [A | da][V; W]) carry different
// product exponents S = eA + eB.  They share one TMEM accumulator: the segment
// with the larger S runs first and the first MMA of the second segment rescales
// the partial sum by 2^-(S1-S2) through tcgen05.mma's scale-input-d operand
// (plus zero-operand MMAs for shifts beyond 15), so the accumulator always holds
// 2^S_last * D exactly as if both products had been formed at the smaller scale.
//
// One CTA = one 128 x BN output tile (BN = 32, 128 or 256), 10 warps:
//   warp 0 lane 0 : TMA producer      (cp.async.bulk.tensor.2d, SWIZZLE_128B)
//   warp 1 lane 0 : MMA issuer        (tcgen05.mma.cta_group::1.kind::f16)
//   warps 2-9     : epilogue          (tcgen05.ld 32x32b -> registers -> 128-bit fused epilogue)
// smem ring of STAGES x {A_hi, A_lo, B_hi, B_lo} 64-deep K slabs, full/empty
// mbarriers between TMA and MMA, tcgen05.commit frees a slab / signals the epilogue.
// Split-K writes fp32 partials (already unscaled) that a fixed-order reduction folds in.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <unordered_map>

#include "common.cuh"
#include "epilogue.cuh"
#include "internal.h"

namespace cv {

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;                   // fp16 elements = 128 bytes = one SWIZZLE_128B row
constexpr int TC_ZERO_BYTES = TC_BM * 32;   // all-zero K-major A tile (SWIZZLE_32B, K=16) for rescaling MMAs
constexpr int TC_STG_BYTES = 2048;          // per epilogue warp: 32 rows x 16 cols, two fp16 planes or one fp32
constexpr int TC_HSTG_BYTES = 1280;        // per epilogue warp: the fused head's W / V rows of one sub-tile (16 x 10 x 2 fp32)
constexpr int TC_STG_TOTAL = 8 * (TC_STG_BYTES + TC_HSTG_BYTES);

struct TcOperand {
  int kmajor;   // 1: K contiguous, 0: M/N contiguous
};

struct TcArgs {
  int M, N;
  int nseg;
  const Scale* asc[2];
  const Scale* bsc[2];
  int kb[2];          // k-blocks per segment
  int kb_total;
  int kb_per_split;
  TcOperand a[2], b[2];
  Epilogue epi;
  const int* skip;
  int lower_only;
  int cyc_nb, cyc_skip;
  int tma_out;        // 0: per-thread stores; 1: fp16 split pair via TMA; 2: fp32 (out or partial) via TMA;
                      // 3: fp32 reduce-add via TMA (accumulating Gram / trailing updates)
  float* partial;     // split-K partials (nullptr: apply the epilogue directly)
  int tiles_m, tiles_n, splits;
};

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
CV_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

CV_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

CV_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

CV_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

CV_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

CV_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

CV_DEV void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// UMMA shared-memory descriptor, version 1 (sm_100), layout 2 = SWIZZLE_128B.
CV_DEV uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)layout << 61;
  return d;
}

// Operand slab descriptors for k-step kk (16 K-elements) of a 64-deep slab:
//   K-major : rows of 128 B (64 fp16), 8-row atoms (SBO 1024), k-step = +32 B in the row.
//   MN-major: 64-wide MN chunks of 64 K-rows x 128 B each (LBO 8192 between chunks),
//             8-row K groups (SBO 1024), k-step = 16 K-rows = +2048 B.
CV_DEV uint64_t op_desc(uint32_t base, int mn, int kk) {
  return mn ? umma_desc(base + kk * 2048, 8192, 1024, 2) : umma_desc(base + kk * 32, 16, 1024, 2);
}

// Instruction descriptor: kind::f16, D f32, A/B f16, majors, N, M.
__host__ __device__ constexpr uint32_t f16_idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// D = A.B + (accum ? D : 0)
template <int CG>
CV_DEV void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  if constexpr (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accum));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

// D = A.B + D * 2^-SH   (scale-input-d, immediate 1..15)
template <int CG, int SH>
CV_DEV void umma_f16_sh(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc) {
  if constexpr (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p, %4;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "n"(SH));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p, %4;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "n"(SH));
}

template <int CG>
CV_DEV void umma_f16_shift(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, int sh) {
  switch (sh) {
#define CV_SH(k) \
  case k:        \
    umma_f16_sh<CG, k>(tmem_d, a, b, idesc); \
    break;
    CV_SH(1) CV_SH(2) CV_SH(3) CV_SH(4) CV_SH(5) CV_SH(6) CV_SH(7) CV_SH(8)
    CV_SH(9) CV_SH(10) CV_SH(11) CV_SH(12) CV_SH(13) CV_SH(14) CV_SH(15)
#undef CV_SH
    default:
      umma_f16<CG>(tmem_d, a, b, idesc, 1u);
      break;
  }
}

// The 3 products of one 16-deep k-step; shift > 0 first rescales the running sum.
template <int CG>
CV_DEV void umma_kstep(uint32_t dtm, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl, uint64_t zero_a,
                       uint32_t idesc, bool accum, int shift) {
  if (accum && shift > 0) {
    while (shift > 15) {  // D <- 0.B + D 2^-15
      umma_f16_shift<CG>(dtm, zero_a, bh, idesc, 15);
      shift -= 15;
    }
    umma_f16_shift<CG>(dtm, ah, bh, idesc, shift);
  } else {
    umma_f16<CG>(dtm, ah, bh, idesc, accum ? 1u : 0u);
  }
  umma_f16<CG>(dtm, ah, bl, idesc, 1u);
  umma_f16<CG>(dtm, al, bh, idesc, 1u);
}

template <int CG>
CV_DEV void umma_commit(uint64_t* bar) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
  } else {
    const uint16_t mask = 3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
  }
}

CV_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

CV_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

CV_DEV void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
CV_DEV void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
// element-wise fp32 add of a staged sub-tile into global memory (the L2 does the
// read-modify-write, one add per element: the accumulating Gram / trailing updates)
CV_DEV void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
CV_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
CV_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
CV_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// product exponents and processing order of the K segments (larger S first)
struct SegPlan {
  int S[2];
  float inv_a[2], inv_b[2];
  int ord;
};

CV_DEV SegPlan seg_plan(const TcArgs& a) {
  SegPlan p;
  for (int s = 0; s < 2; ++s) {
    const int ea = s < a.nseg ? a.asc[s]->e : 0, eb = s < a.nseg ? a.bsc[s]->e : 0;
    p.S[s] = ea + eb;
    p.inv_a[s] = pow2f(-ea);
    p.inv_b[s] = pow2f(-eb);
  }
  p.ord = (a.nseg > 1 && p.S[1] > p.S[0]) ? 1 : 0;
  return p;
}

// virtual k-block v (processing order) -> segment, and the k-block within it
CV_DEV int vseg(const TcArgs& a, const SegPlan& p, int v, int& lkb) {
  const int n0 = a.kb[p.ord];
  if (v < n0) {
    lkb = v;
    return p.ord;
  }
  lkb = v - n0;
  return 1 - p.ord;
}

// descriptor of the zero tile: K-major SWIZZLE_32B, 32-byte rows (K = 16), 8-row atoms of 256 B
CV_DEV uint64_t zero_desc(const uint8_t* z) { return umma_desc(smem_u32(z), 16, 256, 6); }

// zero the rescaling tile (all threads), visible to the tensor core's async proxy
CV_DEV void zero_tile_init(uint8_t* z) {
  for (int i = threadIdx.x; i < TC_ZERO_BYTES / 16; i += blockDim.x) reinterpret_cast<uint4*>(z)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

struct TcMaps {
  CUtensorMap m[2][4];  // [seg][A_hi, A_lo, B_hi, B_lo]
  CUtensorMap o[2];     // TMA-store epilogue: fp16 {hi, lo} boxes {16, 32} SW32, or fp32 {16, 32(,1)} SW64
};

CV_DEV float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
CV_DEV void sts4(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// Fused output-layer head, c = 10: the W and V rows of a 16-column sub-tile (2 x 160
// contiguous fp32, 16-byte aligned) are fetched cooperatively by the warp (lane l
// holds float4 l, l+32, l+64 of the 80), one sub-tile ahead, and staged in the warp's
// smem slot, from which every lane reads them as broadcasts.
CV_DEV void head_fetch10(const Epilogue& e, int nb, int N, int lane, float4 (&hf)[3]) {
  const int64_t lim = (int64_t)N * 10;  // valid floats of the W / V row blocks
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int idx = lane + 32 * u;
    hf[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (idx < 80 && nb < N) {
      const float* base = idx < 40 ? e.head_w : e.head_v;
      const int64_t o = (int64_t)nb * 10 + 4 * (idx % 40);
      if (o + 4 <= lim) {
        hf[u] = __ldg(reinterpret_cast<const float4*>(base + o));
      } else {
        float t[4] = {0.f, 0.f, 0.f, 0.f};
        for (int i = 0; i < 4; ++i)
          if (o + i < lim) t[i] = __ldg(base + o + i);
        hf[u] = make_float4(t[0], t[1], t[2], t[3]);
      }
    }
  }
}

CV_DEV void head_stage10(uint32_t hs, int lane, const float4 (&hf)[3]) {
#pragma unroll
  for (int u = 0; u < 3; ++u)
    if (lane + 32 * u < 80) sts4(hs + 16 * (lane + 32 * u), hf[u]);
}

// d = a * b + c on two fp32 lanes at once (sm_100 FFMA2)
CV_DEV float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

// hacc[k] += sum_j a[j] V[j, k] + t[j] W[j, k] over the staged sub-tile (k pairs on FFMA2)
CV_DEV void head_acc10(uint32_t hs, const float (&av)[16], const float (&t)[16], float (&hacc)[16]) {
  float2 h[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) h[k] = make_float2(hacc[2 * k], hacc[2 * k + 1]);
#pragma unroll
  for (int j0 = 0; j0 < 16; j0 += 2) {
    float2 w[10], v[10];
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      const float4 a = lds4(hs + 4 * (j0 * 10) + 16 * u);
      const float4 b = lds4(hs + 640 + 4 * (j0 * 10) + 16 * u);
      w[2 * u] = make_float2(a.x, a.y);
      w[2 * u + 1] = make_float2(a.z, a.w);
      v[2 * u] = make_float2(b.x, b.y);
      v[2 * u + 1] = make_float2(b.z, b.w);
    }
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      const float2 tt = make_float2(t[j0 + jj], t[j0 + jj]);
      const float2 aa = make_float2(av[j0 + jj], av[j0 + jj]);
#pragma unroll
      for (int k = 0; k < 5; ++k) h[k] = ffma2(aa, v[jj * 5 + k], ffma2(tt, w[jj * 5 + k], h[k]));
    }
  }
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    hacc[2 * k] = h[k].x;
    hacc[2 * k + 1] = h[k].y;
  }
}

// any other head width (<= 16): direct broadcast loads from global
CV_DEV void head_acc_generic(const Epilogue& e, int nb, int N, const float (&av)[16], const float (&t)[16],
                             float (&hacc)[16]) {
  const int hc = e.head_c;
  const float* wr = e.head_w + (int64_t)nb * hc;
  const float* vr = e.head_v + (int64_t)nb * hc;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (nb + j >= N) break;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < hc) hacc[k] = fmaf(av[j], __ldg(vr + j * hc + k), fmaf(t[j], __ldg(wr + j * hc + k), hacc[k]));
  }
}

// Epilogue of one accumulator tile through shared memory and TMA stores (the
// hot modes: split outputs with an optional ReLU mask, fp32 outputs and split-K
// partials).  Each warp owns a 2 KB staging slot and walks its 32 rows in
// 16-column steps: tcgen05.ld -> (mask tile loaded row-contiguously through the
// slot) -> epilogue -> swizzled staging -> one elected lane issues the TMA
// store(s).  Global traffic is full-row, and stores retire asynchronously.
// BITS: the ReLU mask comes as packed bits (Epilogue::mask_bits), compiled as its own
// copy so the fp16-mask prefetch registers and the bit words are never live together.
template <int BN, bool BITS>
CV_DEV void tile_epilogue_tma(const TcArgs& a, const TcMaps& maps, const EpiRt& rt, uint32_t tacc, int m_base, int n0,
                              int split, float inv, int q, int half, int lane, uint8_t* stg, uint8_t* hstg,
                              float& amax) {
  const int r0 = m_base + q * 32;  // this warp's first row
  const int m = r0 + lane;
  const uint32_t trow = tacc + ((uint32_t)(q * 32) << 16);
  constexpr int NSUB = BN / 16;
  constexpr int S0 = NSUB >= 2 ? NSUB / 2 : 1;
  const int sb = half * S0, se = NSUB >= 2 ? (half + 1) * S0 : (half == 0 ? 1 : 0);
  const Epilogue& e = a.epi;
  const bool use_mask = a.tma_out == 1 && (e.mode == EPI_SPLIT_MASK || e.mode == EPI_HVP);
  const bool relu_act = e.act == CV_ACT_RELU;
  const bool head = use_mask && e.head_part != nullptr;
  // forward variant (EPI_SPLIT_ACT): logits partials sum_n act(z)(m, n) W[n, :]
  const bool head_fwd = !use_mask && a.tma_out == 1 && e.mode == EPI_SPLIT_ACT && e.head_part != nullptr;
  const bool head10 = (head || head_fwd) && e.head_c == 10 && !(((uintptr_t)e.head_w | (uintptr_t)e.head_v) & 15);
  const bool store = !(head && e.head_only);
  // packed ReLU bits: the lane's words for all sub-tiles of its half in one go
  const bool use_bits = BITS;
  // up to 8 16-bit words (one per sub-tile) as a 128-bit shift register in 4 registers
  uint64_t wq0 = 0, wq1 = 0;
  if (use_bits) {
#pragma unroll
    for (int i = 0; i < (NSUB >= 2 ? NSUB / 2 : 1) && i < 8; ++i) {
      const int nb = n0 + (sb + i) * 16;
      const uint64_t wd =
          (m < a.M && nb < a.N && sb + i < se) ? (uint64_t)e.mask_bits[(int64_t)m * e.mbits_ld + nb / 16] : 0ull;
      if (i < 4) wq0 |= wd << (16 * i);
      else wq1 |= wd << (16 * (i - 4));
    }
  }
  const bool use_hi = use_mask && !use_bits;
  const uint32_t hs = smem_u32(hstg);
  float4 hf[3];
  if (head10) head_fetch10(e, n0 + sb * 16, a.N, lane, hf);
  // this lane's row of a sub-tile's mask (16 columns = one 32-byte sector), loaded one
  // sub-tile ahead so the global latency overlaps the previous sub-tile; the head also
  // needs the low plane (the activation value, not just its sign)
  auto load_mask = [&](int nb, uint4 (&mv)[2], uint4 (&ml)[2]) {
#pragma unroll
    for (int ch = 0; ch < 2; ++ch) {
      mv[ch] = make_uint4(0, 0, 0, 0);
      ml[ch] = make_uint4(0, 0, 0, 0);
      if (m < a.M && nb + 8 * ch < a.N) {
        const int64_t o = (int64_t)m * e.mask_ld + nb + 8 * ch;
        mv[ch] = *reinterpret_cast<const uint4*>(e.mask_hi + o);
        if (head) ml[ch] = *reinterpret_cast<const uint4*>(e.mask_lo + o);
      }
    }
  };
  uint4 mcur[2], mnext[2], lcur[2], lnext[2];
  float hacc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) hacc[k] = 0.f;
  if (use_hi) load_mask(n0 + sb * 16, mcur, lcur);
#pragma unroll 1
  for (int sbk = sb; sbk < se; ++sbk) {
    const int nb = n0 + sbk * 16;
    if (nb >= a.N) break;
    if (use_hi && sbk + 1 < se) load_mask(nb + 16, mnext, lnext);
    uint32_t r[16];
    tmem_ld16(trow + sbk * 16, r);
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]) * inv;
    if (a.tma_out == 1) {
      // ---- split fp16 output (activations / tangents / cotangents) ----
      float o[16];
      if (use_bits) {
        const uint32_t wd = (uint32_t)(wq0 & 0xFFFFu);
        wq0 = (wq0 >> 16) | (wq1 << 48);
        wq1 >>= 16;
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] = ((wd >> j) & 1u) ? v[j] : 0.f;
      } else if (use_mask) {
        H8 mk[2], ml[2];
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          mk[ch].u = mcur[ch];
          ml[ch].u = lcur[ch];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] = v[j] * (__half2float(mk[j >> 3].h[j & 7]) > 0.f ? 1.f : 0.f);
        if (head) {
          float av[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            av[j] = (__half2float(mk[j >> 3].h[j & 7]) + __half2float(ml[j >> 3].h[j & 7])) * rt.mask_inv;
          if (head10) {
            head_stage10(hs, lane, hf);
            __syncwarp();
            if (sbk + 1 < se) head_fetch10(e, nb + 16, a.N, lane, hf);
            head_acc10(hs, av, o, hacc);
            __syncwarp();  // the slot is rewritten by the next sub-tile
          } else {
            head_acc_generic(e, nb, a.N, av, o, hacc);
          }
        }
        mcur[0] = mnext[0];
        mcur[1] = mnext[1];
        lcur[0] = lnext[0];
        lcur[1] = lnext[1];

      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] = relu_act ? relu_f(v[j]) : tanhf(v[j]);
        if (head_fwd) {
          float zero[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) zero[j] = 0.f;
          if (head10) {
            head_stage10(hs, lane, hf);
            __syncwarp();
            if (sbk + 1 < se) head_fetch10(e, nb + 16, a.N, lane, hf);
            head_acc10(hs, zero, o, hacc);
            __syncwarp();
          } else {
            head_acc_generic(e, nb, a.N, zero, o, hacc);
          }
        }
      }
      if (!store) continue;
      if (m < a.M)
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (nb + j < a.N) amax = fmaxf(amax, fabsf(o[j]));
      H8 h0, h1, l0, l1;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        split16(o[j], rt.out_s, h0.h[j], l0.h[j]);
        split16(o[8 + j], rt.out_s, h1.h[j], l1.h[j]);
      }
      if (e.out_unit && nb + 16 >= a.N && m < a.M) {
        // the ones column of the augmented activation [a | 1] (column N, past the TMA box)
        __half oh, ol;
        split16(1.f, rt.out_s, oh, ol);
        e.out_hi[(int64_t)m * e.ld + a.N] = oh;
        e.out_lo[(int64_t)m * e.ld + a.N] = ol;
        amax = fmaxf(amax, 1.f);
      }
      if (e.bits_out && m < a.M) {
        // packed ReLU sign bits of the stored hi plane (what the hi-mask consumers test)
        uint32_t wd = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          wd |= (__half2float(h0.h[j]) > 0.f ? 1u : 0u) << j;
          wd |= (__half2float(h1.h[j]) > 0.f ? 1u : 0u) << (8 + j);
        }
        e.bits_out[(int64_t)m * e.bits_out_ld + nb / 16] = (uint16_t)wd;
      }
      // the slot must be free: the previous sub-tile's TMA store has read it (waited
      // only now, so that read overlaps this sub-tile's TMEM load and math)
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
      const int sw = (lane >> 2) & 1;
      *reinterpret_cast<uint4*>(stg + lane * 32 + 16 * (0 ^ sw)) = h0.u;
      *reinterpret_cast<uint4*>(stg + lane * 32 + 16 * (1 ^ sw)) = h1.u;
      *reinterpret_cast<uint4*>(stg + 1024 + lane * 32 + 16 * (0 ^ sw)) = l0.u;
      *reinterpret_cast<uint4*>(stg + 1024 + lane * 32 + 16 * (1 ^ sw)) = l1.u;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(&maps.o[0], stg, nb, r0);
        tma_store_2d(&maps.o[1], stg + 1024, nb, r0);
        bulk_commit();
      }
    } else {
      // ---- fp32 output / split-K partial / Gram / accumulation: 32 rows x 64 B, SWIZZLE_64B ----
      if (e.mode == EPI_GRAM && m < a.M) {  // Hadamard factor of the (row, column) examples
        const float* sa = e.sa + (int64_t)((m + e.row0) / e.kdiv) * e.sa_ld;
        int qe = nb / e.kdiv, re = nb - qe * e.kdiv;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          v[j] *= sa[qe];
          if (++re == e.kdiv) {
            re = 0;
            ++qe;
          }
        }
      } else if (e.mode == EPI_ACCUM) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] *= e.alpha;
      }
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
      const int sw = (lane >> 1) & 3;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch)
        *reinterpret_cast<float4*>(stg + lane * 64 + 16 * (ch ^ sw)) =
            make_float4(v[4 * ch], v[4 * ch + 1], v[4 * ch + 2], v[4 * ch + 3]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (a.partial) tma_store_3d(&maps.o[0], stg, nb, r0, split);
        else if (a.tma_out == 3) tma_reduce_add_2d(&maps.o[0], stg, nb, r0);
        else tma_store_2d(&maps.o[0], stg, nb, r0);
        bulk_commit();
      }
    }
  }
  if ((head || head_fwd) && m < a.M) {
    // group = column half of this tile; fixed-order reduction in k_out_reduce
    const int grp = (n0 / BN) * 2 + half;
    float* dst = e.head_part + ((int64_t)grp * a.M + m) * e.head_c;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < e.head_c) dst[k] = hacc[k];
  }
}

// Bulk L2 prefetch of the mask rows (and, for the fused head, the low plane) an
// epilogue warp will read for its next tile: issued before the warp waits for the
// accumulator, so the tile's mainloop hides the DRAM latency of the mask stream.
template <int BN>
CV_DEV void epi_prefetch_mask(const TcArgs& a, int m_base, int n0, int q, int half, int lane) {
  const Epilogue& e = a.epi;
  if (!(a.tma_out == 1 && (e.mode == EPI_SPLIT_MASK || e.mode == EPI_HVP))) return;
  if (e.mask_bits && e.act == CV_ACT_RELU && !e.head_part && e.mask_div == 1) return;  // packed bits: no row stream
  const int m = m_base + q * 32 + lane;
  const int c0 = n0 + half * (BN / 2);
  int cols = a.N - c0 < BN / 2 ? a.N - c0 : BN / 2;
  cols &= ~7;
  if (m >= a.M || cols <= 0) return;
  const int64_t o = (int64_t)m * e.mask_ld + c0;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(e.mask_hi + o), "r"(cols * 2) : "memory");
  if (e.head_part)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(e.mask_lo + o), "r"(cols * 2) : "memory");
}

// The epilogue of one accumulator tile (TMEM -> registers -> fused epilogue), run by
// 8 warps: warp w reads TMEM lane quadrant (w % 4), half = column half.
template <int BN>
CV_DEV void tile_epilogue(const TcArgs& a, const TcMaps& maps, const EpiRt& rt, uint32_t tacc, int m_base, int n0,
                          int split, float inv, int q, int half, int lane, uint8_t* stg, uint8_t* hstg) {
  if (a.tma_out) {
    float amax = 0.f, ramax = 0.f;
    const Epilogue& e = a.epi;
    const bool bits = a.tma_out == 1 && (e.mode == EPI_SPLIT_MASK || e.mode == EPI_HVP) && e.act == CV_ACT_RELU &&
                      !e.head_part && e.mask_bits != nullptr && e.mask_div == 1;
    if (bits) tile_epilogue_tma<BN, true>(a, maps, rt, tacc, m_base, n0, split, inv, q, half, lane, stg, hstg, amax);
    else tile_epilogue_tma<BN, false>(a, maps, rt, tacc, m_base, n0, split, inv, q, half, lane, stg, hstg, amax);
    if (!a.partial) epi_flush_amax(a.epi, amax, ramax);
    return;
  }
  const int m = m_base + q * 32 + lane;
  const uint32_t trow = tacc + ((uint32_t)(q * 32) << 16);
  constexpr int NCH = BN / 32;
  constexpr int C0 = NCH >= 2 ? NCH / 2 : 1;
  float amax = 0.f, ramax = 0.f;
#pragma unroll 1
  for (int c = half * C0; c < (NCH >= 2 ? (half + 1) * C0 : (half == 0 ? 1 : 0)); ++c) {
    uint32_t r[32];
    tmem_ld32(trow + c * 32, r);
    if (m >= a.M) continue;
    const int nb = n0 + c * 32;
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * inv;
    const bool full_chunk = nb + 32 <= a.N && (!a.lower_only || nb + 31 <= lo_row(a, m) + a.lower_only - 1);
    if (a.partial) {
      float* dst = a.partial + ((int64_t)split * a.M + m) * a.N + nb;
      if (full_chunk && al16(dst)) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (nb + j < a.N) dst[j] = v[j];
      }
    } else if (!(full_chunk && epi_applyV<32>(a.epi, rt, m, nb, v, amax, ramax))) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int n = nb + j;
        if (n < a.N && (!a.lower_only || n <= lo_row(a, m) + a.lower_only - 1))
          epi_apply(a.epi, rt, m, n, v[j], amax, ramax);
      }
    }
  }
  if (!a.partial) epi_flush_amax(a.epi, amax, ramax);
}

// ---------------------------------------------------------------------------
// Kernel (1-CTA)
// ---------------------------------------------------------------------------

template <int BN, int STAGES>
struct TcCfg {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;  // 16 KB
  static constexpr int B_BYTES = BN * TC_BK * 2;     // 4 / 16 / 32 KB
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + TC_ZERO_BYTES + TC_STG_TOTAL + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;  // double-buffered accumulator
  static constexpr int THREADS = 320;                          // w0 TMA, w1 MMA, w2..w9 epilogue
};

constexpr int TC_GROUP = 8;

// work item -> (m0, n0, first k-block, k-blocks); split index slowest so that
// co-resident CTAs share K ranges (and therefore L2-resident operand panels)
CV_DEV bool tc_work(const TcArgs& a, int w, int bm, int bn, int& m0, int& n0, int& kb0, int& nkb) {
  const int tiles = a.tiles_m * a.tiles_n;
  const int split = w / tiles, t = w % tiles;
  if (a.tiles_m >= 2 * TC_GROUP && a.tiles_n >= 2 * TC_GROUP) {
    // large grids (Gram, Cholesky trailing updates, C5 layers): bands of TC_GROUP tile
    // rows walked column by column, so the co-resident tiles of a wave share a few A
    // and B slabs in L2 instead of streaming every B slab once per tile row
    const int band = t / (TC_GROUP * a.tiles_n);
    const int r0 = band * TC_GROUP;
    const int rows = a.tiles_m - r0 < TC_GROUP ? a.tiles_m - r0 : TC_GROUP;
    const int r = t - band * TC_GROUP * a.tiles_n;
    m0 = (r0 + r % rows) * bm;
    n0 = (r / rows) * bn;
  } else {
    m0 = (t / a.tiles_n) * bm;
    n0 = (t % a.tiles_n) * bn;
  }
  kb0 = split * a.kb_per_split;
  nkb = min(a.kb_total, kb0 + a.kb_per_split) - kb0;
  return !(a.lower_only && n0 > lo_row(a, m0 + bm - 1) + a.lower_only - 1);
}

// TMA of one operand slab: K-major = one box {64 K, rows}; MN-major = rows/64 boxes
// {64 MN, 64 K} of 8 KB each.
CV_DEV void load_slab(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, bool kmajor, int k0, int r0, int rows) {
  if (kmajor) {
    tma_load_2d(dst, map, bar, k0, r0);
  } else {
    for (int j = 0; j < rows / 64; ++j) tma_load_2d(dst + j * 8192, map, bar, r0 + 64 * j, k0);
  }
}

// Persistent: grid = min(work, SMs); each CTA loops over work items.  The TMEM
// accumulator is double buffered so the epilogue of item i overlaps the
// mainloop of item i+1.
template <int BN, int STAGES>
__global__ void __launch_bounds__(320, 1) k_gemm_tc(const __grid_constant__ TcMaps maps, const TcArgs a) {
  using Cfg = TcCfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* zero = smem + STAGES * Cfg::STAGE_BYTES;
  uint8_t* stg_all = zero + TC_ZERO_BYTES;
  uint64_t* full = (uint64_t*)(stg_all + TC_STG_TOTAL);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = a.tiles_m * a.tiles_n * a.splits;
  zero_tile_init(zero);
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&tfull[b], 1);
        mbar_init(&tempty[b], 8);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int sg = 0; sg < a.nseg; ++sg)
        for (int q = 0; q < 4; ++q) tma_prefetch(&maps.m[sg][q]);
    }
  } else if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // the setup above touches no data of earlier kernels: it overlaps the predecessor's tail
  CV_PDL_ENTRY();
  const bool skipped = skip_if(a.skip);
  const SegPlan plan = skipped ? SegPlan{} : seg_plan(a);

  if (skipped) {
  } else if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    int it = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int m0, n0, kb0, nkb;
      if (!tc_work(a, w, TC_BM, BN, m0, n0, kb0, nkb)) continue;
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
        int lkb;
        const int sg = vseg(a, plan, kb0 + i, lkb);
        const int k0 = lkb * TC_BK;
        uint8_t* st = smem + s * Cfg::STAGE_BYTES;
        mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
        for (int h = 0; h < 2; ++h) {  // hi, lo
          load_slab(st + h * Cfg::A_BYTES, &maps.m[sg][h], &full[s], a.a[sg].kmajor, k0, m0, TC_BM);
          load_slab(st + 2 * Cfg::A_BYTES + h * Cfg::B_BYTES, &maps.m[sg][2 + h], &full[s], a.b[sg].kmajor, k0, n0,
                    BN);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    int it = 0, acc_i = 0;
    const uint64_t zdesc = zero_desc(zero);
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int m0, n0, kb0, nkb;
      if (!tc_work(a, w, TC_BM, BN, m0, n0, kb0, nkb)) continue;
      const int ab = acc_i & 1;
      if (acc_i >= 2) mbar_wait(&tempty[ab], ((acc_i >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dtm = tmem + ab * BN;
      int prev = -1;
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        int lkb;
        const int sg = vseg(a, plan, kb0 + i, lkb);
        const int shift = (prev >= 0 && prev != sg) ? plan.S[prev] - plan.S[sg] : 0;
        prev = sg;
        const int amn = a.a[sg].kmajor ? 0 : 1, bmn = a.b[sg].kmajor ? 0 : 1;
        const uint32_t idesc = f16_idesc(TC_BM, BN, amn, bmn);
        const uint32_t st = smem_u32(smem + s * Cfg::STAGE_BYTES);
        const uint32_t a_hi = st, a_lo = st + Cfg::A_BYTES;
        const uint32_t b_hi = st + 2 * Cfg::A_BYTES, b_lo = b_hi + Cfg::B_BYTES;
#pragma unroll
        for (int kk = 0; kk < TC_BK / 16; ++kk)
          umma_kstep<1>(dtm, op_desc(a_hi, amn, kk), op_desc(a_lo, amn, kk), op_desc(b_hi, bmn, kk),
                        op_desc(b_lo, bmn, kk), zdesc, idesc, i > 0 || kk > 0, kk == 0 ? shift : 0);
        umma_commit<1>(&empty[s]);  // slab free once these MMAs retire
      }
      umma_commit<1>(&tfull[ab]);   // accumulator ready for the epilogue
      ++acc_i;
    }
  } else if (warp >= 2) {
    // ---------------- epilogue ----------------
    const int q = warp & 3, half = (warp - 2) >> 2;
    const EpiRt rt = epi_prepare(a.epi);
    if (blockIdx.x == 0 && warp == 2 && lane == 0 && !a.partial) epi_publish(a.epi, rt);
    int acc_i = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int m0, n0, kb0, nkb;
      if (!tc_work(a, w, TC_BM, BN, m0, n0, kb0, nkb)) continue;
      const int ab = acc_i & 1;
      epi_prefetch_mask<BN>(a, m0, n0, q, half, lane);
      mbar_wait(&tfull[ab], (acc_i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      int lkb;
      const int last = vseg(a, plan, kb0 + nkb - 1, lkb);
      const float inv = plan.inv_a[last] * plan.inv_b[last];
      tile_epilogue<BN>(a, maps, rt, tmem + ab * BN, m0, n0, w / (a.tiles_m * a.tiles_n), inv, q, half, lane,
                        stg_all + (warp - 2) * TC_STG_BYTES, stg_all + 8 * TC_STG_BYTES + (warp - 2) * TC_HSTG_BYTES);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      ++acc_i;
    }
    if (lane == 0) bulk_wait0();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::TMEM_COLS));
  }
}

// split-K reduction in fixed order, then the real epilogue
__global__ void k_splitk_reduce(const float* partial, int splits, int M, int N, Epilogue epi, const int* skip,
                                int lower_only) {
  CV_PDL_ENTRY();
  if (skip_if(skip)) return;
  const EpiRt rt = epi_prepare(epi);
  if (blockIdx.x == 0 && threadIdx.x == 0) epi_publish(epi, rt);
  const int64_t total = (int64_t)M * N;
  float amax = 0.f, ramax = 0.f;
  if ((N & 7) == 0 && !lower_only) {
    // 8 adjacent columns per thread: 128-bit partial loads, vectorized epilogue
    const int64_t oct = total >> 3;
    for (int64_t qd = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; qd < oct; qd += (int64_t)gridDim.x * blockDim.x) {
      float v[8];
      const float4 p0 = *reinterpret_cast<const float4*>(partial + 8 * qd);
      const float4 p1 = *reinterpret_cast<const float4*>(partial + 8 * qd + 4);
      v[0] = p0.x; v[1] = p0.y; v[2] = p0.z; v[3] = p0.w; v[4] = p1.x; v[5] = p1.y; v[6] = p1.z; v[7] = p1.w;
      for (int z = 1; z < splits; ++z) {
        const float4 a0 = *reinterpret_cast<const float4*>(partial + (int64_t)z * total + 8 * qd);
        const float4 a1 = *reinterpret_cast<const float4*>(partial + (int64_t)z * total + 8 * qd + 4);
        v[0] += a0.x; v[1] += a0.y; v[2] += a0.z; v[3] += a0.w; v[4] += a1.x; v[5] += a1.y; v[6] += a1.z; v[7] += a1.w;
      }
      const int m = (int)((8 * qd) / N), n = (int)((8 * qd) % N);
      if (!epi_applyV<8>(epi, rt, m, n, v, amax, ramax))
        for (int t = 0; t < 8; ++t) epi_apply(epi, rt, m, n + t, v[t], amax, ramax);
    }
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
      float s = 0.f;
      for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * total + i];
      const int m = (int)(i / N), n = (int)(i % N);
      if (!lower_only || n <= m + lower_only - 1) epi_apply(epi, rt, m, n, s, amax, ramax);
    }
  }
  epi_flush_amax(epi, amax, ramax);
}

// Split-K form of the fused output-layer JVP (the ReLU tangent GEMM of the last hidden
// layer at batches too small for whole tiles to fill the machine): after the fixed-order
// sum of the partials, one warp per (row, 128-column group) applies the mask, stores the
// split tangent (unless head_only) and accumulates the group's share of the output
// tangent, sum_n a(m, n) V[n, :] + t(m, n) W[n, :] (warp butterfly), into head_part.
constexpr int kHeadGroupCols = 128;
__global__ void __launch_bounds__(256) k_splitk_reduce_head(const float* partial, int splits, int M, int N,
                                                            Epilogue epi, const int* skip) {
  CV_PDL_ENTRY();
  if (skip_if(skip)) return;
  const EpiRt rt = epi_prepare(epi);
  if (blockIdx.x == 0 && threadIdx.x == 0) epi_publish(epi, rt);
  const int lane = threadIdx.x & 31;
  const int groups = (N + kHeadGroupCols - 1) / kHeadGroupCols;
  const int64_t total = (int64_t)M * N;
  const int hc = epi.head_c;
  const bool store = !epi.head_only;
  __shared__ float hred[8][16 * 33];
  float amax = 0.f;
  for (int64_t wk = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); wk < (int64_t)M * groups;
       wk += (int64_t)gridDim.x * 8) {
    const int m = (int)(wk / groups), g = (int)(wk % groups);
    const int n = g * kHeadGroupCols + 4 * lane;
    float v[4] = {0.f, 0.f, 0.f, 0.f}, av[4] = {0.f, 0.f, 0.f, 0.f}, t[4] = {0.f, 0.f, 0.f, 0.f};
    const bool full = n + 3 < N;
    if (n < N) {
      const int64_t o = (int64_t)m * N + n;
      for (int z = 0; z < splits; ++z) {
        if (full) {
          const float4 q = *reinterpret_cast<const float4*>(partial + (int64_t)z * total + o);
          v[0] += q.x; v[1] += q.y; v[2] += q.z; v[3] += q.w;
        } else {
          for (int j = 0; j < 4 && n + j < N; ++j) v[j] += partial[(int64_t)z * total + o + j];
        }
      }
      if (full) {  // 8-byte mask loads and split stores (mask_ld, ld multiples of 8; n of 4)
        H4 mh, ml, oh, ol;
        mh.u = *reinterpret_cast<const uint2*>(epi.mask_hi + (int64_t)m * epi.mask_ld + n);
        ml.u = *reinterpret_cast<const uint2*>(epi.mask_lo + (int64_t)m * epi.mask_ld + n);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float hi = __half2float(mh.h[j]);
          av[j] = (hi + __half2float(ml.h[j])) * rt.mask_inv;
          t[j] = hi > 0.f ? v[j] : 0.f;
          split16(t[j], rt.out_s, oh.h[j], ol.h[j]);
          amax = fmaxf(amax, fabsf(t[j]));
        }
        if (store) {
          *reinterpret_cast<uint2*>(epi.out_hi + (int64_t)m * epi.ld + n) = oh.u;
          *reinterpret_cast<uint2*>(epi.out_lo + (int64_t)m * epi.ld + n) = ol.u;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (n + j >= N) break;
          const int64_t mi = (int64_t)m * epi.mask_ld + n + j;
          const float hi = __half2float(epi.mask_hi[mi]);
          av[j] = (hi + __half2float(epi.mask_lo[mi])) * rt.mask_inv;
          t[j] = hi > 0.f ? v[j] : 0.f;
          if (store) {
            split16(t[j], rt.out_s, epi.out_hi[(int64_t)m * epi.ld + n + j], epi.out_lo[(int64_t)m * epi.ld + n + j]);
            amax = fmaxf(amax, fabsf(t[j]));
          }
        }
      }
    }
    float h[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) h[k] = 0.f;
    if (hc == 10 && full && !(((uintptr_t)epi.head_v | (uintptr_t)epi.head_w) & 15)) {
      // 4 columns x 10 outputs = 10 float4 per matrix, contiguous
      const float4* vq = reinterpret_cast<const float4*>(epi.head_v + (int64_t)n * 10);
      const float4* wq = reinterpret_cast<const float4*>(epi.head_w + (int64_t)n * 10);
#pragma unroll
      for (int u = 0; u < 10; ++u) {
        const float4 vv = __ldg(vq + u), ww = __ldg(wq + u);
        const float ve[4] = {vv.x, vv.y, vv.z, vv.w}, we[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int f = 4 * u + q, j = f / 10, k = f % 10;  // flat index over (column j, output k)
          h[k] = fmaf(av[j], ve[q], fmaf(t[j], we[q], h[k]));
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (n + j >= N) break;
        const float* vr = epi.head_v + (int64_t)(n + j) * hc;
        const float* wr = epi.head_w + (int64_t)(n + j) * hc;
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k < hc) h[k] = fmaf(av[j], __ldg(vr + k), fmaf(t[j], __ldg(wr + k), h[k]));
      }
    }
    // the warp's 32 lane partials per output: through shared memory, fixed order
    float* red = hred[threadIdx.x >> 5];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < hc) red[k * 33 + lane] = h[k];
    __syncwarp();
    if (lane < hc) {
      float x = 0.f;
      for (int l = 0; l < 32; ++l) x += red[lane * 33 + l];
      epi.head_part[((int64_t)g * M + m) * hc + lane] = x;
    }
  }
  float ramax = 0.f;
  epi_flush_amax(epi, amax, ramax);
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

struct MapKey {
  const void* ptr;
  int64_t inner, outer, ld;
  int box0, box1;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && inner == o.inner && outer == o.outer && ld == o.ld && box0 == o.box0 && box1 == o.box1;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = (size_t)k.ptr;
    h = h * 1000003u ^ (size_t)k.inner;
    h = h * 1000003u ^ (size_t)k.outer;
    h = h * 1000003u ^ (size_t)k.ld;
    h = h * 1000003u ^ (size_t)(k.box0 * 4096 + k.box1);
    return h;
  }
};

// 2D fp16 map: dims {inner, outer}, row stride ld elements, OOB zero fill, SWIZZLE_128B
// (the inner box extent is always 64 elements = 128 B).
static CUtensorMap make_map(const __half* ptr, int64_t inner, int64_t outer, int64_t ld, int box0, int box1) {
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  static std::mutex mu;
  MapKey key{ptr, inner, outer, ld, box0, box1};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  auto fn = encode_fn();
  if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)ptr, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, m);
  return m;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// Output map of the TMA-store epilogue (rank 2 or 3), cached like the operand maps.
struct OutKey {
  const void* ptr;
  int64_t d0, d1, d2, s1;
  int fp16;
  bool operator==(const OutKey& o) const {
    return ptr == o.ptr && d0 == o.d0 && d1 == o.d1 && d2 == o.d2 && s1 == o.s1 && fp16 == o.fp16;
  }
};
struct OutKeyHash {
  size_t operator()(const OutKey& k) const {
    size_t h = (size_t)k.ptr;
    h = h * 1000003u ^ (size_t)k.d0;
    h = h * 1000003u ^ (size_t)k.d1;
    h = h * 1000003u ^ (size_t)k.d2;
    h = h * 1000003u ^ (size_t)(k.s1 * 2 + k.fp16);
    return h;
  }
};

// fp16: dims {cols, rows}, row stride ld, box {16, 32}, SWIZZLE_32B.
// fp32: dims {cols, rows}, box {16, 32}, SWIZZLE_64B; split-K partials (slabs > 0):
// dims {cols, rows, slabs}, box {16, 32, 1} -- rank 3 even for a single slab, since the
// partial epilogue always issues the 3-D store.
static CUtensorMap make_out_map(const void* ptr, int fp16, int64_t cols, int64_t rows, int64_t slabs, int64_t ld) {
  static std::unordered_map<OutKey, CUtensorMap, OutKeyHash> cache;
  static std::mutex mu;
  OutKey key{ptr, cols, rows, slabs, ld, fp16};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  auto fn = encode_fn();
  if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
  CUtensorMap m;
  const int esz = fp16 ? 2 : 4;
  const cuuint32_t rank = slabs > 0 ? 3 : 2;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)(slabs > 0 ? slabs : 1)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * esz, (cuuint64_t)ld * esz * rows};
  cuuint32_t box[3] = {16, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(&m, fp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, (void*)ptr, dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  fp16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (out) failed (" + std::to_string((int)r) + ")");
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, m);
  return m;
}

// The TMA-store epilogue a GEMM's output allows without split-K partials:
// 0 none (per-thread stores), 1 fp16 split pair, 2 fp32 (mirrors setup_out).
static int tma_out_mode(const GemmArgs& g) {
  const Epilogue& e = g.epi;
  if (e.mode == EPI_GRAM || e.mode == EPI_ACCUM) {
    // whole computed tiles are written (lower-only GEMMs: also the part of a diagonal tile
    // above the diagonal, which the row lane never reads)
    if ((e.ld & 3) || !aligned16(e.out)) return 0;
    return e.mode == EPI_GRAM && e.first ? 2 : 3;
  }
  if (g.lower_only) return 0;
  if (e.mode == EPI_STORE) return ((e.ld & 3) || !aligned16(e.out)) ? 0 : 2;
  const bool relu_mask = (e.mode == EPI_SPLIT_MASK || e.mode == EPI_HVP) && e.act == CV_ACT_RELU && !e.raw &&
                         e.mask_div == 1 && (e.mask_ld & 7) == 0 && aligned16(e.mask_hi);
  if (!(e.mode == EPI_SPLIT_ACT || relu_mask)) return 0;
  if ((e.ld & 7) || !aligned16(e.out_hi) || !aligned16(e.out_lo)) return 0;
  return 1;
}

// Choose the TMA-store epilogue when the mode and layout allow it.
static void setup_out(const GemmArgs& g, TcMaps& maps, TcArgs& a, float* partial, int splits) {
  a.tma_out = 0;
  const Epilogue& e = g.epi;
  if (!partial && (e.mode == EPI_GRAM || e.mode == EPI_ACCUM)) {
    const int mode = tma_out_mode(g);
    if (!mode) return;
    maps.o[0] = make_out_map(e.out, 0, g.N, g.M, 0, e.ld);
    a.tma_out = mode;
    return;
  }
  if (g.lower_only) return;
  if (partial) {
    if ((g.N & 3) || !aligned16(partial)) return;
    maps.o[0] = make_out_map(partial, 0, g.N, g.M, splits, g.N);
    a.tma_out = 2;
    return;
  }
  if (e.mode == EPI_STORE) {
    if ((e.ld & 3) || !aligned16(e.out)) return;
    maps.o[0] = make_out_map(e.out, 0, g.N, g.M, 0, e.ld);
    a.tma_out = 2;
    return;
  }
  const bool relu_mask = (e.mode == EPI_SPLIT_MASK || e.mode == EPI_HVP) && e.act == CV_ACT_RELU && !e.raw &&
                         e.mask_div == 1 && (e.mask_ld & 7) == 0 && aligned16(e.mask_hi);
  if (!(e.mode == EPI_SPLIT_ACT || relu_mask)) return;
  if ((e.ld & 7) || !aligned16(e.out_hi) || !aligned16(e.out_lo)) return;
  maps.o[0] = make_out_map(e.out_hi, 1, g.N, g.M, 0, e.ld);
  maps.o[1] = make_out_map(e.out_lo, 1, g.N, g.M, 0, e.ld);
  a.tma_out = 1;
}

// Operand majors: A(m,k) = p[m*si + k*sj]; K-major iff sj == 1.
static bool op_ok(const Operand& o) {
  if (o.f32 || !o.hi || !o.lo || !o.sc) return false;
  if (!aligned16(o.hi) || !aligned16(o.lo)) return false;
  const int64_t ld = o.sj == 1 ? o.si : (o.si == 1 ? o.sj : -1);
  return ld > 0 && (ld % 8) == 0 && (o.sj == 1 || o.si == 1);
}

bool gemm_tc_supported(const GemmArgs& g) {
  if (g.M < 64 || g.N < 8) return false;
  for (int s = 0; s < g.nseg; ++s) {
    if (g.seg[s].K < 16) return false;
    if (!op_ok(g.seg[s].A) || !op_ok(g.seg[s].B)) return false;
    // MN-major operands are staged in 64-wide chunks: the narrow (N <= 32) tile
    // takes K-major B only
    if (g.N <= 32 && g.seg[s].B.si != 1) return false;
  }
  return true;
}

// Tensor maps and segment geometry shared by the 1-CTA and 2-CTA launchers.
// A rows per CTA = TC_BM; B box rows = bbox (BN, or BN/2 for the CTA pair).
static void fill_args(const GemmArgs& g, int bbox, TcMaps& maps, TcArgs& a) {
  a.M = g.M;
  a.N = g.N;
  a.nseg = g.nseg;
  a.kb_total = 0;
  for (int s = 0; s < 2; ++s) {
    a.asc[s] = s < g.nseg ? g.seg[s].A.sc : nullptr;
    a.bsc[s] = s < g.nseg ? g.seg[s].B.sc : nullptr;
  }
  for (int s = 0; s < g.nseg; ++s) {
    const GemmSeg& sg = g.seg[s];
    const bool akm = sg.A.sj == 1, bkm = sg.B.si == 1;  // B(k,n) = p[k*si + n*sj]: K-major iff si == 1
    a.a[s].kmajor = akm;
    a.b[s].kmajor = bkm;
    a.kb[s] = (sg.K + TC_BK - 1) / TC_BK;
    a.kb_total += a.kb[s];
    const int64_t lda = akm ? sg.A.si : sg.A.sj;
    const int64_t ldb = bkm ? sg.B.sj : sg.B.si;
    for (int h = 0; h < 2; ++h) {
      const __half* pa = h ? sg.A.lo : sg.A.hi;
      const __half* pb = h ? sg.B.lo : sg.B.hi;
      maps.m[s][h] = akm ? make_map(pa, sg.K, g.M, lda, TC_BK, TC_BM) : make_map(pa, g.M, sg.K, lda, 64, TC_BK);
      maps.m[s][2 + h] = bkm ? make_map(pb, sg.K, g.N, ldb, TC_BK, bbox) : make_map(pb, g.N, sg.K, ldb, 64, TC_BK);
    }
  }
  if (g.nseg < 2) a.kb[1] = 0;
  a.epi = g.epi;
  a.skip = g.skip;
  a.lower_only = g.lower_only;
  a.cyc_nb = g.cyc_nb;
  a.cyc_skip = g.cyc_skip;
}

template <int BN, int STAGES>
static int launch_tc(cv_ctx* ctx, const GemmArgs& g, int splits, float* ext_partial = nullptr) {
  using Cfg = TcCfg<BN, STAGES>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_gemm_tc<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr_set = true;
  }
  TcMaps maps;
  TcArgs a{};
  fill_args(g, BN, maps, a);
  a.kb_per_split = (a.kb_total + splits - 1) / splits;
  splits = (a.kb_total + a.kb_per_split - 1) / a.kb_per_split;
  a.splits = splits;
  a.tiles_m = (g.M + TC_BM - 1) / TC_BM;
  a.tiles_n = (g.N + BN - 1) / BN;
  float* part = nullptr;
  if (ext_partial) {
    a.partial = ext_partial;  // raw split-K partials for the caller, no epilogue
  } else if (splits > 1) {
    part = (float*)ctx->pool.get(sizeof(float) * (size_t)splits * g.M * g.N);
    a.partial = part;
  }
  setup_out(g, maps, a, a.partial, splits);
  if (g.epi.head_part && a.tma_out != 1 && !part)
    throw std::runtime_error("fused output head needs the TMA split epilogue");
  const int work = a.tiles_m * a.tiles_n * splits;
  const int sms = g.max_ctas > 0 && g.max_ctas < ctx->sm_count ? g.max_ctas : ctx->sm_count;
  const int grid = work < sms ? work : sms;
  cudaStream_t st = g.stream ? g.stream : ctx->stream;
  launch_k(st, k_gemm_tc<BN, STAGES>, grid, Cfg::THREADS, Cfg::SMEM, maps, a);
  ctx->launches++;
  if (part) {
    if (g.epi.head_part)
      launch_k(st, k_splitk_reduce_head, 4 * ctx->sm_count, 256, 0, (const float*)part, splits, g.M, g.N, g.epi,
               g.skip);
    else
      launch_k(st, k_splitk_reduce, 4 * ctx->sm_count, 256, 0, part, splits, g.M, g.N, g.epi, g.skip, g.lower_only);
    ctx->launches++;
    if (st == ctx->side2 && st) ctx->deferred2.push_back(part);
    else if (st != ctx->stream) ctx->deferred.push_back(part);  // reused only after the join
    else ctx->pool.put(part);  // stream-ordered reuse: later users enqueue after this kernel
  }
  return splits;
}

#include "gemm_tc2.cuh"

// Tile configuration and split-K factor of a GEMM on `sms` SMs.
struct TcPlan {
  int kind;  // 0: <32,4>, 1: 2-CTA 256x256, 2: <256,2>, 3: <128,3>, 5: <64,4>
  int tiles, kb_total, splits;
  int M, N;
};

static double plan_time(const TcPlan& p, int sms);

static TcPlan tc_plan_kind(const GemmArgs& g, int sms, int kind) {
  TcPlan p;
  p.kind = kind;
  const int bn = kind == 0 ? 32 : (kind == 5 ? 64 : (kind == 3 ? 128 : 256));
  const int bm = kind == 1 ? 256 : TC_BM;
  p.tiles = ((g.M + bm - 1) / bm) * ((g.N + bn - 1) / bn);
  const int slots = kind == 1 ? sms / 2 : sms;  // concurrent work items
  p.kb_total = 0;
  for (int s = 0; s < g.nseg; ++s) p.kb_total += (g.seg[s].K + TC_BK - 1) / TC_BK;
  // split K when the tile grid cannot fill the machine (weight-gradient GEMMs: M, N ~ 1e3, K = batch)
  p.M = g.M;
  p.N = g.N;
  p.splits = 1;
  // split-K when the tiles cannot fill the slots (weight gradients: K = batch; every GEMM
  // at the per-rank batch of a data-parallel run); the fixed-order reduce applies any
  // element-wise epilogue
  const bool splittable = !g.lower_only && (g.epi.mode == EPI_STORE || g.epi.mode == EPI_SPLIT_ACT ||
                                            g.epi.mode == EPI_SPLIT_MASK || g.epi.mode == EPI_HVP);
  if (splittable && p.tiles < slots && !g.unsplit) {
    // the split-K factor whose rounds of items fill the slots best (incl. the partials' round trip)
    double best = 1e300;
    int bs = 1;
    const int smax = p.kb_total / 4 < 32 ? p.kb_total / 4 : 32;
    for (int sp = 1; sp <= smax; ++sp) {
      p.splits = sp;
      const double t = plan_time(p, sms);
      if (t < best) {
        best = t;
        bs = sp;
      }
    }
    p.splits = bs;
  }
  return p;
}

// relative time of a plan: rounds of work items x k-blocks per item (+ fill/epilogue),
// per SM; a 2-CTA tile costs each SM what a 1-CTA 128 x 256 tile does
static double plan_time(const TcPlan& p, int sms) {
  const int slots = p.kind == 1 ? sms / 2 : sms;
  const int items = p.tiles * p.splits;
  const int rounds = (items + slots - 1) / slots;
  const double item_kb = (double)((p.kb_total + p.splits - 1) / p.splits);
  // 2-stage ring / narrower tiles (measured on B200)
  const double pen = p.kind == 2 ? 1.3 : (p.kind == 3 ? 1.2 : (p.kind == 5 ? 1.6 : 1.0));
  const double per_kb = p.kind == 3 ? 0.5 : (p.kind == 5 ? 0.25 : 1.0);  // narrower tiles: less MMA work
  // split-K partials: written once and read once by the fixed-order reduce (units of
  // ~1.2 us, one 256x256x64 3xFP16 k-block on a CTA pair, at ~6.5 TB/s)
  const double red = p.splits > 1 ? (double)(p.splits + 1) * p.M * p.N * 4.0 / 7.8e6 + 2.0 : 0.0;
  return rounds * (item_kb * per_kb * pen + 4.0) + red;
}

static TcPlan tc_plan_search(const GemmArgs& g, int sms);

// Plans depend only on the GEMM's geometry and SM budget: memoised, so the
// co-scheduling split search (gemm_pair) and every launch stay off the host's
// critical path.
struct PlanKey {
  int M, N, K0, K1, nseg, mode, lower, sms, unsplit;
  bool operator==(const PlanKey& o) const {
    return M == o.M && N == o.N && K0 == o.K0 && K1 == o.K1 && nseg == o.nseg && mode == o.mode &&
           lower == o.lower && sms == o.sms && unsplit == o.unsplit;
  }
};
struct PlanKeyHash {
  size_t operator()(const PlanKey& k) const {
    size_t h = (size_t)k.M * 1000003u ^ (size_t)k.N;
    h = h * 1000003u ^ (size_t)k.K0;
    h = h * 1000003u ^ (size_t)k.K1;
    h = h * 1000003u ^ (size_t)(k.nseg * 64 + k.mode * 2 + k.lower);
    return (h * 1000003u ^ (size_t)k.sms) * 2 + (size_t)k.unsplit;
  }
};

static TcPlan tc_plan(const GemmArgs& g, int sms) {
  static std::unordered_map<PlanKey, TcPlan, PlanKeyHash> cache;
  static std::mutex mu;
  const PlanKey key{g.M, g.N, g.seg[0].K, g.nseg > 1 ? g.seg[1].K : 0, g.nseg, g.epi.mode, g.lower_only, sms,
                    g.unsplit};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const TcPlan p = tc_plan_search(g, sms);
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() > 65536) cache.clear();
  cache.emplace(key, p);
  return p;
}

static TcPlan tc_plan_search(const GemmArgs& g, int sms) {
  if (g.N <= 32) return tc_plan_kind(g, sms, 0);
  const bool pair = g.M >= 256 && g.N >= 256;
  const bool wide = g.N >= 512;
  TcPlan best = tc_plan_kind(g, sms, pair ? 1 : (wide ? 2 : 3));
  const int slots = best.kind == 1 ? sms / 2 : sms;
  if (g.epi.mode == EPI_STORE || best.tiles < slots) {
    // split-K weight gradients and under-filled grids: the tile shape that wastes the
    // least of the edges / fills the slots best
    for (int k : {1, 2, 3, 5}) {  // (kind 5, 128x64: only for grids the wider tiles cannot fill)
      if (k == 1 && !pair) continue;
      const TcPlan c = tc_plan_kind(g, sms, k);
      if (plan_time(c, sms) < plan_time(best, sms)) best = c;
    }
  }
  return best;
}

double gemm_tc_estimate(const cv_ctx* ctx, const GemmArgs& g, int ctas) {
  (void)ctx;
  return plan_time(tc_plan(g, ctas), ctas);
}

// Number of column groups of the fused output-layer head this GEMM would write
// (tile_epilogue_tma), or 0 when the GEMM cannot carry the head (engine, layout,
// epilogue mode or tile plan); the caller then runs the output layer separately.
int gemm_tc_head_groups(const cv_ctx* ctx, const GemmArgs& g, int* via_reduce) {
  if (via_reduce) *via_reduce = 0;
  if (ctx->engine == CV_ENGINE_SIMT || !gemm_tc_supported(g) || g.lower_only) return 0;
  const Epilogue& e = g.epi;
  const bool jvp_head = e.mode == EPI_SPLIT_MASK && e.act == CV_ACT_RELU && !e.raw && e.mask_div == 1 &&
                        !(e.mask_ld & 7) && aligned16(e.mask_hi) && aligned16(e.mask_lo);
  const bool fwd_head = e.mode == EPI_SPLIT_ACT && !e.head_only;
  if (!(jvp_head || fwd_head) || (e.ld & 7) || !aligned16(e.out_hi) || !aligned16(e.out_lo)) return 0;
  const int sms = g.max_ctas > 0 && g.max_ctas < ctx->sm_count ? g.max_ctas : ctx->sm_count;
  const TcPlan p = tc_plan(g, sms);
  if (p.kind == 0 || p.splits > 1) return 0;
  if (via_reduce && jvp_head && !g.epi.bits_out) {
    // whole tiles that leave most of the machine idle (small batches): run split-K and
    // form the head in the fixed-order reduction instead (k_splitk_reduce_head)
    GemmArgs gs = g;
    gs.unsplit = 0;
    const TcPlan q = tc_plan(gs, sms);
    if (q.kind != 0 && q.splits > 1 && plan_time(q, sms) < 0.6 * plan_time(p, sms)) {
      *via_reduce = 1;
      return (g.N + kHeadGroupCols - 1) / kHeadGroupCols;
    }
  }
  const int bn = p.kind == 5 ? 64 : (p.kind == 3 ? 128 : 256);
  return 2 * ((g.N + bn - 1) / bn);
}

bool gemm_tc_tma_split(const cv_ctx* ctx, const GemmArgs& g) {
  if (ctx->engine == CV_ENGINE_SIMT || !gemm_tc_supported(g) || tma_out_mode(g) != 1) return false;
  const int sms = g.max_ctas > 0 && g.max_ctas < ctx->sm_count ? g.max_ctas : ctx->sm_count;
  const TcPlan p = tc_plan(g, sms);
  return p.kind != 0 && p.splits == 1;
}

// cv_gemm_bench's plan override (tuning the planner's cost model; never set on a product path)
int g_force_kind = -1, g_force_splits = 0;

void gemm_tc(cv_ctx* ctx, const GemmArgs& g) {
  const int sms = g.max_ctas > 0 && g.max_ctas < ctx->sm_count ? g.max_ctas : ctx->sm_count;
  TcPlan p = tc_plan(g, sms);
  if (g_force_kind >= 0) {
    p = tc_plan_kind(g, sms, g_force_kind);
    if (g_force_splits > 0) p.splits = g_force_splits;
  }
  switch (p.kind) {
    case 0: launch_tc<32, 4>(ctx, g, p.splits); break;
    case 1: launch_tc2<3, 256>(ctx, g, p.splits); break;
    case 2: launch_tc<256, 2>(ctx, g, p.splits); break;
    case 5: launch_tc<64, 4>(ctx, g, p.splits); break;
    default: launch_tc<128, 3>(ctx, g, p.splits); break;
  }
}

// Narrow (N <= 32) GEMM returning raw split-K partials [splits][M][N]: the output
// layer's JVP, whose row-wise loss Hessian cannot be applied per element.
int gemm_tc_partial(cv_ctx* ctx, const GemmArgs& g, float** partial) {
  int kb_total = 0;
  for (int s = 0; s < g.nseg; ++s) kb_total += (g.seg[s].K + TC_BK - 1) / TC_BK;
  const int tiles = (g.M + TC_BM - 1) / TC_BM;
  int splits = tiles < ctx->sm_count ? ctx->sm_count / tiles : 1;
  if (splits > kb_total / 4) splits = kb_total / 4;
  if (splits < 1) splits = 1;
  const int kbs = (kb_total + splits - 1) / splits;
  splits = (kb_total + kbs - 1) / kbs;
  *partial = (float*)ctx->pool.get(sizeof(float) * (size_t)splits * g.M * g.N);
  return launch_tc<32, 4>(ctx, g, splits, *partial);
}

}  // namespace cv
