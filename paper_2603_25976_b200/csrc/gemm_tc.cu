// tcgen05 / TMA split-precision (3xTF32) GEMM engine for sm_100a.
//
//   D[M x N] = sum_seg A_seg[M x K] . B_seg[K x N]        (fp32 accumulate in TMEM)
//   with X = X_hi + X_lo (both stored fp32, hi exactly tf32):
//   D = A_hi.B_hi + A_hi.B_lo + A_lo.B_hi                 (3 tcgen05.mma kind::tf32)
//
// Operands are the split buffers of internal.h (row-major, leading dim ld), each
// either K-major (K contiguous) or MN-major (M/N contiguous); both are native
// tcgen05 operand majors for tf32, so no transposed copies exist anywhere.
//
// One CTA = one 128 x BN output tile (BN = 128 or 256), 8 warps:
//   warp 0 lane 0 : TMA producer      (cp.async.bulk.tensor.2d, SWIZZLE_128B)
//   warp 1 lane 0 : MMA issuer        (tcgen05.mma.cta_group::1.kind::tf32)
//   warps 0-7     : epilogue          (tcgen05.ld 32x32b -> registers -> 128-bit fused epilogue)
// smem ring of STAGES x {A_hi, A_lo, B_hi, B_lo} 32-wide K slabs, full/empty
// mbarriers between TMA and MMA, tcgen05.commit frees a slab / signals the epilogue.
// Split-K (grid.z) writes fp32 partials that a fixed-order reduction folds in.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <stdexcept>
#include <unordered_map>

#include "common.cuh"
#include "epilogue.cuh"
#include "internal.h"

namespace cv {

constexpr int TC_BM = 128;
constexpr int TC_BK = 32;  // fp32 elements = 128 bytes = one SWIZZLE_128B row

struct TcOperand {
  int kmajor;   // 1: K contiguous, 0: M/N contiguous
};

struct TcArgs {
  int M, N;
  int nseg;
  int kb[2];          // k-blocks per segment
  int kb_total;
  int kb_per_split;
  TcOperand a[2], b[2];
  Epilogue epi;
  const int* skip;
  int lower_only;
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

// UMMA shared-memory descriptor, version 1 (sm_100).  layout: 2 = SWIZZLE_128B
// (K-major: 16 B granules, 8-row atoms), 1 = SWIZZLE_128B_BASE32B (the only
// MN-major layout for 32-bit operands: 32 B granules, 4-row atoms).
CV_DEV uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version
  d |= (uint64_t)layout << 61;
  return d;
}

// Instruction descriptor: kind::tf32, D f32, A/B tf32, majors, N, M.
__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

CV_DEV void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

CV_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
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

// ---------------------------------------------------------------------------
// Kernel
// ---------------------------------------------------------------------------
struct TcMaps {
  CUtensorMap m[2][4];  // [seg][A_hi, A_lo, B_hi, B_lo]
};

template <int BN, int STAGES>
struct TcCfg {
  static constexpr int A_BYTES = TC_BM * TC_BK * 4;  // 16 KB
  static constexpr int B_BYTES = BN * TC_BK * 4;     // 16 / 32 KB
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = 2 * BN;           // double-buffered accumulator
  static constexpr int THREADS = 320;                // w0 TMA, w1 MMA, w2..w9 epilogue
};

CV_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// work item -> (m0, n0, first k-block, k-blocks); split index slowest so that
// co-resident CTAs share K ranges (and therefore L2-resident operand panels)
CV_DEV bool tc_work(const TcArgs& a, int w, int bn, int& m0, int& n0, int& kb0, int& nkb) {
  const int tiles = a.tiles_m * a.tiles_n;
  const int split = w / tiles, t = w % tiles;
  m0 = (t / a.tiles_n) * TC_BM;
  n0 = (t % a.tiles_n) * bn;
  kb0 = split * a.kb_per_split;
  nkb = min(a.kb_total, kb0 + a.kb_per_split) - kb0;
  return !(a.lower_only && n0 > m0 + TC_BM - 1);
}

// Persistent: grid = min(work, SMs); each CTA loops over work items.  The TMEM
// accumulator is double buffered so the epilogue of item i overlaps the
// mainloop of item i+1.
template <int BN, int STAGES>
__global__ void __launch_bounds__(320, 1) k_gemm_tc(const __grid_constant__ TcMaps maps, const TcArgs a) {
  using Cfg = TcCfg<BN, STAGES>;
  if (skip_if(a.skip)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = a.tiles_m * a.tiles_n * a.splits;
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

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    int it = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int m0, n0, kb0, nkb;
      if (!tc_work(a, w, BN, m0, n0, kb0, nkb)) continue;
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
        const int kb = kb0 + i;
        const int sg = kb < a.kb[0] ? 0 : 1;
        const int k0 = (sg == 0 ? kb : kb - a.kb[0]) * TC_BK;
        uint8_t* st = smem + s * Cfg::STAGE_BYTES;
        mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
        for (int h = 0; h < 2; ++h) {  // hi, lo
          uint8_t* sa = st + h * Cfg::A_BYTES;
          if (a.a[sg].kmajor) {
            tma_load_2d(sa, &maps.m[sg][h], &full[s], k0, m0);
          } else {
#pragma unroll
            for (int j = 0; j < TC_BM / 32; ++j) tma_load_2d(sa + j * 4096, &maps.m[sg][h], &full[s], m0 + 32 * j, k0);
          }
          uint8_t* sb = st + 2 * Cfg::A_BYTES + h * Cfg::B_BYTES;
          if (a.b[sg].kmajor) {
            tma_load_2d(sb, &maps.m[sg][2 + h], &full[s], k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 32; ++j)
              tma_load_2d(sb + j * 4096, &maps.m[sg][2 + h], &full[s], n0 + 32 * j, k0);
          }
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    int it = 0, acc_i = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int m0, n0, kb0, nkb;
      if (!tc_work(a, w, BN, m0, n0, kb0, nkb)) continue;
      const int ab = acc_i & 1;
      if (acc_i >= 2) mbar_wait(&tempty[ab], ((acc_i >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dtm = tmem + ab * BN;
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int kb = kb0 + i;
        const int sg = kb < a.kb[0] ? 0 : 1;
        const int amn = a.a[sg].kmajor ? 0 : 1, bmn = a.b[sg].kmajor ? 0 : 1;
        const uint32_t idesc = tf32_idesc(TC_BM, BN, amn, bmn);
        const uint32_t st = smem_u32(smem + s * Cfg::STAGE_BYTES);
        const uint32_t a_hi = st, a_lo = st + Cfg::A_BYTES;
        const uint32_t b_hi = st + 2 * Cfg::A_BYTES, b_lo = b_hi + Cfg::B_BYTES;
#pragma unroll
        for (int kk = 0; kk < TC_BK / 8; ++kk) {
          // K-major (SW128): rows of 128 B, 8-row atoms (SBO 1024), k-step = +32 B in the row.
          // MN-major (SW128_BASE32B): 32-wide MN chunks 4 KB apart (LBO), K rows of 128 B in
          // 4-row atoms (SBO 512), k-step = 8 rows = +1024 B.
          const uint32_t aoff = amn ? kk * 1024 : kk * 32;
          const uint32_t boff = bmn ? kk * 1024 : kk * 32;
          const uint32_t albo = amn ? 4096 : 16, blbo = bmn ? 4096 : 16;
          const uint32_t asbo = amn ? 512 : 1024, bsbo = bmn ? 512 : 1024;
          const uint32_t alay = amn ? 1 : 2, blay = bmn ? 1 : 2;
          const uint64_t dah = umma_desc(a_hi + aoff, albo, asbo, alay), dal = umma_desc(a_lo + aoff, albo, asbo, alay);
          const uint64_t dbh = umma_desc(b_hi + boff, blbo, bsbo, blay), dbl = umma_desc(b_lo + boff, blbo, bsbo, blay);
          const uint32_t acc0 = (i > 0 || kk > 0) ? 1u : 0u;
          umma_tf32(dtm, dah, dbh, idesc, acc0);
          umma_tf32(dtm, dah, dbl, idesc, 1u);
          umma_tf32(dtm, dal, dbh, idesc, 1u);
        }
        umma_commit(&empty[s]);  // slab free once these MMAs retire
      }
      umma_commit(&tfull[ab]);   // accumulator ready for the epilogue
      ++acc_i;
    }
  } else if (warp >= 2) {
    // ---------------- epilogue: TMEM -> registers -> fused epilogue ----------------
    // warp w reads TMEM lane quadrant (w % 4); warps 2-5 take the first column half,
    // warps 6-9 the second.
    const int q = warp & 3, half = (warp - 2) >> 2;
    int acc_i = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int m0, n0, kb0, nkb;
      if (!tc_work(a, w, BN, m0, n0, kb0, nkb)) continue;
      const int ab = acc_i & 1;
      mbar_wait(&tfull[ab], (acc_i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int m = m0 + q * 32 + lane;
      const int split = w / (a.tiles_m * a.tiles_n);
      const uint32_t trow = tmem + ab * BN + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c = half; c < BN / 32; c += 2) {
        uint32_t r[32];
        tmem_ld32(trow + c * 32, r);
        if (m >= a.M) continue;
        const int nb = n0 + c * 32;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        const bool full_chunk = nb + 32 <= a.N && (!a.lower_only || nb + 31 <= m);
        if (a.partial) {
          float* dst = a.partial + ((int64_t)split * a.M + m) * a.N + nb;
          if (full_chunk && al16(dst)) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (nb + j < a.N) dst[j] = v[j];
          }
        } else if (!(full_chunk && epi_apply32(a.epi, m, nb, v))) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = nb + j;
            if (n < a.N && (!a.lower_only || n <= m)) epi_apply(a.epi, m, n, v[j]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      ++acc_i;
    }
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
  if (skip_if(skip)) return;
  const int64_t total = (int64_t)M * N;
  if ((N & 3) == 0 && !lower_only) {
    // 4 adjacent columns per thread: 128-bit partial loads, vectorized epilogue
    const int64_t quads = total >> 2;
    for (int64_t qd = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; qd < quads;
         qd += (int64_t)gridDim.x * blockDim.x) {
      float4 s = *reinterpret_cast<const float4*>(partial + 4 * qd);
      for (int z = 1; z < splits; ++z) {
        const float4 p = *reinterpret_cast<const float4*>(partial + (int64_t)z * total + 4 * qd);
        s.x += p.x; s.y += p.y; s.z += p.z; s.w += p.w;
      }
      const int m = (int)((4 * qd) / N), n = (int)((4 * qd) % N);
      const float v[4] = {s.x, s.y, s.z, s.w};
      if (!epi_applyV<4>(epi, m, n, v))
        for (int t = 0; t < 4; ++t) epi_apply(epi, m, n + t, v[t]);
    }
    return;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * total + i];
    const int m = (int)(i / N), n = (int)(i % N);
    if (!lower_only || n <= m) epi_apply(epi, m, n, s);
  }
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
  int box0, box1, mn;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && inner == o.inner && outer == o.outer && ld == o.ld && box0 == o.box0 && box1 == o.box1 &&
           mn == o.mn;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = (size_t)k.ptr;
    h = h * 1000003u ^ (size_t)k.inner;
    h = h * 1000003u ^ (size_t)k.outer;
    h = h * 1000003u ^ (size_t)k.ld;
    h = h * 1000003u ^ (size_t)(k.box0 * 4096 + k.box1 * 2 + k.mn);
    return h;
  }
};

// 2D fp32 map: dims {inner, outer}, row stride ld elements, OOB zero fill; K-major
// operands use SWIZZLE_128B, MN-major ones SWIZZLE_128B_ATOM_32B (UMMA BASE32B).
static CUtensorMap make_map(const float* ptr, int64_t inner, int64_t outer, int64_t ld, int box0, int box1,
                            int mn) {
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  static std::mutex mu;
  MapKey key{ptr, inner, outer, ld, box0, box1, mn};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  auto fn = encode_fn();
  if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, m);
  return m;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// Operand majors: A(m,k) = p[m*si + k*sj]; K-major iff sj == 1.
static bool op_ok(const Operand& o) {
  if (!o.hi || !o.lo) return false;
  if (!aligned16(o.hi) || !aligned16(o.lo)) return false;
  const int64_t ld = o.sj == 1 ? o.si : (o.si == 1 ? o.sj : -1);
  return ld > 0 && (ld % 4) == 0 && (o.sj == 1 || o.si == 1);
}

bool gemm_tc_supported(const GemmArgs& g) {
  if (g.M < 64 || g.N < 8) return false;
  for (int s = 0; s < g.nseg; ++s) {
    if (g.seg[s].K < 8) return false;
    if (!op_ok(g.seg[s].A) || !op_ok(g.seg[s].B)) return false;
  }
  return true;
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
  a.M = g.M;
  a.N = g.N;
  a.nseg = g.nseg;
  a.kb_total = 0;
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
      const float* pa = h ? sg.A.lo : sg.A.hi;
      const float* pb = h ? sg.B.lo : sg.B.hi;
      maps.m[s][h] = akm ? make_map(pa, sg.K, g.M, lda, TC_BK, TC_BM, 0) : make_map(pa, g.M, sg.K, lda, 32, TC_BK, 1);
      maps.m[s][2 + h] = bkm ? make_map(pb, sg.K, g.N, ldb, TC_BK, BN, 0) : make_map(pb, g.N, sg.K, ldb, 32, TC_BK, 1);
    }
  }
  if (g.nseg < 2) a.kb[1] = 0;
  a.epi = g.epi;
  a.skip = g.skip;
  a.lower_only = g.lower_only;
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
  const int work = a.tiles_m * a.tiles_n * splits;
  const int grid = work < ctx->sm_count ? work : ctx->sm_count;
  k_gemm_tc<BN, STAGES><<<grid, Cfg::THREADS, Cfg::SMEM, ctx->stream>>>(maps, a);
  ctx->launches++;
  if (part) {
    k_splitk_reduce<<<4 * ctx->sm_count, 256, 0, ctx->stream>>>(part, splits, g.M, g.N, g.epi, g.skip, g.lower_only);
    ctx->launches++;
    ctx->pool.put(part);  // stream-ordered reuse: later users enqueue after this kernel
  }
  return splits;
}

#include "gemm_tc2.cuh"

void gemm_tc(cv_ctx* ctx, const GemmArgs& g) {
  static const int force_bn = getenv("CURVOPT_TC_BN") ? atoi(getenv("CURVOPT_TC_BN")) : 0;
  static const int use_2sm = getenv("CURVOPT_TC_2SM") ? atoi(getenv("CURVOPT_TC_2SM")) : 1;
  const bool pair = use_2sm && !force_bn && g.M >= 256 && g.N >= 256;
  const bool wide = force_bn ? force_bn == 256 : g.N >= 512;
  const int tiles = pair ? ((g.M + 255) / 256) * ((g.N + 255) / 256) * 2
                         : (wide ? (g.N + 255) / 256 : (g.N + 127) / 128) * ((g.M + TC_BM - 1) / TC_BM);
  int kb_total = 0;
  for (int s = 0; s < g.nseg; ++s) kb_total += (g.seg[s].K + TC_BK - 1) / TC_BK;
  // split K when the tile grid cannot fill the machine (weight-gradient GEMMs: M, N ~ 1e3, K = batch)
  int splits = 1;
  if (g.epi.mode == EPI_STORE && tiles < ctx->sm_count) {
    splits = ctx->sm_count / tiles;
    if (splits > kb_total / 4) splits = kb_total / 4;
    if (splits < 1) splits = 1;
  }
  if (g.N <= 32)
    launch_tc<32, 5>(ctx, g, splits);
  else if (pair)
    launch_tc2<3>(ctx, g, splits);
  else if (wide)
    launch_tc<256, 2>(ctx, g, splits);
  else
    launch_tc<128, 3>(ctx, g, splits);
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
  return launch_tc<32, 5>(ctx, g, splits, *partial);
}

}  // namespace cv
