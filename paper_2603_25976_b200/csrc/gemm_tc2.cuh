// 2-CTA (cta_group::2) variant of the 3xTF32 engine, included by gemm_tc.cu.
//
// A cluster of two CTAs on one TPC computes a 256 x 256 tile with M=256 UMMAs
// issued by the leader CTA only: each CTA stages its own 128 rows of A and its
// own 128 columns of B (so every SM moves half the B bytes of the 1-CTA kernel,
// 64 KB per 32-deep K slab instead of 96 KB), and each CTA's TMEM receives its
// 128 accumulator rows.  Both CTAs' TMA transfers complete on the leader's
// "full" barrier; the leader's tcgen05.commit multicasts "empty"/"tfull" to both
// CTAs; both CTAs' epilogue warps release the accumulator on the leader's
// "tempty" barrier.  Persistent over work items, TMEM double buffered (2 x 256).

constexpr int TC2_BN = 256;

template <int STAGES>
struct Tc2Cfg {
  static constexpr int A_BYTES = TC_BM * TC_BK * 4;         // 16 KB: this CTA's 128 rows
  static constexpr int B_BYTES = (TC2_BN / 2) * TC_BK * 4;  // 16 KB: this CTA's 128 columns
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr int TMEM_COLS = 2 * TC2_BN;
};

CV_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

CV_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cluster address of the same smem object in CTA `rank` of this cluster
CV_DEV uint32_t mapa_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

CV_DEV void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

CV_DEV void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}

CV_DEV void umma_tf32_2sm(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

CV_DEV void umma_commit_2sm(uint64_t* bar) {
  const uint16_t mask = 3;
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

CV_DEV bool tc2_work(const TcArgs& a, int w, int& mt0, int& n0, int& kb0, int& nkb) {
  const int tiles = a.tiles_m * a.tiles_n;
  const int split = w / tiles, t = w % tiles;
  mt0 = (t / a.tiles_n) * 2 * TC_BM;
  n0 = (t % a.tiles_n) * TC2_BN;
  kb0 = split * a.kb_per_split;
  nkb = min(a.kb_total, kb0 + a.kb_per_split) - kb0;
  return !(a.lower_only && n0 > mt0 + 2 * TC_BM - 1);
}

template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
    k_gemm_tc2(const __grid_constant__ TcMaps maps, const TcArgs a) {
  using Cfg = Tc2Cfg<STAGES>;
  if (skip_if(a.skip)) return;  // the flag is identical for both CTAs of the pair
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int total = a.tiles_m * a.tiles_n * a.splits;
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&tfull[b], 1);
        mbar_init(&tempty[b], 16);  // 8 epilogue warps x 2 CTAs
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int sg = 0; sg < a.nseg; ++sg)
        for (int q = 0; q < 4; ++q) tma_prefetch(&maps.m[sg][q]);
    }
  } else if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    int it = 0;
    for (int w = cluster; w < total; w += nclusters) {
      int mt0, n0, kb0, nkb;
      if (!tc2_work(a, w, mt0, n0, kb0, nkb)) continue;
      const int m0 = mt0 + rank * TC_BM;           // this CTA's A rows
      const int nb0 = n0 + rank * (TC2_BN / 2);    // this CTA's B columns
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
        const int kb = kb0 + i;
        const int sg = kb < a.kb[0] ? 0 : 1;
        const int k0 = (sg == 0 ? kb : kb - a.kb[0]) * TC_BK;
        uint8_t* st = smem + s * Cfg::STAGE_BYTES;
        if (rank == 0) mbar_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
        const uint32_t bar = mapa_rank(&full[s], 0);
        for (int h = 0; h < 2; ++h) {
          uint8_t* sa = st + h * Cfg::A_BYTES;
          if (a.a[sg].kmajor) {
            tma_load_2d_2sm(sa, &maps.m[sg][h], bar, k0, m0);
          } else {
#pragma unroll
            for (int j = 0; j < TC_BM / 32; ++j) tma_load_2d_2sm(sa + j * 4096, &maps.m[sg][h], bar, m0 + 32 * j, k0);
          }
          uint8_t* sb = st + 2 * Cfg::A_BYTES + h * Cfg::B_BYTES;
          if (a.b[sg].kmajor) {
            tma_load_2d_2sm(sb, &maps.m[sg][2 + h], bar, k0, nb0);
          } else {
#pragma unroll
            for (int j = 0; j < TC2_BN / 64; ++j)
              tma_load_2d_2sm(sb + j * 4096, &maps.m[sg][2 + h], bar, nb0 + 32 * j, k0);
          }
        }
      }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    // ---------------- MMA issuer (leader CTA) ----------------
    int it = 0, acc_i = 0;
    for (int w = cluster; w < total; w += nclusters) {
      int mt0, n0, kb0, nkb;
      if (!tc2_work(a, w, mt0, n0, kb0, nkb)) continue;
      const int ab = acc_i & 1;
      if (acc_i >= 2) mbar_wait(&tempty[ab], ((acc_i >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dtm = tmem + ab * TC2_BN;
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int kb = kb0 + i;
        const int sg = kb < a.kb[0] ? 0 : 1;
        const int amn = a.a[sg].kmajor ? 0 : 1, bmn = a.b[sg].kmajor ? 0 : 1;
        const uint32_t idesc = tf32_idesc(2 * TC_BM, TC2_BN, amn, bmn);
        const uint32_t st = smem_u32(smem + s * Cfg::STAGE_BYTES);
        const uint32_t a_hi = st, a_lo = st + Cfg::A_BYTES;
        const uint32_t b_hi = st + 2 * Cfg::A_BYTES, b_lo = b_hi + Cfg::B_BYTES;
#pragma unroll
        for (int kk = 0; kk < TC_BK / 8; ++kk) {
          const uint32_t aoff = amn ? kk * 1024 : kk * 32;
          const uint32_t boff = bmn ? kk * 1024 : kk * 32;
          const uint32_t albo = amn ? 4096 : 16, blbo = bmn ? 4096 : 16;
          const uint32_t asbo = amn ? 512 : 1024, bsbo = bmn ? 512 : 1024;
          const uint32_t alay = amn ? 1 : 2, blay = bmn ? 1 : 2;
          const uint64_t dah = umma_desc(a_hi + aoff, albo, asbo, alay), dal = umma_desc(a_lo + aoff, albo, asbo, alay);
          const uint64_t dbh = umma_desc(b_hi + boff, blbo, bsbo, blay), dbl = umma_desc(b_lo + boff, blbo, bsbo, blay);
          const uint32_t acc0 = (i > 0 || kk > 0) ? 1u : 0u;
          umma_tf32_2sm(dtm, dah, dbh, idesc, acc0);
          umma_tf32_2sm(dtm, dah, dbl, idesc, 1u);
          umma_tf32_2sm(dtm, dal, dbh, idesc, 1u);
        }
        umma_commit_2sm(&empty[s]);  // both CTAs' slab s is free once these MMAs retire
      }
      umma_commit_2sm(&tfull[ab]);   // both CTAs' accumulator halves are ready
      ++acc_i;
    }
  } else if (warp >= 2) {
    // ---------------- epilogue (both CTAs) ----------------
    const int q = warp & 3, half = (warp - 2) >> 2;
    const uint32_t tempty0[2] = {mapa_rank(&tempty[0], 0), mapa_rank(&tempty[1], 0)};
    int acc_i = 0;
    for (int w = cluster; w < total; w += nclusters) {
      int mt0, n0, kb0, nkb;
      if (!tc2_work(a, w, mt0, n0, kb0, nkb)) continue;
      const int ab = acc_i & 1;
      mbar_wait(&tfull[ab], (acc_i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int m = mt0 + rank * TC_BM + q * 32 + lane;
      const int split = w / (a.tiles_m * a.tiles_n);
      const uint32_t trow = tmem + ab * TC2_BN + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c = half * (TC2_BN / 64); c < (half + 1) * (TC2_BN / 64); ++c) {
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
      if (lane == 0) mbar_arrive_remote(tempty0[ab]);
      ++acc_i;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::TMEM_COLS));
  }
}

template <int STAGES>
static void launch_tc2(cv_ctx* ctx, const GemmArgs& g, int splits) {
  using Cfg = Tc2Cfg<STAGES>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_gemm_tc2<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
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
    const bool akm = sg.A.sj == 1, bkm = sg.B.si == 1;
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
      maps.m[s][2 + h] = bkm ? make_map(pb, sg.K, g.N, ldb, TC_BK, TC2_BN / 2, 0)
                             : make_map(pb, g.N, sg.K, ldb, 32, TC_BK, 1);
    }
  }
  if (g.nseg < 2) a.kb[1] = 0;
  a.epi = g.epi;
  a.skip = g.skip;
  a.lower_only = g.lower_only;
  a.kb_per_split = (a.kb_total + splits - 1) / splits;
  splits = (a.kb_total + a.kb_per_split - 1) / a.kb_per_split;
  a.splits = splits;
  a.tiles_m = (g.M + 2 * TC_BM - 1) / (2 * TC_BM);
  a.tiles_n = (g.N + TC2_BN - 1) / TC2_BN;
  float* part = nullptr;
  if (splits > 1) {
    part = (float*)ctx->pool.get(sizeof(float) * (size_t)splits * g.M * g.N);
    a.partial = part;
  }
  const int work = a.tiles_m * a.tiles_n * splits;
  const int pairs = ctx->sm_count / 2;
  const int grid = 2 * (work < pairs ? work : pairs);
  k_gemm_tc2<STAGES><<<grid, 320, Cfg::SMEM, ctx->stream>>>(maps, a);
  ctx->launches++;
  if (splits > 1) {
    k_splitk_reduce<<<4 * ctx->sm_count, 256, 0, ctx->stream>>>(part, splits, g.M, g.N, g.epi, g.skip, g.lower_only);
    ctx->launches++;
    ctx->pool.put(part);
  }
}
