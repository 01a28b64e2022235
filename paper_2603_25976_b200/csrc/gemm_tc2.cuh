// 2-CTA (cta_group::2) variant of the 3xFP16 engine, included by gemm_tc.cu.
//
// A cluster of two CTAs on one TPC computes a 256 x 256 tile with M=256 UMMAs
// issued by the leader CTA only: each CTA stages its own 128 rows of A and its
// own 128 columns of B (so every SM moves half the B bytes of the 1-CTA kernel,
// 64 KB per 64-deep K slab), and each CTA's TMEM receives its 128 accumulator
// rows.  Both CTAs' TMA transfers complete on the leader's "full" barrier; the
// leader's tcgen05.commit multicasts "empty"/"tfull" to both CTAs; both CTAs'
// epilogue warps release the accumulator on the leader's "tempty" barrier.
// Persistent over work items, TMEM double buffered (2 x 256 columns).

// TC2_BN = tile width of the pair: 256 (each CTA stages 128 B columns) or 128 (64).
template <int STAGES, int TC2_BN>
struct Tc2Cfg {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;         // 16 KB: this CTA's 128 rows
  static constexpr int B_BYTES = (TC2_BN / 2) * TC_BK * 2;  // 16 / 8 KB: this CTA's 128 / 64 columns
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + TC_ZERO_BYTES + TC_STG_TOTAL + 1024 + 256;
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

CV_DEV void load_slab_2sm(uint8_t* dst, const CUtensorMap* map, uint32_t bar, bool kmajor, int k0, int r0, int rows) {
  if (kmajor) {
    tma_load_2d_2sm(dst, map, bar, k0, r0);
  } else {
    for (int j = 0; j < rows / 64; ++j) tma_load_2d_2sm(dst + j * 8192, map, bar, r0 + 64 * j, k0);
  }
}

// Work item i of this cluster: round robin over the GEMM's items.
CV_DEV bool tc2_item(const TcArgs& a, int cluster, int nclusters, int i, int& w) {
  w = cluster + i * nclusters;
  return w < a.tiles_m * a.tiles_n * a.splits;
}

template <int STAGES, int TC2_BN>
CV_DEV void tc2_body(const TcMaps& mp, const TcArgs& a) {
  using Cfg = Tc2Cfg<STAGES, TC2_BN>;
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
  const uint32_t rank = cluster_ctarank();
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  zero_tile_init(zero);
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
        for (int q = 0; q < 4; ++q) tma_prefetch(&mp.m[sg][q]);
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
  // the setup above touches no data of earlier kernels: it overlaps the predecessor's tail
  CV_PDL_ENTRY();
  const bool skipped = skip_if(a.skip);  // identical for both CTAs
  const SegPlan plan = skipped ? SegPlan{} : seg_plan(a);

  if (skipped) {
  } else if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    int it = 0, w;
    for (int item = 0; tc2_item(a, cluster, nclusters, item, w); ++item) {
      int mt0, n0, kb0, nkb;
      if (!tc_work(a, w, 2 * TC_BM, TC2_BN, mt0, n0, kb0, nkb)) continue;
      const int m0 = mt0 + rank * TC_BM;         // this CTA's A rows
      const int nb0 = n0 + rank * (TC2_BN / 2);  // this CTA's B columns
      for (int i = 0; i < nkb; ++i, ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
        int lkb;
        const int sg = vseg(a, plan, kb0 + i, lkb);
        const int k0 = lkb * TC_BK;
        uint8_t* st = smem + s * Cfg::STAGE_BYTES;
        if (rank == 0) mbar_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
        const uint32_t bar = mapa_rank(&full[s], 0);
        for (int h = 0; h < 2; ++h) {
          load_slab_2sm(st + h * Cfg::A_BYTES, &mp.m[sg][h], bar, a.a[sg].kmajor, k0, m0, TC_BM);
          load_slab_2sm(st + 2 * Cfg::A_BYTES + h * Cfg::B_BYTES, &mp.m[sg][2 + h], bar, a.b[sg].kmajor, k0, nb0,
                        TC2_BN / 2);
        }
      }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    // ---------------- MMA issuer (leader CTA) ----------------
    int it = 0, acc_i = 0, w;
    const uint64_t zdesc = zero_desc(zero);
    for (int item = 0; tc2_item(a, cluster, nclusters, item, w); ++item) {
      int mt0, n0, kb0, nkb;
      if (!tc_work(a, w, 2 * TC_BM, TC2_BN, mt0, n0, kb0, nkb)) continue;
      const int ab = acc_i & 1;
      if (acc_i >= 2) mbar_wait(&tempty[ab], ((acc_i >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dtm = tmem + ab * TC2_BN;
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
        const uint32_t idesc = f16_idesc(2 * TC_BM, TC2_BN, amn, bmn);
        const uint32_t st = smem_u32(smem + s * Cfg::STAGE_BYTES);
        const uint32_t a_hi = st, a_lo = st + Cfg::A_BYTES;
        const uint32_t b_hi = st + 2 * Cfg::A_BYTES, b_lo = b_hi + Cfg::B_BYTES;
#pragma unroll
        for (int kk = 0; kk < TC_BK / 16; ++kk)
          umma_kstep<2>(dtm, op_desc(a_hi, amn, kk), op_desc(a_lo, amn, kk), op_desc(b_hi, bmn, kk),
                        op_desc(b_lo, bmn, kk), zdesc, idesc, i > 0 || kk > 0, kk == 0 ? shift : 0);
        umma_commit<2>(&empty[s]);  // both CTAs' slab s is free once these MMAs retire
      }
      umma_commit<2>(&tfull[ab]);   // both CTAs' accumulator halves are ready
      ++acc_i;
    }
  } else if (warp >= 2) {
    // ---------------- epilogue (both CTAs) ----------------
    const int q = warp & 3, half = (warp - 2) >> 2;
    const uint32_t tempty0[2] = {mapa_rank(&tempty[0], 0), mapa_rank(&tempty[1], 0)};
    const EpiRt rt = epi_prepare(a.epi);
    if (blockIdx.x == 0 && warp == 2 && lane == 0 && !a.partial) epi_publish(a.epi, rt);
    int acc_i = 0, w;
    for (int item = 0; tc2_item(a, cluster, nclusters, item, w); ++item) {
      int mt0, n0, kb0, nkb;
      if (!tc_work(a, w, 2 * TC_BM, TC2_BN, mt0, n0, kb0, nkb)) continue;
      const int ab = acc_i & 1;
      epi_prefetch_mask<TC2_BN>(a, mt0 + rank * TC_BM, n0, q, half, lane);
      mbar_wait(&tfull[ab], (acc_i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      int lkb;
      const int last = vseg(a, plan, kb0 + nkb - 1, lkb);
      const float inv = plan.inv_a[last] * plan.inv_b[last];
      tile_epilogue<TC2_BN>(a, mp, rt, tmem + ab * TC2_BN, mt0 + rank * TC_BM, n0,
                            w / (a.tiles_m * a.tiles_n), inv, q, half, lane, stg_all + (warp - 2) * TC_STG_BYTES,
                            stg_all + 8 * TC_STG_BYTES + (warp - 2) * TC_HSTG_BYTES);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(tempty0[ab]);
      ++acc_i;
    }
    if (lane == 0) bulk_wait0();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::TMEM_COLS));
  }
}

template <int STAGES, int TC2_BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
    k_gemm_tc2(const __grid_constant__ TcMaps maps, const __grid_constant__ TcArgs a) {
  tc2_body<STAGES, TC2_BN>(maps, a);
}

template <int STAGES, int TC2_BN>
static void launch_tc2(cv_ctx* ctx, const GemmArgs& g, int splits) {
  using Cfg = Tc2Cfg<STAGES, TC2_BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_gemm_tc2<STAGES, TC2_BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr_set = true;
  }
  TcMaps maps;
  TcArgs a{};
  fill_args(g, TC2_BN / 2, maps, a);
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
  setup_out(g, maps, a, a.partial, splits);
  if (g.epi.head_part && a.tma_out != 1 && !part)
    throw std::runtime_error("fused output head needs the TMA split epilogue");
  const int work = a.tiles_m * a.tiles_n * splits;
  const int sms = g.max_ctas > 0 && g.max_ctas < ctx->sm_count ? g.max_ctas : ctx->sm_count;
  const int pairs = sms / 2;
  const int grid = 2 * (work < pairs ? work : pairs);
  cudaStream_t st = g.stream ? g.stream : ctx->stream;
  launch_k(st, k_gemm_tc2<STAGES, TC2_BN>, grid, 320, Cfg::SMEM, maps, a);
  ctx->launches++;
  if (splits > 1) {
    if (g.epi.head_part)
      launch_k(st, k_splitk_reduce_head, 4 * ctx->sm_count, 256, 0, (const float*)part, splits, g.M, g.N, g.epi,
               g.skip);
    else
      launch_k(st, k_splitk_reduce, 4 * ctx->sm_count, 256, 0, part, splits, g.M, g.N, g.epi, g.skip, g.lower_only);
    ctx->launches++;
    if (st == ctx->side2 && st) ctx->deferred2.push_back(part);
    else if (st != ctx->stream) ctx->deferred.push_back(part);  // reused only after the join
    else ctx->pool.put(part);
  }
}
