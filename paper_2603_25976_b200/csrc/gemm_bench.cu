// Diagnostic entry point: time one tensor-core GEMM shape in isolation (CUDA
// events, operands resident), for tuning the engine.  Not on any product path.
#include <stdexcept>

#include "common.cuh"
#include "internal.h"

namespace cv {
extern int g_force_kind, g_force_splits;

__global__ void k_fill_split(__half* hi, __half* lo, int64_t n, uint32_t seed) {
  CV_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    const float x = ((float)(h & 0xFFFF) / 32768.f - 1.f) * 1024.f;
    split16(x, 1.f, hi[i], lo[i]);
  }
}

__global__ void k_set_scale(Scale* sc, int n, float amax) {
  CV_PDL_ENTRY();
  if (threadIdx.x < n) {
    sc[threadIdx.x].e = 0;
    sc[threadIdx.x].amax = amax;
  }
}

}  // namespace cv

using namespace cv;

extern "C" __attribute__((visibility("default"))) int cv_gemm_bench(cv_ctx* ctx, int M, int N, int K, int a_kmajor,
                                                                   int b_kmajor, int mode, int iters, float* ms_out) {
  if (!ctx || M <= 0 || N <= 0 || K <= 0 || iters <= 0 || !ms_out) return CV_E_CONTRACT;
  try {
    cudaSetDevice(ctx->device);
    const int64_t lda = a_kmajor ? (K + 7) / 8 * 8 : (M + 7) / 8 * 8;
    const int64_t ldb = b_kmajor ? (K + 7) / 8 * 8 : (N + 7) / 8 * 8;
    const int64_t na = (a_kmajor ? (int64_t)M : K) * lda, nb = (b_kmajor ? (int64_t)N : K) * ldb;
    const int64_t ldo = (N + 7) / 8 * 8;
    const int64_t no = (int64_t)M * ldo;
    __half* buf = (__half*)ctx->pool.get(sizeof(__half) * (size_t)(2 * na + 2 * nb + 4 * no));
    float* outf = (float*)ctx->pool.get(sizeof(float) * (size_t)no);
    Scale* sc = (Scale*)ctx->pool.get(sizeof(Scale) * 4);
    __half *ahi = buf, *alo = ahi + na, *bhi = alo + na, *blo = bhi + nb, *mhi = blo + nb, *mlo = mhi + no,
           *ohi = mlo + no, *olo = ohi + no;
    launch_k(ctx->stream, k_fill_split, 1024, 256, 0, ahi, alo, na, 1u);
    launch_k(ctx->stream, k_fill_split, 1024, 256, 0, bhi, blo, nb, 2u);
    launch_k(ctx->stream, k_fill_split, 1024, 256, 0, mhi, mlo, no, 3u);
    launch_k(ctx->stream, k_set_scale, 1, 32, 0, sc, 4, 1024.f);
    GemmArgs g;
    g.M = M;
    g.N = N;
    g.nseg = 1;
    Operand A, B;
    A.hi = ahi; A.lo = alo; A.sc = sc;
    B.hi = bhi; B.lo = blo; B.sc = sc + 1;
    if (a_kmajor) { A.si = lda; A.sj = 1; } else { A.si = 1; A.sj = lda; }
    if (b_kmajor) { B.si = 1; B.sj = ldb; } else { B.si = ldb; B.sj = 1; }
    g.seg[0].A = A;
    g.seg[0].B = B;
    g.seg[0].K = K;
    // mode: bits 0-7 epilogue (0 store, 1 split+mask); bits 8-15 forced tile kind + 1
    // (0: the planner's choice); bits 16-23 forced split-K factor (0: the kind's default)
    const int fkind = ((mode >> 8) & 0xff) - 1, fsplit = (mode >> 16) & 0xff;
    mode &= 0xff;
    if (mode == 1) {
      g.epi.mode = EPI_SPLIT_MASK;
      g.epi.act = CV_ACT_RELU;
      g.epi.out_hi = ohi;
      g.epi.out_lo = olo;
      g.epi.out_sc = sc + 3;
      g.epi.ld = ldo;
      g.epi.mask_hi = mhi;
      g.epi.mask_lo = mlo;
      g.epi.mask_sc = sc + 2;
      g.epi.mask_ld = ldo;
      g.epi.bound.n = 1;
      g.epi.bound.k[0] = (float)K;
      g.epi.bound.x[0] = &sc[0].amax;
      g.epi.bound.y[0] = &sc[1].amax;
    } else {
      g.epi.mode = EPI_STORE;
      g.epi.out = outf;
      g.epi.ld = ldo;
    }
    if (!gemm_tc_supported(g)) throw std::runtime_error("unsupported shape");
    g_force_kind = fkind;
    g_force_splits = fsplit;
    struct Reset {
      ~Reset() { g_force_kind = -1; g_force_splits = 0; }
    } reset;
    gemm_tc(ctx, g);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, ctx->stream);
    for (int i = 0; i < iters; ++i) gemm_tc(ctx, g);
    cudaEventRecord(e1, ctx->stream);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *ms_out = ms / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    ctx->pool.put(sc);
    ctx->pool.put(outf);
    ctx->pool.put(buf);
    check_launch(ctx);
    return CV_OK;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return CV_E_CUDA;
  }
}

namespace cv {
__global__ void k_scale_copy(const float* x, float s, int64_t n, float* y) {
  CV_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] * s;
}
}  // namespace cv

// Diagnostic/test: two-segment tensor-core GEMM out = A.B + A.(s2 B) (A M x K, B N x K,
// both K-major, fp32 in) -- the two segments carry exponents that differ by
// ~log2(s2), exercising the accumulator rescaling between segments.
extern "C" __attribute__((visibility("default"))) int cv_gemm_test_seg2(cv_ctx* ctx, int M, int N, int K,
                                                                       const float* a, const float* b, float s2,
                                                                       float* out) {
  if (!ctx || M <= 0 || N <= 0 || K <= 0 || (K & 7)) return CV_E_CONTRACT;
  try {
    cudaSetDevice(ctx->device);
    const int64_t na = (int64_t)M * K, nb = (int64_t)N * K;
    __half* buf = (__half*)ctx->pool.get(sizeof(__half) * (size_t)(2 * na + 4 * nb));
    float* b2 = (float*)ctx->pool.get(sizeof(float) * (size_t)nb);
    Scale* sc = (Scale*)ctx->pool.get(sizeof(Scale) * 3);
    __half *ahi = buf, *alo = ahi + na, *bhi = alo + na, *blo = bhi + nb, *b2hi = blo + nb, *b2lo = b2hi + nb;
    launch_k(ctx->stream, k_scale_copy, 1024, 256, 0, b, s2, nb, b2);
    split_mat(ctx, a, K, M, K, ahi, alo, K, 0, sc, 0, nullptr);
    split_mat(ctx, b, K, N, K, bhi, blo, K, 0, sc + 1, 0, nullptr);
    split_mat(ctx, b2, K, N, K, b2hi, b2lo, K, 0, sc + 2, 0, nullptr);
    GemmArgs g;
    g.M = M;
    g.N = N;
    g.nseg = 2;
    for (int s = 0; s < 2; ++s) {
      Operand A, B;
      A.hi = ahi; A.lo = alo; A.sc = sc; A.si = K; A.sj = 1;
      B.hi = s ? b2hi : bhi; B.lo = s ? b2lo : blo; B.sc = sc + 1 + s; B.si = 1; B.sj = K;
      g.seg[s].A = A;
      g.seg[s].B = B;
      g.seg[s].K = K;
    }
    g.epi.mode = EPI_STORE;
    g.epi.out = out;
    g.epi.ld = N;
    if (!gemm_tc_supported(g)) throw std::runtime_error("unsupported shape");
    gemm_tc(ctx, g);
    ctx->pool.put(sc);
    ctx->pool.put(b2);
    ctx->pool.put(buf);
    check_launch(ctx);
    return CV_OK;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return CV_E_CUDA;
  }
}
