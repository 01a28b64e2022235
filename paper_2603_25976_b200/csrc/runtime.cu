// Runtime: caching allocator, NCCL (loaded on demand), GEMM engine dispatch.
#include <dlfcn.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <exception>
#include <stdexcept>

#include "common.cuh"
#include "internal.h"
#include "nccl.h"

namespace cv {

// ---------------------------------------------------------------------------
// Pool
// ---------------------------------------------------------------------------
void* Pool::get(size_t bytes) {
  if (redirect_) return redirect_->get(bytes);
  bytes = (bytes + 255) / 256 * 256;
  if (bytes == 0) bytes = 256;
  auto it = free_.find(bytes);
  void* p = nullptr;
  if (it != free_.end()) {
    p = it->second;
    free_.erase(it);
  } else {
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      // drop cached blocks and retry once
      for (auto& kv : free_) cudaFree(kv.second);
      free_.clear();
      if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        throw std::runtime_error("cudaMalloc failed (" + std::to_string(bytes) + " bytes)");
      }
    }
  }
  live_[p] = bytes;
  return p;
}

void Pool::put(void* p) {
  if (!p) return;
  if (redirect_ && redirect_->owns(p)) {
    redirect_->put(p);
    return;
  }
  auto it = live_.find(p);
  if (it == live_.end()) return;
  free_.emplace(it->second, p);
  live_.erase(it);
}

void Pool::release_all() {
  for (auto& kv : free_) cudaFree(kv.second);
  for (auto& kv : live_) cudaFree(kv.first);
  free_.clear();
  live_.clear();
}

// ---------------------------------------------------------------------------
// NCCL, resolved with dlopen so single-GPU use never needs the library.
// ---------------------------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl_api() {
  static NcclApi api;
  if (api.h) return api;
  const char* cands[] = {getenv("CURVOPT_NCCL_LIB"), "libnccl.so.2",
#ifdef CV_NCCL_LIB_PATH
                         CV_NCCL_LIB_PATH,
#endif
                         nullptr};
  for (const char* c : cands) {
    if (!c) continue;
    api.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (api.h) break;
  }
  if (!api.h) throw std::runtime_error("NCCL library not found (set CURVOPT_NCCL_LIB)");
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.h, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.h, "ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.h, "ncclCommDestroy");
  api.AllReduce = (decltype(api.AllReduce))dlsym(api.h, "ncclAllReduce");
  api.Reduce = (decltype(api.Reduce))dlsym(api.h, "ncclReduce");
  api.AllGather = (decltype(api.AllGather))dlsym(api.h, "ncclAllGather");
  api.Broadcast = (decltype(api.Broadcast))dlsym(api.h, "ncclBroadcast");
  api.GroupStart = (decltype(api.GroupStart))dlsym(api.h, "ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))dlsym(api.h, "ncclGroupEnd");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
  if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.Reduce || !api.AllGather ||
      !api.Broadcast || !api.GroupStart || !api.GroupEnd)
    throw std::runtime_error("NCCL library lacks required symbols");
  return api;
}

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    NcclApi& a = nccl_api();
    throw std::runtime_error(std::string("NCCL ") + what + ": " + (a.GetErrorString ? a.GetErrorString(r) : "error"));
  }
}

void nccl_unique_id(void* out) {
  ncclUniqueId id;
  nccl_check(nccl_api().GetUniqueId(&id), "GetUniqueId");
  memcpy(out, &id, sizeof(id));
}

void nccl_init(cv_ctx* ctx, const void* id_bytes) {
  ncclUniqueId id;
  memcpy(&id, id_bytes, sizeof(id));
  ncclComm_t comm;
  nccl_check(nccl_api().CommInitRank(&comm, ctx->world, id, ctx->rank), "CommInitRank");
  ctx->nccl = comm;
}

void nccl_destroy(cv_ctx* ctx) {
  if (ctx->nccl) nccl_api().CommDestroy((ncclComm_t)ctx->nccl);
  ctx->nccl = nullptr;
}

static void comm_call(cv_ctx* ctx, int dtype, void* buf, int64_t n, cudaStream_t st) {
  const int rc = ctx->comm_fn(ctx->comm_user, dtype, buf, n, (void*)st);
  if (rc != 0) throw std::runtime_error("NCCL-substitute communicator failed (rc " + std::to_string(rc) + ")");
}

void allreduce_f32(cv_ctx* ctx, float* buf, int64_t n) {
  if (ctx->comm_fn) return comm_call(ctx, CV_DTYPE_F32, buf, n, ctx->stream);
  if (!ctx->nccl) return;
  nccl_check(nccl_api().AllReduce(buf, buf, (size_t)n, ncclFloat32, ncclSum, (ncclComm_t)ctx->nccl, ctx->stream),
             "AllReduce");
}

void allreduce_f64(cv_ctx* ctx, double* buf, int64_t n) {
  if (ctx->comm_fn) return comm_call(ctx, CV_DTYPE_F64, buf, n, ctx->stream);
  if (!ctx->nccl) return;
  nccl_check(nccl_api().AllReduce(buf, buf, (size_t)n, ncclFloat64, ncclSum, (ncclComm_t)ctx->nccl, ctx->stream),
             "AllReduce");
}

// Sharded CG (vec.cu cg_run_sharded): rank r owns [r*chunk, (r+1)*chunk) of every
// parameter-space vector.  The block [b0, b1) of a summed product is reduced only onto
// the ranks owning parts of it -- one ncclReduce per owner, grouped -- which moves the
// bytes of a reduce-scatter instead of an all-reduce.  The external communicator only
// sums, so there every rank receives the whole sum (same values on the owned range).
void reduce_to_owners(cv_ctx* ctx, float* buf, int64_t b0, int64_t b1, int64_t chunk, cudaStream_t st) {
  if (ctx->comm_fn) return comm_call(ctx, CV_DTYPE_F32, buf + b0, b1 - b0, st);
  if (!ctx->nccl || b1 <= b0) return;
  NcclApi& a = nccl_api();
  nccl_check(a.GroupStart(), "GroupStart");
  for (int r = (int)(b0 / chunk); r < ctx->world && (int64_t)r * chunk < b1; ++r) {
    const int64_t s0 = std::max(b0, (int64_t)r * chunk), s1 = std::min(b1, (int64_t)(r + 1) * chunk);
    if (s1 > s0)
      nccl_check(a.Reduce(buf + s0, buf + s0, (size_t)(s1 - s0), ncclFloat32, ncclSum, r, (ncclComm_t)ctx->nccl, st),
                 "Reduce");
  }
  nccl_check(a.GroupEnd(), "GroupEnd");
}

// buf holds world*chunk floats; rank r's chunk is valid on rank r; afterwards all are
// valid everywhere.  The external communicator does it as a sum with zeros elsewhere.
void allgather_f32(cv_ctx* ctx, float* buf, int64_t chunk) {
  float* mine = buf + (int64_t)ctx->rank * chunk;
  if (ctx->comm_fn) {
    if (ctx->rank > 0) cudaMemsetAsync(buf, 0, sizeof(float) * (size_t)(mine - buf), ctx->stream);
    const int64_t tail = (int64_t)(ctx->world - 1 - ctx->rank) * chunk;
    if (tail > 0) cudaMemsetAsync(mine + chunk, 0, sizeof(float) * (size_t)tail, ctx->stream);
    return comm_call(ctx, CV_DTYPE_F32, buf, (int64_t)ctx->world * chunk, ctx->stream);
  }
  if (!ctx->nccl) return;
  nccl_check(nccl_api().AllGather(mine, buf, (size_t)chunk, ncclFloat32, (ncclComm_t)ctx->nccl, ctx->stream),
             "AllGather");
}

// root's n elements (CV_DTYPE_*) at buf to every rank, in place, on the context stream.
// The external communicator sums: the other ranks contribute zeros.
void broadcast(cv_ctx* ctx, void* buf, int64_t n, int dtype, int root) {
  if (n <= 0) return;
  const size_t es = dtype == CV_DTYPE_F64 ? 8 : 4;
  if (ctx->comm_fn) {
    if (ctx->rank != root) cudaMemsetAsync(buf, 0, es * (size_t)n, ctx->stream);
    return comm_call(ctx, dtype, buf, n, ctx->stream);
  }
  if (!ctx->nccl) return;
  nccl_check(nccl_api().Broadcast(buf, buf, (size_t)n, dtype == CV_DTYPE_F64 ? ncclFloat64 : ncclFloat32, root,
                                  (ncclComm_t)ctx->nccl, ctx->stream),
             "Broadcast");
}
// NCCL calls between these two are issued as one group (no-op for the external communicator)
void comm_group(cv_ctx* ctx, bool begin) {
  if (!ctx->nccl || ctx->comm_fn) return;
  nccl_check(begin ? nccl_api().GroupStart() : nccl_api().GroupEnd(), begin ? "GroupStart" : "GroupEnd");
}

void LayerAllreduce::ready(int l, cudaStream_t st) {
  if (!ctx->nccl || ctx->comm_fn) return;
  if (!ctx->comm) {
    if (cudaStreamCreateWithFlags(&ctx->comm, cudaStreamNonBlocking) != cudaSuccess)
      throw std::runtime_error("CUDA: cannot create the comm stream");
  }
  while ((int)ctx->comm_ev.size() <= pending) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      throw std::runtime_error("CUDA: cannot create a comm event");
    ctx->comm_ev.push_back(e);
  }
  cudaEventRecord(ctx->comm_ev[pending], st);
  cudaStreamWaitEvent(ctx->comm, ctx->comm_ev[pending], 0);
  ++pending;
  const int64_t b0 = (*off)[l], b1 = l + 1 < (int)off->size() ? (*off)[l + 1] : d;
  if (ctx->shard_chunk) return reduce_to_owners(ctx, out, b0, b1, ctx->shard_chunk, ctx->comm);
  nccl_check(nccl_api().AllReduce(out + b0, out + b0, (size_t)(b1 - b0), ncclFloat32, ncclSum,
                                  (ncclComm_t)ctx->nccl, ctx->comm),
             "AllReduce");
}

void LayerAllreduce::finish() {
  if (!distributed(ctx)) return;
  if (ctx->comm_fn || !pending) {  // external communicator (or nothing bucketed): one reduction
    if (ctx->shard_chunk) reduce_to_owners(ctx, out, 0, d, ctx->shard_chunk, ctx->stream);
    else allreduce_f32(ctx, out, d);
    return;
  }
  cudaEvent_t e = ctx->comm_ev[0];
  cudaEventRecord(e, ctx->comm);
  cudaStreamWaitEvent(ctx->stream, e, 0);
  pending = 0;
}

void check_launch(cv_ctx* ctx) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// GEMM engine dispatch: tensor-core (tcgen05, 3xTF32) where the operand
// geometry allows TMA, exact-fp32 SIMT otherwise.
// ---------------------------------------------------------------------------
static void ensure_side(cv_ctx* ctx) {
  if (ctx->side) return;
  if (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess)
    throw std::runtime_error("CUDA: cannot create the side stream");
}

cudaStream_t side_fork(cv_ctx* ctx) {
  ensure_side(ctx);
  cudaEventRecord(ctx->ev_fork, ctx->stream);
  cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
  ctx->side_live = true;
  return ctx->side;
}

cudaStream_t side2_fork(cv_ctx* ctx) {
  if (!ctx->side2) {
    if (cudaStreamCreateWithFlags(&ctx->side2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_fork2, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_join2, cudaEventDisableTiming) != cudaSuccess)
      throw std::runtime_error("CUDA: cannot create the second side stream");
  }
  cudaEventRecord(ctx->ev_fork2, ctx->stream);
  cudaStreamWaitEvent(ctx->side2, ctx->ev_fork2, 0);
  ctx->side2_live = true;
  return ctx->side2;
}

// Joins only the side streams forked since the last join: a join of an idle side stream
// would make a captured graph depend on work outside the capture.
void side_join(cv_ctx* ctx) {
  if (ctx->side2 && ctx->side2_live) {
    cudaEventRecord(ctx->ev_join2, ctx->side2);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_join2, 0);
    ctx->side2_live = false;
  }
  for (void* p : ctx->deferred2) ctx->pool.put(p);
  ctx->deferred2.clear();
  if (ctx->side && ctx->side_live) {
    cudaEventRecord(ctx->ev_join, ctx->side);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0);
    ctx->side_live = false;
  }
  for (void* p : ctx->deferred) ctx->pool.put(p);
  ctx->deferred.clear();
}

StreamSwap::StreamSwap(cv_ctx* ctx, cudaStream_t s) : c(ctx), prev(ctx->stream), exc(std::uncaught_exceptions()) {
  ctx->stream = s;
}

StreamSwap::~StreamSwap() {
  c->stream = prev;
  if (std::uncaught_exceptions() > exc) {
    try {
      side_join(c);
    } catch (...) {
    }
  }
}

cudaStream_t gemm_pair(cv_ctx* ctx, GemmArgs a, GemmArgs b) {
  const bool tc = ctx->engine != CV_ENGINE_SIMT && gemm_tc_supported(a) && gemm_tc_supported(b);
  if (!tc) {
    gemm(ctx, a);
    gemm(ctx, b);
    return ctx->stream;
  }
  ensure_side(ctx);
  // SM split minimising the slower of the two (even counts: CTA pairs)
  const int sms = ctx->sm_count;
  int best = sms / 2;
  double best_t = 1e300;
  for (int ca = 16; ca <= sms - 16; ca += 2) {
    const double ta = gemm_tc_estimate(ctx, a, ca), tb = gemm_tc_estimate(ctx, b, sms - ca);
    const double t = ta > tb ? ta : tb;
    if (t < best_t) {
      best_t = t;
      best = ca;
    }
  }
  a.max_ctas = best;
  b.max_ctas = sms - best;
  a.stream = ctx->stream;
  b.stream = ctx->side;
  cudaEventRecord(ctx->ev_fork, ctx->stream);
  cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
  gemm(ctx, b);
  gemm(ctx, a);
  cudaEventRecord(ctx->ev_join, ctx->side);
  cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0);
  for (void* p : ctx->deferred) ctx->pool.put(p);  // later users are ordered after the join
  ctx->deferred.clear();
  ctx->side_live = false;
  return ctx->side;
}

void gemm(cv_ctx* ctx, const GemmArgs& a) {
  if (ctx->engine != CV_ENGINE_SIMT && gemm_tc_supported(a)) {
    gemm_tc(ctx, a);
    return;
  }
  gemm_simt(ctx, a);
}

}  // namespace cv
