// Per-rank runtime behind the osh_ctx_* / osh_step C ABI (see runtime.cuh).
#include "runtime.cuh"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "status.hpp"

using namespace optishard;

namespace {

constexpr int64_t kOwnedAlign = 64;  // elements (256 B for fp32)

#define OSH_NCCL_TRY(expr)                                                                     \
  do {                                                                                         \
    ncclResult_t r_ = (expr);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      return osh::fail(OSH_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_));     \
  } while (0)

__global__ void cast_f32_bf16_kernel(const float* src, __nv_bfloat16* dst, long long n) {
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Counter-based N(0,1) * scale for element `idx` of stream `seed`.
__device__ __forceinline__ float synth_normal(uint64_t seed, uint64_t idx) {
  const uint64_t r = mix64(seed ^ mix64(idx));
  const float u1 = (static_cast<float>(r >> 40) + 1.0f) * (1.0f / 16777216.0f);
  const float u2 = static_cast<float>((r >> 16) & 0xFFFFFF) * (1.0f / 16777216.0f);
  return sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
}

// Fills [n] elements starting at flat element `base` of the model.
__global__ void fill_synth_kernel(uint64_t seed, long long base, long long n, float scale,
                                  float* f32, __nv_bfloat16* bf16) {
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x) {
    const float v = scale * synth_normal(seed, static_cast<uint64_t>(base + i));
    if (f32 != nullptr) f32[i] = v;
    if (bf16 != nullptr) bf16[i] = __float2bfloat16_rn(v);
  }
}

unsigned grid_for(long long n) {
  return static_cast<unsigned>(std::min<long long>((n + 255) / 256, 148ll * 16));
}

size_t grad_esize(int dtype) { return dtype == osh::kGradBF16 ? 2 : 4; }

osh_status check_ctx(osh_ctx* ctx, bool need_layout) {
  if (ctx == nullptr) return osh::fail(OSH_ERR_ARG, "null osh_ctx");
  if (need_layout && !ctx->layout_ready)
    return osh::fail(OSH_ERR_PLAN, "osh_ctx_set_layout has not been called");
  if (cudaSetDevice(ctx->device) != cudaSuccess)
    return osh::fail(OSH_ERR_CUDA, "cudaSetDevice failed");
  return OSH_OK;
}

bool distributed(const osh_ctx* ctx) {
  return ctx->comm_mode == OSH_COMM_NCCL && ctx->size > 1 && ctx->comm != nullptr;
}

void destroy_events(std::vector<cudaEvent_t>& v) {
  for (cudaEvent_t e : v) cudaEventDestroy(e);
  v.clear();
}

cudaError_t make_events(std::vector<cudaEvent_t>& v, size_t n) {
  v.assign(n, nullptr);
  for (cudaEvent_t& e : v) {
    const cudaError_t err = cudaEventCreate(&e);
    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

bool is_tp_item(const osh_ctx* ctx, size_t p) {
  if (ctx->tp_size <= 1) return false;
  const ParamSpec& f = ctx->params_full[p];
  return f.tp_splittable != TpSplit::kNone && !f.vocab_space;
}

void free_layout(osh_ctx* ctx) {
  osh::tp_free(ctx);
  ctx->engine.reset();
  destroy_events(ctx->rs_ev);
  destroy_events(ctx->wave_begin);
  destroy_events(ctx->wave_end);
  destroy_events(ctx->pre_ev);
  destroy_events(ctx->ns_ev);
  destroy_events(ctx->h2d_ev);
  destroy_events(ctx->h2d_wave_ev);
  destroy_events(ctx->ag_ev);
  if (ctx->nvls) {
    osh::nvls_free(ctx);
  } else {
    cudaFree(ctx->grad);
    cudaFree(ctx->replica);
  }
  cudaFree(ctx->grad_owned);
  ctx->grad_owned = nullptr;
  cudaFree(ctx->bar);
  ctx->bar = nullptr;
  cudaFree(ctx->w);
  cudaFree(ctx->m);
  ctx->grad = nullptr;
  ctx->replica = nullptr;
  ctx->w = ctx->m = nullptr;
  ctx->layout_ready = false;
}

}  // namespace

namespace osh {

osh_status abort_comms(osh_ctx* ctx, const std::string& why) {
  if (ctx->comm != nullptr) ncclCommAbort(ctx->comm);
  if (ctx->tp_comm != nullptr) ncclCommAbort(ctx->tp_comm);
  ctx->comm = nullptr;
  ctx->tp_comm = nullptr;
  ctx->aborted = true;
  return fail(OSH_ERR_NCCL, why + " (communicators aborted; destroy this ctx)");
}

osh_status wait_stream(osh_ctx* ctx, cudaStream_t stream) {
  if (ctx->comm == nullptr && ctx->tp_comm == nullptr) {
    OSH_CUDA_TRY(cudaStreamSynchronize(stream));
    return OSH_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (int polls = 0;; ++polls) {
    const cudaError_t q = cudaStreamQuery(stream);
    if (q == cudaSuccess) return OSH_OK;
    if (q != cudaErrorNotReady)
      return fail(OSH_ERR_CUDA, std::string("stream wait: ") + cudaGetErrorString(q));
    for (ncclComm_t c : {ctx->comm, ctx->tp_comm}) {
      if (c == nullptr) continue;
      ncclResult_t ae = ncclSuccess;
      if (ncclCommGetAsyncError(c, &ae) != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress))
        return abort_comms(ctx, std::string("NCCL async error: ") + ncclGetErrorString(ae));
    }
    const double waited =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (waited > ctx->timeout_s)
      return abort_comms(ctx, "collective did not complete within " + std::to_string(ctx->timeout_s) +
                                  " s (a peer rank stalled or died)");
    if (polls > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

cudaError_t cast_to_bf16(const float* src, __nv_bfloat16* dst, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  cast_f32_bf16_kernel<<<grid_for(n), 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

// Issues ops [begin, end) of the ctx's collective schedule on `st`; ops of
// one group id go inside one ncclGroupStart / ncclGroupEnd.
osh_status issue_ops(osh_ctx* ctx, int begin, int end, cudaStream_t st) {
  const ncclDataType_t gtype = ctx->grad_dtype == OSH_GRAD_BF16 ? ncclBfloat16 : ncclFloat32;
  const size_t es = grad_esize(ctx->grad_dtype);
  int open_group = -1;
  for (int i = begin; i < end; ++i) {
    const osh_coll_op& o = ctx->sched[static_cast<size_t>(i)];
    if (o.group != open_group) {
      if (open_group >= 0) OSH_NCCL_TRY(ncclGroupEnd());
      OSH_NCCL_TRY(ncclGroupStart());
      open_group = o.group;
    }
    const size_t cnt = static_cast<size_t>(o.count);
    if (o.kind == OSH_OP_REDUCE) {
      const uint8_t* src = static_cast<const uint8_t*>(ctx->grad) + es * static_cast<size_t>(o.offset);
      uint8_t* dst = o.root == ctx->rank
                         ? static_cast<uint8_t*>(ctx->grad_owned) + es * static_cast<size_t>(o.dst_offset)
                         : nullptr;
      OSH_NCCL_TRY(ncclReduce(src, dst, cnt, gtype, ncclSum, o.root, ctx->comm, st));
    } else if (o.kind == OSH_OP_BROADCAST) {
      __nv_bfloat16* ptr = ctx->replica + o.offset;
      OSH_NCCL_TRY(ncclBroadcast(ptr, ptr, cnt, ncclBfloat16, o.root, ctx->comm, st));
    } else {
      uint8_t* base = static_cast<uint8_t*>(ctx->grad) + es * static_cast<size_t>(o.offset);
      OSH_NCCL_TRY(ncclAllReduce(base, base, cnt, gtype, ncclSum, ctx->comm, st));
    }
  }
  if (open_group >= 0) OSH_NCCL_TRY(ncclGroupEnd());
  return OSH_OK;
}

// The bf16 replica from the owners' fp32 masters (checkpoint resume): every
// rank casts the tensors it owns into its replica slots; with TP the hosts
// cast their full masters and scatter each rank its shard (the step's
// pack + scatter path); then the AG-v leg of the schedule broadcasts each
// slice from its owner (the plan's cut owners, or the layer owners under
// NV-layerwise).
osh_status refresh_replica(osh_ctx* ctx) {
  cudaStream_t cs = ctx->compute;
  for (size_t p = 0; p < ctx->params.size(); ++p) {
    if (ctx->owned_off[p] < 0) continue;
    const long long n = ctx->params[p].numel;
    cast_f32_bf16_kernel<<<grid_for(n), 256, 0, cs>>>(ctx->w + ctx->owned_off[p],
                                                     ctx->replica + ctx->flat_off[p], n);
  }
  OSH_CUDA_TRY(cudaGetLastError());
  if (ctx->tp_size > 1)
    if (osh_status st = tp_refresh_replica(ctx, cs); st != OSH_OK) return st;
  const bool ag = ctx->comm_mode == OSH_COMM_NCCL && ctx->size > 1 && ctx->comm != nullptr;
  if (ag && !ctx->sched_ag.empty()) {
    const int b0 = ctx->sched_ag.front().first, b1 = ctx->sched_ag.back().second;
    if (osh_status st = issue_ops(ctx, b0, b1, cs); st != OSH_OK) return st;
  }
  return wait_stream(ctx, cs);
}

// RS-v of bucket b on the comm stream: the owner of each slice receives the
// sum of all ranks' slices in its grad_owned region (local grads intact).
osh_status issue_rs(osh_ctx* ctx, int b) {
  const auto [b0, b1] = ctx->sched_rs[static_cast<size_t>(b)];
  if (osh_status st = issue_ops(ctx, b0, b1, ctx->comm_stream); st != OSH_OK) return st;
  OSH_CUDA_TRY(cudaEventRecord(ctx->rs_ev[b], ctx->comm_stream));
  return OSH_OK;
}

}  // namespace osh

extern "C" {

osh_status osh_nccl_unique_id(uint8_t out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  if (out == nullptr) return osh::fail(OSH_ERR_ARG, "null output");
  ncclUniqueId id;
  OSH_NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return OSH_OK;
}

osh_status osh_ctx_create(int32_t device, int32_t dp_rank, int32_t dp_size, int32_t comm_mode,
                          const uint8_t* nccl_uid, osh_ctx** out) {
  return osh_ctx_create_tp(device, dp_rank, dp_size, 0, 1, comm_mode, nccl_uid, nullptr, out);
}

osh_status osh_ctx_create_tp(int32_t device, int32_t dp_rank, int32_t dp_size, int32_t tp_rank,
                             int32_t tp_size, int32_t comm_mode, const uint8_t* dp_uid,
                             const uint8_t* tp_uid, osh_ctx** out) {
  const uint8_t* nccl_uid = dp_uid;
  if (out == nullptr) return osh::fail(OSH_ERR_ARG, "null output");
  *out = nullptr;
  if (dp_size < 1 || dp_rank < 0 || dp_rank >= dp_size)
    return osh::fail(OSH_ERR_PLAN, "dp_rank/dp_size out of range");
  if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size)
    return osh::fail(OSH_ERR_SHARD, "tp_rank/tp_size out of range");
  if (tp_size > 1 && comm_mode != OSH_COMM_NCCL)
    return osh::fail(OSH_ERR_UNSUPPORTED, "tensor parallelism needs OSH_COMM_NCCL");
  if (comm_mode != OSH_COMM_NCCL && comm_mode != OSH_COMM_NONE)
    return osh::fail(OSH_ERR_ARG, "unknown comm_mode");
  OSH_CUDA_TRY(cudaSetDevice(device));
  std::unique_ptr<osh_ctx> ctx(new osh_ctx());
  ctx->device = device;
  ctx->rank = dp_rank;
  ctx->size = dp_size;
  ctx->comm_mode = comm_mode;
  if (const char* to = std::getenv("OSH_COMM_TIMEOUT_S"); to != nullptr && std::atof(to) > 0.0)
    ctx->timeout_s = std::atof(to);
  OSH_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->compute, cudaStreamNonBlocking));
  OSH_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
  int prio_low = 0, prio_high = 0;
  OSH_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high));
  OSH_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->gemm_stream, cudaStreamNonBlocking, prio_high));
  OSH_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
  OSH_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
  for (cudaEvent_t& e : ctx->ev) OSH_CUDA_TRY(cudaEventCreate(&e));
  for (cudaEvent_t& e : ctx->seq_pre_ev) OSH_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  OSH_CUDA_TRY(cudaEventCreateWithFlags(&ctx->seq_ns_ev, cudaEventDisableTiming));
  if (comm_mode == OSH_COMM_NCCL && dp_size > 1) {
    if (nccl_uid == nullptr) return osh::fail(OSH_ERR_ARG, "nccl_uid required for dp_size > 1");
    ncclUniqueId id;
    std::memcpy(&id, nccl_uid, sizeof(id));
    // OSH_NCCL_MAX_CTAS caps the SMs NCCL's kernels may take from the
    // persistent GEMMs they overlap (NCCL collective path / TP path)
    ncclConfig_t config = NCCL_CONFIG_INITIALIZER;
    if (const char* mc = std::getenv("OSH_NCCL_MAX_CTAS"); mc != nullptr && std::atoi(mc) > 0)
      config.maxCTAs = std::atoi(mc);
    if (const char* cp = std::getenv("OSH_NCCL_CTA_POLICY"); cp != nullptr)
      config.CTAPolicy = std::atoi(cp);  // NCCL_CTA_POLICY_{DEFAULT,EFFICIENCY,ZERO}
    OSH_NCCL_TRY(ncclCommInitRankConfig(&ctx->comm, dp_size, id, dp_rank, &config));
  }
  ctx->tp_rank = tp_rank;
  ctx->tp_size = tp_size;
  if (tp_size > 1) {
    if (tp_uid == nullptr) return osh::fail(OSH_ERR_ARG, "tp_uid required for tp_size > 1");
    ncclUniqueId id;
    std::memcpy(&id, tp_uid, sizeof(id));
    ncclConfig_t config = NCCL_CONFIG_INITIALIZER;
    if (const char* mc = std::getenv("OSH_NCCL_MAX_CTAS"); mc != nullptr && std::atoi(mc) > 0)
      config.maxCTAs = std::atoi(mc);
    if (const char* cp = std::getenv("OSH_NCCL_CTA_POLICY"); cp != nullptr)
      config.CTAPolicy = std::atoi(cp);
    OSH_NCCL_TRY(ncclCommInitRankConfig(&ctx->tp_comm, tp_size, id, tp_rank, &config));
    OSH_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->tp_stream, cudaStreamNonBlocking));
    OSH_CUDA_TRY(cudaEventCreateWithFlags(&ctx->tp_start_ev, cudaEventDisableTiming));
    OSH_CUDA_TRY(cudaEventCreateWithFlags(&ctx->tp_done_ev, cudaEventDisableTiming));
    OSH_CUDA_TRY(cudaEventCreate(&ctx->tp_begin_ev));
    OSH_CUDA_TRY(cudaEventCreate(&ctx->tp_end_ev));
  }
  *out = ctx.release();
  return OSH_OK;
}

osh_status osh_ctx_set_tp_capacity(osh_ctx* ctx, uint64_t c_max) {
  if (ctx == nullptr || c_max == 0) return osh::fail(OSH_ERR_UNSCHEDULABLE, "c_max must be positive");
  ctx->tp_c_max = c_max;
  return OSH_OK;
}

osh_status osh_ctx_set_collectives(osh_ctx* ctx, int32_t mode) {
  if (ctx == nullptr) return osh::fail(OSH_ERR_ARG, "null osh_ctx");
  if (mode != OSH_COLL_AUTO && mode != OSH_COLL_NCCL && mode != OSH_COLL_NVLS)
    return osh::fail(OSH_ERR_ARG, "unknown collectives mode");
  ctx->coll_mode = mode;
  return OSH_OK;
}

osh_status osh_ctx_set_strategy(osh_ctx* ctx, int32_t strategy, const int32_t* layer_of,
                                int32_t n, const osh_cost_model* cost) {
  if (ctx == nullptr) return osh::fail(OSH_ERR_ARG, "null osh_ctx");
  if (strategy < OSH_STRAT_SHARDED || strategy > OSH_STRAT_NV_LAYERWISE)
    return osh::fail(OSH_ERR_CONFIG, "unknown strategy");
  if (strategy != OSH_STRAT_SHARDED && ctx->tp_size > 1)
    return osh::fail(OSH_ERR_UNSUPPORTED, "SC / NV-layerwise baselines run with tp_size == 1");
  if (strategy == OSH_STRAT_NV_LAYERWISE && (layer_of == nullptr || n < 1))
    return osh::fail(OSH_ERR_ARG, "NV-layerwise needs the layer group of every parameter");
  ctx->strategy = strategy;
  ctx->layer_of.clear();
  if (layer_of != nullptr) ctx->layer_of.assign(layer_of, layer_of + n);
  ctx->strategy_cost = CostModel{};
  if (cost != nullptr) {
    if (cost->kind < OSH_COST_NUMEL || cost->kind > OSH_COST_BYTES)
      return osh::fail(OSH_ERR_CONFIG, "unknown cost kind");
    ctx->strategy_cost.kind = static_cast<CostKind>(cost->kind);
    ctx->strategy_cost.ns_steps = cost->ns_steps;
    ctx->strategy_cost.shampoo_coeff = cost->shampoo_coeff;
    ctx->strategy_cost.soap_coeff = cost->soap_coeff;
  }
  return OSH_OK;
}

osh_status osh_shampoo_cfg_default(osh_shampoo_cfg* out) {
  if (out == nullptr) return osh::fail(OSH_ERR_ARG, "null output");
  const osh::ShampooConfig d;
  std::memset(out, 0, sizeof(*out));
  out->beta2 = d.beta2;
  out->eps = d.eps;
  out->block = d.block;
  out->precond_every = d.precond_every;
  out->newton_iters = d.newton_iters;
  return OSH_OK;
}

osh_status osh_ctx_set_optimizer(osh_ctx* ctx, int32_t kind, const osh_shampoo_cfg* cfg) {
  if (ctx == nullptr) return osh::fail(OSH_ERR_ARG, "null osh_ctx");
  if (kind != OSH_OPT_MUON && kind != OSH_OPT_SHAMPOO && kind != OSH_OPT_SOAP)
    return osh::fail(OSH_ERR_ARG, "unknown optimizer");
  if (kind != OSH_OPT_MUON && ctx->tp_size > 1)
    return osh::fail(OSH_ERR_UNSUPPORTED, "Shampoo / SOAP run with tp_size == 1");
  ctx->optimizer = kind;
  if (cfg != nullptr) {
    if (cfg->block < 64 || cfg->block % 64 != 0 || cfg->precond_every < 1 ||
        cfg->newton_iters < 1 || !(cfg->beta2 >= 0.0 && cfg->beta2 <= 1.0) || !(cfg->eps > 0.0))
      return osh::fail(OSH_ERR_CONFIG, "invalid osh_shampoo_cfg");
    ctx->shampoo.beta2 = cfg->beta2;
    ctx->shampoo.eps = cfg->eps;
    ctx->shampoo.block = cfg->block;
    ctx->shampoo.precond_every = cfg->precond_every;
    ctx->shampoo.newton_iters = cfg->newton_iters;
  }
  return OSH_OK;
}

osh_status osh_ctx_destroy(osh_ctx* ctx) {
  if (ctx == nullptr) return OSH_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->compute);
  cudaStreamSynchronize(ctx->comm_stream);
  cudaStreamSynchronize(ctx->gemm_stream);
  cudaStreamSynchronize(ctx->h2d_stream);
  cudaStreamSynchronize(ctx->d2h_stream);
  free_layout(ctx);
  if (ctx->comm != nullptr) ncclCommDestroy(ctx->comm);
  if (ctx->tp_comm != nullptr) ncclCommDestroy(ctx->tp_comm);  // (nullptr once aborted)
  if (ctx->tp_stream != nullptr) {
    cudaStreamSynchronize(ctx->tp_stream);
    cudaStreamDestroy(ctx->tp_stream);
    cudaEventDestroy(ctx->tp_start_ev);
    cudaEventDestroy(ctx->tp_done_ev);
    cudaEventDestroy(ctx->tp_begin_ev);
    cudaEventDestroy(ctx->tp_end_ev);
  }
  for (cudaEvent_t e : ctx->ev) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->seq_pre_ev) cudaEventDestroy(e);
  if (ctx->seq_ns_ev != nullptr) cudaEventDestroy(ctx->seq_ns_ev);
  cudaStreamDestroy(ctx->compute);
  cudaStreamDestroy(ctx->comm_stream);
  cudaStreamDestroy(ctx->gemm_stream);
  cudaStreamDestroy(ctx->h2d_stream);
  cudaStreamDestroy(ctx->d2h_stream);
  delete ctx;
  return OSH_OK;
}

osh_status osh_ctx_set_layout(osh_ctx* ctx, const osh_param_desc* params, int32_t n,
                              int64_t bucket_capacity, const int64_t* cuts, int32_t n_buckets,
                              int32_t grad_dtype, int64_t workspace_bytes) {
  if (osh_status st = check_ctx(ctx, false); st != OSH_OK) return st;
  if (grad_dtype != OSH_GRAD_F32 && grad_dtype != OSH_GRAD_BF16)
    return osh::fail(OSH_ERR_ARG, "grad_dtype must be OSH_GRAD_F32 or OSH_GRAD_BF16");
  if (params == nullptr || cuts == nullptr || n < 1)
    return osh::fail(OSH_ERR_ARG, "params and cuts are required");
  free_layout(ctx);
  try {
    ctx->params.clear();
    for (int32_t i = 0; i < n; ++i) {
      const osh_param_desc& d = params[i];
      if (d.id != i) throw PlanError("parameter ids must be dense 0..n-1 in order");
      ParamSpec p;
      p.id = d.id;
      p.name = "p" + std::to_string(d.id);
      p.shape.assign(d.shape, d.shape + (d.ndim == 2 ? 2 : 1));
      p.numel = 1;
      for (const int64_t e : p.shape) p.numel *= e;
      p.dtype_bytes = d.dtype_bytes;
      p.tp_splittable = d.tp_split == 1 ? TpSplit::kColumn
                        : d.tp_split == 2 ? TpSplit::kRow
                                          : TpSplit::kNone;
      p.vocab_space = d.vocab_space != 0;
      ctx->params.push_back(p);
    }
    if (ctx->tp_size > 1) {
      // params are the FULL tensors; the DP layout / plan are over the shard view
      ctx->params_full = ctx->params;
      ctx->params = apply_tp_sharding(ctx->params_full, ctx->tp_size);
    } else {
      ctx->params_full = ctx->params;
    }
    ctx->layout = build_buffer_layout(ctx->params, bucket_capacity);
    if (static_cast<int32_t>(ctx->layout.buckets.size()) != n_buckets)
      throw PlanError("cut vectors cover " + std::to_string(n_buckets) + " buckets, layout has " +
                      std::to_string(ctx->layout.buckets.size()));
    const int R = ctx->size;
    DpPartitionPlan plan;
    plan.ranks = R;
    plan.atomic = true;
    ctx->cuts.assign(static_cast<size_t>(n_buckets), {});
    for (int32_t b = 0; b < n_buckets; ++b) {
      ctx->cuts[b].assign(cuts + static_cast<size_t>(b) * (R + 1),
                          cuts + static_cast<size_t>(b + 1) * (R + 1));
      plan.cut_vectors.push_back(ctx->cuts[b]);
    }
    detail::fill_rank_sizes(plan);
    // structural checks of validate_plan that do not need the plan's loads
    for (int32_t b = 0; b < n_buckets; ++b) {
      const auto& c = ctx->cuts[b];
      const auto edges = ctx->layout.buckets[b].atomic_boundaries();
      if (c.front() != 0 || c.back() != ctx->layout.buckets[b].numel)
        throw PlanError("bucket " + std::to_string(b) + ": cuts must span [0, numel]");
      for (int r = 0; r <= R; ++r) {
        if (r < R && c[r] > c[r + 1])
          throw PlanError("bucket " + std::to_string(b) + ": cuts are not monotone");
        if (!std::binary_search(edges.begin(), edges.end(), c[r]))
          throw PlanError("bucket " + std::to_string(b) + ": cut " + std::to_string(c[r]) +
                          " splits a tensor (Muon needs an atomic plan)");
      }
    }
    const size_t np = ctx->params.size();
    ctx->flat_off.assign(np, 0);
    ctx->bucket_of.assign(np, 0);
    ctx->owner.assign(np, 0);
    ctx->owned_off.assign(np, -1);
    ctx->engine_index.assign(np, -1);
    ctx->bucket_base.assign(static_cast<size_t>(n_buckets), 0);
    int64_t base = 0;
    for (int32_t b = 0; b < n_buckets; ++b) {
      const Bucket& bk = ctx->layout.buckets[b];
      ctx->bucket_base[b] = base;
      for (size_t j = 0; j < bk.param_ids.size(); ++j) {
        ctx->flat_off[bk.param_ids[j]] = base + bk.param_offsets[j];
        ctx->bucket_of[bk.param_ids[j]] = b;
      }
      base += bk.numel;
    }
    ctx->total_numel = base;
    ctx->owned_numel = 0;
    int64_t alloc = 0;
    // strategy baselines: SC replicates every tensor; NV-layerwise assigns whole
    // layers by LPT (min_heap_balance over the layer costs, simulate.hpp:140-157)
    std::vector<int> layer_owner;  // per parameter (NV-layerwise)
    if (ctx->strategy == OSH_STRAT_NV_LAYERWISE)
      layer_owner = osh::layerwise_owners(ctx->params, ctx->layer_of, ctx->size, ctx->strategy_cost);
    for (size_t p = 0; p < np; ++p) {
      if (ctx->strategy == OSH_STRAT_SC)
        ctx->owner[p] = ctx->rank;
      else if (ctx->strategy == OSH_STRAT_NV_LAYERWISE)
        ctx->owner[p] = layer_owner[p];
      else
        ctx->owner[p] = param_owner(plan, ctx->layout, static_cast<int>(p));
      if (ctx->owner[p] == ctx->rank && !is_tp_item(ctx, p)) {
        ctx->owned_off[p] = alloc;
        alloc += (ctx->params[p].numel + kOwnedAlign - 1) / kOwnedAlign * kOwnedAlign;
        ctx->owned_numel += ctx->params[p].numel;
      }
    }
    ctx->owned_alloc = alloc;
    // the collective schedule every rank issues (identical on all ranks)
    ctx->sched.clear();
    ctx->sched_rs.assign(static_cast<size_t>(n_buckets), {0, 0});
    ctx->sched_ag.assign(static_cast<size_t>(n_buckets), {0, 0});
    if (ctx->comm_mode == OSH_COMM_NCCL && R > 1) {
      std::vector<int64_t> numel(np);
      for (size_t p = 0; p < np; ++p) numel[p] = ctx->params[p].numel;
      ctx->sched = osh::build_comm_schedule(ctx->strategy, ctx->cuts, ctx->bucket_base,
                                            ctx->flat_off, numel, ctx->owner);
      for (int32_t b = 0; b < n_buckets; ++b) {  // op ranges per bucket and leg
        auto& rs = ctx->sched_rs[static_cast<size_t>(b)];
        auto& ag = ctx->sched_ag[static_cast<size_t>(b)];
        rs = ag = {-1, -1};
        for (int i = 0; i < static_cast<int>(ctx->sched.size()); ++i) {
          const osh_coll_op& o = ctx->sched[static_cast<size_t>(i)];
          if (o.bucket != b) continue;
          auto& r = o.phase == OSH_PHASE_RS ? rs : ag;
          if (r.first < 0) r.first = i;
          r.second = i + 1;
        }
        if (rs.first < 0) rs = {0, 0};
        if (ag.first < 0) ag = {0, 0};
      }
    }
  } catch (const PlanError& e) {
    return osh::fail(OSH_ERR_PLAN, std::string("osh_ctx_set_layout: ") + e.what());
  } catch (const ShardError& e) {
    return osh::fail(OSH_ERR_SHARD, std::string("osh_ctx_set_layout: ") + e.what());
  } catch (const LayoutError& e) {
    return osh::fail(OSH_ERR_LAYOUT, std::string("osh_ctx_set_layout: ") + e.what());
  } catch (const std::exception& e) {
    return osh::fail(OSH_ERR_ARG, std::string("osh_ctx_set_layout: ") + e.what());
  }

  ctx->grad_dtype = grad_dtype;
  const size_t es = grad_esize(grad_dtype);
  // NVLS needs every tensor on the 16-byte vector layout (decided from the
  // model alone, so every rank takes the same branch of the collective setup)
  bool nvls_layout = distributed(ctx) && ctx->strategy == OSH_STRAT_SHARDED;
  for (size_t p = 0; p < ctx->params.size() && nvls_layout; ++p) {
    const ParamSpec& ps = ctx->params[p];
    const int64_t inner = ps.is_matrix() ? ps.shape[1] : ps.numel;
    nvls_layout = ctx->flat_off[p] % 8 == 0 && inner % 8 == 0;
  }
  if (ctx->coll_mode == OSH_COLL_NVLS && !nvls_layout)
    return osh::fail(OSH_ERR_UNSUPPORTED,
                     "NVLS collectives need dp_size > 1 and 8-element aligned tensors");
  if (nvls_layout && ctx->coll_mode != OSH_COLL_NCCL) {
    constexpr size_t kGran = 2u << 20;
    const size_t gb = (es * static_cast<size_t>(ctx->total_numel) + kGran - 1) / kGran * kGran;
    const size_t rb = (2 * static_cast<size_t>(ctx->total_numel) + kGran - 1) / kGran * kGran;
    if (osh_status st = osh::nvls_setup(ctx, gb, rb, ctx->coll_mode == OSH_COLL_NVLS); st != OSH_OK)
      return st;
  }
  if (!ctx->nvls) {
    OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&ctx->grad), es * static_cast<size_t>(ctx->total_numel)));
    OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&ctx->replica), 2 * static_cast<size_t>(ctx->total_numel)));
  }
  OSH_CUDA_TRY(cudaMemset(ctx->grad, 0, es * static_cast<size_t>(ctx->total_numel)));
  OSH_CUDA_TRY(cudaMemset(ctx->replica, 0, 2 * static_cast<size_t>(ctx->total_numel)));
  if (distributed(ctx)) OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&ctx->bar), 16));
  // Reduced-gradient slices of this rank (NCCL mode): bucket after bucket.
  // (SC / NV-layerwise all-reduce the whole buffer in place instead.)
  const bool reduce_out = distributed(ctx) && !ctx->nvls && ctx->strategy == OSH_STRAT_SHARDED;
  ctx->owned_slice_off.assign(ctx->cuts.size(), 0);
  int64_t slice_total = 0;
  for (size_t b = 0; b < ctx->cuts.size(); ++b) {
    ctx->owned_slice_off[b] = slice_total;
    slice_total += ctx->cuts[b][ctx->rank + 1] - ctx->cuts[b][ctx->rank];
  }
  if (reduce_out)
    OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&ctx->grad_owned), es * static_cast<size_t>(std::max<int64_t>(slice_total, 1))));
  const size_t owned_bytes = 4 * static_cast<size_t>(std::max<int64_t>(ctx->owned_alloc, 1));
  OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&ctx->w), owned_bytes));
  OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&ctx->m), owned_bytes));
  OSH_CUDA_TRY(cudaMemset(ctx->w, 0, owned_bytes));
  OSH_CUDA_TRY(cudaMemset(ctx->m, 0, owned_bytes));

  std::vector<osh::MuonTensorDesc> tensors;
  for (size_t p = 0; p < ctx->params.size(); ++p) {
    if (ctx->owned_off[p] < 0) continue;
    const ParamSpec& ps = ctx->params[p];
    osh::MuonTensorDesc t;
    t.is_matrix = ps.is_matrix() ? 1 : 0;
    t.vocab_space = ps.vocab_space ? 1 : 0;
    t.bucket = ctx->bucket_of[p];
    t.rows = static_cast<int>(ps.shape[0]);
    t.cols = ps.is_matrix() ? static_cast<int>(ps.shape[1]) : 1;
    t.w = ctx->w + ctx->owned_off[p];
    t.m = ctx->m + ctx->owned_off[p];
    if (ctx->nvls) {
      // the cross-rank sum is read through the multicast address (RS-v fused)
      t.g = static_cast<uint8_t*>(ctx->mc_grad) + es * static_cast<size_t>(ctx->flat_off[p]);
      t.g_mc = 1;
    } else if (reduce_out) {
      // position of p inside this rank's reduced slice of its bucket
      const int bucket = ctx->bucket_of[p];
      const int64_t in_slice = ctx->flat_off[p] - ctx->bucket_base[bucket] - ctx->cuts[bucket][ctx->rank];
      t.g = static_cast<uint8_t*>(ctx->grad_owned) +
            es * static_cast<size_t>(ctx->owned_slice_off[bucket] + in_slice);
    } else {
      t.g = static_cast<uint8_t*>(ctx->grad) + es * static_cast<size_t>(ctx->flat_off[p]);
    }
    t.replica = ctx->replica + ctx->flat_off[p];
    if (ctx->nvls) {
      t.replica = ctx->mc_replica + ctx->flat_off[p];  // multimem.st to every rank (AG-v fused)
      t.rep_mc = 1;
      t.replica_local = ctx->replica + ctx->flat_off[p];
    }
    ctx->engine_index[p] = static_cast<int>(tensors.size());
    tensors.push_back(t);
  }
  size_t budget = workspace_bytes > 0 ? static_cast<size_t>(workspace_bytes) : 0;
  if (budget == 0) {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    budget = std::min<size_t>(24ull << 30, free_b / 3);
  }
  if (ctx->optimizer == OSH_OPT_SHAMPOO) {
    ctx->engine = std::make_unique<osh::ShampooEngine>(ctx->shampoo);
  } else if (ctx->optimizer == OSH_OPT_SOAP) {
    osh::SoapConfig sc;  // osh_shampoo_cfg fields: newton_iters = init_iters
    sc.beta2 = ctx->shampoo.beta2;
    sc.eps = ctx->shampoo.eps;
    sc.block = ctx->shampoo.block;
    sc.precond_every = ctx->shampoo.precond_every;
    sc.init_iters = ctx->shampoo.newton_iters;
    ctx->engine = std::make_unique<osh::SoapEngine>(sc);
  }
  else
    ctx->engine = std::make_unique<osh::MuonEngine>();
  const char* ov = std::getenv("OSH_OVERLAP");
  const bool overlap_on = !(ov != nullptr && std::strcmp(ov, "0") == 0);
  // run_waves_local's schedule (one rank, NVLS, SC / NV-layerwise), or the
  // stage sequence of the NCCL RS-v / AG-v and TP paths (Muon: split phases)
  const bool seq_path = (distributed(ctx) && ctx->strategy == OSH_STRAT_SHARDED && !ctx->nvls) ||
                        ctx->tp_size > 1;
  ctx->overlap = ctx->tp_size == 1 && !reduce_out && overlap_on;
  // (opt-in, OSH_SEQ_OVERLAP=1: measured neutral to slightly slower on these
  // paths — their momentum reads local HBM at full rate and, under the power
  // cap, slows the GEMMs beside it by as much as it hides; profiles/
  // r02_seq_overlap_ab.json)
  const char* so = std::getenv("OSH_SEQ_OVERLAP");
  ctx->seq_overlap = seq_path && overlap_on && ctx->optimizer == OSH_OPT_MUON &&
                     so != nullptr && std::strcmp(so, "1") == 0;
  // (one rank: 16 waves measured 0.7-0.9 % faster than 8 on two boxes,
  // NVLS N=4 neutral: profiles/r02_waves_ab.json)
  int min_waves = ctx->min_waves > 0 ? ctx->min_waves
                  : ctx->overlap ? (distributed(ctx) ? 8 : 16)
                  : (reduce_out && ctx->tp_size == 1) ? 4 : 1;
  if (const char* mw = std::getenv("OSH_MIN_WAVES"); mw != nullptr && std::atoi(mw) > 0)
    min_waves = std::atoi(mw);
  // waves in any order where nothing bucket-ordered waits on them: one rank,
  // or NVLS (the step barrier covers every bucket; collectives are inside the
  // kernels). NCCL RS-v / AG-v, SC / NV-layerwise and TP keep bucket order.
  const char* ro = std::getenv("OSH_WAVE_REORDER");
  const bool reorder = ctx->tp_size == 1 && ctx->strategy == OSH_STRAT_SHARDED &&
                       (!distributed(ctx) || ctx->nvls) && !(ro != nullptr && std::strcmp(ro, "0") == 0);
  ctx->engine->set_wave_reorder(reorder);
  if (osh_status st = ctx->engine->build(tensors, grad_dtype, budget, min_waves,
                                         ctx->overlap || ctx->seq_overlap);
      st != OSH_OK)
    return st;
  {
    const int nw = ctx->engine->num_waves();
    const int nbk = static_cast<int>(ctx->cuts.size());
    std::vector<int> done_at(static_cast<size_t>(nbk), -1);
    ctx->h2d_bucket_order.clear();
    std::vector<char> queued(static_cast<size_t>(nbk), 0);
    for (int w = 0; w < nw; ++w)
      for (int b = ctx->engine->wave_first_bucket(w); b <= ctx->engine->wave_last_bucket(w); ++b) {
        done_at[static_cast<size_t>(b)] = std::max(done_at[static_cast<size_t>(b)], w);
        if (!queued[static_cast<size_t>(b)]) {
          queued[static_cast<size_t>(b)] = 1;
          ctx->h2d_bucket_order.push_back(b);
        }
      }
    for (int b = 0; b < nbk; ++b)
      if (!queued[static_cast<size_t>(b)]) ctx->h2d_bucket_order.push_back(b);
    if (!reorder || distributed(ctx))  // NCCL RS-v waits per bucket in bucket order
      for (int b = 0; b < nbk; ++b) ctx->h2d_bucket_order[static_cast<size_t>(b)] = b;
    ctx->wave_done_buckets.assign(static_cast<size_t>(nw), {});
    for (int b = 0; b < nbk; ++b)  // (buckets no wave touches go with the last wave)
      ctx->wave_done_buckets[static_cast<size_t>(done_at[static_cast<size_t>(b)] >= 0
                                                     ? done_at[static_cast<size_t>(b)]
                                                     : nw - 1)]
          .push_back(b);
    ctx->wave_final_upto.assign(static_cast<size_t>(nw), -1);
    for (int w = 0; w < nw; ++w) {
      int upto = -1;
      while (upto + 1 < nbk && done_at[static_cast<size_t>(upto + 1)] <= w) ++upto;
      ctx->wave_final_upto[static_cast<size_t>(w)] = upto;
    }
  }
  ctx->overlap = ctx->overlap && ctx->engine->double_buffered() && ctx->engine->num_waves() > 1;
  {  // single rank: per-wave host transfer ranges (every tensor owned, each in one wave)
    ctx->wave_io = false;
    ctx->wave_ranges.clear();
    destroy_events(ctx->h2d_wave_ev);
    const int nw = ctx->engine->num_waves();
    std::vector<int> param_of(static_cast<size_t>(ctx->engine->num_tensors()), -1);
    for (size_t p = 0; p < ctx->params.size(); ++p)
      if (ctx->engine_index[p] >= 0) param_of[static_cast<size_t>(ctx->engine_index[p])] = static_cast<int>(p);
    int64_t covered = 0;
    bool ok = ctx->size == 1 && ctx->tp_size == 1 && nw > 0;
    for (int w = 0; w < nw && ok; ++w) {
      const std::vector<int>& ts = ctx->engine->wave_tensors(w);
      if (ts.empty()) ok = false;
      std::vector<std::pair<int64_t, int64_t>> r;
      for (const int ti : ts) {
        const int p = param_of[static_cast<size_t>(ti)];
        if (p < 0) {
          ok = false;
          break;
        }
        const int64_t off = ctx->flat_off[static_cast<size_t>(p)], cnt = ctx->params[static_cast<size_t>(p)].numel;
        if (!r.empty() && r.back().first + r.back().second == off) r.back().second += cnt;
        else r.emplace_back(off, cnt);
        covered += cnt;
      }
      ctx->wave_ranges.push_back(std::move(r));
    }
    ctx->wave_io = ok && covered == ctx->total_numel;
    if (ctx->wave_io) OSH_CUDA_TRY(make_events(ctx->h2d_wave_ev, static_cast<size_t>(nw)));
  }
  if (ctx->tp_size > 1)
    if (osh_status st = osh::tp_setup(ctx, static_cast<int64_t>(budget)); st != OSH_OK) return st;
  OSH_CUDA_TRY(make_events(ctx->rs_ev, ctx->cuts.size()));
  OSH_CUDA_TRY(make_events(ctx->wave_begin, static_cast<size_t>(ctx->engine->num_waves())));
  OSH_CUDA_TRY(make_events(ctx->wave_end, static_cast<size_t>(ctx->engine->num_waves())));
  OSH_CUDA_TRY(make_events(ctx->pre_ev, static_cast<size_t>(ctx->engine->num_waves())));
  OSH_CUDA_TRY(make_events(ctx->h2d_ev, ctx->cuts.size()));
  ctx->bucket_marked.assign(ctx->cuts.size(), 0);
  ctx->n_marked = 0;
  OSH_CUDA_TRY(make_events(ctx->ag_ev, ctx->cuts.size()));
  OSH_CUDA_TRY(make_events(ctx->ns_ev, static_cast<size_t>(ctx->engine->num_waves())));
  // The zero-fills and table uploads above ran on the legacy stream, which the
  // ctx's non-blocking streams do not order against: finish them now.
  OSH_CUDA_TRY(cudaDeviceSynchronize());
  ctx->layout_ready = true;
  return OSH_OK;
}

osh_status osh_ctx_get_info(osh_ctx* ctx, osh_ctx_info* out) {
  if (osh_status st = check_ctx(ctx, true); st != OSH_OK) return st;
  std::memset(out, 0, sizeof(*out));
  out->total_numel = ctx->total_numel;
  out->owned_numel = ctx->owned_numel;
  out->n_params = static_cast<int32_t>(ctx->params.size());
  out->n_buckets = static_cast<int32_t>(ctx->layout.buckets.size());
  out->n_waves = ctx->engine->num_waves();
  out->workspace_bytes = static_cast<int64_t>(ctx->engine->workspace_bytes());
  double flops = 0.0;
  for (size_t p = 0; p < ctx->params.size(); ++p) {
    if (ctx->owned_off[p] < 0) continue;
    ++out->n_owned;
    const ParamSpec& ps = ctx->params[p];
    if (!ps.is_matrix()) continue;
    const double m = static_cast<double>(std::min(ps.shape[0], ps.shape[1]));
    const double nn = static_cast<double>(std::max(ps.shape[0], ps.shape[1]));
    flops += 4.0 * m * m * nn + 2.0 * m * m * m;
  }
  for (const osh_ctx::TpItem& it : ctx->tp_items) {
    if (it.w == nullptr) continue;  // hosted by another TP rank
    const double m = static_cast<double>(std::min(it.full_rows, it.full_cols));
    const double nn = static_cast<double>(std::max(it.full_rows, it.full_cols));
    flops += 4.0 * m * m * nn + 2.0 * m * m * m;
    ++out->n_owned;
  }
  out->ns_flops_per_iter = flops;
  out->collectives = !distributed(ctx) ? 0 : ctx->nvls ? OSH_COLL_NVLS : OSH_COLL_NCCL;
  out->device_bytes = static_cast<int64_t>(
      grad_esize(ctx->grad_dtype) * ctx->total_numel + 2 * ctx->total_numel +
      8 * std::max<int64_t>(ctx->owned_alloc, 1) + ctx->engine->workspace_bytes());
  return OSH_OK;
}

osh_status osh_ctx_buffers(osh_ctx* ctx, void** grad, void** replica) {
  if (osh_status st = check_ctx(ctx, true); st != OSH_OK) return st;
  if (grad != nullptr) *grad = ctx->grad;
  if (replica != nullptr) *replica = ctx->replica;
  return OSH_OK;
}

osh_status osh_load_param(osh_ctx* ctx, int32_t pid, const float* values) {
  if (osh_status st = check_ctx(ctx, true); st != OSH_OK) return st;
  if (pid < 0 || pid >= static_cast<int32_t>(ctx->params.size()) || values == nullptr)
    return osh::fail(OSH_ERR_PLAN, "osh_load_param: unknown parameter");
  std::vector<float> shard_buf;
  if (ctx->tp_size > 1 && ctx->params_full[pid].tp_splittable != TpSplit::kNone) {
    // values are the FULL tensor: keep it whole at a TP host, slice my shard
    const ParamSpec& f = ctx->params_full[pid];
    const int T = ctx->tp_size, t = ctx->tp_rank;
    const int64_t R = f.shape[0], C = f.shape[1];
    const int ti = ctx->tp_item_of.empty() ? -1 : ctx->tp_item_of[pid];
    if (ti >= 0 && ctx->tp_items[ti].host == t) {
      const size_t nf = static_cast<size_t>(R * C);
      OSH_CUDA_TRY(cudaMemcpyAsync(ctx->tp_items[ti].w, values, 4 * nf, cudaMemcpyHostToDevice,
                                   ctx->compute));
      OSH_CUDA_TRY(cudaMemsetAsync(ctx->tp_items[ti].m, 0, 4 * nf, ctx->compute));
      OSH_CUDA_TRY(cudaStreamSynchronize(ctx->compute));
    }
    shard_buf.resize(static_cast<size_t>(R * C / T));
    if (f.tp_splittable == TpSplit::kRow) {
      std::memcpy(shard_buf.data(), values + t * (R / T) * C, 4 * shard_buf.size());
    } else {
      const int64_t cs = C / T;
      for (int64_t i = 0; i < R; ++i)
        std::memcpy(shard_buf.data() + i * cs, values + i * C + t * cs, 4 * static_cast<size_t>(cs));
    }
    values = shard_buf.data();
  }
  const int64_t n = ctx->params[pid].numel;
  float* stage = nullptr;
  OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&stage), 4 * static_cast<size_t>(n)));
  // Pageable H2D copies are ordered only on the stream they are issued on:
  // stage, convert and consume on the ctx's compute stream.
  OSH_CUDA_TRY(cudaMemcpyAsync(stage, values, 4 * static_cast<size_t>(n), cudaMemcpyHostToDevice,
                               ctx->compute));
  cast_f32_bf16_kernel<<<grid_for(n), 256, 0, ctx->compute>>>(stage, ctx->replica + ctx->flat_off[pid], n);
  if (ctx->owned_off[pid] >= 0) {
    OSH_CUDA_TRY(cudaMemcpyAsync(ctx->w + ctx->owned_off[pid], stage, 4 * static_cast<size_t>(n),
                                 cudaMemcpyDeviceToDevice, ctx->compute));
    OSH_CUDA_TRY(cudaMemsetAsync(ctx->m + ctx->owned_off[pid], 0, 4 * static_cast<size_t>(n),
                                 ctx->compute));
  }
  OSH_CUDA_TRY(cudaStreamSynchronize(ctx->compute));
  cudaFree(stage);
  return OSH_OK;
}

osh_status osh_write_grad(osh_ctx* ctx, int32_t pid, const float* values) {
  if (osh_status st = check_ctx(ctx, true); st != OSH_OK) return st;
  if (pid < 0 || pid >= static_cast<int32_t>(ctx->params.size()) || values == nullptr)
    return osh::fail(OSH_ERR_PLAN, "osh_write_grad: unknown parameter");
  const int64_t n = ctx->params[pid].numel;
  if (ctx->grad_dtype == OSH_GRAD_F32) {
    OSH_CUDA_TRY(cudaMemcpyAsync(static_cast<float*>(ctx->grad) + ctx->flat_off[pid], values,
                                 4 * static_cast<size_t>(n), cudaMemcpyHostToDevice, ctx->compute));
    OSH_CUDA_TRY(cudaStreamSynchronize(ctx->compute));
    return OSH_OK;
  }
  float* stage = nullptr;
  OSH_CUDA_TRY(osh::dev_alloc(reinterpret_cast<void**>(&stage), 4 * static_cast<size_t>(n)));
  OSH_CUDA_TRY(cudaMemcpyAsync(stage, values, 4 * static_cast<size_t>(n), cudaMemcpyHostToDevice,
                               ctx->compute));
  cast_f32_bf16_kernel<<<grid_for(n), 256, 0, ctx->compute>>>(
      stage, static_cast<__nv_bfloat16*>(ctx->grad) + ctx->flat_off[pid], n);
  OSH_CUDA_TRY(cudaStreamSynchronize(ctx->compute));
  cudaFree(stage);
  return OSH_OK;
}

osh_status osh_fill_synthetic(osh_ctx* ctx, uint64_t seed, int32_t what, float scale) {
  if (osh_status st = check_ctx(ctx, true); st != OSH_OK) return st;
  for (size_t p = 0; p < ctx->params.size(); ++p) {
    const ParamSpec& ps = ctx->params[p];
    const float s = scale / std::sqrt(static_cast<float>(ps.shape[0]));
    const long long n = ps.numel, base = ctx->flat_off[p];
    if (what == OSH_FILL_WEIGHTS) {
      fill_synth_kernel<<<grid_for(n), 256, 0, ctx->compute>>>(
          seed, base, n, s, ctx->owned_off[p] >= 0 ? ctx->w + ctx->owned_off[p] : nullptr,
          ctx->replica + base);
      if (ctx->owned_off[p] >= 0)
        OSH_CUDA_TRY(cudaMemsetAsync(ctx->m + ctx->owned_off[p], 0, 4 * static_cast<size_t>(n),
                                     ctx->compute));
      const int ti = ctx->tp_item_of.empty() ? -1 : ctx->tp_item_of[p];
      if (ti >= 0 && ctx->tp_items[ti].w != nullptr) {
        const osh_ctx::TpItem& it = ctx->tp_items[ti];
        const long long nf = it.full_rows * it.full_cols;
        fill_synth_kernel<<<grid_for(nf), 256, 0, ctx->compute>>>(seed ^ 0x5bd1e995ull, base, nf, s,
                                                                 it.w, nullptr);
        OSH_CUDA_TRY(cudaMemsetAsync(it.m, 0, 4 * static_cast<size_t>(nf), ctx->compute));
      }
    } else if (what == OSH_FILL_GRADS) {
      if (ctx->grad_dtype == OSH_GRAD_F32)
        fill_synth_kernel<<<grid_for(n), 256, 0, ctx->compute>>>(
            seed, base, n, s, static_cast<float*>(ctx->grad) + base, nullptr);
      else
        fill_synth_kernel<<<grid_for(n), 256, 0, ctx->compute>>>(
            seed, base, n, s, nullptr, static_cast<__nv_bfloat16*>(ctx->grad) + base);
    } else {
      return osh::fail(OSH_ERR_ARG, "osh_fill_synthetic: unknown target");
    }
  }
  OSH_CUDA_TRY(cudaGetLastError());
  OSH_CUDA_TRY(cudaStreamSynchronize(ctx->compute));
  return OSH_OK;
}

namespace {

// Waves on `cs`, either back to back or overlapped: momentum(w+1) and
// apply(w) on cs run while the GEMMs of wave w run on the high-priority
// gemm_stream (MuonEngine::run_pre/run_ns/run_post ordering contract).
// `pipelined`: the step's gradients arrive per bucket on h2d_stream (wave w
// waits for the buckets it reads) and finished replica buckets leave on
// d2h_stream after the wave that completes them.
struct HostIo {
  bool h2d = false;        // wait for h2d_ev before a wave's momentum
  const std::vector<cudaEvent_t>* wait_ev = nullptr;  // per-bucket events to wait instead
  void* replica_out = nullptr;  // per-bucket D2H after each wave (nullptr: none)
  int d2h_next = 0;
  bool nvls_out = false;   // NVLS: a cross-rank barrier per bucket precedes its D2H
  bool per_wave = false;   // single rank: H2D / D2H per wave (ctx->wave_ranges)
};

// OSH_HOST_OUT_OWNED on a sharded multi-rank ctx: each rank reads back only
// the slices it updated (its result); otherwise the whole replica bucket.
bool owned_out(const osh_ctx* ctx) {
  return ctx->host_out_owned && distributed(ctx) && ctx->tp_size == 1 &&
         ctx->strategy == OSH_STRAT_SHARDED;
}

osh_status copy_bucket_out(osh_ctx* ctx, void* host, int b, cudaStream_t st) {
  const int nb = static_cast<int>(ctx->cuts.size());
  int64_t b0 = ctx->bucket_base[b];
  int64_t b1 = b + 1 < nb ? ctx->bucket_base[b + 1] : ctx->total_numel;
  if (owned_out(ctx)) {
    b1 = ctx->bucket_base[b] + ctx->cuts[b][ctx->rank + 1];
    b0 = ctx->bucket_base[b] + ctx->cuts[b][ctx->rank];
  }
  if (b1 > b0)
    OSH_CUDA_TRY(cudaMemcpyAsync(static_cast<__nv_bfloat16*>(host) + b0, ctx->replica + b0,
                                 2 * static_cast<size_t>(b1 - b0), cudaMemcpyDeviceToHost, st));
  return OSH_OK;
}

osh_status d2h_buckets(osh_ctx* ctx, HostIo& io, int upto, cudaEvent_t ready) {
  if (io.replica_out == nullptr || upto < io.d2h_next) return OSH_OK;
  if (owned_out(ctx)) {  // own slices only: final on this rank, no cross-rank wait
    OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->d2h_stream, ready, 0));
    for (int b = io.d2h_next; b <= upto; ++b)
      if (osh_status st = copy_bucket_out(ctx, io.replica_out, b, ctx->d2h_stream); st != OSH_OK)
        return st;
    io.d2h_next = upto + 1;
    return OSH_OK;
  }
  if (io.nvls_out) {
    // every rank's multicast stores into these buckets must have landed: one
    // barrier per bucket on the comm stream (same count and order on every
    // rank, since all ranks share the bucket layout), then the copy
    OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->comm_stream, ready, 0));
    for (int b = io.d2h_next; b <= upto; ++b) {
      OSH_NCCL_TRY(ncclAllReduce(ctx->bar + 1, ctx->bar + 1, 1, ncclFloat32, ncclSum, ctx->comm,
                                 ctx->comm_stream));
      OSH_CUDA_TRY(cudaEventRecord(ctx->ag_ev[b], ctx->comm_stream));
    }
    ready = ctx->ag_ev[upto];
  }
  OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->d2h_stream, ready, 0));
  const int64_t b0 = ctx->bucket_base[io.d2h_next];
  const int64_t b1 = upto + 1 < static_cast<int>(ctx->bucket_base.size()) ? ctx->bucket_base[upto + 1]
                                                                          : ctx->total_numel;
  OSH_CUDA_TRY(cudaMemcpyAsync(static_cast<__nv_bfloat16*>(io.replica_out) + b0, ctx->replica + b0,
                               2 * static_cast<size_t>(b1 - b0), cudaMemcpyDeviceToHost,
                               ctx->d2h_stream));
  io.d2h_next = upto + 1;
  return OSH_OK;
}

osh_status run_waves_local(osh_ctx* ctx, const osh_muon_cfg& cfg, cudaStream_t cs, HostIo& io) {
  osh::OptimizerEngine& eng = *ctx->engine;
  const int nw = eng.num_waves();
  const int nb = static_cast<int>(ctx->cuts.size());
  auto wait_input = [&](int w) -> osh_status {
    if (io.per_wave) {
      OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->h2d_wave_ev[static_cast<size_t>(w)], 0));
      return OSH_OK;
    }
    const std::vector<cudaEvent_t>* ev = io.wait_ev != nullptr ? io.wait_ev
                                         : io.h2d ? &ctx->h2d_ev : nullptr;
    if (ev != nullptr)  // every bucket of the wave (announced buckets may land out of order)
      for (int b = eng.wave_first_bucket(w); b <= eng.wave_last_bucket(w); ++b)
        OSH_CUDA_TRY(cudaStreamWaitEvent(cs, (*ev)[b], 0));
    return OSH_OK;
  };
  // after wave w: the buckets it completes leave at once (one rank / no
  // cross-rank barrier needed); NVLS copies bucket prefixes behind per-bucket
  // barriers issued in the same order on every rank
  auto wave_done = [&](int w) -> osh_status {
    OSH_CUDA_TRY(cudaEventRecord(ctx->wave_end[w], cs));
    if (io.replica_out != nullptr && io.per_wave) {  // exactly this wave's tensors
      OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->d2h_stream, ctx->wave_end[w], 0));
      for (const auto& [off, cnt] : ctx->wave_ranges[static_cast<size_t>(w)])
        OSH_CUDA_TRY(cudaMemcpyAsync(static_cast<__nv_bfloat16*>(io.replica_out) + off,
                                     ctx->replica + off, 2 * static_cast<size_t>(cnt),
                                     cudaMemcpyDeviceToHost, ctx->d2h_stream));
      if (w + 1 == nw) io.d2h_next = nb;
      return OSH_OK;
    }
    if (io.replica_out != nullptr && (!io.nvls_out || owned_out(ctx))) {
      // (owned slices need no cross-rank barrier: this rank wrote them)
      OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->d2h_stream, ctx->wave_end[w], 0));
      for (const int b : ctx->wave_done_buckets[static_cast<size_t>(w)])
        if (osh_status st = copy_bucket_out(ctx, io.replica_out, b, ctx->d2h_stream); st != OSH_OK)
          return st;
      if (w + 1 == nw) io.d2h_next = nb;  // every bucket is out
      return OSH_OK;
    }
    return d2h_buckets(ctx, io, w + 1 < nw ? ctx->wave_final_upto[static_cast<size_t>(w)] : nb - 1,
                       ctx->wave_end[w]);
  };
  if (!ctx->overlap) {
    for (int w = 0; w < nw; ++w) {
      if (osh_status st = wait_input(w); st != OSH_OK) return st;
      OSH_CUDA_TRY(cudaEventRecord(ctx->wave_begin[w], cs));
      if (osh_status st = eng.run_wave(w, cfg, cs); st != OSH_OK) return st;
      OSH_CUDA_TRY(cudaGetLastError());
      if (osh_status st = wave_done(w); st != OSH_OK) return st;
    }
    return OSH_OK;
  }
  cudaStream_t gs = ctx->gemm_stream;
  if (osh_status st = wait_input(0); st != OSH_OK) return st;
  OSH_CUDA_TRY(cudaEventRecord(ctx->wave_begin[0], cs));
  if (osh_status st = eng.run_pre(0, cfg, cs); st != OSH_OK) return st;
  OSH_CUDA_TRY(cudaEventRecord(ctx->pre_ev[0], cs));
  for (int w = 0; w < nw; ++w) {
    if (w + 1 < nw) {
      if (osh_status st = wait_input(w + 1); st != OSH_OK) return st;
      if (osh_status st = eng.run_pre(w + 1, cfg, cs); st != OSH_OK) return st;
      OSH_CUDA_TRY(cudaEventRecord(ctx->pre_ev[w + 1], cs));
    }
    OSH_CUDA_TRY(cudaStreamWaitEvent(gs, ctx->pre_ev[w], 0));
    if (osh_status st = eng.run_ns(w, cfg, gs); st != OSH_OK) return st;
    OSH_CUDA_TRY(cudaEventRecord(ctx->ns_ev[w], gs));
    OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->ns_ev[w], 0));
    if (osh_status st = eng.run_post(w, cfg, cs); st != OSH_OK) return st;
    OSH_CUDA_TRY(cudaGetLastError());
    if (osh_status st = wave_done(w); st != OSH_OK) return st;
  }
  return OSH_OK;
}

}  // namespace

extern "C++" {  // (a template inside the C-ABI block)
namespace {

// One stage of the NCCL / TP step: wave `w` of engine `eng` (the DP engine,
// group -1, or micro group `group`'s engine).
struct Stage {
  osh::OptimizerEngine* eng;
  int w, group;
};

// Runs `stages` on cs in order, `before(i)` ahead of stage i's momentum and
// `after(i)` behind its weight update. Overlapped (ctx->seq_overlap): the
// momentum of stage i+1 runs on cs beside the Newton-Schulz GEMMs of stage i
// on the high-priority gemm stream, as run_waves_local does — across engines
// always, within one engine only when it double-buffers its workspace.
template <typename Before, typename After>
osh_status run_stages(osh_ctx* ctx, const osh_muon_cfg& cfg, cudaStream_t cs,
                      const std::vector<Stage>& stages, Before&& before, After&& after) {
  const int n = static_cast<int>(stages.size());
  if (!ctx->seq_overlap) {
    for (int i = 0; i < n; ++i) {
      if (osh_status st = before(i); st != OSH_OK) return st;
      if (osh_status st = stages[i].eng->run_wave(stages[i].w, cfg, cs); st != OSH_OK) return st;
      OSH_CUDA_TRY(cudaGetLastError());
      if (osh_status st = after(i); st != OSH_OK) return st;
    }
    return OSH_OK;
  }
  cudaStream_t gs = ctx->gemm_stream;
  auto pre = [&](int i) -> osh_status {
    if (osh_status st = before(i); st != OSH_OK) return st;
    if (osh_status st = stages[i].eng->run_pre(stages[i].w, cfg, cs); st != OSH_OK) return st;
    OSH_CUDA_TRY(cudaEventRecord(ctx->seq_pre_ev[i & 1], cs));
    return OSH_OK;
  };
  if (n > 0)
    if (osh_status st = pre(0); st != OSH_OK) return st;
  for (int i = 0; i < n; ++i) {
    const Stage& s = stages[static_cast<size_t>(i)];
    const bool early = i + 1 < n && (stages[i + 1].eng != s.eng || s.eng->double_buffered());
    if (early)
      if (osh_status st = pre(i + 1); st != OSH_OK) return st;
    OSH_CUDA_TRY(cudaStreamWaitEvent(gs, ctx->seq_pre_ev[i & 1], 0));
    if (osh_status st = s.eng->run_ns(s.w, cfg, gs); st != OSH_OK) return st;
    OSH_CUDA_TRY(cudaEventRecord(ctx->seq_ns_ev, gs));
    OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->seq_ns_ev, 0));
    if (osh_status st = s.eng->run_post(s.w, cfg, cs); st != OSH_OK) return st;
    OSH_CUDA_TRY(cudaGetLastError());
    if (osh_status st = after(i); st != OSH_OK) return st;
    if (i + 1 < n && !early)
      if (osh_status st = pre(i + 1); st != OSH_OK) return st;
  }
  return OSH_OK;
}

}  // namespace
}  // extern "C++"

osh_status osh_step(osh_ctx* ctx, const osh_muon_cfg* cfg, const void* host_grads,
                    void* host_replica_out) {
  if (osh_status st = check_ctx(ctx, true); st != OSH_OK) return st;
  if (cfg == nullptr) return osh::fail(OSH_ERR_ARG, "null cfg");
  if (ctx->aborted || (ctx->comm_mode == OSH_COMM_NCCL && ctx->size > 1 && ctx->comm == nullptr))
    return osh::fail(OSH_ERR_NCCL, "osh_step: the communicators were aborted by the watchdog");
  const size_t gbytes = grad_esize(ctx->grad_dtype) * static_cast<size_t>(ctx->total_numel);
  const bool dist = distributed(ctx);
  cudaStream_t cs = ctx->compute, ns = ctx->comm_stream;
  OSH_CUDA_TRY(cudaEventRecord(ctx->ev[5], cs));
  // Host I/O. NVLS and TP: whole-buffer copies on cs (a remote owner may read
  // any bucket after the start barrier; TP groups need every shard). Else the
  // gradient arrives bucket by bucket on h2d_stream and each wave / RS waits
  // only for its own buckets; the replica leaves per finished bucket.
  HostIo io;
  const bool pipelined = !ctx->nvls && ctx->tp_size == 1;
  const int n_buckets = static_cast<int>(ctx->cuts.size());
  const bool marked = ctx->n_marked > 0;  // gradients announced per bucket (osh_bucket_ready)
  const int n_marked = ctx->n_marked;
  std::fill(ctx->bucket_marked.begin(), ctx->bucket_marked.end(), 0);  // reset even on error
  ctx->n_marked = 0;
  if (marked && (n_marked != n_buckets || host_grads != nullptr)) {
    if (distributed(ctx) && !ctx->nvls) cudaStreamSynchronize(ctx->comm_stream);  // drain issued RS
    return osh::fail(OSH_ERR_ARG, "osh_step: osh_bucket_ready must cover every bucket (" +
                                      std::to_string(n_marked) + " of " +
                                      std::to_string(n_buckets) + ") and excludes host_grads");
  }
  if (marked) {
    io.h2d = true;  // waves / barriers wait for the announced buckets
  } else if (host_grads != nullptr && pipelined && ctx->wave_io && !distributed(ctx)) {
    // one rank: each wave's own tensors, in execution order (the first wave
    // starts after its bytes, not after whole buckets)
    io.h2d = true;
    io.per_wave = true;
    const size_t ges = grad_esize(ctx->grad_dtype);
    OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->h2d_stream, ctx->ev[5], 0));
    for (size_t w = 0; w < ctx->wave_ranges.size(); ++w) {
      for (const auto& [off, cnt] : ctx->wave_ranges[w])
        OSH_CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(ctx->grad) + ges * static_cast<size_t>(off),
                                     static_cast<const uint8_t*>(host_grads) + ges * static_cast<size_t>(off),
                                     ges * static_cast<size_t>(cnt), cudaMemcpyHostToDevice,
                                     ctx->h2d_stream));
      OSH_CUDA_TRY(cudaEventRecord(ctx->h2d_wave_ev[w], ctx->h2d_stream));
    }
    for (cudaEvent_t e : ctx->h2d_ev) OSH_CUDA_TRY(cudaEventRecord(e, ctx->h2d_stream));  // all landed
    OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->d2h_stream, ctx->ev[5], 0));
  } else if (host_grads != nullptr && pipelined) {
    io.h2d = true;
    OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->h2d_stream, ctx->ev[5], 0));
    for (const int b : ctx->h2d_bucket_order) {  // the order the waves need them
      const size_t off = grad_esize(ctx->grad_dtype) * static_cast<size_t>(ctx->bucket_base[b]);
      const size_t len = grad_esize(ctx->grad_dtype) * static_cast<size_t>(ctx->layout.buckets[b].numel);
      OSH_CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(ctx->grad) + off,
                                   static_cast<const uint8_t*>(host_grads) + off, len,
                                   cudaMemcpyHostToDevice, ctx->h2d_stream));
      OSH_CUDA_TRY(cudaEventRecord(ctx->h2d_ev[b], ctx->h2d_stream));
    }
    OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->d2h_stream, ctx->ev[5], 0));
  } else if (host_grads != nullptr && !ctx->nvls) {  // (NVLS: copied in its branch)
    OSH_CUDA_TRY(cudaMemcpyAsync(ctx->grad, host_grads, gbytes, cudaMemcpyHostToDevice, cs));
  }
  if (host_replica_out != nullptr && pipelined) {
    io.replica_out = host_replica_out;
    io.per_wave = io.per_wave || (ctx->wave_io && !distributed(ctx) && !marked);
  }
  OSH_CUDA_TRY(cudaEventRecord(ctx->ev[0], cs));
  const int nb = static_cast<int>(ctx->cuts.size());
  osh::OptimizerEngine& eng = *ctx->engine;
  const int nw = eng.num_waves();
  if (osh_status st = eng.begin_step(cs); st != OSH_OK) return st;
  auto all_gather = [&](int b) -> osh_status {
    // AG-v of bucket b: every owner broadcasts its updated bf16 slice.
    const auto [o0, o1] = ctx->sched_ag[static_cast<size_t>(b)];
    if (osh_status st = osh::issue_ops(ctx, o0, o1, ns); st != OSH_OK) return st;
    OSH_CUDA_TRY(cudaEventRecord(ctx->ag_ev[b], ns));
    return d2h_buckets(ctx, io, b, ctx->ag_ev[b]);
  };
  int ag_next = 0;
  ctx->last_seq = false;
  // The stage sequence (NCCL RS-v / AG-v path and TP): this rank's DP waves
  // (bucket order), then the micro groups' waves. Hooks around each stage
  // wait for its inputs and release its outputs: a DP wave waits for the RS-v
  // of its buckets and releases the AG-v of the buckets it completes; a micro
  // group waits for its gather and, after its last wave, packs and scatters.
  // (NVLS + TP: no RS-v / AG-v legs, the step barriers bracket the sequence.)
  auto run_seq = [&]() -> osh_status {
    std::vector<Stage> stages;
    for (int w = 0; w < nw; ++w) stages.push_back(Stage{&eng, w, -1});
    for (int g = 0; g < ctx->tp_groups; ++g)
      for (int w = 0; w < ctx->tp_engines[g]->num_waves(); ++w)
        stages.push_back(Stage{ctx->tp_engines[g].get(), w, g});
    if (ctx->tp_size > 1 && nw == 0) OSH_CUDA_TRY(cudaEventRecord(ctx->ev[1], cs));
    auto before = [&](int i) -> osh_status {
      const Stage& s = stages[static_cast<size_t>(i)];
      if (s.group < 0) {
        for (int b = eng.wave_first_bucket(s.w); b <= eng.wave_last_bucket(s.w); ++b) {
          if (dist && !ctx->nvls) OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->rs_ev[b], 0));
          else if (io.h2d) OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->h2d_ev[b], 0));
        }
        OSH_CUDA_TRY(cudaEventRecord(ctx->wave_begin[s.w], cs));
      } else if (s.w == 0) {
        if (s.group == 0) OSH_CUDA_TRY(cudaEventRecord(ctx->tp_begin_ev, cs));
        if (osh_status st = osh::tp_group_begin(ctx, s.group, cs); st != OSH_OK) return st;
      }
      if (i == 0) OSH_CUDA_TRY(cudaEventRecord(ctx->ev[7], cs));
      return OSH_OK;
    };
    auto after = [&](int i) -> osh_status {
      const Stage& s = stages[static_cast<size_t>(i)];
      if (s.group < 0) {
        OSH_CUDA_TRY(cudaEventRecord(ctx->wave_end[s.w], cs));
        if (dist && !ctx->nvls && ctx->tp_size == 1) {
          // buckets no later wave of this rank touches are final on this rank
          const int done = s.w + 1 < nw ? eng.wave_first_bucket(s.w + 1) - 1 : nb - 1;
          if (done >= ag_next) {
            OSH_CUDA_TRY(cudaStreamWaitEvent(ns, ctx->wave_end[s.w], 0));
            for (; ag_next <= done; ++ag_next)
              if (osh_status st = all_gather(ag_next); st != OSH_OK) return st;
          }
        }
        if (ctx->tp_size > 1 && s.w + 1 == nw)  // every DP (non-TP-plane) wave is done
          OSH_CUDA_TRY(cudaEventRecord(ctx->ev[1], cs));
      } else if (s.w + 1 == s.eng->num_waves()) {
        if (osh_status st = osh::tp_group_end(ctx, s.group, cs); st != OSH_OK) return st;
      }
      return OSH_OK;
    };
    if (osh_status st = run_stages(ctx, *cfg, cs, stages, before, after); st != OSH_OK) return st;
    ctx->last_seq = true;
    if (ctx->tp_size > 1) {
      if (osh_status st = osh::tp_finish(ctx, cs); st != OSH_OK) return st;
      OSH_CUDA_TRY(cudaEventRecord(ctx->tp_end_ev, cs));
      if (dist && !ctx->nvls) {
        // AG-v per bucket, in bucket order on every rank, as soon as the DP
        // waves and the last micro group with a TP item in the bucket have
        // scattered — overlapping the remaining groups' Newton-Schulz
        OSH_CUDA_TRY(cudaStreamWaitEvent(ns, ctx->ev[1], 0));
        for (; ag_next < nb; ++ag_next) {
          const int g = ctx->tp_bucket_group[static_cast<size_t>(ag_next)];
          if (g >= 0) OSH_CUDA_TRY(cudaStreamWaitEvent(ns, ctx->tp_scatter_ev[g], 0));
          if (osh_status st = all_gather(ag_next); st != OSH_OK) return st;
        }
      }
    }
    return OSH_OK;
  };
  if (ctx->nvls) {
    // barrier -> waves (reduce / broadcast inside the kernels) -> barrier.
    // With host buffers the barriers go per bucket on the comm stream: bucket b
    // is "in" once every rank's H2D of b landed, and "out" once every owner's
    // multicast stores into b did, so copies overlap the waves.
    auto barrier = [&](cudaStream_t st) -> osh_status {
      OSH_NCCL_TRY(ncclAllReduce(ctx->bar, ctx->bar, 1, ncclFloat32, ncclSum, ctx->comm, st));
      return OSH_OK;
    };
    HostIo nvls_io;
    const bool tp = ctx->tp_size > 1;  // (TP: whole-buffer host copies)
    const bool pipe_in = host_grads != nullptr && !marked && !tp;
    if (pipe_in) {
      OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->h2d_stream, ctx->ev[5], 0));
      OSH_CUDA_TRY(cudaStreamWaitEvent(ns, ctx->ev[5], 0));
      const size_t ges = grad_esize(ctx->grad_dtype);
      for (int b = 0; b < nb; ++b) {
        const size_t off = ges * static_cast<size_t>(ctx->bucket_base[b]);
        const size_t len = ges * static_cast<size_t>(ctx->layout.buckets[b].numel);
        OSH_CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(ctx->grad) + off,
                                     static_cast<const uint8_t*>(host_grads) + off, len,
                                     cudaMemcpyHostToDevice, ctx->h2d_stream));
        OSH_CUDA_TRY(cudaEventRecord(ctx->h2d_ev[b], ctx->h2d_stream));
        OSH_CUDA_TRY(cudaStreamWaitEvent(ns, ctx->h2d_ev[b], 0));
        if (osh_status st = barrier(ns); st != OSH_OK) return st;
        OSH_CUDA_TRY(cudaEventRecord(ctx->rs_ev[b], ns));
      }
      nvls_io.wait_ev = &ctx->rs_ev;
    } else {
      if (host_grads != nullptr)  // (with announced buckets host_grads was rejected above)
        OSH_CUDA_TRY(cudaMemcpyAsync(ctx->grad, host_grads, gbytes, cudaMemcpyHostToDevice, cs));
      if (marked)
        for (int b = 0; b < nb; ++b) OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->h2d_ev[b], 0));
      if (osh_status st = barrier(cs); st != OSH_OK) return st;
      OSH_CUDA_TRY(cudaEventRecord(ctx->rs_ev.back(), cs));
    }
    if (host_replica_out != nullptr && !tp) {
      nvls_io.replica_out = host_replica_out;
      nvls_io.nvls_out = true;
      OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->d2h_stream, ctx->ev[5], 0));
    }
    if (tp) {
      // TP-plane shards: reduced through the multicast address into the
      // owner's local copy, then gathered to the hosts (TP stream), while the
      // DP waves run; each group's scattered shards are re-stored through the
      // replica's multicast address (AG-v) on the TP stream
      if (osh_status st = osh::tp_gather(ctx, {ctx->rs_ev.back()}); st != OSH_OK) return st;
      if (osh_status st = run_seq(); st != OSH_OK) return st;
    } else if (osh_status st = run_waves_local(ctx, *cfg, cs, nvls_io); st != OSH_OK) {
      return st;
    }
    OSH_CUDA_TRY(cudaEventRecord(ctx->ev[2], cs));
    // end barrier on the comm stream (after any per-bucket barriers there)
    OSH_CUDA_TRY(cudaStreamWaitEvent(ns, ctx->ev[2], 0));
    if (osh_status st = barrier(ns); st != OSH_OK) return st;
    OSH_CUDA_TRY(cudaEventRecord(ctx->ev[3], ns));
    OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->ev[3], 0));
    if (host_replica_out != nullptr && tp) {
      OSH_CUDA_TRY(cudaMemcpyAsync(host_replica_out, ctx->replica,
                                   2 * static_cast<size_t>(ctx->total_numel),
                                   cudaMemcpyDeviceToHost, cs));
    } else if (host_replica_out != nullptr) {
      if (osh_status st = d2h_buckets(ctx, nvls_io, nb - 1, ctx->ev[3]); st != OSH_OK) return st;
      OSH_CUDA_TRY(cudaEventRecord(ctx->ev[6], ctx->d2h_stream));
      OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->ev[6], 0));
    }
    OSH_CUDA_TRY(cudaEventRecord(ctx->ev[4], cs));
    ctx->last_h2d_pipelined = pipe_in;
    const osh::NsLaunchStats& s = eng.stats();
    ctx->last_timing.gemm_launches = s.launches_gemm;
    ctx->last_timing.elementwise_launches = s.launches_elementwise;
    ctx->last_timing.gemm_flops = s.gemm_flops;
    for (const auto& e : ctx->tp_engines) {
      ctx->last_timing.gemm_launches += e->stats().launches_gemm;
      ctx->last_timing.elementwise_launches += e->stats().launches_elementwise;
      ctx->last_timing.gemm_flops += e->stats().gemm_flops;
    }
    if (host_replica_out != nullptr) return osh::wait_stream(ctx, cs);
    return OSH_OK;
  }
  if (dist && ctx->strategy != OSH_STRAT_SHARDED) {
    // SC / NV-layerwise baselines: all-reduce every bucket in place, then the
    // waves (each waits for its buckets), then NV-layerwise broadcasts every
    // tensor from its layer owner. Reduction per bucket overlaps the waves.
    if (marked) return osh::fail(OSH_ERR_UNSUPPORTED, "osh_bucket_ready with SC / NV-layerwise");
    OSH_CUDA_TRY(cudaStreamWaitEvent(ns, ctx->ev[0], 0));
    for (int b = 0; b < nb; ++b) {
      if (io.h2d) OSH_CUDA_TRY(cudaStreamWaitEvent(ns, ctx->h2d_ev[b], 0));
      const auto [o0, o1] = ctx->sched_rs[static_cast<size_t>(b)];  // the bucket's AllReduce
      if (osh_status st = osh::issue_ops(ctx, o0, o1, ns); st != OSH_OK) return st;
      OSH_CUDA_TRY(cudaEventRecord(ctx->rs_ev[b], ns));
    }
    HostIo bio;
    bio.wait_ev = &ctx->rs_ev;
    if (ctx->strategy == OSH_STRAT_SC) {  // replica complete locally after each wave
      bio.replica_out = io.replica_out;
      if (bio.replica_out != nullptr)
        OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->d2h_stream, ctx->ev[5], 0));
    }
    if (osh_status st = run_waves_local(ctx, *cfg, cs, bio); st != OSH_OK) return st;
    OSH_CUDA_TRY(cudaEventRecord(ctx->ev[2], cs));
    OSH_CUDA_TRY(cudaStreamWaitEvent(ns, ctx->ev[2], 0));
    if (ctx->strategy == OSH_STRAT_NV_LAYERWISE) {  // every tensor from its layer owner
      const int o0 = ctx->sched_ag.front().first, o1 = ctx->sched_ag.back().second;
      if (osh_status st = osh::issue_ops(ctx, o0, o1, ns); st != OSH_OK) return st;
    }
    OSH_CUDA_TRY(cudaEventRecord(ctx->ev[3], ns));
    OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->ev[3], 0));
    if (io.h2d)
      for (int b = 0; b < nb; ++b) OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->h2d_ev[b], 0));
    if (bio.replica_out != nullptr) {
      if (osh_status st = d2h_buckets(ctx, bio, nb - 1, ctx->ev[3]); st != OSH_OK) return st;
      OSH_CUDA_TRY(cudaEventRecord(ctx->ev[6], ctx->d2h_stream));
      OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->ev[6], 0));
    } else if (host_replica_out != nullptr) {
      OSH_CUDA_TRY(cudaMemcpyAsync(host_replica_out, ctx->replica,
                                   2 * static_cast<size_t>(ctx->total_numel),
                                   cudaMemcpyDeviceToHost, cs));
    }
    OSH_CUDA_TRY(cudaEventRecord(ctx->ev[4], cs));
    ctx->last_h2d_pipelined = io.h2d;
    const osh::NsLaunchStats& s = eng.stats();
    ctx->last_timing.gemm_launches = s.launches_gemm;
    ctx->last_timing.elementwise_launches = s.launches_elementwise;
    ctx->last_timing.gemm_flops = s.gemm_flops;
    if (host_replica_out != nullptr) return osh::wait_stream(ctx, cs);
    return OSH_OK;
  }
  if (dist && !marked) {
    // RS-v, bucket by bucket (osh_bucket_ready issued them already otherwise)
    OSH_CUDA_TRY(cudaStreamWaitEvent(ns, ctx->ev[0], 0));
    for (int b = 0; b < nb; ++b) {
      if (io.h2d) OSH_CUDA_TRY(cudaStreamWaitEvent(ns, ctx->h2d_ev[b], 0));
      if (osh_status st = osh::issue_rs(ctx, b); st != OSH_OK) return st;
    }
  }
  if (ctx->tp_size > 1) {
    // micro-group gathers need every reduced shard of the TP plane: they go
    // out on the TP stream once the whole reduce-scatter (or H2D) landed,
    // overlapping the DP waves below
    std::vector<cudaEvent_t> ready;
    if (dist) ready = ctx->rs_ev;
    else if (io.h2d) ready = ctx->h2d_ev;
    ready.push_back(ctx->ev[0]);
    if (osh_status st = osh::tp_gather(ctx, ready); st != OSH_OK) return st;
  }
  if (!dist && ctx->tp_size == 1) {
    if (osh_status st = run_waves_local(ctx, *cfg, cs, io); st != OSH_OK) return st;
  } else {
    if (osh_status st = run_seq(); st != OSH_OK) return st;
  }
  OSH_CUDA_TRY(cudaEventRecord(ctx->ev[2], cs));
  if (dist) {
    OSH_CUDA_TRY(cudaStreamWaitEvent(ns, ctx->ev[2], 0));
    for (; ag_next < nb; ++ag_next)
      if (osh_status st = all_gather(ag_next); st != OSH_OK) return st;
    OSH_CUDA_TRY(cudaEventRecord(ctx->ev[3], ns));
    OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->ev[3], 0));
  } else {
    OSH_CUDA_TRY(cudaEventRecord(ctx->ev[3], cs));
  }
  if (io.h2d)
    for (int b = 0; b < nb; ++b) OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->h2d_ev[b], 0));
  if (io.replica_out != nullptr) {
    if (osh_status st = d2h_buckets(ctx, io, nb - 1, ctx->ev[3]); st != OSH_OK) return st;
    OSH_CUDA_TRY(cudaEventRecord(ctx->ev[6], ctx->d2h_stream));
    OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->ev[6], 0));
  } else if (host_replica_out != nullptr) {
    OSH_CUDA_TRY(cudaMemcpyAsync(host_replica_out, ctx->replica,
                                 2 * static_cast<size_t>(ctx->total_numel),
                                 cudaMemcpyDeviceToHost, cs));
  }
  OSH_CUDA_TRY(cudaEventRecord(ctx->ev[4], cs));
  ctx->last_h2d_pipelined = io.h2d;
  const osh::NsLaunchStats& s = ctx->engine->stats();
  ctx->last_timing.gemm_launches = s.launches_gemm;
  ctx->last_timing.elementwise_launches = s.launches_elementwise;
  ctx->last_timing.gemm_flops = s.gemm_flops;
  for (const auto& e : ctx->tp_engines) {  // the micro-group engines are part of the step
    ctx->last_timing.gemm_launches += e->stats().launches_gemm;
    ctx->last_timing.elementwise_launches += e->stats().launches_elementwise;
    ctx->last_timing.gemm_flops += e->stats().gemm_flops;
  }
  if (host_replica_out != nullptr) return osh::wait_stream(ctx, cs);
  return OSH_OK;
}

osh_status osh_bucket_ready(osh_ctx* ctx, int32_t bucket, void* stream) {
  if (osh_status st = check_ctx(ctx, true); st != OSH_OK) return st;
  const int nb = static_cast<int>(ctx->cuts.size());
  if (bucket < 0 || bucket >= nb) return osh::fail(OSH_ERR_ARG, "osh_bucket_ready: bucket out of range");
  if (ctx->bucket_marked[bucket])
    return osh::fail(OSH_ERR_ARG, "osh_bucket_ready: bucket marked twice in one step");
  if (ctx->strategy != OSH_STRAT_SHARDED)
    return osh::fail(OSH_ERR_UNSUPPORTED, "osh_bucket_ready needs the sharded strategy");
  cudaStream_t us = stream != nullptr ? static_cast<cudaStream_t>(stream) : ctx->compute;
  OSH_CUDA_TRY(cudaEventRecord(ctx->h2d_ev[bucket], us));  // "gradient of bucket b landed"
  if (distributed(ctx) && !ctx->nvls) {
    // reduce now, overlapping the rest of the backward pass; the previous
    // step must be done with grad_owned first
    OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev[4], 0));
    OSH_CUDA_TRY(cudaStreamWaitEvent(ctx->comm_stream, ctx->h2d_ev[bucket], 0));
    if (osh_status st = osh::issue_rs(ctx, bucket); st != OSH_OK) return st;
  }
  ctx->bucket_marked[bucket] = 1;
  ++ctx->n_marked;
  return OSH_OK;
}

osh_status osh_ctx_sync(osh_ctx* ctx) {
  if (osh_status st = check_ctx(ctx, false); st != OSH_OK) return st;
  if (osh_status st = osh::wait_stream(ctx, ctx->compute); st != OSH_OK) return st;
  if (osh_status st = osh::wait_stream(ctx, ctx->comm_stream); st != OSH_OK) return st;
  if (ctx->aborted) return osh::fail(OSH_ERR_NCCL, "communicators were aborted by the watchdog");
  return OSH_OK;
}

osh_status osh_ctx_set_host_output(osh_ctx* ctx, int32_t mode) {
  if (ctx == nullptr) return osh::fail(OSH_ERR_ARG, "null osh_ctx");
  if (mode != OSH_HOST_OUT_REPLICA && mode != OSH_HOST_OUT_OWNED)
    return osh::fail(OSH_ERR_ARG, "unknown host output mode");
  ctx->host_out_owned = mode == OSH_HOST_OUT_OWNED;
  return OSH_OK;
}

osh_status osh_ctx_set_timeout(osh_ctx* ctx, double seconds) {
  if (ctx == nullptr) return osh::fail(OSH_ERR_ARG, "null osh_ctx");
  if (!(seconds > 0.0)) return osh::fail(OSH_ERR_CONFIG, "timeout must be positive");
  ctx->timeout_s = seconds;
  return OSH_OK;
}

osh_status osh_ctx_comm_schedule(osh_ctx* ctx, osh_coll_op* out, int32_t cap, int32_t* n_out) {
  if (osh_status st = check_ctx(ctx, true); st != OSH_OK) return st;
  const int32_t n = static_cast<int32_t>(ctx->sched.size());
  if (n_out != nullptr) *n_out = n;
  if (out == nullptr) return OSH_OK;
  if (cap < n) return osh::fail(OSH_ERR_ARG, "osh_ctx_comm_schedule: output array too small");
  std::copy(ctx->sched.begin(), ctx->sched.end(), out);
  return OSH_OK;
}

osh_status osh_ctx_stream(osh_ctx* ctx, void** stream) {
  if (osh_status st = check_ctx(ctx, false); st != OSH_OK) return st;
  *stream = ctx->compute;
  return OSH_OK;
}

osh_status osh_ctx_profile_gemm(osh_ctx* ctx, int32_t enable) {
  if (osh_status st = check_ctx(ctx, true); st != OSH_OK) return st;
  ctx->engine->set_profile(enable != 0);
  for (auto& e : ctx->tp_engines) e->set_profile(enable != 0);  // TP micro-group engines too
  return OSH_OK;
}

osh_status osh_gemm_profile_read(osh_ctx* ctx, osh_gemm_profile* out, int32_t reset) {
  if (osh_status st = osh_ctx_sync(ctx); st != OSH_OK) return st;
  if (!ctx->layout_ready) return osh::fail(OSH_ERR_PLAN, "no layout");
  std::memset(out, 0, sizeof(*out));
  int n = 0;
  ctx->engine->read_profile(&n, &out->flops, &out->exec_flops, &out->ms, reset != 0);
  out->launches = n;
  for (auto& e : ctx->tp_engines) {  // the micro-group engines' GEMMs are part of the step
    int k = 0;
    double f = 0.0, x = 0.0, ms = 0.0;
    e->read_profile(&k, &f, &x, &ms, reset != 0);
    out->launches += k;
    out->flops += f;
    out->exec_flops += x;
    out->ms += ms;
  }
  return OSH_OK;
}

osh_status osh_gemm_profile_dump(osh_ctx* ctx, char* buf, size_t cap, size_t* len) {
  if (osh_status st = osh_ctx_sync(ctx); st != OSH_OK) return st;
  if (!ctx->layout_ready) return osh::fail(OSH_ERR_PLAN, "no layout");
  // start offsets relative to the last step's start (ev[5]): a timeline
  // when a single step was profiled
  std::string s = ctx->engine->profile_text(ctx->ev[5]);
  for (auto& e : ctx->tp_engines) s += e->profile_text(ctx->ev[5]);
  if (len != nullptr) *len = s.size();
  if (buf != nullptr && cap > 0) {
    const size_t n = std::min(s.size(), cap - 1);
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return OSH_OK;
}

osh_status osh_last_timing(osh_ctx* ctx, osh_step_timing* out) {
  if (osh_status st = osh_ctx_sync(ctx); st != OSH_OK) return st;
  auto ms = [&](int a, int b) {
    float t = 0.f;
    return cudaEventElapsedTime(&t, ctx->ev[a], ctx->ev[b]) == cudaSuccess ? t : -1.f;
  };
  auto span = [](cudaEvent_t a, cudaEvent_t b) {
    float t = 0.f;
    return cudaEventElapsedTime(&t, a, b) == cudaSuccess ? t : 0.f;
  };
  osh_step_timing t = ctx->last_timing;
  // pipelined host I/O: h2d_ms = until the last bucket landed (overlaps the
  // waves); d2h_ms = the D2H tail after the last wave / all-gather
  t.h2d_ms = ctx->last_h2d_pipelined && !ctx->h2d_ev.empty() ? span(ctx->ev[5], ctx->h2d_ev.back())
                                                              : ms(5, 0);
  const bool dist = distributed(ctx);
  t.rs_ms = dist && !ctx->rs_ev.empty() ? span(ctx->ev[0], ctx->rs_ev.back()) : 0.f;
  t.compute_ms = 0.f;  // busy time of the waves (excludes waiting for the RS)
  if (ctx->last_seq && ctx->seq_overlap) {  // first stage start -> last stage end
    cudaEvent_t end = ctx->tp_size > 1 ? ctx->tp_end_ev
                      : !ctx->wave_end.empty() ? ctx->wave_end.back() : ctx->ev[7];
    t.compute_ms = span(ctx->ev[7], end);
  } else {
    if (ctx->overlap && !ctx->last_seq && !ctx->wave_begin.empty())
      t.compute_ms = span(ctx->wave_begin.front(), ctx->wave_end.back());
    else
      for (size_t w = 0; w < ctx->wave_begin.size(); ++w)
        t.compute_ms += span(ctx->wave_begin[w], ctx->wave_end[w]);
    if (ctx->tp_size > 1 && ctx->tp_begin_ev != nullptr)  // + the micro groups (gathers overlap the waves)
      t.compute_ms += span(ctx->tp_begin_ev, ctx->tp_end_ev);
  }
  t.ag_ms = ms(2, 3);  // all-gather tail exposed after the last wave
  t.d2h_ms = ms(3, 4);
  t.total_ms = ms(5, 4);
  *out = t;
  return OSH_OK;
}

osh_status osh_update_norms(osh_ctx* ctx, double* out) {
  if (osh_status st = osh_ctx_sync(ctx); st != OSH_OK) return st;
  if (!ctx->layout_ready) return osh::fail(OSH_ERR_PLAN, "no layout");
  const int nt = ctx->engine->num_tensors();
  std::vector<double> sq(static_cast<size_t>(std::max(nt, 1)), 0.0);
  if (nt > 0)
    OSH_CUDA_TRY(cudaMemcpy(sq.data(), ctx->engine->update_sq(), sizeof(double) * nt,
                            cudaMemcpyDeviceToHost));
  for (size_t p = 0; p < ctx->params.size(); ++p)
    out[p] = ctx->engine_index[p] >= 0 ? std::sqrt(sq[ctx->engine_index[p]]) : -1.0;
  // TP-plane tensors: the full-matrix update norm, reported by the host rank
  for (const osh_ctx::TpItem& it : ctx->tp_items) {
    if (it.engine_group < 0) continue;
    double v = 0.0;
    OSH_CUDA_TRY(cudaMemcpy(&v, ctx->tp_engines[it.engine_group]->update_sq() + it.engine_index,
                            sizeof(double), cudaMemcpyDeviceToHost));
    out[it.pid] = std::sqrt(v);
  }
  return OSH_OK;
}

osh_status osh_read_param(osh_ctx* ctx, int32_t pid, int32_t which, float* out) {
  if (osh_status st = osh_ctx_sync(ctx); st != OSH_OK) return st;
  if (!ctx->layout_ready || pid < 0 || pid >= static_cast<int32_t>(ctx->params.size()) ||
      out == nullptr)
    return osh::fail(OSH_ERR_PLAN, "osh_read_param: unknown parameter");
  const size_t n = static_cast<size_t>(ctx->params[pid].numel);
  if (which == OSH_READ_REPLICA) {
    std::vector<uint16_t> h(n);
    OSH_CUDA_TRY(cudaMemcpy(h.data(), ctx->replica + ctx->flat_off[pid], 2 * n,
                            cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < n; ++i) {
      const uint32_t bits = static_cast<uint32_t>(h[i]) << 16;
      std::memcpy(out + i, &bits, 4);
    }
    return OSH_OK;
  }
  const int ti = ctx->tp_item_of.empty() ? -1 : ctx->tp_item_of[pid];
  if (ti >= 0 && ctx->tp_items[ti].w != nullptr) {
    // hosted TP-plane tensor: the FULL master / momentum
    const osh_ctx::TpItem& it = ctx->tp_items[ti];
    const float* src = which == OSH_READ_MASTER ? it.w : it.m;
    OSH_CUDA_TRY(cudaMemcpy(out, src, 4 * static_cast<size_t>(it.full_rows * it.full_cols),
                            cudaMemcpyDeviceToHost));
    return OSH_OK;
  }
  if (ctx->owned_off[pid] < 0)
    return osh::fail(OSH_ERR_PLAN, "osh_read_param: parameter " + std::to_string(pid) +
                                       " is owned by dp rank " + std::to_string(ctx->owner[pid]) +
                                       (ti >= 0 ? " / hosted by tp rank " +
                                                      std::to_string(ctx->tp_items[ti].host)
                                                : std::string()));
  const float* src = (which == OSH_READ_MASTER ? ctx->w : ctx->m) + ctx->owned_off[pid];
  OSH_CUDA_TRY(cudaMemcpy(out, src, 4 * n, cudaMemcpyDeviceToHost));
  return OSH_OK;
}

}  // extern "C"

extern "C" {

osh_status osh_write_state(osh_ctx* ctx, int32_t pid, int32_t which, const float* values) {
  if (osh_status st = osh_ctx_sync(ctx); st != OSH_OK) return st;
  if (!ctx->layout_ready || pid < 0 || pid >= static_cast<int32_t>(ctx->params.size()) ||
      values == nullptr || (which != OSH_READ_MASTER && which != OSH_READ_MOMENTUM))
    return osh::fail(OSH_ERR_PLAN, "osh_write_state: bad parameter or target");
  if (ctx->owned_off[pid] < 0)
    return osh::fail(OSH_ERR_PLAN, "osh_write_state: parameter " + std::to_string(pid) +
                                       " is owned by rank " + std::to_string(ctx->owner[pid]));
  float* dst = (which == OSH_READ_MASTER ? ctx->w : ctx->m) + ctx->owned_off[pid];
  OSH_CUDA_TRY(cudaMemcpyAsync(dst, values, 4 * static_cast<size_t>(ctx->params[pid].numel),
                               cudaMemcpyHostToDevice, ctx->compute));
  OSH_CUDA_TRY(cudaStreamSynchronize(ctx->compute));
  return OSH_OK;
}

namespace {

// NS(x) of one matrix on `device` through the step machinery of a one-rank,
// one-tensor context (same kernels as osh_step): momentum 0, beta 0, grad x,
// w 0 and lr = -1 turn "w -= lr * NS(beta*m + g)" into w = NS(x).
osh_status ns_one_matrix(int32_t device, double* x, int64_t rows, int64_t cols,
                         const osh_muon_cfg& base) {
  osh_ctx* ctx = nullptr;
  if (osh_status st = osh_ctx_create(device, 0, 1, OSH_COMM_NONE, nullptr, &ctx); st != OSH_OK)
    return st;
  struct Guard {
    osh_ctx* c;
    ~Guard() { osh_ctx_destroy(c); }
  } guard{ctx};
  osh_param_desc p{};
  p.ndim = 2;
  p.shape[0] = rows;
  p.shape[1] = cols;
  p.dtype_bytes = 4;
  const int64_t n = rows * cols;
  const int64_t cuts[2] = {0, n};
  if (osh_status st = osh_ctx_set_layout(ctx, &p, 1, n, cuts, 1, OSH_GRAD_F32, 0); st != OSH_OK)
    return st;
  std::vector<float> buf(static_cast<size_t>(n), 0.f);
  if (osh_status st = osh_load_param(ctx, 0, buf.data()); st != OSH_OK) return st;  // w = m = 0
  for (int64_t i = 0; i < n; ++i) buf[static_cast<size_t>(i)] = static_cast<float>(x[i]);
  if (osh_status st = osh_write_grad(ctx, 0, buf.data()); st != OSH_OK) return st;
  osh_muon_cfg cfg = base;
  cfg.lr = -1.0;
  cfg.beta = 0.0;
  if (osh_status st = osh_step(ctx, &cfg, nullptr, nullptr); st != OSH_OK) return st;
  if (osh_status st = osh_read_param(ctx, 0, OSH_READ_MASTER, buf.data()); st != OSH_OK) return st;
  for (int64_t i = 0; i < n; ++i) x[i] = buf[static_cast<size_t>(i)];
  return OSH_OK;
}

}  // namespace

// Host-buffer drop-in of muon_apply (verify.hpp:138-147) on the reference's
// fp64 arrays: the momentum and the final axpy are the reference's own fp64
// expressions on the caller's arrays (so the vector and zero-gradient cases
// stay bit-identical to it); the Newton-Schulz orthogonalisation — all of the
// work — runs on the GPU.
osh_status osh_muon_apply_host(int32_t device, const osh_param_desc* p, const osh_muon_cfg* cfg,
                               double* w, double* m, const double* g, double* update_norm) {
  if (p == nullptr || cfg == nullptr || w == nullptr || m == nullptr || g == nullptr)
    return osh::fail(OSH_ERR_ARG, "osh_muon_apply_host: null argument");
  if (p->ndim != 1 && p->ndim != 2) return osh::fail(OSH_ERR_UNSUPPORTED, "params must be 1-D or 2-D");
  const int64_t rows = p->shape[0], cols = p->ndim == 2 ? p->shape[1] : 1;
  if (rows < 1 || cols < 1) return osh::fail(OSH_ERR_ARG, "osh_muon_apply_host: empty tensor");
  const size_t n = static_cast<size_t>(rows * cols);
  for (size_t i = 0; i < n; ++i) m[i] = cfg->beta * m[i] + g[i];
  std::vector<double> upd(m, m + n);
  if (p->ndim == 2)
    if (osh_status st = ns_one_matrix(device, upd.data(), rows, cols, *cfg); st != OSH_OK) return st;
  double sq = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double before = w[i];
    w[i] -= cfg->lr * upd[i];
    sq += (w[i] - before) * (w[i] - before);
  }
  if (update_norm != nullptr) *update_norm = std::sqrt(sq);
  return OSH_OK;
}

osh_status osh_newton_schulz_host(int32_t device, double* x, int64_t rows, int64_t cols,
                                  int32_t steps) {
  if (x == nullptr || rows < 1 || cols < 1) return osh::fail(OSH_ERR_ARG, "bad matrix");
  if (steps < 0) return osh::fail(OSH_ERR_CONFIG, "negative Newton-Schulz step count");
  osh_muon_cfg cfg;
  osh_muon_cfg_default(&cfg);
  cfg.ns_steps = steps;
  return ns_one_matrix(device, x, rows, cols, cfg);
}

}  // extern "C"
