// Tensor-parallel micro-group path (BASELINE.json config C3, SURVEY.md §8
// A11/E2). Each TP-plane tensor (tp-splittable, not vocab-space,
// workload.hpp:153-159) owned by this DP rank is HOSTED whole on one TP rank,
// chosen by build_micro_groups (tp_schedule.hpp:90-131) over the items my DP
// rank owns; the host keeps that tensor's full fp32 master + momentum. Per
// micro group, in plan order:
//   gather : every TP rank sends its reduced-gradient shard to the host (NVLS:
//            first reduced in place through the DP multicast gradient)
//            (row splits land in place; column splits via a staging block)
//   compute: the host runs the full-matrix Muon update (MuonEngine: momentum,
//            5 Newton-Schulz iterations on tcgen05, weight update)
//   scatter: the host sends each TP rank its updated bf16 shard, which lands
//            in that rank's replica slot (the DP all-gather then spreads it)
//            (NVLS: re-stored through the DP multicast replica)
// All TP traffic is NCCL send/recv on the TP communicator, issued on the TP
// stream and ordered by events with the kernels that produce / consume it.
#include <algorithm>
#include <cstring>
#include <string>

#include "runtime.cuh"
#include "status.hpp"

using namespace optishard;

namespace osh {
namespace {

#define TP_NCCL(expr)                                                                           \
  do {                                                                                          \
    ncclResult_t r_ = (expr);                                                                   \
    if (r_ != ncclSuccess)                                                                      \
      return fail(OSH_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_));            \
  } while (0)

size_t gsize(const osh_ctx* ctx) { return ctx->grad_dtype == OSH_GRAD_BF16 ? 2 : 4; }
ncclDataType_t gtype(const osh_ctx* ctx) {
  return ctx->grad_dtype == OSH_GRAD_BF16 ? ncclBfloat16 : ncclFloat32;
}

// Copy task for a (rows x cols) block of `esize`-byte elements, expressed in
// 16-bit units (fp32 = two units).
CopyTask block(const void* src, long long lds, void* dst, long long ldd, int64_t rows, int64_t cols,
               size_t esize) {
  const long long u = static_cast<long long>(esize / 2);
  CopyTask t{};
  t.src = static_cast<const uint16_t*>(src);
  t.dst = static_cast<uint16_t*>(dst);
  t.lds = lds * u;
  t.ldd = ldd * u;
  t.rows = static_cast<int>(rows);
  t.cols = static_cast<int>(cols * u);
  t.tiles_c = (t.cols + kTile - 1) / kTile;
  return t;
}

void finalize_tiles(std::vector<CopyTask>& v, long long* total) {
  long long tiles = 0;
  for (CopyTask& t : v) {
    t.tile_start = tiles;
    tiles += static_cast<long long>((t.rows + kTile - 1) / kTile) * t.tiles_c;
  }
  *total = tiles;
}

template <typename T>
cudaError_t upload_vec(T** dst, const std::vector<T>& src) {
  *dst = nullptr;
  if (src.empty()) return cudaSuccess;
  cudaError_t e = dev_alloc(reinterpret_cast<void**>(dst), sizeof(T) * src.size());
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice);
}

}  // namespace

// Host -> peers: each TP rank's updated bf16 shard of every group-g item
// lands in its replica slot (tp_pack must have run on `st`'s timeline).
osh_status issue_tp_scatter(osh_ctx* ctx, int g, cudaStream_t st) {
  const int T = ctx->tp_size, me = ctx->tp_rank;
  TP_NCCL(ncclGroupStart());
  for (osh_ctx::TpItem& it : ctx->tp_items) {
    if (it.group != g) continue;
    const size_t shard = static_cast<size_t>(it.full_rows * it.full_cols / T);
    if (it.host != me) {
      TP_NCCL(ncclRecv(ctx->replica + ctx->flat_off[it.pid], shard, ncclBfloat16, it.host,
                       ctx->tp_comm, st));
      continue;
    }
    for (int t = 0; t < T; ++t) {
      if (t == me) continue;
      const void* src = it.split_dim == 0
                            ? static_cast<const void*>(it.rep_full + t * shard)
                            : static_cast<const void*>(reinterpret_cast<__nv_bfloat16*>(it.stage) +
                                                       t * shard);
      TP_NCCL(ncclSend(src, shard, ncclBfloat16, t, ctx->tp_comm, st));
    }
  }
  TP_NCCL(ncclGroupEnd());
  return OSH_OK;
}

// The TP-plane part of the replica from the hosts' fp32 masters (checkpoint
// resume): cast every hosted full master, pack each rank's shard and scatter
// it, group by group, all on `cs`.
osh_status tp_refresh_replica(osh_ctx* ctx, cudaStream_t cs) {
  for (osh_ctx::TpItem& it : ctx->tp_items)
    if (it.w != nullptr)
      OSH_CUDA_TRY(cast_to_bf16(it.w, it.rep_full, it.full_rows * it.full_cols, cs));
  for (int g = 0; g < ctx->tp_groups; ++g) {
    OSH_CUDA_TRY(launch_copy_blocks(ctx->d_tp_pack[g], static_cast<int>(ctx->tp_pack[g].size()),
                                    ctx->tp_pack_tiles[g], cs));
    if (osh_status st = issue_tp_scatter(ctx, g, cs); st != OSH_OK) return st;
  }
  return OSH_OK;
}

void* grad_ptr(osh_ctx* ctx, int pid) {
  const size_t es = gsize(ctx);
  if (ctx->grad_owned != nullptr && ctx->owner[pid] == ctx->rank) {
    const int b = ctx->bucket_of[pid];
    const int64_t in_slice = ctx->flat_off[pid] - ctx->bucket_base[b] - ctx->cuts[b][ctx->rank];
    return static_cast<uint8_t*>(ctx->grad_owned) +
           es * static_cast<size_t>(ctx->owned_slice_off[b] + in_slice);
  }
  return static_cast<uint8_t*>(ctx->grad) + es * static_cast<size_t>(ctx->flat_off[pid]);
}

void tp_free(osh_ctx* ctx) {
  if (ctx->tp_stream != nullptr) cudaStreamSynchronize(ctx->tp_stream);
  ctx->tp_engines.clear();
  for (cudaEvent_t e : ctx->tp_gather_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->tp_pack_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->tp_scatter_ev) cudaEventDestroy(e);
  ctx->tp_gather_ev.clear();
  ctx->tp_pack_ev.clear();
  ctx->tp_scatter_ev.clear();
  ctx->tp_bucket_group.clear();
  for (McReduceTask* p : ctx->d_tp_mc_reduce) cudaFree(p);
  for (McCopyTask* p : ctx->d_tp_mc_copy) cudaFree(p);
  ctx->d_tp_mc_reduce.clear();
  ctx->d_tp_mc_copy.clear();
  ctx->tp_mc_tasks.clear();
  ctx->tp_mc_vecs.clear();
  for (CopyTask* p : ctx->d_tp_unpack) cudaFree(p);
  for (CopyTask* p : ctx->d_tp_pack) cudaFree(p);
  ctx->d_tp_unpack.clear();
  ctx->d_tp_pack.clear();
  ctx->tp_unpack.clear();
  ctx->tp_pack.clear();
  cudaFree(ctx->tp_mem);
  ctx->tp_mem = nullptr;
  ctx->tp_items.clear();
  ctx->tp_groups = 0;
}

osh_status tp_setup(osh_ctx* ctx, int64_t budget) {
  const int T = ctx->tp_size, me = ctx->tp_rank;
  const size_t es = gsize(ctx);
  // ---- the micro-group plan over the TP-plane items my DP rank owns (every
  // TP rank of the group computes the same plan: the scheduler is pure)
  std::vector<TpItem> items;
  for (size_t p = 0; p < ctx->params.size(); ++p) {
    const ParamSpec& full = ctx->params_full[p];
    if (ctx->owner[p] != ctx->rank || full.tp_splittable == TpSplit::kNone || full.vocab_space)
      continue;
    items.push_back(TpItem{static_cast<int>(p), static_cast<Cost>(ctx->params[p].numel)});
  }
  MicroGroupPlan plan;
  try {
    plan = build_micro_groups(items, T, ctx->tp_c_max, CostKind::kNumel);
  } catch (const UnschedulableError& e) {
    return fail(OSH_ERR_UNSCHEDULABLE, std::string("tp micro groups: ") + e.what());
  }
  ctx->tp_item_of.assign(ctx->params.size(), -1);
  ctx->tp_groups = static_cast<int>(plan.groups.size());
  // Execution order of the groups (free: they are independent; the same on
  // every TP rank, since all compute the same plan): largest first, so the
  // last group's pack / scatter / AG-v — the step's unhidden TP tail — is the
  // smallest. Group ids below are execution positions.
  std::vector<size_t> order(plan.groups.size());
  std::vector<int64_t> gsize(plan.groups.size(), 0);
  for (size_t g = 0; g < plan.groups.size(); ++g) {
    order[g] = g;
    for (int r = 0; r < T; ++r)
      for (const int pid : plan.groups[g].rank_params[r]) gsize[g] += ctx->params_full[pid].numel;
  }
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return gsize[a] > gsize[b]; });
  for (size_t g = 0; g < plan.groups.size(); ++g)
    for (int r = 0; r < T; ++r)
      for (const int pid : plan.groups[order[g]].rank_params[r]) {
        osh_ctx::TpItem it;
        it.pid = pid;
        it.group = static_cast<int>(g);
        it.host = r;
        const ParamSpec& full = ctx->params_full[pid];
        it.split_dim = full.tp_splittable == TpSplit::kColumn ? 1 : 0;
        it.full_rows = full.shape[0];
        it.full_cols = full.shape[1];
        ctx->tp_item_of[pid] = static_cast<int>(ctx->tp_items.size());
        ctx->tp_items.push_back(it);
      }

  // ---- host-side memory: full state + gradient / result staging
  size_t bytes = 0;
  auto reserve = [&bytes](size_t n) {
    const size_t off = bytes;
    bytes += (n + 255) / 256 * 256;
    return off;
  };
  std::vector<size_t> offs;
  for (const osh_ctx::TpItem& it : ctx->tp_items) {
    if (it.host != me) continue;
    const size_t n = static_cast<size_t>(it.full_rows * it.full_cols);
    offs.push_back(reserve(4 * n));        // w
    offs.push_back(reserve(4 * n));        // m
    offs.push_back(reserve(es * n));       // g_full
    offs.push_back(reserve(2 * n));        // rep_full
    offs.push_back(reserve(it.split_dim == 1 ? std::max(es, size_t{2}) * n : 0));  // staging
  }
  OSH_CUDA_TRY(dev_alloc(&ctx->tp_mem, std::max<size_t>(bytes, 256)));
  OSH_CUDA_TRY(cudaMemset(ctx->tp_mem, 0, std::max<size_t>(bytes, 256)));
  uint8_t* base = static_cast<uint8_t*>(ctx->tp_mem);
  size_t k = 0;
  for (osh_ctx::TpItem& it : ctx->tp_items) {
    if (it.host != me) continue;
    it.w = reinterpret_cast<float*>(base + offs[k++]);
    it.m = reinterpret_cast<float*>(base + offs[k++]);
    it.g_full = base + offs[k++];
    it.rep_full = reinterpret_cast<__nv_bfloat16*>(base + offs[k++]);
    it.stage = base + offs[k++];
  }

  // ---- per group: engine over the hosted full matrices, unpack / pack tables
  ctx->tp_unpack.assign(ctx->tp_groups, {});
  ctx->tp_pack.assign(ctx->tp_groups, {});
  ctx->tp_unpack_tiles.assign(ctx->tp_groups, 0);
  ctx->tp_pack_tiles.assign(ctx->tp_groups, 0);
  for (int g = 0; g < ctx->tp_groups; ++g) {
    std::vector<MuonTensorDesc> tensors;
    for (osh_ctx::TpItem& it : ctx->tp_items) {
      if (it.group != g || it.host != me) continue;
      MuonTensorDesc t;
      t.rows = static_cast<int>(it.full_rows);
      t.cols = static_cast<int>(it.full_cols);
      t.is_matrix = 1;
      t.w = it.w;
      t.m = it.m;
      t.g = it.g_full;
      t.replica = it.rep_full;
      it.engine_group = g;
      it.engine_index = static_cast<int>(tensors.size());
      tensors.push_back(t);
      const int64_t R = it.full_rows, C = it.full_cols;
      const int64_t shard = R * C / T;
      __nv_bfloat16* my_rep = ctx->replica + ctx->flat_off[it.pid];
      const uint8_t* my_grad = static_cast<const uint8_t*>(grad_ptr(ctx, it.pid));
      if (it.split_dim == 0) {
        // own gradient rows -> their place in the full matrix; own result rows -> replica
        ctx->tp_unpack[g].push_back(block(my_grad, C, static_cast<uint8_t*>(it.g_full) + es * me * shard,
                                          C, R / T, C, es));
        ctx->tp_pack[g].push_back(block(it.rep_full + me * shard, C, my_rep, C, R / T, C, 2));
      } else {
        const int64_t cs = C / T;
        for (int t = 0; t < T; ++t) {
          const uint8_t* src = t == me ? my_grad : it.stage + es * static_cast<size_t>(t) * R * cs;
          ctx->tp_unpack[g].push_back(
              block(src, cs, static_cast<uint8_t*>(it.g_full) + es * t * cs, C, R, cs, es));
          // result columns of rank t -> staging (peers) or my replica slot
          __nv_bfloat16* dst = t == me ? my_rep
                                       : reinterpret_cast<__nv_bfloat16*>(it.stage) +
                                             static_cast<size_t>(t) * R * cs;
          ctx->tp_pack[g].push_back(block(it.rep_full + t * cs, C, dst, cs, R, cs, 2));
        }
      }
    }
    finalize_tiles(ctx->tp_unpack[g], &ctx->tp_unpack_tiles[g]);
    finalize_tiles(ctx->tp_pack[g], &ctx->tp_pack_tiles[g]);
    auto eng = std::make_unique<MuonEngine>();
    if (osh_status st = eng->build(tensors, ctx->grad_dtype, static_cast<size_t>(budget), 1,
                                   ctx->seq_overlap);
        st != OSH_OK)
      return st;
    ctx->tp_engines.push_back(std::move(eng));
  }
  ctx->tp_gather_ev.assign(ctx->tp_groups, nullptr);
  ctx->tp_pack_ev.assign(ctx->tp_groups, nullptr);
  ctx->tp_scatter_ev.assign(ctx->tp_groups, nullptr);
  for (int g = 0; g < ctx->tp_groups; ++g) {
    OSH_CUDA_TRY(cudaEventCreateWithFlags(&ctx->tp_gather_ev[g], cudaEventDisableTiming));
    OSH_CUDA_TRY(cudaEventCreateWithFlags(&ctx->tp_pack_ev[g], cudaEventDisableTiming));
    OSH_CUDA_TRY(cudaEventCreateWithFlags(&ctx->tp_scatter_ev[g], cudaEventDisableTiming));
  }
  // a bucket's AG-v may go once the last group with a TP item in it scattered
  ctx->tp_bucket_group.assign(ctx->cuts.size(), -1);
  for (const osh_ctx::TpItem& it : ctx->tp_items) {
    int& g = ctx->tp_bucket_group[static_cast<size_t>(ctx->bucket_of[it.pid])];
    g = std::max(g, it.group);
  }
  for (int g = 0; g < ctx->tp_groups; ++g) {
    CopyTask* u = nullptr;
    CopyTask* p = nullptr;
    OSH_CUDA_TRY(upload_vec(&u, ctx->tp_unpack[g]));
    OSH_CUDA_TRY(upload_vec(&p, ctx->tp_pack[g]));
    ctx->d_tp_unpack.push_back(u);
    ctx->d_tp_pack.push_back(p);
  }
  if (ctx->nvls) {
    // every TP rank of the owning DP rank holds one shard of each item, at
    // the item's flat offset (8-element aligned: the NVLS layout check)
    for (int g = 0; g < ctx->tp_groups; ++g) {
      std::vector<McReduceTask> red;
      std::vector<McCopyTask> cp;
      long long vecs = 0;
      for (const osh_ctx::TpItem& it : ctx->tp_items) {
        if (it.group != g) continue;
        const int64_t off = ctx->flat_off[it.pid], n = ctx->params[it.pid].numel;
        red.push_back(McReduceTask{static_cast<const uint8_t*>(ctx->mc_grad) + es * static_cast<size_t>(off),
                                   static_cast<uint8_t*>(ctx->grad) + es * static_cast<size_t>(off), n, vecs});
        cp.push_back(McCopyTask{ctx->replica + off, ctx->mc_replica + off, n, vecs});
        vecs += n / 8;
      }
      McReduceTask* dr = nullptr;
      McCopyTask* dc = nullptr;
      OSH_CUDA_TRY(upload_vec(&dr, red));
      OSH_CUDA_TRY(upload_vec(&dc, cp));
      ctx->d_tp_mc_reduce.push_back(dr);
      ctx->d_tp_mc_copy.push_back(dc);
      ctx->tp_mc_tasks.push_back(static_cast<int>(red.size()));
      ctx->tp_mc_vecs.push_back(vecs);
    }
  }
  return OSH_OK;
}

// The TP transfers run on their own stream: all gathers are issued first
// (group order) as soon as the reduced gradients exist — they overlap the DP
// waves of the step — the compute of group g waits only for gather g, and
// the scatter of group g follows its pack, so the gathers / scatters of other
// groups overlap the Newton-Schulz GEMMs. Every TP rank issues the same
// collective sequence on tp_comm (gathers 0..G-1, then scatters 0..G-1).
osh_status tp_gather(osh_ctx* ctx, const std::vector<cudaEvent_t>& ready) {
  const int T = ctx->tp_size, me = ctx->tp_rank;
  const size_t es = gsize(ctx);
  cudaStream_t ts = ctx->tp_stream;
  for (cudaEvent_t e : ready) OSH_CUDA_TRY(cudaStreamWaitEvent(ts, e, 0));
  for (int g = 0; g < ctx->tp_groups; ++g) {
    if (ctx->nvls)  // NVLS: my shards' DP sums first (in place, see McReduceTask)
      OSH_CUDA_TRY(launch_mc_reduce(ctx->d_tp_mc_reduce[g], ctx->tp_mc_tasks[g], ctx->tp_mc_vecs[g],
                                    ctx->grad_dtype == OSH_GRAD_BF16, ts));
    // ---- gather reduced-gradient shards to the hosts
    TP_NCCL(ncclGroupStart());
    for (osh_ctx::TpItem& it : ctx->tp_items) {
      if (it.group != g) continue;
      const size_t shard = static_cast<size_t>(it.full_rows * it.full_cols / T);
      if (it.host != me) {
        TP_NCCL(ncclSend(grad_ptr(ctx, it.pid), shard, gtype(ctx), it.host, ctx->tp_comm, ts));
        continue;
      }
      for (int t = 0; t < T; ++t) {
        if (t == me) continue;
        uint8_t* dst = it.split_dim == 0 ? static_cast<uint8_t*>(it.g_full) + es * t * shard
                                         : it.stage + es * t * shard;
        TP_NCCL(ncclRecv(dst, shard, gtype(ctx), t, ctx->tp_comm, ts));
      }
    }
    TP_NCCL(ncclGroupEnd());
    // the hosted full gradients are assembled here too, off the compute stream
    OSH_CUDA_TRY(launch_copy_blocks(ctx->d_tp_unpack[g], static_cast<int>(ctx->tp_unpack[g].size()),
                                    ctx->tp_unpack_tiles[g], ts));
    OSH_CUDA_TRY(cudaEventRecord(ctx->tp_gather_ev[g], ts));
  }
  return OSH_OK;
}

osh_status tp_group_begin(osh_ctx* ctx, int g, cudaStream_t cs) {
  OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->tp_gather_ev[g], 0));  // gathered + unpacked
  return ctx->tp_engines[g]->begin_step(cs);  // the host's full-matrix Muon follows
}

osh_status tp_group_end(osh_ctx* ctx, int g, cudaStream_t cs) {
  // pack, scatter and AG-v of the group on the TP stream: the compute stream
  // goes straight on to the next group
  cudaStream_t ts = ctx->tp_stream;
  OSH_CUDA_TRY(cudaEventRecord(ctx->tp_pack_ev[g], cs));  // the group's update is done
  OSH_CUDA_TRY(cudaStreamWaitEvent(ts, ctx->tp_pack_ev[g], 0));
  OSH_CUDA_TRY(launch_copy_blocks(ctx->d_tp_pack[g], static_cast<int>(ctx->tp_pack[g].size()),
                                  ctx->tp_pack_tiles[g], ts));
  // ---- scatter updated bf16 shards into every rank's replica slot
  if (osh_status st = issue_tp_scatter(ctx, g, ts); st != OSH_OK) return st;
  if (ctx->nvls)  // AG-v of the group's shards: every DP peer's replica slot
    OSH_CUDA_TRY(launch_mc_copy(ctx->d_tp_mc_copy[g], ctx->tp_mc_tasks[g], ctx->tp_mc_vecs[g], ts));
  OSH_CUDA_TRY(cudaEventRecord(ctx->tp_scatter_ev[g], ts));
  return OSH_OK;
}

osh_status tp_finish(osh_ctx* ctx, cudaStream_t cs) {
  OSH_CUDA_TRY(cudaEventRecord(ctx->tp_done_ev, ctx->tp_stream));
  OSH_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->tp_done_ev, 0));
  return OSH_OK;
}

}  // namespace osh
