// osh_ctx: one data-parallel rank of the Canzona optimizer step on one B200.
//
// HBM layout:
//   grad    [total_numel]  grad dtype   the rank's local gradient buckets, flat
//                                       in declaration order (bucket i starts at
//                                       the sum of earlier bucket sizes)
//   grad_owned [owned]     grad dtype   (R > 1) this rank's reduced slices, bucket
//                                       after bucket: the ncclReduce root output
//   replica [total_numel]  bf16         the model replica every rank forwards
//                                       with; owners write their slices, the
//                                       all-gather (in-place ncclBroadcast)
//                                       distributes them
//   w, m    [owned, 256 B aligned per tensor]  fp32 master weight + momentum
//   NS workspace (MuonEngine)
// Step = RS-v (per bucket: one ncclReduce per rank slice, grouped) ->
//        MuonEngine waves (owned tensors, bucket order) -> AG-v (per bucket:
//        one ncclBroadcast per rank slice, grouped). Collectives run on a comm
//        stream and overlap the compute stream: wave w waits only for the RS
//        of its last bucket, bucket b is all-gathered as soon as the wave that
//        completes it is done. CUDA events time each phase.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include "comm_schedule.hpp"
#include "ns_engine.cuh"
#include "shampoo_engine.cuh"
#include "soap_engine.cuh"
#include "optishard/optishard.hpp"
#include "osh.h"

struct osh_ctx {
  int device = 0;
  int rank = 0, size = 1;
  int comm_mode = 0;  // OSH_COMM_NCCL or OSH_COMM_NONE (caller reduces; no all-gather)
  ncclComm_t comm = nullptr;
  cudaStream_t compute = nullptr, comm_stream = nullptr;
  cudaStream_t gemm_stream = nullptr;   // high priority: NS GEMMs of overlapped schedules
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;  // osh_step host I/O, per bucket
  std::vector<cudaEvent_t> h2d_ev, ag_ev;  // per bucket: gradient landed / all-gathered
  bool last_h2d_pipelined = false;
  std::vector<char> bucket_marked;     // osh_bucket_ready marks of the coming step
  int n_marked = 0;
  cudaEvent_t ev[8] = {};

  // layout
  std::vector<optishard::ParamSpec> params;
  optishard::BufferLayout layout;
  std::vector<std::vector<int64_t>> cuts;  // [bucket][R+1]
  std::vector<int64_t> flat_off;           // per param: element offset in grad/replica
  std::vector<int64_t> bucket_base;        // per bucket: element offset
  std::vector<int> bucket_of;              // per param
  std::vector<int> owner;                  // per param
  std::vector<int64_t> owned_off;          // per param: offset in w/m (-1: not owned)
  std::vector<int> engine_index;           // per param: tensor index in engine (-1)
  int64_t total_numel = 0, owned_numel = 0, owned_alloc = 0;
  int grad_dtype = 0;

  void* grad = nullptr;
  void* grad_owned = nullptr;              // NCCL mode, R > 1: reduced owned slices
  std::vector<int64_t> owned_slice_off;    // per bucket: offset of this rank's slice in grad_owned
  __nv_bfloat16* replica = nullptr;
  float* w = nullptr;
  float* m = nullptr;
  std::unique_ptr<osh::OptimizerEngine> engine;
  std::vector<cudaEvent_t> rs_ev;       // per bucket: reduce-scatter landed
  std::vector<cudaEvent_t> wave_begin;  // per engine wave
  std::vector<cudaEvent_t> wave_end;
  int min_waves = 0;                    // 0: auto (4 with NCCL or overlap, else 1)
  // overlapped schedule (single rank or NVLS): momentum / apply of adjacent
  // waves run on `compute` while the NS GEMMs of the current wave run on the
  // high-priority gemm_stream (double-buffered NS workspace)
  bool overlap = false;
  std::vector<cudaEvent_t> pre_ev, ns_ev;  // per wave
  // the same overlap for the NCCL RS-v / AG-v path and the TP path, over the
  // stage sequence DP waves -> micro-group waves (osh_step run_stages):
  // momentum of stage i+1 beside the GEMMs of stage i; ev[7] marks the first
  // stage's start (compute_ms = ev[7] -> tp_end_ev / last wave_end)
  bool seq_overlap = false;
  bool last_seq = false;                 // the last step ran the stage sequence
  cudaEvent_t seq_pre_ev[2] = {}, seq_ns_ev = nullptr;
  // waves may run out of bucket order (single rank / NVLS, MuonEngine
  // set_wave_reorder): per wave, the last bucket index B such that every
  // bucket <= B is final once the wave is done; and the order in which a
  // single rank's pipelined H2D copies the buckets (first need first)
  std::vector<int> wave_final_upto;
  std::vector<std::vector<int>> wave_done_buckets;  // per wave: buckets it completes
  std::vector<int> h2d_bucket_order;
  // single rank: per wave, the merged flat element ranges (offset, count) of
  // its tensors; host gradients / replica then move wave by wave (the first
  // wave waits for its own tensors only, the last wave's copy-out is its own)
  bool wave_io = false;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> wave_ranges;
  std::vector<cudaEvent_t> h2d_wave_ev;
  // NVLS-fused collectives (nvls.cu): grad / replica are symmetric windows,
  // the update kernels reduce / broadcast through their multicast addresses
  int coll_mode = 0;                    // OSH_COLL_AUTO / _NCCL / _NVLS
  int optimizer = 0;                    // OSH_OPT_MUON / OSH_OPT_SHAMPOO
  int strategy = 0;                     // OSH_STRAT_SHARDED / _SC / _NV_LAYERWISE
  std::vector<int32_t> layer_of;        // NV_LAYERWISE: layer group per parameter
  optishard::CostModel strategy_cost;
  osh::ShampooConfig shampoo;
  bool nvls = false;
  void* nvls_state = nullptr;
  void* mc_grad = nullptr;              // multicast address of grad
  __nv_bfloat16* mc_replica = nullptr;  // multicast address of replica
  std::string nvls_why;                 // why NVLS is off (diagnostics)
  float* bar = nullptr;                 // 1-element buffer of the step barriers
  // DP collective schedule (comm_schedule.hpp): what the NCCL path issues;
  // per bucket, the [begin, end) op ranges of its RS-v and AG-v legs
  std::vector<osh_coll_op> sched;
  std::vector<std::pair<int, int>> sched_rs, sched_ag;
  bool layout_ready = false;
  osh_step_timing last_timing{};
  // watchdog (osh::wait_stream): host waits poll the streams and the NCCL
  // communicators' async errors; past timeout_s the communicators are
  // aborted and the ctx refuses further collective work
  double timeout_s = 600.0;
  bool aborted = false;
  bool host_out_owned = false;  // osh_step host output: own slices only (OSH_HOST_OUT_OWNED)

  // ---- tensor parallelism: micro-group gather -> host Muon -> scatter
  // (paper Alg. 2; state keyed by (dp owner, tp host) as in
  // the reference run_partitioned, verify.hpp:235-286)
  int tp_rank = 0, tp_size = 1;
  ncclComm_t tp_comm = nullptr;
  cudaStream_t tp_stream = nullptr;       // TP gathers / scatters (overlap the group GEMMs)
  cudaEvent_t tp_start_ev = nullptr, tp_done_ev = nullptr;
  cudaEvent_t tp_begin_ev = nullptr, tp_end_ev = nullptr;  // tp_compute span (compute_ms)
  std::vector<cudaEvent_t> tp_gather_ev, tp_pack_ev, tp_scatter_ev;  // per micro group
  std::vector<int> tp_bucket_group;  // per bucket: last micro group with an item in it (-1)
  uint64_t tp_c_max = 268435456ull;  // 512 MiB of bf16 (optishard_cli.cpp:77-82,198)
  std::vector<optishard::ParamSpec> params_full;  // full shapes; `params` is the shard view
  struct TpItem {
    int pid = 0, group = 0, host = 0;
    int split_dim = 0;               // W dimension split across the TP ranks
    int64_t full_rows = 0, full_cols = 0;
    float* w = nullptr;              // host rank only: full fp32 master
    float* m = nullptr;              //                 full fp32 momentum
    void* g_full = nullptr;          //                 assembled reduced gradient
    __nv_bfloat16* rep_full = nullptr;  //              updated full bf16 matrix
    uint8_t* stage = nullptr;        // column splits: per-peer shard staging (host)
    int engine_group = -1, engine_index = -1;
  };
  std::vector<TpItem> tp_items;      // TP-plane tensors my DP rank owns
  std::vector<int> tp_item_of;       // per param: index in tp_items or -1
  int tp_groups = 0;
  std::vector<std::unique_ptr<osh::MuonEngine>> tp_engines;  // per group (hosted items)
  void* tp_mem = nullptr;
  std::vector<std::vector<osh::CopyTask>> tp_unpack, tp_pack;  // per group (host side)
  std::vector<osh::CopyTask*> d_tp_unpack, d_tp_pack;
  std::vector<long long> tp_unpack_tiles, tp_pack_tiles;
  // NVLS + TP, per group: my shards of its items, reduced through the
  // multicast gradient before the gather / re-stored through the multicast
  // replica after the scatter (same regions, same vector counts)
  std::vector<osh::McReduceTask*> d_tp_mc_reduce;
  std::vector<osh::McCopyTask*> d_tp_mc_copy;
  std::vector<int> tp_mc_tasks;
  std::vector<long long> tp_mc_vecs;
};

namespace osh {
// TP helpers (tp.cu)
osh_status tp_setup(osh_ctx* ctx, int64_t workspace_budget);
// TP step in two halves: tp_gather (TP stream, after `ready`) is issued
// before the DP waves so the gathers overlap them; tp_compute (on cs) runs
// each group's full-matrix Muon after its gather, then packs and scatters.
osh_status tp_gather(osh_ctx* ctx, const std::vector<cudaEvent_t>& ready);
// Per micro group g on cs: tp_group_begin (wait for gather g, unpack the
// full gradients, engine begin_step) before its first wave's momentum;
// tp_group_end (pack the result shards, scatter them on the TP stream) after
// its last wave; tp_finish joins the TP stream back into cs.
osh_status tp_group_begin(osh_ctx* ctx, int g, cudaStream_t cs);
osh_status tp_group_end(osh_ctx* ctx, int g, cudaStream_t cs);
osh_status tp_finish(osh_ctx* ctx, cudaStream_t cs);
osh_status tp_refresh_replica(osh_ctx* ctx, cudaStream_t cs);  // checkpoint resume
void tp_free(osh_ctx* ctx);
void* grad_ptr(osh_ctx* ctx, int pid);
osh_status refresh_replica(osh_ctx* ctx);  // runtime.cu (checkpoint load)
// Waits for `stream` like cudaStreamSynchronize, but polls the ctx's NCCL
// communicators: an async NCCL error, or no completion within
// ctx->timeout_s, aborts them (ncclCommAbort) and returns OSH_ERR_NCCL.
osh_status wait_stream(osh_ctx* ctx, cudaStream_t stream);
cudaError_t cast_to_bf16(const float* src, __nv_bfloat16* dst, long long n, cudaStream_t s);
// NVLS helpers (nvls.cu)
osh_status nvls_setup(osh_ctx* ctx, size_t grad_bytes, size_t replica_bytes, bool required);
void nvls_free(osh_ctx* ctx);
}  // namespace osh
