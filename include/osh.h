/*
 * osh.h — C ABI of the B200-native Canzona optimizer step ("optishard" drop-in).
 *
 * This is the boundary between host code that speaks the reference's C++
 * interface (include/optishard/ headers, namespace optishard) and the sm_100a
 * CUDA library libosh.so. Plain C types only: no C++ or torch types cross it.
 * Every entry point returns an osh_status; on failure osh_last_error() holds
 * a thread-local message. No exception crosses the ABI.
 *
 * Reference interfaces replaced (paths relative to the reference checkout):
 *   status codes          proj/include/optishard/common.hpp:19-60 (exception taxonomy)
 *   osh_layout_build      workload.hpp:164-194   build_buffer_layout
 *   osh_param_cost        cost.hpp:81-90         param_cost
 *   osh_plan_dp           dp_partition.hpp:149-293 equal_chunk / atomic_ownership / alpha_balanced
 *   osh_plan_validate     dp_partition.hpp:297-371 validate_plan
 *   osh_param_owner       dp_partition.hpp:374-395 param_owner
 *   osh_plan_tp           tp_schedule.hpp:90-143 build_micro_groups
 *   osh_plan_*_serialize  serialize.hpp:252-366  serialize_dp_plan / serialize_tp_plan
 *   osh_muon_apply        verify.hpp:138-147     muon_apply (one tensor, host buffers)
 *   osh_newton_schulz     verify.hpp:118-134     newton_schulz_orthogonalize
 *   osh_ctx_* / osh_step  verify.hpp:225-322     run_partitioned, executed for real:
 *                          variable-size reduce-scatter -> owner Muon -> all-gather
 */
#ifndef OSH_H_
#define OSH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OSH_ABI_VERSION 1

typedef enum osh_status {
  OSH_OK = 0,
  OSH_ERR_CONFIG = 1,        /* optishard::ConfigError */
  OSH_ERR_LAYOUT = 2,        /* optishard::LayoutError */
  OSH_ERR_SHARD = 3,         /* optishard::ShardError */
  OSH_ERR_UNSUPPORTED = 4,   /* optishard::UnsupportedError */
  OSH_ERR_PLAN = 5,          /* optishard::PlanError */
  OSH_ERR_UNSCHEDULABLE = 6, /* optishard::UnschedulableError */
  OSH_ERR_FORMAT = 7,        /* optishard::FormatError */
  OSH_ERR_CUDA = 16,
  OSH_ERR_NCCL = 17,
  OSH_ERR_OOM = 18,
  OSH_ERR_ARG = 19
} osh_status;

/* Thread-local message of the last failing call on this thread. */
const char* osh_last_error(void);
int osh_abi_version(void);

/* ------------------------------------------------------------ workload
 * One parameter tensor (ParamSpec, workload.hpp:31-44). ndim is 1 or 2;
 * tp_split: 0 none, 1 column, 2 row (TpSplit, workload.hpp:21). */
typedef struct osh_param_desc {
  int32_t id;
  int32_t ndim;
  int64_t shape[2];
  int32_t dtype_bytes;
  int32_t tp_split;
  int32_t vocab_space;
  int32_t reserved_;
} osh_param_desc;

/* Cost kinds (CostKind, cost.hpp:19). */
enum { OSH_COST_NUMEL = 0, OSH_COST_FLOPS_MUON = 1, OSH_COST_FLOPS_SHAMPOO = 2,
       OSH_COST_FLOPS_SOAP = 3, OSH_COST_BYTES = 4 };
/* Plan methods (PlanMethod, dp_partition.hpp:26). */
enum { OSH_PLAN_EQUAL_CHUNK = 0, OSH_PLAN_ATOMIC_OWNERSHIP = 1, OSH_PLAN_ALPHA_BALANCED = 2 };

typedef struct osh_cost_model {
  int32_t kind;
  int32_t ns_steps;       /* default 5 */
  double shampoo_coeff;   /* default 1.0 */
  double soap_coeff;      /* default 2.0 */
} osh_cost_model;

/* Synthetic transformer parameter list (generate_transformer_params,
 * workload.hpp:113-148). With out == NULL only *n_out is written. */
osh_status osh_generate_params(int32_t num_layers, int64_t hidden, int64_t ffn, int32_t heads,
                               int64_t vocab, int32_t dtype_bytes, osh_param_desc* out,
                               int32_t capacity, int32_t* n_out);

/* Per-tensor planning cost (param_cost, cost.hpp:81-90). */
osh_status osh_param_cost(const osh_param_desc* p, const osh_cost_model* model, uint64_t* out);

/* Greedy declaration-order bucket packing (build_buffer_layout). Outputs, per
 * parameter, its bucket index and element offset inside the bucket, plus
 * per-bucket element counts (bucket_numel must hold n entries). */
osh_status osh_layout_build(const osh_param_desc* params, int32_t n, int64_t bucket_capacity,
                            int32_t* bucket_of, int64_t* offset_in_bucket, int64_t* bucket_numel,
                            int32_t* n_buckets);

/* Data-parallel partition plan. cuts: n_buckets x (ranks+1) int64 (row-major),
 * rank_loads: ranks uint64. *atomic receives the plan's atomic flag. */
osh_status osh_plan_dp(const osh_param_desc* params, int32_t n, int64_t bucket_capacity,
                       int32_t ranks, int32_t method, const osh_cost_model* model, double alpha,
                       int64_t* cuts, uint64_t* rank_loads, int32_t* atomic);

/* Serialized dp plan text ("optishard-dp-plan v1", serialize.hpp:252-271).
 * Writes up to cap bytes (NUL-terminated when room) and the full length. */
osh_status osh_plan_dp_serialize(const osh_param_desc* params, int32_t n, int64_t bucket_capacity,
                                 int32_t ranks, int32_t method, const osh_cost_model* model,
                                 double alpha, char* buf, size_t cap, size_t* len);

/* Owning dp rank of every parameter under an atomic plan (param_owner). */
osh_status osh_param_owners(const osh_param_desc* params, int32_t n, int64_t bucket_capacity,
                            int32_t ranks, const int64_t* cuts, int32_t* owner_out);

/* Micro-group plan text ("optishard-tp-plan v1") for the given items
 * (build_micro_groups(items, ranks, c_max, kind), tp_schedule.hpp:90-131). */
osh_status osh_plan_tp_serialize(const int32_t* item_ids, const uint64_t* item_costs, int32_t n,
                                 int32_t ranks, uint64_t c_max, int32_t cost_kind, char* buf,
                                 size_t cap, size_t* len);

/* ---------------------------------------------------------- optimizer */
typedef struct osh_muon_cfg {
  double lr;        /* 0.02 (OptimizerConfig, verify.hpp:31-35) */
  double beta;      /* 0.9 */
  int32_t ns_steps; /* 5 */
  int32_t reserved_;
  double ns_a, ns_b, ns_c; /* 3.4445, -4.7750, 2.0315 (verify.hpp:120) */
} osh_muon_cfg;

/* Fills cfg with the reference defaults. */
void osh_muon_cfg_default(osh_muon_cfg* cfg);

/* Single-tensor host-buffer drop-ins (fp64 host arrays, row-major, the
 * reference's Eigen::MatrixXd values). Each call runs the GPU path on
 * `device` (a temporary one-rank context): the NS iterate is bf16 with fp32
 * accumulation, so results match the fp64 reference to the tolerance stated
 * in tests/test_gpu_parity.py, not bit for bit.
 *   osh_newton_schulz_host  newton_schulz_orthogonalize (verify.hpp:118-134):
 *                           x (rows x cols) is replaced by its orthogonalisation
 *                           (computed on the GPU; zero input stays zero)
 *   osh_muon_apply_host     muon_apply (verify.hpp:138-147): m = beta*m + g;
 *                           matrix: w -= lr*NS(m); vector: w -= lr*m. The two
 *                           elementwise expressions are the reference's fp64
 *                           ones on the caller's fp64 arrays (vector and zero-
 *                           gradient updates stay bit-identical to it); NS(m)
 *                           runs on the GPU.
 *                           *update_norm (nullable) = ||w_new - w_old||_F
 * These serve the reference's fp64 host-array interface (include/optishard/
 * muon.hpp); the production path is osh_step on device-resident buckets. */
osh_status osh_newton_schulz_host(int32_t device, double* x, int64_t rows, int64_t cols,
                                  int32_t steps);
osh_status osh_muon_apply_host(int32_t device, const osh_param_desc* p, const osh_muon_cfg* cfg,
                               double* w, double* m, const double* g, double* update_norm);

/* ------------------------------------------------ kernel-level entry points
 * Device pointers; `stream` is a cudaStream_t (NULL = legacy default). */
typedef struct osh_matrix_ref {
  const void* ptr;    /* bf16, [batch][rows][ld] */
  int32_t batch, rows, cols;
  int32_t reserved_;
  int64_t ld, bstride;
} osh_matrix_ref;

/* OSH_EPI_FINAL targets: a HOST array of `batch` entries per problem. W and
 * the replica move by TMA: both 16-byte aligned, W's row pitch a multiple of
 * 16 bytes and the replica's too (cols % 4 / % 8 of the stored orientation). */
typedef struct osh_final_target {
  float* w;           /* fp32 master weight, original [rows][cols] (device) */
  void* replica;      /* bf16 replica of the same tensor, nullable (device) */
  double* sq_norm;    /* device; += ||lr*update||^2 (fixed-order sum), nullable */
  int32_t transposed; /* tensor is X^T of the Newton-Schulz iterate */
  int32_t reserved_;
} osh_final_target;

typedef struct osh_gemm_problem {
  osh_matrix_ref a;   /* M x K, K-major */
  osh_matrix_ref b;   /* K-major: N x K ; MN-major: K x N */
  int32_t b_mn_major;
  int32_t reserved_;
  osh_matrix_ref out; /* M x N bf16 (OSH_EPI_STAT: fp32) */
  osh_matrix_ref aux; /* M x N bf16 */
  const float* scale; /* per batch, nullable */
  const osh_final_target* final_targets;
  int32_t symmetric;  /* GRAM / POLY / STAT / SPLIT with M == N: upper-triangle tiles, mirror;
                         2 (STAT only): upper triangle written, lower left untouched;
                         3 (GRAM / POLY / SPLIT): upper-tile form — the 256 x 256 tiles on and above
                         the diagonal (diagonal tiles whole), no mirror of the others */
  int32_t out_seg;    /* OSH_EPI_SPLIT: segment width in elements (>= N) */
  int32_t a_upper;    /* A (square) is in the upper-tile form: left-of-diagonal k-blocks are
                         read from the mirrored tiles (2-CTA launches; else A must be full) */
  int32_t b_upper;    /* likewise for a K-major square B */
} osh_gemm_problem;

/* Epilogues (acc = the fp32 tcgen05 accumulator, s = per-batch scale or 1):
 *   GRAM   out = s*acc               POLY  out = alpha*aux + beta*acc
 *   UPDATE out = s*(alpha*aux + acc) FINAL W -= lr*s*(alpha*aux + acc) (+ replica)
 *   STAT   out(fp32) = alpha*out + s*acc   (Shampoo statistics, read-modify-write)
 *   SPLIT  v = s*acc stored as bf16 hi = bf16(v), lo = bf16(v - hi) in four
 *          segments [hi | lo | hi | hi] of out_seg columns: columns
 *          [0, 3*seg) = (hi, lo, hi) are the A view and [seg, 4*seg) =
 *          (lo, hi, hi) the B view of a bf16x3 product hi*lo + lo*hi + hi*hi
 *          (fp32-accurate Newton iterations).
 * alpha == 0 skips reading aux (aux may then be null). */
enum { OSH_EPI_GRAM = 0, OSH_EPI_POLY = 1, OSH_EPI_UPDATE = 2, OSH_EPI_FINAL = 3,
       OSH_EPI_STAT = 4, OSH_EPI_SPLIT = 5 };

/* UMMA CTA group of subsequent GEMM launches (process-wide): 2 = CTA pairs
 * (tcgen05.mma.cta_group::2, 256x256 tiles; default), 1 = single-CTA
 * 128x256 tiles. The environment variable OSH_GEMM_CTA_GROUP=1 sets 1. */
osh_status osh_set_gemm_cta_group(int32_t cg);
int32_t osh_gemm_cta_group(void);

/* One grouped tcgen05 GEMM launch (the Newton-Schulz building block). */
osh_status osh_ns_gemm(int32_t epilogue, const osh_gemm_problem* problems, int32_t n_problems,
                       float alpha, float beta, float lr, void* stream);

/* ------------------------------------------------------- per-rank runtime
 * One osh_ctx per GPU (one process or host thread per ctx; a ctx is not
 * thread-safe). The ctx owns every device buffer it allocates; host arrays
 * passed in are only borrowed for the duration of the call. Work is ordered on
 * the ctx's own streams; osh_step returns once the step is ENQUEUED unless a
 * host output is requested (osh_ctx_sync waits). */
typedef struct osh_ctx osh_ctx;

enum { OSH_COMM_NCCL = 0, /* real NCCL collectives on the dp communicator     */
       OSH_COMM_NONE = 1  /* no collectives: the caller reduces gradients and
                             reads owned results (single-GPU rank simulation) */ };
enum { OSH_GRAD_F32 = 0, OSH_GRAD_BF16 = 1 };
enum { OSH_READ_MASTER = 0, OSH_READ_MOMENTUM = 1, OSH_READ_REPLICA = 2 };
enum { OSH_FILL_WEIGHTS = 1, OSH_FILL_GRADS = 2 };

/* 128-byte ncclUniqueId for rank 0 to broadcast out of band. */
osh_status osh_nccl_unique_id(uint8_t out[128]);

osh_status osh_ctx_create(int32_t device, int32_t dp_rank, int32_t dp_size, int32_t comm_mode,
                          const uint8_t* nccl_uid /* 128 bytes; unused for OSH_COMM_NONE */,
                          osh_ctx** out);
/* Data x tensor parallel rank (dp_rank, tp_rank) of a dp_size x tp_size grid:
 * dp_uid identifies the DP communicator (the dp_size ranks with this
 * tp_rank), tp_uid the TP communicator (the tp_size ranks with this dp_rank).
 * With tp_size > 1, osh_ctx_set_layout takes the FULL parameter list and the
 * DP plan over the TP-sharded view (apply_tp_sharding, workload.hpp:221);
 * TP-plane tensors are hosted whole on one TP rank by the micro-group plan
 * (tp_schedule.hpp:90-131, c_max from osh_ctx_set_tp_capacity). */
osh_status osh_ctx_create_tp(int32_t device, int32_t dp_rank, int32_t dp_size, int32_t tp_rank,
                             int32_t tp_size, int32_t comm_mode, const uint8_t* dp_uid,
                             const uint8_t* tp_uid, osh_ctx** out);
/* Micro-group capacity in numel cost units (default 268435456 = 512 MiB of
 * bf16, as the reference CLI's plan-tp default). Call before set_layout. */
osh_status osh_ctx_set_tp_capacity(osh_ctx* ctx, uint64_t c_max);
osh_status osh_ctx_destroy(osh_ctx* ctx);

/* How the dp reduce-scatter / all-gather move data (dp_size > 1, tp_size 1).
 * Replaces nothing in the reference (its collectives are simulated); the
 * semantics are SURVEY.md §8 row B4. Call before set_layout.
 *   OSH_COLL_NCCL  NCCL kernels on a comm stream (grouped ncclReduce /
 *                  ncclBroadcast per bucket), overlapped with the waves;
 *   OSH_COLL_NVLS  grad / replica in NCCL symmetric windows; the owner's
 *                  momentum kernels read the cross-rank sum with
 *                  multimem.ld_reduce and its apply kernels write the bf16
 *                  replica to every rank with multimem.st (NVSwitch
 *                  multicast); OSH_ERR_UNSUPPORTED if the node cannot;
 *   OSH_COLL_AUTO  NVLS when available, else NCCL (default). */
enum { OSH_COLL_AUTO = 0, OSH_COLL_NCCL = 1, OSH_COLL_NVLS = 2 };
osh_status osh_ctx_set_collectives(osh_ctx* ctx, int32_t mode);

/* Optimizer run on the owned tensors (call before set_layout).
 *   OSH_OPT_MUON     the Canzona/Muon step (default; verify.hpp:118-147)
 *   OSH_OPT_SHAMPOO  builder-defined blocked Shampoo (the reference only costs
 *                    it: cost.hpp:47-48,68-75 — specification and fp64 oracle
 *                    in oracle/shampoo_oracle.py). osh_step's osh_muon_cfg
 *                    supplies lr and beta (= beta1, momentum); ns_* are unused.
 *   OSH_OPT_SOAP     builder-defined blocked SOAP (Adam in the eigenbasis of
 *                    Shampoo's statistics, basis refreshed by shifted power
 *                    iteration + CholeskyQR2, all on this library's own
 *                    kernels; oracle/soap_oracle.py). The
 *                    osh_shampoo_cfg fields read: beta2 (second moment and
 *                    statistics decay, 0.95), eps (Adam epsilon, 1e-8), block
 *                    (multiple of 64, <= 1024), precond_every, newton_iters =
 *                    power iterations of the first refresh (4). osh_muon_cfg
 *                    supplies lr and beta1.
 * Shampoo and SOAP need tp_size == 1. */
typedef struct osh_shampoo_cfg {
  double beta2;           /* statistics decay (0.95) */
  double eps;             /* relative regularisation of the roots (1e-4) */
  int32_t block;          /* max preconditioner dimension, multiple of 64 (1024) */
  int32_t precond_every;  /* inverse-root refresh period in steps (10) */
  int32_t newton_iters;   /* coupled-Newton iterations per root (16) */
  int32_t reserved;
} osh_shampoo_cfg;
enum { OSH_OPT_MUON = 0, OSH_OPT_SHAMPOO = 1, OSH_OPT_SOAP = 2 };

/* Data-parallel optimizer strategy (simulate.hpp:33-39 made executable, the
 * paper's baselines measured on the GPU). Call before
 * set_layout.
 *   OSH_STRAT_SHARDED       the plan's owners (LB-ASC with an α-balanced plan,
 *                           ASC with an atomic-ownership plan): RS-v, owner
 *                           update, AG-v (default)
 *   OSH_STRAT_SC            replicated: all-reduce the gradients, every rank
 *                           updates every tensor, no redistribution
 *   OSH_STRAT_NV_LAYERWISE  whole-layer ownership by LPT over layer costs
 *                           (layerwise_rank_loads, simulate.hpp:140-157):
 *                           all-reduce the gradients, the owner updates its
 *                           layers, then broadcasts them (kBroadcast
 *                           redistribution, simulate.hpp:58-59)
 * layer_of: per parameter, its layer group id (ids in first-appearance
 * order of the name segment before the first '.', simulate.hpp:130-135);
 * required for NV_LAYERWISE. cost: the execution cost model of the LPT. */
enum { OSH_STRAT_SHARDED = 0, OSH_STRAT_SC = 1, OSH_STRAT_NV_LAYERWISE = 2 };
osh_status osh_ctx_set_strategy(osh_ctx* ctx, int32_t strategy, const int32_t* layer_of,
                                int32_t n, const osh_cost_model* cost);
osh_status osh_shampoo_cfg_default(osh_shampoo_cfg* out);

/* The data-parallel collective schedule of one step (csrc/comm_schedule.hpp):
 * every NCCL operation the runtime issues, in issue order, identical on every
 * rank (NCCL requires it). Replaces the reference's analytic RS-v / AG-v
 * (collective.hpp:49-76, simulate.hpp:199-253) with the executed exchange.
 *   kind   OSH_OP_REDUCE     root receives the sum of [offset, offset+count) of
 *                            every rank's flat gradient buffer at element
 *                            dst_offset of its reduced-slice buffer (RS-v leg)
 *          OSH_OP_BROADCAST  root's [offset, offset+count) of the bf16 replica
 *                            is copied in place to every rank (AG-v leg)
 *          OSH_OP_ALLREDUCE  in-place sum of a whole gradient bucket (SC /
 *                            NV-layerwise baselines; root = -1)
 *   phase  OSH_PHASE_RS (before the update) / OSH_PHASE_AG (after)
 *   group  operations sharing a group id are issued inside one
 *          ncclGroupStart / ncclGroupEnd
 * With the NVLS path the same reduce / broadcast pairs run inside the update
 * kernels (multimem.ld_reduce / multimem.st) instead of as NCCL calls. */
enum { OSH_OP_REDUCE = 0, OSH_OP_BROADCAST = 1, OSH_OP_ALLREDUCE = 2 };
enum { OSH_PHASE_RS = 0, OSH_PHASE_AG = 1 };
typedef struct osh_coll_op {
  int32_t kind, phase, bucket, root, group, reserved_;
  int64_t offset, count, dst_offset;
} osh_coll_op;
/* Pure function of the model, bucket capacity and plan (no GPU needed):
 * the schedule a ctx with this layout and strategy issues. layer_of / cost
 * are read for OSH_STRAT_NV_LAYERWISE only. With out == NULL only *n_out is
 * written; otherwise cap must cover the schedule. */
osh_status osh_comm_schedule(const osh_param_desc* params, int32_t n, int64_t bucket_capacity,
                             int32_t ranks, const int64_t* cuts, int32_t n_buckets,
                             int32_t strategy, const int32_t* layer_of,
                             const osh_cost_model* cost, osh_coll_op* out, int32_t cap,
                             int32_t* n_out);
/* The schedule this ctx issues (empty for a single rank / OSH_COMM_NONE). */
osh_status osh_ctx_comm_schedule(osh_ctx* ctx, osh_coll_op* out, int32_t cap, int32_t* n_out);

osh_status osh_ctx_set_optimizer(osh_ctx* ctx, int32_t kind, const osh_shampoo_cfg* cfg);

/* Installs the parameter list (ids dense 0..n-1, declaration order), the
 * bucket capacity and the dp plan's cut vectors (n_buckets x (dp_size+1),
 * e.g. from osh_plan_dp). The plan must be atomic (whole tensors). Allocates
 * grads, replica, owned fp32 state and the Newton-Schulz workspace
 * (workspace_bytes <= 0: default budget). */
osh_status osh_ctx_set_layout(osh_ctx* ctx, const osh_param_desc* params, int32_t n,
                              int64_t bucket_capacity, const int64_t* cuts, int32_t n_buckets,
                              int32_t grad_dtype, int64_t workspace_bytes);

typedef struct osh_ctx_info {
  int64_t total_numel;     /* elements of the full model */
  int64_t owned_numel;     /* elements this rank updates */
  int32_t n_params, n_owned, n_buckets, n_waves;
  int64_t workspace_bytes; /* Newton-Schulz workspace */
  int64_t device_bytes;    /* everything the ctx allocated */
  double ns_flops_per_iter; /* algorithmic GEMM flops (4m^2n + 2m^3 per owned matrix)
                              of ONE Newton-Schulz iteration on this rank */
  int32_t collectives;      /* 0 none (single rank / OSH_COMM_NONE), OSH_COLL_NCCL
                               or OSH_COLL_NVLS: the path set_layout selected */
  int32_t reserved;
} osh_ctx_info;
osh_status osh_ctx_get_info(osh_ctx* ctx, osh_ctx_info* out);

/* Device pointers of the flat gradient buffer (grad dtype) and bf16 replica,
 * both [total_numel] in declaration order: param p starts at the sum of the
 * numels of params 0..p-1. A training loop writes its gradients here. */
osh_status osh_ctx_buffers(osh_ctx* ctx, void** grad, void** replica);

/* Host fp32 values of one parameter -> replica (every rank) and fp32 master
 * weight (owner only); the owner's momentum is reset to zero. With TP the
 * values are the FULL tensor (each rank keeps its shard in the replica; the
 * host keeps the whole master). */
osh_status osh_load_param(osh_ctx* ctx, int32_t param_id, const float* values);
/* Host fp32 gradient of one parameter -> the flat gradient buffer (with TP:
 * this rank's SHARD of the gradient). */
osh_status osh_write_grad(osh_ctx* ctx, int32_t param_id, const float* values);
/* Device-side synthetic fill (counter-based normal draws * scale / sqrt(rows)):
 * OSH_FILL_WEIGHTS sets replica + owned masters (+ zero momentum),
 * OSH_FILL_GRADS the gradient buffer. For benchmarks. */
osh_status osh_fill_synthetic(osh_ctx* ctx, uint64_t seed, int32_t what, float scale);

/* One distributed Muon step: [H2D host_grads (flat, grad dtype) ->]
 * RS-v -> owner Muon -> AG-v [-> D2H updated replica into host_replica_out].
 * Either host pointer may be NULL (device-resident data). What host_replica_out
 * receives (osh_ctx_set_host_output): OSH_HOST_OUT_REPLICA (default) the
 * whole all-gathered replica; OSH_HOST_OUT_OWNED on a sharded multi-rank ctx
 * only the slices this rank updated (at their flat offsets; the rest of the
 * buffer is left untouched) — the rank's result, copied as soon as its wave
 * finishes, without waiting for the all-gather. */
enum { OSH_HOST_OUT_REPLICA = 0, OSH_HOST_OUT_OWNED = 1 };
osh_status osh_ctx_set_host_output(osh_ctx* ctx, int32_t mode);
osh_status osh_step(osh_ctx* ctx, const osh_muon_cfg* cfg, const void* host_grads,
                    void* host_replica_out);
/* Gradient bucket `bucket` is complete in the grad buffer (its writes were
 * enqueued on `stream`, a cudaStream_t; NULL = the ctx stream). Backward-pass
 * overlap: on the NCCL path the bucket's
 * RS-v starts at once on the comm stream while the caller keeps producing the
 * other buckets; single-rank / NVLS steps wait per bucket. Either announce
 * EVERY bucket (any order, the same order on every rank) before osh_step —
 * which then only waits for them — or none. */
osh_status osh_bucket_ready(osh_ctx* ctx, int32_t bucket, void* stream);
/* Waits for the ctx's streams. Every host wait of the library (this, the
 * host-buffer osh_step, checkpoint resume) is a watchdog: it polls the NCCL
 * communicators' async errors, and when a collective reports an error or does
 * not complete within the timeout (default 600 s, OSH_COMM_TIMEOUT_S or
 * osh_ctx_set_timeout) the communicators are aborted (ncclCommAbort) and the
 * call returns OSH_ERR_NCCL instead of hanging; the ctx then refuses further
 * steps and must be destroyed. */
osh_status osh_ctx_sync(osh_ctx* ctx);
osh_status osh_ctx_set_timeout(osh_ctx* ctx, double seconds);
/* The ctx's compute stream (cudaStream_t): the step's last event is recorded
 * on it, so events recorded here bracket whole steps. */
osh_status osh_ctx_stream(osh_ctx* ctx, void** stream);
/* Optional per-GEMM-launch CUDA-event timing inside osh_step (for roofline
 * reporting); costs two event records per launch. */
osh_status osh_ctx_profile_gemm(osh_ctx* ctx, int32_t enable);
typedef struct osh_gemm_profile {
  int32_t launches;       /* GEMM launches timed since the last reset */
  int32_t reserved_;
  double flops;           /* algorithmic flops of those launches (2MNK)      */
  double exec_flops;      /* flops the tensor cores executed (symmetric GRAM /
                             POLY skip the tiles below the diagonal)           */
  double ms;              /* sum of their CUDA-event durations */
} osh_gemm_profile;
/* Accumulated GEMM timing (synchronises); reset != 0 clears it afterwards. */
osh_status osh_gemm_profile_read(osh_ctx* ctx, osh_gemm_profile* out, int32_t reset);
/* The recorded launches as text, one per line:
 * "<gram|poly|update|final> <ms> <flops> <executed flops> <batch x M x N x K[+...]>".
 * Call before osh_gemm_profile_read(..., reset=1). */
osh_status osh_gemm_profile_dump(osh_ctx* ctx, char* buf, size_t cap, size_t* len);

/* CUDA-event timing of the last step: h2d / d2h = host copies, rs_ms = span
 * of the reduce-scatter (it overlaps the first waves), compute_ms = busy time
 * of the Muon waves (excludes waiting for the RS), ag_ms = all-gather tail
 * left exposed after the last wave, total_ms = the whole step. */
typedef struct osh_step_timing {
  float h2d_ms, rs_ms, compute_ms, ag_ms, d2h_ms, total_ms;
  int32_t gemm_launches, elementwise_launches;
  double gemm_flops;
} osh_step_timing;
/* Timing of the last step (synchronises the ctx's streams). */
osh_status osh_last_timing(osh_ctx* ctx, osh_step_timing* out);

/* ||lr * update||_F of every parameter in the last step (owned params;
 * -1 for params another rank owns). */
osh_status osh_update_norms(osh_ctx* ctx, double* out);
/* One parameter to host fp32 (OSH_READ_MASTER / _MOMENTUM: owner only). */
osh_status osh_read_param(osh_ctx* ctx, int32_t param_id, int32_t which, float* out);
/* Host fp32 values into the owner's master weight or momentum (which =
 * OSH_READ_MASTER / OSH_READ_MOMENTUM; owner only; replica untouched). */
osh_status osh_write_state(osh_ctx* ctx, int32_t param_id, int32_t which, const float* values);

/* Sharded optimizer-state checkpoint keyed by the plan (the
 * reference's plan files, serialize.hpp:252-430, say WHAT a rank owns — this
 * file holds that state). Each rank saves its owned fp32 master + momentum
 * (and hosted TP-plane tensors, and the optimizer's extra state: Shampoo
 * statistics, roots, step counter) behind a header with the rank / world /
 * optimizer and a 64-bit hash of the model shapes and the plan's cut vectors.
 * load_state on a ctx with a different plan, model, rank or optimizer fails
 * with OSH_ERR_FORMAT; on success the owned replica slots are rewritten and
 * the replica all-gathered (tp_size == 1), so training resumes bit-exactly. */
osh_status osh_ctx_save_state(osh_ctx* ctx, const char* path);
osh_status osh_ctx_load_state(osh_ctx* ctx, const char* path);

#ifdef __cplusplus
}
#endif
#endif /* OSH_H_ */
