// optishard (B200 build) — the optimizer half of the reference interface
// (proj/include/optishard/verify.hpp:31-147) executed on sm_100a through the
// C ABI of include/osh.h (link with libosh.so).
//
// Source-compatible surface:
//   OptimizerConfig{lr, beta, ns_steps}                 verify.hpp:31-35
//   newton_schulz_orthogonalize(Matrix x, int steps)    verify.hpp:118-134
//   muon_apply(p, cfg, W, M, G)                          verify.hpp:138-147
// `Matrix` stands in for Eigen::MatrixXd (row-major doubles; Eigen is not a
// dependency of this build). Failures throw the reference exception classes
// (errors.hpp) mapped from osh_status — no exception crosses the C ABI.
//
// The distributed step (run_partitioned executed for real: RS-v -> owner
// Muon -> AG-v over NCCL) is the RAII class DistributedMuon below.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "optishard/errors.hpp"
#include "optishard/model.hpp"
#include "optishard/partition.hpp"
#include "osh.h"

namespace optishard {

struct OptimizerConfig {
  double lr = 0.02;
  double beta = 0.9;
  int ns_steps = 5;
};

// Row-major dense matrix of doubles (vectors: cols == 1).
struct Matrix {
  std::int64_t rows = 0, cols = 0;
  std::vector<double> v;
  Matrix() = default;
  Matrix(std::int64_t r, std::int64_t c) : rows(r), cols(c), v(static_cast<std::size_t>(r * c)) {}
  double& operator()(std::int64_t i, std::int64_t j) { return v[static_cast<std::size_t>(i * cols + j)]; }
  double operator()(std::int64_t i, std::int64_t j) const {
    return v[static_cast<std::size_t>(i * cols + j)];
  }
};

namespace detail {

inline void osh_check(osh_status st) {
  if (st == OSH_OK) return;
  const std::string msg = osh_last_error();
  switch (st) {
    case OSH_ERR_CONFIG: throw ConfigError(msg);
    case OSH_ERR_LAYOUT: throw LayoutError(msg);
    case OSH_ERR_SHARD: throw ShardError(msg);
    case OSH_ERR_UNSUPPORTED: throw UnsupportedError(msg);
    case OSH_ERR_PLAN: throw PlanError(msg);
    case OSH_ERR_UNSCHEDULABLE: throw UnschedulableError(msg);
    case OSH_ERR_FORMAT: throw FormatError(msg);
    default: throw std::runtime_error("osh: " + msg);
  }
}

inline osh_param_desc to_desc(const ParamSpec& p) {
  osh_param_desc d{};
  d.id = p.id;
  d.ndim = static_cast<int32_t>(p.shape.size());
  d.shape[0] = p.shape.at(0);
  d.shape[1] = p.is_matrix() ? p.shape[1] : 0;
  d.dtype_bytes = p.dtype_bytes;
  d.tp_split = p.tp_splittable == TpSplit::kColumn ? 1 : p.tp_splittable == TpSplit::kRow ? 2 : 0;
  d.vocab_space = p.vocab_space ? 1 : 0;
  return d;
}

inline osh_muon_cfg to_cfg(const OptimizerConfig& c) {
  osh_muon_cfg o;
  osh_muon_cfg_default(&o);
  o.lr = c.lr;
  o.beta = c.beta;
  o.ns_steps = c.ns_steps;
  return o;
}

}  // namespace detail

// Quintic Newton-Schulz on the GPU (device 0).
inline Matrix newton_schulz_orthogonalize(Matrix x, int steps, int device = 0) {
  detail::osh_check(osh_newton_schulz_host(device, x.v.data(), x.rows, x.cols, steps));
  return x;
}

// momentum = beta*momentum + grad; matrix: weight -= lr*NS(momentum);
// vector: weight -= lr*momentum. Returns ||weight_new - weight_old||_F.
inline double muon_apply(const ParamSpec& p, const OptimizerConfig& cfg, Matrix& weight,
                         Matrix& momentum, const Matrix& grad, int device = 0) {
  const osh_param_desc d = detail::to_desc(p);
  const osh_muon_cfg c = detail::to_cfg(cfg);
  double norm = 0.0;
  detail::osh_check(osh_muon_apply_host(device, &d, &c, weight.v.data(), momentum.v.data(),
                                        grad.v.data(), &norm));
  return norm;
}

// One data-parallel rank of the distributed step (one object per GPU).
class DistributedMuon {
 public:
  // uid: 128-byte ncclUniqueId from rank 0 (osh_nccl_unique_id) when ranks > 1.
  DistributedMuon(const std::vector<ParamSpec>& params, std::int64_t bucket_capacity,
                  const DpPartitionPlan& plan, int rank, int device, const std::uint8_t* uid,
                  int grad_dtype = OSH_GRAD_BF16, std::int64_t workspace_bytes = 0) {
    detail::osh_check(osh_ctx_create(device, rank, plan.ranks, OSH_COMM_NCCL, uid, &ctx_));
    std::vector<osh_param_desc> d;
    for (const ParamSpec& p : params) d.push_back(detail::to_desc(p));
    std::vector<std::int64_t> cuts;
    for (const auto& c : plan.cut_vectors) cuts.insert(cuts.end(), c.begin(), c.end());
    detail::osh_check(osh_ctx_set_layout(ctx_, d.data(), static_cast<int32_t>(d.size()),
                                         bucket_capacity, cuts.data(),
                                         static_cast<int32_t>(plan.cut_vectors.size()),
                                         grad_dtype, workspace_bytes));
  }
  ~DistributedMuon() { osh_ctx_destroy(ctx_); }
  DistributedMuon(const DistributedMuon&) = delete;
  DistributedMuon& operator=(const DistributedMuon&) = delete;

  // Device pointers of the flat gradient buffer and the bf16 replica.
  std::pair<void*, void*> buffers() const {
    void* g = nullptr;
    void* r = nullptr;
    detail::osh_check(osh_ctx_buffers(ctx_, &g, &r));
    return {g, r};
  }
  void step(const OptimizerConfig& cfg, const void* host_grads = nullptr,
            void* host_replica_out = nullptr) {
    const osh_muon_cfg c = detail::to_cfg(cfg);
    detail::osh_check(osh_step(ctx_, &c, host_grads, host_replica_out));
  }
  void sync() { detail::osh_check(osh_ctx_sync(ctx_)); }
  osh_ctx* handle() const { return ctx_; }

 private:
  osh_ctx* ctx_ = nullptr;
};

}  // namespace optishard
