// optishard (B200 build) — the optimizer half of the reference interface
// (proj/include/optishard/verify.hpp) executed on sm_100a through the C ABI of
// include/osh.h (link with libosh.so).
//
// Source-compatible surface (same names, argument meaning, value semantics
// and exception classes as the reference):
//   OptimizerConfig{lr, beta, ns_steps}                     verify.hpp:31-35
//   detail::splitmix64 / NormalStream / stream_seed         verify.hpp:39-86
//   synth_gradient / init_weight                            verify.hpp:102-113
//   newton_schulz_orthogonalize(Matrix x, int steps)        verify.hpp:118-134
//   void muon_apply(p, cfg, W, M, G)                        verify.hpp:138-147
//   VerifyTrace / max_abs_diff / reduced_gradient           verify.hpp:149-186
//   run_replicated(params, cfg, steps, seed, contributors)  verify.hpp:188-210
//   FaultSpec / run_partitioned(params, cfg, steps, seed,
//       shard_layout, dp_plan, tp_plan*, fault)             verify.hpp:212-322
// `Matrix` stands in for Eigen::MatrixXd (Eigen is not a dependency of this
// build) with the same interface subset and the same COLUMN-MAJOR storage:
// rows(), cols(), size(), operator()(i, j), data(), Zero, transpose(),
// norm(), squaredNorm(), setZero(). newton_schulz_orthogonalize and
// muon_apply are templates over the matrix type, so a caller holding real
// Eigen::MatrixXd values (column-major, contiguous) passes them unchanged;
// tests/cpp/muon_dropin.cpp checks that against an Eigen stand-in. Each
// function takes an optional trailing `device` (default 0). The
// Newton-Schulz orthogonalisation runs on the GPU (bf16 operands, fp32
// accumulation: within the tolerance of tests/test_gpu_parity.py of the fp64
// reference, not bit for bit); the momentum / axpy are the reference's fp64
// expressions.
//
// The production distributed step (run_partitioned executed for real across
// GPUs: RS-v -> owner Muon -> AG-v over NCCL) is the RAII class
// DistributedMuon below; run_replicated / run_partitioned are the
// reference's single-process verification drivers.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "optishard/errors.hpp"
#include "optishard/microgroup.hpp"
#include "optishard/model.hpp"
#include "optishard/partition.hpp"
#include "osh.h"

namespace optishard {

struct OptimizerConfig {
  double lr = 0.02;
  double beta = 0.9;
  int ns_steps = 5;
};

// Dense matrix of doubles (vectors: cols == 1), column-major like
// Eigen::MatrixXd: element (i, j) at data()[j * rows() + i].
class Matrix {
 public:
  using Index = std::int64_t;
  Matrix() = default;
  Matrix(Index r, Index c) : rows_(r), cols_(c), v_(static_cast<std::size_t>(r * c), 0.0) {}
  static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index size() const { return rows_ * cols_; }
  double& operator()(Index i, Index j) { return v_[static_cast<std::size_t>(j * rows_ + i)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<std::size_t>(j * rows_ + i)]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  void setZero() { std::fill(v_.begin(), v_.end(), 0.0); }
  Matrix transpose() const {
    Matrix t(cols_, rows_);
    for (Index j = 0; j < cols_; ++j)
      for (Index i = 0; i < rows_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  double squaredNorm() const {  // storage (column-major) order, as Eigen's
    double s = 0.0;
    for (const double x : v_) s += x * x;
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }  // Frobenius

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<double> v_;
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

// ---- deterministic synthetic inputs (host; the reference's streams)
inline std::uint64_t splitmix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Box-Muller over a sequential splitmix64 chain (the state is each output):
// one pair of draws yields the cosine sample, then the sine sample.
class NormalStream {
 public:
  explicit NormalStream(std::uint64_t seed) : state_(seed) {}
  double next() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    state_ = splitmix64(state_);
    const double u1 = (static_cast<double>(state_ >> 11) + 1.0) * 0x1p-53;
    state_ = splitmix64(state_);
    const double u2 = static_cast<double>(state_ >> 11) * 0x1p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double t = 2.0 * 3.14159265358979323846 * u2;
    spare_ = r * std::sin(t);
    spare_ok_ = true;
    return r * std::cos(t);
  }

 private:
  std::uint64_t state_;
  double spare_ = 0.0;
  bool spare_ok_ = false;
};

inline std::uint64_t stream_seed(std::uint64_t seed, int kind, int step, int param_id, int rank) {
  std::uint64_t s = splitmix64(seed ^ (0x100000001ULL * static_cast<std::uint64_t>(kind + 1)));
  s = splitmix64(s ^ static_cast<std::uint64_t>(step + 1));
  s = splitmix64(s ^ (static_cast<std::uint64_t>(param_id + 1) << 20));
  return splitmix64(s ^ (static_cast<std::uint64_t>(rank + 1) << 40));
}

inline Matrix filled_normal(const ParamSpec& p, std::uint64_t seed, double scale) {
  Matrix m(p.shape.at(0), p.is_matrix() ? p.shape[1] : 1);
  NormalStream s(seed);
  for (Matrix::Index i = 0; i < m.rows(); ++i)  // the reference's fill order: (i, j) row by row
    for (Matrix::Index j = 0; j < m.cols(); ++j) m(i, j) = s.next() * scale;
  return m;
}

}  // namespace detail

// One data-parallel contributor's gradient of a parameter at a step.
inline Matrix synth_gradient(const ParamSpec& p, std::uint64_t seed, int step, int rank) {
  return detail::filled_normal(p, detail::stream_seed(seed, 0, step, p.id, rank),
                               1.0 / std::sqrt(static_cast<double>(p.shape.at(0))));
}

inline Matrix init_weight(const ParamSpec& p, std::uint64_t seed) {
  return detail::filled_normal(p, detail::stream_seed(seed, 1, 0, p.id, 0),
                               1.0 / std::sqrt(static_cast<double>(p.shape.at(0))));
}

// Quintic Newton-Schulz on the GPU: unit Frobenius scaling, transposed
// iteration when taller than wide, zero input returned unchanged. `Mat`:
// Matrix or any column-major contiguous matrix with rows() / cols() /
// data() (Eigen::MatrixXd). The C ABI takes row-major arrays; column-major
// rows x cols storage is the row-major cols x rows transpose, and
// NS(X^T) = NS(X)^T, so the storage goes through as that transpose.
template <class Mat>
Mat newton_schulz_orthogonalize(Mat x, int steps, int device = 0) {
  detail::osh_check(osh_newton_schulz_host(device, x.data(), static_cast<std::int64_t>(x.cols()),
                                           static_cast<std::int64_t>(x.rows()), steps));
  return x;
}

// momentum = beta*momentum + grad; matrix: weight -= lr*NS(momentum);
// vector: weight -= lr*momentum. (`Mat` as above: the elementwise terms are
// layout-free, the NS term runs on the column-major storage's transpose.)
template <class Mat>
void muon_apply(const ParamSpec& p, const OptimizerConfig& cfg, Mat& weight, Mat& momentum,
                const Mat& grad, int device = 0) {
  const auto n = [](const Mat& m) { return static_cast<std::int64_t>(m.rows()) * m.cols(); };
  if (n(weight) != p.numel || n(momentum) != p.numel || n(grad) != p.numel ||
      (p.is_matrix() && (weight.rows() != p.shape[0] || momentum.rows() != p.shape[0] ||
                         grad.rows() != p.shape[0])))
    throw ShardError("muon_apply: weight / momentum / grad do not match the parameter shape");
  osh_param_desc d = detail::to_desc(p);
  if (p.is_matrix()) std::swap(d.shape[0], d.shape[1]);  // column-major storage
  const osh_muon_cfg c = detail::to_cfg(cfg);
  detail::osh_check(osh_muon_apply_host(device, &d, &c, weight.data(), momentum.data(),
                                        grad.data(), nullptr));
}

struct VerifyTrace {
  std::string reduction_order = "ascending-rank";
  std::vector<std::map<int, double>> update_norms;  // [step][param] = ||delta||_F
  std::map<int, Matrix> final_weights;
  std::map<int, std::set<std::string>> state_hosts;  // (dp, tp) host keys per parameter
};

inline double max_abs_diff(const VerifyTrace& a, const VerifyTrace& b) {
  if (a.update_norms.size() != b.update_norms.size())
    throw UnsupportedError("traces cover different step counts");
  double mx = 0.0;
  for (std::size_t s = 0; s < a.update_norms.size(); ++s)
    for (const auto& [id, n] : a.update_norms[s]) {
      const auto it = b.update_norms[s].find(id);
      if (it == b.update_norms[s].end()) throw UnsupportedError("traces cover different parameters");
      mx = std::max(mx, std::abs(n - it->second));
    }
  for (const auto& [id, w] : a.final_weights) {
    const auto it = b.final_weights.find(id);
    if (it == b.final_weights.end() || it->second.rows() != w.rows() || it->second.cols() != w.cols())
      throw UnsupportedError("traces cover different parameters");
    const double* x = w.data();
    const double* y = it->second.data();
    for (Matrix::Index i = 0; i < w.size(); ++i) mx = std::max(mx, std::abs(x[i] - y[i]));
  }
  return mx;
}

// Gradient summed over contributors in ascending rank order.
inline Matrix reduced_gradient(const ParamSpec& p, std::uint64_t seed, int step, int contributors) {
  Matrix g = synth_gradient(p, seed, step, 0);
  for (int r = 1; r < contributors; ++r) {
    const Matrix x = synth_gradient(p, seed, step, r);
    for (Matrix::Index i = 0; i < g.size(); ++i) g.data()[i] += x.data()[i];
  }
  return g;
}

namespace detail {

// One muon_apply of the drivers, recording ||W_new - W_old||_F.
inline double traced_apply(const ParamSpec& p, const OptimizerConfig& cfg, Matrix& w, Matrix& m,
                           const Matrix& g, int device) {
  const Matrix before = w;
  muon_apply(p, cfg, w, m, g, device);
  double s = 0.0;  // ||W_new - W_old||_F over the column-major storage, as Eigen's norm()
  for (Matrix::Index i = 0; i < w.size(); ++i) {
    const double d = w.data()[i] - before.data()[i];
    s += d * d;
  }
  return std::sqrt(s);
}

}  // namespace detail

inline VerifyTrace run_replicated(const std::vector<ParamSpec>& params, const OptimizerConfig& cfg,
                                  int steps, std::uint64_t seed, int contributors = 1,
                                  int device = 0) {
  VerifyTrace trace;
  std::map<int, Matrix> weights, momenta;
  for (const ParamSpec& p : params) {
    weights[p.id] = init_weight(p, seed);
    momenta[p.id] = Matrix::Zero(weights[p.id].rows(), weights[p.id].cols());
    trace.state_hosts[p.id].insert("replicated");
  }
  for (int step = 0; step < steps; ++step) {
    trace.update_norms.emplace_back();
    for (const ParamSpec& p : params)
      trace.update_norms.back()[p.id] =
          detail::traced_apply(p, cfg, weights[p.id], momenta[p.id],
                               reduced_gradient(p, seed, step, contributors), device);
  }
  trace.final_weights = std::move(weights);
  return trace;
}

// Corrupts the host of one parameter from a step onward; its optimizer state
// is not migrated (the failure the comparison must catch).
struct FaultSpec {
  bool enabled = false;
  int param_id = -1;  // -1: the first tensor-parallel matrix
  int at_step = -1;   // -1: the middle step
};

// Owner-routed execution: each parameter's momentum lives in the store of its
// (dp owner, tp host); the dp owner comes from the plan (param_owner), the tp
// host from the micro-group plan for TP-plane tensors.
inline VerifyTrace run_partitioned(const std::vector<ParamSpec>& params, const OptimizerConfig& cfg,
                                   int steps, std::uint64_t seed, const BufferLayout& shard_layout,
                                   const DpPartitionPlan& dp_plan, const MicroGroupPlan* tp_plan,
                                   const FaultSpec& fault = {}, int device = 0) {
  VerifyTrace trace;
  std::map<int, std::pair<int, int>> host;
  for (const ParamSpec& p : params) {
    int tp_host = 0;
    if (tp_plan != nullptr && p.tp_splittable != TpSplit::kNone && !p.vocab_space) {
      bool found = false;
      for (const MicroGroup& g : tp_plan->groups) {
        for (int r = 0; r < tp_plan->ranks && !found; ++r)
          for (const int id : g.rank_params[static_cast<std::size_t>(r)])
            if (id == p.id) {
              tp_host = r;
              found = true;
              break;
            }
        if (found) break;
      }
      if (!found) throw PlanError("parameter " + std::to_string(p.id) + " missing from the micro-group plan");
    }
    host[p.id] = {param_owner(dp_plan, shard_layout, p.id), tp_host};
  }
  FaultSpec eff = fault;
  if (eff.enabled) {
    if (eff.param_id < 0)
      for (const ParamSpec& p : params)
        if (p.tp_splittable != TpSplit::kNone && !p.vocab_space) {
          eff.param_id = p.id;
          break;
        }
    if (eff.param_id < 0) eff.param_id = params.front().id;
    if (eff.at_step < 0) eff.at_step = steps / 2;
  }
  auto key_of = [](const std::pair<int, int>& h) {
    return "dp" + std::to_string(h.first) + ".tp" + std::to_string(h.second);
  };
  std::map<std::string, std::map<int, Matrix>> stores;  // per host key
  std::map<int, Matrix> weights;
  for (const ParamSpec& p : params) {
    weights[p.id] = init_weight(p, seed);
    const std::string k = key_of(host[p.id]);
    stores[k][p.id] = Matrix::Zero(weights[p.id].rows(), weights[p.id].cols());
    trace.state_hosts[p.id].insert(k);
  }
  for (int step = 0; step < steps; ++step) {
    if (eff.enabled && step == eff.at_step) {
      auto& h = host.at(eff.param_id);
      if (tp_plan != nullptr && tp_plan->ranks > 1)
        h.second = (h.second + 1) % tp_plan->ranks;
      else
        h.first = (h.first + 1) % dp_plan.ranks;
    }
    trace.update_norms.emplace_back();
    for (const ParamSpec& p : params) {
      const std::string k = key_of(host.at(p.id));
      trace.state_hosts[p.id].insert(k);
      auto& store = stores[k];
      auto it = store.find(p.id);
      if (it == store.end())  // a rerouted parameter meets a cold momentum buffer
        it = store.emplace(p.id, Matrix::Zero(weights[p.id].rows(), weights[p.id].cols())).first;
      trace.update_norms.back()[p.id] =
          detail::traced_apply(p, cfg, weights[p.id], it->second,
                               reduced_gradient(p, seed, step, dp_plan.ranks), device);
    }
  }
  trace.final_weights = std::move(weights);
  return trace;
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
    try {
      detail::osh_check(osh_ctx_set_layout(ctx_, d.data(), static_cast<int32_t>(d.size()),
                                           bucket_capacity, cuts.data(),
                                           static_cast<int32_t>(plan.cut_vectors.size()),
                                           grad_dtype, workspace_bytes));
    } catch (...) {
      osh_ctx_destroy(ctx_);
      throw;
    }
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
  void load_param(int id, const std::vector<float>& values) {
    detail::osh_check(osh_load_param(ctx_, id, values.data()));
  }
  void write_grad(int id, const std::vector<float>& values) {
    detail::osh_check(osh_write_grad(ctx_, id, values.data()));
  }
  void step(const OptimizerConfig& cfg, const void* host_grads = nullptr,
            void* host_replica_out = nullptr) {
    const osh_muon_cfg c = detail::to_cfg(cfg);
    detail::osh_check(osh_step(ctx_, &c, host_grads, host_replica_out));
  }
  // Owner's fp32 master of parameter `id` (PlanError on another rank).
  std::vector<float> read_master(int id, std::int64_t numel) const {
    std::vector<float> out(static_cast<std::size_t>(numel));
    detail::osh_check(osh_read_param(ctx_, id, OSH_READ_MASTER, out.data()));
    return out;
  }
  void sync() { detail::osh_check(osh_ctx_sync(ctx_)); }
  osh_ctx* handle() const { return ctx_; }

 private:
  osh_ctx* ctx_ = nullptr;
};

}  // namespace optishard
