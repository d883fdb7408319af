// The reference's optimizer-half tests (proj/tests/test_verify.cpp:58-229),
// re-expressed against THIS build's C++ drop-in (include/optishard/muon.hpp +
// libosh.so): the same calls, the same assertions, the GPU underneath.
// Built and run by tests/test_gpu_dropin.py (needs a B200):
//   g++ -std=c++20 -O2 -Iinclude -Ioracle/eigen_shim tests/cpp/muon_dropin.cpp
//       -Lpaper_2602_06079_b200 -losh
// (oracle/eigen_shim: a column-major Eigen::MatrixXd stand-in, so the
// entry points are also exercised with the reference's own matrix type)
//   ./muon_dropin <trace-out.bin>
// Prints one "PASS <case>" / "FAIL <case>: <why>" line per case and exits
// non-zero if any case fails. The replicated toy trace (update norms and
// final weights) is written to argv[1] for the Python side to compare with
// the fp64 oracle.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include <Eigen/Dense>

#include "optishard/muon.hpp"

using namespace optishard;

namespace {

int failures = 0;

void report(const std::string& name, bool ok, const std::string& why = "") {
  std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name.c_str(), ok ? "" : ": ", why.c_str());
  if (!ok) ++failures;
}

void run_case(const std::string& name, const std::function<std::string()>& body) {
  try {
    const std::string why = body();
    report(name, why.empty(), why);
  } catch (const std::exception& e) {
    report(name, false, std::string("exception: ") + e.what());
  }
}

ParamSpec matrix_param(int id, std::int64_t rows, std::int64_t cols) {
  ParamSpec p;
  p.id = id;
  p.name = "m" + std::to_string(id);
  p.shape = {rows, cols};
  p.numel = rows * cols;
  return p;
}

ParamSpec vector_param(int id, std::int64_t n) {
  ParamSpec p;
  p.id = id;
  p.name = "v" + std::to_string(id);
  p.shape = {n};
  p.numel = n;
  return p;
}

ModelConfig toy_config() {  // test_verify.cpp toy_config()
  ModelConfig cfg;
  cfg.name = "toy";
  cfg.num_layers = 2;
  cfg.hidden_size = 8;
  cfg.ffn_size = 16;
  cfg.num_heads = 2;
  cfg.vocab_size = 12;
  cfg.bucket_capacity = 200;
  return cfg;
}

Matrix matmul(const Matrix& a, const Matrix& b) {
  Matrix c(a.rows(), b.cols());
  for (std::int64_t i = 0; i < a.rows(); ++i)
    for (std::int64_t k = 0; k < a.cols(); ++k)
      for (std::int64_t j = 0; j < b.cols(); ++j) c(i, j) += a(i, k) * b(k, j);
  return c;
}

// fills x(i, j) row by row from a generator
template <class Mat, class F>
void fill(Mat& x, F&& next) {
  for (std::int64_t i = 0; i < x.rows(); ++i)
    for (std::int64_t j = 0; j < x.cols(); ++j) x(i, j) = next();
}

// One-sided Jacobi SVD (small matrices): A = U diag(s) V^T, thin.
struct Svd {
  Matrix u, v;
  std::vector<double> s;
};

Svd svd(const Matrix& a_in) {
  const bool tall = a_in.rows() >= a_in.cols();
  Matrix a = tall ? a_in : a_in.transpose();  // work on m >= n
  const std::int64_t m = a.rows(), n = a.cols();
  Matrix v(n, n);
  for (std::int64_t i = 0; i < n; ++i) v(i, i) = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (std::int64_t p = 0; p < n; ++p)
      for (std::int64_t q = p + 1; q < n; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (std::int64_t i = 0; i < m; ++i) {
          alpha += a(i, p) * a(i, p);
          beta += a(i, q) * a(i, q);
          gamma += a(i, p) * a(i, q);
        }
        off = std::max(off, std::abs(gamma) / std::sqrt(std::max(alpha * beta, 1e-300)));
        if (std::abs(gamma) < 1e-300) continue;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (std::int64_t i = 0; i < m; ++i) {
          const double x = a(i, p), y = a(i, q);
          a(i, p) = c * x - s * y;
          a(i, q) = s * x + c * y;
        }
        for (std::int64_t i = 0; i < n; ++i) {
          const double x = v(i, p), y = v(i, q);
          v(i, p) = c * x - s * y;
          v(i, q) = s * x + c * y;
        }
      }
    if (off < 1e-15) break;
  }
  Svd r;
  r.u = Matrix(m, n);
  for (std::int64_t j = 0; j < n; ++j) {
    double nrm = 0;
    for (std::int64_t i = 0; i < m; ++i) nrm += a(i, j) * a(i, j);
    nrm = std::sqrt(nrm);
    r.s.push_back(nrm);
    for (std::int64_t i = 0; i < m; ++i) r.u(i, j) = nrm > 0 ? a(i, j) / nrm : 0.0;
  }
  r.v = v;
  if (!tall) std::swap(r.u, r.v);
  return r;
}

std::string in_band(const std::vector<double>& svs, double lo, double hi) {
  for (const double s : svs)
    if (!(s > lo && s < hi)) return "singular value " + std::to_string(s) + " outside (" +
                                   std::to_string(lo) + ", " + std::to_string(hi) + ")";
  return "";
}

template <class A, class B>
double max_abs(const A& a, const B& b) {
  double m = 0;
  for (std::int64_t i = 0; i < a.rows(); ++i)
    for (std::int64_t j = 0; j < a.cols(); ++j) m = std::max(m, std::abs(a(i, j) - b(i, j)));
  return m;
}

}  // namespace

int main(int argc, char** argv) {
  // test_verify.cpp:58-69
  run_case("identity stays a scalar multiple", [] {
    Matrix x(4, 4);
    for (int i = 0; i < 4; ++i) x(i, i) = 1.0;
    const Matrix y = newton_schulz_orthogonalize(x, 5);
    const double d = y(0, 0);
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j)
        if (std::abs(y(i, j) - (i == j ? d : 0.0)) > 1e-9) return std::string("not a scalar multiple");
    return (d > 0.6 && d < 1.4) ? std::string() : "diagonal " + std::to_string(d);
  });
  // :71-82
  run_case("spread spectrum lands in the unit band", [] {
    Matrix x(2, 2);
    x(0, 0) = 2.0;
    x(1, 1) = 0.5;
    return in_band(svd(newton_schulz_orthogonalize(x, 5)).s, 0.6, 1.4);
  });
  // :84-93 — the same bf16 iterate in both orientations, so exactly equal
  run_case("orthogonalization commutes with transposition", [] {
    detail::NormalStream stream(99);
    Matrix x(3, 7);
    fill(x, [&] { return stream.next(); });
    const Matrix a = newton_schulz_orthogonalize(x, 5);
    const Matrix b = newton_schulz_orthogonalize(x.transpose(), 5);
    const double d = max_abs(a.transpose(), b);
    return d == 0.0 ? std::string() : "max |a^T - b| = " + std::to_string(d);
  });
  // :95-98
  run_case("zero input passes through", [] {
    const Matrix y = newton_schulz_orthogonalize(Matrix(3, 5), 5);
    return max_abs(y, Matrix(3, 5)) == 0.0 ? std::string() : std::string("non-zero output");
  });
  // :100-123
  run_case("well-conditioned inputs land in the band", [] {
    std::mt19937_64 rng(7);
    std::normal_distribution<double> normal;
    for (int trial = 0; trial < 40; ++trial) {
      const int rows = 2 + static_cast<int>(rng() % 5), cols = 2 + static_cast<int>(rng() % 5);
      Matrix x(rows, cols);
      fill(x, [&] { return normal(rng); });
      Svd d = svd(x);  // clamp the spectrum into [0.5, 2]
      const std::int64_t k = static_cast<std::int64_t>(d.s.size());
      Matrix us(d.u.rows(), k);
      for (std::int64_t i = 0; i < d.u.rows(); ++i)
        for (std::int64_t j = 0; j < k; ++j) us(i, j) = d.u(i, j) * std::clamp(d.s[j], 0.5, 2.0);
      x = matmul(us, d.v.transpose());
      const std::string why = in_band(svd(newton_schulz_orthogonalize(x, 5)).s, 0.55, 1.45);
      if (!why.empty()) return "trial " + std::to_string(trial) + ": " + why;
    }
    return std::string();
  });
  // :125-136
  run_case("matrix update magnitude tracks the orthogonal scale", [] {
    const ParamSpec p = matrix_param(0, 8, 8);
    OptimizerConfig cfg;
    Matrix w = init_weight(p, 3), m = Matrix::Zero(8, 8);
    const Matrix before = w;
    muon_apply(p, cfg, w, m, synth_gradient(p, 3, 0, 0));
    Matrix d = w;
    for (std::int64_t i = 0; i < d.rows(); ++i)
      for (std::int64_t j = 0; j < d.cols(); ++j) d(i, j) -= before(i, j);
    const double ideal = cfg.lr * std::sqrt(8.0), n = d.norm();
    return (n > 0.6 * ideal && n < 1.4 * ideal) ? std::string() : "norm " + std::to_string(n);
  });
  // :138-150 — bit-identical to the direct expression
  run_case("vector update is plain momentum descent", [] {
    const ParamSpec p = vector_param(0, 16);
    OptimizerConfig cfg;
    Matrix w = init_weight(p, 3), m = Matrix::Zero(16, 1);
    const Matrix g = synth_gradient(p, 3, 0, 0), before = w;
    muon_apply(p, cfg, w, m, g);
    Matrix expected = before;
    for (std::int64_t i = 0; i < expected.rows(); ++i) expected(i, 0) = before(i, 0) - cfg.lr * g(i, 0);
    return max_abs(w, expected) == 0.0 ? std::string() : std::string("differs");
  });
  // :152-160
  run_case("zero gradient leaves cold state untouched", [] {
    const ParamSpec p = matrix_param(0, 4, 4);
    OptimizerConfig cfg;
    Matrix w = init_weight(p, 3), m = Matrix::Zero(4, 4);
    const Matrix before = w;
    muon_apply(p, cfg, w, m, Matrix::Zero(4, 4));
    return max_abs(w, before) == 0.0 ? std::string() : std::string("weight moved");
  });
  // :162-171
  run_case("synthetic gradients are deterministic and stream-distinct", [] {
    const ParamSpec p = matrix_param(2, 4, 6);
    const Matrix a = synth_gradient(p, 11, 3, 1);
    if (max_abs(a, synth_gradient(p, 11, 3, 1)) != 0.0) return std::string("not deterministic");
    if (max_abs(a, synth_gradient(p, 11, 4, 1)) == 0.0 || max_abs(a, synth_gradient(p, 11, 3, 2)) == 0.0 ||
        max_abs(a, synth_gradient(p, 12, 3, 1)) == 0.0)
      return std::string("streams collide");
    return std::string();
  });
  // :173-183
  VerifyTrace replicated_toy;
  run_case("single-rank partitioned run reproduces the replicated run", [&] {
    const auto params = generate_transformer_params(toy_config());
    const auto layout = build_buffer_layout(params, 200);
    CostModel exec;
    const auto plan = alpha_balanced_partition(layout, params, 1, exec, 1.0);
    OptimizerConfig cfg;
    replicated_toy = run_replicated(params, cfg, 6, 42, 1);
    const auto got = run_partitioned(params, cfg, 6, 42, layout, plan, nullptr);
    const double d = max_abs_diff(replicated_toy, got);
    return d == 0.0 ? std::string() : "max_abs_diff " + std::to_string(d);
  });
  // :185-204
  run_case("sharded 4x2 run matches the replicated trajectory bitwise", [] {
    const auto params = generate_transformer_params(toy_config());
    const auto shards = apply_tp_sharding(params, 2);
    const auto layout = build_buffer_layout(shards, 200);
    CostModel exec;
    const auto dp_plan = alpha_balanced_partition(layout, shards, 4, exec, 1.0);
    const auto tp_plan = build_micro_groups(shards, exec, 2, 1u << 20);
    OptimizerConfig opt;
    const auto ref = run_replicated(shards, opt, 8, 42, dp_plan.ranks);
    const auto got = run_partitioned(shards, opt, 8, 42, layout, dp_plan, &tp_plan);
    const double d = max_abs_diff(ref, got);
    if (d != 0.0) return "max_abs_diff " + std::to_string(d);
    for (const auto& [id, hosts] : got.state_hosts)
      if (hosts.size() != 1) return "param " + std::to_string(id) + " on several hosts";
    return std::string();
  });
  // :206-229
  run_case("a mid-run host reassignment makes the trajectories diverge", [] {
    const auto params = generate_transformer_params(toy_config());
    const auto shards = apply_tp_sharding(params, 2);
    const auto layout = build_buffer_layout(shards, 200);
    CostModel exec;
    const auto dp_plan = alpha_balanced_partition(layout, shards, 4, exec, 1.0);
    const auto tp_plan = build_micro_groups(shards, exec, 2, 1u << 20);
    OptimizerConfig opt;
    const auto ref = run_replicated(shards, opt, 8, 42, dp_plan.ranks);
    FaultSpec fault;
    fault.enabled = true;
    const auto bad = run_partitioned(shards, opt, 8, 42, layout, dp_plan, &tp_plan, fault);
    if (!(max_abs_diff(ref, bad) > 1e-6)) return std::string("fault not detected");
    for (const auto& [id, hosts] : bad.state_hosts)
      if (hosts.size() == 2) return std::string();
    return std::string("no two-host trail");
  });
  // the reference's own matrix type (column-major Eigen::MatrixXd) through
  // the same entry points: identical storage, so bit-identical results
  run_case("Eigen::MatrixXd callers get the same results", [] {
    detail::NormalStream stream(5);
    Matrix x(6, 10);
    Eigen::MatrixXd ex(6, 10);
    fill(x, [&] { return stream.next(); });
    for (std::int64_t i = 0; i < 6; ++i)
      for (std::int64_t j = 0; j < 10; ++j) ex(i, j) = x(i, j);
    if (max_abs(newton_schulz_orthogonalize(x, 5), newton_schulz_orthogonalize(ex, 5)) != 0.0)
      return std::string("newton_schulz_orthogonalize differs");
    const ParamSpec p = matrix_param(0, 6, 10);
    OptimizerConfig cfg;
    Matrix w = init_weight(p, 9), m = Matrix::Zero(6, 10);
    const Matrix g = synth_gradient(p, 9, 0, 0);
    Eigen::MatrixXd ew(6, 10), em = Eigen::MatrixXd::Zero(6, 10), eg(6, 10);
    for (std::int64_t i = 0; i < 6; ++i)
      for (std::int64_t j = 0; j < 10; ++j) {
        ew(i, j) = w(i, j);
        eg(i, j) = g(i, j);
      }
    for (int step = 0; step < 3; ++step) {
      muon_apply(p, cfg, w, m, g);
      muon_apply(p, cfg, ew, em, eg);
    }
    if (max_abs(w, ew) != 0.0 || max_abs(m, em) != 0.0) return std::string("muon_apply differs");
    return std::string();
  });
  // errors cross the ABI as the reference's exception classes
  run_case("shape mismatch raises ShardError", [] {
    const ParamSpec p = matrix_param(0, 4, 4);
    Matrix w(3, 3), m(3, 3), g(3, 3);
    try {
      muon_apply(p, OptimizerConfig{}, w, m, g);
    } catch (const ShardError&) {
      return std::string();
    }
    return std::string("no exception");
  });
  run_case("invalid device raises through the C ABI", [] {
    try {
      newton_schulz_orthogonalize(Matrix(2, 2), 5, 4096);
    } catch (const std::runtime_error&) {
      return std::string();
    }
    return std::string("no exception");
  });

  if (argc > 1 && !replicated_toy.update_norms.empty()) {
    // trace dump: steps, params, then per step per param (id, norm); then per
    // param (id, numel, values...)
    std::FILE* f = std::fopen(argv[1], "wb");
    if (f == nullptr) return 2;
    const double steps = static_cast<double>(replicated_toy.update_norms.size());
    const double np = static_cast<double>(replicated_toy.final_weights.size());
    std::fwrite(&steps, 8, 1, f);
    std::fwrite(&np, 8, 1, f);
    for (const auto& step : replicated_toy.update_norms)
      for (const auto& [id, n] : step) {
        const double rec[2] = {static_cast<double>(id), n};
        std::fwrite(rec, 8, 2, f);
      }
    for (const auto& [id, w] : replicated_toy.final_weights) {  // values row by row
      const double hdr[2] = {static_cast<double>(id), static_cast<double>(w.size())};
      std::fwrite(hdr, 8, 2, f);
      for (std::int64_t i = 0; i < w.rows(); ++i)
        for (std::int64_t j = 0; j < w.cols(); ++j) {
          const double x = w(i, j);
          std::fwrite(&x, 8, 1, f);
        }
    }
    if (std::fclose(f) != 0) return 2;
  }
  std::printf("%d failure(s)\n", failures);
  return failures == 0 ? 0 : 1;
}
