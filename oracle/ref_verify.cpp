// Runs the REFERENCE Muon CPU path (proj/include/optishard/verify.hpp,
// compiled unmodified against oracle/eigen_shim) and prints golden vectors
// (TEST INFRASTRUCTURE ONLY; output -> tests/golden/verify_vectors.txt).
// Every double is printed with %.17g so it round-trips exactly.
#include <cstdio>
#include <string>
#include <vector>

#include "optishard/dp_partition.hpp"
#include "optishard/tp_schedule.hpp"
#include "optishard/verify.hpp"
#include "optishard/workload.hpp"

using namespace optishard;

namespace {

void put(const std::string& key, const Eigen::MatrixXd& m) {
  std::printf("%s %td %td", key.c_str(), m.rows(), m.cols());
  for (Eigen::Index i = 0; i < m.rows(); ++i)
    for (Eigen::Index j = 0; j < m.cols(); ++j) std::printf(" %.17g", m(i, j));
  std::printf("\n");
}

ParamSpec mat(int id, std::int64_t r, std::int64_t c) {
  ParamSpec p;
  p.id = id;
  p.name = "m" + std::to_string(id);
  p.shape = {r, c};
  p.numel = r * c;
  return p;
}

ParamSpec vec(int id, std::int64_t n) {
  ParamSpec p;
  p.id = id;
  p.name = "v" + std::to_string(id);
  p.shape = {n};
  p.numel = n;
  return p;
}

ModelConfig toy(int layers) {
  ModelConfig c;
  c.name = "toy";
  c.num_layers = layers;
  c.hidden_size = 8;
  c.ffn_size = 16;
  c.num_heads = 2;
  c.vocab_size = 12;
  c.bucket_capacity = 200;
  return c;
}

void put_trace(const std::string& key, const VerifyTrace& t) {
  for (std::size_t s = 0; s < t.update_norms.size(); ++s) {
    std::printf("%s.norms %zu", key.c_str(), s);
    for (const auto& [id, n] : t.update_norms[s]) std::printf(" %d:%.17g", id, n);
    std::printf("\n");
  }
  for (const auto& [id, w] : t.final_weights) put(key + ".w" + std::to_string(id), w);
}

}  // namespace

int main() {
  // 1) deterministic input streams (verify.hpp:39-113)
  put("grad.m2_4x6.s11.t3.r1", synth_gradient(mat(2, 4, 6), 11, 3, 1));
  put("grad.m7_5x3.s42.t0.r0", synth_gradient(mat(7, 5, 3), 42, 0, 0));
  put("grad.v3_9.s42.t2.r5", synth_gradient(vec(3, 9), 42, 2, 5));
  put("init.m1_6x4.s42", init_weight(mat(1, 6, 4), 42));
  put("init.v0_7.s3", init_weight(vec(0, 7), 3));
  std::printf("seed %llu\n",
              static_cast<unsigned long long>(detail::stream_seed(42, 0, 3, 17, 5)));
  {
    detail::NormalStream s(99);
    std::printf("stream99");
    for (int i = 0; i < 9; ++i) std::printf(" %.17g", s.next());
    std::printf("\n");
  }
  // 2) Newton-Schulz (verify.hpp:118-134)
  put("ns.identity4", newton_schulz_orthogonalize(Eigen::MatrixXd::Identity(4, 4), 5));
  {
    Eigen::MatrixXd d = Eigen::MatrixXd::Zero(2, 2);
    d(0, 0) = 2.0;
    d(1, 1) = 0.5;
    put("ns.diag2", newton_schulz_orthogonalize(d, 5));
  }
  {
    detail::NormalStream s(99);
    Eigen::MatrixXd x(3, 7);
    for (Eigen::Index i = 0; i < 3; ++i)
      for (Eigen::Index j = 0; j < 7; ++j) x(i, j) = s.next();
    put("ns.rand3x7", newton_schulz_orthogonalize(x, 5));
    put("ns.rand7x3", newton_schulz_orthogonalize(x.transpose(), 5));
    put("ns.rand3x7.k1", newton_schulz_orthogonalize(x, 1));
  }
  put("ns.grad20x12", newton_schulz_orthogonalize(synth_gradient(mat(4, 20, 12), 5, 1, 0), 5));
  // 3) muon_apply (verify.hpp:138-147), 3 steps on one matrix and one vector
  for (const ParamSpec& p : {mat(0, 8, 8), mat(9, 24, 10), vec(5, 16)}) {
    OptimizerConfig cfg;
    Eigen::MatrixXd w = init_weight(p, 3);
    Eigen::MatrixXd m = Eigen::MatrixXd::Zero(w.rows(), w.cols());
    for (int step = 0; step < 3; ++step) muon_apply(p, cfg, w, m, synth_gradient(p, 3, step, 0));
    put("muon." + p.name + ".w", w);
    put("muon." + p.name + ".m", m);
  }
  // 4) drivers (verify.hpp:180-322) on the toy model
  {
    const auto params = generate_transformer_params(toy(2));
    const auto layout = build_buffer_layout(params, 200);
    CostModel numel;
    const auto plan = alpha_balanced_partition(layout, params, 1, numel, 1.0);
    OptimizerConfig opt;
    put_trace("rep.toy.c1", run_replicated(params, opt, 6, 42, 1));
    const auto got = run_partitioned(params, opt, 6, 42, layout, plan, nullptr);
    std::printf("part.toy.r1.diff %.17g\n", max_abs_diff(run_replicated(params, opt, 6, 42, 1), got));
  }
  {
    const auto params = apply_tp_sharding(generate_transformer_params(toy(2)), 2);
    const auto layout = build_buffer_layout(params, 200);
    CostModel numel;
    const auto dp = alpha_balanced_partition(layout, params, 4, numel, 1.0);
    const auto tp = build_micro_groups(params, numel, 2, 1u << 20);
    OptimizerConfig opt;
    const auto ref = run_replicated(params, opt, 8, 42, 4);
    put_trace("rep.toytp2.c4", ref);
    std::printf("part.toytp2.diff %.17g\n",
                max_abs_diff(ref, run_partitioned(params, opt, 8, 42, layout, dp, &tp)));
    FaultSpec f;
    f.enabled = true;
    const auto bad = run_partitioned(params, opt, 8, 42, layout, dp, &tp, f);
    std::printf("part.toytp2.fault.diff %.17g\n", max_abs_diff(ref, bad));
    for (const auto& [id, hosts] : bad.state_hosts)
      if (hosts.size() > 1) std::printf("part.toytp2.fault.param %d\n", id);
  }
  return 0;
}
