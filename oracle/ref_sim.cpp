// TEST INFRASTRUCTURE (oracle/): drives the REFERENCE simulator
// (proj/include/optishard/simulate.hpp:163-296, unmodified headers) for the
// measured-vs-simulated calibration of SURVEY.md §8f F4. Built by
// `make -C oracle ref` into oracle/_ref/ref_sim; never linked into the product.
//
//   ref_sim L h f heads v cap ranks strategy exec_cost throughput inter_bw latency [alpha]
//
// strategy: sc | nv-layerwise | asc | lb-asc ; exec_cost: numel | flops-muon
// Prints one JSON object: the optimizer-step part of simulate_dp_step
// (compute from the max rank execution cost / throughput, plus the
// NV-layerwise broadcast) and the per-rank execution costs.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "optishard/simulate.hpp"

using namespace optishard;

int main(int argc, char** argv) {
  if (argc < 13) {
    std::fprintf(stderr, "usage: ref_sim L h f heads v cap ranks strategy exec_cost throughput inter_bw latency [alpha] [trace.json]\n");
    return 2;
  }
  ModelConfig cfg;
  cfg.name = "sim";
  cfg.num_layers = std::atoi(argv[1]);
  cfg.hidden_size = std::atoll(argv[2]);
  cfg.ffn_size = std::atoll(argv[3]);
  cfg.num_heads = std::atoi(argv[4]);
  cfg.vocab_size = std::atoll(argv[5]);
  cfg.bucket_capacity = std::atoll(argv[6]);
  const int ranks = std::atoi(argv[7]);
  const Strategy strategy = parse_strategy(argv[8]);
  CostModel exec;
  exec.kind = std::string(argv[9]) == "flops-muon" ? CostKind::kFlopsMuon : CostKind::kNumel;
  NetModel net;
  net.compute_throughput = std::atof(argv[10]);
  net.inter_bw_bps = std::atof(argv[11]);
  net.latency_s = std::atof(argv[12]);
  const double alpha = argc > 13 ? std::atof(argv[13]) : 1.0;
  const auto params = generate_transformer_params(cfg);
  const auto layout = build_buffer_layout(params, cfg.bucket_capacity);
  CostModel plan_cost;  // numel, as the measured runs
  DpPartitionPlan plan;
  const DpPartitionPlan* pp = nullptr;
  if (strategy == Strategy::kAsc) {
    plan = atomic_ownership_partition(layout, params, ranks, plan_cost);
    pp = &plan;
  } else if (strategy == Strategy::kLbAsc) {
    plan = alpha_balanced_partition(layout, params, ranks, plan_cost, alpha);
    pp = &plan;
  }
  const FwdBwdProfile prof = make_uniform_profile(layout, net);
  const DpSimResult r = simulate_dp_step(layout, params, ranks, strategy, pp, exec, net, prof);
  std::printf("{\"strategy\": \"%s\", \"ranks\": %d, \"optimizer_compute_s\": %.9g, "
              "\"optimizer_comm_s\": %.9g, \"optimizer_s\": %.9g, \"grad_bytes\": %.9g, "
              "\"rank_compute_cost\": [",
              to_string(strategy), ranks, r.optimizer_compute_s, r.optimizer_comm_s,
              r.optimizer_s, r.grad_bytes);
  for (std::size_t i = 0; i < r.rank_compute_cost.size(); ++i)
    std::printf("%s%llu", i ? ", " : "", static_cast<unsigned long long>(r.rank_compute_cost[i]));
  std::printf("]}\n");
  if (argc > 14) {  // the simulated events in Chrome trace-event form (trace.hpp's schema
                    // needs nlohmann/json, absent here; same fields written by hand)
    FILE* f = std::fopen(argv[14], "w");
    if (f) {
      std::fprintf(f, "{\"displayTimeUnit\": \"ms\", \"traceEvents\": [");
      for (std::size_t i = 0; i < r.events.size(); ++i) {
        const SimEvent& e = r.events[i];
        std::fprintf(f, "%s{\"name\": \"%s\", \"cat\": \"%s\", \"ph\": \"X\", \"pid\": 0, "
                        "\"tid\": %d, \"ts\": %.3f, \"dur\": %.3f, \"args\": {\"bytes\": %.0f}}",
                     i ? ", " : "", e.name.c_str(), e.cat.c_str(), e.tid, e.start_s * 1e6,
                     e.dur_s * 1e6, e.bytes);
      }
      std::fprintf(f, "]}\n");
      std::fclose(f);
    }
  }
  return 0;
}
