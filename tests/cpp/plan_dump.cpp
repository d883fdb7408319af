// Differential plan dump (test infrastructure).
//
// The same source is compiled twice:
//   * against the reference headers (/root/reference/proj/include) by
//     oracle/Makefile -> oracle/_ref/ref_plan_dump, which writes the golden
//     files under tests/golden/ (tests/golden/make_golden.sh);
//   * against this repo's include/optishard by the test build -> the output
//     must match the golden bytes exactly (tests/test_planner_golden.py).
// It prints, for every (config, R, method, cost, alpha), the serialized dp
// plan, its balance metrics (%.17g) and the owner table; then micro-group
// plans; then an a1-style fuzz corpus (acceptance_main.cpp:102-152 shape).
#include <cstdio>
#include <cstdint>
#include <iostream>
#include <random>
#include <string>
#include <vector>

#ifdef OSH_REFERENCE_HEADERS
#include "optishard/config.hpp"
#include "optishard/cost.hpp"
#include "optishard/dp_partition.hpp"
#include "optishard/metrics.hpp"
#include "optishard/serialize.hpp"
#include "optishard/tp_schedule.hpp"
#include "optishard/workload.hpp"
#else
#include "optishard/balance.hpp"
#include "optishard/costing.hpp"
#include "optishard/microgroup.hpp"
#include "optishard/model.hpp"
#include "optishard/partition.hpp"
#include "optishard/planfile.hpp"
#include "optishard/runconfig.hpp"
#endif

using namespace optishard;

namespace {

std::string g17(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

void emit_plan(const std::string& tag, const DpPartitionPlan& plan, const BufferLayout& layout,
               const std::vector<ParamSpec>& params, const CostModel& model) {
  std::cout << "## " << tag << "\n" << serialize_dp_plan(plan);
  const auto v = validate_plan(plan, layout, params, model);
  std::cout << "violations " << v.size() << "\n";
  const auto row = summarize_plan(tag, plan, layout, params);
  std::cout << "metrics " << g17(row.r_lb_cost) << " " << g17(row.r_lb_flops) << " "
            << g17(row.r_lb_memory) << " " << g17(row.j_dp) << " " << g17(row.j_comm) << "\n";
  if (plan.atomic) {
    std::cout << "owners";
    for (const ParamSpec& p : params) std::cout << " " << param_owner(plan, layout, p.id);
    std::cout << "\n";
  }
}

CostModel model_of(const std::string& kind) {
  CostModel m;
  m.kind = parse_cost_kind(kind);
  return m;
}

void dump_config(const std::string& path) {
  const RunFileConfig cfg = load_config_file(path);
  const auto full = generate_transformer_params(cfg.model);
  const int tps[] = {1, 2, 4, 8};
  for (const int tp : tps) {
    std::vector<ParamSpec> params;
    try {
      params = apply_tp_sharding(full, tp);
    } catch (const ShardError&) {
      continue;
    }
    const std::int64_t cap = tp == 1 ? cfg.model.bucket_capacity : cfg.model.bucket_capacity / tp;
    BufferLayout layout;
    try {
      layout = build_buffer_layout(params, cap);
    } catch (const LayoutError& e) {
      std::cout << "## " << cfg.model.name << " tp " << tp << " layout-error " << e.what() << "\n";
      continue;
    }
    std::cout << "# " << cfg.model.name << " tp " << tp << " params " << params.size()
              << " buckets " << layout.buckets.size() << " numel " << layout.total_numel << "\n";
    for (const char* kind : {"numel", "flops-muon", "flops-shampoo", "flops-soap", "bytes"}) {
      const CostModel model = model_of(kind);
      for (const int R : {1, 2, 3, 4, 8, 16, 32}) {
        const std::string base = cfg.model.name + " tp " + std::to_string(tp) + " R " +
                                 std::to_string(R) + " " + kind;
        for (const double a : {0.0, 0.25, 0.5, 0.75, 1.0})
          emit_plan(base + " alpha-balanced " + g17(a),
                    alpha_balanced_partition(layout, params, R, model, a), layout, params, model);
        emit_plan(base + " atomic-ownership",
                  atomic_ownership_partition(layout, params, R, model), layout, params, model);
        emit_plan(base + " equal-chunk", equal_chunk_partition(layout, params, R, model), layout,
                  params, model);
      }
    }
    if (tp > 1) {
      const auto plane = tp_plane_params(params);
      for (const char* kind : {"numel", "flops-muon"}) {
        const CostModel model = model_of(kind);
        Cost total = 0;
        for (const ParamSpec& p : plane) total += param_cost(p, model);
        const Cost caps[] = {total > 0 ? total : 1, 268435456ull, 134217728ull};
        for (const Cost c_max : caps) {
          std::cout << "## tp-plan " << cfg.model.name << " tp " << tp << " " << kind << " cmax "
                    << c_max << "\n";
          try {
            std::cout << serialize_tp_plan(build_micro_groups(plane, model, tp, c_max));
          } catch (const UnschedulableError& e) {
            std::cout << "unschedulable " << e.what() << "\n";
          }
        }
      }
    }
  }
}

// a1-shaped random workloads: mixed small matrices / vectors, bounded bucket
// counts, R in {2,4,8,16}, cost kinds and alphas cycling.
std::vector<ParamSpec> random_params(std::mt19937_64& rng, int count) {
  std::uniform_int_distribution<std::int64_t> side(1, 64);
  std::uniform_int_distribution<int> kind(0, 3);
  std::vector<ParamSpec> ps;
  for (int i = 0; i < count; ++i) {
    ParamSpec p;
    p.id = i;
    p.name = "p" + std::to_string(i);
    p.dtype_bytes = 2;
    if (kind(rng) == 0) {
      p.shape = {side(rng)};
    } else {
      const std::int64_t r = side(rng);
      const std::int64_t c = side(rng);
      p.shape = {r, c};
      p.tp_splittable = kind(rng) == 1 ? TpSplit::kRow : TpSplit::kColumn;
    }
    p.numel = 1;
    for (const auto e : p.shape) p.numel *= e;
    ps.push_back(p);
  }
  return ps;
}

void dump_fuzz(std::uint64_t seed, int count) {
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> n_params(5, 200);
  std::uniform_int_distribution<int> n_buckets(1, 8);
  std::uniform_int_distribution<int> pick(0, 3);
  const int ranks[4] = {2, 4, 8, 16};
  const char* kinds[3] = {"numel", "flops-muon", "bytes"};
  const double alphas[3] = {0.0, 0.5, 1.0};
  for (int t = 0; t < count; ++t) {
    const auto params = random_params(rng, n_params(rng));
    std::int64_t total = 0, biggest = 1;
    for (const auto& p : params) {
      total += p.numel;
      biggest = std::max(biggest, p.numel);
    }
    const int nb = n_buckets(rng);
    const std::int64_t cap = std::max(biggest, (total + nb - 1) / nb);
    const auto layout = build_buffer_layout(params, cap);
    const int R = ranks[pick(rng)];
    const CostModel model = model_of(kinds[t % 3]);
    const double a = alphas[(t / 3) % 3];
    const std::string tag = "fuzz " + std::to_string(t) + " R " + std::to_string(R);
    emit_plan(tag + " balanced", alpha_balanced_partition(layout, params, R, model, a), layout,
              params, model);
    emit_plan(tag + " strided", atomic_ownership_partition(layout, params, R, model), layout,
              params, model);
    std::vector<TpItem> items;
    for (const auto& p : tp_plane_params(params)) items.push_back({p.id, param_cost(p, model)});
    Cost mx = 1;
    for (const auto& it : items) mx = std::max(mx, it.cost);
    std::cout << "## " << tag << " groups\n"
              << serialize_tp_plan(build_micro_groups(items, 1 + t % 4, mx + mx / 2, model.kind));
  }
}

// One plan of one config: the parameter list, the serialized plan and the
// owner table (bench.py's reference arm plans with the reference's own
// planner through this mode; oracle/cpu_step.py parses it).
void dump_one(const std::string& path, int R, const std::string& method, const std::string& kind,
              double alpha) {
  const RunFileConfig cfg = load_config_file(path);
  const auto params = generate_transformer_params(cfg.model);
  const BufferLayout layout = build_buffer_layout(params, cfg.model.bucket_capacity);
  const CostModel model = model_of(kind);
  const PlanMethod m = parse_plan_method(method);
  const DpPartitionPlan plan = m == PlanMethod::kAlphaBalanced
                                   ? alpha_balanced_partition(layout, params, R, model, alpha)
                               : m == PlanMethod::kAtomicOwnership
                                   ? atomic_ownership_partition(layout, params, R, model)
                                   : equal_chunk_partition(layout, params, R, model);
  for (const ParamSpec& p : params) {
    std::cout << "param " << p.id << " " << p.name;
    for (const auto e : p.shape) std::cout << " " << e;
    std::cout << "\n";
  }
  std::cout << serialize_dp_plan(plan);
  if (plan.atomic) {
    std::cout << "owners";
    for (const ParamSpec& p : params) std::cout << " " << param_owner(plan, layout, p.id);
    std::cout << "\n";
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr,
                 "usage: %s config <file.cfg> | fuzz <seed> <count> | "
                 "plan <file.cfg> <ranks> <method> <cost> <alpha>\n",
                 argv[0]);
    return 2;
  }
  const std::string mode = argv[1];
  try {
    if (mode == "config" && argc == 3) {
      dump_config(argv[2]);
    } else if (mode == "plan" && argc == 7) {
      dump_one(argv[2], std::stoi(argv[3]), argv[4], argv[5], std::stod(argv[6]));
    } else if (mode == "fuzz" && argc == 4) {
      dump_fuzz(std::stoull(argv[2]), std::stoi(argv[3]));
    } else {
      std::fprintf(stderr, "bad arguments\n");
      return 2;
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
