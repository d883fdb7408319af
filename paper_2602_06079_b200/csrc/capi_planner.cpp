// C-ABI wrappers of the host planner (include/optishard/*.hpp). Every C++
// exception is caught here and turned into the matching osh_status, so no
// exception crosses the ABI (osh.h).
#include <cstring>
#include <string>
#include <vector>

#include "optishard/optishard.hpp"
#include "comm_schedule.hpp"
#include "osh.h"
#include "status.hpp"

using namespace optishard;

namespace {

template <typename F>
osh_status guarded(const char* where, F&& body) {
  try {
    body();
    return OSH_OK;
  } catch (const ConfigError& e) {
    return osh::fail(OSH_ERR_CONFIG, std::string(where) + ": " + e.what());
  } catch (const LayoutError& e) {
    return osh::fail(OSH_ERR_LAYOUT, std::string(where) + ": " + e.what());
  } catch (const ShardError& e) {
    return osh::fail(OSH_ERR_SHARD, std::string(where) + ": " + e.what());
  } catch (const UnsupportedError& e) {
    return osh::fail(OSH_ERR_UNSUPPORTED, std::string(where) + ": " + e.what());
  } catch (const PlanError& e) {
    return osh::fail(OSH_ERR_PLAN, std::string(where) + ": " + e.what());
  } catch (const UnschedulableError& e) {
    return osh::fail(OSH_ERR_UNSCHEDULABLE, std::string(where) + ": " + e.what());
  } catch (const FormatError& e) {
    return osh::fail(OSH_ERR_FORMAT, std::string(where) + ": " + e.what());
  } catch (const std::bad_alloc&) {
    return osh::fail(OSH_ERR_OOM, std::string(where) + ": out of host memory");
  } catch (const std::exception& e) {
    return osh::fail(OSH_ERR_ARG, std::string(where) + ": " + e.what());
  }
}

ParamSpec to_spec(const osh_param_desc& d) {
  if (d.ndim != 1 && d.ndim != 2) throw UnsupportedError("params must be 1-D or 2-D");
  ParamSpec p;
  p.id = d.id;
  p.name = "p" + std::to_string(d.id);
  p.shape.assign(d.shape, d.shape + d.ndim);
  p.numel = 1;
  for (const std::int64_t e : p.shape) p.numel *= e;
  p.dtype_bytes = d.dtype_bytes;
  p.tp_splittable = d.tp_split == 1 ? TpSplit::kColumn : d.tp_split == 2 ? TpSplit::kRow
                                                                        : TpSplit::kNone;
  p.vocab_space = d.vocab_space != 0;
  return p;
}

osh_param_desc to_desc(const ParamSpec& p) {
  osh_param_desc d{};
  d.id = p.id;
  d.ndim = static_cast<int32_t>(p.shape.size());
  for (std::size_t i = 0; i < p.shape.size() && i < 2; ++i) d.shape[i] = p.shape[i];
  d.dtype_bytes = p.dtype_bytes;
  d.tp_split = p.tp_splittable == TpSplit::kColumn ? 1 : p.tp_splittable == TpSplit::kRow ? 2 : 0;
  d.vocab_space = p.vocab_space ? 1 : 0;
  return d;
}

// Params are indexed by id in the reference (params.at(id)); the C caller
// passes them in id order 0..n-1.
std::vector<ParamSpec> to_specs(const osh_param_desc* params, int32_t n) {
  if (n < 0 || (n > 0 && params == nullptr)) throw UnsupportedError("bad parameter array");
  std::vector<ParamSpec> v;
  v.reserve(static_cast<std::size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    if (params[i].id != i) throw PlanError("parameter ids must be dense 0..n-1 in order");
    v.push_back(to_spec(params[i]));
  }
  return v;
}

CostModel to_model(const osh_cost_model* m) {
  CostModel c;
  if (m == nullptr) return c;
  if (m->kind < OSH_COST_NUMEL || m->kind > OSH_COST_BYTES) throw ConfigError("unknown cost kind");
  c.kind = static_cast<CostKind>(m->kind);
  c.ns_steps = m->ns_steps;
  c.shampoo_coeff = m->shampoo_coeff;
  c.soap_coeff = m->soap_coeff;
  return c;
}

DpPartitionPlan make_plan(const std::vector<ParamSpec>& specs, const BufferLayout& layout,
                          int32_t ranks, int32_t method, const CostModel& model, double alpha) {
  switch (method) {
    case OSH_PLAN_EQUAL_CHUNK: return equal_chunk_partition(layout, specs, ranks, model);
    case OSH_PLAN_ATOMIC_OWNERSHIP: return atomic_ownership_partition(layout, specs, ranks, model);
    case OSH_PLAN_ALPHA_BALANCED:
      return alpha_balanced_partition(layout, specs, ranks, model, alpha);
    default: throw FormatError("unknown plan method");
  }
}

void copy_text(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len != nullptr) *len = s.size();
  if (buf != nullptr && cap > 0) {
    const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
}

}  // namespace

extern "C" {

void osh_muon_cfg_default(osh_muon_cfg* cfg) {
  if (cfg == nullptr) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->lr = 0.02;
  cfg->beta = 0.9;
  cfg->ns_steps = 5;
  cfg->ns_a = 3.4445;
  cfg->ns_b = -4.7750;
  cfg->ns_c = 2.0315;
}

osh_status osh_generate_params(int32_t num_layers, int64_t hidden, int64_t ffn, int32_t heads,
                               int64_t vocab, int32_t dtype_bytes, osh_param_desc* out,
                               int32_t capacity, int32_t* n_out) {
  return guarded("osh_generate_params", [&] {
    ModelConfig c;
    c.name = "capi";
    c.num_layers = num_layers;
    c.hidden_size = hidden;
    c.ffn_size = ffn;
    c.num_heads = heads;
    c.vocab_size = vocab;
    c.dtype_bytes = dtype_bytes;
    const std::vector<ParamSpec> ps = generate_transformer_params(c);
    if (n_out != nullptr) *n_out = static_cast<int32_t>(ps.size());
    if (out == nullptr) return;
    if (capacity < static_cast<int32_t>(ps.size()))
      throw UnsupportedError("output array too small");
    for (std::size_t i = 0; i < ps.size(); ++i) out[i] = to_desc(ps[i]);
  });
}

osh_status osh_param_cost(const osh_param_desc* p, const osh_cost_model* model, uint64_t* out) {
  return guarded("osh_param_cost", [&] {
    if (p == nullptr || out == nullptr) throw UnsupportedError("null argument");
    *out = param_cost(to_spec(*p), to_model(model));
  });
}

osh_status osh_layout_build(const osh_param_desc* params, int32_t n, int64_t bucket_capacity,
                            int32_t* bucket_of, int64_t* offset_in_bucket, int64_t* bucket_numel,
                            int32_t* n_buckets) {
  return guarded("osh_layout_build", [&] {
    const std::vector<ParamSpec> specs = to_specs(params, n);
    const BufferLayout layout = build_buffer_layout(specs, bucket_capacity);
    for (const Bucket& b : layout.buckets) {
      for (std::size_t j = 0; j < b.param_ids.size(); ++j) {
        const int id = b.param_ids[j];
        if (bucket_of != nullptr) bucket_of[id] = b.index;
        if (offset_in_bucket != nullptr) offset_in_bucket[id] = b.param_offsets[j];
      }
      if (bucket_numel != nullptr) bucket_numel[b.index] = b.numel;
    }
    if (n_buckets != nullptr) *n_buckets = static_cast<int32_t>(layout.buckets.size());
  });
}

osh_status osh_plan_dp(const osh_param_desc* params, int32_t n, int64_t bucket_capacity,
                       int32_t ranks, int32_t method, const osh_cost_model* model, double alpha,
                       int64_t* cuts, uint64_t* rank_loads, int32_t* atomic) {
  return guarded("osh_plan_dp", [&] {
    const std::vector<ParamSpec> specs = to_specs(params, n);
    const BufferLayout layout = build_buffer_layout(specs, bucket_capacity);
    const DpPartitionPlan plan = make_plan(specs, layout, ranks, method, to_model(model), alpha);
    if (cuts != nullptr)
      for (std::size_t i = 0; i < plan.cut_vectors.size(); ++i)
        std::memcpy(cuts + i * static_cast<std::size_t>(ranks + 1), plan.cut_vectors[i].data(),
                    sizeof(int64_t) * static_cast<std::size_t>(ranks + 1));
    if (rank_loads != nullptr)
      std::memcpy(rank_loads, plan.rank_loads.data(), sizeof(uint64_t) * plan.rank_loads.size());
    if (atomic != nullptr) *atomic = plan.atomic ? 1 : 0;
  });
}

osh_status osh_plan_dp_serialize(const osh_param_desc* params, int32_t n, int64_t bucket_capacity,
                                 int32_t ranks, int32_t method, const osh_cost_model* model,
                                 double alpha, char* buf, size_t cap, size_t* len) {
  return guarded("osh_plan_dp_serialize", [&] {
    const std::vector<ParamSpec> specs = to_specs(params, n);
    const BufferLayout layout = build_buffer_layout(specs, bucket_capacity);
    copy_text(serialize_dp_plan(make_plan(specs, layout, ranks, method, to_model(model), alpha)),
              buf, cap, len);
  });
}

osh_status osh_param_owners(const osh_param_desc* params, int32_t n, int64_t bucket_capacity,
                            int32_t ranks, const int64_t* cuts, int32_t* owner_out) {
  return guarded("osh_param_owners", [&] {
    const std::vector<ParamSpec> specs = to_specs(params, n);
    const BufferLayout layout = build_buffer_layout(specs, bucket_capacity);
    if (ranks < 1) throw PlanError("ranks must be >= 1");
    DpPartitionPlan plan;
    plan.ranks = ranks;
    for (std::size_t i = 0; i < layout.buckets.size(); ++i)
      plan.cut_vectors.emplace_back(cuts + i * static_cast<std::size_t>(ranks + 1),
                                    cuts + (i + 1) * static_cast<std::size_t>(ranks + 1));
    for (const ParamSpec& p : specs) owner_out[p.id] = param_owner(plan, layout, p.id);
  });
}

osh_status osh_plan_tp_serialize(const int32_t* item_ids, const uint64_t* item_costs, int32_t n,
                                 int32_t ranks, uint64_t c_max, int32_t cost_kind, char* buf,
                                 size_t cap, size_t* len) {
  return guarded("osh_plan_tp_serialize", [&] {
    std::vector<TpItem> items;
    for (int32_t i = 0; i < n; ++i) items.push_back(TpItem{item_ids[i], item_costs[i]});
    if (cost_kind < OSH_COST_NUMEL || cost_kind > OSH_COST_BYTES)
      throw ConfigError("unknown cost kind");
    copy_text(serialize_tp_plan(build_micro_groups(std::move(items), ranks, c_max,
                                                   static_cast<CostKind>(cost_kind))),
              buf, cap, len);
  });
}

osh_status osh_comm_schedule(const osh_param_desc* params, int32_t n, int64_t bucket_capacity,
                             int32_t ranks, const int64_t* cuts, int32_t n_buckets,
                             int32_t strategy, const int32_t* layer_of,
                             const osh_cost_model* cost, osh_coll_op* out, int32_t cap,
                             int32_t* n_out) {
  return guarded("osh_comm_schedule", [&] {
    const std::vector<ParamSpec> specs = to_specs(params, n);
    const BufferLayout layout = build_buffer_layout(specs, bucket_capacity);
    if (ranks < 1) throw PlanError("ranks must be >= 1");
    if (cuts == nullptr || n_buckets != static_cast<int32_t>(layout.buckets.size()))
      throw PlanError("cut vectors must cover every bucket of the layout");
    if (strategy < OSH_STRAT_SHARDED || strategy > OSH_STRAT_NV_LAYERWISE)
      throw ConfigError("unknown strategy");
    std::vector<std::vector<int64_t>> cv;
    std::vector<int64_t> bucket_base, flat_off(specs.size()), numel(specs.size());
    int64_t base = 0;
    for (const Bucket& b : layout.buckets) {
      cv.emplace_back(cuts + static_cast<std::size_t>(b.index) * (ranks + 1),
                      cuts + static_cast<std::size_t>(b.index + 1) * (ranks + 1));
      if (cv.back().front() != 0 || cv.back().back() != b.numel)
        throw PlanError("bucket " + std::to_string(b.index) + ": cuts must span [0, numel]");
      bucket_base.push_back(base);
      for (std::size_t j = 0; j < b.param_ids.size(); ++j)
        flat_off[static_cast<std::size_t>(b.param_ids[j])] = base + b.param_offsets[j];
      base += b.numel;
    }
    for (const ParamSpec& p : specs) numel[static_cast<std::size_t>(p.id)] = p.numel;
    std::vector<int> owner(specs.size(), 0);
    if (strategy == OSH_STRAT_NV_LAYERWISE) {
      if (layer_of == nullptr) throw PlanError("NV-layerwise needs the layer group of every parameter");
      owner = osh::layerwise_owners(specs, std::vector<int32_t>(layer_of, layer_of + n), ranks,
                                    to_model(cost));
    }
    const std::vector<osh_coll_op> ops =
        ranks > 1 ? osh::build_comm_schedule(strategy, cv, bucket_base, flat_off, numel, owner)
                  : std::vector<osh_coll_op>{};
    if (n_out != nullptr) *n_out = static_cast<int32_t>(ops.size());
    if (out == nullptr) return;
    if (cap < static_cast<int32_t>(ops.size())) throw UnsupportedError("output array too small");
    std::copy(ops.begin(), ops.end(), out);
  });
}

}  // extern "C"
