// The data-parallel collective schedule of one optimizer step, as a value.
//
// The runtime (runtime.cu) issues exactly these operations to NCCL, in this
// order, on every rank, and osh_comm_schedule / osh_ctx_comm_schedule export
// them through the C ABI so the exchange can be executed and checked without
// a GPU (tests/test_multi_rank_cpu.py runs it over gloo against the oracle).
//
// Sharded strategy (the Canzona step, the reference models it
// analytically in collective.hpp:49-76 / simulate.hpp:199-253):
//   RS-v, per bucket b (one NCCL group per bucket): for every rank r with a
//     non-empty slice [cuts[b][r], cuts[b][r+1]), a Reduce rooted at r of that
//     slice of the flat gradient buffer into r's reduced-slice buffer at
//     dst_offset (r's slices of the earlier buckets come first);
//   AG-v, per bucket b: a Broadcast rooted at r of the same slice of the bf16
//     replica, in place.
// SC: an AllReduce of every bucket, no redistribution (simulate.hpp:33-39).
// NV-layerwise: an AllReduce of every bucket, then a Broadcast of every tensor
// from the owner of its layer (kBroadcast redistribution, simulate.hpp:58-59).
#pragma once

#include <cstdint>
#include <vector>

#include "optishard/optishard.hpp"
#include "osh.h"

namespace osh {

// Whole-layer owners of the NV-layerwise baseline: LPT over the layer costs
// (min_heap_balance, simulate.hpp:140-157).
inline std::vector<int> layerwise_owners(const std::vector<optishard::ParamSpec>& params,
                                         const std::vector<int32_t>& layer_of, int ranks,
                                         const optishard::CostModel& cost) {
  using namespace optishard;
  if (layer_of.size() != params.size()) throw PlanError("layer_of must cover every parameter");
  std::vector<Cost> layer_cost;
  for (std::size_t p = 0; p < params.size(); ++p) {
    if (layer_of[p] < 0) throw PlanError("negative layer id");
    const std::size_t l = static_cast<std::size_t>(layer_of[p]);
    if (layer_cost.size() <= l) layer_cost.resize(l + 1, 0);
    layer_cost[l] += param_cost(params[p], cost);
  }
  std::vector<TpItem> items;
  for (std::size_t l = 0; l < layer_cost.size(); ++l) items.push_back({static_cast<int>(l), layer_cost[l]});
  const HeapAssignment a = min_heap_balance(items, ranks);
  std::vector<int> layer_owner(layer_cost.size(), 0);
  for (std::size_t r = 0; r < a.rank_params.size(); ++r)
    for (const int l : a.rank_params[r]) layer_owner[static_cast<std::size_t>(l)] = static_cast<int>(r);
  std::vector<int> owner(params.size(), 0);
  for (std::size_t p = 0; p < params.size(); ++p)
    owner[p] = layer_owner[static_cast<std::size_t>(layer_of[p])];
  return owner;
}

// cuts: [bucket][R+1]; bucket_base: flat element offset of each bucket;
// flat_off / numel / owner: per parameter (owner used by NV-layerwise only).
inline std::vector<osh_coll_op> build_comm_schedule(int strategy,
                                                    const std::vector<std::vector<int64_t>>& cuts,
                                                    const std::vector<int64_t>& bucket_base,
                                                    const std::vector<int64_t>& flat_off,
                                                    const std::vector<int64_t>& numel,
                                                    const std::vector<int>& owner) {
  std::vector<osh_coll_op> ops;
  const int nb = static_cast<int>(cuts.size());
  auto op = [&](int kind, int phase, int bucket, int root, int group, int64_t off, int64_t cnt,
                int64_t dst) {
    osh_coll_op o{};
    o.kind = kind;
    o.phase = phase;
    o.bucket = bucket;
    o.root = root;
    o.group = group;
    o.offset = off;
    o.count = cnt;
    o.dst_offset = dst;
    ops.push_back(o);
  };
  if (strategy == OSH_STRAT_SHARDED) {
    const int R = nb > 0 ? static_cast<int>(cuts[0].size()) - 1 : 1;
    std::vector<int64_t> slice_off(static_cast<std::size_t>(R), 0);  // per root: reduced-slice cursor
    for (int b = 0; b < nb; ++b)
      for (int r = 0; r < R; ++r) {
        const int64_t cnt = cuts[b][r + 1] - cuts[b][r];
        if (cnt == 0) continue;
        op(OSH_OP_REDUCE, OSH_PHASE_RS, b, r, b, bucket_base[b] + cuts[b][r], cnt, slice_off[r]);
        slice_off[r] += cnt;
      }
    for (int b = 0; b < nb; ++b)
      for (int r = 0; r < R; ++r) {
        const int64_t cnt = cuts[b][r + 1] - cuts[b][r];
        if (cnt == 0) continue;
        op(OSH_OP_BROADCAST, OSH_PHASE_AG, b, r, nb + b, bucket_base[b] + cuts[b][r], cnt, -1);
      }
    return ops;
  }
  for (int b = 0; b < nb; ++b)  // cuts[b].back() is the bucket's numel
    op(OSH_OP_ALLREDUCE, OSH_PHASE_RS, b, -1, b, bucket_base[b], cuts[b].back(), -1);
  if (strategy == OSH_STRAT_NV_LAYERWISE) {
    // params in declaration order = flat order; bucket of each from its offset
    int b = 0;
    for (std::size_t p = 0; p < flat_off.size(); ++p) {
      while (b + 1 < nb && flat_off[p] >= bucket_base[b + 1]) ++b;
      op(OSH_OP_BROADCAST, OSH_PHASE_AG, b, owner[p], nb, flat_off[p], numel[p], -1);
    }
  }
  return ops;
}

}  // namespace osh
