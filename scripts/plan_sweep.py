"""Partitioner sweep (BASELINE.json config C5): per model and R,
the max/mean rank load of equal-chunk, atomic-ownership and alpha-balanced
(alpha in {0, .25, .5, 1}) plans, planned on numel. Each cell is
"plan-cost r_lb / NS GEMM-flop r_lb" where the second number re-costs every
rank's owned tensors with 5*(4m^2n + 2m^3) (what the GPUs execute).
Equal-chunk splits tensors (Muon cannot run it): its flop column pro-rates
partial tensors exactly (no uint64 wrap)."""
import json
import os
import sys
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_06079_b200 import planner as P  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ns_flops(p):
    if not p.is_matrix:
        return 0
    m, n = min(p.shape), max(p.shape)
    return 5 * (4 * m * m * n + 2 * m ** 3)


def rlb(x):
    x = [float(v) for v in x]
    return max(x) / (sum(x) / len(x)) if sum(x) else 1.0


def flop_loads(params, layout, plan):
    loads = [Fraction(0)] * plan.ranks
    for b, ids in enumerate(layout.buckets):
        cuts = plan.cut_vectors[b]
        for pid in ids:
            p = params[pid]
            s = int(layout.offset[pid])
            e = s + p.numel
            for r in range(plan.ranks):
                ov = min(e, int(cuts[r + 1])) - max(s, int(cuts[r]))
                if ov > 0:
                    loads[r] += Fraction(ns_flops(p) * ov, p.numel)
    return loads


def main():
    out = []
    for cfg_name in ["qwen3-8b-like", "qwen3-1p7b-like", "qwen3-32b-like"]:
        cfg = P.load_config(os.path.join(ROOT, "configs", cfg_name + ".cfg"))
        params = P.generate_transformer_params(cfg)
        layout = P.build_buffer_layout(params, cfg.bucket_capacity)
        for R in (2, 4, 8):
            row = {"model": cfg_name, "R": R}
            for label, method, alpha in [("equal-chunk", "equal-chunk", 1.0),
                                         ("atomic-ownership", "atomic-ownership", 1.0),
                                         ("alpha=0", "alpha-balanced", 0.0),
                                         ("alpha=0.25", "alpha-balanced", 0.25),
                                         ("alpha=0.5", "alpha-balanced", 0.5),
                                         ("alpha=1", "alpha-balanced", 1.0)]:
                plan = P.plan_dp(params, cfg.bucket_capacity, R, method, "numel", alpha)
                row[label] = f"{rlb(plan.rank_loads):.3f}/{rlb(flop_loads(params, layout, plan)):.3f}"
            out.append(row)
    cols = ["model", "R", "equal-chunk", "atomic-ownership", "alpha=0", "alpha=0.25", "alpha=0.5",
            "alpha=1"]
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for r in out:
        print("| " + " | ".join(str(r[c]) for c in cols) + " |")
    with open(os.path.join(ROOT, "profiles", "r01_plan_sweep.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
