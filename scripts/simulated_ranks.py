"""Per-rank optimizer compute at R ranks measured on ONE B200, one rank at a
time (comm='none': each rank's ctx updates exactly the tensors the plan gives
it; reduced gradients are synthetic). This measures the compute half of an
R-GPU step — and the measured max/mean rank load — for R beyond the GPUs a
box has (the 8-GPU configs C2 / M0 of SURVEY.md §8 D2).

    python scripts/simulated_ranks.py CONFIG RANKS METHOD [ALPHA] [STEPS]
prints one JSON line.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig  # noqa: E402


def main():
    cfg_path, R, method = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    alpha = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    steps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
    cfg = P.load_config(cfg_path)
    params = P.generate_transformer_params(cfg)
    cap = cfg.bucket_capacity
    plan = P.plan_dp(params, cap, R, method, "numel", alpha)
    per_rank = []
    for r in range(R):
        with DistributedMuon(params, cap, plan, rank=r, comm="none", grad_dtype="bf16") as e:
            e.fill_synthetic(42, "weights")
            e.fill_synthetic(1000 + r, "grads")
            for _ in range(2):
                e.step(OptimizerConfig())
            e.sync()
            s = torch.cuda.ExternalStream(e.stream())
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(steps):
                e.step(OptimizerConfig())
            b.record(s)
            b.synchronize()
            per_rank.append(a.elapsed_time(b) / steps)
    loads = [float(x) for x in plan.rank_loads]
    mean = sum(per_rank) / R
    print(json.dumps({"config": os.path.basename(cfg_path), "ranks": R, "method": method,
                      "alpha": alpha if method == "alpha-balanced" else None,
                      "per_rank_compute_ms": [round(x, 2) for x in per_rank],
                      "max_compute_ms": round(max(per_rank), 2),
                      "measured_max_mean": round(max(per_rank) / mean, 4),
                      "plan_numel_max_mean": round(max(loads) / (sum(loads) / R), 4),
                      "note": "ranks run one at a time on one B200 (comm none): the compute "
                              "half of an R-GPU step, no collectives"}))


if __name__ == "__main__":
    main()
