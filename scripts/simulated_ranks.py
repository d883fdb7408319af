"""Per-rank optimizer compute at R ranks measured on ONE B200, one rank at a
time (comm='none': each rank's ctx updates exactly the tensors the plan gives
it; reduced gradients are synthetic). This measures the compute half of an
R-GPU step — and the measured max/mean rank load — for R beyond the GPUs a
box has (the 8-GPU configs C2 / M0 of SURVEY.md §8 D2).

    python scripts/simulated_ranks.py CONFIG RANKS METHOD [ALPHA] [STEPS] [ROUNDS]
prints one JSON line. ALPHA may be "auto" (planner.choose_alpha).
OSH_SIMRANK_OPT=shampoo|soap runs the builder-defined blocked Shampoo / SOAP
instead of Muon (config C4) and also times one preconditioner-refresh step per rank;
OSH_SIMRANK_WS_GB caps the NS / Shampoo workspace (default: the runtime's).

Every rank is measured ROUNDS times, the ranks interleaved (rank 0..R-1, then
again), and each rank's median is reported: one B200 under its power cap
drifts by a few percent over a minute, and the max over R single samples
is biased upward by exactly that drift. OSH_SIMRANK_BREAKDOWN=1 adds the
per-mode kernel times (GEMM modes and elementwise kernels, summed CUDA-event
durations of one profiled step) of every rank.
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import (DistributedMuon, OptimizerConfig, ShampooConfig,  # noqa: E402
                                          SoapConfig)

OPT = os.environ.get("OSH_SIMRANK_OPT", "muon")  # muon | shampoo | soap
WS = int(float(os.environ.get("OSH_SIMRANK_WS_GB", "0")) * (1 << 30))
PRECOND_EVERY = 10


def ns_flops_per_rank(params, cap, plan, R):
    owners = P.param_owners(params, cap, plan)
    fl = [0.0] * R
    for p, o in zip(params, owners):
        if len(p.shape) == 2:
            m, n = sorted(p.shape)
            fl[int(o)] += 5.0 * (4.0 * m * m * n + 2.0 * m ** 3)
    return fl


def timed(e, n):
    s = torch.cuda.ExternalStream(e.stream())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(n):
        e.step(OptimizerConfig())
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / n


def measure_rank(params, cap, plan, r, steps, breakdown):
    sh = (ShampooConfig(precond_every=PRECOND_EVERY) if OPT == "shampoo" else
          SoapConfig(precond_every=PRECOND_EVERY) if OPT == "soap" else None)
    with DistributedMuon(params, cap, plan, rank=r, comm="none", grad_dtype="bf16",
                         optimizer=OPT, shampoo=sh, workspace_bytes=WS) as e:
        e.fill_synthetic(42, "weights")
        e.fill_synthetic(1000 + r, "grads")
        for _ in range(2):  # (Shampoo: step 0 is a refresh step)
            e.step(OptimizerConfig())
        e.sync()
        ms = timed(e, min(steps, PRECOND_EVERY - 2) if sh else steps)
        refresh = None
        if sh is not None:  # advance to the next refresh step and time it alone
            done = 2 + min(steps, PRECOND_EVERY - 2)
            for _ in range((-done) % PRECOND_EVERY):
                e.step(OptimizerConfig())
            e.sync()
            refresh = timed(e, 1)
        refresh_modes = None
        if sh is not None and breakdown:  # one more refresh step, profiled
            for _ in range(PRECOND_EVERY - 1):
                e.step(OptimizerConfig())
            e.sync()
            e.profile_gemm(True)
            e.step(OptimizerConfig())
            e.sync()
            e.profile_gemm(False)
            refresh_modes = {}
            for mode, lms, _fl, _ex, _what in e.gemm_profile_launches():
                refresh_modes[mode] = round(refresh_modes.get(mode, 0.0) + lms, 3)
            e.gemm_profile(reset=True)
        modes = None
        if breakdown:
            e.profile_gemm(True)
            e.step(OptimizerConfig())
            e.sync()
            e.profile_gemm(False)
            modes = {}
            for mode, lms, _fl, _ex, _what in e.gemm_profile_launches():
                modes[mode] = round(modes.get(mode, 0.0) + lms, 3)
            e.gemm_profile(reset=True)
            if refresh_modes is not None:
                modes = {"step": modes, "refresh_step": refresh_modes}
        return ms, modes, refresh


def main():
    cfg_path, R, method = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    alpha = sys.argv[4] if len(sys.argv) > 4 else "1.0"
    steps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
    rounds = int(sys.argv[6]) if len(sys.argv) > 6 else 1
    breakdown = os.environ.get("OSH_SIMRANK_BREAKDOWN", "0") == "1"
    cfg = P.load_config(cfg_path)
    params = P.generate_transformer_params(cfg)
    cap = cfg.bucket_capacity
    alpha = P.choose_alpha(params, cap, R)[0] if alpha == "auto" else float(alpha)
    plan = P.plan_dp(params, cap, R, method, "numel", alpha)
    samples = [[] for _ in range(R)]
    modes = [None] * R
    refresh = [[] for _ in range(R)]
    for k in range(rounds):
        for r in range(R):
            ms, md, rf = measure_rank(params, cap, plan, r, steps, breakdown and k == 0)
            samples[r].append(ms)
            if rf is not None:
                refresh[r].append(rf)
            if md is not None:
                modes[r] = md
    per_rank = [statistics.median(s) for s in samples]
    loads = [float(x) for x in plan.rank_loads]
    fl = ns_flops_per_rank(params, cap, plan, R)
    mean = sum(per_rank) / R
    out = {"config": os.path.basename(cfg_path), "optimizer": OPT, "ranks": R, "method": method,
           "alpha": alpha if method == "alpha-balanced" else None,
           "rounds": rounds, "steps_per_sample": steps,
           "per_rank_compute_ms": [round(x, 2) for x in per_rank],
           "per_rank_samples_ms": [[round(x, 2) for x in s] for s in samples],
           "per_rank_ns_tflop": [round(x / 1e12, 2) for x in fl],
           "per_rank_alg_tflops": [round(f / (t * 1e-3) / 1e12, 1) for f, t in zip(fl, per_rank)],
           "max_compute_ms": round(max(per_rank), 2),
           "measured_max_mean": round(max(per_rank) / mean, 4),
           "plan_numel_max_mean": round(max(loads) / (sum(loads) / R), 4),
           "plan_nsflops_max_mean": round(max(fl) / (sum(fl) / R), 4),
           "note": "ranks run one at a time on one B200 (comm none): the compute "
                   "half of an R-GPU step, no collectives; per-rank median over "
                   "interleaved rounds"}
    if OPT in ("shampoo", "soap"):
        # Newton-Schulz flops do not apply; the per-step ratio is the measured one
        for k in ("per_rank_ns_tflop", "per_rank_alg_tflops", "plan_nsflops_max_mean"):
            out.pop(k)
        rf = [statistics.median(x) for x in refresh]
        amort = [(t * (PRECOND_EVERY - 1) + f) / PRECOND_EVERY for t, f in zip(per_rank, rf)]
        out.update({"precond_every": PRECOND_EVERY,
                    "per_rank_refresh_ms": [round(x, 1) for x in rf],
                    "per_rank_amortized_ms": [round(x, 2) for x in amort],
                    "measured_max_mean_amortized": round(max(amort) / (sum(amort) / R), 4)})
    if breakdown:
        out["per_rank_modes_ms"] = modes
    print(json.dumps(out))


if __name__ == "__main__":
    main()
