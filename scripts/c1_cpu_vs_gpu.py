"""A MEASURED full CPU step next to the GPU step on config C1 (Qwen3-0.6B
shapes): no sampling, no extrapolation.

CPU: the reference's run_replicated step (verify.hpp:188-210) restated in
oracle/ (fp64, NS in the reference's 3-product form through OpenBLAS on every
host core), over all 143 tensors with R = 2 contributors. Timed twice:
  * optimizer: muon_apply over every tensor on pre-generated reduced
    gradients (the optimizer step proper),
  * full:      the same plus the per-step gradient synthesis and ascending
    rank sum of run_replicated.
GPU: the same model on one B200 through the C ABI (osh_step, device-resident
bf16 gradients), CUDA events on the ctx stream, after warm-up.

    python scripts/c1_cpu_vs_gpu.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

CFG = os.path.join(ROOT, "configs", "qwen3-0p6b-like.cfg")
SEED, R = 42, 2


def cpu_step():
    from oracle import cpu_step as C

    plan = C.reference_plan(CFG, 1)
    fast = O.set_fast_blas(True)
    O.lib().orc_set_threads(os.cpu_count())
    params = [(pid, shape) for pid, _, shape in plan.params]
    w = {pid: O.init_weight(s, pid, SEED) for pid, s in params}
    m = {pid: np.zeros_like(w[pid]) for pid, _ in params}
    cfg = O.OptimizerConfig()
    t0 = time.perf_counter()
    grads = {pid: O.reduced_gradient(s, pid, SEED, 0, R) for pid, s in params}
    t_synth = time.perf_counter() - t0
    t0 = time.perf_counter()
    for pid, s in params:
        O.muon_apply(len(s) == 2, cfg, w[pid], m[pid], grads[pid])
    t_opt = time.perf_counter() - t0
    return {"optimizer_ms": round(1e3 * t_opt, 1), "full_ms": round(1e3 * (t_opt + t_synth), 1),
            "gradient_synthesis_ms": round(1e3 * t_synth, 1), "cores": O.lib().orc_get_threads(),
            "blas": "numpy OpenBLAS (ILP64 dgemm)" if fast else "blocked C GEMM",
            "tensors": len(params), "contributors": R, "planner": plan.source}


def gpu_step(steps=10, warmup=3):
    import torch

    from paper_2602_06079_b200 import planner as P
    from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig

    cfg = P.load_config(CFG)
    params = P.generate_transformer_params(cfg)
    plan = P.plan_dp(params, cfg.bucket_capacity, 1)
    with DistributedMuon(params, cfg.bucket_capacity, plan, comm="none", grad_dtype="bf16") as eng:
        eng.fill_synthetic(42, "weights")
        eng.fill_synthetic(1000, "grads")
        stream = torch.cuda.ExternalStream(eng.stream())
        for _ in range(warmup):
            eng.step(OptimizerConfig())
        eng.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            eng.step(OptimizerConfig())
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
    return {"step_ms": round(ms, 3), "steps": steps, "warmup": warmup, "grad_dtype": "bf16",
            "device": torch.cuda.get_device_name(0)}


def main():
    out = {"config": "C1 qwen3-0p6b-like (143 tensors, 604,795,904 params), R=1 GPU step vs "
                     "the reference's fp64 CPU step with 2 contributors",
           "gpu": gpu_step(), "cpu": cpu_step()}
    out["cpu_over_gpu_optimizer"] = round(out["cpu"]["optimizer_ms"] / out["gpu"]["step_ms"], 1)
    line = json.dumps(out)
    print(line)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
