"""Two Muon steps on the 1.7B-shaped config (R=1) — for ncu captures of the
momentum / apply kernels at realistic sizes."""
import os
import sys

sys.path.insert(0, ".")
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig  # noqa: E402

cfg = P.load_config(os.path.join("configs", "qwen3-1p7b-like.cfg"))
params = P.generate_transformer_params(cfg)
plan = P.plan_dp(params, cfg.bucket_capacity, 1)
with DistributedMuon(params, cfg.bucket_capacity, plan, comm="none", grad_dtype="bf16") as eng:
    eng.fill_synthetic(42, "weights")
    eng.fill_synthetic(7, "grads")
    for _ in range(2):
        eng.step(OptimizerConfig())
    eng.sync()
print("ok")
