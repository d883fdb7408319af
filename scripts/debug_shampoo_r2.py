"""Shampoo R=2 owner debug (OSH_SHAMPOO_DEBUG=1 prints per-block sums)."""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_gpu_shampoo import params  # noqa: E402
from paper_2602_06079_b200 import planner as P  # noqa: E402

ps = params()
plan = P.plan_dp(ps, 10 ** 9, 2, "alpha-balanced", "numel", 1.0)
print("owners", P.param_owners(ps, 10 ** 9, plan), flush=True)
import numpy as np  # noqa: E402
from test_gpu_shampoo import run_gpu  # noqa: E402
from paper_2602_06079_b200.engine import OptimizerConfig, ShampooConfig  # noqa: E402
import test_gpu_shampoo as T  # noqa: E402
T.STEPS = 1
b, _ = run_gpu(ps, 2, OptimizerConfig(), ShampooConfig(block=256, precond_every=2))
print({p.name: float(np.abs(b[p.id]).max()) for p in ps})
