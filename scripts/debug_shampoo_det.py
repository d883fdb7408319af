"""Shampoo determinism: R=1 twice and R=2 vs R=1, max |diff| per tensor."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_gpu_shampoo import params, run_gpu  # noqa: E402
from paper_2602_06079_b200.engine import OptimizerConfig, ShampooConfig  # noqa: E402

ps = params()
cfg = OptimizerConfig()
scfg = ShampooConfig(block=256, precond_every=2)
a, _ = run_gpu(ps, 1, cfg, scfg)
a2, _ = run_gpu(ps, 1, cfg, scfg)
b, _ = run_gpu(ps, 2, cfg, scfg)
for p in ps:
    print(p.name, p.shape, "R1 vs R1", np.abs(a[p.id] - a2[p.id]).max(), "R2 vs R1",
          np.abs(a[p.id] - b[p.id]).max(), "scale", np.abs(a[p.id]).max())
