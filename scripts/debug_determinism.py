import sys; sys.path.insert(0, ".")
import numpy as np
sys.path.insert(0, "tests")
from test_gpu_parity import run_gpu, mixed_params, toy_params
params = mixed_params()[:3]
runs = [run_gpu(params, 8_000_000, 1, 2, 1, grad_dtype=gd) for gd in ("f32", "bf16", "f32", "bf16", "f32")]
for i in range(1, len(runs)):
    for p in params:
        d = np.abs(runs[0][0][p.id] - runs[i][0][p.id]).max() if i % 2 == 0 else np.abs(runs[1][0][p.id] - runs[i][0][p.id]).max()
        print("run", i, p.name, "diff vs same-dtype run", d)
for p in params:
    print(p.name, "f32 vs bf16", np.abs(runs[0][0][p.id] - runs[1][0][p.id]).max() / np.abs(runs[0][0][p.id]).max())
