import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from test_gpu_parity import run_gpu, mixed_params, toy_params
for name, params, cap in [("mixed3", mixed_params()[:3], 8_000_000), ("toy", toy_params(), 200), ("mixed", mixed_params(), 8_000_000)]:
    for gd in ("f32", "bf16"):
        w, n, b = run_gpu(params, cap, 1, 2, 1, grad_dtype=gd)
        bad = [p.name for p in params if not np.isfinite(w[p.id]).all()]
        nn = [p.name for p, v in zip(params, n[-1]) if not np.isfinite(v)]
        print(name, gd, "nonfinite W:", bad, "nonfinite norms:", nn)
