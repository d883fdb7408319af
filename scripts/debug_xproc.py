import hashlib, sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from test_gpu_parity import run_gpu, mixed_params
params = mixed_params()[:3]
for gd in ("f32", "bf16"):
    w, n, b = run_gpu(params, 8_000_000, 1, 2, 1, grad_dtype=gd)
    print(gd, " ".join(hashlib.sha1(w[p.id].tobytes()).hexdigest()[:10] for p in params),
          " ".join(hashlib.sha1(b[p.id].tobytes()).hexdigest()[:10] for p in params))
