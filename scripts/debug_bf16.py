import sys; sys.path.insert(0, ".")
import numpy as np
from oracle import oracle as O
from paper_2602_06079_b200 import planner as P
from paper_2602_06079_b200.engine import DistributedMuon
params = [P.ParamSpec(0, "a", (1024, 3072)), P.ParamSpec(1, "b", (3072, 1024)), P.ParamSpec(2, "c", (512, 96)), P.ParamSpec(3, "d", (96, 512))]
plan = P.plan_dp(params, 8_000_000, 1)
out = {}
for gd in ("f32", "bf16"):
    c = DistributedMuon(params, 8_000_000, plan, comm="none", grad_dtype=gd)
    for p in params:
        c.load_param(p.id, O.init_weight(p.shape, p.id, 42))
        c.write_grad(p.id, O.synth_gradient(p.shape, p.id, 42, 0, 0))
    c.step()
    out[gd] = {p.id: (c.read_param(p.id, "momentum"), c.read_param(p.id, "master"), c.read_param(p.id, "replica")) for p in params}
    out[gd]["norms"] = c.update_norms()
    c.close()
for p in params:
    g = O.synth_gradient(p.shape, p.id, 42, 0, 0).reshape(p.shape)
    mf, wf, rf = out["f32"][p.id]; mb, wb, rb = out["bf16"][p.id]
    print(p.name, p.shape, "mom f32-vs-g", np.abs(mf - g).max(), "mom bf16-vs-g", np.abs(mb - g).max(), "rel", np.abs(mb-g).max()/np.abs(g).max(),
          "W diff", np.abs(wf - wb).max(), "W", np.abs(wf).max(), "dW f32", np.abs(wf - O.init_weight(p.shape, p.id, 42).reshape(p.shape)).max())
print(out["f32"]["norms"], out["bf16"]["norms"])
