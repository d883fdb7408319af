import sys; sys.path.insert(0, ".")
import numpy as np
from oracle import oracle as O
from paper_2602_06079_b200 import planner as P
from paper_2602_06079_b200.engine import DistributedMuon
params = [P.ParamSpec(0, "a", (1024, 3072)), P.ParamSpec(1, "b", (1024, 1024)), P.ParamSpec(2, "c", (3072, 1024))]
plan = P.plan_dp(params, 8_000_000, 1)
res = {}
for gd in ("f32", "bf16"):
    c = DistributedMuon(params, 8_000_000, plan, comm="none", grad_dtype=gd)
    for p in params:
        c.load_param(p.id, O.init_weight(p.shape, p.id, 42))
    ws = []
    for step in range(3):
        for p in params:
            c.write_grad(p.id, O.reduced_gradient(p.shape, p.id, 42, step, 1))
        c.step()
        ws.append({p.id: (c.read_param(p.id, "master"), c.read_param(p.id, "momentum")) for p in params})
        print(gd, step, c.update_norms())
    res[gd] = ws
    c.close()
for step in range(3):
    for p in params:
        wf, mf = res["f32"][step][p.id]; wb, mb = res["bf16"][step][p.id]
        print(step, p.name, "Wdiff", np.abs(wf - wb).max(), "Wmax", np.abs(wf).max(), "Mdiff rel", np.abs(mf - mb).max() / np.abs(mf).max())
