import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from oracle import oracle as O
from paper_2602_06079_b200 import planner as P
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig
for shapes in ([(64, 96)], [(96, 64)], [(64, 96), (32,)], [(256, 512), (512, 256), (128,)]):
    params = [P.ParamSpec(i, f"t{i}", s) for i, s in enumerate(shapes)]
    plan = P.plan_dp(params, 10_000_000, 1)
    with DistributedMuon(params, 10_000_000, plan, comm="none") as c:
        w0 = {p.id: O.init_weight(p.shape, p.id, 42) for p in params}
        for p in params:
            c.load_param(p.id, w0[p.id]); c.write_grad(p.id, O.synth_gradient(p.shape, p.id, 42, 0, 0))
        c.step(OptimizerConfig())
        n = c.update_norms()
        for p in params:
            w = w0[p.id].copy(); m = np.zeros_like(w)
            rn = O.muon_apply(p.is_matrix, O.OptimizerConfig(), w, m, O.synth_gradient(p.shape, p.id, 42, 0, 0))
            got = c.read_param(p.id, "master").reshape(w.shape)
            dg = got - w0[p.id]; dr = w - w0[p.id]
            print(shapes, p.shape, "norm gpu", n[p.id], "ref", rn, "dW relerr", np.linalg.norm(dg - dr) / np.linalg.norm(dr),
                  "ratio", np.linalg.norm(dg) / np.linalg.norm(dr))
