"""Shampoo GPU vs spec on one tensor, one step, beta1 = 0 (dW = lr * grafted U)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from oracle import shampoo_oracle as S  # noqa: E402
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig, ShampooConfig  # noqa: E402

CASES = [((256, 256), 256, 16), ((256, 256), 256, 1), ((256, 256), 256, 2),
         ((256, 512), 256, 16), ((128, 128), 1024, 16), ((512, 768), 256, 16)]
if len(sys.argv) > 1:
    CASES = CASES[:int(sys.argv[1])]
for shape, block, iters in CASES:
    ps = [P.ParamSpec(0, "t", shape)]
    plan = P.plan_dp(ps, 10 ** 9, 1, "alpha-balanced", "numel", 1.0)
    scfg = ShampooConfig(block=block, precond_every=1, newton_iters=iters)
    e = DistributedMuon(ps, 10 ** 9, plan, comm="none", optimizer="shampoo", shampoo=scfg)
    w0 = O.init_weight(shape, 0, 42)
    g = O.reduced_gradient(shape, 0, 42, 0, 1)
    e.load_param(0, w0)
    e.write_grad(0, g)
    cfg = OptimizerConfig(lr=1.0, beta=0.0)
    e.step(cfg)
    e.sync()
    got = e.read_param(0, "master").astype(np.float64) - w0
    e.close()
    ocfg = S.ShampooConfig(lr=1.0, beta1=0.0, block=block, precond_every=1, newton_iters=iters)
    st = S.ShampooTensorState(shape, ocfg, True)
    w = w0.copy()
    S.shampoo_apply(st, ocfg, w, g, 0)
    ref = w - w0
    for k, (r0, p, c0, q) in enumerate(st.blocks):
        gb = g[r0:r0 + p, c0:c0 + q]
        u = st.PL[k] @ gb @ st.PR[k]
        print("ref block", k, "gsq", (gb ** 2).sum(), "usq(unscaled U)", (u ** 2).sum(),
              "ssqL", (st.L[k] ** 2).sum(), "ssqR", (st.R[k] ** 2).sum(), flush=True)
    print(shape, block, iters, "|dW| gpu", np.linalg.norm(got), "ref", np.linalg.norm(ref), "|g|",
          np.linalg.norm(g), "rel err", np.linalg.norm(got - ref) / np.linalg.norm(ref), flush=True)
