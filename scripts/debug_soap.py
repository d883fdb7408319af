"""SOAP GPU vs the fp64 spec and its bf16-emulating variant, per step and
tensor (relative Frobenius error of each step's update)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from oracle import soap_oracle as S  # noqa: E402
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig, SoapConfig  # noqa: E402

SEED = 42
pe = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
shapes = [(512, 768), (768,), (256, 256), (200, 328), (333, 96), (1000, 256), (64, 64)]
ps = [P.ParamSpec(i, f"t{i}", s) for i, s in enumerate(shapes)]
ps[5] = P.ParamSpec(5, "vocab", (1000, 256), 2, 0, True)
cfg = OptimizerConfig(lr=0.02, beta=0.9)
scfg = SoapConfig(block=256, precond_every=pe)
ocfg = S.SoapConfig(lr=cfg.lr, beta1=cfg.beta, beta2=scfg.beta2, shampoo_beta=scfg.beta2,
                    eps=scfg.eps, block=scfg.block, precond_every=pe, init_iters=scfg.init_iters)
cap = 10 ** 9
plan = P.plan_dp(ps, cap, 1, "alpha-balanced", "numel", 1.0)
e = DistributedMuon(ps, cap, plan, rank=0, comm="none", grad_dtype="f32", optimizer="soap", shampoo=scfg)
for p in ps:
    e.load_param(p.id, O.init_weight(p.shape, p.id, SEED))
w64 = {p.id: O.init_weight(p.shape, p.id, SEED).reshape(S._shape2(p)) for p in ps}
wem = {k: v.copy() for k, v in w64.items()}
st64 = {p.id: S.SoapTensorState(S._shape2(p), ocfg, S.is_preconditioned(p)) for p in ps}
stem = {p.id: S.SoapTensorState(S._shape2(p), ocfg, S.is_preconditioned(p)) for p in ps}
for s in range(steps):
    before = {p.id: e.read_param(p.id, "master").astype(np.float64).reshape(S._shape2(p)) for p in ps}
    b64 = {k: v.copy() for k, v in w64.items()}
    bem = {k: v.copy() for k, v in wem.items()}
    for p in ps:
        g = O.reduced_gradient(p.shape, p.id, SEED, s, 1)
        e.write_grad(p.id, g)
        S.soap_apply(st64[p.id], ocfg, w64[p.id], g.reshape(S._shape2(p)), s)
        S.soap_apply(stem[p.id], ocfg, wem[p.id], g.reshape(S._shape2(p)), s, emulate_bf16=True)
    e.step(cfg)
    row = []
    for p in ps:
        got = e.read_param(p.id, "master").astype(np.float64).reshape(S._shape2(p))
        dg = got - before[p.id]
        d64 = w64[p.id] - b64[p.id]
        dem = wem[p.id] - bem[p.id]
        row.append(f"{p.name}: fp64 {np.linalg.norm(dg - d64) / np.linalg.norm(d64):.3e} "
                   f"em {np.linalg.norm(dg - dem) / np.linalg.norm(dem):.3e} "
                   f"em-vs-64 {np.linalg.norm(dem - d64) / np.linalg.norm(d64):.3e}")
        # keep the GPU trajectory as the baseline for the next step
        w64[p.id] = w64[p.id] - d64 + (got - before[p.id]) * 0 + 0
    print(f"step {s}:")
    for r in row:
        print("   ", r)
e.close()
