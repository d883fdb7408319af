"""Config C1 end to end: the whole qwen3-0.6B-like model
(604,795,904 parameters, 143 tensors incl. the two 1024x151936 vocabulary
matrices), bucket capacity 155,582,464 (4 buckets), the α-balanced plan at
R = 2 (two ranks simulated on one B200, comm none), one step of the product
path against the fp64 oracle (reference algorithm, OpenBLAS dgemm) on the
reference generator's inputs. Every tensor must meet the tolerances of
tests/test_gpu_parity.py; the plan's max/mean equals the reference planner's
(1.000 at R = 2 under numel).
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = 42
TOL_DW, TOL_W, TOL_VEC = 3e-2, 2.5e-3, 1e-5


def test_c1_full_model_two_ranks_match_oracle():
    cfg = P.load_config(os.path.join(ROOT, "configs", "qwen3-0p6b-like.cfg"))
    params = P.generate_transformer_params(cfg)
    cap = cfg.bucket_capacity
    plan = P.plan_dp(params, cap, 2, "alpha-balanced", "numel", 1.0)
    loads = [float(x) for x in plan.rank_loads]
    assert max(loads) / (sum(loads) / 2) < 1.001
    owners = P.param_owners(params, cap, plan)
    ctxs = [DistributedMuon(params, cap, plan, rank=r, comm="none", grad_dtype="f32")
            for r in range(2)]
    w0, g0 = {}, {}
    for p in params:
        w0[p.id] = O.init_weight(p.shape, p.id, SEED)
        g0[p.id] = O.reduced_gradient(p.shape, p.id, SEED, 0, 2)
        for c in ctxs:
            c.load_param(p.id, w0[p.id])
            c.write_grad(p.id, g0[p.id])
    for c in ctxs:
        c.step(OptimizerConfig())
    got = {p.id: ctxs[owners[p.id]].read_param(p.id, "master").astype(np.float64) for p in params}
    for c in ctxs:
        c.close()
    O.set_fast_blas(True)
    ocfg = O.OptimizerConfig()
    worst = {}
    for p in params:
        w = w0[p.id].copy()
        O.muon_apply(p.is_matrix, ocfg, w, np.zeros_like(w), g0[p.id])
        gw = got[p.id].reshape(w.shape)
        e_dw = np.linalg.norm((gw - w0[p.id]) - (w - w0[p.id])) / np.linalg.norm(w - w0[p.id])
        e_w = np.abs(gw - w).max() / np.abs(w).max()
        tol_dw, tol_w = (TOL_DW, TOL_W) if p.is_matrix else (TOL_VEC, TOL_VEC)
        assert e_dw <= tol_dw and e_w <= tol_w, (p.name, e_dw, e_w)
        worst[p.name] = e_dw
    assert len(worst) == 143
