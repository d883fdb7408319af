"""GPU blocked Shampoo (ShampooEngine through the C ABI) against the fp64
specification oracle/shampoo_oracle.py on the same inputs.

Parity is UNPINNED against the reference (it has no Shampoo mathematics, only
its cost, cost.hpp:47-48,68-75); the oracle is this build's specification.
Stated tolerances (bf16 G / P / U operands, fp32 statistics, inverse roots by
bf16x3 split GEMMs ~ fp32):
  TOL_DW  relative Frobenius error of the last step's update per tensor  <= 5e-2
  TOL_W   max error of the final weights relative to max|W_ref|         <= 2.5e-3
  vectors / vocabulary matrices (momentum SGD in fp32)                  <= 1e-5
Runs 4 steps with a root refresh every 2 steps (refresh and cached roots),
block 256 so tensors split into full and ragged blocks. The sharded run
(R = 2, comm none) equals the R = 1 run bit for bit.
"""
import numpy as np
import pytest

pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from oracle import shampoo_oracle as S  # noqa: E402
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig, ShampooConfig  # noqa: E402

pytestmark = pytest.mark.gpu
SEED = 42
TOL_DW, TOL_W, TOL_VEC = 5e-2, 2.5e-3, 1e-5
STEPS = 4


def params():
    shapes = [(512, 768), (768,), (256, 256), (200, 328), (333, 96), (1000, 256), (64, 64)]
    ps = [P.ParamSpec(i, f"t{i}", s) for i, s in enumerate(shapes)]
    ps[5] = P.ParamSpec(5, "vocab", (1000, 256), 2, 0, True)  # vocabulary: momentum SGD
    return ps


def run_gpu(ps, ranks, cfg, scfg, grad_dtype="f32"):
    cap = 10 ** 9
    plan = P.plan_dp(ps, cap, ranks, "alpha-balanced", "numel", 1.0)
    owners = P.param_owners(ps, cap, plan)
    ctxs = [DistributedMuon(ps, cap, plan, rank=r, comm="none", grad_dtype=grad_dtype,
                            optimizer="shampoo", shampoo=scfg) for r in range(ranks)]
    for p in ps:
        for c in ctxs:
            c.load_param(p.id, O.init_weight(p.shape, p.id, SEED))
    before = {}
    for s in range(STEPS):
        if s == STEPS - 1:
            before = {p.id: ctxs[owners[p.id]].read_param(p.id, "master").astype(np.float64)
                      for p in ps}
        for c in ctxs:
            for p in ps:
                c.write_grad(p.id, O.reduced_gradient(p.shape, p.id, SEED, s, 1))
            c.step(cfg)
    out = {p.id: ctxs[owners[p.id]].read_param(p.id, "master").astype(np.float64) for p in ps}
    for c in ctxs:
        c.close()
    return out, before


def oracle_run(ps, cfg, scfg):
    ocfg = S.ShampooConfig(lr=cfg.lr, beta1=cfg.beta, beta2=scfg.beta2, eps=scfg.eps,
                           block=scfg.block, precond_every=scfg.precond_every,
                           newton_iters=scfg.newton_iters)
    w = {p.id: O.init_weight(p.shape, p.id, SEED).reshape(S._shape2(p)) for p in ps}
    st = {p.id: S.ShampooTensorState(S._shape2(p), ocfg, S.is_preconditioned(p)) for p in ps}
    before = {}
    for s in range(STEPS):
        if s == STEPS - 1:
            before = {k: v.copy() for k, v in w.items()}
        for p in ps:
            g = O.reduced_gradient(p.shape, p.id, SEED, s, 1).reshape(S._shape2(p))
            S.shampoo_apply(st[p.id], ocfg, w[p.id], g, s)
    return w, before


@pytest.mark.parametrize("grad_dtype", ["f32", "bf16"])
def test_shampoo_matches_fp64_spec(grad_dtype):
    ps = params()
    cfg = OptimizerConfig(lr=0.02, beta=0.9)
    scfg = ShampooConfig(block=256, precond_every=2)
    got, got_before = run_gpu(ps, 1, cfg, scfg, grad_dtype)
    ref, ref_before = oracle_run(ps, cfg, scfg)
    for p in ps:
        g, r = got[p.id].reshape(-1), ref[p.id].reshape(-1)
        dg = g - got_before[p.id].reshape(-1)
        dr = r - ref_before[p.id].reshape(-1)
        e_w = np.abs(g - r).max() / np.abs(r).max()
        e_dw = np.linalg.norm(dg - dr) / np.linalg.norm(dr)
        pre = S.is_preconditioned(p)
        tol_dw = TOL_DW if pre else (TOL_VEC if grad_dtype == "f32" else 1e-2)
        assert e_dw <= tol_dw, (p.name, e_dw)
        assert e_w <= (TOL_W if pre or grad_dtype == "bf16" else TOL_VEC), (p.name, e_w)


def test_shampoo_sharded_equals_replicated_bitwise():
    ps = params()
    cfg = OptimizerConfig()
    scfg = ShampooConfig(block=256, precond_every=2)
    a, _ = run_gpu(ps, 1, cfg, scfg)
    b, _ = run_gpu(ps, 2, cfg, scfg)
    for p in ps:
        assert np.array_equal(a[p.id], b[p.id]), p.name


def test_shampoo_rejects_bad_config():
    ps = params()
    plan = P.plan_dp(ps, 10 ** 9, 1, "alpha-balanced", "numel", 1.0)
    with pytest.raises(Exception):
        DistributedMuon(ps, 10 ** 9, plan, comm="none", optimizer="shampoo",
                        shampoo=ShampooConfig(block=100))
