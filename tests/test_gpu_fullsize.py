"""Parity at the benchmark's FULL size (qwen3-8b-like, 7.28e9 parameters, one
B200): the whole model is stepped once through the product path, and the
tensors of the three non-vocabulary shape classes of layer 0 — qkv 4096x12288,
attn_out 4096x4096, ffn_down 12288x4096 (transposed in the momentum kernel) —
carry the reference generator's weights/gradients (verify.hpp:102-113) and are
compared with the fp64 oracle (oracle/, OpenBLAS dgemm) at the tolerances of
tests/test_gpu_parity.py. The vocabulary matrices (4096x151936, 51.7 TFLOP
per step in fp64 — minutes on the host) are checked through a size-independent
property instead: the applied update equals lr x an orthogonalised matrix,
so its singular values cluster in the quintic's band (test_verify.cpp:100-123
analogue: >= 99 % of them in (0.55, 1.45) for a Gaussian momentum).
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
TOL_DW, TOL_W = 3e-2, 2.5e-3


@pytest.fixture(scope="module")
def stepped():
    if torch.cuda.get_device_properties(0).total_memory < 150 * (1 << 30):
        pytest.skip("needs a 180 GB B200")
    cfg = P.load_config(os.path.join(ROOT, "configs", "qwen3-8b-like.cfg"))
    params = P.generate_transformer_params(cfg)
    cap = cfg.bucket_capacity
    plan = P.plan_dp(params, cap, 1, "alpha-balanced", "numel", 1.0)
    eng = DistributedMuon(params, cap, plan, rank=0, comm="nccl", grad_dtype="f32")
    eng.fill_synthetic(42, "weights")
    eng.fill_synthetic(1000, "grads")
    by_name = {p.name: p for p in params}
    chosen = [by_name[n] for n in ("layer0.qkv", "layer0.attn_out", "layer0.ffn_down")]
    vocab = [p for p in params if p.vocab_space and p.is_matrix]
    inputs = {}
    for p in chosen:
        w0 = O.init_weight(p.shape, p.id, SEED)
        g = O.reduced_gradient(p.shape, p.id, SEED, 0, 1)
        eng.load_param(p.id, w0)
        eng.write_grad(p.id, g)
        inputs[p.id] = (w0, g)
    before = {p.id: eng.read_param(p.id, "master") for p in vocab}
    eng.step(OptimizerConfig())
    eng.sync()
    after = {p.id: eng.read_param(p.id, "master") for p in chosen + vocab}
    eng.close()
    return chosen, vocab, inputs, before, after


def test_layer0_classes_match_fp64_oracle(stepped):
    chosen, _, inputs, _, after = stepped
    O.set_fast_blas(True)
    cfg = O.OptimizerConfig()
    for p in chosen:
        w0, g = inputs[p.id]
        w = w0.copy()
        mom = np.zeros_like(w)
        O.muon_apply(True, cfg, w, mom, g)
        got = after[p.id].astype(np.float64).reshape(w.shape)
        dw_ref, dw_got = w - w0, got - w0
        e_dw = np.linalg.norm(dw_got - dw_ref) / np.linalg.norm(dw_ref)
        e_w = np.abs(got - w).max() / np.abs(w).max()
        assert e_dw <= TOL_DW, (p.name, e_dw)
        assert e_w <= TOL_W, (p.name, e_w)


def test_vocab_update_is_orthogonalised(stepped):
    _, vocab, _, before, after = stepped
    lr = OptimizerConfig().lr
    for p in vocab:
        x = (torch.tensor(before[p.id]).cuda() - torch.tensor(after[p.id]).cuda()) / lr
        x = x.reshape(p.shape).double()
        if x.shape[0] > x.shape[1]:
            x = x.t()
        sv = torch.linalg.eigvalsh(x @ x.t()).clamp_min(0).sqrt()
        inside = ((sv > 0.55) & (sv < 1.45)).double().mean().item()
        assert inside >= 0.99, (p.name, inside, sv.min().item(), sv.max().item())
