"""GPU Muon step (libosh.so, C ABI) against the fp64 oracle on the same inputs.

The oracle (oracle/muon_oracle.c) is pinned bit-for-bit to the reference's
verify.hpp (tests/test_oracle.py). The GPU iterates Newton-Schulz with bf16
operands and fp32 accumulation/state, so parity is a stated tolerance:

  TOL_DW  per-tensor relative Frobenius error of the last step's update
          ||dW_gpu - dW_ref|| / ||dW_ref||            <= 3e-2 (min side >= 64)
          <= 1e-1 for tiny matrices (min side < 64): their smallest singular
          directions are amplified ~a^k = 3.4445^5 ~ 480x by the quintic, so the
          bf16 operand rounding shows (toy 8x8: 5.9e-2 measured)
  TOL_W   max-abs error of the final weights relative to max|W_ref|  <= 2.5e-3
          (after <= 6 steps; measured <= 1.4e-3 on the toy model)
  TOL_N   relative error of the reported update norms ||lr*dW||      <= 3e-2
  vectors (plain momentum SGD in fp32)                                <= 1e-5

Bitwise property (reference test_verify.cpp:173-204 analogue): the sharded
run (R ranks, each updating only the tensors it owns) equals the R=1 run
bit for bit, because every tensor's computation is independent of which
tensors share its launches and all reductions are in a fixed order.
"""
import numpy as np
import pytest

pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig  # noqa: E402

pytestmark = pytest.mark.gpu

TOL_DW, TOL_DW_SMALL, TOL_W, TOL_N, TOL_VEC = 3e-2, 1e-1, 2.5e-3, 3e-2, 1e-5
SEED = 42


def toy_params(layers=2):
    cfg = P.ModelConfig(name="toy", num_layers=layers, hidden_size=8, ffn_size=16, num_heads=2,
                        vocab_size=12, bucket_capacity=200)
    return P.generate_transformer_params(cfg)


def mixed_params():
    """Every code path at moderate size: K-major/MN-major, transposed
    (rows > cols), ragged (non-multiple-of-tile) and vocab-like tall shapes."""
    shapes = [(1024, 3072), (1024, 1024), (3072, 1024), (1024,), (4000, 1024), (200, 328),
              (333, 96), (1024,), (64, 64)]
    return [P.ParamSpec(i, f"t{i}", s) for i, s in enumerate(shapes)]


def run_gpu(params, cap, ranks, steps, contributors, cfg=OptimizerConfig(), reset=None,
            grad_dtype="f32"):
    """R simulated ranks on one GPU (comm='none': gradients are reduced by the
    oracle and written to every rank). Returns (weights, norms per step,
    weights before the last step)."""
    plan = P.plan_dp(params, cap, ranks, "alpha-balanced", "numel", 1.0)
    owners = P.param_owners(params, cap, plan)
    ctxs = [DistributedMuon(params, cap, plan, rank=r, comm="none", grad_dtype=grad_dtype)
            for r in range(ranks)]
    for p in params:
        w0 = O.init_weight(p.shape, p.id, SEED)
        for c in ctxs:
            c.load_param(p.id, w0)
    norms, before = [], {}
    for step in range(steps):
        grads = {p.id: O.reduced_gradient(p.shape, p.id, SEED, step, contributors) for p in params}
        if reset is not None and step == reset[1]:
            pid = reset[0]  # cold momentum on a new host (FaultSpec semantics)
            c = ctxs[owners[pid]]
            c.load_param(pid, c.read_param(pid, "master"))
        if step == steps - 1:
            before = {p.id: ctxs[owners[p.id]].read_param(p.id, "master").astype(np.float64)
                      for p in params}
        for c in ctxs:
            for p in params:
                c.write_grad(p.id, grads[p.id])
            c.step(cfg)
        n = np.full(len(params), -1.0)
        for c in ctxs:
            un = c.update_norms()
            n = np.where(un >= 0, un, n)
        norms.append(n)
    weights = {p.id: ctxs[owners[p.id]].read_param(p.id, "master").astype(np.float64)
               for p in params}
    for c in ctxs:
        c.close()
    return weights, norms, before


def oracle_run(params, steps, contributors, reset=None):
    cfg = O.OptimizerConfig()
    w = {p.id: O.init_weight(p.shape, p.id, SEED) for p in params}
    m = {p.id: np.zeros_like(w[p.id]) for p in params}
    norms, before = [], {}
    for step in range(steps):
        if reset is not None and step == reset[1]:
            m[reset[0]] = np.zeros_like(m[reset[0]])
        if step == steps - 1:
            before = {k: v.copy() for k, v in w.items()}
        row = []
        for p in params:
            g = O.reduced_gradient(p.shape, p.id, SEED, step, contributors)
            row.append(O.muon_apply(len(p.shape) == 2, cfg, w[p.id], m[p.id], g))
        norms.append(np.array(row))
    return w, norms, before


def errors(params, got, ref):
    gw, gn, gb = got
    rw, rn, rb = ref
    out = {}
    for p in params:
        g1, g0 = gw[p.id].reshape(-1), gb[p.id].reshape(-1)
        r1, r0 = rw[p.id].reshape(-1), rb[p.id].reshape(-1)
        dg, dr = g1 - g0, r1 - r0
        out[p.id] = dict(
            dw=np.linalg.norm(dg - dr) / max(np.linalg.norm(dr), 1e-30),
            w=np.abs(g1 - r1).max() / max(np.abs(r1).max(), 1e-30),
            n=max(abs(a[p.id] - b[p.id]) / max(b[p.id], 1e-30) for a, b in zip(gn, rn)),
        )
    return out


def assert_within(params, errs):
    for p in params:
        e = errs[p.id]
        if p.is_matrix:
            tol_dw = TOL_DW if min(p.shape) >= 64 else TOL_DW_SMALL
            tol_n = TOL_N if min(p.shape) >= 64 else TOL_DW_SMALL
            assert e["dw"] <= tol_dw and e["w"] <= TOL_W and e["n"] <= tol_n, (p, e)
        else:
            assert e["dw"] <= TOL_VEC and e["w"] <= TOL_VEC and e["n"] <= TOL_VEC, (p, e)


@pytest.mark.parametrize("ranks,contributors", [(1, 1), (4, 4)])
def test_toy_model_matches_oracle(ranks, contributors):
    params = toy_params()
    got = run_gpu(params, 200, ranks, 6, contributors)
    ref = oracle_run(params, 6, contributors)
    errs = errors(params, got, ref)
    print({p.name: {k: f"{v:.2e}" for k, v in errs[p.id].items()} for p in params})
    assert_within(params, errs)


def test_sharded_equals_replicated_bitwise():
    params = toy_params(layers=4)
    one = run_gpu(params, 200, 1, 5, 4)
    four = run_gpu(params, 200, 4, 5, 4)
    for p in params:
        assert np.array_equal(one[0][p.id], four[0][p.id]), p.name
    assert all(np.array_equal(a, b) for a, b in zip(one[1], four[1]))


def test_mixed_shapes_match_oracle():
    params = mixed_params()
    O.set_fast_blas(True)
    try:
        ref = oracle_run(params, 3, 2)
    finally:
        O.set_fast_blas(False)
    got = run_gpu(params, 8_000_000, 2, 3, 2)
    errs = errors(params, got, ref)
    print({p.name: {k: f"{v:.2e}" for k, v in errs[p.id].items()} for p in params})
    assert_within(params, errs)


def test_cold_momentum_fault_is_detected():
    """FaultSpec analogue (verify.hpp:212-219): a tensor whose optimizer state
    lands on a cold host mid-run must break the tolerance."""
    params = toy_params()
    fault_pid = P.tp_plane_params(params)[0].id
    got = run_gpu(params, 200, 2, 6, 2, reset=(fault_pid, 3))
    ref = oracle_run(params, 6, 2)
    errs = errors(params, got, ref)
    assert errs[fault_pid]["w"] > TOL_W or errs[fault_pid]["dw"] > TOL_DW_SMALL
    others = [p for p in params if p.id != fault_pid]
    assert_within(others, errs)


def test_zero_gradient_and_zero_norm_passthrough():
    params = [P.ParamSpec(0, "m", (64, 96)), P.ParamSpec(1, "v", (64,))]
    plan = P.plan_dp(params, 10_000, 1)
    with DistributedMuon(params, 10_000, plan, comm="none") as c:
        w = [np.random.default_rng(0).standard_normal(p.shape).astype(np.float32) for p in params]
        for p in params:
            c.load_param(p.id, w[p.id])
        c.step()  # grads are zero, momentum is zero -> NS returns the zero iterate
        for p in params:
            assert np.array_equal(c.read_param(p.id, "master"), w[p.id])
        assert np.array_equal(c.update_norms(), [0.0, 0.0])


def test_bf16_gradients_close_to_fp32():
    params = mixed_params()[:3]
    a = run_gpu(params, 8_000_000, 1, 2, 1, grad_dtype="f32")
    b = run_gpu(params, 8_000_000, 1, 2, 1, grad_dtype="bf16")
    for p in params:
        rel = np.abs(a[0][p.id] - b[0][p.id]).max() / np.abs(a[0][p.id]).max()
        print("bf16-vs-f32", p.name, rel)
        assert rel < TOL_W, (p.name, rel)


def test_stream_k_gram_matches_oracle_and_is_plan_invariant(monkeypatch):
    """OSH_STREAM_K=1 (opt-in): a 4096 x 16384 matrix's GRAM (136 symmetric
    256 x 256 tiles, 256 k-blocks: more tiles than CTA pairs, a part-empty
    last round) runs its first round whole and cuts the 62 tail tiles into
    equal k-parts, finished by a fixed-order fixup. The cut points depend
    only on the matrix, so the result is the same bits whichever plan / wave
    the tensor lands in, and it matches the fp64 oracle."""
    monkeypatch.setenv("OSH_STREAM_K", "1")
    params = [P.ParamSpec(0, "wide", (4096, 16384)), P.ParamSpec(1, "m", (1024, 3072)),
              P.ParamSpec(2, "v", (4096,))]
    one = run_gpu(params, 100_000_000, 1, 1, 1)
    two = run_gpu(params, 100_000_000, 2, 1, 1)
    for p in params:
        assert np.array_equal(one[0][p.id], two[0][p.id]), p.name
    O.set_fast_blas(True)
    try:
        ref = oracle_run(params, 1, 1)
    finally:
        O.set_fast_blas(False)
    errs = errors(params, one, ref)
    print({p.name: {k: f"{v:.2e}" for k, v in errs[p.id].items()} for p in params})
    assert_within(params, errs)
    # the launch really was stream-K
    plan = P.plan_dp(params, 100_000_000, 1, "alpha-balanced", "numel", 1.0)
    with DistributedMuon(params, 100_000_000, plan, comm="none") as c:
        c.fill_synthetic(1, "weights")
        c.fill_synthetic(2, "grads")
        c.profile_gemm(True)
        c.step()
        c.sync()
        grams = [w for mode, _, _, _, w in c.gemm_profile_launches() if mode == "gram"]
        c.profile_gemm(False)
    assert grams and all("stream-k" in w for w in grams if "16384" in w), grams
