"""The reference's Newton-Schulz properties (proj/tests/test_verify.cpp:57-136)
checked on the PRODUCT path: every input is a gradient of a tensor stepped
once through osh_step with lr = 1, beta = 0 and W0 = 0, so -W1 is exactly the
tcgen05 Newton-Schulz output (bf16 operands, fp32 accumulation).

  identity -> scalar multiple in (0.6, 1.4)            test_verify.cpp:57-68
  spread spectrum diag(2 .. 0.5) -> band (0.6, 1.4)    :70-81
  transposition commutes, EXACTLY (bitwise)            :83-93
  clamped spectra [0.5, 2] -> band (0.55, 1.45)        :100-123
  matrix update magnitude ~ lr * sqrt(min side)        :125-136
(Sizes are >= 8 per side: a TMA row is at least 16 bytes of bf16.)
"""
import numpy as np
import pytest

pytest.importorskip("torch")

from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig  # noqa: E402

pytestmark = pytest.mark.gpu


def ns_outputs(mats):
    ps = [P.ParamSpec(i, f"x{i}", m.shape) for i, m in enumerate(mats)]
    cap = max(p.numel for p in ps) * 4
    plan = P.plan_dp(ps, cap, 1, "alpha-balanced", "numel", 1.0)
    with DistributedMuon(ps, cap, plan, comm="none") as e:
        for p, m in zip(ps, mats):
            e.load_param(p.id, np.zeros(m.shape))
            e.write_grad(p.id, m)
        e.step(OptimizerConfig(lr=1.0, beta=0.0))
        e.sync()
        return [-e.read_param(p.id, "master").astype(np.float64).reshape(m.shape)
                for p, m in zip(ps, mats)]


def test_identity_stays_a_scalar_multiple():
    (y,) = ns_outputs([np.eye(8)])
    d = y[0, 0]
    assert np.allclose(y, d * np.eye(8), atol=1e-6 + 1e-2 * abs(d))
    assert 0.6 < d < 1.4


def test_spread_spectrum_lands_in_the_band():
    (y,) = ns_outputs([np.diag(np.linspace(2.0, 0.5, 8))])
    s = np.linalg.svd(y, compute_uv=False)
    assert (s > 0.6).all() and (s < 1.4).all(), s


def test_transposition_commutes_exactly():
    rng = np.random.default_rng(99)
    x = rng.standard_normal((24, 56))
    a, b = ns_outputs([x, np.ascontiguousarray(x.T)])
    assert np.array_equal(a.T, b)


def test_clamped_spectra_land_in_the_band():
    rng = np.random.default_rng(7)
    mats = []
    for _ in range(12):
        r, c = 8 * int(rng.integers(1, 9)), 8 * int(rng.integers(1, 9))
        u, s, vt = np.linalg.svd(rng.standard_normal((r, c)), full_matrices=False)
        mats.append((u * np.clip(s, 0.5, 2.0)) @ vt)
    for y in ns_outputs(mats):
        s = np.linalg.svd(y, compute_uv=False)
        assert (s > 0.55).all() and (s < 1.45).all(), s


def test_update_magnitude_tracks_the_orthogonal_scale():
    rng = np.random.default_rng(3)
    (y,) = ns_outputs([rng.standard_normal((64, 64)) / 8.0])
    ideal = np.sqrt(64.0)  # lr = 1
    assert 0.6 * ideal < np.linalg.norm(y) < 1.4 * ideal
