"""Backward-pass overlap (osh_bucket_ready): gradients
announced bucket by bucket — in REVERSE bucket order, as a backward pass
produces them — give bit-for-bit the result of a plain step (single rank and
rank-simulated), and misuse is rejected."""
import numpy as np
import pytest

pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2602_06079_b200 import _lib  # noqa: E402
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig  # noqa: E402

pytestmark = pytest.mark.gpu
SEED = 42


def params():
    shapes = [(512, 768), (768,), (256, 256), (768, 512), (200, 328), (1024,), (64, 64)]
    return [P.ParamSpec(i, f"t{i}", s) for i, s in enumerate(shapes)]


def run(announce, ranks=1):
    ps = params()
    cap = 400_000
    plan = P.plan_dp(ps, cap, ranks, "alpha-balanced", "numel", 1.0)
    ctxs = [DistributedMuon(ps, cap, plan, rank=r, comm="none") for r in range(ranks)]
    out = []
    for c in ctxs:
        assert len(c.bucket_params()) > 2
        for p in ps:
            c.load_param(p.id, O.init_weight(p.shape, p.id, SEED))
        for s in range(3):
            if announce:
                for b in reversed(range(len(c.bucket_params()))):
                    for pid in c.bucket_params()[b]:
                        c.write_grad(pid, O.reduced_gradient(ps[pid].shape, pid, SEED, s, 1))
                    c.bucket_ready(b)
            else:
                for p in ps:
                    c.write_grad(p.id, O.reduced_gradient(p.shape, p.id, SEED, s, 1))
            c.step(OptimizerConfig())
        c.sync()
        out.append(c.read_param(0, "replica"))
    return out


@pytest.mark.parametrize("ranks", [1, 2])
def test_announced_buckets_equal_plain_step(ranks):
    a, b = run(False, ranks), run(True, ranks)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_partial_announcement_is_rejected():
    ps = params()
    plan = P.plan_dp(ps, 400_000, 1, "alpha-balanced", "numel", 1.0)
    c = DistributedMuon(ps, 400_000, plan, comm="none")
    c.bucket_ready(0)
    with pytest.raises(_lib.OshError):
        c.bucket_ready(0)  # twice
    with pytest.raises(_lib.OshError):
        c.step(OptimizerConfig())  # not every bucket
    c.step(OptimizerConfig())  # marks were reset: a plain step works
