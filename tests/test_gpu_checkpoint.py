"""Sharded optimizer-state checkpoint keyed by the plan (osh_ctx_save_state /
osh_ctx_load_state): resuming from a checkpoint continues
the trajectory BIT FOR BIT (master, momentum, replica; Muon, Shampoo and
SOAP, including the Shampoo statistics, roots and refresh counter and the
SOAP statistics, bases, second moments and step counter), and a
checkpoint refuses to load under a different plan or rank.
"""
import numpy as np
import pytest

pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2602_06079_b200 import _lib  # noqa: E402
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import (DistributedMuon, OptimizerConfig, ShampooConfig,  # noqa: E402
                                          SoapConfig)

pytestmark = pytest.mark.gpu
SEED = 42


def params():
    shapes = [(512, 768), (768,), (256, 256), (200, 328), (1000, 256), (64, 64)]
    ps = [P.ParamSpec(i, f"t{i}", s) for i, s in enumerate(shapes)]
    ps[4] = P.ParamSpec(4, "vocab", (1000, 256), 2, 0, True)
    return ps


def make(ps, ranks, opt, method="alpha-balanced"):
    plan = P.plan_dp(ps, 600_000, ranks, method, "numel", 1.0)
    kw = (dict(optimizer=opt, shampoo=ShampooConfig(block=256, precond_every=2)) if opt == "shampoo"
          else dict(optimizer=opt, shampoo=SoapConfig(block=256, precond_every=2)) if opt == "soap"
          else {})
    return [DistributedMuon(ps, 600_000, plan, rank=r, comm="none", grad_dtype="f32", **kw)
            for r in range(ranks)]


def steps(ctxs, ps, s0, s1):
    for s in range(s0, s1):
        for c in ctxs:
            for p in ps:
                c.write_grad(p.id, O.reduced_gradient(p.shape, p.id, SEED, s, 1))
            c.step(OptimizerConfig())


def snapshot(ctxs, ps):
    out = []
    for r, c in enumerate(ctxs):
        d = {}
        for p in ps:
            try:
                d[("master", p.id)] = c.read_param(p.id, "master")
                d[("momentum", p.id)] = c.read_param(p.id, "momentum")
            except _lib.OshError:
                continue  # not owned by this rank (comm none: its replica slot is not ours)
            d[("replica", p.id)] = c.read_param(p.id, "replica")
        out.append(d)
    return out


@pytest.mark.parametrize("opt", ["muon", "shampoo", "soap"])
@pytest.mark.parametrize("ranks", [1, 2])
def test_resume_is_bit_exact(tmp_path, opt, ranks):
    ps = params()
    a = make(ps, ranks, opt)
    for c in a:
        for p in ps:
            c.load_param(p.id, O.init_weight(p.shape, p.id, SEED))
    steps(a, ps, 0, 3)
    for r, c in enumerate(a):
        c.save_state(str(tmp_path / f"rank{r}.osh"))
    steps(a, ps, 3, 6)
    want = snapshot(a, ps)
    for c in a:
        c.close()
    b = make(ps, ranks, opt)
    for r, c in enumerate(b):
        c.load_state(str(tmp_path / f"rank{r}.osh"))
    steps(b, ps, 3, 6)
    got = snapshot(b, ps)
    for r in range(ranks):
        assert want[r].keys() == got[r].keys()
        for k in want[r]:
            assert np.array_equal(want[r][k], got[r][k]), (r, k)
    for c in b:
        c.close()


def test_checkpoint_refuses_other_plan_or_rank(tmp_path):
    ps = params()
    a = make(ps, 2, "muon")
    a[0].save_state(str(tmp_path / "r0.osh"))
    p1 = P.plan_dp(ps, 600_000, 2, "alpha-balanced", "numel", 1.0)
    p2 = P.plan_dp(ps, 600_000, 2, "atomic-ownership", "numel", 1.0)
    assert [list(c) for c in p1.cut_vectors] != [list(c) for c in p2.cut_vectors]
    other = make(ps, 2, "muon", method="atomic-ownership")
    with pytest.raises(_lib.OshError) as e:
        other[0].load_state(str(tmp_path / "r0.osh"))
    assert e.value.code == 7
    with pytest.raises(_lib.OshError) as e:
        a[1].load_state(str(tmp_path / "r0.osh"))
    assert e.value.code == 7
    sh = make(ps, 2, "shampoo")
    with pytest.raises(_lib.OshError) as e:
        sh[0].load_state(str(tmp_path / "r0.osh"))
    assert e.value.code == 7
    ps2 = params()
    ps2[0] = P.ParamSpec(0, "t0", (512, 704))  # another model
    m2 = make(ps2, 2, "muon")
    with pytest.raises(_lib.OshError) as e:
        m2[0].load_state(str(tmp_path / "r0.osh"))
    assert e.value.code == 7


def test_damaged_checkpoint_leaves_state_untouched(tmp_path):
    """A truncated file, or one saved with another gradient dtype, is refused
    before any device state is written; saving goes through a temporary file
    that is renamed into place (no '.tmp' left behind)."""
    ps = params()
    a = make(ps, 1, "muon")
    for p in ps:
        a[0].load_param(p.id, O.init_weight(p.shape, p.id, SEED))
    steps(a, ps, 0, 2)
    path = tmp_path / "r0.osh"
    a[0].save_state(str(path))
    assert path.exists() and not (tmp_path / "r0.osh.tmp").exists()
    before = snapshot(a, ps)
    raw = path.read_bytes()
    cut = tmp_path / "cut.osh"
    cut.write_bytes(raw[: len(raw) - 4096])
    b = make(ps, 1, "muon")
    for p in ps:
        b[0].load_param(p.id, np.zeros(p.shape, np.float32))
    pristine = snapshot(b, ps)
    with pytest.raises(_lib.OshError) as e:
        b[0].load_state(str(cut))
    assert e.value.code == 7
    after = snapshot(b, ps)
    for k in pristine[0]:
        assert np.array_equal(pristine[0][k], after[0][k]), k  # nothing half restored
    plan = P.plan_dp(ps, 600_000, 1, "alpha-balanced", "numel", 1.0)
    with DistributedMuon(ps, 600_000, plan, comm="none", grad_dtype="bf16") as bf:
        with pytest.raises(_lib.OshError) as e:
            bf.load_state(str(path))
        assert e.value.code == 7
    b[0].load_state(str(path))  # the intact file still restores exactly
    got = snapshot(b, ps)
    for k in before[0]:
        assert np.array_equal(before[0][k], got[0][k]), k
