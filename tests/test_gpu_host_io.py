"""osh_step with HOST buffers (the e2e entry point a training loop uses):
gradients in from host memory, the updated bf16 replica out to host memory.

On a single rank and on the NCCL path the gradient is copied bucket by bucket
and each wave waits only for the buckets it reads; finished replica buckets
are copied back while later waves still run. The result must equal the
device-buffer path (write_grad + step + read the replica) BIT FOR BIT, for
pageable and pinned host memory, fp32 and bf16 gradients, overlapped and
back-to-back wave schedules.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig  # noqa: E402

pytestmark = pytest.mark.gpu
SEED = 42
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def params():
    shapes = [(1024, 3072), (1024,), (1024, 1024), (3072, 1024), (512, 1536), (1536, 512),
              (200, 328), (1024,), (4000, 1024), (64, 64)]
    return [P.ParamSpec(i, f"t{i}", s) for i, s in enumerate(shapes)]


def flat_grads(ps, step, dtype):
    g = np.concatenate([O.reduced_gradient(p.shape, p.id, SEED, step, 1).reshape(-1) for p in ps])
    t = torch.tensor(g.astype(np.float32))
    return t.bfloat16() if dtype == "bf16" else t


def run(ps, cap, grad_dtype, host, pinned, steps=3):
    plan = P.plan_dp(ps, cap, 1, "alpha-balanced", "numel", 1.0)
    eng = DistributedMuon(ps, cap, plan, rank=0, comm="nccl", grad_dtype=grad_dtype)
    assert eng.info()["n_buckets"] > 2
    for p in ps:
        eng.load_param(p.id, O.init_weight(p.shape, p.id, SEED))
    total = sum(p.numel for p in ps)
    out = torch.empty(total, dtype=torch.bfloat16, pin_memory=pinned)
    for s in range(steps):
        g = flat_grads(ps, s, grad_dtype)
        if host:
            hg = g.pin_memory() if pinned else g.clone()
            eng.step(OptimizerConfig(), host_grads=hg.data_ptr(), host_replica_out=out.data_ptr())
            eng.sync()
        else:
            off = 0
            for p in ps:
                eng.write_grad(p.id, g[off:off + p.numel].float().numpy())
                off += p.numel
            eng.step(OptimizerConfig())
            eng.sync()
    if not host:
        out = torch.cat([torch.tensor(eng.read_param(p.id, "replica").reshape(-1)).bfloat16()
                         for p in ps])
    eng.close()
    return out.float().numpy()


@pytest.mark.parametrize("grad_dtype", ["f32", "bf16"])
@pytest.mark.parametrize("pinned", [False, True])
def test_host_buffers_equal_device_path(grad_dtype, pinned):
    ps = params()
    cap = 4_200_000  # several buckets
    ref = run(ps, cap, grad_dtype, host=False, pinned=False)
    got = run(ps, cap, grad_dtype, host=True, pinned=pinned)
    assert np.array_equal(got, ref)


def test_host_buffers_back_to_back_schedule():
    env = dict(os.environ, OSH_OVERLAP="0")
    code = ("import sys; sys.path[:0] = [%r, %r]; import numpy as np; "
            "from test_gpu_host_io import run, params; ps = params(); "
            "a = run(ps, 4_200_000, 'bf16', False, False); b = run(ps, 4_200_000, 'bf16', True, True); "
            "print('EQUAL' if np.array_equal(a, b) else 'DIFF')" % (ROOT, os.path.join(ROOT, "tests")))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=600)
    assert "EQUAL" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]
