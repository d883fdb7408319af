"""One Muon step of a single vocabulary-class matrix (default 4096 x 151936)
through the engine — for ncu captures of its GRAM / POLY / UPDATE / FINAL."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon  # noqa: E402

shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4096x151936").split("x"))
params = [P.ParamSpec(0, "vocab", shape)]
cap = shape[0] * shape[1]
with DistributedMuon(params, cap, P.plan_dp(params, cap, 1), comm="none", grad_dtype="bf16") as e:
    e.fill_synthetic(1, "weights")
    e.fill_synthetic(2, "grads")
    e.step()
    e.sync()
print("ok")
