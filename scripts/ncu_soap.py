"""A small blocked-SOAP workload for ncu: 2 x (4096 x 4096) matrices (32
blocks of 1024^2), bf16 gradients, one init call (statistics + the initial
4-iteration basis refresh) and one regular step. Capture e.g.
    ncu --set full -k regex:"ns_gemm_kernel|soap_chol|soap_prep" -c 8 python scripts/ncu_soap.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig, SoapConfig  # noqa: E402

ps = [P.ParamSpec(0, "a", (4096, 4096)), P.ParamSpec(1, "b", (4096, 4096))]
plan = P.plan_dp(ps, 10 ** 9, 1, "alpha-balanced", "numel", 1.0)
with DistributedMuon(ps, 10 ** 9, plan, comm="none", grad_dtype="bf16", optimizer="soap",
                     shampoo=SoapConfig(block=1024, precond_every=10)) as e:
    e.fill_synthetic(42, "weights")
    e.fill_synthetic(7, "grads")
    for _ in range(2):
        e.step(OptimizerConfig())
    e.sync()
print("ok")
