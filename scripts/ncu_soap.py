"""Blocked-SOAP workload for ncu. Default: 12 x (4096 x 12288) matrices (576
blocks of 1024^2, the 8B FFN shapes), bf16 gradients. The first call
(statistics + the initial 4-iteration basis refresh) runs outside the
profiled range; the second, a regular step, is bracketed by
cudaProfilerStart/Stop:
    ncu --profile-from-start off --set full -k regex:"ns_gemm_kernel|soap_" \
        python scripts/ncu_soap.py
`--refresh` profiles the init call instead (the refresh kernels).
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig, SoapConfig  # noqa: E402

refresh = "--refresh" in sys.argv
ps = [P.ParamSpec(i, f"ffn{i}", (4096, 12288)) for i in range(12)]
plan = P.plan_dp(ps, 10 ** 10, 1, "alpha-balanced", "numel", 1.0)
with DistributedMuon(ps, 10 ** 10, plan, comm="none", grad_dtype="bf16", optimizer="soap",
                     shampoo=SoapConfig(block=1024, precond_every=10)) as e:
    e.fill_synthetic(42, "weights")
    e.fill_synthetic(7, "grads")
    e.sync()
    if refresh:
        torch.cuda.profiler.start()
    e.step(OptimizerConfig())
    e.sync()
    if refresh:
        torch.cuda.profiler.stop()
    else:
        torch.cuda.profiler.start()
        e.step(OptimizerConfig())
        e.sync()
        torch.cuda.profiler.stop()
print("ok")
