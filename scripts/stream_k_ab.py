"""A/B of the stream-K GRAM on the vocabulary class (4096 x 151936), same
process, same GPU, alternating engines built with OSH_STREAM_K=1 and =0.
Prints per-variant median GRAM / step ms of one matrix's Muon step."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig  # noqa: E402

shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4096x151936").split("x"))
params = [P.ParamSpec(0, "vocab", shape)]
cap = shape[0] * shape[1]
plan = P.plan_dp(params, cap, 1)
engs = {}
for v in ("1", "0"):
    os.environ["OSH_STREAM_K"] = v
    e = DistributedMuon(params, cap, plan, comm="none", grad_dtype="bf16")
    e.fill_synthetic(1, "weights")
    e.fill_synthetic(2, "grads")
    engs[v] = e
res = {v: {"gram": [], "step": []} for v in engs}
for rnd in range(6):
    for v, e in engs.items():
        st = torch.cuda.ExternalStream(e.stream())
        e.step()
        e.sync()
        e.profile_gemm(True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        e.step()
        b.record(st)
        b.synchronize()
        e.sync()
        e.profile_gemm(False)
        g = sum(ms for mode, ms, _, _, _ in e.gemm_profile_launches() if mode == "gram")
        e.gemm_profile(reset=True)
        if rnd > 0:
            res[v]["gram"].append(g)
            res[v]["step"].append(a.elapsed_time(b))
out = {("stream_k" if v == "1" else "lpt"): {k: round(statistics.median(x), 3) for k, x in d.items()}
       for v, d in res.items()}
out["shape"] = "x".join(map(str, shape))
print(json.dumps(out))
