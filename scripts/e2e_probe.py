import os, sys, json, torch
sys.path.insert(0, ".")
from paper_2602_06079_b200 import planner as P
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig
cfg = P.load_config("configs/qwen3-8b-like.cfg")
params = P.generate_transformer_params(cfg)
plan = P.plan_dp(params, cfg.bucket_capacity, 1)
eng = DistributedMuon(params, cfg.bucket_capacity, plan, comm="nccl", grad_dtype="bf16")
eng.fill_synthetic(42, "weights"); eng.fill_synthetic(7, "grads")
total = eng.info()["total_numel"]
hg = torch.empty(total, dtype=torch.bfloat16, pin_memory=True); hr = torch.empty(total, dtype=torch.bfloat16, pin_memory=True)
hg.fill_(0.01)
st = torch.cuda.ExternalStream(eng.stream())
for _ in range(2): eng.step()
eng.sync()
out = {}
for mode in ("device", "h2d_only", "d2h_only", "both"):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kw = {}
    if mode in ("h2d_only", "both"): kw["host_grads"] = hg.data_ptr()
    if mode in ("d2h_only", "both"): kw["host_replica_out"] = hr.data_ptr()
    eng.step(OptimizerConfig(), **kw); eng.sync()
    a.record(st)
    for _ in range(4): eng.step(OptimizerConfig(), **kw)
    b.record(st); b.synchronize(); eng.sync()
    out[mode] = {"ms": round(a.elapsed_time(b) / 4, 1), "timing": {k: round(v, 1) for k, v in eng.timing().items() if isinstance(v, float)}}
# raw copy bandwidth
d = torch.empty(total, dtype=torch.bfloat16, device="cuda")
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); d.copy_(hg, non_blocking=True); b.record(); b.synchronize()
out["h2d_GBps"] = round(2 * total / a.elapsed_time(b) / 1e6, 1)
a.record(); hr.copy_(d, non_blocking=True); b.record(); b.synchronize()
out["d2h_GBps"] = round(2 * total / a.elapsed_time(b) / 1e6, 1)
print(json.dumps(out))
