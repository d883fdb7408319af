"""One profiled step's launch timeline per rank (which kernels ran when, and
the idle gaps between them on the rank's streams), for the DP x TP or DP
step of the 8B config.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 scripts/timeline.py TP [auto|nccl] [out_dir]

Writes <out_dir>/timeline_rank<r>.json: step ms, the launches (mode, start,
ms), the union of their busy time and the gaps longer than 0.3 ms.
"""
import json
import os
import sys

import torch
import torch.distributed as td

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig, nccl_unique_id  # noqa: E402


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    coll = sys.argv[2] if len(sys.argv) > 2 else "auto"
    out_dir = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/timeline"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    D = world // T
    d, t = rank // T, rank % T
    td.init_process_group("gloo")
    torch.cuda.set_device(local)
    cfg = P.load_config(os.path.join(ROOT, "configs", "qwen3-8b-like.cfg"))
    params = P.generate_transformer_params(cfg)
    view = P.apply_tp_sharding(params, T)
    cap = cfg.bucket_capacity // T
    plan = P.plan_dp(view, cap, D, "alpha-balanced", "numel", 1.0)
    mine = {"dp": nccl_unique_id() if d == 0 and D > 1 else None,
            "tp": nccl_unique_id() if t == 0 and T > 1 else None}
    ids = [None] * world
    td.all_gather_object(ids, mine)
    eng = DistributedMuon(params, cap, plan, rank=d, device=local, comm="nccl", nccl_uid=ids[t]["dp"],
                          grad_dtype="bf16", tp_rank=t, tp_size=T,
                          tp_uid=ids[d * T]["tp"] if T > 1 else None,
                          tp_capacity=268435456 if T > 1 else None, collectives=coll)
    eng.fill_synthetic(42, "weights")
    eng.fill_synthetic(1000 + rank, "grads")
    for _ in range(3):
        eng.step(OptimizerConfig())
    eng.sync()
    td.barrier()
    eng.profile_gemm(True)
    eng.step(OptimizerConfig())
    eng.sync()
    eng.profile_gemm(False)
    tl = eng.gemm_profile_timeline()
    tm = eng.timing()
    # busy union and gaps
    iv = sorted((s, s + ms, m) for m, s, ms, _ in tl)
    busy, gaps, cur_s, cur_e, last_mode = 0.0, [], None, None, None
    for s, e, m in iv:
        if cur_e is None:
            cur_s, cur_e, last_mode = s, e, m
            continue
        if s > cur_e:
            busy += cur_e - cur_s
            if s - cur_e > 0.3:
                gaps.append({"at": round(cur_e, 3), "ms": round(s - cur_e, 3), "after": last_mode, "before": m})
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
        last_mode = m if e >= cur_e else last_mode
    if cur_e is not None:
        busy += cur_e - cur_s
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, f"timeline_rank{rank}.json"), "w") as f:
        json.dump({"rank": rank, "dp": d, "tp": t, "collectives": coll, "timing": tm,
                   "first_launch_ms": round(iv[0][0], 3) if iv else None,
                   "last_end_ms": round(max(e for _, e, _ in iv), 3) if iv else None,
                   "busy_union_ms": round(busy, 3), "gaps": gaps,
                   "launches": [(m, round(s, 3), round(ms, 3)) for m, s, ms, _ in tl]}, f)
    eng.close()
    td.barrier()
    if rank == 0:
        print(json.dumps({"ok": True}))


if __name__ == "__main__":
    main()
