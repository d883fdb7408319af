"""The NCCL watchdog on real GPUs: a peer that dies mid-run must turn the
survivor's step into an OSH_ERR_NCCL error within the timeout, not a hang.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/watchdog_check.py

Rank 1 leaves right after both ranks built their contexts (os._exit: no
NCCL teardown, like a crashed process); rank 0 runs a step with host buffers
(osh_step waits on its streams) under a 15 s timeout. Prints one JSON line.
"""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as td

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_06079_b200 import _lib, planner as P  # noqa: E402
from paper_2602_06079_b200.engine import DistributedMuon, OptimizerConfig, nccl_unique_id  # noqa: E402

TIMEOUT = 15.0


def main():
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    td.init_process_group("gloo")
    torch.cuda.set_device(local)
    params = [P.ParamSpec(i, f"t{i}", s) for i, s in enumerate([(1024, 3072), (1024,), (3072, 1024)])]
    cap = 10_000_000
    plan = P.plan_dp(params, cap, 2, "alpha-balanced", "numel", 1.0)
    uid = [nccl_unique_id() if rank == 0 else None]
    td.broadcast_object_list(uid, src=0)
    eng = DistributedMuon(params, cap, plan, rank=rank, device=local, comm="nccl", nccl_uid=uid[0],
                          grad_dtype="bf16", collectives="nccl")
    eng.set_timeout(TIMEOUT)
    eng.fill_synthetic(42, "weights")
    eng.fill_synthetic(1000 + rank, "grads")
    eng.step(OptimizerConfig())  # one healthy step together
    eng.sync()
    td.barrier()
    if rank == 1:
        os._exit(0)  # the peer dies without tearing anything down
    total = sum(p.numel for p in params)
    hg = torch.zeros(total, dtype=torch.bfloat16).pin_memory()
    hr = torch.empty(total, dtype=torch.bfloat16).pin_memory()
    t0 = time.time()
    code, msg = 0, ""
    try:
        eng.step(OptimizerConfig(), host_grads=hg.data_ptr(), host_replica_out=hr.data_ptr())
        eng.sync()
    except _lib.OshError as e:
        code, msg = e.code, str(e)
    waited = time.time() - t0
    refused = None
    try:
        eng.step(OptimizerConfig())
    except _lib.OshError as e:
        refused = e.code
    ok = code == 17 and waited < TIMEOUT + 30 and refused == 17
    print(json.dumps({"ok": ok, "status": code, "waited_s": round(waited, 1), "timeout_s": TIMEOUT,
                      "next_step_status": refused, "message": msg[:300]}), flush=True)
    os._exit(0 if ok else 1)


if __name__ == "__main__":
    main()
