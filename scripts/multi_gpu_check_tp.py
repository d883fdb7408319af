"""DP x TP correctness of the micro-group path (config C3 semantics).

    torchrun --nproc-per-node D*T --master-addr 127.0.0.1 scripts/multi_gpu_check_tp.py \
        D T [steps] [ckpt|-] [auto|nccl] [f32|bf16]

Collectives: "auto" takes NVLS on an NVSwitch node when D > 1 (the TP-plane
shards are reduced through the multicast gradient into the DP owner's copy
before the gather, and re-stored through the multicast replica after the
scatter); "nccl" forces the NCCL reduce / broadcast legs.

Global rank = d*T + t. Every rank loads the FULL initial weights, writes its
own gradient SHARD (the full synthetic gradient of contributor d split along
the tensor's TP dimension — SURVEY.md §8 D2 "TP input rule"), and runs the
real step: DP reduce-scatter -> per-micro-group gather to the TP host ->
full-matrix Muon -> scatter -> DP all-gather. The fp64 oracle runs:
  * TP-plane tensors (tp-splittable, not vocab-space): full-tensor Muon on the
    reduced full gradient (paper semantics);
  * vocab-space shards: Muon on each shard separately (reference-literal:
    they are not in the TP plane, verify.hpp:299-301);
  * vectors: full (replicated) momentum SGD.
Checks the tolerances of tests/test_gpu_parity.py and that every rank's bf16
replica shard equals bf16 of the final master. One JSON line on rank 0.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as td

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2602_06079_b200 import planner as P  # noqa: E402
from paper_2602_06079_b200.engine import (COLLECTIVE_NAMES, DistributedMuon, OptimizerConfig,  # noqa: E402
                                          nccl_unique_id)

SEED = 42


def shard_of(x, p, T, t):
    """TP shard t of a full array (workload.hpp:197-216 geometry)."""
    if p.tp_split == P.TP_ROW:
        r = x.shape[0] // T
        return x[t * r:(t + 1) * r]
    if p.tp_split == P.TP_COLUMN:
        c = x.shape[1] // T
        return x[:, t * c:(t + 1) * c]
    return x


def bf16(x):
    return torch.tensor(np.ascontiguousarray(x, dtype=np.float32)).bfloat16().float().numpy()


def main():
    D, T = int(sys.argv[1]), int(sys.argv[2])
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    ckpt = len(sys.argv) > 4 and sys.argv[4] == "ckpt"  # save / reload: replica rebuilt?
    coll = sys.argv[5] if len(sys.argv) > 5 else "auto"
    gdt = sys.argv[6] if len(sys.argv) > 6 else "f32"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert world == D * T
    d, t = rank // T, rank % T
    local = int(os.environ.get("LOCAL_RANK", rank))
    td.init_process_group("gloo")
    torch.cuda.set_device(local)
    cfg = P.ModelConfig(name="tpcheck", num_layers=2, hidden_size=256, ffn_size=768, num_heads=4,
                        vocab_size=1000)
    full = P.generate_transformer_params(cfg)
    shards = P.apply_tp_sharding(full, T)
    cap = 400_000
    plan = P.plan_dp(shards, cap, D, "alpha-balanced", "numel", 1.0)
    owners = P.param_owners(shards, cap, plan)
    # unique ids: DP group of tp rank t is created by global rank t, TP group of
    # dp rank d by global rank d*T
    mine = {"dp": nccl_unique_id() if d == 0 else None, "tp": nccl_unique_id() if t == 0 else None}
    allids = [None] * world
    td.all_gather_object(allids, mine)
    dp_uid, tp_uid = allids[t]["dp"], allids[d * T]["tp"]
    eng = DistributedMuon(full, cap, plan, rank=d, device=local, comm="nccl", nccl_uid=dp_uid,
                          grad_dtype=gdt, tp_rank=t, tp_size=T, tp_uid=tp_uid,
                          tp_capacity=200_000, collectives=coll)
    path = COLLECTIVE_NAMES[eng.info()["collectives"]]
    for p in full:
        eng.load_param(p.id, O.init_weight(p.shape, p.id, SEED).reshape(p.shape))
    norms = []
    for step in range(steps):
        for p in full:
            g = O.synth_gradient(p.shape, p.id, SEED, step, d).reshape(p.shape)
            eng.write_grad(p.id, shard_of(g, p, T, t))
        eng.step(OptimizerConfig())
        eng.sync()
        norms.append(eng.update_norms())
    res = {}
    for p in full:
        plane = p.tp_split != P.TP_NONE and not p.vocab_space
        if owners[p.id] != d:
            continue
        try:
            if plane:
                res[p.id] = ("full", eng.read_param(p.id, "master", shape=p.shape))
            else:
                res[p.id] = ("shard", eng.read_param(p.id, "master", shape=shards[p.id].shape))
        except Exception:
            pass  # TP-plane tensor hosted by the other TP rank
    replica = {p.id: eng.read_param(p.id, "replica", shape=shards[p.id].shape) for p in full}
    ckpt_ok = True
    if ckpt:
        # every rank saves its state, a FRESH ctx (zero replica) loads it: the
        # TP hosts' masters must come back as every rank's replica shards
        import tempfile
        path = os.path.join(tempfile.gettempdir(), f"osh_tp_ckpt_{os.getpid()}.osh")
        eng.save_state(path)
        eng.close()
        mine2 = {"dp": nccl_unique_id() if d == 0 else None, "tp": nccl_unique_id() if t == 0 else None}
        ids2 = [None] * world
        td.all_gather_object(ids2, mine2)
        eng = DistributedMuon(full, cap, plan, rank=d, device=local, comm="nccl",
                              nccl_uid=ids2[t]["dp"], grad_dtype=gdt, tp_rank=t, tp_size=T,
                              tp_uid=ids2[d * T]["tp"], tp_capacity=200_000, collectives=coll)
        eng.load_state(path)
        os.remove(path)
        again = {p.id: eng.read_param(p.id, "replica", shape=shards[p.id].shape) for p in full}
        ckpt_ok = all(np.array_equal(again[k], replica[k]) for k in replica)
    gathered = [None] * world
    td.all_gather_object(gathered, (d, t, res, norms, replica, ckpt_ok))
    eng.close()
    if rank != 0:
        return 0
    # ---- oracle
    ocfg = O.OptimizerConfig()
    ref_w = {}
    for p in full:
        w0 = O.init_weight(p.shape, p.id, SEED).reshape(p.shape) if p.is_matrix else \
            O.init_weight(p.shape, p.id, SEED).reshape(p.shape[0], 1)
        plane = p.tp_split != P.TP_NONE and not p.vocab_space
        pieces = [w0] if (plane or not p.is_matrix) else [np.ascontiguousarray(shard_of(w0, p, T, k))
                                                          for k in range(T)]
        moms = [np.zeros_like(x) for x in pieces]
        for s in range(steps):
            gfull = O.reduced_gradient(p.shape, p.id, SEED, s, D)
            gfull = gfull.reshape(p.shape) if p.is_matrix else gfull.reshape(-1, 1)
            gp = [gfull] if len(pieces) == 1 else [np.ascontiguousarray(shard_of(gfull, p, T, k))
                                                  for k in range(T)]
            for x, mo, g in zip(pieces, moms, gp):
                O.muon_apply(p.is_matrix, ocfg, x, mo, np.ascontiguousarray(g))
        ref_w[p.id] = pieces
    ok, report = True, {}
    for p in full:
        plane = p.tp_split != P.TP_NONE and not p.vocab_space
        found = [(gt, r[p.id]) for (gd, gt, r, _, _, _) in gathered if p.id in r]
        if not found:
            ok = False
            report[p.name] = {"ok": False, "why": "no rank returned it"}
            continue
        if plane or not p.is_matrix:
            got_full = found[0][1][1].reshape(p.shape)       # host (full) or replicated vector
            ref_full = ref_w[p.id][0].reshape(p.shape)
        else:  # vocab tensor: per-shard Muon on each TP rank of the owner
            parts = [a for _, (_, a) in sorted(found, key=lambda x: x[0])]
            axis = 0 if p.tp_split == P.TP_ROW else 1
            got_full = np.concatenate(parts, axis=axis)
            ref_full = np.concatenate(ref_w[p.id], axis=axis)
        e_w = float(np.abs(got_full - ref_full).max() / np.abs(ref_full).max())
        tol = 2.5e-3 if p.is_matrix else (1e-5 if gdt == "f32" else 1e-3)
        rep_ok = all(np.array_equal(rep[p.id].reshape(-1), bf16(shard_of(got_full, p, T, gt)).reshape(-1))
                     for (gd, gt, _, _, rep, _) in gathered)
        good = e_w <= tol and rep_ok
        ok &= good
        report[p.name] = {"owner": int(owners[p.id]), "tp_plane": plane, "w": f"{e_w:.2e}",
                          "replica_bitexact": rep_ok, "ok": good}
    ckpt_ok = all(g[5] for g in gathered)
    ok &= ckpt_ok
    print(json.dumps({"dp": D, "tp": T, "steps": steps, "collectives": path, "grad_dtype": gdt, "checkpoint_replica_ok": ckpt_ok if ckpt else None,
                      "ok": ok, "params": report}))
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
