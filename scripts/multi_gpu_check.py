"""N-GPU correctness of the real NCCL path (RS-v -> owner Muon -> AG-v).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/multi_gpu_check.py [steps] [auto|nccl|nvls] [muon|shampoo|soap]

The optional second argument selects the DP collective path (engine.py
``collectives``); the JSON line reports the path the runtime actually took.

Every rank writes ITS OWN contributor gradient (synth_gradient(..., rank=r),
verify.hpp:102-107) into its local buckets; the NCCL reduce-scatter must
deliver sum_r g_r to the owner, the owner's Muon update must match the fp64
oracle (reduced_gradient with R contributors, ascending-rank sum) within the
tolerances of tests/test_gpu_parity.py, and after the all-gather every rank's
bf16 replica must equal bf16(owner's fp32 master) bit for bit.
Prints one JSON line on rank 0 and exits non-zero on failure.
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
from oracle import shampoo_oracle as S  # noqa: E402
from oracle import soap_oracle as SO  # noqa: E402
from paper_2602_06079_b200.engine import (COLLECTIVE_NAMES, DistributedMuon, OptimizerConfig,  # noqa: E402
                                          ShampooConfig, SoapConfig, nccl_unique_id)

SEED = 42
SCFG = ShampooConfig(block=512, precond_every=2)
SOCFG = SoapConfig(block=512, precond_every=2)


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    coll = sys.argv[2] if len(sys.argv) > 2 else "auto"
    opt = sys.argv[3] if len(sys.argv) > 3 else "muon"
    announce = len(sys.argv) > 4 and sys.argv[4] == "buckets"  # osh_bucket_ready, reverse order
    host = len(sys.argv) > 4 and sys.argv[4] in ("host", "host_owned")  # e2e entry: host buffers
    host_owned = len(sys.argv) > 4 and sys.argv[4] == "host_owned"  # D2H of own slices only
    ckpt = len(sys.argv) > 4 and sys.argv[4] == "ckpt"  # save / reload into a fresh ctx
    strategy = sys.argv[5] if len(sys.argv) > 5 else "sharded"  # or the sc / nv-layerwise baselines
    gdt = sys.argv[6] if len(sys.argv) > 6 else "f32"  # bf16: NVLS reduces bf16x8 with fp32 accumulation
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    td.init_process_group("gloo")
    torch.cuda.set_device(local)
    shapes = [(1024, 3072), (1024, 1024), (3072, 1024), (1024,), (4000, 1024), (200, 328),
              (333, 96), (1024,), (64, 64), (512, 1536), (1536, 512), (512,)]
    params = [P.ParamSpec(i, f"t{i}", s) for i, s in enumerate(shapes)]
    cap = int(os.environ.get("OSH_CHECK_CAP", 5_000_000))
    plan = P.plan_dp(params, cap, world, "alpha-balanced", "numel", 1.0)
    owners = P.param_owners(params, cap, plan)
    uid = [nccl_unique_id() if rank == 0 else None]
    td.broadcast_object_list(uid, src=0)
    eng = DistributedMuon(params, cap, plan, rank=rank, device=local, comm="nccl", nccl_uid=uid[0],
                          grad_dtype=gdt, collectives=coll, optimizer=opt,
                          shampoo=(SCFG if opt == "shampoo" else SOCFG if opt == "soap" else None),
                          strategy=strategy)
    path = COLLECTIVE_NAMES[eng.info()["collectives"]]
    # the ctx issues exactly the schedule the pure planner function exports
    # (the one tests/test_multi_rank_cpu.py executes over gloo)
    from paper_2602_06079_b200.engine import layer_groups
    sched_ok = eng.comm_schedule() == P.comm_schedule(
        params, cap, plan, strategy, layer_groups(params) if strategy == "nv-layerwise" else None)
    for p in params:
        eng.load_param(p.id, O.init_weight(p.shape, p.id, SEED))
    norms = []
    total = sum(p.numel for p in params)
    hrep = torch.empty(total, dtype=torch.bfloat16).pin_memory() if host else None
    if host_owned:
        eng.set_host_output("owned")
        hrep.view(torch.int16).fill_(-1)  # sentinel: slices of other ranks stay untouched
    for step in range(steps):
        if host:
            hg = torch.from_numpy(np.concatenate(
                [O.synth_gradient(p.shape, p.id, SEED, step, rank).reshape(-1) for p in params])
                .astype(np.float32))
            hg = (hg.bfloat16() if gdt == "bf16" else hg).pin_memory()
            eng.step(OptimizerConfig(), host_grads=hg.data_ptr(), host_replica_out=hrep.data_ptr())
            eng.sync()
            norms.append(eng.update_norms())
            continue
        if announce:
            for b in reversed(range(len(eng.bucket_params()))):
                for pid in eng.bucket_params()[b]:
                    eng.write_grad(pid, O.synth_gradient(params[pid].shape, pid, SEED, step, rank))
                eng.bucket_ready(b)
        else:
            for p in params:
                eng.write_grad(p.id, O.synth_gradient(p.shape, p.id, SEED, step, rank))
        eng.step(OptimizerConfig())
        eng.sync()
        norms.append(eng.update_norms())
    mine = {}
    for p in params:  # whatever this rank owns under its strategy
        try:
            mine[p.id] = eng.read_param(p.id, "master").astype(np.float64)
        except Exception:
            pass
    replica = {p.id: eng.read_param(p.id, "replica") for p in params}
    ckpt_ok = True
    if ckpt:
        # a FRESH ctx (zeroed replica) restored from this rank's file must
        # rebuild every rank's full replica from the owners' masters
        import tempfile
        path = os.path.join(tempfile.gettempdir(), f"osh_ckpt_{os.getpid()}.osh")
        eng.save_state(path)
        eng.close()
        uid2 = [nccl_unique_id() if rank == 0 else None]
        td.broadcast_object_list(uid2, src=0)
        eng = DistributedMuon(params, cap, plan, rank=rank, device=local, comm="nccl",
                              nccl_uid=uid2[0], grad_dtype=gdt, collectives=coll, optimizer=opt,
                              shampoo=(SCFG if opt == "shampoo" else SOCFG if opt == "soap" else None),
                              strategy=strategy)
        eng.load_state(path)
        os.remove(path)
        again = {p.id: eng.read_param(p.id, "replica") for p in params}
        ckpt_ok = all(np.array_equal(again[k], replica[k]) for k in replica)
    if host:  # the replica the step copied out must equal the device replica
        off = 0
        for p in params:
            got = hrep[off:off + p.numel]
            if host_owned and owners[p.id] != rank:  # another rank's result: untouched
                assert bool((got.view(torch.int16) == -1).all()), p.name
            else:
                assert np.array_equal(got.float().numpy(), replica[p.id].reshape(-1)), p.name
            off += p.numel
    gathered = [None] * world
    td.all_gather_object(gathered, (mine, norms, replica, ckpt_ok))
    eng.close()
    if rank != 0:
        return 0
    weights, gnorms = {}, np.full((steps, len(params)), -1.0)
    for m, n, _, _ in gathered:
        weights.update(m)
        for s in range(steps):
            gnorms[s] = np.where(n[s] >= 0, n[s], gnorms[s])
    # oracle with R contributors
    cfg = O.OptimizerConfig()
    w = {p.id: O.init_weight(p.shape, p.id, SEED) for p in params}
    mom = {p.id: np.zeros_like(w[p.id]) for p in params}
    rnorms = np.zeros((steps, len(params)))
    if opt == "shampoo":
        scfg = S.ShampooConfig(lr=cfg.lr, beta1=cfg.beta, beta2=SCFG.beta2, eps=SCFG.eps,
                               block=SCFG.block, precond_every=SCFG.precond_every,
                               newton_iters=SCFG.newton_iters)
        st = {p.id: S.ShampooTensorState(w[p.id].shape, scfg, S.is_preconditioned(p)) for p in params}
    if opt == "soap":
        socfg = SO.SoapConfig(lr=cfg.lr, beta1=cfg.beta, beta2=SOCFG.beta2, shampoo_beta=SOCFG.beta2,
                              eps=SOCFG.eps, block=SOCFG.block, precond_every=SOCFG.precond_every,
                              init_iters=SOCFG.init_iters)
        st = {p.id: SO.SoapTensorState(w[p.id].shape, socfg, SO.is_preconditioned(p)) for p in params}
    for s in range(steps):
        for p in params:
            if opt == "soap" and gdt == "bf16":
                # SOAP's basis is ill-conditioned in its statistics (DESIGN.md
                # 3c): the spec gets the GPU's input, the bf16 rank gradients
                # summed in fp32 and rounded to bf16 (multimem.ld_reduce
                # .acc::f32 .bf16x2 and NCCL's bf16 reduction alike)
                acc = sum(torch.from_numpy(O.synth_gradient(p.shape, p.id, SEED, s, r))
                          .bfloat16().float() for r in range(world))
                g = acc.bfloat16().double().numpy()
            else:
                g = O.reduced_gradient(p.shape, p.id, SEED, s, world)
            if opt == "shampoo":
                rnorms[s, p.id] = S.shampoo_apply(st[p.id], scfg, w[p.id], g.reshape(w[p.id].shape), s)
            elif opt == "soap":
                rnorms[s, p.id] = SO.soap_apply(st[p.id], socfg, w[p.id], g.reshape(w[p.id].shape), s)
            else:
                rnorms[s, p.id] = O.muon_apply(p.is_matrix, cfg, w[p.id], mom[p.id], g)
    ckpt_all = all(g[3] for g in gathered)
    report, ok = {}, sched_ok and ckpt_all
    for p in params:
        got, ref = weights[p.id].reshape(-1), w[p.id].reshape(-1)
        e_w = float(np.abs(got - ref).max() / np.abs(ref).max())
        live = rnorms[:, p.id] > 0  # (SOAP's first call only builds its statistics)
        e_n = float(np.max(np.abs(gnorms[live, p.id] - rnorms[live, p.id]) / rnorms[live, p.id]))
        tol_w = 2.5e-3 if p.is_matrix else (1e-5 if gdt == "f32" else 1e-3)
        tol_n = (3e-2 if min(p.shape) >= 64 else 1e-1) if p.is_matrix else (1e-5 if gdt == "f32" else 1e-2)
        if opt == "shampoo" and p.is_matrix:
            tol_n = 5e-2
        if opt == "soap" and p.is_matrix:
            # Adam-type steps move every element by ~lr and a handful of
            # near-zero rotated entries may flip: judge the direction of the
            # total change in Frobenius norm (tests/test_gpu_soap.py tolerances)
            w0 = O.init_weight(p.shape, p.id, SEED).reshape(-1).astype(np.float64)
            e_w = float(np.linalg.norm((got - w0) - (ref - w0)) / np.linalg.norm(ref - w0))
            # (elongated blocks rotate only their short side — soap_oracle.py
            # frozen(): the rank-deficient side's basis is not data-determined)
            tol_n, tol_w = 5e-2, 5e-2
        rep_ok = all(np.array_equal(g[2][p.id].reshape(-1),
                                    torch.tensor(weights[p.id].reshape(-1)).float().bfloat16().float().numpy())
                     for g in gathered)
        good = e_w <= tol_w and e_n <= tol_n and rep_ok
        ok &= good
        report[p.name] = {"plan_owner": int(owners[p.id]), "w": f"{e_w:.2e}", "norm": f"{e_n:.2e}",
                          "replica_bitexact": rep_ok, "ok": good}
    print(json.dumps({"world": world, "steps": steps, "collectives": path, "optimizer": opt,
                      "bucket_ready": announce, "host_buffers": host, "strategy": strategy,
                      "grad_dtype": gdt, "schedule_matches": sched_ok,
                      "checkpoint_replica_ok": ckpt_all if ckpt else None, "ok": ok,
                      "params": report}))
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
