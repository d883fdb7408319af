"""N>1 host-side logic on CPU with real processes (torch.distributed gloo).

Every rank plans independently through the C ABI (as every GPU process of
bench.py does), then the ranks exchange what they computed:
  * all ranks hold byte-identical plans and owner tables (the planner is a
    pure function: SPEC.md "same inputs, same bytes out"),
  * owned tensor sets partition the parameter list and owned slices tile
    every bucket (the RS-v / AG-v counts NCCL will be given),
  * bench.py's plumbing (NCCL unique-id broadcast, all-gather of per-rank
    records) round-trips.
"""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as td  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    from paper_2602_06079_b200 import planner as P

    try:
        dist = bench.Dist()
        cfg = P.load_config(os.path.join(ROOT, "configs", "qwen3-8b-like.cfg"))
        params = P.generate_transformer_params(cfg)
        text = P.serialize_dp_plan(params, cfg.bucket_capacity, world)
        plan = P.plan_dp(params, cfg.bucket_capacity, world)
        owners = P.param_owners(params, cfg.bucket_capacity, plan).tolist()
        layout = P.build_buffer_layout(params, cfg.bucket_capacity)
        owned = [p.id for p in params if owners[p.id] == rank]
        slices = [(int(c[rank]), int(c[rank + 1])) for c in plan.cut_vectors]
        uid = dist.bcast_bytes(bytes(range(128)) if rank == 0 else None)
        recs = dist.gather({"text": text, "owners": owners, "owned": owned, "slices": slices,
                            "uid": uid, "numel": [int(x) for x in layout.bucket_numel]})
        if rank == 0:
            q.put(recs)
        dist.barrier()
        td.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(repr(e))


@pytest.mark.parametrize("world", [2, 4])
def test_ranks_agree_and_partition(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    recs = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert not isinstance(recs, str), recs
    assert len(recs) == world
    assert all(r["text"] == recs[0]["text"] for r in recs)
    assert all(r["owners"] == recs[0]["owners"] for r in recs)
    assert all(r["uid"] == bytes(range(128)) for r in recs)
    owned = sorted(pid for r in recs for pid in r["owned"])
    assert owned == list(range(len(recs[0]["owners"])))
    for b, numel in enumerate(recs[0]["numel"]):
        edges = [recs[r]["slices"][b] for r in range(world)]
        assert edges[0][0] == 0 and edges[-1][1] == numel
        assert all(edges[r][1] == edges[r + 1][0] for r in range(world - 1))


# ---------------------------------------------------------------------------
# The DP data plane executed on CPU: the RS-v / AG-v schedule the runtime hands
# NCCL (osh_comm_schedule, the function csrc/runtime.cu builds its collectives
# from) is run over gloo on the oracle's per-rank gradients.
SEED = 42


def _exchange_worker(rank, world, port, q, strategy):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import numpy as np

    from oracle import oracle as O
    from paper_2602_06079_b200 import planner as P
    from paper_2602_06079_b200.engine import layer_groups

    try:
        td.init_process_group("gloo", rank=rank, world_size=world)
        cfg = P.ModelConfig(name="x", num_layers=2, hidden_size=64, ffn_size=192, num_heads=4,
                            vocab_size=500, bucket_capacity=45_000)
        params = P.generate_transformer_params(cfg)
        cap = cfg.bucket_capacity
        plan = P.plan_dp(params, cap, world, "alpha-balanced", "numel", 1.0)
        lay = layer_groups(params) if strategy == "nv-layerwise" else None
        sched = P.comm_schedule(params, cap, plan, strategy, lay)
        flat = {}
        off = 0
        for p in params:
            flat[p.id] = off
            off += p.numel
        total = off
        step = 0
        # this rank's contributor gradient (verify.hpp:102-107), flat declaration order
        grad = torch.from_numpy(np.concatenate(
            [O.synth_gradient(p.shape, p.id, SEED, step, rank).reshape(-1) for p in params]))
        owned_sizes = sum(o["count"] for o in sched if o["kind"] == "reduce" and o["root"] == rank)
        reduced = torch.full((max(owned_sizes, 1),), float("nan"), dtype=torch.float64)
        replica = torch.full((total,), -1.0, dtype=torch.bfloat16)
        # ---- RS leg, in issue order (every rank walks the same list)
        for o in sched:
            if o["phase"] != "rs":
                continue
            t = grad[o["offset"]:o["offset"] + o["count"]].clone()
            if o["kind"] == "reduce":
                td.reduce(t, dst=o["root"], op=td.ReduceOp.SUM)
                if rank == o["root"]:
                    reduced[o["dst_offset"]:o["dst_offset"] + o["count"]] = t
            else:  # allreduce (SC / NV-layerwise)
                td.all_reduce(t, op=td.ReduceOp.SUM)
                grad[o["offset"]:o["offset"] + o["count"]] = t
        # ---- owners: the oracle's Muon on the reduced slice
        owners = (P.param_owners(params, cap, plan) if strategy == "sharded"
                  else None)
        if strategy == "nv-layerwise":
            owners = np.zeros(len(params), np.int64)
            for o in sched:
                if o["phase"] == "ag":
                    pid = next(p.id for p in params if flat[p.id] == o["offset"])
                    owners[pid] = o["root"]
        ocfg = O.OptimizerConfig()
        sum_err, exact = 0.0, True
        for p in params:
            if strategy != "sc" and owners[p.id] != rank:
                continue
            ref = O.reduced_gradient(p.shape, p.id, SEED, step, world).reshape(-1)
            if strategy == "sharded":
                b = next(o for o in sched if o["kind"] == "reduce" and o["root"] == rank
                         and o["offset"] <= flat[p.id] < o["offset"] + o["count"])
                at = b["dst_offset"] + flat[p.id] - b["offset"]
                g = reduced[at:at + p.numel].numpy()
            else:
                g = grad[flat[p.id]:flat[p.id] + p.numel].numpy()
            exact &= bool(np.array_equal(g, ref))
            sum_err = max(sum_err, float(np.abs(g - ref).max() / max(np.abs(ref).max(), 1e-300)))
            w = O.init_weight(p.shape, p.id, SEED)
            m = np.zeros_like(w)
            O.muon_apply(p.is_matrix, ocfg, w, m, g.reshape(w.shape).copy())
            replica[flat[p.id]:flat[p.id] + p.numel] = torch.from_numpy(w.reshape(-1)).to(torch.bfloat16)
        # ---- AG leg: in-place broadcasts of the owners' bf16 slices
        for o in sched:
            if o["phase"] != "ag":
                continue
            t = replica[o["offset"]:o["offset"] + o["count"]].view(torch.uint8).clone()  # (gloo has no 16-bit ints)
            td.broadcast(t, src=o["root"])
            replica[o["offset"]:o["offset"] + o["count"]] = t.view(torch.bfloat16)
        # every rank's replica against the replicated oracle (run_replicated, R contributors)
        want = torch.cat([torch.from_numpy(
            O.run_replicated([p], ocfg, 1, SEED, world).final_weights[p.id].reshape(-1))
            .to(torch.bfloat16) for p in params])
        rep_ok = bool(torch.equal(replica.view(torch.int16), want.view(torch.int16)))
        rec = {"rank": rank, "n_ops": len(sched), "exact_sum": exact, "sum_err": sum_err,
               "replica_ok": rep_ok, "sched": sched}
        out = [None] * world
        td.all_gather_object(out, rec)
        if rank == 0:
            q.put(out)
        td.barrier()
        td.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback

        q.put(repr(e) + traceback.format_exc())


@pytest.mark.parametrize("world,strategy", [(2, "sharded"), (4, "sharded"), (4, "nv-layerwise"),
                                            (2, "sc")])
def test_dp_exchange_schedule_over_gloo(world, strategy):
    """RS-v delivers the ascending-rank gradient sum (verify.hpp:180-186) to
    each slice owner; after the owners' Muon, AG-v leaves every rank with the
    owner's bf16 master (the replica the next forward pass reads)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q, strategy))
             for r in range(world)]
    for p in procs:
        p.start()
    recs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert not isinstance(recs, str), recs
    assert all(r["sched"] == recs[0]["sched"] for r in recs)  # identical on every rank
    kinds = {o["kind"] for o in recs[0]["sched"]}
    assert kinds == ({"reduce", "broadcast"} if strategy == "sharded" else
                     {"allreduce", "broadcast"} if strategy == "nv-layerwise" else {"allreduce"})
    for r in recs:
        # gloo sums in its own order for > 2 ranks (as NCCL does): exact for
        # two contributors, within a few ulp of the ascending-rank sum beyond
        assert r["exact_sum"] or (world > 2 and r["sum_err"] < 1e-14), r["sum_err"]
        assert r["replica_ok"], f"rank {r['rank']}: replica differs from bf16(owner master)"
