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
