"""Real multi-GPU paths (NCCL over NVLink): run the torchrun checks when the
box has enough GPUs (skipped on single-GPU boxes; the CPU-side multi-rank
logic is covered by tests/test_multi_rank_cpu.py).

* scripts/multi_gpu_check.py     DP ZeRO-1: RS-v -> owner Muon -> AG-v vs the
                                 fp64 oracle with R real contributors
* scripts/multi_gpu_check_tp.py  DP x TP micro-group gather/host-Muon/scatter
"""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(nproc, script, *args):
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "scripts", script), *map(str, args)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert lines, out.stdout[-2000:] + out.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"], json.dumps(res)[:3000]
    return res


def test_dp2_nccl_matches_oracle():
    res = _run(2, "multi_gpu_check.py", 3, "nccl")
    assert res["collectives"] == "nccl"


def test_dp2_auto_matches_oracle():
    # NVLS-fused reduce / broadcast when the box has NVSwitch multicast
    _run(2, "multi_gpu_check.py", 3, "auto")


def test_tp2_micro_groups_match_oracle():
    _run(2, "multi_gpu_check_tp.py", 1, 2, 3)


@pytest.mark.parametrize("coll,gdt", [("auto", "f32"), ("nccl", "f32"), ("auto", "bf16")])
def test_dp2_tp2_micro_groups_match_oracle(coll, gdt):
    # auto = NVLS on NVSwitch boxes: TP-plane shards reduced through the
    # multicast gradient before the gathers, scattered shards re-stored
    # through the multicast replica; nccl = NCCL reduce / broadcast legs
    res = _run(4, "multi_gpu_check_tp.py", 2, 2, 3, "-", coll, gdt)
    if coll == "nccl":
        assert res["collectives"] == "nccl"
    assert res["grad_dtype"] == gdt


def test_stage_overlap_opt_in_matches_oracle(monkeypatch):
    # OSH_SEQ_OVERLAP=1: momentum of stage i+1 beside the GEMMs of stage i on
    # the NCCL RS-v / AG-v path and across TP micro groups (opt-in schedule)
    monkeypatch.setenv("OSH_SEQ_OVERLAP", "1")
    assert _run(2, "multi_gpu_check.py", 3, "nccl")["collectives"] == "nccl"
    _run(2, "multi_gpu_check_tp.py", 1, 2, 3)


def test_dp2_nccl_bucket_ready_matches_oracle():
    # gradients announced bucket by bucket in reverse order: the RS-v of each
    # bucket starts before the next one is written (backward overlap)
    res = _run(2, "multi_gpu_check.py", 3, "nccl", "muon", "buckets")
    assert res["bucket_ready"]


def test_dp2_host_buffers_nvls_and_nccl():
    # the e2e entry (host gradients in, replica out) on both collective paths,
    # whole replica and own slices only (OSH_HOST_OUT_OWNED)
    for coll in ("auto", "nccl"):
        for mode in ("host", "host_owned"):
            res = _run(2, "multi_gpu_check.py", 2, coll, "muon", mode)
            assert res["host_buffers"]


@pytest.mark.parametrize("strategy", ["sc", "nv-layerwise"])
def test_dp2_baseline_strategies_match_oracle(strategy):
    # the paper's baselines executed for real: same trajectory as the oracle
    res = _run(2, "multi_gpu_check.py", 2, "auto", "muon", "-", strategy)
    assert res["strategy"] == strategy


def test_dp2_bf16_gradients_both_paths():
    # bf16 gradients: NVLS multimem.ld_reduce (bf16x8, fp32 accumulation in
    # the switch) and NCCL's bf16 reduce against the fp64 oracle
    for coll in ("auto", "nccl"):
        res = _run(2, "multi_gpu_check.py", 2, coll, "muon", "-", "sharded", "bf16")
        assert res["grad_dtype"] == "bf16"


def test_dp2_shampoo_matches_spec():
    res = _run(2, "multi_gpu_check.py", 3, "auto", "shampoo")
    assert res["optimizer"] == "shampoo"


def test_dp2_soap_matches_spec():
    # NVLS-fused prep / apply and the NCCL RS-v / AG-v path. f32 gradients:
    # SOAP's basis amplifies input differences ~3000x, so the
    # spec must see bit-identical reduced gradients; bf16-gradient parity is
    # pinned single-GPU (tests/test_gpu_soap.py) where the inputs are exact
    for coll, gdt in (("auto", "f32"), ("nccl", "f32")):
        res = _run(2, "multi_gpu_check.py", 4, coll, "soap", "-", "sharded", gdt)
        assert res["optimizer"] == "soap"


def test_dp4_nccl_matches_oracle():
    _run(4, "multi_gpu_check.py", 3, "nccl")


def test_dp4_auto_matches_oracle():
    _run(4, "multi_gpu_check.py", 3, "auto")


@pytest.mark.parametrize("strategy,coll", [("nv-layerwise", "nccl"), ("sharded", "auto")])
def test_dp2_checkpoint_restores_replica(strategy, coll):
    # a fresh ctx restored from each rank's file rebuilds every rank's replica
    # (NV-layerwise: broadcast from the layer owners, not the plan's cuts)
    res = _run(2, "multi_gpu_check.py", 2, coll, "muon", "ckpt", strategy)
    assert res["checkpoint_replica_ok"] is True


def test_tp2_checkpoint_restores_replica():
    # TP hosts cast their full masters and scatter the shards on resume
    res = _run(2, "multi_gpu_check_tp.py", 1, 2, 2, "ckpt")
    assert res["checkpoint_replica_ok"] is True


@pytest.mark.parametrize("coll", ["auto", "nccl"])
def test_dp2_tp2_checkpoint_restores_replica(coll):
    res = _run(4, "multi_gpu_check_tp.py", 2, 2, 2, "ckpt", coll)
    assert res["checkpoint_replica_ok"] is True


def test_dp2_watchdog_turns_dead_peer_into_error():
    # a peer dies mid-run: the survivor's step returns OSH_ERR_NCCL within the
    # timeout (communicators aborted) instead of hanging
    res = _run(2, "watchdog_check.py")
    assert res["status"] == 17 and res["next_step_status"] == 17
