#!/usr/bin/env python
"""bench.py — Canzona distributed Muon optimizer step, Qwen3-8B shapes, on B200.

One "step" = the reference's distributed optimizer step executed for real
(SURVEY.md §8 D1): from "every rank holds its local bf16 gradient buckets" to
"every rank holds the updated bf16 replica": variable-size NCCL reduce-scatter
to the alpha-balanced owners -> per-owner Muon (momentum + 5 quintic
Newton-Schulz iterations on tcgen05 + fused weight update) -> variable-size
NCCL all-gather. Workload: configs/qwen3-8b-like.cfg (183 tensors, 7.28e9
params, 12 buckets of <= 622,329,856 elements), plan alpha-balanced alpha=1
numel over N = --gpus data-parallel ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torch.distributed.run (one process per GPU); torch's gloo
group only carries the NCCL unique id and the max-over-ranks reductions.
Rank 0 prints ONE JSON line. `value` is the device-resident step time (CUDA
events on the ctx's compute stream, max over ranks); `e2e` repeats the step
through the C ABI with host (pinned) gradients in and the updated replica out.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Muon optimizer step ms (Qwen3-8B shapes) at 1/2/4/8 B200; max/mean rank load"
METRIC_SHAMPOO = ("Shampoo optimizer step ms (Qwen3-8B shapes, builder-defined blocked Shampoo; "
                  "not the BASELINE metric); max/mean rank load")
CONFIG = os.path.join(ROOT, "configs", "qwen3-8b-like.cfg")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--alpha", default="auto",
                    help="alpha of the alpha-balanced plan, or 'auto': the alpha of {1, .75, .5, "
                         ".25, 0} with the lowest planned per-rank NS-flop max/mean, kept at 1 "
                         "unless another plans > 1.5 %% better (planner.choose_alpha)")
    ap.add_argument("--method", default="alpha-balanced",
                    choices=["alpha-balanced", "atomic-ownership"],
                    help="executable (atomic) partition; equal-chunk splits tensors, see "
                         "scripts/plan_sweep.py")
    ap.add_argument("--cost", default="numel")
    ap.add_argument("--grad-dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workspace-gb", type=float, default=0.0)
    ap.add_argument("--optimizer", default="muon", choices=["muon", "shampoo", "soap"],
                    help="muon = the headline metric; shampoo / soap = builder-defined blocked "
                         "Shampoo / SOAP")
    ap.add_argument("--shampoo-block", type=int, default=1024)
    ap.add_argument("--precond-every", type=int, default=10)
    ap.add_argument("--strategy", default="sharded", choices=["sharded", "sc", "nv-layerwise"],
                    help="sharded = the plan's owners (LB-ASC with --method alpha-balanced); "
                         "sc / nv-layerwise = the paper's baselines executed for real")
    ap.add_argument("--collectives", default="auto", choices=["auto", "nccl", "nvls"],
                    help="DP RS/AG path: NCCL kernels or NVLS multicast fused into the update")
    ap.add_argument("--tp", type=int, default=1,
                    help="tensor-parallel degree T (config C3: --gpus 8 --tp 2 = DP4 x TP2); "
                         "TP-plane tensors go through the micro-group gather/compute/scatter path")
    ap.add_argument("--tp-cmax", type=int, default=268435456,
                    help="micro-group capacity in numel (default 512 MiB of bf16)")
    return ap.parse_args()


# ------------------------------------------------------------------ plumbing
class Dist:
    def __init__(self):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch.distributed as td

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            td.init_process_group("gloo", rank=self.rank, world_size=self.world)
            self.pg = td

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def bcast_bytes(self, b: bytes | None) -> bytes:
        if not self.pg:
            return b
        obj = [b]
        self.pg.broadcast_object_list(obj, src=0)
        return obj[0]

    def gather(self, x):
        if not self.pg:
            return [x]
        out = [None] * self.world
        self.pg.all_gather_object(out, x)
        return out


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
         "power.limit")

    def __init__(self):
        self.proc, self.lines = None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self, n_gpus):
        if self.proc is None:
            return None
        time.sleep(0.3)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, pw, lim, reasons = [], [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9 or not f[0].isdigit() or int(f[0]) >= n_gpus:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            try:  # (power: the energy budget the step runs against under sw_power_cap)
                pw.append((float(f[1]), float(f[3])))
                if len(f) > 9:
                    lim.append(float(f[9]))
            except ValueError:
                pass
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return None
        load = [s for s in sm if s > 0.5 * max(sm)] or sm
        out = {"sm_mhz": statistics.median(load), "sm_max_mhz": max(mx), "samples": len(sm),
               "reasons": sorted(reasons)}
        busy = [p for s, p in pw if s > 0.5 * max(sm)]
        if busy:
            out["power_w"] = round(statistics.median(busy), 1)
        if lim:
            out["power_limit_w"] = max(lim)
        return out


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d, "MEASURED_PEAKS.json"
    except Exception:
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}, \
            "fallback (B200_PROFILING.md)"


def host_mem_available():
    """MemAvailable of this host in bytes (None if unknown)."""
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except Exception:
        pass
    return None


def gpu_local_cpus(torch, dev):
    """Binds the calling thread to the CPUs NVML names as close to GPU `dev`,
    so pinned host buffers allocated next land on that GPU's NUMA node (the
    caller restores its affinity after allocating). True when bound."""
    try:
        import pynvml
        pynvml.nvmlInit()
        uuid = str(torch.cuda.get_device_properties(dev).uuid)
        h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        pynvml.nvmlDeviceSetCpuAffinity(h)
        return True
    except Exception:
        return False


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant GEMM from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ns_gemm_ncu.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------ CPU side
def cpu_reference_step(cfg_path, ranks, method, cost, alpha, threads=None, steps=1, warmup=0):
    """The reference's CPU Muon step (oracle/cpu_step.py: reference planner
    from oracle/_ref, fp64 restatement of verify.hpp on every host core),
    timed on bounded samples — complete Newton-Schulz iterations on full-size
    matrices of each shape class — and extrapolated to the full step."""
    from oracle import cpu_step as C

    plan = C.reference_plan(cfg_path, ranks, method, cost, alpha)
    cs = C.CpuStep(plan, ranks, threads)
    for _ in range(warmup):
        cs.warmup_sample()
    samples = []
    for i in range(steps):
        dt, what = cs.sample(i)
        samples.append((dt, what))
    est = cs.estimate()
    O = C.O
    O.set_fast_blas(False)
    return {**est, "cores": cs.cores, "blas": "numpy OpenBLAS (ILP64 dgemm)" if cs.fast
            else "exact blocked GEMM", "sample": cs.describe(), "samples": samples,
            "planner": plan.source}


# ------------------------------------------------------------------ our arm
def resolve_alpha(P, a, params, cap, ranks):
    """--alpha auto: the planner's own choice (planner.choose_alpha)."""
    a.alpha_auto = a.alpha == "auto"
    if not a.alpha_auto:
        return float(a.alpha)
    if a.method != "alpha-balanced" or a.optimizer != "muon":
        return 1.0
    return P.choose_alpha(params, cap, ranks, a.cost)[0]


def run_ours(a, dist: Dist):
    import numpy as np
    import torch

    from paper_2602_06079_b200 import planner as P
    from paper_2602_06079_b200.engine import (COLLECTIVE_NAMES, DistributedMuon, OptimizerConfig,
                                              ShampooConfig, SoapConfig, nccl_unique_id)

    N = dist.world
    T = a.tp
    if N % T:
        raise SystemExit(f"--tp {T} must divide the number of ranks {N}")
    D = N // T
    d, t = dist.rank // T, dist.rank % T
    torch.cuda.set_device(dist.local)
    cfg = P.load_config(a.config)
    params = P.generate_transformer_params(cfg)
    view = P.apply_tp_sharding(params, T)     # the DP partition is over the TP shards
    cap = cfg.bucket_capacity // T
    t_plan = time.perf_counter()
    a.alpha = resolve_alpha(P, a, view, cap, D)
    plan = P.plan_dp(view, cap, D, a.method, a.cost, a.alpha)
    plan_us = (time.perf_counter() - t_plan) * 1e6
    if T == 1:
        uid = dist.bcast_bytes(nccl_unique_id() if dist.rank == 0 and N > 1 else None)
        tp_uid = None
    else:
        ids = dist.gather({"dp": nccl_unique_id() if d == 0 and D > 1 else None,
                           "tp": nccl_unique_id() if t == 0 else None})
        uid, tp_uid = ids[t]["dp"], ids[d * T]["tp"]
    eng = DistributedMuon(params, cap, plan, rank=d, device=dist.local,
                          comm="nccl", nccl_uid=uid, grad_dtype=a.grad_dtype,
                          workspace_bytes=int(a.workspace_gb * (1 << 30)), tp_rank=t, tp_size=T,
                          tp_uid=tp_uid, tp_capacity=a.tp_cmax if T > 1 else None,
                          collectives=a.collectives, optimizer=a.optimizer, strategy=a.strategy,
                          shampoo=(ShampooConfig(block=a.shampoo_block, precond_every=a.precond_every)
                                   if a.optimizer == "shampoo" else
                                   SoapConfig(block=a.shampoo_block, precond_every=a.precond_every)
                                   if a.optimizer == "soap" else None))
    info = eng.info()
    coll_path = COLLECTIVE_NAMES[info["collectives"]]
    eng.fill_synthetic(42, "weights")
    eng.fill_synthetic(1000 + dist.rank, "grads")
    ocfg = OptimizerConfig()
    stream = torch.cuda.ExternalStream(eng.stream())
    # Shampoo / SOAP refresh their preconditioner on calls i with
    # i % precond_every == 0 (engine step counter): every measured leg below
    # starts on a call i % pe == 1 so its steps stay refresh-free when they fit
    # in one period, and the refresh step is timed on its own
    pe = a.precond_every if a.optimizer in ("shampoo", "soap") else 0
    calls = [0]

    def step(**kw):
        eng.step(ocfg, **kw)
        calls[0] += 1

    def align(k):  # untimed steps until the next leg of k steps avoids a refresh
        if pe and k < pe:
            while calls[0] % pe != 1:
                step()

    for _ in range(a.warmup):
        step()
    align(a.steps)
    eng.sync()
    dist.barrier()

    clocks = ClockSampler() if dist.rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.4)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    eng.sync()
    dist.barrier()
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    e1.synchronize()
    eng.sync()
    ms = e0.elapsed_time(e1) / a.steps
    last = eng.timing()
    clock = clocks.stop(torch.cuda.device_count()) if clocks else None
    # per-launch breakdown in a separate, untimed pass: the profiler's two
    # events per GEMM launch stay out of the headline step time
    prof_steps = max(1, min(a.steps, 3))
    align(prof_steps)
    eng.profile_gemm(True)
    for _ in range(prof_steps):
        step()
    eng.sync()
    eng.profile_gemm(False)
    launches = eng.gemm_profile_launches()
    prof = eng.gemm_profile(reset=True)
    by_mode = {}
    for mode, lms, fl, ex, what in launches:
        d = by_mode.setdefault(mode, {"ms": 0.0, "flops": 0.0, "exec_flops": 0.0, "launches": 0})
        d["ms"] += lms
        d["flops"] += fl
        d["exec_flops"] += ex
        d["launches"] += 1
    for mode, d in by_mode.items():
        if mode in GEMM_MODES:
            d["tflops_alg"] = round(d["flops"] / (d["ms"] * 1e-3) / 1e12, 1) if d["ms"] else 0.0
            d["tflops_exec"] = round(d["exec_flops"] / (d["ms"] * 1e-3) / 1e12, 1) if d["ms"] else 0.0
        elif d["flops"] > 0:  # elementwise: algorithmic bytes in the flops column
            d["gbps_alg"] = round(d["flops"] / (d["ms"] * 1e-3) / 1e9, 1) if d["ms"] else 0.0
        d["ms_per_step"] = round(d["ms"] / prof_steps, 2)
        for k in ("ms", "flops", "exec_flops"):
            d.pop(k)
    if os.environ.get("OSH_BENCH_LAUNCHES") and dist.rank == 0:
        for rec in launches:
            print("launch", *rec, file=sys.stderr)
    refresh_ms, refresh_modes = None, None
    if a.optimizer in ("shampoo", "soap"):
        # the timed steps avoid the root refresh (align above); time one
        # refresh step on its own: the next call i with i % precond_every == 0
        while calls[0] % pe != 0:
            step()
        eng.sync()
        dist.barrier()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.profile_gemm(True)
        r0.record(stream)
        step()
        r1.record(stream)
        r1.synchronize()
        eng.sync()
        refresh_ms = r0.elapsed_time(r1)
        refresh_modes = {}
        for mode, lms, fl, ex, what in eng.gemm_profile_launches():
            d = refresh_modes.setdefault(mode, {"launches": 0, "ms": 0.0, "flops": 0.0})
            d["launches"] += 1
            d["ms"] += lms
            d["flops"] += fl
        for mode, d in refresh_modes.items():
            if mode in GEMM_MODES and d["ms"] > 0:
                d["tflops_alg"] = round(d["flops"] / (d["ms"] * 1e-3) / 1e12, 1)
            d["ms"] = round(d["ms"], 2)
            d.pop("flops")
        eng.gemm_profile(reset=True)
        eng.profile_gemm(False)

    # e2e through the C ABI with host buffers (pinned)
    e2e = None
    e2e_skip = None
    if not a.no_e2e and a.e2e_steps > 0:
        total = info["total_numel"]
        gdt = torch.bfloat16 if a.grad_dtype == "bf16" else torch.float32
        # every rank pins a full gradient and replica (N x 29 GB at 8B bf16):
        # all ranks take the e2e leg together or none does
        numa = os.environ.get("OSH_BENCH_NUMA", "1") != "0"
        saved_cpus = os.sched_getaffinity(0)
        # every local rank pins its buffers at once: skip the leg (all ranks
        # agree below) rather than let pinned pages exhaust the host's memory
        need = dist.world * total * (torch.tensor([], dtype=gdt).element_size() + 2)
        avail = host_mem_available()
        hg = hr = None
        if avail is not None and need > 0.8 * avail:
            pinned = (f"host memory: {dist.world} ranks x {need / dist.world / 1e9:.1f} GB pinned "
                      f"> 80 % of MemAvailable {avail / 1e9:.1f} GB")
        else:
            if numa:
                numa = gpu_local_cpus(torch, dist.local)
            try:
                hg = torch.empty(total, dtype=gdt, pin_memory=True)
                hr = torch.empty(total, dtype=torch.bfloat16, pin_memory=True)
                pinned = True
            except RuntimeError as exc:  # pinned host memory exhausted
                hg = hr = None
                pinned = str(exc).splitlines()[0][:200]
            finally:  # (the pages stay where they were allocated)
                os.sched_setaffinity(0, saved_cpus)
        flags = dist.gather(pinned)
        if any(f is not True for f in flags):
            e2e_skip = next(f for f in flags if f is not True)
            del hg, hr
    if not a.no_e2e and a.e2e_steps > 0 and e2e_skip is None:
        # host gradients: synthetic bf16/f32 values staged through the device in
        # 256M-element chunks (outside the timed region)
        chunk = 1 << 28
        for off in range(0, total, chunk):
            c = min(chunk, total - off)
            hg[off:off + c].copy_(torch.randn(c, device="cuda", dtype=gdt).mul_(0.01))
        torch.cuda.synchronize()
        dist.barrier()
        eng.sync()
        # N > 1 (sharded, TP 1): each rank reads back the parameters it updated
        # (its owned slices, as soon as its wave is done); the full replica
        # stays all-gathered on the devices for the next forward pass
        owned_out = N > 1 and T == 1 and a.strategy == "sharded"
        if owned_out:
            eng.set_host_output("owned")
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        align(a.e2e_steps)
        eng.sync()
        f0.record(stream)
        for _ in range(a.e2e_steps):
            step(host_grads=hg.data_ptr(), host_replica_out=hr.data_ptr())
        f1.record(stream)
        f1.synchronize()
        e2e_ms = f0.elapsed_time(f1) / a.e2e_steps
        e2e = {"e2e_ms": e2e_ms, "h2d": total * hg.element_size(),
               "d2h": (info["owned_numel"] if owned_out else total) * 2,
               "d2h_what": "own updated slices" if owned_out else "full bf16 replica",
               "numa_local": bool(numa)}
        del hg, hr

    rec = {"ms": ms, "prof": prof, "prof_steps": prof_steps, "by_mode": by_mode, "last": last, "info": info, "e2e": e2e,
           "e2e_skip": e2e_skip,
           "owned_numel": info["owned_numel"],
           "ns_flops": (info["ns_flops_per_iter"] * 5 if a.optimizer == "muon"
                        else float(last["gemm_flops"])),
           "refresh_ms": refresh_ms,
           "refresh_modes": refresh_modes if a.optimizer != "muon" else None}
    allrec = dist.gather(rec)
    eng.close()
    if dist.rank != 0:
        return None

    peaks, peak_src = measured_peaks()
    ms_max = max(r["ms"] for r in allrec)
    flops = [r["ns_flops"] for r in allrec]
    comp = [r["last"]["compute_ms"] for r in allrec]
    numel_loads = [float(x) for x in plan.rank_loads]

    def rlb(v):
        v = [float(x) for x in v]
        return max(v) / (sum(v) / len(v)) if sum(v) > 0 else 1.0

    p0 = allrec[0]["prof"]
    achieved = p0["flops"] / (p0["ms"] * 1e-3) / 1e12 if p0["ms"] > 0 else 0.0
    achieved_exec = p0["exec_flops"] / (p0["ms"] * 1e-3) / 1e12 if p0["ms"] > 0 else 0.0
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1400.0)))
    alpha_src = (" (auto: planner.choose_alpha over {1,.75,.5,.25,0} by planned NS-flop max/mean)"
                 if a.alpha_auto else "")
    out = {
        "metric": (METRIC if a.optimizer == "muon" else METRIC_SHAMPOO if a.optimizer == "shampoo"
                   else METRIC_SHAMPOO.replace("Shampoo", "SOAP")),
        "value": round(ms_max, 3),
        "unit": "ms",
        "n_gpus": N,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": round(ms_max, 3),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16 NS operands / fp32 accum+state / " + a.grad_dtype + " grads",
        "data": "synthetic: counter-based normal weights/grads of the reference generator's shapes",
        "config": {
            "workload": "qwen3-8b-like Muon step (L36 h4096 f12288 v151936: 183 tensors, "
                        f"{info['total_numel']} params, {info['n_buckets']} buckets cap {cap})",
            "plan": (f"alpha-balanced alpha={a.alpha}{alpha_src}" if a.method == "alpha-balanced"
                     else a.method) + f" cost={a.cost}",
            "ranks": N, "ns_steps": 5, "grad_dtype": a.grad_dtype, "collectives": coll_path,
            "strategy": a.strategy,
            "parallelism": ((f"dp{N} (ZeRO-1 variable-size RS/AG fused into the update kernels: "
                             "multimem.ld_reduce / multimem.st over NVSwitch)" if coll_path == "nvls"
                             else f"dp{N} (ZeRO-1 variable-size RS/AG over NCCL)") if T == 1 else
                            f"dp{D} x tp{T} (ZeRO-1 RS/AG over the TP shards + micro-group "
                            f"gather/host-Muon/scatter, c_max {a.tp_cmax})"),
            "l2": "inputs (weights, momentum, grads) >> 126 MB L2; no flush needed",
        },
        "max_mean_rank_load": {
            "plan_numel": round(rlb(numel_loads), 4),
            "ns_gemm_flops": round(rlb(flops), 4),
            "measured_compute_ms": round(rlb(comp), 4),
            "per_rank_compute_ms": [round(c, 2) for c in comp],
        },
        "phases_ms_rank0": {k: round(allrec[0]["last"][k], 3)
                            for k in ("rs_ms", "compute_ms", "ag_ms", "total_ms")},
        "gpu_launches": int(a.steps * (allrec[0]["last"]["gemm_launches"] +
                                       allrec[0]["last"]["elementwise_launches"])),
        "roofline": {
            "bound": "tensor",
            "kernel": "ns_gemm_kernel (tcgen05 UMMA 128x256, all NS GEMM launches)",
            "achieved": round(achieved, 1),
            "peak": peak,
            "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4),
            "peak_source": peak_src + " bf16_tflops_sustained",
            "traffic": ncu_traffic(),
            "achieved_executed": round(achieved_exec, 1),
            "frac_executed": round(achieved_exec / peak, 4),
            "note": "achieved = algorithmic NS flops 2MNK per GEMM (4m^2n+2m^3 per matrix-iteration) "
                    "/ summed CUDA-event launch time; symmetric GRAM/POLY tiles execute fewer flops "
                    "(achieved_executed = tensor-core flops actually issued)",
            "by_mode": allrec[0]["by_mode"],
            "launches_timed": p0["launches"],
            "gemm_ms_per_step": round(p0["ms"] / allrec[0]["prof_steps"], 3),
            "step_frac_in_gemm": round(p0["ms"] / allrec[0]["prof_steps"] / allrec[0]["ms"], 4),
            "profiled_steps": allrec[0]["prof_steps"],
        },
        "planner_us": round(plan_us, 1),
    }
    if clock:
        out["clocks"] = clock
    if allrec[0]["e2e_skip"] is not None:
        out["e2e"] = {"value": None, "unit": "ms", "skipped": "pinned host buffers unavailable: "
                      + str(allrec[0]["e2e_skip"])}
    if allrec[0]["e2e"]:
        e = max(r["e2e"]["e2e_ms"] for r in allrec)
        out["e2e"] = {"value": round(e, 3), "unit": "ms",
                      "h2d_bytes_per_step": allrec[0]["e2e"]["h2d"],
                      "d2h_bytes_per_step": allrec[0]["e2e"]["d2h"],
                      "note": "per rank: H2D its full local bf16 gradient (pinned), D2H "
                              + allrec[0]["e2e"]["d2h_what"] + "; bytes are rank 0's"
                              + ("; pinned buffers on each GPU's NUMA node" if allrec[0]["e2e"]["numa_local"]
                                 else "")}
    if a.optimizer == "soap":
        rms = max(r["refresh_ms"] for r in allrec)
        out["soap"] = {"block": a.shampoo_block, "precond_every": a.precond_every,
                       "timed_steps_refresh_free": a.steps < a.precond_every,
                       "refresh_step_ms": round(rms, 3),
                       "refresh_by_mode_rank0": allrec[0]["refresh_modes"],
                       "amortized_step_ms": round(ms_max + (rms - ms_max) / a.precond_every, 3),
                       "note": "value = a step without the eigenbasis refresh; the refresh step "
                               "(power iteration + CholeskyQR2) is timed separately"}
    if a.optimizer == "shampoo":
        rms = max(r["refresh_ms"] for r in allrec)
        out["shampoo"] = {"block": a.shampoo_block, "precond_every": a.precond_every,
                       "timed_steps_refresh_free": a.steps < a.precond_every,
                          "newton_iters": 16, "refresh_step_ms": round(rms, 3),
                          "refresh_by_mode_rank0": allrec[0]["refresh_modes"],
                          "amortized_step_ms": round(ms_max + (rms - ms_max) / a.precond_every, 3),
                          "note": "value = a step without the inverse-root refresh; the refresh "
                                  "step (coupled Newton, bf16x3 split GEMMs) is timed separately"}
        out["config"]["workload"] = out["config"]["workload"].replace("Muon step", "Shampoo step")
        out["roofline"]["kernel"] = "ns_gemm_kernel (STAT / UPDATE / GRAM GEMMs of the step)"
    if N == 1 and not a.no_cpu_baseline and a.optimizer == "muon" and T == 1:
        cb = cpu_reference_step(a.config, 1, a.method, a.cost, a.alpha, os.cpu_count(), steps=1)
        out["cpu_baseline"] = {"value": round(cb["critical_path_ms"], 1), "unit": "ms",
                               "cores": cb["cores"], "kind": "port", "sample": cb["sample"],
                               "extrapolated": True, "blas": cb["blas"],
                               "iter_ms": cb["iter_ms"], "elem_ns": cb["elem_ns"],
                               "sampled_s": round(sum(t for t, _ in cb["samples"]), 1)}
    return out


# ------------------------------------------------------------------ reference arm
def run_reference(a, dist: Dist):
    """The reference arm: the reference's CPU step on this host's cores,
    planned by the REFERENCE planner (oracle/_ref), never by this package."""
    if dist.rank != 0:
        return None
    from oracle import cpu_step as C

    N = dist.world
    alpha_auto = a.alpha == "auto"
    if alpha_auto and a.method == "alpha-balanced" and a.optimizer == "muon":
        alpha = C.choose_alpha(a.config, N, a.cost)[0]
    else:
        alpha = 1.0 if a.alpha == "auto" else float(a.alpha)
    threads = os.cpu_count()
    t0 = time.perf_counter()
    cb = cpu_reference_step(a.config, N, a.method, a.cost, alpha, threads, steps=a.steps,
                            warmup=a.warmup)
    wall = time.perf_counter() - t0
    v = cb["critical_path_ms"]
    sampled = [round(1e3 * t, 1) for t, _ in cb["samples"]]
    return {
        "metric": METRIC, "value": round(v, 1), "unit": "ms", "n_gpus": N, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(v, 1), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "extrapolated": True,
        "measured": {"sample_ms_per_step": round(statistics.mean(sampled), 1),
                     "samples_ms": sampled, "sampled": [w for _, w in cb["samples"]],
                     "wall_s": round(wall, 1),
                     "note": "each timed step runs a bounded sample of the CPU step (see "
                             "cpu_baseline.sample); value extrapolates the latest sample of "
                             "every shape class to the full step, so value x steps is NOT the "
                             "wall time of this run"},
        "data": "synthetic normal matrices of the reference generator's shapes",
        "config": {"workload": f"{os.path.splitext(os.path.basename(a.config))[0]} Muon step, "
                               "CPU fp64 (reference algorithm)",
                   "ranks": N, "plan": f"{a.method} alpha={alpha}"
                   f"{' (auto, same rule as our arm)' if alpha_auto else ''} cost={a.cost}",
                   "planner": cb["planner"]},
        "cpu_baseline": {"value": round(v, 1), "unit": "ms", "cores": cb["cores"],
                         "kind": "port", "sample": cb["sample"], "blas": cb["blas"],
                         "extrapolated": True, "iter_ms": cb["iter_ms"], "elem_ns": cb["elem_ns"],
                         "rank_ms": [round(x, 1) for x in cb["rank_ms"]],
                         "replicated_full_step_ms": round(cb["full_ms"], 1)},
        "e2e": {"value": round(v, 1), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


GEMM_MODES = ("gram", "poly", "update", "final", "stat", "split")


def main():
    a = parse_args()
    dist = Dist()
    if a.impl == "reference":
        out = run_reference(a, dist)
    else:
        out = run_ours(a, dist)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
