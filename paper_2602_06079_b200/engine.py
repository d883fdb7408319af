"""Per-rank driver of the B200 Canzona optimizer step (Python mirror of the
reference's ``run_partitioned``, proj/include/optishard/verify.hpp:225-322,
executed for real: variable-size NCCL reduce-scatter -> owner Muon on sm_100a
-> variable-size all-gather). All work happens in libosh.so behind the C ABI;
this module only marshals arguments.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .planner import DpPartitionPlan, ParamSpec, _desc_array, apply_tp_sharding, build_buffer_layout

GRAD_DTYPES = {"f32": 0, "fp32": 0, "float32": 0, "bf16": 1, "bfloat16": 1}
READ = {"master": 0, "momentum": 1, "replica": 2}


@dataclass
class OptimizerConfig:
    """OptimizerConfig (verify.hpp:31-35) + the quintic coefficients (:120)."""
    lr: float = 0.02
    beta: float = 0.9
    ns_steps: int = 5
    ns_a: float = 3.4445
    ns_b: float = -4.7750
    ns_c: float = 2.0315

    def c(self) -> _lib.MuonCfgC:
        return _lib.MuonCfgC(self.lr, self.beta, self.ns_steps, 0, self.ns_a, self.ns_b, self.ns_c)


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _lib.check(_lib.lib().osh_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return bytes(buf)


@dataclass
class ShampooConfig:
    """Builder-defined blocked Shampoo (osh.h osh_shampoo_cfg; specification
    oracle/shampoo_oracle.py). lr / beta1 come from OptimizerConfig."""
    beta2: float = 0.95
    eps: float = 1e-4
    block: int = 1024
    precond_every: int = 10
    newton_iters: int = 16

    def c(self) -> _lib.ShampooCfgC:
        return _lib.ShampooCfgC(self.beta2, self.eps, self.block, self.precond_every,
                                self.newton_iters, 0)


@dataclass
class SoapConfig:
    """Builder-defined blocked SOAP (osh.h OSH_OPT_SOAP; specification
    oracle/soap_oracle.py). lr / beta1 come from OptimizerConfig; beta2 is
    both the second-moment and the statistics decay; init_iters = power
    iterations of the first basis refresh. Carried in osh_shampoo_cfg."""
    beta2: float = 0.95
    eps: float = 1e-8
    block: int = 1024
    precond_every: int = 10
    init_iters: int = 4

    def c(self) -> _lib.ShampooCfgC:
        return _lib.ShampooCfgC(self.beta2, self.eps, self.block, self.precond_every,
                                self.init_iters, 0)


OPTIMIZERS = {"muon": 0, "shampoo": 1, "soap": 2}
STRATEGIES = {"sharded": 0, "sc": 1, "nv-layerwise": 2}


def layer_groups(params) -> np.ndarray:
    """Layer group id per parameter: the name segment before the first '.',
    ids in first-appearance order (simulate.hpp:130-135,140-152)."""
    ids, out = {}, []
    for p in params:
        key = p.name.split(".", 1)[0]
        out.append(ids.setdefault(key, len(ids)))
    return np.asarray(out, dtype=np.int32)
COLLECTIVES = {"auto": 0, "nccl": 1, "nvls": 2}
COLLECTIVE_NAMES = {0: "none", 1: "nccl", 2: "nvls"}


class DistributedMuon:
    """One data-parallel rank. ``comm='nccl'`` runs the real collectives
    (dp_size > 1 needs ``nccl_uid``); ``comm='none'`` skips them: the caller
    supplies already-reduced gradients and reads its owned results."""

    def __init__(self, params: Sequence[ParamSpec], bucket_capacity: int, plan: DpPartitionPlan,
                 rank: int = 0, device: int = 0, comm: str = "nccl",
                 nccl_uid: Optional[bytes] = None, grad_dtype: str = "f32",
                 workspace_bytes: int = 0, tp_rank: int = 0, tp_size: int = 1,
                 tp_uid: Optional[bytes] = None, tp_capacity: Optional[int] = None,
                 collectives: str = "auto", optimizer: str = "muon",
                 shampoo: Optional[ShampooConfig] = None, strategy: str = "sharded",
                 strategy_cost: str = "numel"):
        """With tp_size > 1: ``params`` are the FULL tensors, ``plan`` /
        ``bucket_capacity`` describe the DP partition of the TP-sharded view
        (planner.apply_tp_sharding), ``rank`` is the DP rank.

        ``collectives`` (dp_size > 1): "nccl" = NCCL reduce-scatter /
        all-gather kernels overlapped with the update, "nvls" = reduction and
        broadcast fused into the update kernels through NVSwitch multicast
        (OshError when the node cannot), "auto" = nvls when available.
        ``optimizer``: "muon" (the reference's step) or "shampoo" (builder-
        defined blocked Shampoo, ``shampoo`` = its ShampooConfig).
        ``strategy``: "sharded" (the plan's owners: LB-ASC / ASC), or the
        paper's baselines "sc" (replicated update after an all-reduce) and
        "nv-layerwise" (whole-layer LPT owners over ``strategy_cost``,
        all-reduce, owner update, broadcast)."""
        L = _lib.lib()
        self.params = list(params)
        self.rank, self.world = rank, plan.ranks
        self.tp_rank, self.tp_size = tp_rank, tp_size
        self.grad_dtype = grad_dtype
        ctx = ctypes.c_void_p()

        def buf(b):
            return None if b is None else ctypes.cast(ctypes.create_string_buffer(b, 128),
                                                      ctypes.c_void_p)
        _lib.check(L.osh_ctx_create_tp(device, rank, plan.ranks, tp_rank, tp_size,
                                       0 if comm == "nccl" else 1, buf(nccl_uid), buf(tp_uid),
                                       ctypes.byref(ctx)))
        self._ctx = ctx
        if tp_capacity is not None:
            _lib.check(L.osh_ctx_set_tp_capacity(ctx, tp_capacity))
        _lib.check(L.osh_ctx_set_collectives(ctx, COLLECTIVES[collectives]))
        if optimizer != "muon" or shampoo is not None:
            sc = (shampoo or (SoapConfig() if optimizer == "soap" else ShampooConfig())).c()
            _lib.check(L.osh_ctx_set_optimizer(ctx, OPTIMIZERS[optimizer], ctypes.byref(sc)))
        self.optimizer = optimizer
        if strategy != "sharded":
            from .planner import cost_model
            lay = layer_groups(self.params)
            cm = cost_model(strategy_cost)
            _lib.check(L.osh_ctx_set_strategy(ctx, STRATEGIES[strategy],
                                              lay.ctypes.data_as(ctypes.c_void_p), len(lay),
                                              ctypes.byref(cm)))
        self.strategy = strategy
        view = apply_tp_sharding(self.params, tp_size) if tp_size > 1 else self.params
        self._bucket_params = [list(b) for b in build_buffer_layout(view, bucket_capacity).buckets]
        cuts = np.ascontiguousarray(plan.cut_vectors, dtype=np.int64)
        _lib.check(L.osh_ctx_set_layout(ctx, _desc_array(self.params), len(self.params),
                                        bucket_capacity,
                                        cuts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                        cuts.shape[0], GRAD_DTYPES[grad_dtype], workspace_bytes))

    # ------------------------------------------------------------ lifetime
    def close(self):
        if self._ctx is not None and self._ctx.value:
            _lib.check(_lib.lib().osh_ctx_destroy(self._ctx))
        self._ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ data
    def info(self) -> dict:
        i = _lib.CtxInfo()
        _lib.check(_lib.lib().osh_ctx_get_info(self._ctx, ctypes.byref(i)))
        return {k: getattr(i, k) for k, _ in _lib.CtxInfo._fields_}

    def buffers(self):
        g, r = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(_lib.lib().osh_ctx_buffers(self._ctx, ctypes.byref(g), ctypes.byref(r)))
        return g.value, r.value

    @staticmethod
    def _f32(a) -> np.ndarray:
        return np.ascontiguousarray(np.asarray(a, dtype=np.float32)).reshape(-1)

    def load_param(self, pid: int, values) -> None:
        v = self._f32(values)
        _lib.check(_lib.lib().osh_load_param(self._ctx, pid,
                                             v.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))

    def write_grad(self, pid: int, values) -> None:
        v = self._f32(values)
        _lib.check(_lib.lib().osh_write_grad(self._ctx, pid,
                                             v.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))

    def fill_synthetic(self, seed: int, what: str, scale: float = 1.0) -> None:
        _lib.check(_lib.lib().osh_fill_synthetic(self._ctx, seed, 1 if what == "weights" else 2,
                                                 scale))

    def read_param(self, pid: int, which: str = "master", shape=None) -> np.ndarray:
        """``shape``: the shape to read (with TP: the shard shape for the
        replica or a non-hosted tensor, the full shape for a hosted master)."""
        p = self.params[pid]
        shape = tuple(shape) if shape is not None else tuple(p.shape)
        n = 1
        for e in shape:
            n *= int(e)
        out = np.empty(n, np.float32)
        _lib.check(_lib.lib().osh_read_param(self._ctx, pid, READ[which],
                                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
        return out.reshape(shape)

    # ------------------------------------------------------------ step
    def step(self, cfg: OptimizerConfig = OptimizerConfig(), host_grads=None,
             host_replica_out=None) -> None:
        """host_grads / host_replica_out: objects with a data pointer (int) —
        e.g. pinned torch tensors' data_ptr() — or None for device-resident."""
        c = cfg.c()
        _lib.check(_lib.lib().osh_step(self._ctx, ctypes.byref(c), host_grads, host_replica_out))

    def sync(self) -> None:
        _lib.check(_lib.lib().osh_ctx_sync(self._ctx))

    def set_host_output(self, mode: str) -> None:
        """What step(host_replica_out=...) receives: "replica" (the whole
        all-gathered bf16 replica, default) or "owned" (only the slices this
        rank updated, at their flat offsets)."""
        _lib.check(_lib.lib().osh_ctx_set_host_output(self._ctx, {"replica": 0, "owned": 1}[mode]))

    def set_timeout(self, seconds: float) -> None:
        """Watchdog timeout of the ctx's host waits (osh_ctx_set_timeout): a
        collective that does not complete in time aborts the communicators
        and raises OshError (code 17) instead of hanging."""
        _lib.check(_lib.lib().osh_ctx_set_timeout(self._ctx, float(seconds)))

    def timing(self) -> dict:
        t = _lib.StepTiming()
        _lib.check(_lib.lib().osh_last_timing(self._ctx, ctypes.byref(t)))
        return {k: getattr(t, k) for k, _ in _lib.StepTiming._fields_}

    def stream(self) -> int:
        """cudaStream_t of the ctx's compute stream (wrap with torch.cuda.ExternalStream)."""
        s = ctypes.c_void_p()
        _lib.check(_lib.lib().osh_ctx_stream(self._ctx, ctypes.byref(s)))
        return s.value or 0

    def profile_gemm(self, enable: bool = True) -> None:
        _lib.check(_lib.lib().osh_ctx_profile_gemm(self._ctx, 1 if enable else 0))

    def gemm_profile_launches(self) -> list:
        """Per-launch records [(mode, ms, flops, exec_flops, shapes)] since the last reset."""
        n = ctypes.c_size_t(0)
        L = _lib.lib()
        _lib.check(L.osh_gemm_profile_dump(self._ctx, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _lib.check(L.osh_gemm_profile_dump(self._ctx, buf, n.value + 1, ctypes.byref(n)))
        out = []
        for line in buf.value.decode().splitlines():
            mode, ms, fl, ex, what = line.split()[:5]
            out.append((mode, float(ms), float(fl), float(ex), what))
        return out

    def gemm_profile_timeline(self) -> list:
        """Per-launch [(mode, start_ms, ms, shapes)], start relative to the last
        step's start: a timeline when exactly one step was profiled."""
        n = ctypes.c_size_t(0)
        L = _lib.lib()
        _lib.check(L.osh_gemm_profile_dump(self._ctx, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _lib.check(L.osh_gemm_profile_dump(self._ctx, buf, n.value + 1, ctypes.byref(n)))
        out = []
        for line in buf.value.decode().splitlines():
            f = line.split()
            if len(f) >= 6 and f[5].startswith("@"):
                out.append((f[0], float(f[5][1:]), float(f[1]), f[4]))
        return sorted(out, key=lambda r: r[1])

    def gemm_profile(self, reset: bool = True) -> dict:
        p = _lib.GemmProfile()
        _lib.check(_lib.lib().osh_gemm_profile_read(self._ctx, ctypes.byref(p), 1 if reset else 0))
        return {"launches": p.launches, "flops": p.flops, "exec_flops": p.exec_flops, "ms": p.ms}

    def bucket_ready(self, bucket: int, stream: Optional[int] = None) -> None:
        """Announce that gradient bucket ``bucket`` is complete (work on
        ``stream``, a raw cudaStream_t; None = the ctx stream). NCCL path: its
        reduce-scatter starts now, overlapping the rest of the backward pass."""
        _lib.check(_lib.lib().osh_bucket_ready(self._ctx, bucket, stream))

    def bucket_params(self) -> list:
        """Parameter ids of every bucket (declaration order, planner layout)."""
        return self._bucket_params

    def save_state(self, path: str) -> None:
        """This rank's optimizer state (osh_ctx_save_state; one file per rank)."""
        _lib.check(_lib.lib().osh_ctx_save_state(self._ctx, path.encode()))

    def load_state(self, path: str) -> None:
        """Restore a state saved under the same plan/model/rank (else OshError,
        code 7 = OSH_ERR_FORMAT); rewrites and all-gathers the replica."""
        _lib.check(_lib.lib().osh_ctx_load_state(self._ctx, path.encode()))

    def comm_schedule(self) -> list:
        """The collective schedule this ctx issues (osh_ctx_comm_schedule; see
        planner.comm_schedule for the record fields)."""
        from .planner import _ops_to_records
        L = _lib.lib()
        n = ctypes.c_int32(0)
        _lib.check(L.osh_ctx_comm_schedule(self._ctx, None, 0, ctypes.byref(n)))
        arr = (_lib.CollOp * max(n.value, 1))()
        _lib.check(L.osh_ctx_comm_schedule(self._ctx, arr, n.value, ctypes.byref(n)))
        return _ops_to_records(arr, n.value)

    def update_norms(self) -> np.ndarray:
        out = np.zeros(len(self.params))
        _lib.check(_lib.lib().osh_update_norms(
            self._ctx, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out
