"""Python face of the fp64 Muon oracle (TEST INFRASTRUCTURE / CPU BASELINE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` leg
may import this module; it is the checker, never the product. Numerics live
in liboracle.so (muon_oracle.c); the drivers below restate the reference's
``run_replicated`` / ``run_partitioned`` / ``max_abs_diff``
(proj/include/optishard/verify.hpp:149-322) around those kernels.
"""
from __future__ import annotations

import ctypes
import glob
import os
import subprocess
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Set, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64, _u64, _int, _dbl = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-C", HERE, "liboracle.so"], check=True,
                           stdout=subprocess.DEVNULL)
        L = ctypes.CDLL(path)
        L.orc_splitmix64.restype = _u64
        L.orc_splitmix64.argtypes = [_u64]
        L.orc_stream_seed.restype = _u64
        L.orc_stream_seed.argtypes = [_u64, _int, _int, _int, _int]
        L.orc_normal_fill.argtypes = [_u64, _dbl, _i64, _dp]
        L.orc_synth_gradient.argtypes = [_i64, _i64, _int, _u64, _int, _int, _dp]
        L.orc_init_weight.argtypes = [_i64, _i64, _int, _u64, _dp]
        L.orc_reduced_gradient.argtypes = [_i64, _i64, _int, _u64, _int, _int, _dp]
        L.orc_newton_schulz.restype = _int
        L.orc_newton_schulz.argtypes = [_dp, _i64, _i64, _int]
        L.orc_muon_apply.argtypes = [_i64, _i64, _int, _dbl, _dbl, _int, _dp, _dp, _dp, _dp]
        L.orc_norm.restype = _dbl
        L.orc_norm.argtypes = [_dp, _i64, _i64]
        L.orc_set_blas.restype = _int
        L.orc_set_blas.argtypes = [ctypes.c_char_p, ctypes.c_char_p]
        L.orc_set_threads.argtypes = [_int]
        L.orc_get_threads.restype = _int
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def _rc(shape: Sequence[int]) -> Tuple[int, int]:
    return (int(shape[0]), int(shape[1])) if len(shape) == 2 else (int(shape[0]), 1)


def set_fast_blas(enable: bool = True) -> bool:
    """FAST mode: products through numpy's bundled ILP64 OpenBLAS (timed CPU
    baseline). Returns False when no such library is present."""
    if not enable:
        lib().orc_set_blas(None, None)
        return True
    import numpy  # noqa: F401

    base = os.path.dirname(os.path.dirname(np.__file__))
    for path in glob.glob(os.path.join(base, "numpy.libs", "libscipy_openblas64_*.so")):
        if lib().orc_set_blas(path.encode(), b"scipy_cblas_dgemm64_") == 0:
            return True
    return False


def stream_seed(seed, kind, step, param_id, rank) -> int:
    return int(lib().orc_stream_seed(seed, kind, step, param_id, rank))


def normal_stream(seed: int, n: int) -> np.ndarray:
    out = np.empty(n)
    lib().orc_normal_fill(seed, 1.0, n, _ptr(out))
    return out


def synth_gradient(shape, param_id, seed, step, rank) -> np.ndarray:
    r, c = _rc(shape)
    out = np.empty((r, c))
    lib().orc_synth_gradient(r, c, param_id, seed, step, rank, _ptr(out))
    return out


def init_weight(shape, param_id, seed) -> np.ndarray:
    r, c = _rc(shape)
    out = np.empty((r, c))
    lib().orc_init_weight(r, c, param_id, seed, _ptr(out))
    return out


def reduced_gradient(shape, param_id, seed, step, contributors) -> np.ndarray:
    r, c = _rc(shape)
    out = np.empty((r, c))
    lib().orc_reduced_gradient(r, c, param_id, seed, step, contributors, _ptr(out))
    return out


def newton_schulz(x: np.ndarray, steps: int = 5) -> np.ndarray:
    y = np.ascontiguousarray(x, dtype=np.float64).copy()
    lib().orc_newton_schulz(_ptr(y), y.shape[0], y.shape[1], steps)
    return y


def norm(x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib().orc_norm(_ptr(x), x.shape[0], x.shape[1] if x.ndim == 2 else 1))


@dataclass
class OptimizerConfig:
    lr: float = 0.02
    beta: float = 0.9
    ns_steps: int = 5


def muon_apply(is_matrix: bool, cfg: OptimizerConfig, w: np.ndarray, m: np.ndarray,
               g: np.ndarray) -> float:
    """In place on w, m; returns ||w_new - w_old||_F."""
    assert w.shape == m.shape == g.shape
    g = np.ascontiguousarray(g, dtype=np.float64)
    out = ctypes.c_double(0.0)
    r, c = w.shape
    lib().orc_muon_apply(r, c, 1 if is_matrix else 0, cfg.lr, cfg.beta, cfg.ns_steps, _ptr(w),
                         _ptr(m), _ptr(g), ctypes.byref(out))
    return out.value


@dataclass
class VerifyTrace:
    reduction_order: str = "ascending-rank"
    update_norms: List[Dict[int, float]] = field(default_factory=list)
    final_weights: Dict[int, np.ndarray] = field(default_factory=dict)
    state_hosts: Dict[int, Set[str]] = field(default_factory=dict)


def max_abs_diff(a: VerifyTrace, b: VerifyTrace) -> float:
    mx = 0.0
    if len(a.update_norms) != len(b.update_norms):
        raise ValueError("traces cover different step counts")
    for sa, sb in zip(a.update_norms, b.update_norms):
        for pid, n in sa.items():
            mx = max(mx, abs(n - sb[pid]))
    for pid, w in a.final_weights.items():
        mx = max(mx, float(np.abs(w - b.final_weights[pid]).max()))
    return mx


def run_replicated(params, cfg: OptimizerConfig, steps: int, seed: int,
                   contributors: int = 1) -> VerifyTrace:
    """verify.hpp:188-210. ``params``: objects with id, shape."""
    t = VerifyTrace()
    w = {p.id: init_weight(p.shape, p.id, seed) for p in params}
    m = {p.id: np.zeros_like(w[p.id]) for p in params}
    for p in params:
        t.state_hosts.setdefault(p.id, set()).add("replicated")
    for step in range(steps):
        t.update_norms.append({})
        for p in params:
            g = reduced_gradient(p.shape, p.id, seed, step, contributors)
            t.update_norms[-1][p.id] = muon_apply(len(p.shape) == 2, cfg, w[p.id], m[p.id], g)
    t.final_weights = w
    return t


@dataclass
class FaultSpec:
    enabled: bool = False
    param_id: int = -1
    at_step: int = -1


def run_partitioned(params, cfg: OptimizerConfig, steps: int, seed: int,
                    owners: Dict[int, int], tp_hosts: Optional[Dict[int, int]], dp_ranks: int,
                    tp_ranks: int = 1, fault: FaultSpec = FaultSpec()) -> VerifyTrace:
    """verify.hpp:225-322 with the plan lookups pre-resolved: ``owners`` maps
    param id -> dp owner (param_owner), ``tp_hosts`` param id -> tp host."""
    t = VerifyTrace()
    host = {p.id: [owners[p.id], (tp_hosts or {}).get(p.id, 0)] for p in params}
    eff = FaultSpec(fault.enabled, fault.param_id, fault.at_step)
    if eff.enabled:
        if eff.param_id < 0:
            for p in params:
                if getattr(p, "tp_split", 0) != 0 and not getattr(p, "vocab_space", False):
                    eff.param_id = p.id
                    break
        if eff.param_id < 0:
            eff.param_id = params[0].id
        if eff.at_step < 0:
            eff.at_step = steps // 2

    def key(h):
        return f"dp{h[0]}.tp{h[1]}"

    moms: Dict[str, Dict[int, np.ndarray]] = {}
    w = {}
    for p in params:
        w[p.id] = init_weight(p.shape, p.id, seed)
        moms.setdefault(key(host[p.id]), {})[p.id] = np.zeros_like(w[p.id])
        t.state_hosts.setdefault(p.id, set()).add(key(host[p.id]))
    for step in range(steps):
        if eff.enabled and step == eff.at_step:
            h = host[eff.param_id]
            if tp_hosts is not None and tp_ranks > 1:
                h[1] = (h[1] + 1) % tp_ranks
            else:
                h[0] = (h[0] + 1) % dp_ranks
        t.update_norms.append({})
        for p in params:
            g = reduced_gradient(p.shape, p.id, seed, step, dp_ranks)
            k = key(host[p.id])
            t.state_hosts[p.id].add(k)
            store = moms.setdefault(k, {})
            if p.id not in store:
                store[p.id] = np.zeros_like(w[p.id])
            t.update_norms[-1][p.id] = muon_apply(len(p.shape) == 2, cfg, w[p.id], store[p.id], g)
    t.final_weights = w
    return t
