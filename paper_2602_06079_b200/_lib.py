"""ctypes binding of libosh.so (the C ABI declared in include/osh.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2602_06079_b200/csrc``). There is no fallback: if the library
is missing every entry point raises ``OshLibraryMissing`` — the product path
never silently runs on the CPU.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int32, c_int64, c_size_t, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OSH_LIB") or os.path.join(_HERE, "libosh.so")  # (OSH_LIB: A/B builds)


class OshLibraryMissing(RuntimeError):
    pass


class OshError(RuntimeError):
    """Raised for a non-zero osh_status; ``code`` holds the status."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"osh status {code}: {msg}")
        self.code = code


# osh_status values (osh.h) -> names of the reference exception classes
STATUS_NAMES = {
    1: "ConfigError", 2: "LayoutError", 3: "ShardError", 4: "UnsupportedError",
    5: "PlanError", 6: "UnschedulableError", 7: "FormatError",
    16: "CudaError", 17: "NcclError", 18: "OutOfMemory", 19: "ArgumentError",
}


class ParamDesc(ctypes.Structure):
    _fields_ = [("id", c_int32), ("ndim", c_int32), ("shape", c_int64 * 2),
                ("dtype_bytes", c_int32), ("tp_split", c_int32), ("vocab_space", c_int32),
                ("reserved_", c_int32)]


class CostModelC(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("ns_steps", c_int32), ("shampoo_coeff", c_double),
                ("soap_coeff", c_double)]


class MuonCfgC(ctypes.Structure):
    _fields_ = [("lr", c_double), ("beta", c_double), ("ns_steps", c_int32),
                ("reserved_", c_int32), ("ns_a", c_double), ("ns_b", c_double),
                ("ns_c", c_double)]


class MatrixRef(ctypes.Structure):
    _fields_ = [("ptr", c_void_p), ("batch", c_int32), ("rows", c_int32), ("cols", c_int32),
                ("reserved_", c_int32), ("ld", c_int64), ("bstride", c_int64)]


class FinalTarget(ctypes.Structure):
    _fields_ = [("w", c_void_p), ("replica", c_void_p), ("sq_norm", c_void_p),
                ("transposed", c_int32), ("reserved_", c_int32)]


class CtxInfo(ctypes.Structure):
    _fields_ = [("total_numel", c_int64), ("owned_numel", c_int64), ("n_params", c_int32),
                ("n_owned", c_int32), ("n_buckets", c_int32), ("n_waves", c_int32),
                ("workspace_bytes", c_int64), ("device_bytes", c_int64),
                ("ns_flops_per_iter", c_double), ("collectives", c_int32),
                ("reserved", c_int32)]


class ShampooCfgC(ctypes.Structure):
    _fields_ = [("beta2", c_double), ("eps", c_double), ("block", c_int32),
                ("precond_every", c_int32), ("newton_iters", c_int32), ("reserved", c_int32)]


class StepTiming(ctypes.Structure):
    _fields_ = [("h2d_ms", c_float), ("rs_ms", c_float), ("compute_ms", c_float),
                ("ag_ms", c_float), ("d2h_ms", c_float), ("total_ms", c_float),
                ("gemm_launches", c_int32), ("elementwise_launches", c_int32),
                ("gemm_flops", c_double)]


class GemmProfile(ctypes.Structure):
    _fields_ = [("launches", c_int32), ("reserved_", c_int32), ("flops", c_double),
                ("exec_flops", c_double), ("ms", c_double)]


class GemmProblem(ctypes.Structure):
    _fields_ = [("a", MatrixRef), ("b", MatrixRef), ("b_mn_major", c_int32),
                ("reserved_", c_int32), ("out", MatrixRef), ("aux", MatrixRef),
                ("scale", c_void_p), ("final_targets", c_void_p), ("symmetric", c_int32),
                ("out_seg", c_int32), ("a_upper", c_int32), ("b_upper", c_int32)]


class CollOp(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("phase", c_int32), ("bucket", c_int32), ("root", c_int32),
                ("group", c_int32), ("reserved_", c_int32), ("offset", c_int64),
                ("count", c_int64), ("dst_offset", c_int64)]


_lib = None


def lib() -> ctypes.CDLL:
    """Loads libosh.so once; raises OshLibraryMissing when it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OshLibraryMissing(
                f"{LIB_PATH} not found: run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the CUDA extension is required; there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().osh_last_error().decode(errors="replace")
        raise OshError(status, f"{STATUS_NAMES.get(status, 'error')}: {msg}")


def _declare(L: ctypes.CDLL) -> None:
    def d(name, restype, *argtypes):
        fn = getattr(L, name)
        fn.restype = restype
        fn.argtypes = list(argtypes)

    d("osh_last_error", c_char_p)
    d("osh_abi_version", c_int32)
    d("osh_ns_gemm", c_int32, c_int32, POINTER(GemmProblem), c_int32, c_float, c_float, c_float,
      c_void_p)
    optional = [
        ("osh_generate_params", c_int32, c_int32, c_int64, c_int64, c_int32, c_int64, c_int32,
         POINTER(ParamDesc), c_int32, POINTER(c_int32)),
        ("osh_param_cost", c_int32, POINTER(ParamDesc), POINTER(CostModelC), POINTER(c_uint64)),
        ("osh_layout_build", c_int32, POINTER(ParamDesc), c_int32, c_int64, POINTER(c_int32),
         POINTER(c_int64), POINTER(c_int64), POINTER(c_int32)),
        ("osh_plan_dp", c_int32, POINTER(ParamDesc), c_int32, c_int64, c_int32, c_int32,
         POINTER(CostModelC), c_double, POINTER(c_int64), POINTER(c_uint64), POINTER(c_int32)),
        ("osh_plan_dp_serialize", c_int32, POINTER(ParamDesc), c_int32, c_int64, c_int32, c_int32,
         POINTER(CostModelC), c_double, ctypes.c_char_p, c_size_t, POINTER(c_size_t)),
        ("osh_param_owners", c_int32, POINTER(ParamDesc), c_int32, c_int64, c_int32,
         POINTER(c_int64), POINTER(c_int32)),
        ("osh_plan_tp_serialize", c_int32, POINTER(c_int32), POINTER(c_uint64), c_int32, c_int32,
         c_uint64, c_int32, ctypes.c_char_p, c_size_t, POINTER(c_size_t)),
        ("osh_muon_cfg_default", None, POINTER(MuonCfgC)),
        ("osh_nccl_unique_id", c_int32, c_void_p),
        ("osh_ctx_create", c_int32, c_int32, c_int32, c_int32, c_int32, c_void_p,
         POINTER(c_void_p)),
        ("osh_ctx_destroy", c_int32, c_void_p),
        ("osh_ctx_create_tp", c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32,
         c_void_p, c_void_p, POINTER(c_void_p)),
        ("osh_ctx_set_tp_capacity", c_int32, c_void_p, c_uint64),
        ("osh_ctx_set_collectives", c_int32, c_void_p, c_int32),
        ("osh_shampoo_cfg_default", c_int32, POINTER(ShampooCfgC)),
        ("osh_ctx_set_optimizer", c_int32, c_void_p, c_int32, POINTER(ShampooCfgC)),
        ("osh_ctx_save_state", c_int32, c_void_p, c_char_p),
        ("osh_bucket_ready", c_int32, c_void_p, c_int32, c_void_p),
        ("osh_ctx_set_strategy", c_int32, c_void_p, c_int32, c_void_p, c_int32, c_void_p),
        ("osh_ctx_load_state", c_int32, c_void_p, c_char_p),
        ("osh_ctx_set_layout", c_int32, c_void_p, POINTER(ParamDesc), c_int32, c_int64,
         POINTER(c_int64), c_int32, c_int32, c_int64),
        ("osh_ctx_get_info", c_int32, c_void_p, POINTER(CtxInfo)),
        ("osh_ctx_buffers", c_int32, c_void_p, POINTER(c_void_p), POINTER(c_void_p)),
        ("osh_load_param", c_int32, c_void_p, c_int32, POINTER(c_float)),
        ("osh_write_grad", c_int32, c_void_p, c_int32, POINTER(c_float)),
        ("osh_fill_synthetic", c_int32, c_void_p, c_uint64, c_int32, c_float),
        ("osh_step", c_int32, c_void_p, POINTER(MuonCfgC), c_void_p, c_void_p),
        ("osh_ctx_sync", c_int32, c_void_p),
        ("osh_last_timing", c_int32, c_void_p, POINTER(StepTiming)),
        ("osh_update_norms", c_int32, c_void_p, POINTER(c_double)),
        ("osh_read_param", c_int32, c_void_p, c_int32, c_int32, POINTER(c_float)),
        ("osh_ctx_stream", c_int32, c_void_p, POINTER(c_void_p)),
        ("osh_set_gemm_cta_group", c_int32, c_int32),
        ("osh_gemm_cta_group", c_int32),
        ("osh_ctx_profile_gemm", c_int32, c_void_p, c_int32),
        ("osh_gemm_profile_read", c_int32, c_void_p, POINTER(GemmProfile), c_int32),
        ("osh_gemm_profile_dump", c_int32, c_void_p, ctypes.c_char_p, c_size_t, POINTER(c_size_t)),
        ("osh_comm_schedule", c_int32, POINTER(ParamDesc), c_int32, c_int64, c_int32,
         POINTER(c_int64), c_int32, c_int32, c_void_p, c_void_p, POINTER(CollOp), c_int32,
         POINTER(c_int32)),
        ("osh_ctx_comm_schedule", c_int32, c_void_p, POINTER(CollOp), c_int32, POINTER(c_int32)),
        ("osh_ctx_set_timeout", c_int32, c_void_p, c_double),
        ("osh_ctx_set_host_output", c_int32, c_void_p, c_int32),
        ("osh_write_state", c_int32, c_void_p, c_int32, c_int32, POINTER(c_float)),
        ("osh_muon_apply_host", c_int32, c_int32, POINTER(ParamDesc), POINTER(MuonCfgC),
         POINTER(c_double), POINTER(c_double), POINTER(c_double), POINTER(c_double)),
        ("osh_newton_schulz_host", c_int32, c_int32, POINTER(c_double), c_int64, c_int64, c_int32),
    ]
    for name, restype, *args in optional:
        if hasattr(L, name):
            d(name, restype, *args)
