"""Times the symmetric POLY GEMM (B = b·A + c·A·A) of the NS iteration at
in-step batch sizes, for a same-box A/B of two builds:

    OSH_LIB=ab/libosh_base.so python scripts/poly_ab.py   vs   python scripts/poly_ab.py

One JSON line: ms and executed TFLOP/s (symmetric tiles only) per shape.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_06079_b200 import _lib  # noqa: E402


def mref(t):
    m = _lib.MatrixRef()
    m.ptr = t.data_ptr(); m.batch, m.rows, m.cols = t.shape
    m.ld = t.stride(1); m.bstride = t.stride(0)
    return m


def main():
    L = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    out = {"lib": os.environ.get("OSH_LIB", "libosh.so")}
    for bt, m in [(20, 4096), (16, 1024)]:
        a = torch.randn(bt, m, m, device="cuda").mul_(0.01).bfloat16()
        a = (a + a.transpose(1, 2)).contiguous()
        o = torch.empty_like(a)
        p = _lib.GemmProblem(); p.a = mref(a); p.b = mref(a); p.out = mref(o); p.aux = mref(a)
        p.symmetric = 1
        arr = (_lib.GemmProblem * 1)(p)
        for _ in range(3):
            _lib.check(L.osh_ns_gemm(1, arr, 1, -4.775, 2.0315, 0.0, s))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 20
        e0.record()
        for _ in range(iters):
            _lib.check(L.osh_ns_gemm(1, arr, 1, -4.775, 2.0315, 0.0, s))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        tiles = (m // 256) * (m // 256 + 1) // 2
        f = bt * tiles * 2.0 * 256 * 256 * m
        out[f"poly_{bt}x{m}"] = {"ms": round(ms, 4), "tflops_exec": round(f / ms / 1e9, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
