"""Isolated GRAM / POLY / UPDATE timings (8 x 4096x12288 iterate, CUDA events,
20 launches each after warm-up) for a same-box A/B of two builds:
    OSH_LIB=ab/other.so python scripts/iso_gemm_ab.py [--upper]
--upper: the step's upper-tile form (symmetric = 3 outputs, a_upper / b_upper)."""
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
    up = "--upper" in sys.argv or "--upper2" in sys.argv
    full_in = "--upper2" in sys.argv  # GRAM mirrored, POLY reads it whole, POLY out upper-form
    bt, m, n = 8, 4096, 12288
    x = torch.randn(bt, m, n, device="cuda").mul_(0.01).bfloat16()
    a = torch.randn(bt, m, m, device="cuda").mul_(0.01)
    a = (a + a.transpose(1, 2)).mul_(0.5).bfloat16().contiguous()
    oa, ox = torch.empty_like(a), torch.empty_like(x)
    g = _lib.GemmProblem(); g.a = mref(x); g.b = mref(x); g.out = mref(oa)
    g.symmetric = 3 if up and not full_in else 1
    pl = _lib.GemmProblem(); pl.a = mref(a); pl.b = mref(a); pl.out = mref(oa); pl.aux = mref(a)
    pl.symmetric = 3 if up else 1
    if up and not full_in:
        pl.a_upper = pl.b_upper = 1
    u = _lib.GemmProblem(); u.a = mref(a); u.b = mref(x); u.b_mn_major = 1; u.out = mref(ox)
    if up:
        u.a_upper = 1
    L = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    out = {"lib": os.environ.get("OSH_LIB", "libosh.so"), "upper": up, "poly_reads_full": full_in}
    for name, mode, p, al, be in (("gram", 0, g, 0.0, 0.0), ("poly", 1, pl, -4.775, 2.0315),
                                  ("update", 2, u, 0.0, 0.0)):
        arr = (_lib.GemmProblem * 1)(p)
        for _ in range(3):
            _lib.check(L.osh_ns_gemm(mode, arr, 1, al, be, 0.0, s))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            _lib.check(L.osh_ns_gemm(mode, arr, 1, al, be, 0.0, s))
        e1.record()
        torch.cuda.synchronize()
        out[name] = round(e0.elapsed_time(e1) / 20, 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
