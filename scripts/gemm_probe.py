"""Times the grouped tcgen05 NS GEMM at the Qwen3-8B shape classes (CUDA events)."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_06079_b200 import _lib  # noqa: E402


def mref(t):
    m = _lib.MatrixRef()
    m.ptr = t.data_ptr(); m.batch, m.rows, m.cols = t.shape
    m.ld = t.stride(1); m.bstride = t.stride(0)
    return m


def bench(mode, probs, alpha=0.0, beta=0.0, iters=5, lr=0.0):
    arr = (_lib.GemmProblem * len(probs))(*probs)
    s = torch.cuda.current_stream().cuda_stream
    L = _lib.lib()
    for _ in range(2):
        _lib.check(L.osh_ns_gemm(mode, arr, len(probs), alpha, beta, lr, s))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        _lib.check(L.osh_ns_gemm(mode, arr, len(probs), alpha, beta, lr, s))
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    out = {}
    for (bt, m, n) in [(4, 4096, 12288), (4, 4096, 4096), (1, 4096, 151936), (32, 1024, 3072)]:
        x = torch.randn(bt, m, n, device="cuda").mul_(0.01).bfloat16()
        a = torch.randn(bt, m, m, device="cuda").mul_(0.01).bfloat16()
        o_mm = torch.empty(bt, m, m, device="cuda", dtype=torch.bfloat16)
        o_mn = torch.empty_like(x)
        p = _lib.GemmProblem(); p.a = mref(x); p.b = mref(x); p.out = mref(o_mm)
        t = bench(0, [p]); f = 2.0 * bt * m * m * n
        out[f"gram_{bt}x{m}x{n}"] = {"ms": t, "tflops": f / t / 1e9}
        p = _lib.GemmProblem(); p.a = mref(a); p.b = mref(a); p.out = mref(o_mm); p.aux = mref(a)
        t = bench(1, [p], -4.775, 2.0315); f = 2.0 * bt * m * m * m
        out[f"poly_{bt}x{m}x{m}"] = {"ms": t, "tflops": f / t / 1e9}
        p = _lib.GemmProblem(); p.a = mref(a); p.b = mref(x); p.b_mn_major = 1; p.out = mref(o_mn); p.aux = mref(x)
        t = bench(2, [p], 3.4445); f = 2.0 * bt * m * m * n
        out[f"update_{bt}x{m}x{n}"] = {"ms": t, "tflops": f / t / 1e9}
        p.aux = _lib.MatrixRef()
        t = bench(2, [p], 0.0)
        out[f"update_noaux_{bt}x{m}x{n}"] = {"ms": t, "tflops": f / t / 1e9}
        # FINAL: W -= lr * (A X) in the epilogue, W fp32 in both orientations
        if bt * m * n <= 4 * 4096 * 12288:
            for tr in (0, 1):
                w = torch.zeros(bt, n, m, device="cuda") if tr else torch.zeros(bt, m, n, device="cuda")
                rep = torch.empty(w.shape, device="cuda", dtype=torch.bfloat16)
                tg = (_lib.FinalTarget * bt)()
                for i in range(bt):
                    tg[i].w = w[i].data_ptr(); tg[i].replica = rep[i].data_ptr(); tg[i].transposed = tr
                p.final_targets = ctypes.addressof(tg)
                t = bench(3, [p], 0.0, lr=0.02)
                out[f"final_t{tr}_{bt}x{m}x{n}"] = {"ms": t, "tflops": f / t / 1e9}
                del w, rep
        del x, a, o_mm, o_mn
        torch.cuda.empty_cache()
    # cuBLAS reference point for the same shapes
    x = torch.randn(4, 4096, 12288, device="cuda").bfloat16()
    torch.matmul(x, x.transpose(1, 2)); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        torch.matmul(x, x.transpose(1, 2))
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 5
    out["cublas_gram_4x4096x12288"] = {"ms": t, "tflops": 2.0 * 4 * 4096 * 4096 * 12288 / t / 1e9}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
