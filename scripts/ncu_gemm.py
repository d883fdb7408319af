"""One launch of each NS GEMM mode at Qwen3-8B shape classes (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_06079_b200 import _lib  # noqa: E402


def mref(t):
    m = _lib.MatrixRef()
    m.ptr = t.data_ptr()
    m.batch, m.rows, m.cols = t.shape
    m.ld = t.stride(1)
    m.bstride = t.stride(0)
    return m


def run(mode, p, alpha=0.0, beta=0.0):
    arr = (_lib.GemmProblem * 1)(p)
    _lib.check(_lib.lib().osh_ns_gemm(mode, arr, 1, alpha, beta, 0.0,
                                      torch.cuda.current_stream().cuda_stream))


bt, m, n = 8, 4096, 12288
x = torch.randn(bt, m, n, device="cuda").mul_(0.01).bfloat16()
a = torch.randn(bt, m, m, device="cuda").mul_(0.01).bfloat16()
oa = torch.empty_like(a)
ox = torch.empty_like(x)
# --upper: the step's upper-tile form (GRAM / POLY outputs without the
# off-diagonal mirror, POLY / UPDATE reading left-of-diagonal k-blocks from it)
up = '--upper' in sys.argv
sym = (3 if up else 1) if '--sym' in sys.argv else 0
a = (a.float() + a.float().transpose(1, 2)).mul_(0.5).bfloat16().contiguous()  # symmetric
g = _lib.GemmProblem(); g.a = mref(x); g.b = mref(x); g.out = mref(oa); g.symmetric = sym
pl = _lib.GemmProblem(); pl.a = mref(a); pl.b = mref(a); pl.out = mref(oa); pl.aux = mref(a); pl.symmetric = sym
pl.a_upper = pl.b_upper = int(up)
u = _lib.GemmProblem(); u.a = mref(a); u.b = mref(x); u.b_mn_major = 1; u.out = mref(ox); u.aux = mref(x)
u.a_upper = int(up)
# --noaux: the step's UPDATE form (the 'a X' term folded into B by POLY: no aux read)
ua = 0.0 if '--noaux' in sys.argv else 3.4445
for _ in range(2):  # warm-up
    run(0, g); run(1, pl, -4.775, 2.0315); run(2, u, ua)
torch.cuda.synchronize()
run(0, g); run(1, pl, -4.775, 2.0315); run(2, u, ua)
torch.cuda.synchronize()
print("ok")
