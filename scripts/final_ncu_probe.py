import ctypes, sys, torch
sys.path.insert(0, ".")
from paper_2602_06079_b200 import _lib
def mref(t):
    m = _lib.MatrixRef(); m.ptr = t.data_ptr(); m.batch, m.rows, m.cols = t.shape
    m.ld = t.stride(1); m.bstride = t.stride(0); return m
bt, m, n = 4, 4096, 12288
x = torch.randn(bt, m, n, device="cuda").mul_(0.01).bfloat16()
a = torch.randn(bt, m, m, device="cuda").mul_(0.01).bfloat16()
o = torch.empty_like(x)
L = _lib.lib(); s = torch.cuda.current_stream().cuda_stream
p = _lib.GemmProblem(); p.a = mref(a); p.b = mref(x); p.b_mn_major = 1; p.out = mref(o)
arr = (_lib.GemmProblem * 1)(p)
_lib.check(L.osh_ns_gemm(2, arr, 1, 0.0, 0.0, 0.0, s))
for tr in (0, 1):
    w = torch.zeros(bt, n, m, device="cuda") if tr else torch.zeros(bt, m, n, device="cuda")
    rep = torch.empty(w.shape, device="cuda", dtype=torch.bfloat16)
    tg = (_lib.FinalTarget * bt)()
    for i in range(bt):
        tg[i].w = w[i].data_ptr(); tg[i].replica = rep[i].data_ptr(); tg[i].transposed = tr
    p.final_targets = ctypes.addressof(tg)
    arr = (_lib.GemmProblem * 1)(p)
    _lib.check(L.osh_ns_gemm(3, arr, 1, 0.0, 0.0, 0.02, s))
torch.cuda.synchronize()
print("ok")
