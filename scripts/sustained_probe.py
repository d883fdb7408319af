"""Sustained (seconds-long, back-to-back) throughput of the NS GEMM vs cuBLAS."""
import json, subprocess, sys, threading, time
import torch
sys.path.insert(0, ".")
from paper_2602_06079_b200 import _lib
from scripts.ncu_gemm import mref, run  # noqa  (module runs its own small launches)

def clocks_during(fn, secs):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "100", "-i", "0"], stdout=subprocess.PIPE, text=True)
    lines = []
    th = threading.Thread(target=lambda: lines.extend(p.stdout), daemon=True); th.start()
    r = fn(secs)
    p.terminate(); time.sleep(0.2)
    vals = [l.split(",") for l in lines if "," in l]
    sm = sorted(float(v[0]) for v in vals); pw = sorted(float(v[1]) for v in vals)
    return r, (sm[len(sm)//2] if sm else None), (pw[len(pw)//2] if pw else None)

def loop(launch, flops):
    def f(secs):
        torch.cuda.synchronize(); t0 = time.time(); n = 0
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        while time.time() - t0 < secs:
            for _ in range(10): launch()
            n += 10
            torch.cuda.synchronize()
        e1.record(); torch.cuda.synchronize()
        return flops * n / (e0.elapsed_time(e1) * 1e-3) / 1e12
    return f

bt, m, n = 8, 4096, 12288
x = torch.randn(bt, m, n, device="cuda").mul_(0.01).bfloat16()
a = torch.randn(bt, m, m, device="cuda").mul_(0.01).bfloat16()
oa = torch.empty_like(a); ox = torch.empty_like(x)
g = _lib.GemmProblem(); g.a = mref(x); g.b = mref(x); g.out = mref(oa)
u = _lib.GemmProblem(); u.a = mref(a); u.b = mref(x); u.b_mn_major = 1; u.out = mref(ox); u.aux = mref(x)
gs = _lib.GemmProblem(); gs.a = mref(x); gs.b = mref(x); gs.out = mref(oa); gs.symmetric = 1
xt = x.transpose(1, 2).contiguous()
uk = _lib.GemmProblem(); uk.a = mref(a); uk.b = mref(xt); uk.b_mn_major = 0; uk.out = mref(ox)
F = 2.0 * bt * m * m * n
res = {}
for name, fn in [("ours_gram", lambda: run(0, g)), ("ours_update", lambda: run(2, u, 3.4445)),
                 ("ours_update_noaux", lambda: run(2, u, 0.0)),
                 ("ours_update_kmajor_b", lambda: run(2, uk, 0.0)),
                 ("ours_gram_sym(alg flops)", lambda: run(0, gs)),
                 ("cublas_gram", lambda: torch.matmul(x, x.transpose(1, 2), out=oa)),
                 ("cublas_update", lambda: torch.matmul(a, x, out=ox))]:
    tf, sm, pw = clocks_during(loop(fn, F), 4.0)
    res[name] = {"tflops": round(tf, 1), "sm_mhz_median": sm, "power_w_median": pw,
                 "tflops_per_mhz": round(tf / sm, 4) if sm else None,
                 "gflop_per_joule": round(tf * 1e3 / pw, 1) if pw else None}
print(json.dumps(res, indent=1))
