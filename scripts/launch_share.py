"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
`bench.py --steps S --warmup W`: per-kernel serialized time and share of the
optimizer-step kernels (setup kernels such as fill_synth / cast are excluded).

    python scripts/launch_share.py profiles/r01_ncu_launches_bench_n1_final.csv [out.json]
"""
import csv
import json
import re
import sys
from collections import defaultdict

SETUP = ("fill_synth_kernel", "cast_f32_bf16_kernel", "multicast_base_kernel")


def short(name):
    name = re.sub(r"\(.*", "", name.split("::")[-1] if "::" in name else name)
    return name


def main():
    rows = []
    with open(sys.argv[1]) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r["Metric Unit"], 1e-6)
        rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")) * scale))
    per = defaultdict(lambda: [0, 0.0])
    for name, ms in rows:
        k = name.split("(")[0]
        k = re.sub(r"^void ", "", k)
        k = re.sub(r"<unnamed>::|\(anonymous namespace\)::|osh::", "", k)
        per[k][0] += 1
        per[k][1] += ms
    step = {k: v for k, v in per.items() if not any(s in k for s in SETUP)}
    total = sum(v[1] for v in step.values())
    out = {"source": sys.argv[1], "launches": len(rows),
           "step_kernel_ms_serialized": round(total, 3),
           "kernels": {k: {"launches": v[0], "ms": round(v[1], 3), "share_of_step": round(v[1] / total, 4)}
                       for k, v in sorted(step.items(), key=lambda kv: -kv[1][1])},
           "excluded_setup": {k: {"launches": v[0], "ms": round(v[1], 3)} for k, v in per.items()
                              if any(s in k for s in SETUP)}}
    gemm = sum(v[1] for k, v in step.items() if "ns_gemm_kernel" in k)
    out["gemm_share_of_step"] = round(gemm / total, 4)
    txt = json.dumps(out, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
