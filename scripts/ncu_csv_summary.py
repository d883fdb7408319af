"""Summarise an `ncu --metrics ... --csv` capture (one row per kernel
launch and metric) into per-kernel totals: launches, time, tensor-pipe
utilisation (time-weighted), DRAM bytes.

    python scripts/ncu_csv_summary.py capture.csv [out.json] [source note]
"""
import csv
import json
import re
import sys
from collections import defaultdict


def main():
    lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    launches = defaultdict(dict)
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        v = r["Metric Value"].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        unit = r["Metric Unit"]
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ns": 1e-6, "us": 1e-3,
                 "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1.0)
        launches[key][r["Metric Name"]] = v * scale
    per = defaultdict(lambda: {"launches": 0, "ms": 0.0, "tensor_pct_x_ms": 0.0, "dram_bytes": 0.0})
    for (lid, name), m in launches.items():
        k = re.sub(r"\(.*", "", name).replace("void ", "")
        k = re.sub(r"unnamed>::|\(anonymous namespace\)::|osh::", "", k)
        d = per[k]
        ms = m.get("gpu__time_duration.sum", 0.0)
        d["launches"] += 1
        d["ms"] += ms
        d["tensor_pct_x_ms"] += ms * m.get(
            "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", 0.0)
        d["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    out = {"source": sys.argv[3] if len(sys.argv) > 3 else sys.argv[1], "kernels": {}}
    total = sum(d["ms"] for d in per.values())
    for k, d in sorted(per.items(), key=lambda kv: -kv[1]["ms"]):
        out["kernels"][k] = {"launches": d["launches"], "ms": round(d["ms"], 3),
                             "share": round(d["ms"] / total, 4) if total else 0.0,
                             "tensor_pipe_pct": round(d["tensor_pct_x_ms"] / d["ms"], 1) if d["ms"] else 0.0,
                             "dram_GB": round(d["dram_bytes"] / 1e9, 3),
                             "dram_GBps": round(d["dram_bytes"] / (d["ms"] * 1e-3) / 1e9, 1) if d["ms"] else 0.0}
    txt = json.dumps(out, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
