"""Measured-vs-simulated calibration, run HERE (needs the
reference simulator built by `make -C oracle ref` into oracle/_ref/ref_sim).

The reference prices the optimizer step as max-rank execution cost /
compute_throughput (+ the NV-layerwise broadcast), simulate.hpp:268-295. We
calibrate compute_throughput (flops-muon cost units per second) on ONE
measured number — the N=1 step (profiles/r01_bench_n1_final.json) — and the
inter-GPU bandwidth on the NVLS traffic measured per GPU (~750 GB/s), then
compare the simulator's prediction for every strategy at N=2/4 with the
step times measured on B200 (profiles/r01_strategies_n2_n4.jsonl).
Writes profiles/r01_sim_calibration.json and the simulated LB-ASC N=4 step
as a Chrome trace (profiles/r01_sim_trace_lbasc_n4.json).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SIM = os.path.join(ROOT, "oracle", "_ref", "ref_sim")
MODEL = ["36", "4096", "12288", "32", "151936", "622329856"]
BW, LAT = 750e9, 10e-6


def sim(ranks, strategy, throughput, trace=None):
    args = [SIM, *MODEL, str(ranks), strategy, "flops-muon", repr(throughput), repr(BW), repr(LAT), "1.0"]
    if trace:
        args.append(trace)
    return json.loads(subprocess.run(args, check=True, capture_output=True, text=True).stdout)


def main():
    if not os.path.exists(SIM):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    n1 = json.load(open(os.path.join(ROOT, "profiles", "r01_bench_n1_final.json")))
    # calibration: the R=1 simulated cost with throughput 1 is the total cost
    total_cost = sim(1, "sc", 1.0)["optimizer_compute_s"]
    throughput = total_cost / (n1["value"] * 1e-3)
    measured = {}
    for line in open(os.path.join(ROOT, "profiles", "r01_strategies_n2_n4.jsonl")):
        d = json.loads(line)
        strat = d["config"]["strategy"]
        if strat == "sharded":
            strat = "asc" if d["config"]["plan"].startswith("atomic") else "lb-asc"
        measured[(d["n_gpus"], strat)] = d["value"]
    rows = []
    for n in (2, 4):
        for strat in ("sc", "nv-layerwise", "asc", "lb-asc"):
            s = sim(n, strat, throughput,
                    os.path.join(ROOT, "profiles", "r01_sim_trace_lbasc_n4.json")
                    if (n, strat) == (4, "lb-asc") else None)
            m = measured.get((n, strat))
            rows.append({"ranks": n, "strategy": strat, "simulated_optimizer_ms": round(s["optimizer_s"] * 1e3, 2),
                         "simulated_compute_ms": round(s["optimizer_compute_s"] * 1e3, 2),
                         "simulated_comm_ms": round(s["optimizer_comm_s"] * 1e3, 2),
                         "measured_step_ms": m,
                         "measured_over_simulated": round(m / (s["optimizer_s"] * 1e3), 3) if m else None})
    out = {"calibration": {"exec_cost": "flops-muon", "compute_throughput_cost_per_s": throughput,
                           "from": f"N=1 measured step {n1['value']} ms (profiles/r01_bench_n1_final.json)",
                           "inter_bw_Bps": BW, "latency_s": LAT},
           "note": "the simulator's optimizer step excludes the RS-v / all-reduce it places in the "
                   "backward pass and the AG-v it places in the next forward; the measured step "
                   "includes them (NVLS-fused for LB-ASC / ASC, NCCL for SC / NV-layerwise)",
           "rows": rows}
    json.dump(out, open(os.path.join(ROOT, "profiles", "r01_sim_calibration.json"), "w"), indent=1)
    for r in rows:
        print(r)


if __name__ == "__main__":
    main()
