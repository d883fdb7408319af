"""Measured step timelines (scripts/timeline.py output, one file per rank) as
a Chrome trace in the schema of the reference's trace.hpp export
(proj/include/optishard/trace.hpp:24-49: traceEvents, "M" process / thread
names, "X" events with name, cat, ts and dur in microseconds), so a measured
B200 step opens beside the reference simulator's trace
(profiles/r01_sim_trace_lbasc_n4.json) in chrome://tracing / Perfetto.

    python scripts/measured_trace.py out.json timeline_rank0.json [timeline_rank1.json ...]

pid = rank; tid 0 = elementwise kernels (momentum, partial sums, multicast
copies), tid 2 = Newton-Schulz GEMMs (the GEMM stream of the overlapped
schedule). Collectives fused into the kernels (NVLS) have no event of their own.
"""
import json
import sys

GEMM = {"gram", "poly", "update", "final", "stat", "split"}


def main():
    out, files = sys.argv[1], sys.argv[2:]
    ev = []
    for f in files:
        d = json.load(open(f))
        r = int(d["rank"])
        ev.append({"name": "process_name", "ph": "M", "pid": r, "tid": 0,
                   "args": {"name": f"rank {r} (dp {d['dp']}, tp {d['tp']}, {d['collectives']})"}})
        for tid, tname in ((0, "elementwise"), (2, "ns_gemm")):
            ev.append({"name": "thread_name", "ph": "M", "pid": r, "tid": tid, "args": {"name": tname}})
        for mode, start, ms in d["launches"]:
            gemm = mode in GEMM
            ev.append({"name": mode, "cat": "gemm" if gemm else "compute", "ph": "X", "pid": r,
                       "tid": 2 if gemm else 0, "ts": round(start * 1e3, 3), "dur": round(ms * 1e3, 3),
                       "args": {}})
    with open(out, "w") as fo:
        json.dump({"displayTimeUnit": "ms", "traceEvents": ev}, fo)
    print(f"{out}: {sum(1 for e in ev if e['ph'] == 'X')} events from {len(files)} ranks")


if __name__ == "__main__":
    main()
