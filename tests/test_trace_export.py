"""scripts/measured_trace.py: a measured step timeline becomes a Chrome trace
in the reference's trace.hpp schema (traceEvents; "M" process / thread
names; "X" events with name, cat, ph, pid, tid, ts, dur in microseconds)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_measured_timeline_to_chrome_trace(tmp_path):
    tl = {"rank": 1, "dp": 0, "tp": 1, "collectives": "auto",
          "launches": [["momentum_matrix", 0.05, 1.25], ["gram", 1.3, 2.0], ["final", 3.4, 0.5]]}
    src = tmp_path / "timeline_rank1.json"
    src.write_text(json.dumps(tl))
    out = tmp_path / "trace.json"
    subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "measured_trace.py"), str(out), str(src)],
                   check=True, capture_output=True)
    d = json.loads(out.read_text())
    ev = d["traceEvents"]
    x = [e for e in ev if e["ph"] == "X"]
    assert [e["name"] for e in x] == ["momentum_matrix", "gram", "final"]
    for e in x:
        assert set(e) == {"name", "cat", "ph", "pid", "tid", "ts", "dur", "args"}
        assert e["pid"] == 1
    assert x[1]["cat"] == "gemm" and x[1]["tid"] == 2 and x[0]["tid"] == 0
    assert x[1]["ts"] == 1300.0 and x[1]["dur"] == 2000.0  # microseconds
    meta = [e for e in ev if e["ph"] == "M"]
    assert {e["name"] for e in meta} == {"process_name", "thread_name"}
