"""Regenerates tests/golden/ from the REFERENCE planner (test infrastructure).

oracle/_ref/ref_plan_dump is tests/cpp/plan_dump.cpp compiled unmodified
against /root/reference/proj/include (oracle/Makefile, target `ref`). Every
'## <tag>' block of its output is stored as a sha256 digest; a few blocks are
also stored verbatim (*.plan) for the C-ABI serializer tests and for humans.

    make -C oracle ref && python tests/golden/make_golden.py
"""
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref", "ref_plan_dump")
CONFIGS = ["toy", "qwen3-0p6b-like", "qwen3-1p7b-like", "qwen3-8b-like", "qwen3-14b-like",
           "qwen3-32b-like"]
FUZZ = ("20260819", "1000")
VERBATIM = {  # (config, tag prefix) -> file
    ("toy", "toy tp 1 R 4 flops-muon alpha-balanced 1"): "toy_R4_flops-muon_a1.plan",
    ("toy", "toy tp 2 R 4 numel alpha-balanced 1"): "toy_tp2_R4_numel_a1.plan",
}
for R in (1, 2, 4, 8):
    VERBATIM[("qwen3-8b-like", f"qwen3-8b-like tp 1 R {R} numel alpha-balanced 1")] = \
        f"qwen3-8b-like_R{R}_numel_a1.plan"
    VERBATIM[("qwen3-0p6b-like", f"qwen3-0p6b-like tp 1 R {R} numel alpha-balanced 1")] = \
        f"qwen3-0p6b-like_R{R}_numel_a1.plan"


def blocks(text):
    """Splits dump output into (tag, body) pairs at '## ' lines."""
    out, tag, body = [], None, []
    for line in text.splitlines(keepends=True):
        if line.startswith("## "):
            if tag is not None:
                out.append((tag, "".join(body)))
            tag, body = line[3:].rstrip("\n"), []
        elif line.startswith("# "):
            if tag is not None:
                out.append((tag, "".join(body)))
            tag, body = None, []
            out.append((line[2:].rstrip("\n"), ""))
        else:
            body.append(line)
    if tag is not None:
        out.append((tag, "".join(body)))
    return out


def digest_lines(text):
    return "".join(f"{hashlib.sha256((t + '\n' + b).encode()).hexdigest()[:24]}  {t}\n"
                   for t, b in blocks(text))


def main():
    if not os.path.exists(REF):
        sys.exit(f"{REF} missing: run `make -C oracle ref` (needs /root/reference)")
    for cfg in CONFIGS:
        text = subprocess.run([REF, "config", os.path.join(ROOT, "configs", cfg + ".cfg")],
                              check=True, capture_output=True, text=True).stdout
        with open(os.path.join(HERE, f"plans_{cfg}.sha"), "w") as f:
            f.write(digest_lines(text))
        for tag, body in blocks(text):
            name = VERBATIM.get((cfg, tag))
            if name:
                plan = body.split("violations")[0]
                with open(os.path.join(HERE, name), "w") as f:
                    f.write(plan)
    text = subprocess.run([REF, "fuzz", *FUZZ], check=True, capture_output=True, text=True).stdout
    with open(os.path.join(HERE, "plans_fuzz.sha"), "w") as f:
        f.write(digest_lines(text))
    print("golden files written to", HERE)


if __name__ == "__main__":
    main()
