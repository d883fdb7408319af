"""Bit-exact partition assignment (north star item 1).

Golden files in tests/golden/ come from the REFERENCE planner
(oracle/_ref/ref_plan_dump = tests/cpp/plan_dump.cpp compiled unmodified
against /root/reference/proj/include; tests/golden/make_golden.py). Here the
same dump program is compiled against this repo's include/optishard and every
plan block (serialized plan, validation, %.17g metrics, owner table, micro-group
plans, a1-style fuzz corpus) must hash identically. The C ABI (libosh.so) must
serialize the verbatim golden plans byte for byte.
"""
import glob
import hashlib
import os
import subprocess

import numpy as np
import pytest

from paper_2602_06079_b200 import _lib
from paper_2602_06079_b200 import planner as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
DUMP = os.path.join(ROOT, "build", "plan_dump")
CONFIGS = ["toy", "qwen3-0p6b-like", "qwen3-1p7b-like", "qwen3-8b-like", "qwen3-14b-like",
           "qwen3-32b-like"]


@pytest.fixture(scope="module")
def dump_bin():
    src = os.path.join(ROOT, "tests", "cpp", "plan_dump.cpp")
    headers = glob.glob(os.path.join(ROOT, "include", "optishard", "*.hpp"))
    newest = max(os.path.getmtime(p) for p in headers + [src])
    if not os.path.exists(DUMP) or os.path.getmtime(DUMP) < newest:
        os.makedirs(os.path.dirname(DUMP), exist_ok=True)
        subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-Wall", "-Wextra",
                        "-I", os.path.join(ROOT, "include"), src, "-o", DUMP], check=True)
    return DUMP


def digests(text):
    out, tag, body = [], None, []

    def flush():
        if tag is not None:
            out.append(f"{hashlib.sha256((tag + chr(10) + ''.join(body)).encode()).hexdigest()[:24]}  {tag}")

    for line in text.splitlines(keepends=True):
        if line.startswith("## "):
            flush()
            tag, body = line[3:].rstrip("\n"), []
        elif line.startswith("# "):
            flush()
            tag, body = None, []
            t = line[2:].rstrip("\n")
            out.append(f"{hashlib.sha256((t + chr(10)).encode()).hexdigest()[:24]}  {t}")
        else:
            body.append(line)
    flush()
    return out


def compare(got_lines, gold_path):
    want = open(gold_path).read().splitlines()
    assert len(got_lines) == len(want), (len(got_lines), len(want))
    bad = [(g, w) for g, w in zip(got_lines, want) if g != w]
    assert not bad, f"{len(bad)} blocks differ, first: {bad[0]}"


@pytest.mark.parametrize("cfg", CONFIGS)
def test_cpp_planner_matches_reference(dump_bin, cfg):
    text = subprocess.run([dump_bin, "config", os.path.join(ROOT, "configs", cfg + ".cfg")],
                          check=True, capture_output=True, text=True).stdout
    compare(digests(text), os.path.join(GOLD, f"plans_{cfg}.sha"))


def test_cpp_planner_fuzz_corpus_matches_reference(dump_bin):
    text = subprocess.run([dump_bin, "fuzz", "20260819", "1000"], check=True, capture_output=True,
                          text=True).stdout
    compare(digests(text), os.path.join(GOLD, "plans_fuzz.sha"))


def _params(name):
    return P.generate_transformer_params(P.load_config(os.path.join(ROOT, "configs", name + ".cfg")))


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "*.plan"))))
def test_capi_serializes_golden_plans(path):
    base = os.path.basename(path)[:-5]
    parts = base.split("_")
    cfg = P.load_config(os.path.join(ROOT, "configs", parts[0] + ".cfg"))
    tp = 1
    rest = parts[1:]
    if rest[0].startswith("tp"):
        tp = int(rest[0][2:])
        rest = rest[1:]
    R, cost, alpha = int(rest[0][1:]), rest[1], float(rest[2][1:])
    params = P.apply_tp_sharding(P.generate_transformer_params(cfg), tp)
    cap = cfg.bucket_capacity if tp == 1 else cfg.bucket_capacity // tp
    got = P.serialize_dp_plan(params, cap, R, "alpha-balanced", cost, alpha)
    assert got == open(path).read()


def test_readme_toy_plan():
    """proj/README.md:93-99: toy, dp 4, flops-muon, alpha 1."""
    params = _params("toy")
    plan = P.plan_dp(params, 200, 4, "alpha-balanced", "flops-muon", 1.0)
    assert plan.rank_loads.tolist() == [49920, 40960, 65280, 40984]


# ---- hand traces of proj/tests/test_dp_partition.cpp, through the C ABI ----
def vec_params(numels):
    return [P.ParamSpec(i, f"p{i}", (n,)) for i, n in enumerate(numels)]


def test_single_bucket_even_split():  # test_dp_partition.cpp:58-69
    plan = P.plan_dp(vec_params([8, 4, 2, 2]), 16, 2)
    assert plan.cut_vectors.tolist() == [[0, 8, 16]] and plan.rank_loads.tolist() == [8, 8]
    assert plan.atomic and plan.alpha == 1.0


def test_cross_bucket_compensation():  # :71-89
    plan = P.plan_dp(vec_params([7, 3, 3, 3]), 10, 2)
    assert plan.cut_vectors.tolist() == [[0, 7, 10], [0, 0, 6]]
    assert plan.rank_loads.tolist() == [7, 9]


def test_tie_takes_smaller_offset():  # :91-99
    plan = P.plan_dp(vec_params([2]), 2, 2, alpha=0.0)
    assert plan.cut_vectors.tolist() == [[0, 0, 2]] and plan.rank_loads.tolist() == [0, 2]


def test_stride_ownership():  # :101-119, :272-281
    ps = vec_params([4, 2, 2])
    plan = P.plan_dp(ps, 8, 4, "atomic-ownership")
    assert plan.rank_loads.tolist() == [4, 0, 2, 2]
    assert plan.cut_vectors.tolist() == [[0, 4, 4, 6, 8]]
    assert P.param_owners(ps, 8, plan).tolist() == [0, 2, 3]
    assert P.plan_dp(vec_params([3, 3, 2]), 8, 2, "atomic-ownership").rank_loads.tolist() == [6, 2]


def test_equal_chunk():  # :121-133
    plan = P.plan_dp(vec_params([10]), 10, 4, "equal-chunk")
    assert plan.cut_vectors.tolist() == [[0, 3, 5, 8, 10]] and not plan.atomic
    assert plan.rank_sizes.tolist() == [[3, 2, 3, 2]]


def test_single_rank_owns_everything():  # :135-150
    for method in P.METHODS:
        plan = P.plan_dp(vec_params([5, 9, 2]), 16, 1, method)
        assert plan.rank_loads.tolist() == [16] and plan.atomic


def test_error_taxonomy():  # :152-161 and workload/layout errors
    with pytest.raises(_lib.OshError) as e:
        P.plan_dp(vec_params([4]), 4, 2, alpha=1.5)
    assert e.value.code == 1  # ConfigError
    with pytest.raises(_lib.OshError) as e:
        P.plan_dp(vec_params([4]), 4, 2, alpha=-0.1)
    assert e.value.code == 1
    with pytest.raises(_lib.OshError) as e:
        P.plan_dp(vec_params([4]), 4, 0)
    assert e.value.code == 5  # PlanError
    with pytest.raises(_lib.OshError) as e:
        P.build_buffer_layout(vec_params([5]), 4)
    assert e.value.code == 2  # LayoutError
    with pytest.raises(_lib.OshError) as e:
        P.serialize_tp_plan([(0, 7), (1, 2)], 2, 6)
    assert e.value.code == 6 and "param 0" in str(e.value) and "7" in str(e.value)


def test_micro_group_hand_traces():  # test_tp_schedule.cpp:328-337
    text = P.serialize_tp_plan([(0, 6), (1, 5), (2, 4)], 2, 6)
    groups = P.parse_tp_plan(text)
    assert groups == {0: (0, 0), 1: (0, 1), 2: (1, 0)}
    assert "group 0 lmax 6" in text and "group 1 lmax 4" in text


def test_big_model_balance_a2():
    """acceptance a2 (acceptance_main.cpp:156-175): 32B-like, R=32, flops."""
    cfg = P.load_config(os.path.join(ROOT, "configs", "qwen3-32b-like.cfg"))
    params = P.generate_transformer_params(cfg)
    strided = P.plan_dp(params, cfg.bucket_capacity, 32, "atomic-ownership", "flops-muon")
    bal = P.plan_dp(params, cfg.bucket_capacity, 32, "alpha-balanced", "flops-muon")

    def rlb(x):
        x = np.asarray(x, dtype=np.float64)
        return x.max() / x.mean()

    assert rlb(strided.rank_loads) >= 2.0 and rlb(bal.rank_loads) <= 1.5
    assert rlb(strided.rank_sizes.sum(0)) >= 1.8 and rlb(bal.rank_sizes.sum(0)) <= 1.3
