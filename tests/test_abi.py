"""The C ABI boundary without a GPU: libosh.so loads, exports every function
include/osh.h declares, the ctypes mirrors in _lib.py have the C structs'
sizes and field offsets, and the GPU-free entry points validate arguments.
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2602_06079_b200 import _lib
from paper_2602_06079_b200 import planner as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "osh.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?(?:osh_status|int32_t|int|void|char\s*\*|const char\s*\*)\s*\*?\s*"
                       r"(osh_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_every_declared_function_is_exported():
    names = declared_functions()
    assert len(names) >= 45, names
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert _lib.lib().osh_abi_version() == 1


STRUCTS = {
    "osh_param_desc": _lib.ParamDesc, "osh_cost_model": _lib.CostModelC,
    "osh_muon_cfg": _lib.MuonCfgC, "osh_matrix_ref": _lib.MatrixRef,
    "osh_final_target": _lib.FinalTarget, "osh_gemm_problem": _lib.GemmProblem,
    "osh_ctx_info": _lib.CtxInfo, "osh_shampoo_cfg": _lib.ShampooCfgC,
    "osh_step_timing": _lib.StepTiming, "osh_gemm_profile": _lib.GemmProfile,
    "osh_coll_op": _lib.CollOp,
}


def test_ctypes_structs_match_the_header(tmp_path):
    """sizeof and every field offset of the C structs, from a C compiler,
    equal the ctypes mirrors the Python side passes across the ABI."""
    lines = ["#include <stddef.h>", "#include <stdio.h>", '#include "osh.h"', "int main(void) {"]
    for cname, py in STRUCTS.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = {}
    for line in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines():
        cname, key, val = line.split()
        got[(cname, key)] = int(val)
    for cname, py in STRUCTS.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)


def test_gpu_free_entry_points_validate_arguments():
    L = _lib.lib()
    assert L.osh_ctx_set_timeout(None, 1.0) == 19           # OSH_ERR_ARG
    assert L.osh_ctx_set_host_output(None, 0) == 19
    assert L.osh_ctx_comm_schedule(None, None, 0, None) == 19
    params = P.generate_transformer_params(P.load_config(os.path.join(ROOT, "configs", "toy.cfg")))
    cap = 200
    plan = P.plan_dp(params, cap, 4)
    sched = P.comm_schedule(params, cap, plan)
    # every RS-v leg reduces a slice to its owner; every AG-v leg broadcasts it back
    rs = [(o["offset"], o["count"], o["root"]) for o in sched if o["phase"] == "rs"]
    ag = [(o["offset"], o["count"], o["root"]) for o in sched if o["phase"] == "ag"]
    assert rs == ag and sum(c for _, c, _ in rs) == sum(p.numel for p in params)
    bad = P.DpPartitionPlan(plan.ranks, plan.method, plan.cost_kind, plan.alpha, plan.atomic,
                            plan.cut_vectors[:-1], plan.rank_loads)
    with pytest.raises(_lib.OshError) as e:
        P.comm_schedule(params, cap, bad)
    assert e.value.code == 5  # PlanError: cut vectors must cover every bucket
    broken = plan.cut_vectors.copy()
    broken[0, -1] += 1
    with pytest.raises(_lib.OshError) as e:
        P.comm_schedule(params, cap, P.DpPartitionPlan(plan.ranks, plan.method, plan.cost_kind,
                                                       plan.alpha, plan.atomic, broken,
                                                       plan.rank_loads))
    assert e.value.code == 5
    one = P.plan_dp(params, cap, 1)
    assert P.comm_schedule(params, cap, one) == []  # a single rank exchanges nothing
    assert np.asarray(plan.cut_vectors).shape[1] == 5
