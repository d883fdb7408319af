"""The reference's CPU optimizer step, timed — bench.py's reference arm and
cpu_baseline leg (TEST INFRASTRUCTURE / CPU BASELINE ONLY; nothing under
paper_2602_06079_b200/ is imported here).

Planning uses the REFERENCE planner: oracle/_ref/ref_plan_dump is
tests/cpp/plan_dump.cpp compiled unmodified against
/root/reference/proj/include (oracle/Makefile `ref`); its `plan` mode prints
the parameter list (generate_transformer_params, workload.hpp:113-148), the
serialized plan (serialize.hpp:252-271) and the owner table
(dp_partition.hpp:374-395).

The step is the reference's run_replicated / run_partitioned per-step work
(verify.hpp:180-210,225-322) restated in oracle/muon_oracle.c: per owned
tensor, the ascending-rank gradient sum (reduced_gradient), the momentum,
the 5-iteration Newton-Schulz in the reference's 3-product form
(verify.hpp:126-130: A = X Xᵀ, B = A X, C = A B — 6 m² n flops per
iteration) through numpy's OpenBLAS dgemm on every host core, and the
update. A full 8B step is ~4.5 PFLOP of fp64 — about an hour on a 16-core
host — so each timed step is a BOUNDED SAMPLE of it:

  * one COMPLETE Newton-Schulz iteration on a FULL-SIZE matrix of one of the
    model's shape classes (rotating over the classes step by step; at 8B
    4096x4096, 4096x12288 and the 4096x151936 vocabulary class), and
  * one elementwise pass (contributor sum + momentum + update) over 1e8
    elements,

and the step time is extrapolated from the latest sample of every class:
t_rank = Σ_{owned matrices} 5 · t_iter(class) + t_elem · owned elements,
value = max over ranks (the per-rank critical path; = the replicated
run_replicated step at R = 1). Nothing is scaled along a matrix dimension.
"""
from __future__ import annotations

import os
import subprocess
import time
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_PLAN_DUMP = os.path.join(HERE, "_ref", "ref_plan_dump")
ALPHA_GRID = (1.0, 0.75, 0.5, 0.25, 0.0)


class RefPlan:
    """One reference plan: params [(id, name, shape)], cuts [bucket][R+1],
    rank loads, owners per param, and the serialized text."""

    def __init__(self, text: str, source: str):
        self.params: List[Tuple[int, str, Tuple[int, ...]]] = []
        self.cuts: List[List[int]] = []
        self.loads: List[int] = []
        self.owners: List[int] = []
        self.source = source
        body = []
        for line in text.splitlines():
            f = line.split()
            if not f:
                continue
            if f[0] == "param":
                self.params.append((int(f[1]), f[2], tuple(int(x) for x in f[3:])))
                continue
            if f[0] == "owners":
                self.owners = [int(x) for x in f[1:]]
                continue
            body.append(line)
            if f[0] == "bucket":
                self.cuts.append([int(x) for x in f[3:]])
            elif f[0] == "loads":
                self.loads = [int(x) for x in f[1:]]
            elif f[0] == "ranks":
                self.ranks = int(f[1])
        self.text = "\n".join(body) + "\n"


def reference_plan(cfg_path: str, ranks: int, method: str = "alpha-balanced", cost: str = "numel",
                   alpha: float = 1.0) -> RefPlan:
    if os.access(REF_PLAN_DUMP, os.X_OK):
        out = subprocess.run([REF_PLAN_DUMP, "plan", cfg_path, str(ranks), method, cost,
                              repr(float(alpha))], check=True, capture_output=True, text=True)
        return RefPlan(out.stdout, "reference planner (oracle/_ref/ref_plan_dump)")
    raise RuntimeError("the reference planner is not built on this host: run "
                       "`make -C oracle ref` where /root/reference exists (oracle/_ref travels "
                       "with the repository snapshot)")


def ns_gemm_flops(shape: Sequence[int], ns_steps: int = 5) -> float:
    """Algorithmic GEMM flops of the polynomial form, 5·(4m²n + 2m³) (the
    bench's roofline unit)."""
    if len(shape) != 2:
        return 0.0
    m, n = float(min(shape)), float(max(shape))
    return ns_steps * (4.0 * m * m * n + 2.0 * m * m * m)


def choose_alpha(cfg_path: str, ranks: int, cost: str = "numel", min_gain: float = 0.015):
    """The bench's α rule on the REFERENCE planner: α = 1 (the paper's
    default) unless another α of the grid lowers the planned per-rank
    NS-flop max/mean by more than `min_gain` (relative)."""
    best, base = None, None
    for a in ALPHA_GRID:
        plan = reference_plan(cfg_path, ranks, "alpha-balanced", cost, a)
        per = [0.0] * ranks
        for (pid, _, shape), o in zip(plan.params, plan.owners):
            per[o] += ns_gemm_flops(shape)
        mean = sum(per) / ranks
        ratio = max(per) / mean if mean > 0 else 1.0
        if base is None:
            best, base = (a, ratio), ratio
        elif ratio < best[1] - 1e-12 and ratio < base * (1.0 - min_gain):
            best = (a, ratio)
    return best


class CpuStep:
    """Samples and extrapolates the reference CPU step (see module doc)."""

    def __init__(self, plan: RefPlan, contributors: int, threads: Optional[int] = None,
                 elem_sample: int = 100_000_000, budget_s: float = 150.0):
        self.plan = plan
        self.R = contributors
        self.fast = O.set_fast_blas(True)
        if threads:
            O.lib().orc_set_threads(threads)
        self.cores = O.lib().orc_get_threads()
        self.classes: Dict[Tuple[int, int], int] = {}
        for _, _, shape in plan.params:
            if len(shape) == 2:
                k = (min(shape), max(shape))
                self.classes[k] = self.classes.get(k, 0) + 1
        self.order = sorted(self.classes)  # smallest first
        self.t_iter: Dict[Tuple[int, int], float] = {}
        self.t_elem: Optional[float] = None
        self.elem_sample = elem_sample
        self.budget_s = budget_s  # re-samples after the first round stay within this
        self.spent_s = 0.0
        self.rng = np.random.default_rng(0)

    def _time_iteration(self, cls: Tuple[int, int]) -> float:
        m, n = cls
        x = self.rng.standard_normal((m, n))
        t0 = time.perf_counter()
        O.newton_schulz(x, 1)
        return time.perf_counter() - t0

    def _time_elementwise(self) -> float:
        """Per element: R-1 contributor adds + momentum + update (fp64)."""
        k = self.elem_sample
        if not hasattr(self, "_ew"):
            self._ew = (np.zeros((k, 1)), np.zeros((k, 1)), self.rng.standard_normal((k, 1)))
        w, mo, g = self._ew
        t0 = time.perf_counter()
        acc = g.copy()
        for _ in range(1, self.R):
            acc += g
        O.muon_apply(False, O.OptimizerConfig(), w, mo, acc)
        return (time.perf_counter() - t0) / k

    def warmup_sample(self) -> float:
        """A warm-up step: the smallest class only (BLAS threads / page
        faults); its timing is discarded."""
        t0 = time.perf_counter()
        self._time_iteration(self.order[0])
        return time.perf_counter() - t0

    def sample(self, i: int) -> Tuple[float, str]:
        """Timed step i. The first timed step runs one complete iteration of
        EVERY class; later steps re-sample the classes in rotation (class
        i mod #classes), skipping to the cheapest class when the rotation's
        class would overrun the run's time budget (the 8B vocabulary class
        costs ~15 TFLOP per iteration). Every step also times the elementwise
        pass. Returns (wall seconds of the sample, what was sampled)."""
        t0 = time.perf_counter()
        todo = [c for c in self.order if c not in self.t_iter]
        if not todo:
            c = self.order[i % len(self.order)]
            if self.spent_s + self.t_iter[c] > self.budget_s:
                c = self.order[0]
            todo = [c]
        for c in todo:
            self.t_iter[c] = self._time_iteration(c)
        self.t_elem = self._time_elementwise()
        dt = time.perf_counter() - t0
        self.spent_s += dt
        return dt, ",".join(f"{m}x{n}" for m, n in todo)

    def estimate(self) -> dict:
        ranks = self.plan.ranks
        rank_s = [0.0] * ranks
        for (pid, _, shape), o in zip(self.plan.params, self.plan.owners):
            numel = int(np.prod(shape))
            t = self.t_elem * numel
            if len(shape) == 2:
                t += 5 * self.t_iter[(min(shape), max(shape))]
            rank_s[o] += t
        return {"critical_path_ms": 1e3 * max(rank_s), "full_ms": 1e3 * sum(rank_s),
                "rank_ms": [1e3 * t for t in rank_s],
                "iter_ms": {f"{m}x{n}": round(1e3 * t, 1) for (m, n), t in sorted(self.t_iter.items())},
                "elem_ns": round(1e9 * self.t_elem, 3)}

    def describe(self) -> str:
        cls = ", ".join(f"{m}x{n} x{c}" for (m, n), c in sorted(self.classes.items()))
        return (f"complete fp64 Newton-Schulz iterations (reference 3-product form, "
                f"{'OpenBLAS dgemm' if self.fast else 'blocked C GEMM'}, {self.cores} threads) on "
                f"full-size matrices of the shape classes [{cls}]: every class in the first timed "
                f"step, then one class per step in rotation within a {self.budget_s:.0f} s "
                f"budget; plus a {self.elem_sample:.0e}-element contributor-sum/momentum/update "
                f"pass per step; extrapolated to 5 iterations x every owned tensor, max over "
                f"ranks")
