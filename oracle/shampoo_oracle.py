"""fp64 oracle of the BUILDER-DEFINED blocked Shampoo step (TEST INFRASTRUCTURE ONLY).

The reference has no Shampoo/SOAP mathematics — only their planning cost
(proj/include/optishard/cost.hpp:47-48,68-75; SPEC.md:8 puts the optimizer
internals out of scope), so parity is UNPINNED against the reference: this
file is the specification the GPU path (paper_2602_06079_b200/csrc/shampoo*.cu)
is checked against, written in plain numpy fp64 from the published algorithm
(Gupta et al. 2018 "Shampoo", with block partitioning and SGD-norm grafting as
in the Distributed Shampoo implementation; coupled Newton inverse roots,
Higham "Functions of Matrices" 7.3 / Guo & Higham 2006).

Per 2-D tensor that is not vocabulary-space (SURVEY.md §8 A19 policy), the
tensor W (r x c) is cut into blocks of at most `block` rows and columns
(ragged last blocks). For each block with gradient G (p x q), at step t:

    L <- beta2 * L + G G^T            R <- beta2 * R + G^T G          (fp32 state)
    if t % precond_every == 0:        for S in (L, R):
        c = ||S||_F ;  A = S / c + eps * I
        P_S = inv_root4(A, newton_iters) * c^(-1/4)
    U = P_L G P_R
    U <- U * ||G||_F / ||U||_F        (SGD-norm grafting; U = 0 when ||U|| = 0)
    M <- beta1 * M + U ;  W <- W - lr * M

inv_root4 (coupled Newton for A^(-1/4), X0 = I, M0 = A, eigenvalues of A in
(0, 1 + eps]):
    T = (5 I - M) / 4 ;  X <- X T ;  M <- T^4 M         (newton_iters times)

Vectors and vocabulary-space matrices: M <- beta1 M + G ; W <- W - lr M (the
Muon path's vector rule, verify.hpp:143-146).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Tuple

import numpy as np


@dataclass
class ShampooConfig:
    lr: float = 0.02
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-4
    block: int = 1024
    precond_every: int = 10
    newton_iters: int = 16


def blocks(rows: int, cols: int, b: int) -> List[Tuple[int, int, int, int]]:
    """(r0, p, c0, q) of every block, row-major block order."""
    out = []
    for r0 in range(0, rows, b):
        for c0 in range(0, cols, b):
            out.append((r0, min(b, rows - r0), c0, min(b, cols - c0)))
    return out


def inv_root4(a: np.ndarray, iters: int) -> np.ndarray:
    n = a.shape[0]
    eye = np.eye(n)
    x, m = eye.copy(), a.copy()
    for _ in range(iters):
        t = (5.0 * eye - m) / 4.0
        x = x @ t
        t2 = t @ t
        m = (t2 @ t2) @ m
    return x


def inv_root4_exact(a: np.ndarray) -> np.ndarray:
    w, v = np.linalg.eigh(a)
    return (v * w ** -0.25) @ v.T


def precond_root(s: np.ndarray, cfg: ShampooConfig) -> np.ndarray:
    c = float(np.linalg.norm(s))
    if c == 0.0:
        return np.eye(s.shape[0])  # no statistics yet: identity preconditioner
    a = s / c + cfg.eps * np.eye(s.shape[0])
    return inv_root4(a, cfg.newton_iters) * c ** -0.25


class ShampooTensorState:
    def __init__(self, shape, cfg: ShampooConfig, preconditioned: bool):
        self.shape = tuple(shape)
        self.m = np.zeros(self.shape)
        self.pre = preconditioned
        self.blocks = blocks(self.shape[0], self.shape[1], cfg.block) if preconditioned else []
        self.L = [np.zeros((p, p)) for (_, p, _, q) in self.blocks]
        self.R = [np.zeros((q, q)) for (_, p, _, q) in self.blocks]
        self.PL = [np.eye(p) for (_, p, _, q) in self.blocks]
        self.PR = [np.eye(q) for (_, p, _, q) in self.blocks]


def shampoo_apply(st: ShampooTensorState, cfg: ShampooConfig, w: np.ndarray, g: np.ndarray,
                  step: int) -> float:
    """In place on w and the state; returns ||W_new - W_old||_F."""
    g = np.asarray(g, dtype=np.float64).reshape(st.shape)
    if not st.pre:
        st.m = cfg.beta1 * st.m + g
        upd = cfg.lr * st.m
        w -= upd
        return float(np.linalg.norm(upd))
    u_full = np.zeros(st.shape)
    for k, (r0, p, c0, q) in enumerate(st.blocks):
        gb = g[r0:r0 + p, c0:c0 + q]
        st.L[k] = cfg.beta2 * st.L[k] + gb @ gb.T
        st.R[k] = cfg.beta2 * st.R[k] + gb.T @ gb
        if step % cfg.precond_every == 0:
            st.PL[k] = precond_root(st.L[k], cfg)
            st.PR[k] = precond_root(st.R[k], cfg)
        u = st.PL[k] @ gb @ st.PR[k]
        nu, ng = np.linalg.norm(u), np.linalg.norm(gb)
        u_full[r0:r0 + p, c0:c0 + q] = u * (ng / nu) if nu > 0 else 0.0
    st.m = cfg.beta1 * st.m + u_full
    upd = cfg.lr * st.m
    w -= upd
    return float(np.linalg.norm(upd))


def is_preconditioned(p) -> bool:
    """SURVEY.md §8 A19 policy: 2-D, not vocabulary-space."""
    return len(p.shape) == 2 and not p.vocab_space


def run(params, cfg: ShampooConfig, steps: int, seed: int, contributors: int = 1,
        init=None, grad=None) -> Tuple[Dict[int, np.ndarray], List[np.ndarray]]:
    """Replicated trajectory over `params` (planner ParamSpecs) with the
    reference generator's inputs (oracle.init_weight / reduced_gradient)."""
    from oracle import oracle as O
    init = init or (lambda p: O.init_weight(p.shape, p.id, seed).reshape(_shape2(p)))
    grad = grad or (lambda p, s: O.reduced_gradient(p.shape, p.id, seed, s, contributors)
                    .reshape(_shape2(p)))
    w = {p.id: init(p).astype(np.float64) for p in params}
    st = {p.id: ShampooTensorState(_shape2(p), cfg, is_preconditioned(p)) for p in params}
    norms = []
    for s in range(steps):
        n = np.zeros(len(params))
        for p in params:
            n[p.id] = shampoo_apply(st[p.id], cfg, w[p.id], grad(p, s), s)
        norms.append(n)
    return w, norms


def _shape2(p):
    return tuple(p.shape) if len(p.shape) == 2 else (p.shape[0], 1)
