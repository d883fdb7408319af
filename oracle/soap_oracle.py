"""fp64 oracle of the BUILDER-DEFINED blocked SOAP step (TEST INFRASTRUCTURE ONLY).

The reference has no SOAP mathematics — only its planning cost
(proj/include/optishard/cost.hpp:47-48,68-75; SPEC.md:8 puts optimizer
internals out of scope), so parity is UNPINNED against the reference: this
file is the specification the GPU path (paper_2602_06079_b200/csrc/soap*.cu)
is checked against, written in plain numpy fp64 from the published algorithm
(Vyas et al. 2024, "SOAP: Improving and Stabilizing Shampoo using Adam",
Algorithm 3: Adam in the eigenbasis of Shampoo's preconditioner, the basis
refreshed every `precond_every` steps by one step of power iteration + QR).

Per 2-D tensor that is not vocabulary-space (SURVEY.md §8 A19 policy), the
tensor W is cut into blocks of at most `block` rows and columns (ragged last
blocks). Step order follows the published implementation (Vyas et al.,
github.com/nikhilvyas/SOAP, soap.py): the FIRST call only accumulates the
statistics and computes the initial basis (no parameter, momentum or second
moment update); every later call s = 1, 2, ... first takes the Adam step in
the current basis and then updates the statistics, refreshing the basis
every `precond_every` calls. For each block with gradient G (p x q):

    s == 0:
        L = (1 - bs) G G^T ;  R = (1 - bs) G^T G
        Q_L, Q_R <- refresh(L, I), refresh(R, I)   (init_iters iterations)
    s >= 1 (t = s):
        G' = Q_L^T G Q_R
        M  <- b1 M + (1 - b1) G                           (original space)
        V  <- b2 V + (1 - b2) G'^2                        (eigenbasis)
        N' = (Q_L^T M Q_R / (1 - b1^t)) / (sqrt(V / (1 - b2^t)) + eps)
        W  <- W - lr * Q_L N' Q_R^T
        L  <- bs L + (1 - bs) G G^T ;  R <- bs R + (1 - bs) G^T G   (fp32 state)
        if s % precond_every == 0:   Q_L, Q_R <- refresh (one iteration),
                                     V <- V[order_L, :][:, order_R]

refresh(S, Q), `iters` times:
    c = shift * ||S||_F           (c == 0: the basis is kept)
    Y = S Q + c Q                 est_j = (Q^T Y)_jj
    order = stable argsort of -est
    Q <- qr(Y[:, order])          (R with a positive diagonal)

The shift keeps the power iteration well defined when S is rank deficient
(non-square blocks, early steps): the columns of Q in S's null space stay
the previous basis, orthogonalised against the range, instead of whatever
rounding noise a QR of a singular matrix returns — this is what makes the
basis a deterministic function of the inputs on both the fp64 oracle and
the fp32 GPU path.

Elongated blocks (one side more than twice the other, e.g. 333 x 96): the
long side's statistics have rank <= the short side, so more than half of its
eigenbasis would be an arbitrary basis of the null space — a function of
rounding, not of the data. That side is not rotated (Q = I, order =
identity, never refreshed): one-sided SOAP on the short side, the Adam
second moment living in the half-rotated space.

Vectors and vocabulary-space matrices: elementwise Adam with the same b1,
b2, eps and bias correction (also skipped on the first call).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Tuple

import numpy as np


@dataclass
class SoapConfig:
    lr: float = 0.02
    beta1: float = 0.9
    beta2: float = 0.95
    shampoo_beta: float = 0.95
    eps: float = 1e-8
    block: int = 1024
    precond_every: int = 10
    init_iters: int = 4
    shift: float = 1e-3


def blocks(rows: int, cols: int, b: int) -> List[Tuple[int, int, int, int]]:
    """(r0, p, c0, q) of every block, row-major block order."""
    out = []
    for r0 in range(0, rows, b):
        for c0 in range(0, cols, b):
            out.append((r0, min(b, rows - r0), c0, min(b, cols - c0)))
    return out


def qr_pos(y: np.ndarray) -> np.ndarray:
    """Q of y = Q R with diag(R) >= 0 (the QR the GPU's CholeskyQR2 returns)."""
    q, r = np.linalg.qr(y)
    d = np.sign(np.diag(r))
    d[d == 0] = 1.0
    return q * d


def frozen(n: int, other: int) -> bool:
    """The side of size n of an n x other block keeps Q = I (elongated block)."""
    return n > 2 * other


def refresh_basis(s: np.ndarray, q: np.ndarray, cfg: SoapConfig, iters: int,
                  other: int = None) -> Tuple[np.ndarray, np.ndarray]:
    """One (or `iters`) shifted power-iteration steps; returns (Q, order of
    the LAST step) — the permutation V must follow. A frozen side (`other` =
    the block's other dimension) keeps its basis."""
    n = s.shape[0]
    order = np.arange(n)
    if other is not None and frozen(n, other):
        return q, order
    c = cfg.shift * float(np.linalg.norm(s))
    if c == 0.0:
        return q, order
    for _ in range(iters):
        y = s @ q + c * q
        est = np.einsum("ij,ij->j", q, y)
        order = np.argsort(-est, kind="stable")
        q = qr_pos(y[:, order])
    return q, order


class SoapTensorState:
    def __init__(self, shape, cfg: SoapConfig, preconditioned: bool):
        self.shape = tuple(shape)
        self.m = np.zeros(self.shape)
        self.v = np.zeros(self.shape)  # vectors / vocabulary matrices (elementwise Adam)
        self.pre = preconditioned
        self.blocks = blocks(self.shape[0], self.shape[1], cfg.block) if preconditioned else []
        self.L = [np.zeros((p, p)) for (_, p, _, q) in self.blocks]
        self.R = [np.zeros((q, q)) for (_, p, _, q) in self.blocks]
        self.QL = [np.eye(p) for (_, p, _, q) in self.blocks]
        self.QR = [np.eye(q) for (_, p, _, q) in self.blocks]
        self.V = [np.zeros((p, q)) for (_, p, _, q) in self.blocks]


def _bf16(x: np.ndarray) -> np.ndarray:
    """Round to the nearest bfloat16 (ties to even), returned as float64."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def soap_apply(st: SoapTensorState, cfg: SoapConfig, w: np.ndarray, g: np.ndarray,
               step: int, emulate_bf16: bool = False) -> float:
    """In place on w and the state; returns ||W_new - W_old||_F.

    emulate_bf16: round where the GPU path stores plain bf16 — the
    back-projection operands and intermediates (Q_L, Q_R, N', T3, N); the
    statistics and the projections G', M' run in bf16x3 there (fp32-level,
    treated as exact here). A precision model of the GPU, used to separate
    implementation errors from the rounding the fp64 comparison measures."""
    r = _bf16 if emulate_bf16 else (lambda x: x)
    g = np.asarray(g, dtype=np.float64).reshape(st.shape)
    bs = cfg.shampoo_beta
    if step == 0:  # statistics and the initial basis only
        for k, (r0, p, c0, q) in enumerate(st.blocks):
            gs = g[r0:r0 + p, c0:c0 + q]
            st.L[k] = (1.0 - bs) * (gs @ gs.T)
            st.R[k] = (1.0 - bs) * (gs.T @ gs)
            st.QL[k], _ = refresh_basis(st.L[k], st.QL[k], cfg, cfg.init_iters, q)
            st.QR[k], _ = refresh_basis(st.R[k], st.QR[k], cfg, cfg.init_iters, p)
        return 0.0
    t = step
    bc1, bc2 = 1.0 - cfg.beta1 ** t, 1.0 - cfg.beta2 ** t
    st.m = cfg.beta1 * st.m + (1.0 - cfg.beta1) * g
    if not st.pre:
        st.v = cfg.beta2 * st.v + (1.0 - cfg.beta2) * g * g
        upd = cfg.lr * (st.m / bc1) / (np.sqrt(st.v / bc2) + cfg.eps)
        w -= upd
        return float(np.linalg.norm(upd))
    upd = np.zeros(st.shape)
    for k, (r0, p, c0, q) in enumerate(st.blocks):
        gs = g[r0:r0 + p, c0:c0 + q]
        ql, qr = st.QL[k], st.QR[k]
        gp = ql.T @ gs @ qr
        st.V[k] = cfg.beta2 * st.V[k] + (1.0 - cfg.beta2) * gp * gp
        mp = ql.T @ st.m[r0:r0 + p, c0:c0 + q] @ qr
        n_rot = r((mp / bc1) / (np.sqrt(st.V[k] / bc2) + cfg.eps))
        upd[r0:r0 + p, c0:c0 + q] = cfg.lr * r(r(r(ql) @ n_rot) @ r(qr).T)
        st.L[k] = bs * st.L[k] + (1.0 - bs) * (gs @ gs.T)
        st.R[k] = bs * st.R[k] + (1.0 - bs) * (gs.T @ gs)
        if step % cfg.precond_every == 0:
            st.QL[k], ol = refresh_basis(st.L[k], st.QL[k], cfg, 1, q)
            st.QR[k], orr = refresh_basis(st.R[k], st.QR[k], cfg, 1, p)
            st.V[k] = st.V[k][ol, :][:, orr]
    w -= upd
    return float(np.linalg.norm(upd))


def is_preconditioned(p) -> bool:
    """SURVEY.md §8 A19 policy: 2-D, not vocabulary-space."""
    return len(p.shape) == 2 and not p.vocab_space


def run(params, cfg: SoapConfig, steps: int, seed: int, contributors: int = 1,
        init=None, grad=None) -> Tuple[Dict[int, np.ndarray], List[np.ndarray]]:
    """Replicated trajectory over `params` (planner ParamSpecs) with the
    reference generator's inputs (oracle.init_weight / reduced_gradient)."""
    from oracle import oracle as O
    init = init or (lambda p: O.init_weight(p.shape, p.id, seed).reshape(_shape2(p)))
    grad = grad or (lambda p, s: O.reduced_gradient(p.shape, p.id, seed, s, contributors)
                    .reshape(_shape2(p)))
    w = {p.id: init(p).astype(np.float64) for p in params}
    st = {p.id: SoapTensorState(_shape2(p), cfg, is_preconditioned(p)) for p in params}
    norms = []
    for s in range(steps):
        n = np.zeros(len(params))
        for p in params:
            n[p.id] = soap_apply(st[p.id], cfg, w[p.id], grad(p, s), s)
        norms.append(n)
    return w, norms


def _shape2(p):
    return tuple(p.shape) if len(p.shape) == 2 else (p.shape[0], 1)
