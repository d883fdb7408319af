"""The builder-defined Shampoo specification (oracle/shampoo_oracle.py) on CPU.

The reference has no Shampoo mathematics (cost model only, cost.hpp:47-48,
68-75), so these tests pin the specification itself: the coupled-Newton
inverse 4th root converges to the eigendecomposition root, blocks tile the
tensor exactly, grafting preserves the gradient norm per block, the zero
gradient is a fixed point, and the planner's Shampoo cost matches the formula
the reference uses (test_cost.cpp:91-101 values are pinned in test_planner_golden).
"""
import numpy as np

from oracle import shampoo_oracle as S


def test_blocks_tile_the_tensor():
    for rows, cols, b in [(512, 768, 256), (333, 96, 256), (4096, 12288, 1024), (64, 64, 1024)]:
        cover = np.zeros((rows, cols), dtype=int)
        for r0, p, c0, q in S.blocks(rows, cols, b):
            assert 0 < p <= b and 0 < q <= b
            cover[r0:r0 + p, c0:c0 + q] += 1
        assert (cover == 1).all()


def test_newton_root_matches_eigh():
    rng = np.random.default_rng(1)
    for p, q in [(64, 192), (128, 128), (96, 40)]:
        g = rng.standard_normal((p, q))
        for s in (g @ g.T, g.T @ g):
            c = np.linalg.norm(s)
            a = s / c + 1e-4 * np.eye(s.shape[0])
            x = S.inv_root4(a, 16)
            e = S.inv_root4_exact(a)
            assert np.linalg.norm(x - e) / np.linalg.norm(e) < 1e-10


def test_graft_keeps_block_gradient_norm():
    cfg = S.ShampooConfig(lr=1.0, beta1=0.0, block=64, precond_every=1)
    st = S.ShampooTensorState((128, 96), cfg, True)
    rng = np.random.default_rng(2)
    g = rng.standard_normal((128, 96))
    w = np.zeros((128, 96))
    S.shampoo_apply(st, cfg, w, g, 0)
    for r0, p, c0, q in st.blocks:  # beta1 = 0, lr = 1: -w is the grafted update
        u = -w[r0:r0 + p, c0:c0 + q]
        assert abs(np.linalg.norm(u) - np.linalg.norm(g[r0:r0 + p, c0:c0 + q])) < 1e-9 * np.linalg.norm(u)


def test_zero_gradient_is_a_fixed_point():
    cfg = S.ShampooConfig(block=64)
    st = S.ShampooTensorState((64, 128), cfg, True)
    w = np.ones((64, 128))
    n = S.shampoo_apply(st, cfg, w, np.zeros((64, 128)), 0)
    assert n == 0.0 and (w == 1.0).all()
    for pl in st.PL:
        assert np.array_equal(pl, np.eye(pl.shape[0]))


def test_vectors_use_momentum_sgd():
    cfg = S.ShampooConfig()
    st = S.ShampooTensorState((10, 1), cfg, False)
    w = np.zeros((10, 1))
    g = np.arange(10.0).reshape(10, 1)
    S.shampoo_apply(st, cfg, w, g, 0)
    S.shampoo_apply(st, cfg, w, g, 1)
    assert np.allclose(w, -cfg.lr * (g + (cfg.beta1 * g + g)))
