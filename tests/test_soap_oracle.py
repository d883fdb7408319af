"""fp64 SOAP specification (oracle/soap_oracle.py) — properties that pin it
without a reference implementation (the reference only costs SOAP,
cost.hpp:47-48,68-75):
  * the refreshed basis is orthogonal and, iterated, diagonalises S with a
    descending diagonal (power iteration + QR converges to the eigenbasis);
  * diagonal gradients give diagonal statistics, so the eigenbasis is a
    signed permutation and SOAP is exactly elementwise Adam;
  * the update is invariant to the sign of the basis columns;
  * zero gradients give zero updates (no NaN), and the shifted refresh keeps
    the basis when S = 0;
  * vectors / vocabulary matrices take elementwise Adam.
"""
import numpy as np

from oracle import soap_oracle as S


def adam_ref(gs, cfg):
    """Elementwise Adam over gs[1:] (the first call only initialises)."""
    m = np.zeros_like(gs[0])
    v = np.zeros_like(gs[0])
    out = [np.zeros_like(gs[0])]
    for t, g in enumerate(gs[1:], start=1):
        m = cfg.beta1 * m + (1 - cfg.beta1) * g
        v = cfg.beta2 * v + (1 - cfg.beta2) * g * g
        out.append(cfg.lr * (m / (1 - cfg.beta1 ** t)) / (np.sqrt(v / (1 - cfg.beta2 ** t)) + cfg.eps))
    return out


def test_refresh_orthogonal_and_converges():
    rng = np.random.default_rng(0)
    v, _ = np.linalg.qr(rng.standard_normal((48, 48)))
    s = (v * (0.8 ** np.arange(48))) @ v.T  # well separated spectrum
    cfg = S.SoapConfig()
    q, _ = S.refresh_basis(s, np.eye(48), cfg, 1)
    assert np.abs(q.T @ q - np.eye(48)).max() < 1e-12
    q, _ = S.refresh_basis(s, np.eye(48), cfg, 400)
    d = q.T @ s @ q
    # eigenvalues well above the shift (c = 1e-3 ||S||_F) converge fast; the
    # shifted tail converges at (l_i+1 + c)/(l_i + c) per iteration
    top = d[:16, :16]
    assert np.abs(top - np.diag(np.diag(top))).max() < 1e-9
    assert np.abs(d[:16, 16:]).max() < 1e-9
    w = np.linalg.eigvalsh(s)[::-1]
    np.testing.assert_allclose(np.diag(d)[:16], w[:16], rtol=1e-9)
    assert np.all(np.diff(np.diag(d)) <= 1e-12)


def test_diagonal_gradients_reduce_to_adam():
    cfg = S.SoapConfig(block=64, precond_every=3)
    rng = np.random.default_rng(1)
    gs = [np.diag(rng.standard_normal(32) * (1 + i)) for i in range(7)]
    st = S.SoapTensorState((32, 32), cfg, True)
    w = np.zeros((32, 32))
    ref = adam_ref(gs, cfg)
    for s, g in enumerate(gs):
        before = w.copy()
        S.soap_apply(st, cfg, w, g, s)
        np.testing.assert_allclose(before - w, ref[s], rtol=1e-7, atol=1e-8)


def test_sign_invariance_of_the_update():
    cfg = S.SoapConfig(block=64, precond_every=100)
    rng = np.random.default_rng(2)
    gs = [rng.standard_normal((24, 40)) for _ in range(3)]
    outs = []
    for flip in (False, True):
        st = S.SoapTensorState((24, 40), cfg, True)
        w = np.zeros((24, 40))
        for s, g in enumerate(gs):
            if s == 1 and flip:  # flip basis column signs after the first refresh
                st.QL[0] = st.QL[0] * np.where(np.arange(24) % 2, -1.0, 1.0)
                st.QR[0] = st.QR[0] * np.where(np.arange(40) % 3, 1.0, -1.0)
            S.soap_apply(st, cfg, w, g, s)
        outs.append(w)
    np.testing.assert_allclose(outs[0], outs[1], rtol=1e-10, atol=1e-13)


def test_zero_gradient_and_zero_statistics():
    cfg = S.SoapConfig(block=64)
    st = S.SoapTensorState((16, 24), cfg, True)
    w = np.ones((16, 24))
    for s in range(3):
        assert S.soap_apply(st, cfg, w, np.zeros((16, 24)), s) == 0.0
    assert np.all(w == 1.0)
    assert np.array_equal(st.QL[0], np.eye(16)) and np.array_equal(st.QR[0], np.eye(24))


def test_vectors_take_adam():
    cfg = S.SoapConfig()
    rng = np.random.default_rng(3)
    gs = [rng.standard_normal((50, 1)) for _ in range(4)]
    st = S.SoapTensorState((50, 1), cfg, False)
    w = np.zeros((50, 1))
    ref = adam_ref(gs, cfg)
    for s, g in enumerate(gs):
        before = w.copy()
        S.soap_apply(st, cfg, w, g, s)
        np.testing.assert_allclose(before - w, ref[s], rtol=1e-12)


def test_first_call_initialises_only():
    cfg = S.SoapConfig(block=64)
    rng = np.random.default_rng(5)
    st = S.SoapTensorState((40, 24), cfg, True)
    w = np.ones((40, 24))
    assert S.soap_apply(st, cfg, w, rng.standard_normal((40, 24)), 0) == 0.0
    assert np.all(w == 1.0) and np.all(st.m == 0.0) and np.all(st.V[0] == 0.0)
    assert np.abs(st.QL[0].T @ st.QL[0] - np.eye(40)).max() < 1e-12
    assert not np.allclose(st.QL[0], np.eye(40))


def test_ragged_blocks_cover_the_tensor():
    cfg = S.SoapConfig(block=64, precond_every=2)
    rng = np.random.default_rng(4)
    st = S.SoapTensorState((130, 70), cfg, True)
    assert [b[1] for b in st.blocks] == [64, 64, 64, 64, 2, 2]
    w = np.zeros((130, 70))
    for s in range(4):
        S.soap_apply(st, cfg, w, rng.standard_normal((130, 70)), s)
    assert np.all(np.isfinite(w)) and np.all(w != 0.0)


def test_bf16_rounding_matches_torch():
    """The precision model's bf16 rounding (oracle.soap_oracle._bf16) is
    round-to-nearest-even, as the GPU's __float2bfloat16_rn."""
    torch = __import__("pytest").importorskip("torch")
    rng = np.random.default_rng(6)
    x = np.concatenate([rng.standard_normal(10000) * 10.0 ** rng.integers(-8, 8, 10000),
                        [0.0, -0.0, 1.0, 1.00390625, 1.01171875, -3.5]])
    ref = torch.from_numpy(x.astype(np.float32)).bfloat16().double().numpy()
    np.testing.assert_array_equal(S._bf16(x), ref)


def test_elongated_block_rotates_only_its_short_side():
    """A p x q block with p > 2q keeps Q_L = I (its statistics have rank <= q:
    most of that basis would be rounding noise); Q_R is refreshed."""
    cfg = S.SoapConfig(block=512, precond_every=1)
    st = S.SoapTensorState((300, 60), cfg, True)
    w = np.zeros((300, 60))
    g = np.random.default_rng(3).standard_normal((300, 60))
    for step in range(3):
        S.soap_apply(st, cfg, w, g, step)
    assert np.array_equal(st.QL[0], np.eye(300))
    assert not np.allclose(st.QR[0], np.eye(60))
    assert S.frozen(300, 60) and not S.frozen(60, 300) and not S.frozen(200, 100)
