"""Numerics of the grouped tcgen05 Newton-Schulz GEMM (osh_ns_gemm) against a
plain PyTorch fp32 reference of the same contraction on the same bf16 inputs.

Tolerance: outputs are bf16 (8-bit mantissa), accumulation fp32, so the
max-abs error relative to the max-abs reference value must stay below 1e-2.
"""
import ctypes

import pytest

torch = pytest.importorskip("torch")

from paper_2602_06079_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu

A, B, C = 3.4445, -4.7750, 2.0315


@pytest.fixture(autouse=True, params=[2, 1], ids=["cta_pair", "cta1"])
def cta_group(request):
    """Every numerics test runs on both UMMA variants (cta_group::2 and ::1)."""
    L = _lib.lib()
    before = L.osh_gemm_cta_group()
    _lib.check(L.osh_set_gemm_cta_group(request.param))
    yield request.param
    _lib.check(L.osh_set_gemm_cta_group(before))


def mref(t, rows=None, cols=None, batch=None):
    """MatrixRef for a [batch][rows][ld] bf16 tensor (logical rows x cols)."""
    assert t.dtype == torch.bfloat16 and t.is_cuda and t.dim() == 3
    bt, r, ld = t.shape
    m = _lib.MatrixRef()
    m.ptr = t.data_ptr()
    m.batch = bt if batch is None else batch
    m.rows = r if rows is None else rows
    m.cols = ld if cols is None else cols
    m.ld = t.stride(1)
    m.bstride = t.stride(0)
    return m


def run(mode, probs, alpha=0.0, beta=0.0, lr=0.0):
    arr = (_lib.GemmProblem * len(probs))(*probs)
    _lib.check(_lib.lib().osh_ns_gemm(mode, arr, len(probs), alpha, beta, lr,
                                      torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()


def padded(batch, rows, cols, ld=None, scale=1.0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    ld = ld or cols
    t = torch.zeros(batch, rows, ld, device="cuda", dtype=torch.bfloat16)
    t[:, :, :cols] = (torch.randn(batch, rows, cols, device="cuda", generator=g) * scale).bfloat16()
    return t


def relerr(got, ref):
    return ((got.float() - ref.float()).abs().max() / ref.float().abs().max().clamp_min(1e-30)).item()


@pytest.mark.parametrize("batch,m,n,ld", [(1, 128, 256, 256), (2, 256, 768, 768), (3, 200, 300, 304),
                                          (1, 8, 24, 24), (2, 64, 12, 16), (1, 1024, 3072, 3072)])
def test_gram(batch, m, n, ld):
    x = padded(batch, m, n, ld, scale=0.05)
    out = torch.zeros(batch, m, m + (-m) % 8, device="cuda", dtype=torch.bfloat16)
    scale = torch.full((batch,), 0.5, device="cuda")
    p = _lib.GemmProblem()
    p.a = mref(x, cols=n)
    p.b = mref(x, cols=n)
    p.b_mn_major = 0
    p.out = mref(out, cols=m)
    p.scale = scale.data_ptr()
    run(0, [p])
    xf = x[:, :, :n].float()
    ref = 0.5 * xf @ xf.transpose(1, 2)
    assert relerr(out[:, :, :m], ref) < 1e-2


@pytest.mark.parametrize("batch,m", [(1, 128), (2, 512), (4, 100)])
def test_poly(batch, m):
    x = padded(batch, m, 2 * m, scale=0.05)
    a = (x.float() @ x.float().transpose(1, 2)).bfloat16()
    ld = m + (-m) % 8
    a_p = torch.zeros(batch, m, ld, device="cuda", dtype=torch.bfloat16)
    a_p[:, :, :m] = a
    out = torch.zeros_like(a_p)
    p = _lib.GemmProblem()
    p.a = mref(a_p, cols=m)
    p.b = mref(a_p, cols=m)
    p.out = mref(out, cols=m)
    p.aux = mref(a_p, cols=m)
    run(1, [p], alpha=B, beta=C)
    af = a.float()
    ref = B * af + C * af @ af
    assert relerr(out[:, :, :m], ref) < 1e-2


@pytest.mark.parametrize("batch,m,n", [(1, 128, 256), (2, 256, 1000), (3, 64, 4000), (1, 8, 24)])
def test_update_mn_major(batch, m, n):
    ld = n + (-n) % 8
    x = padded(batch, m, n, ld, scale=0.1)
    bm = padded(batch, m, m, m + (-m) % 8, scale=0.1, seed=1)
    out = torch.zeros_like(x)
    scale = torch.full((batch,), 0.25, device="cuda")
    p = _lib.GemmProblem()
    p.a = mref(bm, cols=m)
    p.b = mref(x, cols=n)        # K x N = m x n, N contiguous
    p.b_mn_major = 1
    p.out = mref(out, cols=n)
    p.aux = mref(x, cols=n)
    p.scale = scale.data_ptr()
    run(2, [p], alpha=A)
    xf = x[:, :, :n].float()
    ref = 0.25 * (A * xf + bm[:, :, :m].float() @ xf)
    assert relerr(out[:, :, :n], ref) < 1e-2


@pytest.mark.parametrize("transposed", [0, 1])
@pytest.mark.parametrize("batch,m,n,alpha", [(2, 128, 384, A), (1, 256, 512, 0.0), (3, 200, 328, 0.0),
                                             (1, 96, 1000, A), (1, 8, 24, 0.0)])
def test_final_weight_update(transposed, batch, m, n, alpha):
    """FINAL: W -= lr * (alpha X + B X) straight from the accumulator, W and
    the bf16 replica moved by TMA boxes in the tensor's stored orientation."""
    x = padded(batch, m, n, scale=0.1)
    bm = padded(batch, m, m, scale=0.1, seed=2)
    w0 = torch.randn(batch, m, n, device="cuda")
    if transposed:
        w = w0.transpose(1, 2).contiguous()   # tensor stored as [n][m]
    else:
        w = w0.clone()
    rep = torch.zeros(w.shape, device="cuda", dtype=torch.bfloat16)
    sq = torch.full((batch,), 0.5, device="cuda", dtype=torch.float64)  # accumulates (+=)
    tg = (_lib.FinalTarget * batch)()   # host array (osh.h)
    for i in range(batch):
        tg[i].w = w[i].data_ptr()
        tg[i].replica = rep[i].data_ptr()
        tg[i].sq_norm = sq[i:].data_ptr()
        tg[i].transposed = transposed
    p = _lib.GemmProblem()
    p.a = mref(bm)
    p.b = mref(x)
    p.b_mn_major = 1
    p.aux = mref(x)
    p.final_targets = ctypes.addressof(tg)
    lr = 0.02
    run(3, [p], alpha=alpha, lr=lr)
    upd = lr * (alpha * x.float() + bm.float() @ x.float())
    ref = w0 - upd
    got = w.transpose(1, 2) if transposed else w
    assert (got - ref).abs().max().item() < 1e-3 * upd.abs().max().item() + 1e-6
    assert torch.equal(rep, w.bfloat16())
    want_sq = 0.5 + (upd.double() ** 2).sum(dim=(1, 2))
    assert torch.allclose(sq, want_sq, rtol=1e-2)


def test_final_rejects_unaligned_pitch():
    """A row pitch TMA cannot address is refused (the engine then keeps the
    streaming update path for that wave)."""
    m, n = 8, 22
    x = padded(1, m, n, ld=24, scale=0.1)
    bm = padded(1, m, m, scale=0.1, seed=2)
    w = torch.zeros(1, m, n, device="cuda")
    tg = (_lib.FinalTarget * 1)()
    tg[0].w = w.data_ptr()
    p = _lib.GemmProblem()
    p.a = mref(bm)
    p.b = mref(x, cols=n)
    p.b_mn_major = 1
    p.aux = mref(x, cols=n)
    p.final_targets = ctypes.addressof(tg)
    arr = (_lib.GemmProblem * 1)(p)
    st = _lib.lib().osh_ns_gemm(3, arr, 1, 0.0, 0.0, 0.02, torch.cuda.current_stream().cuda_stream)
    assert st == 19  # OSH_ERR_ARG


def test_grouped_problems_one_launch():
    shapes = [(2, 128, 384), (5, 64, 192), (1, 256, 256)]
    xs, outs, ps = [], [], []
    for i, (bt, m, n) in enumerate(shapes):
        x = padded(bt, m, n, scale=0.05, seed=10 + i)
        out = torch.zeros(bt, m, m, device="cuda", dtype=torch.bfloat16)
        p = _lib.GemmProblem()
        p.a = mref(x)
        p.b = mref(x)
        p.out = mref(out)
        xs.append(x)
        outs.append(out)
        ps.append(p)
    run(0, ps)
    for x, out in zip(xs, outs):
        xf = x.float()
        assert relerr(out, xf @ xf.transpose(1, 2)) < 1e-2


@pytest.mark.parametrize("batch,m,n", [(2, 256, 768), (1, 1024, 3072), (3, 200, 300), (1, 8, 24),
                                       (2, 640, 128)])
def test_gram_symmetric_tiles(batch, m, n):
    """Upper-triangle tiles + mirrored epilogue == the full product, and the
    output is exactly symmetric (each element has a single writer)."""
    ld = n + (-n) % 8
    x = padded(batch, m, n, ld, scale=0.05, seed=3)
    ldm = m + (-m) % 8
    out = torch.full((batch, m, ldm), float("nan"), device="cuda", dtype=torch.bfloat16)
    p = _lib.GemmProblem()
    p.a = mref(x, cols=n)
    p.b = mref(x, cols=n)
    p.out = mref(out, cols=m)
    p.symmetric = 1
    run(0, [p])
    o = out[:, :, :m]
    assert not torch.isnan(o).any()
    assert torch.equal(o, o.transpose(1, 2))
    xf = x[:, :, :n].float()
    assert relerr(o, xf @ xf.transpose(1, 2)) < 1e-2


@pytest.mark.parametrize("batch,m", [(2, 512), (1, 4096), (3, 100)])
def test_poly_symmetric_tiles(batch, m):
    x = padded(batch, m, 2 * m, scale=0.05, seed=4)
    a = (x.float() @ x.float().transpose(1, 2)).bfloat16()
    a = ((a.float() + a.float().transpose(1, 2)) * 0.5).bfloat16()   # exactly symmetric input
    ld = m + (-m) % 8
    a_p = torch.zeros(batch, m, ld, device="cuda", dtype=torch.bfloat16)
    a_p[:, :, :m] = a
    out = torch.full_like(a_p, float("nan"))
    p = _lib.GemmProblem()
    p.a = mref(a_p, cols=m)
    p.b = mref(a_p, cols=m)
    p.out = mref(out, cols=m)
    p.aux = mref(a_p, cols=m)
    p.symmetric = 1
    run(1, [p], alpha=B, beta=C)
    o = out[:, :, :m]
    assert not torch.isnan(o).any() and torch.equal(o, o.transpose(1, 2))
    af = a.float()
    assert relerr(o, B * af + C * af @ af) < 1e-2


def mref32(t):
    """MatrixRef for a [batch][rows][ld] fp32 tensor (STAT output)."""
    assert t.dtype == torch.float32 and t.is_cuda and t.dim() == 3
    m = _lib.MatrixRef()
    m.ptr = t.data_ptr()
    m.batch, m.rows, m.cols = t.shape
    m.ld = t.stride(1)
    m.bstride = t.stride(0)
    return m


@pytest.mark.parametrize("alpha", [0.95, 0.0])
@pytest.mark.parametrize("sym", [1, 0, 2])
@pytest.mark.parametrize("batch,m,n", [(2, 256, 768), (1, 200, 328), (3, 512, 512)])
def test_stat_fp32_accumulate(batch, m, n, sym, alpha):
    """Shampoo statistics: L = beta2 * L + G G^T in fp32 (read-modify-write).
    sym = 2 (the engines' per-step statistics): the upper triangle only, the
    lower one left as it was, and bit-identical to the mirrored (sym = 1)
    result where written."""
    g = padded(batch, m, n, n + (-n) % 8, scale=0.3)
    l0 = torch.randn(batch, m, m, device="cuda")
    l0 = l0 + l0.transpose(1, 2)  # symmetric like a statistics matrix
    out = l0.clone()
    p = _lib.GemmProblem()
    p.a = mref(g, cols=n)
    p.b = mref(g, cols=n)
    p.out = mref32(out)
    p.symmetric = sym
    run(4, [p], alpha=alpha)
    gf = g[:, :, :n].float()
    ref = alpha * l0 + gf @ gf.transpose(1, 2)
    if sym == 2:
        up = torch.ones(m, m, device="cuda", dtype=torch.bool).triu()
        assert relerr(out[:, up], ref[:, up]) < 1e-5
        assert torch.equal(out[:, ~up], l0[:, ~up])  # lower triangle untouched
        full = l0.clone()
        p.out = mref32(full)
        p.symmetric = 1
        run(4, [p], alpha=alpha)
        assert torch.equal(out[:, up], full[:, up])
    else:
        assert relerr(out, ref) < 1e-5
    if sym == 1:
        assert torch.equal(out, out.transpose(1, 2))


def split4(x):
    """[hi | lo | hi | hi] bf16 layout of an fp32 [b][n][n] matrix."""
    hi = x.bfloat16()
    lo = (x - hi.float()).bfloat16()
    return torch.cat([hi, lo, hi, hi], dim=2).contiguous()


@pytest.mark.parametrize("sym", [1, 0])
@pytest.mark.parametrize("batch,n", [(2, 256), (1, 320), (3, 512)])
def test_split_bf16x3_product(batch, n, sym):
    """bf16x3 product of split operands: fp32-level accuracy (the Shampoo
    coupled-Newton iteration), output again in the split layout."""
    gen = torch.Generator(device="cuda").manual_seed(7)
    a = torch.randn(batch, n, n, device="cuda", generator=gen, dtype=torch.float64) / n ** 0.5
    a = (a + a.transpose(1, 2)) / 2
    b = a @ a + 0.1 * a  # commutes with a: a @ b is symmetric
    sa, sb = split4(a.float()), split4(b.float())
    out = torch.zeros(batch, n, 4 * n, device="cuda", dtype=torch.bfloat16)
    p = _lib.GemmProblem()
    p.a = mref(sa, cols=3 * n)                       # A view: columns [0, 3n) = (hi, lo, hi)
    bview = sb[:, :, n:]
    p.b = _lib.MatrixRef()
    p.b.ptr, p.b.batch, p.b.rows, p.b.cols = bview.data_ptr(), batch, n, 3 * n
    p.b.ld, p.b.bstride = sb.stride(1), sb.stride(0)  # B view: columns [n, 4n) = (lo, hi, hi)
    p.out = mref(out, cols=n)
    p.out_seg = n
    p.symmetric = sym
    run(5, [p])
    ref = a @ b
    got = out[:, :, :n].double() + out[:, :, n:2 * n].double()
    err = ((got - ref).abs().max() / ref.abs().max()).item()
    assert err < 5e-5, err  # bf16 alone would be ~4e-3
    assert torch.equal(out[:, :, :n], out[:, :, 2 * n:3 * n])
    assert torch.equal(out[:, :, :n], out[:, :, 3 * n:4 * n])


def test_poly_alpha_zero_skips_aux():
    x = padded(2, 256, 256, scale=0.1)
    out = torch.zeros_like(x)
    p = _lib.GemmProblem()
    p.a = mref(x)
    p.b = mref(x)
    p.out = mref(out)
    run(1, [p], alpha=0.0, beta=2.0)  # aux is null: must not be read
    xf = x.float()
    assert relerr(out, 2.0 * xf @ xf.transpose(1, 2)) < 1e-2


def test_poly_diagonal_add():
    """POLY's lr * I term (the Newton-Schulz 'a' folded into B)."""
    a = padded(2, 256, 256, scale=0.1)
    a = ((a.float() + a.float().transpose(1, 2)) / 2).bfloat16().contiguous()
    out = torch.zeros_like(a)
    for sym in (1, 0):
        p = _lib.GemmProblem()
        p.a = mref(a)
        p.b = mref(a)
        p.out = mref(out)
        p.aux = mref(a)
        p.symmetric = sym
        run(1, [p], alpha=B, beta=C, lr=A)
        af = a.float()
        ref = B * af + C * af @ af + A * torch.eye(256, device="cuda")
        assert relerr(out, ref) < 1e-2


@pytest.mark.parametrize("batch,m,n", [(2, 512, 768), (1, 1024, 3072), (3, 300, 328)])
def test_upper_tile_form_chain(batch, m, n, cta_group):
    """GRAM and POLY in the upper-tile form (symmetric = 3: no mirror of the
    off-diagonal tiles) feeding POLY / UPDATE that read the left-of-diagonal
    k-blocks from the mirrored tiles (a_upper / b_upper): the chain equals the
    fully mirrored chain bit for bit, and the torch fp32 reference within
    the bf16 tolerance. (1-CTA launches fall back to full matrices.)"""
    x = padded(batch, m, n, n + (-n) % 8, scale=0.02)

    ldm = m + (-m) % 8  # 16-byte row pitch (TMA)

    def chain(upper):
        a = torch.zeros(batch, m, ldm, device="cuda", dtype=torch.bfloat16)
        b = torch.zeros_like(a)
        xo = torch.zeros_like(x)
        g = _lib.GemmProblem()
        g.a = mref(x, cols=n)
        g.b = mref(x, cols=n)
        g.out = mref(a, cols=m)
        g.symmetric = 3 if upper else 1
        run(0, [g])
        p = _lib.GemmProblem()
        p.a = mref(a, cols=m)
        p.b = mref(a, cols=m)
        p.out = mref(b, cols=m)
        p.aux = mref(a, cols=m)
        p.symmetric = 3 if upper else 1
        p.a_upper = p.b_upper = int(upper)
        run(1, [p], alpha=B, beta=C, lr=A)
        u = _lib.GemmProblem()
        u.a = mref(b, cols=m)
        u.b = mref(x, cols=n)
        u.b_mn_major = 1
        u.out = mref(xo, cols=n)
        u.a_upper = int(upper)
        run(2, [u], alpha=0.0)
        return a, b, xo

    a1, b1, x1 = chain(False)
    a3, b3, x3 = chain(True)
    a1, b1, a3, b3 = (t[:, :, :m] for t in (a1, b1, a3, b3))
    up = torch.ones(m, m, device="cuda", dtype=torch.bool).triu()
    assert torch.equal(a3[:, up], a1[:, up]) and torch.equal(b3[:, up], b1[:, up])
    assert torch.equal(x3[:, :, :n], x1[:, :, :n])
    xf = x[:, :, :n].float()
    af = xf @ xf.transpose(1, 2)
    bf = A * torch.eye(m, device="cuda") + B * af + C * (af @ af)
    ref = bf @ xf
    assert relerr(x3[:, :, :n], ref) < 2e-2
