"""L0 operator parity on the GPU (reference tensor.py API) against the oracle restatement."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import ops

pytestmark = pytest.mark.gpu


def test_gelu_values_and_backward(cuda, rng):
    from paper_2507_05753_b200 import tensor as T
    x = torch.tensor([0.0, 1.0, 10.0, -3.0], device=cuda)
    y = T.gelu(x).cpu().numpy()
    assert y[0] == 0.0 and abs(y[1] - 0.841345) < 1e-6 and abs(y[2] - 10.0) < 1e-6  # test_tensor.py:73-81
    xs = rng.standard_normal((37, 53))
    up = rng.standard_normal((37, 53))
    got = T.gelu_backward(torch.tensor(xs, dtype=torch.float32, device=cuda),
                          torch.tensor(up, dtype=torch.float32, device=cuda)).cpu().numpy()
    assert rel_err(got, ops.gelu_backward(xs, up)) < 1e-5


def test_layer_norm_and_backward(cuda, rng):
    from paper_2507_05753_b200 import tensor as T
    x = rng.standard_normal((3, 40, 72)) * 2 + 0.5
    gam, bet, up = rng.standard_normal(72), rng.standard_normal(72), rng.standard_normal((3, 40, 72))
    f = lambda a: torch.tensor(a, dtype=torch.float32, device=cuda)  # noqa: E731
    assert rel_err(T.layer_norm(f(x), f(gam), f(bet)).cpu().numpy(), ops.layer_norm(x, gam, bet)) < 1e-5
    dx, dg, db = T.layer_norm_backward(f(x), f(gam), 1e-5, f(up))
    rdx, rdg, rdb = ops.layer_norm_backward(x, gam, 1e-5, up)
    assert rel_err(dx.cpu().numpy(), rdx) < 1e-4
    assert rel_err(dg.cpu().numpy(), rdg) < 1e-5 and rel_err(db.cpu().numpy(), rdb) < 1e-5
    two = T.layer_norm(f(np.array([[1.0, 3.0, 1.0, 3.0]])), f(np.ones(4)), f(np.zeros(4)), eps=1e-12)
    assert np.allclose(two.cpu().numpy(), [[-1, 1, -1, 1]], atol=1e-5)  # test_tensor.py:99-104
    with pytest.raises(ValueError):
        T.layer_norm(f(x), f(gam), f(bet), eps=0.0)


@pytest.mark.parametrize("shape,patch", [((2, 32, 64, 8), (4, 4)), ((1, 16, 24, 70), (8, 8)), ((1, 8, 12, 3), (2, 3))])
def test_patchify_round_trip(cuda, rng, shape, patch):
    from paper_2507_05753_b200 import tensor as T
    from paper_2507_05753_b200.errors import ShapeError
    x = rng.standard_normal(shape)
    t = T.patchify(torch.tensor(x, dtype=torch.float32, device=cuda), *patch)
    assert np.array_equal(t.cpu().numpy(), ops.patchify(x.astype(np.float32), *patch))
    back = T.unpatchify(t, shape[1], shape[2], *patch)
    assert np.array_equal(back.cpu().numpy(), x.astype(np.float32))
    with pytest.raises(ShapeError):
        T.patchify(torch.zeros((1, 5, 8, 2), device=cuda), 2, 2)


def test_matmul_dtype_mismatch_raises(cuda):
    from paper_2507_05753_b200 import tensor as T
    from paper_2507_05753_b200.errors import ShapeError
    with pytest.raises(ShapeError, match="dtype mismatch"):
        T.matmul(torch.zeros(4, 4, device=cuda), torch.zeros(4, 4, device=cuda, dtype=torch.bfloat16))
    with pytest.raises(ShapeError, match="incompatible"):
        T.matmul(torch.zeros(4, 3, device=cuda), torch.zeros(4, 3, device=cuda), "NN")


@pytest.mark.parametrize("shape,patch,gdt", [((2, 16, 32, 8), (4, 4), torch.float32), ((1, 16, 24, 70), (8, 8), torch.bfloat16),
                                             ((1, 8, 12, 35), (2, 2), torch.bfloat16), ((1, 8, 12, 3), (2, 3), torch.float32),
                                             ((1, 16, 16, 5), (8, 8), torch.float32)])
def test_blend_loss_kernel(cuda, rng, shape, patch, gdt):
    """jg_blend_loss (unpatchify + blend + lat-weighted MSE + dL/d(dec tokens) + blend-weight
    gradient) against a float64 torch restatement of the same formulas; vector (pw 2/4/8) and
    scalar (pw 3) token paths, fp32 and bf16 gradient tokens, target and external-gradient forms."""
    from paper_2507_05753_b200 import kernels as K
    from paper_2507_05753_b200 import tensor as T
    B, lat, lon, C = shape
    pl, pw = patch
    f = lambda a: torch.tensor(a, dtype=torch.float32, device=cuda)  # noqa: E731
    x, tgt = rng.standard_normal(shape), rng.standard_normal(shape)
    dec_g = rng.standard_normal(shape)
    w, latw, varw = rng.random(C), rng.random(lat), rng.random(C)
    dec_tok = T.patchify(f(dec_g), pl, pw)
    inv, ls = 1.0 / x.size, 3.0
    # float64 restatement
    out = w * dec_g + (1 - w) * x
    wt = latw[None, :, None, None] * varw[None, None, None, :]
    er = out - tgt
    loss = (wt * er * er).sum() * inv
    g = 2 * wt * er * inv * ls
    gblend = (g * (dec_g - x)).sum(axis=(0, 1, 2))
    gdec = ops.patchify((g * w).astype(np.float32), pl, pw)
    for mode in ("target", "ext"):
        lossd, gb = torch.zeros(1, device=cuda), torch.zeros(C, device=cuda)
        gd = torch.zeros(dec_tok.shape, dtype=gdt, device=cuda)
        o = torch.zeros(shape, device=cuda)
        K.blend_loss(dec_tok, f(x), f(tgt) if mode == "target" else None, f(w), f(latw), f(varw),
                     f(g) if mode == "ext" else None, o, lossd, gb, gd, B, lat, lon, C, pl, pw, inv, ls)
        tol = 1e-5 if gdt == torch.float32 else 8e-3
        assert rel_err(o.cpu().numpy(), out) < 1e-6
        assert rel_err(gd.float().cpu().numpy(), gdec) < tol
        assert rel_err(gb.cpu().numpy(), gblend) < 1e-4
        if mode == "target":
            assert abs(lossd.item() - loss) / loss < 1e-5


@pytest.mark.parametrize("rows,cols,ld,dt", [(8190, 2160, 2160, torch.bfloat16), (300, 72, 80, torch.float32),
                                             (77, 13, 13, torch.float32), (1000, 264, 264, torch.float32)])
def test_colsum_rowsum_kernels(cuda, rows, cols, ld, dt):
    """Bias-gradient reductions (reference _sum_except, parallel.py:552-561): column and row sums
    accumulate into fp32 outputs; vector (16-byte) and scalar paths, padded leading dimension."""
    from paper_2507_05753_b200 import kernels as K
    g = torch.Generator(device=cuda).manual_seed(5)
    x = torch.randn(rows, ld, device=cuda, generator=g).to(dt)
    ref = x[:, :cols].double()
    cs = torch.ones(cols, device=cuda)
    K.colsum(x, cs, rows, cols, ld=ld)
    assert rel_err(cs.cpu().numpy(), (ref.sum(0) + 1).cpu().numpy()) < 1e-5
    rs = torch.ones(rows, device=cuda)
    K.rowsum(x, rs, rows, cols, ld=ld)
    assert rel_err(rs.cpu().numpy(), (ref.sum(1) + 1).cpu().numpy()) < 1e-5


def test_epilogue_and_ln_kernels_tile_shapes(cuda):
    """Jigsaw epilogue (planes summed + row bias + residual + LN moments; col bias + GELU) and the
    layer-norm phases at 2x2-tile-like shapes with ragged column chunks, against fp64 torch."""
    from paper_2507_05753_b200 import kernels as K, _lib
    g = torch.Generator(device=cuda).manual_seed(7)
    M, N = 515, 1080  # 1080 = 4 full 256-column chunks + a partial one
    planes = torch.randn(2, M, N, device=cuda, generator=g).to(torch.bfloat16)
    bias, resid = torch.randn(M, device=cuda, generator=g), torch.randn(M, N, device=cuda, generator=g)
    d, st = torch.empty(M, N, device=cuda), torch.zeros(M, 2, device=cuda)
    K.epilogue(planes, M, N, acc_bs=M * N, nplanes=2, epi=_lib.EPI_BIAS_ROW | _lib.EPI_RESID | _lib.EPI_STATS,
               bias=bias, resid=resid, d=d, stats=st)
    ref = planes.double().sum(0) + bias.double()[:, None] + resid.double()
    assert rel_err(d.cpu().numpy(), ref.cpu().numpy()) < 1e-6
    assert rel_err(st[:, 0].cpu().numpy(), ref.sum(1).cpu().numpy()) < 1e-5
    assert rel_err(st[:, 1].cpu().numpy(), (ref * ref).sum(1).cpu().numpy()) < 1e-5
    cb = torch.randn(N, device=cuda, generator=g)
    h, a = torch.empty(M, N, device=cuda), torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    K.epilogue(planes, M, N, acc_bs=M * N, nplanes=2, epi=_lib.EPI_BIAS_COL | _lib.EPI_GELU_FWD, bias=cb, d=h, d2=a)
    hr = planes.double().sum(0) + cb.double()
    assert rel_err(h.cpu().numpy(), hr.cpu().numpy()) < 1e-6
    assert rel_err(a.double().cpu().numpy(), torch.nn.functional.gelu(hr).cpu().numpy()) < 8e-3
    # layer norm over the split axis: moments from the epilogue, apply, backward phases
    gam, bet = torch.randn(N, device=cuda, generator=g), torch.randn(N, device=cuda, generator=g)
    u, mr = torch.empty(M, N, device=cuda), torch.empty(M, 2, device=cuda)
    K.ln_apply(d, st, gam, bet, u, mr, M, N, N, 1e-5)
    mean = ref.mean(1, keepdim=True)
    xh = (ref - mean) / torch.sqrt(ref.var(1, unbiased=False, keepdim=True) + 1e-5)
    assert rel_err(u.cpu().numpy(), (xh * gam.double() + bet.double()).cpu().numpy()) < 1e-4
    gin = torch.randn(M, N, device=cuda, generator=g)
    bst = torch.zeros(M, 2, device=cuda)
    K.ln_bwd_moments(d, gin, gam, mr, bst, M, N)
    hh = gin.double() * gam.double()
    assert rel_err(bst[:, 0].cpu().numpy(), hh.sum(1).cpu().numpy()) < 1e-5
    out, dg, db = torch.empty(M, N, device=cuda), torch.zeros(N, device=cuda), torch.zeros(N, device=cuda)
    K.ln_bwd_apply(d, gin, gam, mr, bst, resid, out, None, dg, db, M, N, N)
    rstd = 1 / torch.sqrt(ref.var(1, unbiased=False, keepdim=True) + 1e-5)
    dx = rstd * (hh - hh.mean(1, keepdim=True) - xh * (hh * xh).mean(1, keepdim=True)) + resid.double()
    assert rel_err(out.cpu().numpy(), dx.cpu().numpy()) < 1e-4
    assert rel_err(dg.cpu().numpy(), (gin.double() * xh).sum(0).cpu().numpy()) < 1e-4
    assert rel_err(db.cpu().numpy(), gin.double().sum(0).cpu().numpy()) < 1e-5


@pytest.mark.parametrize("rows,cols,period", [(130, 1030, 65), (600, 2160, 300), (16380, 4320, 16380)])
def test_ln_bwd_apply_fused_bias_sums(cuda, rows, cols, period):
    """Layer-norm backward with the fused bias-gradient sums (row sums folded by r % period for
    the tok2 row bias, column sums for ch2 / encoder): same results as the exact torch double."""
    import cpu_kernels as CK
    from paper_2507_05753_b200 import kernels as K
    g = torch.Generator(device=cuda).manual_seed(rows + cols)
    r = lambda *s: torch.randn(*s, device=cuda, generator=g)  # noqa: E731
    x, gin, resid, gam = r(rows, cols), r(rows, cols), r(rows, cols), r(cols)
    mr = torch.stack([x.mean(1), 1 / torch.sqrt(x.var(1, unbiased=False) + 1e-5)], 1).contiguous()
    bst = r(rows, 2)
    outs = []
    for impl in (K, CK):
        out = torch.empty(rows, cols, device=cuda)
        dg, db = torch.zeros(cols, device=cuda), torch.zeros(cols, device=cuda)
        rs, cs = torch.full((period,), 0.5, device=cuda), torch.zeros(cols, device=cuda)
        impl.ln_bwd_apply(x, gin, gam, mr, bst, resid, out, None, dg, db, rows, cols, cols,
                          rowsum=rs, rowsum_period=period, colsum=cs)
        outs.append((out, dg, db, rs, cs))
    for a, b in zip(*outs):
        assert rel_err(a.double().cpu().numpy(), b.double().cpu().numpy()) < 1e-4
