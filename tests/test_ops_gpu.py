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
