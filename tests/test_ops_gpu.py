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
