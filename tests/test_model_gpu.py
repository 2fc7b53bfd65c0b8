"""Single-GPU WeatherMixer parity: fused sm_100a forward/backward vs the reference (golden
vectors from running the reference, tests/golden) and vs the oracle at C2 scale."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

from conftest import rel_err

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden():
    z = np.load(os.path.join(GOLD, "wm_golden.npz"))
    meta = json.load(open(os.path.join(GOLD, "comm_golden.json")))
    return z, meta


def _model(cfg_dict, dtype):
    from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel
    cfg = ModelConfig.from_dict(cfg_dict)
    ctx = MpContext(Communicator.local(), [0])
    return WeatherMixerModel(ctx, cfg, seed=0, dtype=dtype)


@pytest.mark.parametrize("dtype,tol_out,tol_grad", [("f32", 1e-4, 1e-4), ("bf16", 2e-2, 2e-2)])
def test_forward_backward_vs_reference(cuda, dtype, tol_out, tol_grad):
    z, meta = _golden()
    m = _model(meta["config"], dtype)
    # init is the reference's, bit for bit in fp32
    from oracle import model as om
    cfg_o = om.Config(**{**meta["config"], "grid": tuple(meta["config"]["grid"]), "patch": tuple(meta["config"]["patch"])})
    ref_params = om.init_params(cfg_o, 0, np.float32)
    for name, arr in ref_params.items():
        assert np.array_equal(m.params[name].data.cpu().numpy(), arr), name
    m.zero_grads()
    out = m.forward(torch.tensor(z["x"], dtype=torch.float32))
    m.backward(torch.tensor(z["g_out"], dtype=torch.float32))
    m.grad_sync()
    torch.cuda.synchronize()
    e = rel_err(out.cpu().numpy(), z["out_f64"])
    assert e < tol_out, e
    worst = 0.0
    for name in meta["param_names"]:
        ge = rel_err(m.params[name].grad.cpu().numpy(), z["grad_f64/" + name])
        worst = max(worst, ge)
        assert ge < tol_grad, (name, ge)
    print(f"{dtype}: out {e:.2e} worst grad {worst:.2e}")


def test_rollout_vs_reference(cuda):
    z, meta = _golden()
    m = _model(meta["config"], "f32")
    m.zero_grads()
    out = m.forward(torch.tensor(z["x"][:1], dtype=torch.float32), r=2)
    m.backward(torch.tensor(z["g_out"][:1], dtype=torch.float32))
    assert rel_err(out.cpu().numpy(), z["rollout_out_f64"]) < 1e-4
    for name in meta["param_names"]:
        assert rel_err(m.params[name].grad.cpu().numpy(), z["rollout_grad_f64/" + name]) < 1e-4, name


def test_backward_without_forward_raises(cuda):
    z, meta = _golden()
    m = _model(meta["config"], "bf16")
    with pytest.raises(RuntimeError):
        m.backward(torch.zeros(1, 32, 64, 8))


@pytest.mark.parametrize("dtype,tol", [("f32", 1e-4), ("bf16", 2e-2)])
def test_c2_vs_oracle(cuda, dtype, tol):
    """C2 (5.625 deg, 69 -> 70 channels, 12 blocks) against the f64 oracle."""
    from oracle import model as om
    cfg = dict(n_vars=70, grid=(32, 64), patch=(2, 2), d_emb=512, d_tok=1024, d_ch=512, n_blocks=12)
    m = _model(cfg, dtype)
    oc = om.Config(**cfg)
    ref = om.SerialModel(oc, om.init_params(oc, 0, np.float64))
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1, 32, 64, 70))
    g = rng.standard_normal((1, 32, 64, 70))
    out_ref = ref.forward(x)
    grads_ref = ref.backward(g)
    m.zero_grads()
    out = m.forward(torch.tensor(x, dtype=torch.float32))
    m.backward(torch.tensor(g, dtype=torch.float32))
    torch.cuda.synchronize()
    e = rel_err(out.cpu().numpy(), out_ref)
    assert e < tol, e
    worst = max(rel_err(m.params[k].grad.cpu().numpy(), v) for k, v in grads_ref.items())
    print(f"C2 {dtype}: out {e:.2e} worst grad {worst:.2e}")
    assert worst < tol
