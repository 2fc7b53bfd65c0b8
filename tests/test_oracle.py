"""Pin the oracle (CPU restatement) to the reference: known-answer tests copied in spirit from
reference pkg/tests/test_tensor.py and golden vectors produced by running the reference itself
(tests/golden/make_golden.py). CPU only."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from conftest import rel_err
from oracle import model as om
from oracle import ops, train, volume

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def golden():
    z = np.load(os.path.join(GOLD, "wm_golden.npz"))
    meta = json.load(open(os.path.join(GOLD, "comm_golden.json")))
    return z, meta


def gcfg(meta):
    c = dict(meta["config"])
    c["grid"], c["patch"] = tuple(c["grid"]), tuple(c["patch"])
    return om.Config(**c)


# ----------------------------------------------------------------- tensor.py known answers
def test_matmul_fixed_nt_example():
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[5.0, 6.0], [7.0, 8.0]])
    assert ops.matmul(a, b, "NT").tolist() == [[17.0, 23.0], [39.0, 53.0]]  # test_tensor.py:23-28


def test_matmul_modes_vs_loops(rng):
    a, b = rng.standard_normal((5, 4)), rng.standard_normal((4, 3))
    ref = np.array([[sum(a[i, k] * b[k, j] for k in range(4)) for j in range(3)] for i in range(5)])
    assert rel_err(ops.matmul(a, b, "NN"), ref) < 1e-12
    assert rel_err(ops.matmul(a, b.T.copy(), "NT"), ref) < 1e-12
    assert rel_err(ops.matmul(a.T.copy(), b, "TN"), ref) < 1e-12
    with pytest.raises(ops.OracleShapeError):
        ops.matmul(a, b, "NT")


def test_gelu_values():
    assert ops.gelu(np.array(0.0)) == 0.0
    assert abs(ops.gelu(np.array(1.0)) - 0.841345) < 1e-6  # test_tensor.py:73-81
    assert abs(ops.gelu(np.array(10.0)) - 10.0) < 1e-6


def test_gelu_backward_fd(rng):
    x = rng.standard_normal(20)
    h = 1e-6
    fd = (ops.gelu(x + h) - ops.gelu(x - h)) / (2 * h)
    assert np.max(np.abs(ops.gelu_backward(x, np.ones_like(x)) - fd)) < 1e-6


def test_layer_norm_closed_forms():
    g, b = np.ones(4), np.zeros(4)
    assert np.allclose(ops.layer_norm(np.full((1, 4), 3.0), g, b), 0.0)
    y = ops.layer_norm(np.array([[1.0, 3.0]]), np.ones(2), np.zeros(2), eps=1e-12)
    assert np.allclose(y, [[-1.0, 1.0]], atol=1e-6)
    with pytest.raises(ValueError):
        ops.layer_norm(np.ones((1, 2)), np.ones(2), np.zeros(2), eps=0)


def test_layer_norm_backward_fd(rng):
    x, gam, up = rng.standard_normal((3, 6)), rng.standard_normal(6), rng.standard_normal((3, 6))
    dx, dg, db = ops.layer_norm_backward(x, gam, 1e-5, up)
    h = 1e-6
    f = lambda xx: float((ops.layer_norm(xx, gam, np.zeros(6)) * up).sum())  # noqa: E731
    num = np.zeros_like(x)
    for i in np.ndindex(x.shape):
        e = np.zeros_like(x)
        e[i] = h
        num[i] = (f(x + e) - f(x - e)) / (2 * h)
    assert np.max(np.abs(num - dx)) < 1e-5
    assert np.allclose(db, up.sum(0))


def test_patchify_identities(rng):
    x = rng.standard_normal((2, 8, 12, 3))
    t = ops.patchify(x, 4, 4)
    assert t.shape == (2, 6, 48)
    assert np.array_equal(ops.unpatchify(t, 8, 12, 4, 4), x)
    # unit patches keep row-major token order (test_tensor.py:157-160)
    assert np.array_equal(ops.patchify(x, 1, 1)[0, :, 0], x[0, :, :, 0].reshape(-1))
    with pytest.raises(ops.OracleShapeError):
        ops.patchify(x, 3, 5)


# ----------------------------------------------------------------- model golden (reference run)
def test_init_bit_exact(golden):
    _, meta = golden
    cfg = gcfg(meta)
    assert om.params_digest(om.init_params(cfg, 0, np.float64)) == meta["init_digest_f64"]
    assert om.params_digest(om.init_params(cfg, 0, np.float32)) == meta["init_digest_f32"]
    assert list(om.init_params(cfg, 0)) == meta["param_names"]


def test_serial_model_matches_reference_f64(golden):
    z, meta = golden
    cfg = gcfg(meta)
    m = om.SerialModel(cfg, om.init_params(cfg, 0, np.float64))
    out = m.forward(z["x"])
    assert rel_err(out, z["out_f64"]) < 1e-12
    grads = m.backward(z["g_out"])
    for name in meta["param_names"]:
        ref = z["grad_f64/" + name]
        assert rel_err(grads[name], ref) < 1e-12, name


def test_serial_model_rollout_matches_reference(golden):
    z, meta = golden
    cfg = gcfg(meta)
    m = om.SerialModel(cfg, om.init_params(cfg, 0, np.float64))
    out = m.forward(z["x"][:1], r=2)
    assert rel_err(out, z["rollout_out_f64"]) < 1e-12
    grads = m.backward(z["g_out"][:1])
    for name in meta["param_names"]:
        assert rel_err(grads[name], z["rollout_grad_f64/" + name]) < 1e-12, name


def test_serial_model_f32_close_to_reference_f32(golden):
    z, meta = golden
    cfg = gcfg(meta)
    m = om.SerialModel(cfg, om.init_params(cfg, 0, np.float32))
    out = m.forward(z["x"].astype(np.float32))
    assert rel_err(out, z["out_f32"]) < 1e-5
    grads = m.backward(z["g_out"].astype(np.float32))
    for name in meta["param_names"]:
        assert rel_err(grads[name], z["grad_f32/" + name]) < 1e-4, name


def test_local_layouts_match_reference_tiles(golden):
    """local_sample on the R x C grid reproduces the reference n=2 / n=4 per-rank blocks."""
    z, meta = golden
    cfg = gcfg(meta)
    for pos in range(2):
        assert rel_err(om.local_sample(cfg, z["out_f64"], 1, 2, 0, pos), z[f"n2_out_local/{pos}"]) < 1e-12
    for pos in range(4):
        assert rel_err(om.local_sample(cfg, z["out_f64"], 2, 2, pos // 2, pos % 2), z[f"n4_out_local/{pos}"]) < 1e-12


def test_flops_formula(golden):
    _, meta = golden
    cfg = gcfg(meta)
    assert om.train_flops(cfg, meta["batch"]) == meta["flops_n1"] == meta["flops_n4"]


def test_comm_volume_tables(golden):
    _, meta = golden
    cfg = gcfg(meta)
    for key, val in meta["primitive_send_elements"].items():
        mode, n, a_s, b_s = key.split("/")
        if isinstance(val, str):
            continue
        assert volume.primitive_send_elements(mode, int(n), eval(a_s), eval(b_s)) == val, key
    for key, (fwd, bwd) in meta["comm_volume"].items():
        mode, n, dims = key.split("/")
        m, k, no, b = dims.split(",")
        f, bk = volume.comm_volume(int(m), int(k), int(no), int(n), mode, batch=int(b[1:]))
        assert (f, bk) == (fwd, bwd), key
    for key, val in meta["step_comm_volume"].items():
        n, b, r = (int(s[1:]) for s in key.split("_"))
        got = volume.step_comm_volume(cfg, n, b, r, volume.dup_elements_per_rank(cfg, n))
        assert got == val, key


# ----------------------------------------------------------------- SPEC worked examples (loss, Adam)
def test_lat_weights_spec_example():
    w = train.lat_weights(3)
    assert np.allclose(w, [0.5 / (2 / 3), 1.0 / (2 / 3), 0.5 / (2 / 3)])
    pred = np.zeros((1, 3, 1, 1))
    target = np.zeros_like(pred)
    target[0, 1] = 1.0
    rmse = train.lat_weighted_rmse(pred, target, w)
    assert abs(rmse[0] - np.sqrt(1.5 / 3)) < 1e-12
    assert abs(train.lat_weights(721).mean() - 1.0) < 1e-12


def test_weighted_mse_spec_examples(rng):
    pred, target = rng.standard_normal((2, 4, 5, 3)), rng.standard_normal((2, 4, 5, 3))
    loss, g = train.weighted_mse_loss(pred, target, np.ones(4), np.ones(3))
    assert abs(loss - np.mean((pred - target) ** 2)) < 1e-12
    pw = np.array(train.PRESSURE_WEIGHTS)
    e50 = np.zeros((1, 1, 1, 13))
    e50[..., -1] = 1.0
    e1000 = np.zeros((1, 1, 1, 13))
    e1000[..., 0] = 1.0
    l50, _ = train.weighted_mse_loss(e50, np.zeros_like(e50), np.ones(1), pw)
    l1000, _ = train.weighted_mse_loss(e1000, np.zeros_like(e1000), np.ones(1), pw)
    assert abs(l50 / l1000 - 0.3) < 1e-12


def test_adam_spec_examples():
    p, m, v = np.array([1.0, -2.0]), np.zeros(2), np.zeros(2)
    train.adam_step(p, np.zeros(2), m, v, 1, 0.1)
    assert np.array_equal(p, [1.0, -2.0])  # zero grad -> unchanged
    p, m, v = np.array([1.0, -2.0]), np.zeros(2), np.zeros(2)
    train.adam_step(p, np.array([0.3, -5.0]), m, v, 1, 0.01)
    assert np.allclose(p, [1.0 - 0.01, -2.0 + 0.01], atol=1e-7)  # step 1 ~ -lr sign(g)
    x, m, v = np.array([1.0]), np.zeros(1), np.zeros(1)
    for t in range(1, 101):
        train.adam_step(x, 2 * x, m, v, t, 0.1)
    assert abs(x[0]) < 0.1
    clipped, _ = train.clip_grads([np.array([3.0, 4.0])], 1.0)
    assert np.allclose(clipped[0], [0.6, 0.8])
