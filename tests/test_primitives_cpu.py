"""Collective primitives pnt / pnn / ptn and the reference layer API (ShardedLinear,
ShardedLayerNorm, MixerBlock) over gloo worlds of 1 / 2 / 4 / 8 processes, with the kernel
layer replaced by the exact tests/cpu_kernels.py double.

Known answers are SPEC.md's (:210 2-way NT, :219 4-way blocks, :228-229 backward, :235 TN
identity, :244 comm count); layouts are the reference's for n = 2 (column blocks) and n = 4
(2 x 2 blocks, rank r owns block (r // 2, r % 2), parallel.py:1-10), and the 4 x 2 grid for
n = 8. Every gathered result is compared with the serial product."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from spmd import run_spmd

X = [[1.0, 2.0], [3.0, 4.0]]
W = [[5.0, 6.0], [7.0, 8.0]]


def _grid(n):
    return {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (4, 2)}[n]


def _block(a: np.ndarray, R: int, C: int, r: int, c: int) -> np.ndarray:
    """Block (r, c) of the last two dims: rows split R ways, columns C ways (contiguous)."""
    m, k = a.shape[-2:]
    return np.ascontiguousarray(a[..., r * m // R:(r + 1) * m // R, c * k // C:(c + 1) * k // C])


def _ctx(comm):
    from paper_2507_05753_b200 import MpContext
    return MpContext(comm, list(range(comm.world_size)))


def _kat_forward(comm):
    from paper_2507_05753_b200 import pnt
    ctx = _ctx(comm)
    R, C = ctx.R, ctx.C
    x = torch.tensor(_block(np.array(X), R, C, ctx.r, ctx.c))
    w = torch.tensor(_block(np.array(W), R, C, ctx.r, ctx.c))
    return pnt(ctx, x, w, b_is_param=True).tolist(), ctx.flops, ctx.param_buffer_peak


def test_spec_2way_nt_example():
    # rank 0 yields [[17], [39]], rank 1 yields [[23], [53]]
    res = run_spmd(2, _kat_forward)
    assert res[0][0] == [[17.0], [39.0]] and res[1][0] == [[23.0], [53.0]]


def test_spec_4way_blocks():
    # Y blocks 17, 23, 39, 53 land on ranks 0, 1, 2, 3
    res = run_spmd(4, _kat_forward)
    assert [r[0] for r in res] == [[[17.0]], [[23.0]], [[39.0]], [[53.0]]]
    # FLOPs: every rank does exactly 1/n of the serial 2*m*n*k (balanced schedule)
    assert [r[1] for r in res] == [2 * 2 * 2 * 2 // 4] * 4
    # the gathered weight block (B's other row) is a live parameter buffer during the call
    assert all(r[2] == 1 for r in res)


def _kat_backward(comm, wmat):
    from paper_2507_05753_b200 import pnn, ptn
    ctx = _ctx(comm)
    R, C = ctx.R, ctx.C
    x = torch.tensor(_block(np.array(X), R, C, ctx.r, ctx.c))
    w = torch.tensor(_block(np.array(wmat), R, C, ctx.r, ctx.c))
    g = torch.ones_like(x)  # L = sum(Y): unit upstream
    return pnn(ctx, g, w).tolist(), ptn(ctx, g, x).tolist()


@pytest.mark.parametrize("n", [2, 4])
def test_spec_backward_examples(n):
    # W = I -> grad_X gathers to ones; W = [[5,6],[7,8]] -> grad_W = [[4,6],[4,6]]
    R, C = _grid(n)
    eye = run_spmd(n, _kat_backward, [[1.0, 0.0], [0.0, 1.0]])
    full = run_spmd(n, _kat_backward, W)
    for pos, (gx, _) in enumerate(eye):
        assert np.array_equal(np.array(gx), _block(np.ones((2, 2)), R, C, pos // C, pos % C))
    for pos, (_, gw) in enumerate(full):
        assert np.array_equal(np.array(gw), _block(np.array([[4.0, 6.0], [4.0, 6.0]]), R, C, pos // C, pos % C))


def _kat_tn(comm):
    from paper_2507_05753_b200 import ptn
    ctx = _ctx(comm)
    x = torch.tensor(_block(np.array(X), ctx.R, ctx.C, ctx.r, ctx.c))
    w = torch.tensor(_block(np.eye(2), ctx.R, ctx.C, ctx.r, ctx.c))
    return ptn(ctx, x, w).tolist()


@pytest.mark.parametrize("n", [2, 4])
def test_spec_tn_identity_is_transpose(n):
    # X^T I == X^T
    R, C = _grid(n)
    res = run_spmd(n, _kat_tn)
    for pos, got in enumerate(res):
        assert np.array_equal(np.array(got), _block(np.array(X).T, R, C, pos // C, pos % C))


def test_spec_comm_count():
    # m = 2, n_out = 2, n = 2 -> 2 elements sent per rank (reference schedule table)
    from paper_2507_05753_b200 import comm_volume
    rep = comm_volume(2, 2, 2, 2, "NT")
    assert rep.forward_sent == [2, 2]
    assert comm_volume(2, 2, 2, 1, "NT").total_sent == 0


def _random(comm, seed):
    from paper_2507_05753_b200 import pnn, pnt, ptn
    ctx = _ctx(comm)
    R, C = ctx.R, ctx.C
    rng = np.random.default_rng(seed)
    m, k, n = 16, 24, 8 * C * R
    a = rng.standard_normal((3, m, k))
    b_nt = rng.standard_normal((n, k))
    b_nn = rng.standard_normal((k, n))
    bl = lambda t: torch.tensor(_block(t, R, C, ctx.r, ctx.c), dtype=torch.float32)  # noqa: E731
    out = {
        "NT": pnt(ctx, bl(a), bl(b_nt)).numpy(),
        "NN": pnn(ctx, bl(a), bl(b_nn)).numpy(),
        "TN": ptn(ctx, bl(a), bl(rng.standard_normal((3, m, n)))).numpy(),
    }
    return out, ctx.flops


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_random_equivalence_all_modes(n):
    """gather(primitive_n(A, B)) == serial product (f32 rel <= 1e-5, SPEC.md invariants), and the
    per-rank FLOPs add up to the serial count."""
    R, C = _grid(n)
    res = run_spmd(n, _random, 11)
    rng = np.random.default_rng(11)
    m, k, nn = 16, 24, 8 * C * R
    a = rng.standard_normal((3, m, k))
    b_nt, b_nn = rng.standard_normal((nn, k)), rng.standard_normal((k, nn))
    b_tn = rng.standard_normal((3, m, nn))
    serial = {"NT": a @ b_nt.T, "NN": a @ b_nn, "TN": np.swapaxes(a, -1, -2) @ b_tn}
    for pos, (out, _) in enumerate(res):
        for mode, full in serial.items():
            exp = _block(full, R, C, pos // C, pos % C)
            np.testing.assert_allclose(out[mode], exp, rtol=1e-5, atol=1e-5 * np.abs(full).max())
    total = sum(f for _, f in res)
    assert total == 3 * 2 * (m * nn * k + m * nn * k + k * nn * m)


# ------------------------------------------------------------------ reference layer API
def _block_layers(comm):
    """MixerBlock (layers.py) of a WeatherMixerModel built on this rank's tiles: forward, then
    backward of an upstream gradient; returns the local output / input grad / param grads."""
    import json
    import os
    from oracle import model as om
    from paper_2507_05753_b200 import ModelConfig, MpContext, WeatherMixerModel
    here = os.path.dirname(os.path.abspath(__file__))
    meta = json.load(open(os.path.join(here, "golden", "comm_golden.json")))
    cfg = ModelConfig.from_dict(meta["config"])
    ctx = MpContext(comm, list(range(comm.world_size)))
    model = WeatherMixerModel(ctx, cfg, seed=0, dtype="f32", device="cpu")
    oc = om.Config(**{**meta["config"], "grid": tuple(meta["config"]["grid"]), "patch": tuple(meta["config"]["patch"])})
    rng = np.random.default_rng(4)
    h = rng.standard_normal((2, oc.tokens, oc.d_emb))
    g = rng.standard_normal((2, oc.tokens, oc.d_emb))
    ts = model.sets["T"][ctx.r]
    es = model.sets["E_C"][ctx.c]
    hl = torch.tensor(h[:, ts][:, :, es], dtype=torch.float32)
    gl = torch.tensor(g[:, ts][:, :, es], dtype=torch.float32)
    model.zero_grads()
    blk = model.blocks[0]
    y, cache = blk.forward(hl)
    gx = blk.backward(cache, gl)
    model.grad_sync()
    grads = {k: p.grad.numpy().copy() for k, p in model.params.items() if k.startswith("block0.")}
    return {"rc": (ctx.R, ctx.C, ctx.r, ctx.c), "y": y.numpy(), "gx": gx.numpy(), "grads": grads,
            "flops": ctx.flops, "ts": ts, "es": es}


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_mixer_block_layer_api_matches_oracle(n):
    import json
    import os
    from oracle import model as om
    here = os.path.dirname(os.path.abspath(__file__))
    meta = json.load(open(os.path.join(here, "golden", "comm_golden.json")))
    oc = om.Config(**{**meta["config"], "grid": tuple(meta["config"]["grid"]), "patch": tuple(meta["config"]["patch"])})
    P = om.init_params(oc, 0, np.float64)
    P = {k: v.astype(np.float32).astype(np.float64) for k, v in P.items()}
    rng = np.random.default_rng(4)
    h = rng.standard_normal((2, oc.tokens, oc.d_emb))
    g = rng.standard_normal((2, oc.tokens, oc.d_emb))
    ref = om.SerialModel(oc, P)
    y, cache = ref.block_forward(0, h)
    grads = {k: np.zeros_like(v) for k, v in P.items()}
    gx = ref.block_backward(0, cache, g, grads)
    res = run_spmd(n, _block_layers)
    for d in res:
        R, C, r, c = d["rc"]
        ts, es = d["ts"], d["es"]
        np.testing.assert_allclose(d["y"], y[:, ts][:, :, es], rtol=0, atol=1e-5 * np.abs(y).max())
        np.testing.assert_allclose(d["gx"], gx[:, ts][:, :, es], rtol=0, atol=1e-5 * np.abs(gx).max())
        for k, got in d["grads"].items():
            exp = om.local_tile(oc, k, grads[k], R, C, r, c)
            np.testing.assert_allclose(got, exp, rtol=0, atol=1e-5 * max(np.abs(grads[k]).max(), 1e-30), err_msg=k)
    # forward + backward of one block: 3 x (4 T E (d_tok + d_ch)) per sample, split evenly
    per_sample = 3 * 4 * oc.tokens * oc.d_emb * (oc.d_tok + oc.d_ch)
    assert sum(d["flops"] for d in res) == 2 * per_sample
