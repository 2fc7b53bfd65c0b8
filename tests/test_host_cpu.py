"""Host-side API parity on CPU: layout API (reference test_sharding.py), config validation and
hashing (model.py:73-111), process groups (test_comm.py:214-236), parameter layouts
(model.py:124-197) and the analytic communication volume (parallel.py:361-466)."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

from oracle import model as om
from paper_2507_05753_b200 import ConfigError, ModelConfig, ProcessGroup, ShardSpec, gather, shard
from paper_2507_05753_b200.config import token_sets
from paper_2507_05753_b200.model import Layout
from paper_2507_05753_b200.parallel import comm_volume, primitive_send_elements
from paper_2507_05753_b200.sharding import contiguous_split, pad_axes, padded_size

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ sharding (test_sharding.py)
def test_two_way_placement_and_round_trip(rng):
    x = rng.standard_normal((3, 5, 7))
    specs = [ShardSpec(2, r, x.shape) for r in range(2)]
    blocks = [shard(x, s) for s in specs]
    assert blocks[0].shape == (3, 5, 4) and specs[1].pad_cols == 1
    assert np.array_equal(blocks[1][..., -1], np.zeros((3, 5)))  # high-side zero padding
    assert np.array_equal(gather(blocks, specs), x)


def test_four_and_eight_way_round_trip_numpy_and_torch(rng):
    for n in (4, 8):
        x = rng.standard_normal((2, 9, 6))
        specs = [ShardSpec(n, r, x.shape) for r in range(n)]
        blocks = [shard(x, s) for s in specs]
        assert np.array_equal(gather(blocks, specs), x)
        xt = torch.tensor(x)
        tb = [shard(xt, s) for s in specs]
        assert torch.equal(gather(tb, specs), xt)
    s = ShardSpec(4, 3, (6, 8))
    assert (s.block_row, s.block_col, s.local_shape) == (1, 1, (3, 4))


def test_shard_errors():
    with pytest.raises(ValueError):
        ShardSpec(3, 0, (4, 4))
    with pytest.raises(ValueError):
        ShardSpec(2, 2, (4, 4))
    with pytest.raises(ValueError):
        ShardSpec(4, 0, (4,))
    with pytest.raises(ValueError):
        gather([np.zeros((2, 2))], [ShardSpec(2, 0, (2, 4))])
    with pytest.raises(ValueError):
        pad_axes(np.zeros(4), {0: 2})
    assert padded_size(7, 2) == 8
    assert [list(c) for c in contiguous_split(5, 2)] == [[0, 1, 2], [3, 4, 5]]


def test_custom_strided_split_round_trip(rng):
    x = rng.standard_normal((4, 8))
    split = (np.array([0, 2, 4, 6]), np.array([1, 3, 5, 7]))
    specs = [ShardSpec(2, r, x.shape, col_split=split) for r in range(2)]
    blocks = [shard(x, s) for s in specs]
    assert np.array_equal(blocks[1], x[:, 1::2])
    assert np.array_equal(gather(blocks, specs), x)


# ------------------------------------------------------------------ config (model.py:41-111)
def test_validate_rules():
    ModelConfig().validate(1)
    with pytest.raises(ConfigError, match="n_vars"):
        ModelConfig(n_vars=7).validate(2)
    with pytest.raises(ConfigError, match="longitude patches"):
        ModelConfig(grid=(32, 60), patch=(4, 4)).validate(4)  # 15 lon patches
    with pytest.raises(ConfigError, match="not divisible"):
        ModelConfig(grid=(30, 64)).validate(1)
    with pytest.raises(ConfigError):
        ModelConfig(d_emb=0).validate(1)
    ModelConfig(grid=(32, 64), patch=(4, 4)).validate(8)  # 16 lon patches / 4
    c4 = ModelConfig(n_vars=70, grid=(728, 1440), patch=(8, 8), d_emb=4320, d_tok=8640, d_ch=4320, n_blocks=3)
    for n in (1, 2, 4, 8):
        c4.validate(n)
    assert abs(c4.train_flops() / 1e9 - 36818.7) < 0.1  # GFLOP per sample, BASELINE.md C4


def test_content_hash_matches_reference_algorithm():
    import hashlib
    c = ModelConfig()
    expect = hashlib.sha256(json.dumps(c.to_dict(), sort_keys=True).encode()).hexdigest()[:16]
    assert c.content_hash() == expect
    assert ModelConfig.from_dict(c.to_dict()) == c


def test_token_sets_match_reference():
    cfg = ModelConfig()
    oc = om.Config()
    for a, b in zip(token_sets(cfg), om.token_sets(oc)):
        assert np.array_equal(a, b)


# ------------------------------------------------------------------ process groups (comm.py:319-361)
def test_process_groups():
    assert ProcessGroup.dp_groups(8, 2) == [[0, 2, 4, 6], [1, 3, 5, 7]]
    assert ProcessGroup.dp_groups(8, 4) == [[0, 4], [1, 5], [2, 6], [3, 7]]
    pg = ProcessGroup(8, 4, 5)
    assert pg.mp_group == [4, 5, 6, 7] and pg.mp_pos == 1 and pg.dp_group == [1, 5] and pg.dp_replicas == 2
    pg8 = ProcessGroup(8, 8, 3)
    assert pg8.mp_group == list(range(8))
    with pytest.raises(ValueError):
        ProcessGroup(6, 4, 0)


# ------------------------------------------------------------------ parameter layouts
@pytest.mark.parametrize("n", [2, 4, 8])
def test_layout_local_matches_grid_tiles(n, rng):
    cfg = om.Config()
    from paper_2507_05753_b200.sharding import grid_shape
    R, C = grid_shape(n)
    sets = {"T": om.token_sets(cfg, R) if R > 1 else None, "K": contiguous_split(cfg.d_tok, C)}
    glob = rng.standard_normal((cfg.tokens, cfg.d_tok))
    lay = Layout(n, "matrix", glob.shape, row_sets=sets["T"], col_sets=sets["K"])
    out = np.zeros_like(glob)
    for pos in range(n):
        loc = lay.local(glob, pos)
        assert np.array_equal(loc, om.local_tile(cfg, "block0.tok1.w", glob, R, C, pos // C, pos % C))
        lay.place(out, pos, loc)
    assert np.array_equal(out, glob)
    # dup positions of a column vector = the column group; of tok2.b = the row group
    vcol = Layout(n, "vec_col", (cfg.d_emb,), col_sets=contiguous_split(cfg.d_emb, C))
    vrow = Layout(n, "vec_row", (cfg.tokens,), row_sets=sets["T"])
    for pos in range(n):
        r, c = pos // C, pos % C
        assert vcol.dup_positions(pos) == (tuple(i * C + c for i in range(R)) if R > 1 else ())
        assert vrow.dup_positions(pos) == tuple(r * C + j for j in range(C))
    if n in (2, 4):  # the reference's own rule (model.py:168-173)
        ref_col = lambda p: (p, p ^ 2) if n == 4 else ()  # noqa: E731
        ref_row = lambda p: (0, 1) if n == 2 else (p, p ^ 1)  # noqa: E731
        for pos in range(n):
            assert sorted(vcol.dup_positions(pos)) == sorted(ref_col(pos))
            assert sorted(vrow.dup_positions(pos)) == sorted(ref_row(pos))


def test_layout_to_local_index():
    cfg = om.Config()
    sets = om.token_sets(cfg, 2)
    lay = Layout(4, "matrix", (cfg.tokens, cfg.d_tok), row_sets=sets, col_sets=contiguous_split(cfg.d_tok, 2))
    t = int(sets[1][5])
    assert lay.to_local_index(3, (t, 70)) == (5, 6)
    assert lay.to_local_index(0, (t, 70)) is None


# ------------------------------------------------------------------ analytic volume (product copy)
def test_product_comm_volume_matches_reference_tables():
    meta = json.load(open(os.path.join(GOLD, "comm_golden.json")))
    for key, val in meta["primitive_send_elements"].items():
        mode, n, a_s, b_s = key.split("/")
        if isinstance(val, str):
            continue
        assert primitive_send_elements(mode, int(n), eval(a_s), eval(b_s)) == val, key
    for key, (fwd, bwd) in meta["comm_volume"].items():
        mode, n, dims = key.split("/")
        m, k, no, b = dims.split(",")
        rep = comm_volume(int(m), int(k), int(no), int(n), mode, batch=int(b[1:]))
        assert (rep.forward_sent, rep.backward_sent) == (fwd, bwd), key
        assert rep.total_sent == sum(fwd) + sum(bwd) == rep.total_received


def test_lr_schedule_spec_examples():
    """step 0 -> 1e-6, end of epoch 1 -> 1e-4 (body), last step -> 1e-5; the
    warm-up end equals the cosine start; host mirror == oracle restatement; out-of-range raises."""
    import math
    from oracle import train as ot
    from paper_2507_05753_b200.train import AdamConfig
    a = AdamConfig(warmup_steps=100, total_steps=10000)
    assert math.isclose(a.lr_at(0), 1e-6)
    assert math.isclose(a.lr_at(100), 1e-4)
    assert math.isclose(a.lr_at(9999), 1e-5)
    assert math.isclose(a.lr_at(9999, "encdec"), 2e-6)
    assert abs(a.lr_at(99) - a.lr_at(100)) < 1e-6  # continuous across the warm-up end
    for s in (0, 1, 50, 99, 100, 101, 5000, 9998, 9999):
        assert math.isclose(a.lr_at(s), ot.lr_at(s, 10000, 100), rel_tol=1e-12)
    with pytest.raises(ValueError):
        a.lr_at(10000)
    assert AdamConfig().lr_at(123, "encdec") == 2e-5  # no schedule: constant class lr


def test_clip_spec_examples():
    from oracle import train as ot
    g, norm = ot.clip_grads([np.array([3.0, 4.0])], 1.0)
    assert np.allclose(g[0], [0.6, 0.8]) and norm == 5.0
    g, _ = ot.clip_grads([np.array([0.3, 0.4])], 1.0)
    assert np.allclose(g[0], [0.3, 0.4])


def test_dp_groups_rule():
    """SPEC.md:491-499 examples: n=2 in 8 ranks -> {0,2,4,6},{1,3,5,7}; n=4 -> {0,4},..."""
    from paper_2507_05753_b200.comm import ProcessGroup
    assert ProcessGroup.dp_groups(8, 2) == [[0, 2, 4, 6], [1, 3, 5, 7]]
    assert ProcessGroup.dp_groups(8, 4) == [[0, 4], [1, 5], [2, 6], [3, 7]]
    assert ProcessGroup(4, 4, 1).dp_replicas == 1


def test_tile_loader_reads_rank_tiles_with_padding(tmp_path):
    """each rank reads exactly oracle.local_sample of the zero-padded sample (and of
    sample + lead as the target); mp-group members share the order, dp replicas split it."""
    from types import SimpleNamespace
    from paper_2507_05753_b200.data import TileLoader
    cfg = ModelConfig(n_vars=8, grid=(32, 64), patch=(4, 4), d_emb=64, d_tok=128, d_ch=64, n_blocks=1)
    oc = om.Config(n_vars=8, grid=(32, 64), patch=(4, 4), d_emb=64, d_tok=128, d_ch=64, n_blocks=1)
    rng = np.random.default_rng(3)
    src = rng.standard_normal((9, 30, 64, 7)).astype(np.float32)  # 30 real rows, 7 real vars
    np.save(tmp_path / "era.npy", src)
    padded = np.zeros((9, 32, 64, 8), np.float32)
    padded[:, :30, :, :7] = src
    for (R, C) in ((1, 1), (1, 2), (2, 2), (4, 2)):
        for r in range(R):
            for c in range(C):
                ctx = SimpleNamespace(R=R, C=C, r=r, c=c, dp_index=0, dp_replicas=1)
                ld = TileLoader(str(tmp_path / "era.npy"), cfg, ctx, lead=2, batch=2, seed=5, pin=False)
                order = ld.order(0)
                got = [(x.clone(), t.clone()) for x, t in ld.epoch(0)]
                assert len(got) == ld.steps_per_epoch() == 3
                for s, (x, t) in enumerate(got):
                    ids = order[2 * s:2 * s + 2]
                    assert np.array_equal(x.numpy(), om.local_sample(oc, padded[ids], R, C, r, c))
                    assert np.array_equal(t.numpy(), om.local_sample(oc, padded[ids + 2], R, C, r, c))
    base = TileLoader(src, cfg, SimpleNamespace(R=1, C=2, r=0, c=1, dp_index=0, dp_replicas=1), pin=False).order(1)
    shares = [TileLoader(src, cfg, SimpleNamespace(R=1, C=2, r=0, c=0, dp_index=k, dp_replicas=2), pin=False).order(1)
              for k in range(2)]
    assert len(shares[0]) == len(shares[1]) and not set(shares[0]) & set(shares[1])
    assert set(shares[0]) | set(shares[1]) <= set(base)
    with pytest.raises(ConfigError):
        TileLoader(src[:, :, :32], cfg, SimpleNamespace(R=1, C=1, r=0, c=0), pin=False)


def test_adam_push_split_respects_segment_limit():
    """26 panel segments (12 blocks at R > 1) -> Adam calls of <= 16 segments each, covering
    the class range exactly once, segments re-based to their call and never split."""
    from paper_2507_05753_b200.engine import split_push
    lo, hi = 1000, 1000 + 26 * 100 + 37
    segs = [(i * 100 + 5, 90, [i]) for i in reversed(range(26))]
    calls = list(split_push(lo, hi, segs, 16))
    assert calls[0][0] == lo and calls[-1][1] == hi
    assert all(a1 == b0 for (_, a1, _), (b0, _, _) in zip(calls, calls[1:]))
    assert all(len(sub) <= 16 for _, _, sub in calls)
    got = sorted((a0 + st, n, tuple(ad)) for a0, a1, sub in calls for st, n, ad in sub)
    assert got == sorted((lo + st, n, tuple(ad)) for st, n, ad in segs)
    for a0, a1, sub in calls:
        assert all(0 <= st and a0 + st + n <= a1 for st, n, _ in sub)
    assert list(split_push(lo, hi, [], 16)) == [(lo, hi, [])]
