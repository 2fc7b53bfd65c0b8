"""ORACLE (test infrastructure): analytic communication volume of the reference schedules.

Restates primitive_send_elements (parallel.py:361-401), comm_volume (parallel.py:430-462) and
WeatherMixerModel.step_comm_volume (model.py:483-529), all in elements sent per rank.
"""
from __future__ import annotations

import numpy as np


def _lead(shape):
    return int(np.prod(shape[:-2], dtype=np.int64)) if len(shape) > 2 else 1


def primitive_send_elements(mode: str, n: int, a_shape, b_shape):
    la, lb = _lead(a_shape), _lead(b_shape)
    lc = max(la, lb)
    if n == 1:
        return [0]
    if mode == "NT":
        m, k, no = a_shape[-2], a_shape[-1], b_shape[-2]
        if n == 2:
            return [la * m * (no // 2)] * 2
        raw = lb * (no // 2) * (k // 2) + la * (m // 2) * (k // 2)
        part = 2 * lc * (m // 2) * (no // 2)
        return [raw, part, part, raw]
    if mode == "NN":
        m, k, no = a_shape[-2], a_shape[-1], b_shape[-1]
        if n == 2:
            return [la * m * (k // 2)] * 2
        a_blk = la * (m // 2) * (k // 2)
        b_blk = lb * (k // 2) * (no // 2)
        part = lc * (m // 2) * (no // 2)
        return [a_blk + b_blk, a_blk + part, a_blk + part, b_blk + a_blk]
    p, q, s = a_shape[-2], a_shape[-1], b_shape[-1]
    if n == 2:
        return [la * p * (q // 2)] * 2
    a_blk = la * (p // 2) * (q // 2)
    b_blk = lb * (p // 2) * (s // 2)
    part = 2 * lc * (q // 2) * (s // 2)
    return [a_blk + b_blk, part, part, b_blk + a_blk]


def _vsum(a, b):
    return [x + y for x, y in zip(a, b)]


def comm_volume(m, k, n_out, n_way, mode="NT", batch=1):
    """(forward_sent, backward_sent) per position (parallel.py:430-462)."""
    if mode == "NT":
        x, w, y = (batch, m, k), (n_out, k), (batch, m, n_out)
        return (primitive_send_elements("NT", n_way, x, w),
                _vsum(primitive_send_elements("NN", n_way, y, w), primitive_send_elements("TN", n_way, y, x)))
    if mode == "NN":
        x, w, y = (batch, m, k), (k, n_out), (batch, m, n_out)
        return (primitive_send_elements("NN", n_way, x, w),
                _vsum(primitive_send_elements("NT", n_way, y, w), primitive_send_elements("TN", n_way, x, y)))
    x, w, y = (batch, m, k), (m, n_out), (batch, k, n_out)
    return (primitive_send_elements("TN", n_way, x, w),
            _vsum(primitive_send_elements("NT", n_way, w, y), primitive_send_elements("NN", n_way, x, y)))


def step_comm_volume(cfg, n: int, batch: int, r: int = 1, dup_elements_per_rank: int = 0) -> int:
    """Total elements sent across the mp group per fwd+bwd (model.py:483-529).

    dup_elements_per_rank: elements of duplicated vector params held per rank (grad sync).
    """
    if n == 1:
        return 0
    m_tok = batch * cfg.tokens

    def layer(m, k, no, mode):
        f, b = comm_volume(m, k, no, n, mode)
        return sum(f) + sum(b)

    total = layer(m_tok, cfg.patch_features, cfg.d_emb, "NT")
    wb, hb, ob = (cfg.tokens, cfg.d_tok), (batch, cfg.d_emb, cfg.d_tok), (batch, cfg.tokens, cfg.d_emb)
    tok2 = (sum(primitive_send_elements("NT", n, wb, hb)) + sum(primitive_send_elements("NN", n, ob, hb))
            + sum(primitive_send_elements("TN", n, ob, wb)))
    per_block = (layer(m_tok, cfg.d_emb, cfg.d_tok, "TN") + tok2 + layer(m_tok, cfg.d_emb, cfg.d_ch, "NT")
                 + layer(m_tok, cfg.d_ch, cfg.d_emb, "NT"))
    total += r * cfg.n_blocks * per_block
    total += layer(m_tok, cfg.d_emb, cfg.patch_features, "NT")
    rows = batch * cfg.tokens if n == 2 else batch * cfg.tokens // 2
    total += r * cfg.n_blocks * 2 * 2 * (rows * 2) * n
    total += dup_elements_per_rank * n
    return total


def dup_elements_per_rank(cfg, n: int) -> int:
    """Elements of duplicated vector params per rank (Layout.dup_positions, model.py:168-173)."""
    if n == 1:
        return 0
    E, F, K, H, C, T = cfg.d_emb, cfg.patch_features, cfg.d_tok, cfg.d_ch, cfg.n_vars, cfg.tokens
    if n == 2:
        return cfg.n_blocks * T  # tok2.b replicated on both positions
    col = E + F + C + cfg.n_blocks * (4 * E + K + H + E)  # enc.b, dec.b, blend, ln1/ln2 gamma/beta, tok1.b, ch1.b, ch2.b
    return col // 2 + cfg.n_blocks * T // 2
