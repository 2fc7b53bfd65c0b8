"""ORACLE (test infrastructure): the bounded CPU-baseline sample for bench.py.

Times the reference algorithm (this package's numpy restatement, kind "port") on the host
cores: one WeatherMixer block forward + backward at the benchmark's full shape (the repeated
unit that carries >= 90% of the step's FLOPs at C4), f32, OpenBLAS using every host core.
The full-step time is extrapolated by FLOP count: t_step = t_block * F_train / F_block.
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import model as om


def block_flops(cfg: om.Config, batch: int = 1) -> int:
    """2 m n k per linear, backward = 2 x forward, one mixer block."""
    return 3 * batch * 4 * cfg.tokens * cfg.d_emb * (cfg.d_tok + cfg.d_ch)


def time_block(cfg: om.Config, batch: int = 1, repeats: int = 1, seed: int = 0, dtype=np.float32):
    """Seconds per block fwd+bwd (min over `repeats` timed runs after one untimed run)."""
    one = om.Config(n_vars=cfg.n_vars, grid=cfg.grid, patch=cfg.patch, d_emb=cfg.d_emb,
                    d_tok=cfg.d_tok, d_ch=cfg.d_ch, n_blocks=1)
    rng = np.random.default_rng(seed)
    E, K, H, Tn = cfg.d_emb, cfg.d_tok, cfg.d_ch, cfg.tokens
    p = {
        "block0.ln1.gamma": np.ones(E, dtype), "block0.ln1.beta": np.zeros(E, dtype),
        "block0.tok1.w": rng.uniform(-Tn ** -0.5, Tn ** -0.5, (Tn, K)).astype(dtype),
        "block0.tok1.b": np.zeros(K, dtype),
        "block0.tok2.w": rng.uniform(-K ** -0.5, K ** -0.5, (Tn, K)).astype(dtype),
        "block0.tok2.b": np.zeros(Tn, dtype),
        "block0.ln2.gamma": np.ones(E, dtype), "block0.ln2.beta": np.zeros(E, dtype),
        "block0.ch1.w": rng.uniform(-E ** -0.5, E ** -0.5, (H, E)).astype(dtype),
        "block0.ch1.b": np.zeros(H, dtype),
        "block0.ch2.w": rng.uniform(-H ** -0.5, H ** -0.5, (E, H)).astype(dtype),
        "block0.ch2.b": np.zeros(E, dtype),
    }
    model = om.SerialModel(one, p)
    h = rng.standard_normal((batch, Tn, E)).astype(dtype)
    g = rng.standard_normal((batch, Tn, E)).astype(dtype)

    def run():
        grads = {k: np.zeros_like(v) for k, v in p.items()}
        _, cache = model.block_forward(0, h)
        model.block_backward(0, cache, g, grads)

    times = []
    for i in range(repeats + 1):
        t0 = time.perf_counter()
        run()
        if i:
            times.append(time.perf_counter() - t0)
    return min(times)


def step_estimate(cfg: om.Config, batch: int = 1, repeats: int = 1):
    """(seconds per full training step, seconds of the timed block sample, host cores)."""
    tb = time_block(cfg, batch, repeats)
    ftrain = om.train_flops(cfg, batch)
    return tb * ftrain / block_flops(cfg, batch), tb, os.cpu_count()
