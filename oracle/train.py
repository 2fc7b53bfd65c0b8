"""ORACLE (test infrastructure): loss and optimiser of the SPEC `data` / `train` modules.

The reference package ships no loss or optimiser code; these restate SPEC.md and are pinned
to SPEC's worked examples only (tests/test_oracle.py):
  lat_weights            SPEC.md:396-400  w_i = cos(phi_i) / mean_j cos(phi_j), cell centres
  weighted_mse_loss      SPEC.md:401-407  mean of lat_w * var_w * (pred - target)^2
  adam_step              SPEC.md:482-490  bias-corrected Adam, betas (0.9, 0.999), eps 1e-8
  clip_grads
  lr_at                  SPEC.md:464-472  linear warm-up from 1e-6 over epoch 1, cosine to 1e-5
Conventions fixed here (stated in DESIGN.md): the mean runs over B x lat_real x lon x C_real;
zero-padded rows (721 -> 728) and channels get weight 0; p -= lr * mhat / (sqrt(vhat) + eps).
"""
from __future__ import annotations

import numpy as np

PRESSURE_WEIGHTS = [1, 1, 1, 1, 1, 1, 0.9, 0.8, 0.7, 0.6, 0.5, 0.4, 0.3]  # SPEC.md:434, high -> low pressure


def lat_weights(n_lat: int, n_real: int | None = None) -> np.ndarray:
    """Cell-centre latitudes phi_i = 90 - (i + 0.5) * 180 / n_real; padded rows get 0."""
    n_real = n_lat if n_real is None else n_real
    phi = np.deg2rad(90.0 - (np.arange(n_real) + 0.5) * 180.0 / n_real)
    w = np.cos(phi)
    w = w / w.mean()
    out = np.zeros(n_lat)
    out[:n_real] = w
    return out


def weighted_mse_loss(pred, target, lat_w, var_w, count=None):
    """Returns (loss, dloss/dpred). count defaults to pred.size."""
    count = pred.size if count is None else count
    wt = lat_w[None, :, None, None] * var_w[None, None, None, :]
    e = pred - target
    loss = float((wt * e * e).sum() / count)
    return loss, 2.0 * wt * e / count


def lat_weighted_rmse(pred, target, lat_w):
    """Per-variable RMSE."""
    e2 = lat_w[None, :, None, None] * (pred - target) ** 2
    return np.sqrt(e2.mean(axis=(0, 1, 2)))


def adam_step(p, g, m, v, step, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """In-place bias-corrected Adam; step counts from 1."""
    m *= beta1
    m += (1 - beta1) * g
    v *= beta2
    v += (1 - beta2) * g * g
    mhat = m / (1 - beta1 ** step)
    vhat = v / (1 - beta2 ** step)
    p -= lr * mhat / (np.sqrt(vhat) + eps)
    return p


def clip_grads(grads, clip_norm):
    norm = float(np.sqrt(sum(float((g * g).sum()) for g in grads)))
    if norm > clip_norm:
        return [g * (clip_norm / norm) for g in grads], norm
    return list(grads), norm


def lr_at(step, total_steps, warmup_steps, base=1e-4, warm_start=1e-6, final=1e-5):
    """SPEC lr_at: linear from warm_start to base across the warm-up (epoch 1), then
    final + (base - final) / 2 * (1 + cos(pi t)), t = progress through the remaining steps."""
    if not 0 <= step < total_steps:
        raise ValueError("step out of range")
    if step < warmup_steps:
        return warm_start + (base - warm_start) * step / warmup_steps
    t = (step - warmup_steps) / max(1, total_steps - 1 - warmup_steps)
    return final + (base - final) / 2.0 * (1.0 + np.cos(np.pi * t))
