"""Loss weights and optimiser hyper-parameters of the WeatherMixer step (SPEC data/train modules).

The reference package ships no loss or optimiser; these follow SPEC.md:
  lat_weights      SPEC.md:396-400  w_i = cos(phi_i) / mean_j cos(phi_j), cell-centre rows
  var weights      SPEC.md:401-407, 433-434 (pressure-level vector; default all ones)
  Adam             SPEC.md:482-490, lr 1e-4 body / 2e-5 encdec
  lr_at            SPEC.md:464-472 (linear warm-up from 1e-6 over epoch 1, cosine to 1e-5)
  clipping         SPEC.md:473-481 (global L2 norm over the sharded parameter set, 1.0)
The device work is done by jg_blend_loss (fused loss), jg_opt_schedule (lr + clip factor, read
from device memory so one captured graph serves every step) and jg_adam (fused optimiser).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

PRESSURE_WEIGHTS = (1, 1, 1, 1, 1, 1, 0.9, 0.8, 0.7, 0.6, 0.5, 0.4, 0.3)  # SPEC.md:434, high -> low pressure


def lat_weights(n_lat: int, n_real: int | None = None) -> np.ndarray:
    """Cell-centre latitude weights normalised to mean 1 over the real rows; padded rows 0."""
    n_real = n_lat if n_real is None else n_real
    if n_real < 1:
        raise ValueError("lat_weights: all-zero weights (degenerate grid)")
    phi = np.deg2rad(90.0 - (np.arange(n_real) + 0.5) * 180.0 / n_real)
    w = np.cos(phi)
    w = w / w.mean()
    out = np.zeros(n_lat)
    out[:n_real] = w
    return out


def var_weights(n_vars: int, n_real: int | None = None, per_var=None) -> np.ndarray:
    """Per-channel loss weights; padded channels get 0."""
    n_real = n_vars if n_real is None else n_real
    out = np.zeros(n_vars)
    out[:n_real] = 1.0 if per_var is None else np.asarray(per_var, dtype=np.float64)[:n_real]
    return out


@dataclass
class AdamConfig:
    """Adam hyper-parameters plus the SPEC schedule. total_steps == 0 keeps the lr constant at the
    class base; clip_norm None disables clipping. The encdec class runs the same curve scaled by
    lr_encdec / lr_body (warm-up start excepted: both classes start from warm_start)."""
    lr_body: float = 1e-4
    lr_encdec: float = 2e-5
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    warm_start: float = 1e-6
    final_lr_body: float = 1e-5
    warmup_steps: int = 0        # steps of epoch 1
    total_steps: int = 0         # 0: no schedule
    clip_norm: float | None = None

    def lr(self, lr_class: str) -> float:
        return self.lr_encdec if lr_class == "encdec" else self.lr_body

    def final_lr(self, lr_class: str) -> float:
        return self.final_lr_body * self.lr(lr_class) / self.lr_body

    def schedule(self, lr_class: str) -> tuple:
        """Fields of jg_lr_schedule for one class."""
        return (self.lr(lr_class), self.warm_start, self.final_lr(lr_class), self.warmup_steps, self.total_steps)

    def lr_at(self, step: int, lr_class: str = "body") -> float:
        """SPEC lr_at(step, total_steps, cfg, class) for 0 <= step < total_steps (host mirror of
        the device schedule)."""
        if self.total_steps <= 0:
            return self.lr(lr_class)
        if not 0 <= step < self.total_steps:
            raise ValueError(f"lr_at: step {step} outside [0, {self.total_steps})")
        base, final = self.lr(lr_class), self.final_lr(lr_class)
        if step < self.warmup_steps:
            return self.warm_start + (base - self.warm_start) * step / self.warmup_steps
        span = self.total_steps - 1 - self.warmup_steps
        u = (step - self.warmup_steps) / span if span > 0 else 1.0
        return final + 0.5 * (base - final) * (1.0 + math.cos(math.pi * u))
