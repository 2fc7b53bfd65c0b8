"""Loss weights and optimiser hyper-parameters of the WeatherMixer step (SPEC data/train modules).

The reference package ships no loss or optimiser; these follow SPEC.md:
  lat_weights      SPEC.md:396-400  w_i = cos(phi_i) / mean_j cos(phi_j), cell-centre rows
  var weights      SPEC.md:401-407, 433-434 (pressure-level vector; default all ones)
  Adam             SPEC.md:482-490, lr 1e-4 body / 2e-5 encdec
The device work is done by jg_blend_loss (fused loss) and jg_adam (fused optimiser).
"""
from __future__ import annotations

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
    lr_body: float = 1e-4
    lr_encdec: float = 2e-5
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    def lr(self, lr_class: str) -> float:
        return self.lr_encdec if lr_class == "encdec" else self.lr_body
