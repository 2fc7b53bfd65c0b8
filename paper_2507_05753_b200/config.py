"""ModelConfig / ConfigError / token_sets — reference model.py:37-121, extended to 8-way grids.

`validate(n)` keeps the reference rules (model.py:73-92: every width >= 1, even widths for a
split, even longitude patches at n = 4) and generalises them to the R x C Jigsaw grid of
sharding.grid_shape(n): n_vars, d_emb, d_tok, d_ch, patch features divisible by C; d_emb,
d_ch, patch features divisible by R; longitude patches divisible by R.
"""
from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError
from .sharding import grid_shape

__all__ = ["ModelConfig", "ConfigError", "token_sets", "pad_grid"]


@dataclass
class ModelConfig:
    n_vars: int = 8
    grid: tuple[int, int] = (32, 64)
    patch: tuple[int, int] = (4, 4)
    d_emb: int = 64
    d_tok: int = 128
    d_ch: int = 64
    n_blocks: int = 3
    dropout_rate: float = 0.0

    @property
    def lat(self) -> int:
        return self.grid[0]

    @property
    def lon(self) -> int:
        return self.grid[1]

    @property
    def patch_grid(self) -> tuple[int, int]:
        return self.grid[0] // self.patch[0], self.grid[1] // self.patch[1]

    @property
    def tokens(self) -> int:
        gl, gw = self.patch_grid
        return gl * gw

    @property
    def patch_features(self) -> int:
        return self.patch[0] * self.patch[1] * self.n_vars

    def validate(self, n: int = 1) -> None:
        for name in ("n_vars", "d_emb", "d_tok", "d_ch", "n_blocks"):
            if getattr(self, name) < 1:
                raise ConfigError(f"model.{name} must be >= 1")
        if not 0.0 <= self.dropout_rate < 1.0:
            raise ConfigError("model.dropout_rate must be in [0, 1)")
        if self.lat % self.patch[0] or self.lon % self.patch[1]:
            raise ConfigError(f"model.grid {self.grid} not divisible by model.patch {self.patch}")
        try:
            R, C = grid_shape(n)
        except ValueError as e:
            raise ConfigError(str(e)) from None
        if n >= 2:
            for name in ("n_vars", "d_emb", "d_tok", "d_ch"):
                if getattr(self, name) % C:
                    word = "even" if C == 2 else f"divisible by {C}"
                    raise ConfigError(f"model.{name} must be {word} for {n}-way sharding")
        if R > 1:
            if self.patch_grid[1] % R:
                raise ConfigError(
                    f"model.grid longitude patches ({self.patch_grid[1]}) must be "
                    f"{'even' if R == 2 else f'divisible by {R}'} for {n}-way sharding")
            for name in ("d_emb", "d_ch"):
                if getattr(self, name) % R:
                    raise ConfigError(f"model.{name} must be divisible by {R} for {n}-way sharding")
            if self.patch_features % R:
                raise ConfigError(f"model patch features ({self.patch_features}) must be divisible by {R}")
        # TMA row strides are 16-byte multiples: every per-rank contiguous width (bf16) must be a
        # multiple of 8 elements. Pad n_vars (zero-weight channels) when the patch features miss it.
        for name, width in (("d_emb", self.d_emb), ("d_tok", self.d_tok), ("d_ch", self.d_ch),
                            ("n_vars (patch features)", self.patch_features)):
            if (width // C) % 8:
                raise ConfigError(f"model.{name}: per-rank width {width // C} at {n}-way must be a multiple of 8 "
                                  f"(16-byte TMA rows); pad the global width")

    def to_dict(self) -> dict:
        return {
            "n_vars": self.n_vars, "grid": list(self.grid), "patch": list(self.patch),
            "d_emb": self.d_emb, "d_tok": self.d_tok, "d_ch": self.d_ch,
            "n_blocks": self.n_blocks, "dropout_rate": self.dropout_rate,
        }

    @classmethod
    def from_dict(cls, d: dict) -> "ModelConfig":
        d = dict(d)
        if "grid" in d:
            d["grid"] = tuple(d["grid"])
        if "patch" in d:
            d["patch"] = tuple(d["patch"])
        return cls(**d)

    def content_hash(self) -> str:
        return hashlib.sha256(json.dumps(self.to_dict(), sort_keys=True).encode()).hexdigest()[:16]

    def train_flops(self, batch: int = 1, r: int = 1) -> int:
        """Algorithmic FLOPs of one training step: 2 m n k per linear, backward = 2 x forward
        (equals the sum of the reference's MpContext.flops, parallel.py:65-69)."""
        T, F, E = self.tokens, self.patch_features, self.d_emb
        return 3 * batch * (4 * T * F * E + r * self.n_blocks * 4 * T * E * (self.d_tok + self.d_ch))


def token_sets(cfg: ModelConfig, parts: int = 2) -> list[np.ndarray]:
    """Token indices owned by each longitude part, row-major token order (model.py:114-121)."""
    gl, gw = cfg.patch_grid
    w = gw // parts
    return [np.array([a * gw + b for a in range(gl) for b in range(i * w, (i + 1) * w)], dtype=np.int64)
            for i in range(parts)]


def pad_grid(lat: int, n_vars: int, p_lat: int, n_way: int = 1) -> tuple[int, int]:
    """Zero-padding rule for ERA5 shapes: rows up to a multiple of the patch,
    channels up to a multiple of the channel split (and even)."""
    C = grid_shape(n_way)[1]
    lat_p = -(-lat // p_lat) * p_lat
    mult = max(2, C)
    return lat_p, -(-n_vars // mult) * mult
