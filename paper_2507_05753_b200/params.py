"""Parameter shards in flat HBM buffers (reference Param, parallel.py:469-493).

Every local parameter shard of a model is a view into a handful of flat device buffers, one
per role, laid out lr-class by lr-class so the optimiser is one fused kernel per class:

  master fp32  (Param.data)   grad fp32 (Param.grad)   m, v fp32 (Adam moments)
  op           GEMM-operand copy: bf16 in bf16 mode (written by the Adam kernel), or the
               master itself in fp32 mode.

Offsets are aligned to 64 elements so every view satisfies the 16-byte TMA / vector-access
alignment. Zeroing all gradients is one memset (reference zero_grads, model.py:447-449).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

ALIGN = 64


@dataclass
class Param:
    """One locally stored parameter shard with gradient accumulation (parallel.py:469-493)."""

    name: str
    data: torch.Tensor
    lr_class: str = "body"
    dup_positions: tuple[int, ...] = ()
    grad: torch.Tensor | None = field(default=None, repr=False)
    op: torch.Tensor | None = field(default=None, repr=False)  # GEMM operand copy (bf16 or == data)

    @property
    def dup_factor(self) -> int:
        return max(1, len(self.dup_positions))

    def zero_grad(self) -> None:
        if self.grad is None:
            self.grad = torch.zeros_like(self.data)
        else:
            self.grad.zero_()

    def add_grad(self, g: torch.Tensor) -> None:
        if self.grad is None:
            self.grad = torch.zeros_like(self.data)
        self.grad += g


class FlatParams:
    """Owns the flat buffers; hands out Param views in registration order."""

    CLASSES = ("encdec", "body")

    KINDS = ("matrix", "vec_col", "vec_row")

    def __init__(self, specs, device, op_dtype: torch.dtype):
        # specs: list of (name, local_shape, lr_class, dup_positions, kind) in registration order.
        # Storage order: lr class, then kind, so each (class, kind) is one contiguous range:
        # Adam runs once per class and the duplicated-vector gradient sync is one all-reduce
        # per (class, vector kind).
        self.specs = list(specs)
        self.device = device
        self.op_dtype = op_dtype
        self.offsets: dict[str, int] = {}
        self.class_range: dict[str, tuple[int, int]] = {}
        self.kind_range: dict[tuple[str, str], tuple[int, int]] = {}
        off = 0
        for cls in self.CLASSES:
            start = off
            for kind in self.KINDS:
                kstart = off
                for name, shape, lr_class, _, pkind in self.specs:
                    if lr_class != cls or pkind != kind:
                        continue
                    self.offsets[name] = off
                    numel = 1
                    for s in shape:
                        numel *= s
                    off += -(-numel // ALIGN) * ALIGN
                self.kind_range[(cls, kind)] = (kstart, off)
            self.class_range[cls] = (start, off)
        self.total = off
        f32 = dict(dtype=torch.float32, device=device)
        self.master = torch.zeros(self.total, **f32)
        self.grad = torch.zeros(self.total, **f32)
        self.m = torch.zeros(self.total, **f32)
        self.v = torch.zeros(self.total, **f32)
        self.op = self.master if op_dtype == torch.float32 else torch.zeros(self.total, dtype=op_dtype, device=device)
        self.params: dict[str, Param] = {}
        for name, shape, lr_class, dup, _ in self.specs:
            o = self.offsets[name]
            numel = 1
            for s in shape:
                numel *= s
            p = Param(name, self.master[o:o + numel].view(shape), lr_class, tuple(dup))
            p.grad = self.grad[o:o + numel].view(shape)
            p.op = self.op[o:o + numel].view(shape)
            self.params[name] = p

    def zero_grads(self) -> None:
        from . import kernels as K  # (jg_memset: one launch for every gradient of the model)
        K.zero(self.grad)

    def view(self, name: str, buf: torch.Tensor) -> torch.Tensor:
        """`name`'s view into another flat buffer (m, v, ...) with the same layout."""
        p = self.params[name]
        o = self.offsets[name]
        return buf[o:o + p.data.numel()].view(p.data.shape)

    def vec_range(self, cls: str) -> tuple[int, int]:
        """Contiguous range of all vector parameters (column then row) of one lr class."""
        return self.kind_range[(cls, "vec_col")][0], self.kind_range[(cls, "vec_row")][1]

    def numel(self) -> int:
        return sum(p.data.numel() for p in self.params.values())
