"""Jigsaw distributed linear algebra on B200 — reference parallel.py API over NCCL + tcgen05.

Three collective primitives cover every layer multiplication (parallel.py:1-25):

    pnt(a, b) = a @ b.T      pnn(a, b) = a @ b      ptn(a, b) = a.T @ b

Each rank holds one block of every operand and gets its output block in the same layout, so
layers chain without redistribution. The reference runs fixed point-to-point schedules for
n = 2 and a 1:3:3:1 FLOP-imbalanced schedule for n = 4 (measured). Here the group
is an R x C grid (sharding.grid_shape: 1x2, 2x2, 4x2) and every primitive is the balanced
"gather the operand panel along one grid axis, one local tcgen05 GEMM, reduce-scatter the
partials along the other" schedule of SURVEY 8e, each rank doing exactly 1/n of the FLOPs:

  C(i, j) = sum_l A(i, l) B(j, l)^T on a grid where rank (r, c) holds A(r, c), B(r, c):
    pnt:  AG B over the column group -> B(:, c);  P = A(r, c) B(:, c)^T  [m_r, n];
          RS P over the row group along n  -> C(r, c)
  pnn / ptn reduce to pnt by the backward-composition table (parallel.py:20-24).

Generic primitives (any operands) live here; the WeatherMixer model drives the same
collectives through its fused per-layer paths (model.py).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import tensor as T
from .comm import Communicator, ProcessGroup
from .errors import ShapeError
from .params import Param  # noqa: F401  (re-exported: reference parallel.Param)
from .sharding import grid_shape
from .tensor import MatmulMode


class MpContext:
    """One rank's view of its model-parallel group (parallel.py:44-76), as an R x C grid."""

    def __init__(self, comm: Communicator, group: list[int]):
        group = sorted(group)
        if comm.rank not in group:
            raise ValueError(f"rank {comm.rank} not in model-parallel group {group}")
        if len(group) not in (1, 2, 4, 8):
            raise ValueError(f"model-parallel group must have 1, 2, 4 or 8 ranks, got {group}")
        self.comm = comm
        self.group = group
        self.n = len(group)
        self.pos = group.index(comm.rank)
        self.R, self.C = grid_shape(self.n)
        self.r, self.c = self.pos // self.C, self.pos % self.C
        self.flops = 0
        self.param_buffer_elements = 0
        self.param_buffer_peak = 0
        self.row_ranks = [group[self.r * self.C + j] for j in range(self.C)]
        self.col_ranks = [group[i * self.C + self.c] for i in range(self.R)]
        self.row_group = self.col_group = None
        self.mp_group = None
        self.dp_group = None
        pg = ProcessGroup(comm.world_size, self.n, comm.rank) if comm.world_size % self.n == 0 else None
        self.dp_replicas = pg.dp_replicas if pg is not None else 1
        self.dp_index = pg.dp_index if pg is not None else 0
        if self.n > 1:
            self._build_groups()
        if self.dp_replicas > 1:
            # dp groups {r : r % n == c} (comm.py:346-361), created in the same order on every rank
            for ranks in ProcessGroup.dp_groups(comm.world_size, self.n):
                g = comm.group(ranks)
                if comm.rank in ranks:
                    self.dp_group = g

    def _build_groups(self) -> None:
        # new_group is collective over the whole world: every rank creates every mp group's row
        # and column groups in the same order, keeping only its own.
        pg = ProcessGroup(self.comm.world_size, self.n, self.comm.rank)
        for k in range(pg.dp_replicas):
            base = k * self.n
            g = self.comm.group(list(range(base, base + self.n)))
            if self.comm.rank in range(base, base + self.n):
                self.mp_group = g
            for i in range(self.R):
                ranks = [base + i * self.C + j for j in range(self.C)]
                g = self.comm.group(ranks) if self.C > 1 else None
                if self.comm.rank in ranks:
                    self.row_group = g
            for j in range(self.C):
                ranks = [base + i * self.C + j for i in range(self.R)]
                g = self.comm.group(ranks) if self.R > 1 else None
                if self.comm.rank in ranks:
                    self.col_group = g

    def rank_at(self, pos: int) -> int:
        return self.group[pos]

    def _count(self, m: int, n: int, k: int, batch: int = 1) -> None:
        self.flops += 2 * m * n * k * batch

    # -- collectives on the grid axes (device tensors, current stream) --------
    def all_gather_row(self, x: torch.Tensor) -> torch.Tensor:
        """[C, *x.shape] stack of the row group's blocks (ordered by column index)."""
        out = torch.empty((self.C, *x.shape), dtype=x.dtype, device=x.device)
        if self.C == 1:
            out[0].copy_(x)
        else:
            dist.all_gather_into_tensor(out, x.contiguous(), group=self.row_group)
        return out

    def all_gather_col(self, x: torch.Tensor) -> torch.Tensor:
        out = torch.empty((self.R, *x.shape), dtype=x.dtype, device=x.device)
        if self.R == 1:
            out[0].copy_(x)
        else:
            dist.all_gather_into_tensor(out, x.contiguous(), group=self.col_group)
        return out

    def reduce_scatter_row(self, planes: torch.Tensor) -> torch.Tensor:
        """planes [C, ...] -> sum over the row group of plane c (this rank's column index)."""
        if self.C == 1:
            return planes[0]
        out = torch.empty(planes.shape[1:], dtype=planes.dtype, device=planes.device)
        dist.reduce_scatter_tensor(out, planes.contiguous(), group=self.row_group)
        return out

    def reduce_scatter_col(self, planes: torch.Tensor) -> torch.Tensor:
        if self.R == 1:
            return planes[0]
        out = torch.empty(planes.shape[1:], dtype=planes.dtype, device=planes.device)
        dist.reduce_scatter_tensor(out, planes.contiguous(), group=self.col_group)
        return out

    # -- into pre-allocated outputs (graph-capture friendly; used by the fused model path) --
    def ag_row_into(self, out: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
        if self.C == 1:
            out.view(-1).copy_(x.reshape(-1))
        else:
            dist.all_gather_into_tensor(out.view(-1), x.reshape(-1), group=self.row_group)
        return out

    def ag_col_into(self, out: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
        if self.R == 1:
            out.view(-1).copy_(x.reshape(-1))
        else:
            dist.all_gather_into_tensor(out.view(-1), x.reshape(-1), group=self.col_group)
        return out

    def rs_row_into(self, out: torch.Tensor, planes: torch.Tensor) -> torch.Tensor:
        dist.reduce_scatter_tensor(out.view(-1), planes.reshape(-1), group=self.row_group)
        return out

    def rs_col_into(self, out: torch.Tensor, planes: torch.Tensor) -> torch.Tensor:
        dist.reduce_scatter_tensor(out.view(-1), planes.reshape(-1), group=self.col_group)
        return out

    def all_reduce_all(self, x: torch.Tensor) -> torch.Tensor:
        if self.n > 1:
            dist.all_reduce(x, group=self.mp_group)
        return x

    def all_reduce_dp_mean(self, x: torch.Tensor) -> torch.Tensor:
        """dp_reduce: mean of this shard's gradient over the replicas holding
        the same shard; a no-op for a single replica."""
        if self.dp_replicas > 1:
            dist.all_reduce(x, group=self.dp_group)
            x.mul_(1.0 / self.dp_replicas)
        return x

    def all_reduce_row(self, x: torch.Tensor) -> torch.Tensor:
        if self.C > 1:
            dist.all_reduce(x, group=self.row_group)
        return x

    def all_reduce_col(self, x: torch.Tensor) -> torch.Tensor:
        if self.R > 1:
            dist.all_reduce(x, group=self.col_group)
        return x


# ----------------------------------------------------------------------------- primitives
def _check_dtypes(name, a, b):
    if a.dtype != b.dtype:
        raise ShapeError(f"{name} dtype mismatch: {a.dtype} vs {b.dtype}")


def _split_even(size: int, parts: int, what: str) -> int:
    if size % parts:
        raise ShapeError(f"{what} of size {size} cannot split in {parts}; pad the global tensor first")
    return size // parts


def pnt(ctx: MpContext, a: torch.Tensor, b: torch.Tensor, *, a_is_param: bool = False,
        b_is_param: bool = False) -> torch.Tensor:
    """Collective C = A B^T on block operands (parallel.py:107-116).

    Rank (r, c) holds A(r, c) [..., m/R, k/C] and B(r, c) [n/R, k/C] (trailing two dims;
    n = 2 splits only the last dim) and returns C(r, c) [..., m/R, n/C].
    """
    _check_dtypes("pnt", a, b)
    if ctx.n == 1:
        out = T.matmul(a, b, MatmulMode.NT)
        ctx._count(out.shape[-2], out.shape[-1], a.shape[-1], out[..., 0, 0].numel())
        return out
    # gather B's rows (all n) for this column block
    b_col = ctx.all_gather_col(b)                          # [R, n/R, k/C]
    b_panel = b_col.reshape(-1, b.shape[-1])               # [n, k/C]
    n_total = b_panel.shape[0]
    _split_even(n_total, ctx.C, "pnt output dimension")
    part = T.matmul(a, b_panel, MatmulMode.NT)             # [..., m/R, n] partial over k/C
    ctx._count(part.shape[-2], part.shape[-1], a.shape[-1], part[..., 0, 0].numel())
    planes = torch.stack(part.split(n_total // ctx.C, dim=-1))  # [C, ..., m/R, n/C]
    return ctx.reduce_scatter_row(planes)


def pnn(ctx: MpContext, a: torch.Tensor, b: torch.Tensor, *, a_is_param: bool = False,
        b_is_param: bool = False) -> torch.Tensor:
    """Collective C = A B (parallel.py:189-198): rank holds A(r,c) [m/R, k/C], B(r,c) [k/R, n/C]."""
    _check_dtypes("pnn", a, b)
    if ctx.n == 1:
        out = T.matmul(a, b, MatmulMode.NN)
        ctx._count(out.shape[-2], out.shape[-1], a.shape[-1], out[..., 0, 0].numel())
        return out
    # A B = A (B^T)^T: transpose-gather B so the column split of the product is over n.
    # Gather B over the column group -> B(:, c) = rows k (all), cols n/C (this column block).
    b_full_k = ctx.all_gather_col(b).reshape(-1, b.shape[-1])      # [k, n/C]
    # A's k-columns are split over the row group: gather them -> A(r, :) [m/R, k]
    a_row = ctx.all_gather_row(a)                                    # [C, ..., m/R, k/C]
    a_full = torch.cat(list(a_row), dim=-1)                          # [..., m/R, k]
    out = T.matmul(a_full, b_full_k, MatmulMode.NN)
    ctx._count(out.shape[-2], out.shape[-1], a_full.shape[-1], out[..., 0, 0].numel())
    return out


def ptn(ctx: MpContext, a: torch.Tensor, b: torch.Tensor, *, a_is_param: bool = False,
        b_is_param: bool = False) -> torch.Tensor:
    """Collective C = A^T B (parallel.py:276-285): rank holds A(r,c) [p/R, q/C], B(r,c) [p/R, s/C];
    returns C(r, c) [q/R, s/C]."""
    _check_dtypes("ptn", a, b)
    if ctx.n == 1:
        out = T.matmul(a, b, MatmulMode.TN)
        ctx._count(out.shape[-2], out.shape[-1], a.shape[-2], out[..., 0, 0].numel())
        return out
    a_row = ctx.all_gather_row(a)                                    # [C, ..., p/R, q/C]
    a_full = torch.cat(list(a_row), dim=-1)                          # [..., p/R, q]
    part = T.matmul(a_full, b, MatmulMode.TN)                        # [..., q, s/C] partial over p/R
    ctx._count(part.shape[-2], part.shape[-1], a_full.shape[-2], part[..., 0, 0].numel())
    q = part.shape[-2]
    _split_even(q, ctx.R, "ptn output rows")
    planes = torch.stack(part.split(q // ctx.R, dim=-2))            # [R, ..., q/R, s/C]
    return ctx.reduce_scatter_col(planes)


PRIMITIVES = {MatmulMode.NT: pnt, MatmulMode.NN: pnn, MatmulMode.TN: ptn}


# ----------------------------------------------------------------------------- analytic volume
def _lead(shape) -> int:
    return int(np.prod(shape[:-2], dtype=np.int64)) if len(shape) > 2 else 1


def primitive_send_elements(mode, n: int, a_shape, b_shape) -> list[int]:
    """Elements the REFERENCE schedule sends per position (parallel.py:361-401)."""
    mode = MatmulMode(mode)
    la, lb = _lead(a_shape), _lead(b_shape)
    lc = max(la, lb)
    if n == 1:
        return [0]
    if n not in (2, 4):
        raise ValueError("the reference schedules exist for n = 2 and 4 only")
    if mode is MatmulMode.NT:
        m, k, no = a_shape[-2], a_shape[-1], b_shape[-2]
        if n == 2:
            return [la * m * (no // 2)] * 2
        raw = lb * (no // 2) * (k // 2) + la * (m // 2) * (k // 2)
        part = 2 * lc * (m // 2) * (no // 2)
        return [raw, part, part, raw]
    if mode is MatmulMode.NN:
        m, k, no = a_shape[-2], a_shape[-1], b_shape[-1]
        if n == 2:
            return [la * m * (k // 2)] * 2
        a_blk, b_blk, part = la * (m // 2) * (k // 2), lb * (k // 2) * (no // 2), lc * (m // 2) * (no // 2)
        return [a_blk + b_blk, a_blk + part, a_blk + part, b_blk + a_blk]
    p, q, s = a_shape[-2], a_shape[-1], b_shape[-1]
    if n == 2:
        return [la * p * (q // 2)] * 2
    a_blk, b_blk, part = la * (p // 2) * (q // 2), lb * (p // 2) * (s // 2), 2 * lc * (q // 2) * (s // 2)
    return [a_blk + b_blk, part, part, b_blk + a_blk]


@dataclass
class CommVolumeReport:
    """Per-rank element counts for one sharded linear layer (parallel.py:404-427)."""

    n_way: int
    mode: MatmulMode
    forward_sent: list[int]
    backward_sent: list[int]

    @property
    def forward_total(self) -> int:
        return sum(self.forward_sent)

    @property
    def backward_total(self) -> int:
        return sum(self.backward_sent)

    @property
    def total_sent(self) -> int:
        return self.forward_total + self.backward_total

    @property
    def total_received(self) -> int:
        return self.total_sent


def comm_volume(m: int, k: int, n_out: int, n_way: int, mode=MatmulMode.NT, batch: int = 1) -> CommVolumeReport:
    """Analytic transfer counts of the reference schedules for one linear layer (parallel.py:430-462)."""
    if min(m, k, n_out) <= 0:
        raise ValueError(f"layer dims must be positive, got {(m, k, n_out)}")
    mode = MatmulMode(mode)

    def vs(a, b):
        return [x + y for x, y in zip(a, b)]

    if mode is MatmulMode.NT:
        x, w, y = (batch, m, k), (n_out, k), (batch, m, n_out)
        fwd = primitive_send_elements(mode, n_way, x, w)
        bwd = vs(primitive_send_elements(MatmulMode.NN, n_way, y, w), primitive_send_elements(MatmulMode.TN, n_way, y, x))
    elif mode is MatmulMode.NN:
        x, w, y = (batch, m, k), (k, n_out), (batch, m, n_out)
        fwd = primitive_send_elements(mode, n_way, x, w)
        bwd = vs(primitive_send_elements(MatmulMode.NT, n_way, y, w), primitive_send_elements(MatmulMode.TN, n_way, x, y))
    else:
        x, w, y = (batch, m, k), (m, n_out), (batch, k, n_out)
        fwd = primitive_send_elements(mode, n_way, x, w)
        bwd = vs(primitive_send_elements(MatmulMode.NT, n_way, w, y), primitive_send_elements(MatmulMode.NN, n_way, x, y))
    return CommVolumeReport(n_way, mode, fwd, bwd)
