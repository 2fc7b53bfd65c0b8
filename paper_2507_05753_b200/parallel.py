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
        self.allreduce_bytes = 0.0  # ring all-reduce payload this rank sends (2 (G-1)/G per buffer)
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

    def _buf_acquire(self, size: int) -> None:
        """Live communication buffers holding parameter blocks, and their watermark (parallel.py:71-76)."""
        self.param_buffer_elements += size
        self.param_buffer_peak = max(self.param_buffer_peak, self.param_buffer_elements)

    def _buf_release(self, size: int) -> None:
        self.param_buffer_elements -= size

    # -- collectives on the grid axes (device tensors, current stream) --------
    def all_gather_row(self, x: torch.Tensor) -> torch.Tensor:
        """[C, *x.shape] stack of the row group's blocks (ordered by column index)."""
        out = torch.empty((self.C, *x.shape), dtype=x.dtype, device=x.device)
        if self.C == 1:
            out[0].copy_(x)
        else:
            dist.all_gather_into_tensor(out.view(-1), x.contiguous().view(-1), group=self.row_group)
        return out

    def all_gather_col(self, x: torch.Tensor) -> torch.Tensor:
        out = torch.empty((self.R, *x.shape), dtype=x.dtype, device=x.device)
        if self.R == 1:
            out[0].copy_(x)
        else:
            dist.all_gather_into_tensor(out.view(-1), x.contiguous().view(-1), group=self.col_group)
        return out

    def reduce_scatter_row(self, planes: torch.Tensor) -> torch.Tensor:
        """planes [C, ...] -> sum over the row group of plane c (this rank's column index)."""
        if self.C == 1:
            return planes[0]
        out = torch.empty(planes.shape[1:], dtype=planes.dtype, device=planes.device)
        dist.reduce_scatter_tensor(out.view(-1), planes.contiguous().view(-1), group=self.row_group)
        return out

    def reduce_scatter_col(self, planes: torch.Tensor) -> torch.Tensor:
        if self.R == 1:
            return planes[0]
        out = torch.empty(planes.shape[1:], dtype=planes.dtype, device=planes.device)
        dist.reduce_scatter_tensor(out.view(-1), planes.contiguous().view(-1), group=self.col_group)
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

    def _ar_count(self, G: int, x: torch.Tensor) -> None:
        self.allreduce_bytes += 2.0 * (G - 1) / G * x.numel() * x.element_size()

    def all_reduce_all(self, x: torch.Tensor) -> torch.Tensor:
        if self.n > 1:
            self._ar_count(self.n, x)
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
            self._ar_count(self.C, x)
            dist.all_reduce(x, group=self.row_group)
        return x

    def all_reduce_col(self, x: torch.Tensor) -> torch.Tensor:
        if self.R > 1:
            self._ar_count(self.R, x)
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


def _gather_axis(blocks: torch.Tensor, axis: int) -> torch.Tensor:
    """[G, *shape] stack of gathered blocks -> one tensor concatenated along `axis` (< 0) of shape."""
    g = blocks.shape[0]
    moved = blocks.movedim(0, blocks.dim() + axis - 1)  # G just before the target axis
    shape = list(blocks.shape[1:])
    shape[axis] *= g
    return moved.reshape(shape)


def _lead_pad(t: torch.Tensor, lead: int) -> torch.Tensor:
    """View with `lead` leading batch dims (singletons prepended) so plane-batched operands broadcast."""
    return t.reshape((1,) * (lead - (t.dim() - 2)) + tuple(t.shape))


def _count_out(ctx: MpContext, out_shape, k: int) -> None:
    """The reference's FLOP counter: 2 * out.size * k per local GEMM (parallel.py:65-69)."""
    n = 1
    for s in out_shape:
        n *= int(s)
    ctx.flops += 2 * n * int(k)


def _param_blocks(ctx: MpContext, gathered: torch.Tensor, own: torch.Tensor, is_param: bool):
    """Account received parameter blocks in the buffer watermark (parallel.py:71-76, 79-97)."""
    if is_param:
        ctx._buf_acquire(gathered.numel() - own.numel())
    return gathered.numel() - own.numel() if is_param else 0


def pnt(ctx: MpContext, a: torch.Tensor, b: torch.Tensor, *, a_is_param: bool = False,
        b_is_param: bool = False) -> torch.Tensor:
    """Collective C = A B^T on block operands (parallel.py:107-116).

    Rank (r, c) of the R x C grid holds A(r, c) [..., m/R, k/C] and B(r, c) [..., n/R, k/C] and
    returns C(r, c) [..., m/R, n/C] — for n = 2 (1 x 2) and n = 4 (2 x 2) exactly the reference's
    column-block / 2 x 2-block layouts (parallel.py:1-10). Schedule: all-gather B over the
    column group (B(:, c), all n rows), one local GEMM per output plane (partials over k/C),
    reduce-scatter the planes over the row group; every rank does 1/n of the FLOPs.
    """
    _check_dtypes("pnt", a, b)
    if ctx.n == 1:
        out = T.matmul(a, b, MatmulMode.NT)
        _count_out(ctx, out.shape, a.shape[-1])
        return out
    held = 0
    try:
        panel = _gather_axis(ctx.all_gather_col(b), -2) if ctx.R > 1 else b   # [..., n, k/C]
        held = _param_blocks(ctx, panel, b, b_is_param)
        n_c = _split_even(panel.shape[-2], ctx.C, "pnt output dimension")
        # planes [C, ..., m/R, n/C]: plane j = A B_panel[j-th n chunk]^T (broadcast batch, no copies)
        lead = max(a.dim(), panel.dim()) - 2
        pl = _lead_pad(panel, lead)
        bp = pl.reshape(*pl.shape[:-2], ctx.C, n_c, pl.shape[-1]).movedim(-3, 0)
        planes = T.matmul(_lead_pad(a, lead).unsqueeze(0), bp, MatmulMode.NT)
        _count_out(ctx, planes.shape, a.shape[-1])
        return ctx.reduce_scatter_row(planes)
    finally:
        ctx._buf_release(held)


def pnn(ctx: MpContext, a: torch.Tensor, b: torch.Tensor, *, a_is_param: bool = False,
        b_is_param: bool = False) -> torch.Tensor:
    """Collective C = A B (parallel.py:189-198): rank holds A(r, c) [..., m/R, k/C] and
    B(r, c) [..., k/R, n/C], returns C(r, c) [..., m/R, n/C]. Schedule: all-gather A over the
    row group (all k columns) and B over the column group (all k rows), one local GEMM."""
    _check_dtypes("pnn", a, b)
    if ctx.n == 1:
        out = T.matmul(a, b, MatmulMode.NN)
        _count_out(ctx, out.shape, a.shape[-1])
        return out
    held = 0
    try:
        b_full = _gather_axis(ctx.all_gather_col(b), -2) if ctx.R > 1 else b   # [..., k, n/C]
        held += _param_blocks(ctx, b_full, b, b_is_param)
        a_full = _gather_axis(ctx.all_gather_row(a), -1) if ctx.C > 1 else a   # [..., m/R, k]
        held += _param_blocks(ctx, a_full, a, a_is_param)
        out = T.matmul(a_full, b_full, MatmulMode.NN)
        _count_out(ctx, out.shape, a_full.shape[-1])
        return out
    finally:
        ctx._buf_release(held)


def ptn(ctx: MpContext, a: torch.Tensor, b: torch.Tensor, *, a_is_param: bool = False,
        b_is_param: bool = False) -> torch.Tensor:
    """Collective C = A^T B (parallel.py:276-285): rank holds A(r, c) [..., p/R, q/C] and
    B(r, c) [..., p/R, s/C], returns C(r, c) [..., q/R, s/C] (n = 2: the two q halves stacked,
    as _tn2). Schedule: all-gather A over the row group (all q columns), one local GEMM per
    output plane (partials over p/R), reduce-scatter the planes over the column group."""
    _check_dtypes("ptn", a, b)
    if ctx.n == 1:
        out = T.matmul(a, b, MatmulMode.TN)
        _count_out(ctx, out.shape, a.shape[-2])
        return out
    held = 0
    try:
        a_full = _gather_axis(ctx.all_gather_row(a), -1) if ctx.C > 1 else a   # [..., p/R, q]
        held = _param_blocks(ctx, a_full, a, a_is_param)
        q_r = _split_even(a_full.shape[-1], ctx.R, "ptn output rows")
        # planes [R, ..., q/R, s/C]: plane i = A_full[:, i-th q chunk]^T B
        lead = max(a_full.dim(), b.dim()) - 2
        af = _lead_pad(a_full, lead)
        ap = af.reshape(*af.shape[:-1], ctx.R, q_r).movedim(-2, 0)
        planes = T.matmul(ap, _lead_pad(b, lead).unsqueeze(0), MatmulMode.TN)
        _count_out(ctx, planes.shape, a_full.shape[-2])
        return ctx.reduce_scatter_col(planes)
    finally:
        ctx._buf_release(held)


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
