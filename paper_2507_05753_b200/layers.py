"""Reference layer API over the sm_100a kernels: ShardedLinear, ShardedLayerNorm, MixerBlock.

Layer objects with the reference's constructors, `forward(x) -> (y, cache)` and
`backward(cache, g) -> gx` contracts, gradients accumulated in place into `Param.grad`:

  ShardedLinear(ctx, weight, bias, mode, weight_first)   parallel.py:496-549
  ShardedLayerNorm(ctx, gamma, beta, c_total, eps)       model.py:200-250
  MixerBlock(ctx, ln1, tok1, tok2, ln2, ch1, ch2, dropout_rate, rng)   model.py:253-297

They run one operation at a time through the collective primitives (parallel.pnt / pnn / ptn:
tcgen05 GEMMs + NCCL gather / reduce-scatter on the R x C grid) and the row-wise kernels
(layer-norm moments / apply / backward, GELU, bias add and bias-gradient sums), so a caller of
the reference's layer API can drop them in. The training step does NOT use them: it runs the
fused per-block schedule of model.py / jigsaw_grid.py (epilogue fusions, NVLink peer stores,
one CUDA graph), which computes the same functions; tests/test_layers_* check both against the
oracle.

Layouts are the model's (jigsaw_grid.py docstring): activations [..., T_r, E/C], tok1 output
[..., E/R, d_tok/C]; the layer-norm's normalised axis is split over the row group, whose
moments are all-reduced (the reference's stats_peer exchange, model.py:220-231).
"""
from __future__ import annotations

import torch

from . import _lib
from . import kernels as K
from .errors import ConfigError, ShapeError
from .parallel import PRIMITIVES, MpContext, pnn, pnt, ptn
from .params import Param
from .tensor import MatmulMode


def _operand(p: Param, dtype: torch.dtype) -> torch.Tensor:
    """The parameter as a GEMM operand of the activations' dtype (bf16 copy or fp32 master)."""
    if p.op is not None and p.op.dtype == dtype:
        return p.op
    return p.data if p.data.dtype == dtype else p.data.to(dtype)


def _rows(x: torch.Tensor) -> int:
    r = 1
    for s in x.shape[:-1]:
        r *= s
    return r


def _flatten_lead(arr: torch.Tensor) -> torch.Tensor:
    """Sum away broadcast batch dims so weight grads stay 2-D (parallel.py:552-556)."""
    return arr if arr.dim() == 2 else arr.sum(dim=tuple(range(arr.dim() - 2)))


class ShardedLinear:
    """Linear layer whose weight and bias exist only as this rank's blocks (parallel.py:496-549).

    mode NT computes y = x W^T, NN y = x W, TN y = x^T W. weight_first=True (NT only) computes
    y = W x^T with a row bias (the second token-mixing linear)."""

    def __init__(self, ctx: MpContext, weight: Param, bias: Param | None, mode=MatmulMode.NT,
                 weight_first: bool = False):
        if weight_first and MatmulMode(mode) is not MatmulMode.NT:
            raise ValueError("weight_first is only defined for NT layers")
        self.ctx, self.weight, self.bias = ctx, weight, bias
        self.mode = MatmulMode(mode)
        self.weight_first = weight_first

    def _add_bias(self, y: torch.Tensor) -> torch.Tensor:
        """y + bias (column bias, or row bias for weight_first), one jg_epilogue launch."""
        rows, n = y.shape[-2], y.shape[-1]
        batch = _rows(y) // rows
        out = torch.empty_like(y)
        if self.weight_first:
            K.epilogue(y, rows, n, batch=batch, acc_bs=rows * n, epi=_lib.EPI_BIAS_ROW, d=out, d_bs=rows * n,
                       bias=self.bias.data)
        else:
            K.epilogue(y, batch * rows, n, epi=_lib.EPI_BIAS_COL, d=out, bias=self.bias.data)
        return out

    def forward(self, x: torch.Tensor):
        w = _operand(self.weight, x.dtype)
        if self.weight_first:
            y = pnt(self.ctx, w, x, a_is_param=True)
        else:
            y = PRIMITIVES[self.mode](self.ctx, x, w, b_is_param=True)
        if self.bias is not None:
            y = self._add_bias(y)
        return y, x

    def _bias_grad(self, g: torch.Tensor, row: bool) -> None:
        gb = self.bias.grad if self.bias.grad is not None else torch.zeros_like(self.bias.data)
        self.bias.grad = gb
        g = g.contiguous()
        rows, n = g.shape[-2], g.shape[-1]
        if row:  # sum over everything but axis -2 (parallel.py:536, 559-561)
            for gi in g.reshape(-1, rows, n):
                K.rowsum(gi, gb, rows, n)
        else:
            K.colsum(g, gb, _rows(g), n)

    def backward(self, cache, g: torch.Tensor) -> torch.Tensor:
        x, ctx = cache, self.ctx
        w = _operand(self.weight, g.dtype)
        if self.weight_first:
            self.weight.add_grad(_flatten_lead(pnn(ctx, g, x)).to(self.weight.data.dtype))
            gx = ptn(ctx, g, w, b_is_param=True)
            if self.bias is not None:
                self._bias_grad(g, row=True)
            return gx
        if self.mode is MatmulMode.NT:
            gx = pnn(ctx, g, w, b_is_param=True)
            gw = ptn(ctx, g, x)
        elif self.mode is MatmulMode.NN:
            gx = pnt(ctx, g, w, b_is_param=True)
            gw = ptn(ctx, x, g)
        else:  # TN
            gx = pnt(ctx, w, g, a_is_param=True)
            gw = pnn(ctx, x, g)
        self.weight.add_grad(_flatten_lead(gw).to(self.weight.data.dtype))
        if self.bias is not None:
            self._bias_grad(g, row=False)
        return gx


class ShardedLayerNorm:
    """Last-axis layer norm whose normalised axis may be split over the row group (model.py:200-250).

    forward(x fp32) -> (y, cache); backward(cache, g fp32) -> dx, accumulating gamma / beta
    gradients. Row moments (sum x, sum x^2) and the backward's (sum g*gamma, sum g*gamma*xhat)
    are all-reduced over the row group — the grid form of the reference's stats_peer."""

    def __init__(self, ctx: MpContext, gamma: Param, beta: Param, c_total: int, eps: float = 1e-5,
                 out_dtype: torch.dtype | None = None):
        if eps <= 0:
            raise ValueError(f"layer_norm eps must be > 0, got {eps}")
        self.ctx, self.gamma, self.beta, self.c_total, self.eps = ctx, gamma, beta, c_total, eps
        self.out_dtype = out_dtype
        self.stats_peer = None if ctx.n == 1 or ctx.C == 1 else [r for r in ctx.row_ranks if r != ctx.comm.rank]

    def forward(self, x: torch.Tensor):
        if x.dtype != torch.float32:
            raise ShapeError("ShardedLayerNorm input must be float32 (the residual stream)")
        x = x.contiguous()
        rows, cols = _rows(x), x.shape[-1]
        stats = torch.zeros((rows, 2), dtype=torch.float32, device=x.device)
        K.ln_moments(x, stats, rows, cols)
        self.ctx.all_reduce_row(stats)
        y = torch.empty(x.shape, dtype=self.out_dtype or x.dtype, device=x.device)
        mr = torch.empty((rows, 2), dtype=torch.float32, device=x.device)
        K.ln_apply(x, stats, self.gamma.data, self.beta.data, y, mr, rows, cols, self.c_total, self.eps)
        return y, (x, mr)

    def backward(self, cache, g: torch.Tensor) -> torch.Tensor:
        x, mr = cache
        g = g.float().contiguous()
        rows, cols = _rows(x), x.shape[-1]
        bst = torch.zeros((rows, 2), dtype=torch.float32, device=x.device)
        K.ln_bwd_moments(x, g, self.gamma.data, mr, bst, rows, cols)
        self.ctx.all_reduce_row(bst)
        for p in (self.gamma, self.beta):
            if p.grad is None:
                p.grad = torch.zeros_like(p.data)
        dx = torch.empty_like(x)
        K.ln_bwd_apply(x, g, self.gamma.data, mr, bst, None, dx, None, self.gamma.grad, self.beta.grad, rows, cols,
                       self.c_total)
        return dx


def _gelu(x: torch.Tensor) -> torch.Tensor:
    y = torch.empty_like(x)
    K.gelu_fwd(x.contiguous(), y)
    return y


def _gelu_backward(x: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    dx = torch.empty_like(x)
    K.gelu_bwd(x.contiguous(), g.contiguous(), dx)
    return dx


class MixerBlock:
    """Token mixing then channel mixing, each pre-normed with a residual (model.py:253-297)."""

    def __init__(self, ctx: MpContext, ln1: ShardedLayerNorm, tok1: ShardedLinear, tok2: ShardedLinear,
                 ln2: ShardedLayerNorm, ch1: ShardedLinear, ch2: ShardedLinear, dropout_rate: float = 0.0, rng=None):
        if dropout_rate != 0.0:
            raise ConfigError("dropout_rate > 0 is not supported on the sm_100a path (the reference default is 0)")
        self.ctx = ctx
        self.ln1, self.tok1, self.tok2, self.ln2, self.ch1, self.ch2 = ln1, tok1, tok2, ln2, ch1, ch2
        self.dropout_rate, self.rng = dropout_rate, rng

    def forward(self, x: torch.Tensor):
        u, c_ln1 = self.ln1.forward(x)
        h, c_t1 = self.tok1.forward(u)          # x^T W: [B, E/R, d_tok/C] blocks
        ha = _gelu(h)
        o, c_t2 = self.tok2.forward(ha)         # W h^T: back to [B, T_r, E/C]
        x2 = x + o.float()
        v, c_ln2 = self.ln2.forward(x2)
        c, c_c1 = self.ch1.forward(v)
        ca = _gelu(c)
        z, c_c2 = self.ch2.forward(ca)
        y = x2 + z.float()
        return y, (c_ln1, c_t1, h, c_t2, c_ln2, c_c1, c, c_c2)

    def backward(self, cache, g: torch.Tensor) -> torch.Tensor:
        c_ln1, c_t1, h, c_t2, c_ln2, c_c1, c, c_c2 = cache
        od = h.dtype
        g_z = self.ch2.backward(c_c2, g.to(od))
        g_c = _gelu_backward(c, g_z)
        g_v = self.ch1.backward(c_c1, g_c)
        g_x2 = g + self.ln2.backward(c_ln2, g_v)
        g_o = self.tok2.backward(c_t2, g_x2.to(od))
        g_h = _gelu_backward(h, g_o)
        g_u = self.tok1.backward(c_t1, g_h)
        return g_x2 + self.ln1.backward(c_ln1, g_u)
