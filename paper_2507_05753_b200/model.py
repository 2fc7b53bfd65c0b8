"""WeatherMixer over Jigsaw tiles on B200 — reference model.py API, fused sm_100a execution.

Public surface (reference model.py): ModelConfig, ConfigError, token_sets, Layout,
WeatherMixerModel(ctx, cfg, seed=0, dtype=..., eps=1e-5) with forward(x_local, r=1),
backward(g_out_local), zero_grads(), grad_sync(), params / layouts, gather_global,
set_param_entry / get_param_entry, param_elements(), step_comm_volume(batch, r), local_grid.

Execution is not layer-object by layer-object: one step is a fixed sequence of fused kernels
over pre-allocated HBM workspaces (CUDA-graph capturable, see engine.TrainStep):

  forward, per block (model.py:268-282):
    ln_apply(x, stats1)                         -> u (GEMM operand), (mean, rstd)
    tok1  h = u^T W1 + b1, a = gelu(h)          one tcgen05 GEMM, bias + GELU epilogue
    tok2  x2 = x + W2 a^T + b2[:, None]         one GEMM, row bias + residual + LN2 moments
    ln_apply(x2, stats2)                        -> v
    ch1   c = v Wc1^T + bc1, ca = gelu(c)       one GEMM, bias + GELU epilogue
    ch2   y = x2 + ca Wc2^T + bc2               one GEMM, bias + residual + next LN1 moments
  backward, per block (model.py:284-297): 8 GEMMs (dX with GELU' epilogues, dW accumulating
  into fp32 gradients with the batch folded into K), two-phase layer-norm backward kernels,
  bias-gradient reductions.

dtype: "bf16" (bf16 GEMM operands, fp32 accumulate / residual stream / statistics /
gradients / optimiser) or "f32" (everything fp32; GEMMs in 3xTF32). f64 is rejected.

Jigsaw tiling (n = 2, 4, 8): rank (r, c) of the R x C grid holds activations
[B, T_r, E/C], weights as listed in Layout, and runs the gather / local-GEMM /
reduce-scatter schedule of parallel.py through NCCL on the compute stream.
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from . import kernels as K
from .config import ConfigError, ModelConfig, token_sets  # noqa: F401  (re-exported)
from .errors import ShapeError
from .params import FlatParams, Param
from .parallel import MpContext, comm_volume, primitive_send_elements
from .sharding import contiguous_split

KM, MN = _lib.JG_KMAJOR, _lib.JG_MNMAJOR
E_ACC, E_BCOL, E_BROW, E_RES = _lib.EPI_ACCUM, _lib.EPI_BIAS_COL, _lib.EPI_BIAS_ROW, _lib.EPI_RESID
E_GF, E_GB, E_CP, E_ST = _lib.EPI_GELU_FWD, _lib.EPI_GELU_BWD, _lib.EPI_COPY_D2, _lib.EPI_STATS
E_LNB = _lib.EPI_LNB

DTYPES = {"bf16": torch.bfloat16, "f32": torch.float32}


# ----------------------------------------------------------------------------------- layout
class Layout:
    """Maps one parameter's global tensor to local shards per mp position (model.py:124-197).

    Matrices: rows split R ways (row_sets), columns C ways (col_sets). Column vectors split C
    ways (duplicated over the column group), row vectors (tok2.b) split R ways (duplicated
    over the row group). n = 2 / 4 reproduce the reference exactly; n = 8 is the 4 x 2 grid.
    """

    def __init__(self, n: int, kind: str, shape: tuple[int, ...], row_sets=None, col_sets=None):
        from .sharding import grid_shape
        self.n, self.kind, self.shape = n, kind, shape
        self.R, self.C = grid_shape(n)
        self.row_sets, self.col_sets = row_sets, col_sets

    def _rc(self, pos):
        return pos // self.C, pos % self.C

    def local(self, global_arr: np.ndarray, pos: int) -> np.ndarray:
        if self.n == 1:
            return np.array(global_arr, copy=True)
        r, c = self._rc(pos)
        if self.kind == "matrix":
            out = global_arr
            if self.C > 1:
                out = out[:, self.col_sets[c]]
            if self.R > 1:
                out = out[self.row_sets[r], :]
            return np.ascontiguousarray(out)
        if self.kind == "vec_col":
            return np.ascontiguousarray(global_arr[self.col_sets[c]] if self.C > 1 else global_arr)
        return np.ascontiguousarray(global_arr[self.row_sets[r]] if self.R > 1 else global_arr)

    def place(self, out: np.ndarray, pos: int, local: np.ndarray) -> None:
        if self.n == 1:
            out[...] = local
            return
        r, c = self._rc(pos)
        if self.kind == "matrix":
            rows = self.row_sets[r] if self.R > 1 else np.arange(out.shape[0])
            cols = self.col_sets[c] if self.C > 1 else np.arange(out.shape[1])
            out[np.ix_(rows, cols)] = local
        elif self.kind == "vec_col":
            out[self.col_sets[c] if self.C > 1 else slice(None)] = local
        else:
            out[self.row_sets[r] if self.R > 1 else slice(None)] = local

    def dup_positions(self, pos: int) -> tuple[int, ...]:
        """Positions holding an identical copy (model.py:168-173, grid generalisation)."""
        if self.n == 1 or self.kind == "matrix":
            return ()
        r, c = self._rc(pos)
        if self.kind == "vec_col":
            return tuple(i * self.C + c for i in range(self.R)) if self.R > 1 else ()
        return tuple(r * self.C + j for j in range(self.C)) if self.C > 1 else ()

    def to_local_index(self, pos: int, idx: tuple[int, ...]):
        """Local index of a global entry on this position, or None (model.py:175-197)."""
        if self.n == 1:
            return idx
        r, c = self._rc(pos)

        def find(sets, part, v):
            hit = np.nonzero(sets[part] == v)[0]
            return int(hit[0]) if hit.size else None

        if self.kind == "matrix":
            li = idx[0] if self.R == 1 else find(self.row_sets, r, idx[0])
            lj = idx[1] if self.C == 1 else find(self.col_sets, c, idx[1])
            return None if li is None or lj is None else (li, lj)
        if self.kind == "vec_col":
            v = idx[0] if self.C == 1 else find(self.col_sets, c, idx[0])
        else:
            v = idx[0] if self.R == 1 else find(self.row_sets, r, idx[0])
        return None if v is None else (v,)


# ----------------------------------------------------------------------------------- model
class WeatherMixerModel:
    """Encoder, mixing-block stack, decoder and blend over local Jigsaw tiles (model.py:300-529)."""

    def __init__(self, ctx: MpContext, cfg: ModelConfig, seed: int = 0, dtype: str = "bf16",
                 eps: float = 1e-5, init: str = "reference", device=None, *, lat_real: int | None = None,
                 vars_real: int | None = None):
        """lat_real / vars_real: rows and channels of the unpadded data (e.g. 721 of 728 rows, 69 of
        70 channels at 0.25 deg). The loss gives padded rows / channels weight 0 and averages over
        B x lat_real x lon x vars_real. Default: nothing padded."""
        cfg.validate(ctx.n)
        if dtype not in DTYPES:
            raise ShapeError(f"dtype {dtype!r} not supported on sm_100a (use 'bf16' or 'f32'; f64 lives in oracle/)")
        if cfg.dropout_rate != 0.0:
            raise ConfigError("model.dropout_rate > 0 is not supported by the fused B200 path")
        if eps <= 0:
            raise ValueError(f"layer_norm eps must be > 0, got {eps}")
        self.ctx, self.cfg, self.seed, self.eps = ctx, cfg, seed, eps
        self.lat_real = cfg.grid[0] if lat_real is None else int(lat_real)
        self.vars_real = cfg.n_vars if vars_real is None else int(vars_real)
        if not (1 <= self.lat_real <= cfg.grid[0] and 1 <= self.vars_real <= cfg.n_vars):
            raise ConfigError(f"lat_real {self.lat_real} / vars_real {self.vars_real} outside the padded grid "
                              f"{cfg.grid[0]} rows x {cfg.n_vars} channels")
        self.dtype_name = dtype
        self.op_dtype = DTYPES[dtype]
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        n = ctx.n
        self.R, self.C, self.r, self.c = ctx.R, ctx.C, ctx.r, ctx.c
        # axis splits (model.py:316-321): strided longitude token sets, contiguous channel chunks
        self.t_sets = token_sets(cfg, self.R) if self.R > 1 else [np.arange(cfg.tokens)]
        split = lambda size, parts: contiguous_split(size, parts) if parts > 1 else [np.arange(size)]  # noqa: E731
        E, Kd, H, F = cfg.d_emb, cfg.d_tok, cfg.d_ch, cfg.patch_features
        self.sets = {
            "T": self.t_sets, "E_R": split(E, self.R), "E_C": split(E, self.C), "K_C": split(Kd, self.C),
            "H_R": split(H, self.R), "H_C": split(H, self.C), "F_R": split(F, self.R), "F_C": split(F, self.C),
            "V_C": split(cfg.n_vars, self.C),
        }
        self.layouts: dict[str, Layout] = {}
        self._specs = []  # (name, global_shape, fan_in, kind, row_sets, col_sets, lr_class, const)
        self._register_all()
        local_specs = []
        for name, gshape, _, kind, rs, cs, lr_class, _ in self._specs:
            lay = self.layouts[name]
            local_specs.append((name, self._local_shape(lay), lr_class, lay.dup_positions(ctx.pos), kind))
        self.flat = FlatParams(local_specs, self.device, self.op_dtype)
        self.params: dict[str, Param] = self.flat.params
        self._init(init)
        self._ws = None
        self._cache_valid = False

    # -- registration (model.py:336-389) --------------------------------------------------
    def _register_all(self):
        cfg, s, n = self.cfg, self.sets, self.ctx.n
        E, Kd, H, F, Tn, Cv = cfg.d_emb, cfg.d_tok, cfg.d_ch, cfg.patch_features, cfg.tokens, cfg.n_vars

        def weight(name, shape, fan_in, row_sets, col_sets, lr_class="body"):
            self.layouts[name] = Layout(n, "matrix", shape, row_sets, col_sets)
            self._specs.append((name, shape, fan_in, "matrix", row_sets, col_sets, lr_class, None))

        def vec(name, size, sets, kind, init=0.0, lr_class="body"):
            self.layouts[name] = Layout(n, kind, (size,), row_sets=sets if kind == "vec_row" else None,
                                        col_sets=sets if kind == "vec_col" else None)
            self._specs.append((name, (size,), None, kind, None, None, lr_class, init))

        weight("enc.w", (E, F), F, s["E_R"], s["F_C"], "encdec")
        vec("enc.b", E, s["E_C"], "vec_col", lr_class="encdec")
        for i in range(cfg.n_blocks):
            p = f"block{i}."
            vec(p + "ln1.gamma", E, s["E_C"], "vec_col", init=1.0)
            vec(p + "ln1.beta", E, s["E_C"], "vec_col")
            weight(p + "tok1.w", (Tn, Kd), Tn, s["T"], s["K_C"])
            vec(p + "tok1.b", Kd, s["K_C"], "vec_col")
            weight(p + "tok2.w", (Tn, Kd), Kd, s["T"], s["K_C"])
            vec(p + "tok2.b", Tn, s["T"], "vec_row")
            vec(p + "ln2.gamma", E, s["E_C"], "vec_col", init=1.0)
            vec(p + "ln2.beta", E, s["E_C"], "vec_col")
            weight(p + "ch1.w", (H, E), E, s["H_R"], s["E_C"])
            vec(p + "ch1.b", H, s["H_C"], "vec_col")
            weight(p + "ch2.w", (E, H), H, s["E_R"], s["H_C"])
            vec(p + "ch2.b", E, s["E_C"], "vec_col")
        weight("dec.w", (F, E), E, s["F_R"], s["E_C"], "encdec")
        vec("dec.b", F, s["F_C"], "vec_col", lr_class="encdec")
        vec("blend.w", Cv, s["V_C"], "vec_col", init=0.5)

    def _local_shape(self, lay: Layout):
        if lay.kind == "matrix":
            rows = lay.shape[0] // (self.R if lay.R > 1 else 1)
            cols = lay.shape[1] // (self.C if lay.C > 1 else 1)
            return (rows, cols)
        if lay.kind == "vec_col":
            return (lay.shape[0] // self.C,)
        return (lay.shape[0] // self.R,)

    def _init(self, mode: str):
        """Global init exactly as the reference draws it (model.py:312, 323-334), then sliced."""
        pos = self.ctx.pos
        if mode == "reference":
            rng = np.random.default_rng(self.seed)
            for name, shape, fan_in, kind, _, _, _, const in self._specs:
                if fan_in is not None:
                    bound = 1.0 / np.sqrt(fan_in)
                    glob = rng.uniform(-bound, bound, size=shape)
                else:
                    glob = np.full(shape, const)
                local = self.layouts[name].local(glob, pos).astype(np.float32)
                self.params[name].data.copy_(torch.from_numpy(local))
        elif mode == "fast":
            # device-side init with the reference's bounds (bench-scale models; not bit-exact)
            g = torch.Generator(device=self.device).manual_seed(self.seed * 1000003 + pos)
            for name, shape, fan_in, kind, _, _, _, const in self._specs:
                p = self.params[name].data
                if fan_in is not None:
                    bound = 1.0 / np.sqrt(fan_in)
                    p.uniform_(-bound, bound, generator=g)
                else:
                    p.fill_(const)
        else:
            raise ValueError(f"unknown init mode {mode!r}")
        self.sync_operand_copies()

    def sync_operand_copies(self):
        """Refresh the bf16 GEMM-operand copy of the master weights (after init / external edits).
        Collective in effect: every rank calls it, and `weights_version` (which tells a TrainStep
        that its optimiser-pushed weight panels are stale) advances on every rank."""
        if self.flat.op is not self.flat.master:
            K.cast_bf16(self.flat.master, self.flat.op)
        self.weights_version = getattr(self, "weights_version", 0) + 1

    # -- reference layer objects (model.py:336-389) -----------------------------------------
    def _layer_objects(self) -> dict:
        """encoder / blocks / decoder / blend as the reference exposes them: layer objects of
        layers.py over this model's Params (one op at a time; the training step instead runs
        the fused schedule below over the same Params)."""
        if getattr(self, "_layer_objs", None) is None:
            from .layers import MixerBlock, ShardedLayerNorm, ShardedLinear
            from .tensor import MatmulMode
            p, ctx, E = self.params, self.ctx, self.cfg.d_emb

            def ln(pre):
                return ShardedLayerNorm(ctx, p[pre + "gamma"], p[pre + "beta"], E, self.eps, out_dtype=self.op_dtype)

            blocks = []
            for i in range(self.cfg.n_blocks):
                b = f"block{i}."
                blocks.append(MixerBlock(
                    ctx, ln(b + "ln1."), ShardedLinear(ctx, p[b + "tok1.w"], p[b + "tok1.b"], MatmulMode.TN),
                    ShardedLinear(ctx, p[b + "tok2.w"], p[b + "tok2.b"], MatmulMode.NT, weight_first=True),
                    ln(b + "ln2."), ShardedLinear(ctx, p[b + "ch1.w"], p[b + "ch1.b"], MatmulMode.NT),
                    ShardedLinear(ctx, p[b + "ch2.w"], p[b + "ch2.b"], MatmulMode.NT), self.cfg.dropout_rate))
            self._layer_objs = {
                "encoder": ShardedLinear(ctx, p["enc.w"], p["enc.b"], MatmulMode.NT),
                "blocks": blocks,
                "decoder": ShardedLinear(ctx, p["dec.w"], p["dec.b"], MatmulMode.NT),
            }
        return self._layer_objs

    @property
    def encoder(self):
        return self._layer_objects()["encoder"]

    @property
    def blocks(self):
        return self._layer_objects()["blocks"]

    @property
    def decoder(self):
        return self._layer_objects()["decoder"]

    @property
    def blend(self) -> Param:
        return self.params["blend.w"]

    # -- introspection (model.py:462-529) -------------------------------------------------
    @property
    def local_grid(self) -> tuple[int, int]:
        lat, lon = self.cfg.grid
        return lat, lon // self.R

    @property
    def local_vars(self) -> int:
        return self.cfg.n_vars // self.C

    def param_elements(self) -> int:
        return sum(p.data.numel() for p in self.params.values())

    def gather_global(self, name: str, locals_by_pos: dict) -> np.ndarray:
        lay = self.layouts[name]
        out = np.zeros(lay.shape, dtype=np.float64)
        for pos, local in locals_by_pos.items():
            loc = local.detach().double().cpu().numpy() if isinstance(local, torch.Tensor) else np.asarray(local)
            lay.place(out, pos, loc)
        return out

    def set_param_entry(self, name: str, idx: tuple[int, ...], value: float) -> None:
        li = self.layouts[name].to_local_index(self.ctx.pos, idx)
        if li is not None:
            self.params[name].data[li] = value
        self.sync_operand_copies()  # every rank: keeps weights_version equal across ranks

    def get_param_entry(self, name, idx):
        li = self.layouts[name].to_local_index(self.ctx.pos, idx)
        return None if li is None else float(self.params[name].data[li])

    def step_flops(self, batch: int, r: int = 1) -> tuple[int, int]:
        """(forward, backward) GEMM FLOPs THIS rank executes per call, counted like the reference's
        MpContext._mm (2 * out.size * k per GEMM, parallel.py:65-69). Every rank of the balanced
        grid does exactly 1/n of them. The backward skips the encoder's input gradient, which the
        reference computes and discards (model.py:444-445): 2 T F E per sample fewer."""
        cfg, n = self.cfg, self.ctx.n
        T, F, E = cfg.tokens, cfg.patch_features, cfg.d_emb
        fwd = batch * (4 * T * F * E + r * cfg.n_blocks * 4 * T * E * (cfg.d_tok + cfg.d_ch))
        bwd = 2 * fwd - batch * 2 * T * F * E
        return fwd // n, bwd // n

    def step_comm_volume(self, batch: int, r: int = 1) -> int:
        """Elements the REFERENCE schedules send per fwd+bwd (model.py:483-529), for n = 1, 2, 4."""
        cfg, n = self.cfg, self.ctx.n
        if n == 1:
            return 0
        m_tok = batch * cfg.tokens

        def layer(m, k, n_out, mode):
            return comm_volume(m, k, n_out, n, mode).total_sent

        total = layer(m_tok, cfg.patch_features, cfg.d_emb, "NT")
        wb, hb, ob = (cfg.tokens, cfg.d_tok), (batch, cfg.d_emb, cfg.d_tok), (batch, cfg.tokens, cfg.d_emb)
        tok2 = (sum(primitive_send_elements("NT", n, wb, hb)) + sum(primitive_send_elements("NN", n, ob, hb))
                + sum(primitive_send_elements("TN", n, ob, wb)))
        per_block = (layer(m_tok, cfg.d_emb, cfg.d_tok, "TN") + tok2 + layer(m_tok, cfg.d_emb, cfg.d_ch, "NT")
                     + layer(m_tok, cfg.d_ch, cfg.d_emb, "NT"))
        total += r * cfg.n_blocks * per_block + layer(m_tok, cfg.d_emb, cfg.patch_features, "NT")
        rows = batch * cfg.tokens if n == 2 else batch * cfg.tokens // 2
        total += r * cfg.n_blocks * 2 * 2 * (rows * 2) * n
        for p in self.params.values():
            if len(p.dup_positions) > 1:
                total += p.data.numel() * n
        return total

    # -- workspace --------------------------------------------------------------------------
    def workspace(self, batch: int, r: int = 1):
        """Pre-allocated activations for (batch, rollout r); reused across steps."""
        if self._ws is not None and self._ws.key == (batch, r):
            return self._ws
        self._ws = _Workspace(self, batch, r)
        return self._ws

    # -- execution ----------------------------------------------------------------------------
    def zero_grads(self) -> None:
        self.flat.zero_grads()

    def forward(self, x: torch.Tensor, r: int = 1) -> torch.Tensor:
        """Forecast from a local sample block, applying the processor r times (model.py:406-426)."""
        if r < 1:
            raise ValueError(f"rollout length must be >= 1, got {r}")
        x = self._check_sample(x)
        ws = self.workspace(x.shape[0], r)
        ws.xin.copy_(x)
        self._forward(ws)
        out = torch.empty_like(ws.xin)
        self._blend(ws, out=out)
        self._cache_valid = True
        self.ctx.flops += self.step_flops(ws.B, r)[0]
        return out

    def backward(self, g_out: torch.Tensor) -> None:
        """Accumulate parameter gradients from dL/dout; call grad_sync() afterwards (model.py:428-445)."""
        if not self._cache_valid or self._ws is None:
            raise RuntimeError("backward called without a cached forward")
        self._cache_valid = False
        ws = self._ws
        g_out = self._check_sample(g_out)
        self._blend(ws, g_ext=g_out)
        self._backward(ws)
        self.ctx.flops += self.step_flops(ws.B, ws.r)[1]

    def grad_sync(self) -> None:
        """Sum gradients of duplicated vector parameters over their sharing group (model.py:451-460)."""
        if self.ctx.n == 1:
            return
        self._grad_sync()

    def _check_sample(self, x: torch.Tensor) -> torch.Tensor:
        lat, lon = self.local_grid
        if not isinstance(x, torch.Tensor) or x.dim() != 4 or tuple(x.shape[1:]) != (lat, lon, self.local_vars):
            raise ShapeError(f"expected a local sample [B, {lat}, {lon}, {self.local_vars}], got "
                             f"{tuple(x.shape) if isinstance(x, torch.Tensor) else type(x)}")
        return x.to(device=self.device, dtype=torch.float32).contiguous()

    # ======================================================================= kernels (n = 1)
    def _gemm(self, out, a, b, am, bm, m, n, k, *batch_args, **kw):
        K.gemm(out, a, b, am, bm, m, n, k, *batch_args, **kw)

    def _forward(self, ws: "_Workspace") -> None:
        if self.ctx.n > 1:
            return self._forward_grid(ws)
        cfg, p, B = self.cfg, self.params, ws.B
        Tn, E, F, Kd, H = cfg.tokens, cfg.d_emb, cfg.patch_features, cfg.d_tok, cfg.d_ch
        lat, lon = self.local_grid
        M = B * Tn
        K.zero(ws.stats)
        K.patchify(ws.xin, ws.xp, B, lat, lon, cfg.n_vars, cfg.patch[0], cfg.patch[1])
        # encoder: res0 = xp Wenc^T + benc, with LN1 moments of block 0
        self._gemm(ws.res[0], ws.xp, p["enc.w"].op, KM, KM, M, E, F, epi=E_BCOL | E_ST,
                   bias=p["enc.b"].data, stats=ws.st1[0])
        nj = ws.r * cfg.n_blocks
        for j in range(nj):
            b = f"block{j % cfg.n_blocks}."
            x = ws.res[j]
            K.ln_apply(x, ws.st1[j], p[b + "ln1.gamma"].data, p[b + "ln1.beta"].data, ws.u[j], ws.mr1[j], M, E, E,
                       self.eps)
            # tok1 (TN, per sample): h = u^T W1 + b1 ; a = gelu(h)
            self._gemm(ws.h[j], ws.u[j], p[b + "tok1.w"].op, MN, MN, E, Kd, Tn, B, Tn * E, 0,
                       epi=E_BCOL | E_GF, bias=p[b + "tok1.b"].data, d2=ws.a[j])
            # tok2 (weight-first NT): x2 = x + W2 a^T + b2[:, None] ; LN2 moments
            self._gemm(ws.x2[j], p[b + "tok2.w"].op, ws.a[j], KM, KM, Tn, E, Kd, B, 0, E * Kd,
                       epi=E_BROW | E_RES | E_ST, bias=p[b + "tok2.b"].data, resid=x, stats=ws.st2[j],
                       stats_bs=2 * Tn)
            K.ln_apply(ws.x2[j], ws.st2[j], p[b + "ln2.gamma"].data, p[b + "ln2.beta"].data, ws.v[j], ws.mr2[j],
                       M, E, E, self.eps)
            # ch1: c = v Wc1^T + bc1 ; ca = gelu(c)
            self._gemm(ws.c[j], ws.v[j], p[b + "ch1.w"].op, KM, KM, M, H, E, epi=E_BCOL | E_GF,
                       bias=p[b + "ch1.b"].data, d2=ws.ca[j])
            # ch2: y = x2 + ca Wc2^T + bc2 ; next LN1 moments (or the decoder operand copy)
            last = j == nj - 1
            copy_y = last and ws.y_op is not ws.res[nj]
            self._gemm(ws.res[j + 1], ws.ca[j], p[b + "ch2.w"].op, KM, KM, M, E, H,
                       epi=E_BCOL | E_RES | (E_CP if copy_y else 0) | (0 if last else E_ST),
                       bias=p[b + "ch2.b"].data, resid=ws.x2[j],
                       stats=None if last else ws.st1[j + 1], d2=ws.y_op if copy_y else None)
        # decoder: d = y Wdec^T + bdec (token layout, fp32)
        self._gemm(ws.dec, ws.y_op, p["dec.w"].op, KM, KM, M, F, E, epi=E_BCOL, bias=p["dec.b"].data)

    def _blend(self, ws, out=None, g_ext=None, target=None, loss=None, loss_scale=1.0):
        """Decoder tail: unpatchify + blend (+ loss and its gradient, or an external gradient)."""
        cfg = self.cfg
        lat, lon = self.local_grid
        bw = self.params["blend.w"]
        want_grad = g_ext is not None or target is not None
        gd, hd = (ws.gd if want_grad else None), None
        if want_grad and self.ctx.n > 1 and self.C > 1:
            # Jigsaw: the decoder-output gradient goes straight into the row group's gather slot
            # (own plane + peer planes, stored by this kernel) for the decoder's backward GEMMs
            from .jigsaw_grid import _gw
            g = _gw(self, ws)
            hd = g.row.dest((ws.B * ws.Tl, ws.Fl), self.op_dtype, slot="gd")
            gd = hd.own.view(ws.gd.shape)
        K.blend_loss(ws.dec, ws.xin, target, bw.data, ws.lat_w, ws.var_w, g_ext, out, loss,
                     bw.grad if want_grad else None, gd, ws.B, lat, lon, self.local_vars,
                     cfg.patch[0], cfg.patch[1], ws.inv_count, loss_scale, bcast=hd.peers if hd is not None else None)
        if hd is not None:
            g.row.publish(hd)
        ws.gd_row = hd

    # -- weight-gradient sink ---------------------------------------------------------------
    def _wgrad(self, name):
        """(out, epilogue kwargs) for the GEMM producing weight `name`'s complete gradient.

        Normally the gradient accumulates into Param.grad (reference add_grad, parallel.py:490-493).
        Inside TrainStep with fused Adam (rollout 1: each weight gets exactly one gradient GEMM)
        the GEMM epilogue applies Adam to the master weight directly (JG_EPI_ADAM) and the
        gradient never touches HBM; the caller orders every dX GEMM before its dW GEMM.
        """
        p = self.params[name]
        fa = getattr(self, "_fused_adam", None)
        if fa is None:
            # inside TrainStep (rollout 1) each weight's gradient comes from exactly one GEMM:
            # overwrite (TMA-store epilogue) instead of read-modify-write, no zeroing needed
            return p.grad, {"epi": 0 if getattr(self, "_grad_overwrite", False) else E_ACC}
        step, cfg = fa
        f = self.flat
        return p.data, {"epi": _lib.EPI_ADAM, "adam": (f.view(name, f.m), f.view(name, f.v),
                                                      None if f.op is f.master else p.op, step, cfg.lr(p.lr_class),
                                                      cfg.beta1, cfg.beta2, cfg.eps)}

    def _wgrad_reduced(self, name, red):
        """Sink for a weight gradient that arrived reduced (NCCL reduce-scatter) in `red`."""
        p = self.params[name]
        fa = getattr(self, "_fused_adam", None)
        if fa is None:
            if getattr(self, "_grad_overwrite", False):
                K.sum_planes(p.grad, red, p.grad.numel(), 1, 0)
            else:
                K.sum_planes(p.grad, red, p.grad.numel(), 1, 0, accumulate=True)
            return
        step, cfg = fa
        f = self.flat
        K.adam(p.data, red, f.view(name, f.m), f.view(name, f.v), None if f.op is f.master else p.op,
               p.data.numel(), cfg.lr(p.lr_class), cfg.beta1, cfg.beta2, cfg.eps, step)

    def _backward(self, ws: "_Workspace") -> None:
        if self.ctx.n > 1:
            return self._backward_grid(ws)
        cfg, p, B = self.cfg, self.params, ws.B
        Tn, E, F, Kd, H = cfg.tokens, cfg.d_emb, cfg.patch_features, cfg.d_tok, cfg.d_ch
        M = B * Tn
        K.zero(ws.bstats)
        # decoder (NT): g = gd Wdec ; dW += gd^T y ; db += sum gd
        g, g_op = ws.g, ws.g_op
        self._gemm(g, ws.gd, p["dec.w"].op, KM, MN, M, E, F, epi=0 if g_op is g else E_CP,
                   d2=None if g_op is g else g_op)
        out, kw = self._wgrad("dec.w")
        self._gemm(out, ws.gd, ws.y_op, MN, MN, F, E, M, **kw)
        K.colsum(ws.gd, p["dec.b"].grad, M, F)
        nj = ws.r * cfg.n_blocks
        for j in reversed(range(nj)):
            b = f"block{j % cfg.n_blocks}."
            # ch2: gc = (g Wc2) * gelu'(c) ; dWc2 += g^T ca ; dbc2 += sum g
            self._gemm(ws.gc, g_op, p[b + "ch2.w"].op, KM, MN, M, H, E, epi=E_GB, pre=ws.c[j])
            out, kw = self._wgrad(b + "ch2.w")
            self._gemm(out, g_op, ws.ca[j], MN, MN, E, H, M, **kw)
            if j == nj - 1:  # (later blocks get this column sum from the LN1-backward pass below)
                K.colsum(g, p[b + "ch2.b"].grad, M, E)
            # ch1: gv = gc Wc1 ; dWc1 += gc^T v ; dbc1 += sum gc
            # (epilogue: LN2-backward row moments of gv, so _ln_bwd needs only its apply pass)
            self._gemm(ws.gv, ws.gc, p[b + "ch1.w"].op, KM, MN, M, E, H, epi=E_LNB, stats=ws.bst2[j],
                       lnb=(ws.x2[j], p[b + "ln2.gamma"].data, ws.mr2[j]))
            out, kw = self._wgrad(b + "ch1.w")
            self._gemm(out, ws.gc, ws.v[j], MN, MN, H, E, M, **kw)
            K.colsum(ws.gc, p[b + "ch1.b"].grad, M, H)
            # ln2 backward + residual: g_x2 = g + LN2'(gv)
            # (same pass: tok2's row-bias gradient = row sums of g_x2, folded over the B samples)
            self._ln_bwd(ws.x2[j], ws.gv, b + "ln2.", ws.mr2[j], ws.bst2[j], g, ws.gx2, ws.gx2_op, M, E,
                         moments=False, sums=dict(rowsum=p[b + "tok2.b"].grad, rowsum_period=Tn))
            # tok2 (weight-first): gh = (g_x2^T W2) * gelu'(h) ; dW2 += sum_b g_x2 a ; db2 += row sums
            self._gemm(ws.gh, ws.gx2_op, p[b + "tok2.w"].op, MN, MN, E, Kd, Tn, B, Tn * E, 0, epi=E_GB, pre=ws.h[j])
            out, kw = self._wgrad(b + "tok2.w")
            self._gemm(out, ws.gx2_op, ws.a[j], KM, MN, Tn, Kd, E, B, Tn * E, E * Kd, reduce_batch=True, **kw)
            K.colsum(ws.gh, p[b + "tok1.b"].grad, B * E, Kd)
            # tok1 (TN): gu = W1 gh^T ; dW1 += sum_b u gh
            self._gemm(ws.gu, p[b + "tok1.w"].op, ws.gh, KM, KM, Tn, E, Kd, B, 0, E * Kd, epi=E_LNB,
                       stats=ws.bst1[j], lnb=(ws.res[j], p[b + "ln1.gamma"].data, ws.mr1[j]))
            out, kw = self._wgrad(b + "tok1.w")
            self._gemm(out, ws.u[j], ws.gh, KM, MN, Tn, Kd, E, B, Tn * E, E * Kd, reduce_batch=True, **kw)
            # ln1 backward + residual: g = g_x2 + LN1'(gu)
            # (same pass: the column sums of g = the bias gradient of the next layer down — the
            # previous block's ch2, or the encoder)
            nxt = f"block{(j - 1) % cfg.n_blocks}.ch2.b" if j > 0 else "enc.b"
            self._ln_bwd(ws.res[j], ws.gu, b + "ln1.", ws.mr1[j], ws.bst1[j], ws.gx2, g, g_op, M, E, moments=False,
                         sums=dict(colsum=p[nxt].grad))
            hook = getattr(self, "_after_block_bwd", None)
            if hook is not None:  # block j's weight gradients are complete (TrainStep: early Adam)
                hook(j)
        # encoder (NT): dWenc += g^T xp ; db += sum g (the input gradient is not needed, model.py:444-445)
        out, kw = self._wgrad("enc.w")
        self._gemm(out, g_op, ws.xp, MN, MN, E, F, M, **kw)

    def _ln_bwd(self, x, gin, pre, mr, bst, resid, out, out_op, rows, cols, c_total=None, row_reduce=None, bcast=None,
                moments=True, sums=None):
        """Two-phase layer-norm backward + residual add (model.py:242-250): row sums (all-reduced
        over the row group by `row_reduce` when the normalised axis is split), then apply.
        moments=False: the GEMM producing `gin` already accumulated them (JG_EPI_LNB)."""
        p = self.params
        c_total = c_total or cols
        if moments:
            K.ln_bwd_moments(x, gin, p[pre + "gamma"].data, mr, bst, rows, cols)
        if row_reduce is not None:
            row_reduce(bst)
        if out_op is not None and out_op is not out and out_op.dtype == torch.float32:
            # fp32 mode: the kernel's operand copy is bf16-only; copy (and push) the fp32 result
            K.ln_bwd_apply(x, gin, p[pre + "gamma"].data, mr, bst, resid, out, None, p[pre + "gamma"].grad,
                           p[pre + "beta"].grad, rows, cols, c_total, **(sums or {}))
            K.copy_async(out_op.data_ptr(), out, out.numel() * 4)
            for addr in bcast or []:
                K.copy_async(addr, out, out.numel() * 4)
            return
        K.ln_bwd_apply(x, gin, p[pre + "gamma"].data, mr, bst, resid, out, out_op, p[pre + "gamma"].grad,
                       p[pre + "beta"].grad, rows, cols, c_total, bcast=bcast, **(sums or {}))

    # grid paths are implemented in jigsaw_grid.py (bound below)
    def _forward_grid(self, ws):
        from .jigsaw_grid import forward_grid
        return forward_grid(self, ws)

    def _backward_grid(self, ws):
        from .jigsaw_grid import backward_grid
        return backward_grid(self, ws)

    def _grad_sync(self):
        from .jigsaw_grid import grad_sync
        return grad_sync(self)


class _Workspace:
    """All activations of one (batch, rollout) shape, allocated once in HBM."""

    def __init__(self, model: WeatherMixerModel, B: int, r: int):
        cfg, dev = model.cfg, model.device
        self.key, self.B, self.r = (B, r), B, r
        od = model.op_dtype
        f32 = dict(dtype=torch.float32, device=dev)
        opk = dict(dtype=od, device=dev)
        R, C = model.R, model.C
        Tl = cfg.tokens // R
        El, Kl, Hl, Fl = cfg.d_emb // C, cfg.d_tok // C, cfg.d_ch // C, cfg.patch_features // C
        Er = cfg.d_emb // R
        lat, lon = model.local_grid
        nv = model.local_vars
        nj = r * cfg.n_blocks
        M = B * Tl
        self.Tl, self.El, self.Kl, self.Hl, self.Fl, self.Er = Tl, El, Kl, Hl, Fl, Er
        self.xin = torch.empty((B, lat, lon, nv), **f32)
        self.xp = torch.empty((B, Tl, Fl), **opk)
        # statistics: one buffer, one memset per forward / backward
        self.stats = torch.zeros((2 * nj + 1, M, 2), **f32)
        self.st1 = [self.stats[2 * j] for j in range(nj + 1)]
        self.st2 = [self.stats[2 * j + 1] for j in range(nj)]
        self.mr = torch.zeros((2 * nj, M, 2), **f32)
        self.mr1 = [self.mr[2 * j] for j in range(nj)]
        self.mr2 = [self.mr[2 * j + 1] for j in range(nj)]
        self.bstats = torch.zeros((2 * nj, M, 2), **f32)
        self.bst1 = [self.bstats[2 * j] for j in range(nj)]
        self.bst2 = [self.bstats[2 * j + 1] for j in range(nj)]
        self.res = [torch.empty((B, Tl, El), **f32) for _ in range(nj + 1)]
        self.u = [torch.empty((B, Tl, El), **opk) for _ in range(nj)]
        # GELU pre-activations (kept only for GELU' in the backward): operand dtype, i.e. bf16 in
        # bf16 mode — half the epilogue stores and backward reads (JIGSAW_PRE_FP32=1 keeps fp32)
        prek = f32 if os.environ.get("JIGSAW_PRE_FP32", "0") == "1" else opk
        self.h = [torch.empty((B, Er, Kl), **prek) for _ in range(nj)]
        self.a = [torch.empty((B, Er, Kl), **opk) for _ in range(nj)]
        self.x2 = [torch.empty((B, Tl, El), **f32) for _ in range(nj)]
        self.v = [torch.empty((B, Tl, El), **opk) for _ in range(nj)]
        self.c = [torch.empty((B, Tl, Hl), **prek) for _ in range(nj)]
        self.ca = [torch.empty((B, Tl, Hl), **opk) for _ in range(nj)]
        self.y_op = self.res[nj] if od == torch.float32 else torch.empty((B, Tl, El), **opk)
        self.dec = torch.empty((B, Tl, Fl), **f32)
        # backward
        self.gd = torch.empty((B, Tl, Fl), **opk)
        self.g = torch.empty((B, Tl, El), **f32)
        self.g_op = self.g if od == torch.float32 else torch.empty((B, Tl, El), **opk)
        self.gx2 = torch.empty((B, Tl, El), **f32)
        self.gx2_op = self.gx2 if od == torch.float32 else torch.empty((B, Tl, El), **opk)
        self.gc = torch.empty((B, Tl, Hl), **opk)
        self.gv = torch.empty((B, Tl, El), **f32)
        self.gh = torch.empty((B, Er, Kl), **opk)
        self.gu = torch.empty((B, Tl, El), **f32)
        # loss weights over the local grid block (padded rows / channels weigh 0)
        from .train import lat_weights, var_weights
        lat_real, vars_real = model.lat_real, model.vars_real
        self.lat_w = torch.tensor(lat_weights(lat, lat_real), **f32)
        vw = var_weights(cfg.n_vars, vars_real)
        c0 = model.sets["V_C"][model.c][0] if C > 1 else 0
        self.var_w = torch.tensor(vw[c0:c0 + nv], **f32)
        self.inv_count = 1.0 / (B * lat_real * cfg.lon * vars_real)
        self.loss = torch.zeros(1, **f32)
