"""One WeatherMixer training step as a single CUDA graph (the hot path of BASELINE north_star).

    step = TrainStep(model, batch=1)
    loss = step(x_host, target_host)        # public API: host buffers in, host loss out
    step.run_device()                       # inputs already resident (bench `value` leg)

Per step, on one stream: zero gradients (one memset) -> fused forward -> fused blend +
lat-weighted MSE + its gradient (jg_blend_loss) -> fused backward -> gradient sync of
duplicated vectors (NCCL, n > 1) -> Adam, one fused kernel per lr class, writing the bf16
operand copies (jg_adam). The reference has no loss / optimiser; they follow SPEC.md:396-413
and 482-490 (see train.py).
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from . import kernels as K
from . import tensor as T
from .errors import ConfigError
from .model import WeatherMixerModel
from .train import AdamConfig


def split_push(lo: int, hi: int, segs, max_segs: int):
    """Split the Adam range [lo, hi) at panel-segment starts so that each jg_adam_push call
    carries at most `max_segs` segments (e.g. 12 blocks = 26 channel-mixing panels at R > 1).
    segs: [(start - lo, numel, addrs)]; yields (a0, a1, segments re-based to a0)."""
    segs = sorted(segs, key=lambda t: t[0])
    cuts = [lo] + [lo + segs[j][0] for j in range(max_segs, len(segs), max_segs)]
    for a0, a1 in zip(cuts, cuts[1:] + [hi]):
        yield a0, a1, [(st - (a0 - lo), n, addrs) for st, n, addrs in segs if a0 <= lo + st < a1]


class TrainStep:
    def __init__(self, model: WeatherMixerModel, batch: int = 1, r: int = 1, adam: AdamConfig | None = None,
                 graph: bool = True, loss_scale: float = 1.0, fused_adam: bool = False,
                 step_count: torch.Tensor | None = None):
        self.model, self.batch, self.r = model, batch, r
        # Every weight receives exactly one gradient GEMM per step at rollout 1 (one per sample
        # on the grid path): the GEMM overwrites the fp32 gradient (no zeroing, no read-back) and
        # one HBM-roofline Adam kernel per lr class follows. fused_adam=True instead applies Adam
        # inside the weight-gradient GEMM epilogue (JG_EPI_ADAM; measured no faster on C4, the
        # 4 epilogue warps cannot hide 26 B/param behind the MMA).
        self.overwrite = r == 1
        self.fused_adam = fused_adam and r == 1 and (model.ctx.n == 1 or batch == 1)
        self.adam = adam or AdamConfig()
        a = self.adam
        self.clip = float(a.clip_norm) if a.clip_norm is not None and a.clip_norm > 0 else None
        self.scheduled = a.total_steps > 0
        if self.fused_adam and (self.clip is not None or model.ctx.dp_replicas > 1):
            raise ConfigError("fused_adam applies Adam inside the gradient GEMMs; clipping and dp_reduce "
                              "need the whole gradient first")
        self.loss_scale = loss_scale
        self.ws = model.workspace(batch, r)
        dev = model.device
        self.target = torch.zeros_like(self.ws.xin)
        # Adam step counter (device; shared by the per-rollout steps of one Trainer)
        self.step_count = step_count if step_count is not None else torch.zeros(1, dtype=torch.int32, device=dev)
        self.lr_dev = torch.zeros(_lib.JG_MAX_LR_CLASSES, dtype=torch.float32, device=dev)  # this step's lr per class
        self.grad_scale = torch.ones(1, dtype=torch.float32, device=dev)                # clip factor
        self.sqsum = torch.zeros(1, dtype=torch.float32, device=dev)                    # global squared grad norm
        self.use_graph = graph
        self._dry = False
        self.graph = None
        self.launches_per_step = None
        self._pinned_loss = torch.zeros(1, dtype=torch.float32, pin_memory=dev.type == "cuda")
        self._h2d_bytes = 2 * self.ws.xin.numel() * 4
        self._d2h_bytes = 4
        # Jigsaw R > 1 over symmetric memory: Adam stores each channel-mixing weight's new bf16
        # copy straight into the column group's panel slots (jg_adam_push), so the next forward
        # replaces the per-panel all-gathers with one barrier. The slots then hold the weights as
        # of this TrainStep's last update: `_panel_version` tracks model.weights_version and a
        # stale step (external weight edit, or another TrainStep's update) re-gathers eagerly.
        self.push_panels = (model.ctx.n > 1 and model.R > 1 and not self.fused_adam
                            and os.environ.get("JIGSAW_PANEL_PUSH", "1") == "1")
        self._panel_version = None
        # Adam overlapped with the backward (1 GPU): once block j's weight gradients are complete
        # (the backward runs blocks last-to-first), its matrices' Adam runs on a side stream pinned
        # to `adam_sms` SMs (jg_adam_sms) while the remaining backward GEMMs use the other SMs
        # (jg_gemm_desc.max_sms); the first block, the encoder / decoder and the vectors are updated
        # after the backward on every SM. Needs the whole step's gradient-free schedule: no
        # clipping (global norm first), no dp_reduce, one gradient GEMM per weight (rollout 1).
        # Measured NOT faster on C4 (power-capped: the GEMMs lose what Adam gains; 25.4-25.9 vs
        # 25.9-26.0 samples/s with 16 / 24 SMs, 20 with 8), so it is an option, off by default.
        self.adam_sms = int(os.environ.get("JIGSAW_ADAM_SMS", "16"))
        self.adam_overlap = (os.environ.get("JIGSAW_ADAM_OVERLAP", "0") == "1" and self.adam_sms > 0
                             and model.ctx.n == 1 and r == 1 and not self.fused_adam and self.clip is None
                             and model.ctx.dp_replicas == 1 and model.device.type == "cuda"
                             and model.cfg.n_blocks > 1)
        self._early: list[tuple[int, int]] = []
        self._adam_stream = None

    # -- the step body --------------------------------------------------------------------
    def _body(self) -> None:
        self._body_fwd()
        self._body_bwd()

    def _body_fwd(self) -> None:
        """Step counter, gradient zeroing, forward (needs only x)."""
        m, ws, f = self.model, self.ws, self.model.flat
        if not self._dry:
            K.step_increment(self.step_count)
        if self.fused_adam or self.overwrite:
            for cls in f.CLASSES:  # matrix gradients are written whole by their GEMM; vectors accumulate
                lo, hi = f.vec_range(cls)
                K.zero(f.grad[lo:hi])
        else:
            m.zero_grads()
        m._panels_pushed = self._pushing()
        try:
            m._forward(ws)
        finally:
            m._panels_pushed = False

    def _body_bwd(self) -> None:
        """Loss against the target, backward, gradient sync, Adam."""
        m, ws = self.model, self.ws
        K.zero(ws.loss)
        m._blend(ws, target=self.target, loss=ws.loss, loss_scale=self.loss_scale)
        if m.ctx.n > 1:
            m.ctx.all_reduce_all(ws.loss)  # the loss is a sum of per-tile terms
        m._fused_adam = (self.step_count, self.adam) if self.fused_adam and not self._dry else None
        m._grad_overwrite = self.overwrite
        overlap = self.adam_overlap and not self._dry
        self._early = []
        if overlap:
            if self.scheduled:  # this step's lr (no clipping here: it needs no gradient)
                K.opt_schedule(self.step_count, [self.adam.schedule(c) for c in m.flat.CLASSES], self.sqsum, None,
                               self.lr_dev, self.grad_scale)
            m._after_block_bwd = self._early_adam
        try:
            m._backward(ws)
        finally:
            m._fused_adam = None
            m._grad_overwrite = False
            m._after_block_bwd = None
            T.GEMM_SM_CAP = 0
        m.grad_sync()
        m.ctx.all_reduce_dp_mean(m.flat.grad)  # dp_reduce over replicas of this shard (no-op for one)
        if self._dry:
            return
        if self.clip is not None:
            self._global_sqnorm()
        if (self.clip is not None or self.scheduled) and not overlap:
            K.opt_schedule(self.step_count, [self.adam.schedule(c) for c in m.flat.CLASSES], self.sqsum, self.clip,
                           self.lr_dev, self.grad_scale)
        self._adam()
        if self._early:
            torch.cuda.current_stream().wait_stream(self._adam_stream)  # join the early updates

    def _block_range(self, j: int) -> tuple[int, int]:
        """Flat range of block j's weight matrices (contiguous: lr class, then kind, then order)."""
        f = self.model.flat
        names = [f"block{j}.{w}" for w in ("tok1.w", "tok2.w", "ch1.w", "ch2.w")]
        lo = min(f.offsets[n] for n in names)
        hi = max(f.offsets[n] + f.params[n].data.numel() for n in names)
        return lo, hi

    def _early_adam(self, j: int) -> None:
        """Backward hook after block j: its matrices' Adam on the side stream, pinned to adam_sms
        SMs; the GEMMs issued from here on leave those SMs free. Block 0 (last in the backward)
        waits for the full-GPU Adam after the backward."""
        if j == 0:
            return
        m, f, a = self.model, self.model.flat, self.adam
        if self._adam_stream is None:
            self._adam_stream = torch.cuda.Stream(device=m.device)
        lo, hi = self._block_range(j)
        cls = "body"
        ci = list(f.class_range).index(cls)
        op_copy = f.op if f.op is not f.master else None
        cur, side = torch.cuda.current_stream(), self._adam_stream
        side.wait_stream(cur)  # block j's gradients are written
        with torch.cuda.stream(side):
            K.adam(f.master[lo:], f.grad[lo:], f.m[lo:], f.v[lo:], None if op_copy is None else op_copy[lo:], hi - lo,
                   a.lr(cls), a.beta1, a.beta2, a.eps, self.step_count,
                   lr_dev=self.lr_dev[ci:ci + 1] if self.scheduled else None, sms=self.adam_sms)
        self._early.append((lo, hi))
        T.GEMM_SM_CAP = _lib.num_sms() - self.adam_sms

    def _global_sqnorm(self) -> None:
        """Squared L2 norm of the global gradient: local shards summed over the
        mp group, duplicated vectors counted once (weight 1/R for column vectors shared by the
        column group, 1/C for the row vector shared by the row group; parallel.py:483-485)."""
        m, f = self.model, self.model.flat
        K.zero(self.sqsum)
        for cls in f.CLASSES:
            for kind, w in (("matrix", 1.0), ("vec_col", 1.0 / m.R), ("vec_row", 1.0 / m.C)):
                lo, hi = f.kind_range[(cls, kind)]
                if hi > lo:
                    K.sqnorm(f.grad[lo:hi], self.sqsum, w)
        m.ctx.all_reduce_all(self.sqsum)

    def _pushing(self) -> bool:
        """Adam pushes the weight panels (and the forward only barriers) in this step body."""
        g = getattr(self.ws, "grid", None)
        return (self.push_panels and not self._dry and g is not None and g.kind == "symm"
                and bool(g.panel_names) and self.model.flat.op is not self.model.flat.master)

    def _adam(self) -> None:
        from .jigsaw_grid import panel_push_segments
        f, a = self.model.flat, self.adam
        op_copy = f.op if f.op is not f.master else None
        if self._early:
            # the rest of every class after the early (overlapped) block updates
            for i, (cls, (lo, hi)) in enumerate(f.class_range.items()):
                cuts = sorted(r for r in self._early if lo <= r[0] < hi)
                pos = lo
                for a0, a1 in cuts + [(hi, hi)]:
                    if a0 > pos:
                        K.adam(f.master[pos:], f.grad[pos:], f.m[pos:], f.v[pos:],
                               None if op_copy is None else op_copy[pos:], a0 - pos, a.lr(cls), a.beta1, a.beta2,
                               a.eps, self.step_count, lr_dev=self.lr_dev[i:i + 1] if self.scheduled else None)
                    pos = max(pos, a1)
            return
        push = self._pushing()
        if push:
            # no column-group member may still be reading this step's panels (the encoder's dW
            # GEMM is the last reader) when the pushes land in its slots
            self.ws.grid.col.barrier()
        for i, (cls, (lo, hi)) in enumerate(f.class_range.items()):
            if self.fused_adam:
                lo, hi = f.vec_range(cls)
            if hi <= lo:
                continue
            segs = panel_push_segments(self.model, self.ws.grid, lo, hi) if push else []
            for a0, a1, sub in split_push(lo, hi, segs, _lib.JG_MAX_PUSH_SEGS):
                K.adam(f.master[a0:], f.grad[a0:], f.m[a0:], f.v[a0:], None if op_copy is None else op_copy[a0:],
                       a1 - a0, a.lr(cls), a.beta1, a.beta2, a.eps, self.step_count,
                       grad_scale=self.grad_scale if self.clip is not None else None,
                       lr_dev=self.lr_dev[i:i + 1] if self.scheduled else None, push=sub or None)

    def _refresh_panels(self) -> None:
        """Before a step whose forward relies on pushed panels: if the weights changed since this
        TrainStep's last update (init, checkpoint load, another TrainStep), gather them now."""
        m = self.model
        if not self._pushing():
            return
        v = getattr(m, "weights_version", 0)
        if self._panel_version != v:
            from .jigsaw_grid import gather_panels
            gather_panels(m, self.ws.grid)

    def _updated(self) -> None:
        """After a step's Adam: the model changed and this TrainStep's panel slots hold it."""
        m = self.model
        m.weights_version = getattr(m, "weights_version", 0) + 1
        self._panel_version = m.weights_version

    def capture(self) -> None:
        """Warm up on a side stream with a dry step (forward, loss, backward, gradient sync: no
        optimiser update, no step count — lazy initialisation of communicators and kernels
        happens outside the capture and the training state is untouched), then capture the step
        into two CUDA graphs (forward | loss + backward + Adam) sharing one memory pool, so the
        public call can overlap the target's host->device copy with the forward."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self._dry = True
            try:
                self._body()
            finally:
                self._dry = False
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        before = _lib.launch_count()
        g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1):
            self._body_fwd()
        with torch.cuda.graph(g2, pool=g1.pool()):
            self._body_bwd()
        self.launches_per_step = _lib.launch_count() - before
        self.graph = (g1, g2)
        torch.cuda.synchronize()

    def run_device(self, target_ready: torch.cuda.Event | None = None) -> torch.Tensor:
        """One step on resident inputs (self.ws.xin / self.target); returns the device loss.
        `target_ready`: event the loss half of the step waits on (target still in flight)."""
        if self.use_graph:
            if self.graph is None:
                self.capture()
            self._refresh_panels()
            self.graph[0].replay()
            if target_ready is not None:
                torch.cuda.current_stream().wait_event(target_ready)
            self.graph[1].replay()
        else:
            before = _lib.launch_count()
            self._refresh_panels()
            self._body_fwd()
            if target_ready is not None:
                torch.cuda.current_stream().wait_event(target_ready)
            self._body_bwd()
            self.launches_per_step = _lib.launch_count() - before
        self._updated()
        self.model.ctx.flops += sum(self.model.step_flops(self.batch, self.r))  # MpContext counter, per step
        return self.ws.loss

    def _streams(self):
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream()
            self._target_ev = torch.cuda.Event()
            self._stage = None      # device staging buffers of a prefetched step
            self._staged = None     # (x, target) host tensors the staging buffers hold
            self._stage_ev = torch.cuda.Event()
        return self._copy_stream

    def prefetch(self, x: torch.Tensor, target: torch.Tensor) -> None:
        """Start the host->device copy of the NEXT step's inputs (pinned host tensors) on the copy
        stream, into device staging buffers, so it overlaps the step running now; the next call
        with these same tensors waits for it and moves them into place with one device copy.
        (Pipelined input feeding, as a training loop with a read-ahead loader does.)"""
        if self.model.device.type != "cuda":
            return
        cs = self._streams()
        if self._stage is None:  # (allocated once, at the first prefetch; see warm_prefetch)
            self._stage = (torch.empty_like(self.ws.xin), torch.empty_like(self.target))
        # after everything queued so far (incl. the device copy consuming the previous staged
        # inputs), but ahead of the step about to be launched
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            self._stage[0].copy_(x, non_blocking=True)
            self._stage[1].copy_(target, non_blocking=True)
            self._stage_ev.record(cs)
        self._staged = (x, target)

    def warm_prefetch(self) -> None:
        """Allocate the prefetch staging buffers now (outside any timed region)."""
        if self.model.device.type == "cuda":
            self._streams()
            if self._stage is None:
                self._stage = (torch.empty_like(self.ws.xin), torch.empty_like(self.target))

    def __call__(self, x: torch.Tensor, target: torch.Tensor, prefetch_next=None) -> float:
        """Public step: copy this step's inputs from (pinned) host memory, run, read the loss.
        Without a prefetch the target is copied on a side stream while the forward runs (x is
        needed first). `prefetch_next=(x_next, target_next)` also starts the next step's copies
        behind this step's compute (see prefetch)."""
        cur = torch.cuda.current_stream() if self.model.device.type == "cuda" else None
        ev = None
        if cur is not None:
            cs = self._streams()
            if self._staged is not None and self._staged[0] is x and self._staged[1] is target:
                cur.wait_event(self._stage_ev)
                # staged inputs into place with an SM copy (jg_push), not a copy-engine memcpy that
                # would queue behind the next step's host->device prefetch on the copy engines
                K.push(self._stage[0], [self.ws.xin.data_ptr()])
                K.push(self._stage[1], [self.target.data_ptr()])
                self._staged = None
            else:
                cs.wait_stream(cur)  # the previous step's loss half has finished reading the target
                self.ws.xin.copy_(x, non_blocking=True)
                with torch.cuda.stream(cs):
                    self.target.copy_(target, non_blocking=True)
                    self._target_ev.record(cs)
                ev = self._target_ev
            if prefetch_next is not None:
                self.prefetch(*prefetch_next)
        else:
            self.ws.xin.copy_(x)
            self.target.copy_(target)
        loss = self.run_device(ev)
        self._pinned_loss.copy_(loss, non_blocking=cur is not None)
        if cur is not None:
            cur.synchronize()
        return float(self._pinned_loss.item())

    def sync_loss(self) -> float:
        return float(self.ws.loss.item())

    @property
    def h2d_bytes_per_step(self) -> int:
        return self._h2d_bytes

    @property
    def d2h_bytes_per_step(self) -> int:
        return self._d2h_bytes


class Trainer:
    """train_epoch / finetune_rollout: per step load this
    rank's tile (data.TileLoader, read ahead on a host thread), run the captured step (forward
    with rollout r, loss vs the target at lead r, backward, grad sync, dp_reduce, clip, scheduled
    Adam). Fine-tuning draws r ~ Uniform{1..r_max} from default_rng(seed), the same sequence on
    every rank; one CUDA graph per r, all sharing one Adam step counter."""

    def __init__(self, model: WeatherMixerModel, batch: int = 1, adam: AdamConfig | None = None, r_max: int = 1,
                 seed: int = 0, graph: bool = True):
        self.model, self.batch, self.adam, self.r_max, self.graph = model, batch, adam or AdamConfig(), r_max, graph
        self.rng = np.random.default_rng(seed)
        self.step_count = torch.zeros(1, dtype=torch.int32, device=model.device)
        self.steps: dict[int, TrainStep] = {}
        # position for checkpoint / resume: the epoch in progress, the batches of it already
        # trained, and the rollout RNG state from before that epoch's draws
        self.epoch, self.step_in_epoch = 0, 0
        self._epoch_rng_state = self.rng.bit_generator.state

    def step_for(self, r: int) -> TrainStep:
        if r not in self.steps:
            self.steps[r] = TrainStep(self.model, self.batch, r, self.adam, graph=self.graph,
                                      step_count=self.step_count)
        return self.steps[r]

    def draw_rollouts(self, n: int) -> np.ndarray:
        if self.r_max == 1:
            return np.ones(n, dtype=np.int64)
        return self.rng.integers(1, self.r_max + 1, size=n)

    def train_epoch(self, loader, epoch: int = 0, max_steps: int | None = None, start: int = 0) -> dict:
        """One pass over this replica's share of the samples; returns mean loss, per-step losses
        and rollouts, and the wall time. `start`: batches of this epoch already trained (resume;
        the RNG must hold the epoch-start state, as load_checkpoint restores it)."""
        import time
        nb = loader.steps_per_epoch() if max_steps is None else min(start + max_steps, loader.steps_per_epoch())
        if (loader.lat_real, loader.vars_real) != (self.model.lat_real, self.model.vars_real):
            raise ConfigError(f"loader data is {loader.lat_real} rows x {loader.vars_real} channels but the model's "
                              f"loss mask is {self.model.lat_real} x {self.model.vars_real}: build the model with "
                              f"lat_real=loader.lat_real, vars_real=loader.vars_real")
        self._epoch_rng_state = self.rng.bit_generator.state
        self.epoch, self.step_in_epoch = epoch, start
        rs = self.draw_rollouts(loader.steps_per_epoch())
        if self.r_max > 1 and loader.lead < self.r_max:
            raise ConfigError(f"loader lead {loader.lead} < r_max {self.r_max}: build it with lead=r_max")
        losses = []
        t0 = time.perf_counter()
        for s, (x, t) in enumerate(loader.epoch(epoch, leads=rs if self.r_max > 1 else None, start=start), start):
            if s >= nb:
                break
            losses.append(self.step_for(int(rs[s]))(x, t))
            self.step_in_epoch = s + 1
        return {"loss": float(np.mean(losses)) if losses else float("nan"), "losses": losses,
                "rollouts": rs[start:start + len(losses)].tolist(), "seconds": time.perf_counter() - t0}

    def save_checkpoint(self, directory: str) -> str | None:
        """This rank's shard (weights, Adam state, step) plus the training position: epoch, batches
        done in it, and the rollout RNG's epoch-start state."""
        from . import checkpoint
        step = next(iter(self.steps.values()), None) or self.step_for(1)
        return checkpoint.save(step, directory, extra={"trainer": {
            "epoch": self.epoch, "step_in_epoch": self.step_in_epoch, "rng_state": self._epoch_rng_state}})

    def load_checkpoint(self, directory: str) -> tuple[int, int]:
        """Restore a shard written by save_checkpoint; returns (epoch, start) for train_epoch, which
        then reproduces the uninterrupted run (same rollout draws, same samples)."""
        from . import checkpoint
        header = checkpoint.load(self.step_for(1), directory)
        tr = header.get("trainer")
        if tr is None:
            return 0, 0
        self.rng.bit_generator.state = tr["rng_state"]
        self._epoch_rng_state = tr["rng_state"]
        self.epoch, self.step_in_epoch = int(tr["epoch"]), int(tr["step_in_epoch"])
        return self.epoch, self.step_in_epoch

    finetune_rollout = train_epoch
