"""Domain-parallel data path.

Each rank reads only its own tile of every sample — longitude part r, channel part c of the
zero-padded [lat, lon, vars] grid (the layout model.forward expects, oracle local_sample) —
straight from a memory-mapped global array into pinned host buffers, on a background thread
that runs ahead of the training step (the step's public call then copies the tile to HBM).

    loader = TileLoader("era5.npy", cfg, ctx, lead=1, seed=0)     # [N, lat_real, lon, vars_real]
    for x, target in loader.epoch(e):                              # pinned [B, lat, lon/R, vars/C]
        loss = step(x, target)

Sample order: one permutation per epoch from default_rng(seed + epoch), identical on every rank,
so all members of a model-parallel group load the same sample; data-parallel replicas take
disjoint round-robin shares (index dp_index of every dp_replicas), truncated to equal length so
every rank agrees on the epoch length up front. Target = sample i + lead.
Padding rows (721 -> 728) and channels (69 -> 70/72) are zero.
"""
from __future__ import annotations

import queue
import threading

import numpy as np
import torch

from .errors import ConfigError


class TileLoader:
    def __init__(self, source, cfg, ctx, *, lead: int = 1, batch: int = 1, seed: int = 0, shuffle: bool = True,
                 prefetch: int = 2, pin: bool | None = None):
        if isinstance(source, str):
            source = np.load(source, mmap_mode="r")
        if source.ndim != 4:
            raise ConfigError(f"source must be [N, lat, lon, vars], got shape {source.shape}")
        n, lat_r, lon, vars_r = source.shape
        lat_p, lon_p = cfg.grid
        if lon != lon_p or lat_r > lat_p or vars_r > cfg.n_vars:
            raise ConfigError(f"source grid {lat_r}x{lon}x{vars_r} does not fit the padded model grid "
                              f"{lat_p}x{lon_p}x{cfg.n_vars}")
        if n <= lead:
            raise ConfigError(f"need more than lead={lead} samples, have {n}")
        R, C = ctx.R, ctx.C
        self.src, self.cfg, self.lead, self.batch, self.seed, self.shuffle = source, cfg, lead, batch, seed, shuffle
        self.lat_real, self.vars_real = lat_r, vars_r
        self.lon_l, self.v_l = lon // R, cfg.n_vars // C
        self.lon0, self.v0 = ctx.r * self.lon_l, ctx.c * self.v_l
        self.nv = max(0, min(self.v_l, vars_r - self.v0))      # real channels in this chunk
        self.dp_index, self.dp_replicas = getattr(ctx, "dp_index", 0), getattr(ctx, "dp_replicas", 1)
        self.shape = (batch, lat_p, self.lon_l, self.v_l)
        pin = torch.cuda.is_available() if pin is None else pin
        self.slots = [tuple(torch.zeros(self.shape, dtype=torch.float32, pin_memory=pin) for _ in range(2))
                      for _ in range(prefetch + 1)]

    # -- sample order --------------------------------------------------------------------
    def order(self, epoch: int) -> np.ndarray:
        idx = np.arange(self.src.shape[0] - self.lead)
        if self.shuffle:
            idx = np.random.default_rng(self.seed + epoch).permutation(idx)
        per = len(idx) // self.dp_replicas
        return idx[self.dp_index::self.dp_replicas][:per]

    def steps_per_epoch(self) -> int:
        return len(self.order(0)) // self.batch

    # -- tile reads ----------------------------------------------------------------------
    def read_tile(self, i: int, out: np.ndarray) -> None:
        """out [lat_p, lon_l, v_l] = this rank's tile of sample i (zero padding)."""
        out[self.lat_real:] = 0
        if self.nv < self.v_l:
            out[:, :, self.nv:] = 0
        if self.nv:
            out[:self.lat_real, :, :self.nv] = self.src[i, :, self.lon0:self.lon0 + self.lon_l,
                                                        self.v0:self.v0 + self.nv]

    def _fill(self, slot, ids, lead) -> None:
        x, t = slot
        xn, tn = x.numpy(), t.numpy()
        for b, i in enumerate(ids):
            self.read_tile(int(i), xn[b])
            self.read_tile(int(i) + lead, tn[b])

    def epoch(self, epoch: int = 0, leads=None, start: int = 0):
        """Yields pinned (x, target) batches; a background thread reads ahead into free slots.
        A yielded pair stays valid until the next item is requested. `leads[s]` (<= lead) is
        batch s's target lead (rollout fine-tuning), default `lead`. `start`: skip the epoch's
        first batches (resuming from a mid-epoch checkpoint)."""
        ids = self.order(epoch)
        if leads is not None and max(leads, default=0) > self.lead:
            raise ConfigError(f"target lead {max(leads)} exceeds the loader's lead {self.lead}")
        nb = len(ids) // self.batch
        free, ready = queue.Queue(), queue.Queue()
        for k in range(len(self.slots)):
            free.put(k)
        stop = threading.Event()

        def work():
            for s in range(start, nb):
                k = free.get()
                if stop.is_set():
                    return
                try:
                    self._fill(self.slots[k], ids[s * self.batch:(s + 1) * self.batch],
                               self.lead if leads is None or s >= len(leads) else int(leads[s]))
                except BaseException as e:  # noqa: BLE001  surfaced in the consumer
                    ready.put(e)
                    return
                ready.put(k)

        th = threading.Thread(target=work, daemon=True)
        th.start()
        try:
            for _ in range(max(0, nb - start)):
                k = ready.get()
                if isinstance(k, BaseException):
                    raise k
                yield self.slots[k]
                free.put(k)
        finally:
            stop.set()
            free.put(0)
            th.join(timeout=10)
