"""Jigsaw exchange transports for one grid axis (the row group or the column group of a rank).

Two implementations of the same two operations used by jigsaw_grid.py:

  ag(x, slot)          all-gather: returns the local [G, *x.shape] planes of the group members'
                       blocks (ordered by group index)
  rs_gemm(shape, fn)   reduce-scatter of a GEMM's partial products: `fn(planes, d_planes)` runs
                       the plane-batched GEMM; returns (acc, nplanes, plane_stride) for the
                       consuming epilogue (which sums the planes)

* NcclTransport — NCCL all_gather_into_tensor / reduce_scatter_tensor on the compute stream
  (also the gloo path of the CPU tests).
* SymmTransport — NVLink peer memory (torch symmetric memory, CUDA backend): the GEMM epilogue
  stores each partial plane straight into its owner's buffer (`d_planes`, remote st.global
  over NVLink, overlapping the transfer with the MMA tile by tile); gathers are copy-engine
  pushes into the peers' buffers; a 7 us device barrier (graph-capturable) publishes them.
  Buffers: one symmetric arena per group = a named slot per gather role (u rows, gelu(h)
  columns, weight panels, the g / gc / g_x2 gradient gathers, a copy-engine scratch) + two
  rotating regions for reduce-scatter partials. A slot is rewritten only after the barrier of a
  later exchange, which every member passes only after its consumer of the previous contents
  (stream order), so no peer can overwrite data another member is still reading; partial
  planes are summed right after their barrier, so two rotating regions suffice.
"""
from __future__ import annotations

import ctypes
import os

import torch
import torch.distributed as dist

from . import _lib
from . import kernels as K


class Gather:
    """A reserved all-gather destination: the producer writes its block to `own` and (symmetric
    memory) also stores it at every address in `peers`; after publish(), `planes` [G, *shape]
    holds every member's block."""

    def __init__(self, planes, own, peers, pm=None):
        self.planes, self.own, self.peers = planes, own, peers
        self.pm = pm  # plane-major destination (slot tensor, sub, nsub, q) of dest_pm, NCCL publish


def pm_block(r: int, sub: int, nsub: int, q: int) -> int:
    """Block index of member r's sample `sub` in a plane-major gather slot [G/q][nsub][q][block]:
    members r = j*q .. j*q+q-1 (one chunk j of the gathered rows) of every sample next to each
    other, chunk-major over the samples — so chunk j of sample b sits at (j*nsub + b) * q blocks,
    one uniform stride for a GEMM batched over (chunk, sample)."""
    return ((r // q) * nsub + sub) * q + r % q


class NcclTransport:
    kind = "nccl"

    def __init__(self, group, G: int, idx: int, device):
        self.group, self.G, self.idx, self.device = group, G, idx, device
        self._persist: dict[str, torch.Tensor] = {}
        self._scratch = {}
        self.bytes_sent = 0  # payload bytes this member sends to its peers (host-side count per issue)

    def reserve(self, name: str, shape, dtype) -> None:
        self._persist[name] = torch.empty(shape, dtype=dtype, device=self.device)

    def persistent(self, name: str) -> torch.Tensor:
        return self._persist[name]

    def _slot(self, name, numel, dtype):
        t = self._persist.get(name)
        if t is None or t.numel() < numel or t.dtype != dtype:
            assert name not in self._persist or t.numel() >= numel, f"slot {name} too small"
            t = torch.empty(numel, dtype=dtype, device=self.device)
            self._persist[name] = t
        return t.reshape(-1)[:numel]

    def _buf(self, key, numel, dtype):
        b = self._scratch.get((key, dtype))
        if b is None or b.numel() < numel:
            b = torch.empty(numel, dtype=dtype, device=self.device)
            self._scratch[(key, dtype)] = b
        return b[:numel]

    def ag(self, x: torch.Tensor, slot: str = "tmp", sub: int = 0, nsub: int = 1) -> torch.Tensor:
        """Planes [G, *x.shape] in the named slot (viewed [nsub, G, *x.shape], entry sub)."""
        out = self._slot(slot, nsub * self.G * x.numel(), x.dtype).view(nsub, self.G, *x.shape)[sub]
        self.bytes_sent += (self.G - 1) * x.numel() * x.element_size()
        if self.G == 1:
            out[0].copy_(x)
        else:
            dist.all_gather_into_tensor(out.view(-1), x.reshape(-1), group=self.group)
        return out

    def dest(self, shape, dtype, slot: str, sub: int = 0, nsub: int = 1) -> Gather:
        n = 1
        for s_ in shape:
            n *= s_
        planes = self._slot(slot, nsub * self.G * n, dtype).view(nsub, self.G, *shape)[sub]
        return Gather(planes, self._buf(("own", slot, sub), n, dtype).view(*shape), [])

    def dest_pm(self, shape, dtype, slot: str, sub: int, nsub: int, q: int) -> Gather:
        """Gather destination whose members' blocks land plane-major in `slot` (see pm_block)."""
        n = 1
        for s_ in shape:
            n *= s_
        return Gather(None, self._buf(("own", slot, sub), n, dtype).view(*shape), [],
                      pm=(self._persist[slot], sub, nsub, q))

    def publish(self, h: Gather) -> None:
        self.bytes_sent += (self.G - 1) * h.own.numel() * h.own.element_size()
        if h.pm is not None:
            slot, sub, nsub, q = h.pm
            tmp = self._buf(("pm", h.own.numel()), self.G * h.own.numel(), h.own.dtype)
            if self.G == 1:
                tmp.copy_(h.own.reshape(-1))
            else:
                dist.all_gather_into_tensor(tmp, h.own.reshape(-1), group=self.group)
            n = h.own.numel()
            dst = slot.view(-1)[:self.G * nsub * n].view(self.G // q, nsub, q * n)[:, sub]
            dst.copy_(tmp.view(self.G // q, q * n))  # (NCCL path: the scatter into the plane-major slot)
            return
        if self.G == 1:
            h.planes[0].copy_(h.own)
        else:
            dist.all_gather_into_tensor(h.planes.view(-1), h.own.reshape(-1), group=self.group)

    def rs_gemm(self, rows: int, cols: int, dtype, fn, q: int = 1, out: torch.Tensor | None = None, key: int = 0):
        """fn(s, D, d_bs, d_planes) for s < q computes GEMM batches j writing owner plane j*q + s."""
        planes = self._buf(("rs", key), self.G * rows * cols, dtype).view(self.G, rows, cols)
        for s in range(q):
            fn(s, planes[s], q * rows * cols, None)
        self.bytes_sent += (self.G - 1) * rows * cols * planes.element_size()
        if self.G == 1:
            return planes[0], 1, 0
        use_out = out is not None and out.dtype == dtype
        red = out if use_out else self._buf(("red", key), rows * cols, dtype).view(rows, cols)
        dist.reduce_scatter_tensor(red.view(-1), planes.view(-1), group=self.group)
        return red, 1, 0

    def rs_gemm_multi(self, rows: int, cols: int, dtype, fns, q: int = 1, outs=None, run=None):
        """Several independent reduce-scatters of the same shape (e.g. one per sample). `run`
        launches a list of closures (e.g. concurrently on side streams); then one NCCL
        reduce-scatter per item."""
        outs = outs or [None] * len(fns)
        planes = [self._buf(("rs", k), self.G * rows * cols, dtype).view(self.G, rows, cols) for k in range(len(fns))]
        calls = [lambda fn=fn, pl=pl, s=s: fn(s, pl[s], q * rows * cols, None)
                 for fn, pl in zip(fns, planes) for s in range(q)]
        (run or _run_all)(calls)
        res = []
        for k, (pl, o) in enumerate(zip(planes, outs)):
            self.bytes_sent += (self.G - 1) * rows * cols * pl.element_size()
            if self.G == 1:
                res.append((pl[0], 1, 0))
                continue
            red = o if o is not None and o.dtype == dtype else self._buf(("red", k), rows * cols, dtype).view(rows, cols)
            dist.reduce_scatter_tensor(red.view(-1), pl.reshape(-1), group=self.group)
            res.append((red, 1, 0))
        return res

    def rs_gemm_batched(self, rows: int, cols: int, dtype, nsamples: int, fns, fn_batched=None, q: int = 1,
                        outs=None, run=None):
        """(peer-memory transport: one launch for all samples) here: per-sample reduce-scatters."""
        return self.rs_gemm_multi(rows, cols, dtype, fns, q=q, outs=outs, run=run)

    def publish_all(self, hs) -> None:
        for h in hs:
            self.publish(h)


FLAG_CAP = 1 << 15  # arrival counters per reduce-scatter region (jg_gemm_desc.rs_flag_cap)
PUSH_SM_BYTES = 4 << 20  # gathers up to this size are pushed by an SM kernel (jg_push), larger by copy engines


def _run_all(calls) -> None:
    for c in calls:
        c()


class Fanout:
    """Launch independent closures concurrently on a few side streams forked from the current
    stream and joined back into it (graph-capturable: the capture records the fork / join as
    parallel branches). Used for the per-sample token-mixing GEMMs of a B > 1 grid step: each
    alone has too few tiles to fill 148 SMs (C3 at 1x2: 16-32 tiles), side by side they do."""

    def __init__(self, device, width: int):
        self.cuda = device.type == "cuda" and width > 1
        self.streams = [torch.cuda.Stream(device=device) for _ in range(width)] if self.cuda else []

    def __call__(self, calls) -> None:
        if not self.cuda or len(calls) < 2:
            _run_all(calls)
            return
        cur = torch.cuda.current_stream()
        used = self.streams[:min(len(self.streams), len(calls))]
        for s in used:
            s.wait_stream(cur)
        for i, c in enumerate(calls):
            with torch.cuda.stream(used[i % len(used)]):
                c()
        for s in used:
            cur.wait_stream(s)


def fused_rs_enabled() -> bool:
    """GEMM + reduce-scatter + epilogue as one kernel (JIGSAW_FUSED_RS=1; the default is the
    GEMM -> barrier -> jg_epilogue sequence, measured faster)."""
    return os.environ.get("JIGSAW_FUSED_RS", "0") == "1"


class SymmTransport:
    kind = "symm"

    def __init__(self, group, G: int, idx: int, device, scratch_bytes: int, persist_spec):
        self.group, self.G, self.idx, self.device = group, G, idx, device
        self.offsets: dict[str, tuple[int, tuple, torch.dtype]] = {}
        off = 0
        for name, shape, dtype in persist_spec:
            n = 1
            for s in shape:
                n *= s
            self.offsets[name] = (off, tuple(shape), dtype)
            off += -(-n * torch.empty((), dtype=dtype).element_size() // 256) * 256
        self.scratch_off = off
        self.scratch_bytes = -(-scratch_bytes // 256) * 256
        self.flag_off = off + 2 * self.scratch_bytes  # per region: FLAG_CAP arrival counters (fused RS)
        self.bar_off = self.flag_off + 2 * FLAG_CAP * 4  # G arrival counters of jg_group_barrier
        self.k = 0
        self.bytes_sent = 0  # payload bytes this member stores into its peers (host-side count per issue)
        self._alloc(self.bar_off + 256)
        self.buf[self.flag_off:].zero_()
        # JIGSAW_BARRIER=jg: jg_group_barrier (one 32-thread kernel: release-add into each peer's
        # counter, acquire-spin on its own); measured no faster than the default, torch's barrier
        self._jg_bar = False
        self.barrier()  # every member's counters are zero before anyone signals
        self._jg_bar = os.environ.get("JIGSAW_BARRIER", "torch") == "jg"
        self._bar_peers = (ctypes.c_void_p * 8)(*[b + self.bar_off for b in self.base])
        self._bar_epoch = torch.zeros(1, dtype=torch.int32, device=device)

    def _alloc(self, total: int) -> None:
        """One symmetric arena per group member; self.base[j] = member j's arena address."""
        import torch.distributed._symmetric_memory as symm
        name = self.group.group_name
        try:
            symm.enable_symm_mem_for_group(name)
        except Exception:  # noqa: BLE001  (newer torch enables on demand)
            pass
        self.buf = symm.empty(total, dtype=torch.uint8, device=self.device)
        self.hdl = symm.rendezvous(self.buf, name)
        self.base = [int(p) for p in self.hdl.buffer_ptrs]

    def reserve(self, name, shape, dtype):  # persistent slots are fixed at construction
        assert name in self.offsets, name

    def _view(self, off: int, shape, dtype) -> torch.Tensor:
        n = 1
        for s in shape:
            n *= s
        es = torch.empty((), dtype=dtype).element_size()
        return self.buf[off:off + n * es].view(dtype).view(*shape)

    def persistent(self, name: str) -> torch.Tensor:
        off, shape, dtype = self.offsets[name]
        return self._view(off, shape, dtype)

    def _region(self) -> int:
        r = self.scratch_off + (self.k % 2) * self.scratch_bytes
        self.k += 1
        return r

    def barrier(self) -> None:
        if self._jg_bar:
            _lib.call("jg_group_barrier", self._bar_peers, self.base[self.idx] + self.bar_off,
                      self._bar_epoch.data_ptr(), self.G, self.idx)
        else:
            self.hdl.barrier(channel=0)

    def _slot_off(self, slot: str, sub: int, nbytes: int) -> int:
        off, shape, dtype = self.offsets[slot]
        cap = torch.empty((), dtype=dtype).element_size()
        for s_ in shape:
            cap *= s_
        assert (sub + 1) * self.G * nbytes <= cap, f"slot {slot} too small"
        return off + sub * self.G * nbytes

    def ag(self, x: torch.Tensor, slot: str = "tmp", sub: int = 0, nsub: int = 1) -> torch.Tensor:
        nbytes = x.numel() * x.element_size()
        off = self._slot_off(slot, sub, nbytes)
        x = x.contiguous()
        dsts = [self.base[j] + off + self.idx * nbytes for j in range(self.G)]
        if nbytes <= PUSH_SM_BYTES and self.G <= 4 and nbytes % 8 == 0 and x.data_ptr() % 8 == 0 and off % 8 == 0:
            # small gathers (layer-norm moments): stores from the SMs, so they never queue behind a
            # bulk host->device copy on the copy engines (the e2e input feed)
            K.push(x, dsts, nbytes)
        else:
            for d in dsts:  # push my block into slot idx of every member (copy engine)
                K.copy_async(d, x, nbytes)
        self.bytes_sent += (self.G - 1) * nbytes
        self.barrier()
        return self._view(off, (self.G, *x.shape), x.dtype)

    def dest(self, shape, dtype, slot: str, sub: int = 0, nsub: int = 1) -> Gather:
        n = 1
        for s_ in shape:
            n *= s_
        nbytes = n * torch.empty((), dtype=dtype).element_size()
        off = self._slot_off(slot, sub, nbytes)
        planes = self._view(off, (self.G, *shape), dtype)
        peers = [self.base[j] + off + self.idx * nbytes for j in range(self.G) if j != self.idx]
        return Gather(planes, planes[self.idx], peers)

    def dest_pm(self, shape, dtype, slot: str, sub: int, nsub: int, q: int) -> Gather:
        """Gather destination whose members' blocks land plane-major in `slot` (see pm_block):
        the producer stores its block at the same position of every member's slot."""
        n = 1
        for s_ in shape:
            n *= s_
        nbytes = n * torch.empty((), dtype=dtype).element_size()
        blk = pm_block(self.idx, sub, nsub, q)
        off = self._slot_off(slot, 0, nsub * nbytes)  # (capacity check for G x nsub blocks)
        pos = off + blk * nbytes
        own = self._view(pos, shape, dtype)
        peers = [self.base[j] + pos for j in range(self.G) if j != self.idx]
        return Gather(None, own, peers, pm=(self.persistent(slot), sub, nsub, q))

    def publish(self, h: Gather) -> None:
        self.bytes_sent += len(h.peers) * h.own.numel() * h.own.element_size()
        self.barrier()

    def rs_gemm(self, rows: int, cols: int, dtype, fn, q: int = 1, out: torch.Tensor | None = None):
        es = torch.empty((), dtype=dtype).element_size()
        pbytes = rows * cols * es
        off = self._region()
        assert self.G * pbytes <= self.scratch_bytes
        local = self._view(off, (self.G, rows, cols), dtype)
        # owner plane o of my partial goes to slot idx of member o's region (remote epilogue stores)
        for s in range(q):
            fn(s, local[0], 0, [self.base[j * q + s] + off + self.idx * pbytes for j in range(self.G // q)])
        self.bytes_sent += (self.G - 1) * pbytes
        self.barrier()
        return local, self.G, rows * cols

    def rs_gemm_multi(self, rows: int, cols: int, dtype, fns, q: int = 1, outs=None, run=None):
        """Several independent reduce-scatters of one shape (the B samples of a token layer): every
        GEMM stores its partial planes into its own part of one region, then ONE barrier
        publishes them all — B times fewer barriers than a reduce-scatter per sample. `run`
        launches the GEMM closures (e.g. concurrently on side streams, so B small GEMMs fill the
        GPU together)."""
        es = torch.empty((), dtype=dtype).element_size()
        pbytes = rows * cols * es
        off = self._region()
        assert len(fns) * self.G * pbytes <= self.scratch_bytes, "reduce-scatter region too small"
        res, calls = [], []
        for k, fn in enumerate(fns):
            ko = off + k * self.G * pbytes
            local = self._view(ko, (self.G, rows, cols), dtype)
            for s in range(q):
                dpl = [self.base[j * q + s] + ko + self.idx * pbytes for j in range(self.G // q)]
                calls.append(lambda fn=fn, local=local, s=s, dpl=dpl: fn(s, local[0], 0, dpl))
            self.bytes_sent += (self.G - 1) * pbytes
            res.append((local, self.G, rows * cols))
        (run or _run_all)(calls)
        self.barrier()
        return res

    def rs_gemm_batched(self, rows: int, cols: int, dtype, nsamples: int, fns, fn_batched=None, q: int = 1,
                        outs=None, run=None):
        """rs_gemm_multi with ONE GEMM launch per owner sub-chunk for all samples:
        fn_batched(s, D, d_planes, plane_div, planes_bs) (D: a tensor of the partial dtype) multiplies every (plane, sample) item at
        once, batch b -> owner plane b / nsamples at sample b % nsamples of its region (sample
        stride G * rows * cols elements: the per-sample regions of rs_gemm_multi)."""
        if fn_batched is None:
            return self.rs_gemm_multi(rows, cols, dtype, fns, q=q, outs=outs, run=run)
        es = torch.empty((), dtype=dtype).element_size()
        pbytes = rows * cols * es
        off = self._region()
        assert nsamples * self.G * pbytes <= self.scratch_bytes, "reduce-scatter region too small"
        local = self._view(off, (self.G, rows, cols), dtype)  # (its dtype = the partial planes' dtype)
        for s in range(q):
            fn_batched(s, local[0], [self.base[j * q + s] + off + self.idx * pbytes for j in range(self.G // q)],
                       nsamples, self.G * rows * cols)
        self.bytes_sent += nsamples * (self.G - 1) * pbytes
        self.barrier()
        return [(self._view(off + k * self.G * pbytes, (self.G, rows, cols), dtype), self.G, rows * cols)
                for k in range(nsamples)]

    def publish_all(self, hs) -> None:
        """One barrier publishes several producer-pushed gathers."""
        for h in hs:
            self.bytes_sent += len(h.peers) * h.own.numel() * h.own.element_size()
        self.barrier()

    def rs_gemm_fused(self, rows: int, cols: int, dtype, fn, q: int = 1, **epi) -> None:
        """Reduce-scatter fused into the GEMM (jg_gemm_desc rs_*): each launch stores its
        partial tiles raw into the owners' region slots and counts their arrival on the owners'
        flags; the launch holding this rank's own plane runs those tiles last, waits per tile for
        every peer's partial, sums the planes in member order and applies the epilogue `epi`
        (jg_epilogue's arguments; d = the output) — no barrier, no separate epilogue pass.
        Region reuse is safe without a barrier: a member writes region k again only two
        reduce-scatters later, and it cannot finish the one in between before this rank has
        started it, i.e. finished reading region k (stream order)."""
        es = torch.empty((), dtype=dtype).element_size()
        pbytes = rows * cols * es
        fl = self.flag_off + (self.k % 2) * FLAG_CAP * 4
        off = self._region()
        assert self.G * pbytes <= self.scratch_bytes
        local = self._view(off, (self.G, rows, cols), dtype)
        d = epi.pop("d")
        for bad in ("ldd", "ldd2", "ldr", "ldp", "batch", "acc_ld"):
            assert bad not in epi, f"fused reduce-scatter epilogue: unsupported argument {bad}"
        part = _lib.dtype_code(local)
        nb = self.G // q
        self.bytes_sent += (self.G - 1) * pbytes
        for s in range(q):
            dpl, fpeers, own = [], [], -1
            for j in range(nb):
                o = j * q + s
                if o == self.idx:
                    own = j
                    dpl.append(None)
                    fpeers.append(None)
                else:
                    dpl.append(self.base[o] + off + self.idx * pbytes)
                    fpeers.append(self.base[o] + fl)
            rs = dict(flags=self.base[self.idx] + fl if own >= 0 else None, flag_peers=fpeers,
                      src=self.base[self.idx] + off, src_stride=rows * cols, part_type=part, nsrc=self.G,
                      src_idx=self.idx, own=own, need=self.G - 1, flag_cap=FLAG_CAP)
            if own >= 0:
                fn(s, d, 0, dpl, rs=rs, **epi)
            else:
                fn(s, None, 0, dpl, rs=rs)
