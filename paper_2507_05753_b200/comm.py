"""Rank transport over torch.distributed (NCCL on B200, gloo for CPU tests).

Replaces the reference's message-passing layer (comm.py: in-process mailboxes / TCP mesh,
JGSW frames) with one process per GPU over torch.distributed. The hot path does not use this
API — it runs NCCL sub-communicators and NVLink peer memory (parallel.MpContext, transport.py)
— but the reference's public surface is kept with its semantics:

  Communicator       rank / world_size; isend(peer, tag, arr) snapshots the payload and returns
                     at once; irecv(peer, tag) -> PendingTransfer whose wait() (exactly once)
                     returns a fresh tensor of the SENDER's shape and dtype; recv; reserve_tags;
                     allreduce_sum / allreduce_mean (gather to the lowest rank in ascending rank
                     order, then broadcast: identical bytes on every member); pairwise_sum /
                     pairwise_reduce_mean (summed in rank order); barrier; message / element /
                     byte counters                             (comm.py:72-287)
  ProcessGroup       mp groups = consecutive blocks, dp groups = r % n  (comm.py:319-361)
  CommError / CommTimeout

Frames: a fixed int64 header (magic, src, dst, tag, dtype code, ndim, dims) followed by the
payload, both as torch.distributed point-to-point messages. Messages between one (src, dst)
pair arrive in issue order; a receive for tag t takes the next frame with tag t from that peer
and stashes frames with other tags for later receives (the reference's per-(src, tag) mailbox,
comm.py:93-128). Group reductions are built from these frames, so — unlike a
torch.distributed sub-group — any subset of ranks can reduce without the rest of the world
taking part. pairwise_sum exchanges through one batched isend/irecv (deadlock-free under NCCL,
whose send and receive to the same peer are otherwise serialised on one stream).
"""
from __future__ import annotations

import collections
import datetime
import os

import torch
import torch.distributed as dist

from .errors import CommError, CommTimeout  # noqa: F401  (re-exported)

COLLECTIVE_TAG_BASE = 1 << 48
DEFAULT_TIMEOUT = 30.0
MAGIC = 0x4A475357  # "JGSW", the reference's frame magic (comm.py:27)
MAX_DIMS = 8
HEADER = 6 + MAX_DIMS
_DTYPES = [torch.float32, torch.float64, torch.bfloat16, torch.float16, torch.int32, torch.int64, torch.uint8,
           torch.bool, torch.int8, torch.int16]
_CODE = {d: i for i, d in enumerate(_DTYPES)}


class PendingTransfer:
    """Handle of a non-blocking transfer; wait() exactly once (comm.py:72-90). A receive returns
    the received tensor, a send returns None."""

    def __init__(self, comm: "Communicator", peer: int, tag: int, direction: str, works=()):
        self.comm, self.peer, self.tag, self.direction = comm, peer, tag, direction
        self._works = list(works)
        self._done = False

    def wait(self, timeout: float | None = None):
        if self._done:
            raise CommError(f"transfer (peer={self.peer}, tag={self.tag}, {self.direction}) already waited on")
        self._done = True
        t = self.comm.timeout if timeout is None else timeout
        if self.direction == "send":
            for w in self._works:
                self.comm._wait(w, t, self.peer, self.tag)
            return None
        return self.comm._finish_recv(self.peer, self.tag, t)


class Communicator:
    """Per-rank endpoint over the default torch.distributed group."""

    def __init__(self, rank: int = 0, world_size: int = 1, timeout: float = DEFAULT_TIMEOUT):
        if not 0 <= rank < world_size:
            raise CommError(f"rank {rank} outside world of size {world_size}")
        self.rank, self.world_size, self.timeout = rank, world_size, timeout
        self._coll_seq = 0
        self._groups: dict[tuple[int, ...], object] = {}
        self._stash: dict[tuple[int, int], collections.deque] = collections.defaultdict(collections.deque)
        self.reset_counters()

    # -- construction --------------------------------------------------------
    @classmethod
    def local(cls) -> "Communicator":
        """Single-rank communicator (n = 1; no process group needed)."""
        return cls(0, 1)

    @classmethod
    def from_env(cls, backend: str | None = None, timeout: float = DEFAULT_TIMEOUT) -> "Communicator":
        """Join the torchrun world (RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT)."""
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if world == 1:
            return cls.local()
        if not dist.is_initialized():
            backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
            if backend == "nccl":
                torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
            dist.init_process_group(backend, timeout=datetime.timedelta(seconds=max(timeout, 60)))
        return cls(dist.get_rank(), dist.get_world_size(), timeout)

    # -- groups --------------------------------------------------------------
    def group(self, ranks) -> object:
        """torch.distributed sub-group for `ranks` (the hot path's NCCL sub-communicators).
        new_group is collective over the whole world: every rank must request the same groups in
        the same order (MpContext does, at construction)."""
        key = tuple(sorted(ranks))
        if len(key) == self.world_size:
            return dist.group.WORLD if dist.is_initialized() else None
        if key not in self._groups:
            self._groups[key] = dist.new_group(list(key))
        return self._groups[key]

    # -- frames --------------------------------------------------------------
    def _device(self, like: torch.Tensor | None = None) -> torch.device:
        if dist.is_initialized() and dist.get_backend() == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    def _check_peer(self, peer: int) -> None:
        if not 0 <= peer < self.world_size:
            raise CommError(f"unknown peer {peer} in world of size {self.world_size}")
        if peer == self.rank:
            raise CommError(f"rank {self.rank} cannot transfer to itself")

    def _frame(self, peer: int, tag: int, arr: torch.Tensor):
        if arr.dtype not in _CODE:
            raise CommError(f"unsupported dtype {arr.dtype}")
        if arr.dim() > MAX_DIMS:
            raise CommError(f"at most {MAX_DIMS} dims per message, got {arr.dim()}")
        dev = self._device()
        hdr = torch.zeros(HEADER, dtype=torch.int64)
        hdr[:6] = torch.tensor([MAGIC, self.rank, peer, tag, _CODE[arr.dtype], arr.dim()])
        hdr[6:6 + arr.dim()] = torch.tensor(list(arr.shape), dtype=torch.int64)
        payload = arr.detach().to(dev).clone().contiguous()  # snapshot: the caller may reuse `arr`
        return hdr.to(dev), payload

    def _wait(self, work, timeout: float, peer: int, tag: int) -> None:
        try:
            ok = work.wait(datetime.timedelta(seconds=timeout)) if timeout else work.wait()
        except RuntimeError as e:  # gloo / NCCL report a timed-out wait as a RuntimeError
            raise CommTimeout(f"timed out after {timeout:.1f}s waiting for peer={peer}, tag={tag}: {e}") from e
        if ok is False:
            raise CommTimeout(f"timed out after {timeout:.1f}s waiting for peer={peer}, tag={tag}")

    def _count_send(self, payload: torch.Tensor):
        self.sent_messages += 1
        self.sent_elements += payload.numel()
        self.sent_bytes += payload.numel() * payload.element_size() + 8 * HEADER

    def _count_recv(self, payload: torch.Tensor):
        self.recv_messages += 1
        self.recv_elements += payload.numel()
        self.recv_bytes += payload.numel() * payload.element_size() + 8 * HEADER

    def _recv_frame(self, peer: int, timeout: float, want: int) -> tuple[int, torch.Tensor]:
        dev = self._device()
        hdr = torch.empty(HEADER, dtype=torch.int64, device=dev)
        self._wait(dist.irecv(hdr, peer), timeout, peer, want)
        h = hdr.cpu().tolist()
        magic, src, dst, tag, code, ndim = h[:6]
        if magic != MAGIC:
            raise CommError(f"bad frame magic {magic:#x} from rank {peer}")
        if (src, dst) != (peer, self.rank):
            raise CommError(f"frame routing mismatch: got ({src}->{dst}), expected ({peer}->{self.rank})")
        payload = torch.empty(h[6:6 + ndim], dtype=_DTYPES[code], device=dev)
        if payload.numel():
            self._wait(dist.irecv(payload, peer), timeout, peer, tag)
        self._count_recv(payload)
        return tag, payload

    def _finish_recv(self, peer: int, tag: int, timeout: float) -> torch.Tensor:
        q = self._stash[(peer, tag)]
        if q:
            return q.popleft()
        while True:
            got, payload = self._recv_frame(peer, timeout, tag)
            if got == tag:
                return payload
            self._stash[(peer, got)].append(payload)  # another tag's frame: keep it for its receive

    # -- point to point ------------------------------------------------------
    def isend(self, peer: int, tag: int, arr: torch.Tensor) -> PendingTransfer:
        """Queue a tensor for delivery and return immediately; the payload is snapshotted here, so
        the caller may reuse `arr` at once (comm.py:165-177)."""
        self._check_peer(peer)
        hdr, payload = self._frame(peer, tag, arr)
        works = [dist.isend(hdr, peer)]
        if payload.numel():
            works.append(dist.isend(payload, peer))
        self._count_send(payload)
        return PendingTransfer(self, peer, tag, "send", works)

    def irecv(self, peer: int, tag: int) -> PendingTransfer:
        """Receive the next frame tagged `tag` from `peer`; wait() returns it (comm.py:179-181)."""
        self._check_peer(peer)
        return PendingTransfer(self, peer, tag, "recv")

    def recv(self, peer: int, tag: int) -> torch.Tensor:
        return self.irecv(peer, tag).wait()

    def reserve_tags(self, count: int) -> int:
        """Reserve a block of collective tags; SPMD callers advance in lockstep (comm.py:203-207)."""
        base = COLLECTIVE_TAG_BASE + self._coll_seq
        self._coll_seq += count
        return base

    # -- collectives ---------------------------------------------------------
    def _reduce_to_root(self, group, arr, tag, sends):
        root = group[0]
        if self.rank == root:
            acc = arr.detach().clone()
            for r in group[1:]:
                acc = acc + self.recv(r, tag).to(acc.device)  # ascending rank order: deterministic
            return acc
        sends.append(self.isend(root, tag, arr))
        return None

    def _broadcast(self, group, arr, tag, sends):
        root = group[0]
        if self.rank == root:
            for r in group[1:]:
                sends.append(self.isend(r, tag, arr))
            return arr
        return self.recv(root, tag)

    def _allreduce(self, group, arr: torch.Tensor, mean: bool) -> torch.Tensor:
        group = sorted(group)
        if self.rank not in group:
            raise CommError(f"rank {self.rank} not in reduction group {group}")
        if len(group) == 1:
            return arr.detach().clone()
        tag = self.reserve_tags(2)
        sends: list[PendingTransfer] = []
        total = self._reduce_to_root(group, arr, tag, sends)
        if total is not None and mean:
            total = total / len(group)
        out = self._broadcast(group, total, tag + 1, sends)
        for s in sends:
            s.wait()
        return out.to(arr.device)

    def allreduce_sum(self, group, arr: torch.Tensor) -> torch.Tensor:
        """Elementwise sum over `group` (list of ranks), identical bytes on every member: gather to
        the lowest rank, summed in ascending rank order, then broadcast (comm.py:229-243)."""
        return self._allreduce(group, arr, mean=False)

    def allreduce_mean(self, group, arr: torch.Tensor) -> torch.Tensor:
        """Elementwise arithmetic mean over the group, deterministic order (comm.py:245-256)."""
        return self._allreduce(group, arr, mean=True)

    def _pairwise(self, peer: int, arr: torch.Tensor):
        """Exchange with one peer; returns (lower-rank tensor, higher-rank tensor) (comm.py:258-268)."""
        self._check_peer(peer)
        tag = self.reserve_tags(1)  # lockstep tag, as the reference's schedule (comm.py:262)
        hdr, payload = self._frame(peer, tag, arr)
        other = torch.empty_like(payload)
        ops = [dist.P2POp(dist.isend, payload, peer), dist.P2POp(dist.irecv, other, peer)]
        hdr_in = torch.empty_like(hdr)
        hops = [dist.P2POp(dist.isend, hdr, peer), dist.P2POp(dist.irecv, hdr_in, peer)]
        for w in dist.batch_isend_irecv(hops):
            self._wait(w, self.timeout, peer, -1)
        h = hdr_in.cpu().tolist()
        if h[0] != MAGIC or h[3] != tag:
            raise CommError(f"pairwise exchange with rank {peer} out of order: got tag {h[3]}, expected {tag}")
        if h[4] != hdr.cpu().tolist()[4] or h[6:6 + h[5]] != list(arr.shape):
            raise CommError(f"pairwise shape mismatch: local {tuple(arr.shape)} vs peer {tuple(h[6:6 + h[5]])}")
        if payload.numel():
            for w in dist.batch_isend_irecv(ops):
                self._wait(w, self.timeout, peer, -1)
        self._count_send(payload)
        self._count_recv(other)
        other = other.to(arr.device)
        mine = payload.to(arr.device)
        return (mine, other) if self.rank < peer else (other, mine)

    def pairwise_sum(self, peer: int, arr: torch.Tensor) -> torch.Tensor:
        """t_self + t_peer, summed in rank order so both members agree bitwise (comm.py:275-278)."""
        lo, hi = self._pairwise(peer, arr)
        return lo + hi

    def pairwise_reduce_mean(self, peer: int, arr: torch.Tensor) -> torch.Tensor:
        """(t_self + t_peer) / 2, summed in rank order on both members (comm.py:270-273)."""
        lo, hi = self._pairwise(peer, arr)
        return (lo + hi) / 2

    def barrier(self, group=None) -> None:
        """All members of `group` (default: the world) have arrived (comm.py:280-283)."""
        group = list(range(self.world_size)) if group is None else list(group)
        if len(group) > 1:
            self.allreduce_sum(group, torch.zeros(1))

    def close(self) -> None:
        pass

    def reset_counters(self) -> None:
        self.sent_messages = self.sent_elements = self.sent_bytes = 0
        self.recv_messages = self.recv_elements = self.recv_bytes = 0


class ProcessGroup:
    """World split into model-parallel and data-parallel groups (comm.py:319-361).

    mp groups are consecutive blocks [k n, k n + n); the dp group of rank r is every rank with
    the same r % n. n may be 1, 2, 4 or 8 (the reference stops at 4).
    """

    def __init__(self, world_size: int, n: int, rank: int):
        if n not in (1, 2, 4, 8):
            raise ValueError(f"model-parallel degree must be 1, 2, 4 or 8, got {n}")
        if world_size % n:
            raise ValueError(f"world size {world_size} not divisible by n={n}")
        if not 0 <= rank < world_size:
            raise ValueError(f"rank {rank} outside world of size {world_size}")
        self.world_size, self.n, self.rank = world_size, n, rank

    @property
    def mp_group(self) -> list[int]:
        k = self.rank // self.n
        return list(range(k * self.n, (k + 1) * self.n))

    @property
    def mp_pos(self) -> int:
        return self.rank % self.n

    @property
    def dp_group(self) -> list[int]:
        return [r for r in range(self.world_size) if r % self.n == self.rank % self.n]

    @property
    def dp_index(self) -> int:
        return self.rank // self.n

    @property
    def dp_replicas(self) -> int:
        return self.world_size // self.n

    @staticmethod
    def dp_groups(world_size: int, n: int) -> list[list[int]]:
        return [[r for r in range(world_size) if r % n == c] for c in range(n)]
