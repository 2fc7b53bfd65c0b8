"""Rank transport over torch.distributed (NCCL on B200, gloo for CPU tests).

Replaces the reference's message-passing layer (comm.py: in-process mailboxes / TCP mesh,
JGSW frames) with one process per GPU and NCCL collectives over NVLink 5 / NVSwitch. The
reference's public surface is kept where the hot path uses it:

  Communicator       rank / world_size, isend / irecv / recv (PendingTransfer.wait once),
                     pairwise_sum, allreduce_sum / allreduce_mean, barrier, reserve_tags,
                     message / element / byte counters          (comm.py:131-287)
  ProcessGroup       mp groups = consecutive blocks, dp groups = r % n  (comm.py:319-361)
  CommError / CommTimeout

Tags are kept for API compatibility; NCCL point-to-point matches by issue order per peer,
which the SPMD lockstep of the reference (comm.py:203-207) already guarantees.
"""
from __future__ import annotations

import datetime
import os

import torch
import torch.distributed as dist

from .errors import CommError, CommTimeout  # noqa: F401  (re-exported)

COLLECTIVE_TAG_BASE = 1 << 48
DEFAULT_TIMEOUT = 30.0


class PendingTransfer:
    """Handle of a non-blocking transfer; wait() exactly once (comm.py:72-90)."""

    def __init__(self, work, kind: str, peer: int, tag: int, tensor=None):
        self._work, self.kind, self.peer, self.tag, self._tensor = work, kind, peer, tag, tensor
        self._done = False

    def wait(self):
        if self._done:
            raise CommError(f"transfer ({self.kind} peer {self.peer}, tag {self.tag}) already waited")
        self._done = True
        if self._work is not None:
            self._work.wait()
        return self._tensor if self.kind == "recv" else None


class Communicator:
    """Per-rank endpoint over the default torch.distributed group."""

    def __init__(self, rank: int = 0, world_size: int = 1, timeout: float = DEFAULT_TIMEOUT):
        if not 0 <= rank < world_size:
            raise CommError(f"rank {rank} outside world of size {world_size}")
        self.rank, self.world_size, self.timeout = rank, world_size, timeout
        self._coll_seq = 0
        self._groups: dict[tuple[int, ...], object] = {}
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
        """torch.distributed sub-group for `ranks` (created collectively on first use: every rank
        must request the same groups in the same order, as new_group requires)."""
        key = tuple(sorted(ranks))
        if len(key) == self.world_size:
            return dist.group.WORLD if dist.is_initialized() else None
        if key not in self._groups:
            self._groups[key] = dist.new_group(list(key))
        return self._groups[key]

    # -- point to point ------------------------------------------------------
    def _check_peer(self, peer: int) -> None:
        if not 0 <= peer < self.world_size:
            raise CommError(f"unknown peer {peer} in world of size {self.world_size}")
        if peer == self.rank:
            raise CommError(f"rank {self.rank} cannot transfer to itself")

    def _count_send(self, t: torch.Tensor):
        self.sent_messages += 1
        self.sent_elements += t.numel()
        self.sent_bytes += t.numel() * t.element_size()

    def _count_recv(self, t: torch.Tensor):
        self.recv_messages += 1
        self.recv_elements += t.numel()
        self.recv_bytes += t.numel() * t.element_size()

    def isend(self, peer: int, tag: int, arr: torch.Tensor) -> PendingTransfer:
        """Queue a tensor for delivery; the payload is snapshotted (comm.py:165-177)."""
        self._check_peer(peer)
        payload = arr.detach().clone().contiguous()
        work = dist.isend(payload, peer)
        self._count_send(payload)
        return PendingTransfer(work, "send", peer, tag, payload)

    def irecv(self, peer: int, tag: int, like: torch.Tensor) -> PendingTransfer:
        """Receive into a fresh tensor shaped like `like` (NCCL needs the size up front)."""
        self._check_peer(peer)
        buf = torch.empty_like(like)
        work = dist.irecv(buf, peer)
        self._count_recv(buf)
        return PendingTransfer(work, "recv", peer, tag, buf)

    def recv(self, peer: int, tag: int, like: torch.Tensor) -> torch.Tensor:
        return self.irecv(peer, tag, like).wait()

    def reserve_tags(self, count: int) -> int:
        base = COLLECTIVE_TAG_BASE + self._coll_seq
        self._coll_seq += count
        return base

    # -- collectives ---------------------------------------------------------
    def allreduce_sum(self, group, arr: torch.Tensor) -> torch.Tensor:
        """Elementwise sum over `group` (list of ranks); identical on every member (comm.py:229-243)."""
        group = sorted(group)
        if self.rank not in group:
            raise CommError(f"rank {self.rank} not in reduction group {group}")
        out = arr.clone()
        if len(group) > 1:
            dist.all_reduce(out, group=self.group(group))
            self._count_send(out)
        return out

    def allreduce_mean(self, group, arr: torch.Tensor) -> torch.Tensor:
        out = self.allreduce_sum(group, arr)
        if len(group) > 1:
            out /= len(group)
        return out

    def pairwise_sum(self, peer: int, arr: torch.Tensor) -> torch.Tensor:
        """t_self + t_peer, identical on both members (comm.py:275-278)."""
        self._check_peer(peer)
        return self.allreduce_sum([self.rank, peer], arr)

    def barrier(self, group=None) -> None:
        if self.world_size > 1:
            dist.barrier(group=None if group is None else self.group(group))

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
