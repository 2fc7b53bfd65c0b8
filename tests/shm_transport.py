"""TEST DOUBLE (tests only): the symmetric-memory transport on CPU.

SymmTransport's buffer plumbing (named gather slots, rotating reduce-scatter regions, peer
addresses `base[j] + off + idx * bytes`, producer pushes, the q-way owner sub-chunking of the
4 x 2 grid) is exercised without GPUs: each group member's arena is a shared file under
/dev/shm mapped by every rank, the addresses handed to the kernels are synthetic and resolved by
tests/cpu_kernels.py, and the device barrier becomes a gloo barrier on the group.
"""
from __future__ import annotations

import itertools
import os

import torch
import torch.distributed as dist

import cpu_kernels
from paper_2507_05753_b200.transport import SymmTransport

_gid = itertools.count(1)


class ShmSymmTransport(SymmTransport):
    kind = "symm"

    def _alloc(self, total: int) -> None:
        gid = next(_gid)  # same creation order on every rank -> same id per group
        ranks = dist.get_process_group_ranks(self.group)
        tag = f"{os.environ.get('MASTER_PORT', '0')}_{gid}_{'-'.join(map(str, ranks))}"
        paths = [f"/dev/shm/jg_test_{tag}_{j}" for j in range(self.G)]
        own = torch.from_file(paths[self.idx], shared=True, size=total, dtype=torch.uint8)
        own.zero_()
        dist.barrier(group=self.group)
        self.bufs = [own if j == self.idx else torch.from_file(paths[j], shared=True, size=total, dtype=torch.uint8)
                     for j in range(self.G)]
        dist.barrier(group=self.group)
        os.unlink(paths[self.idx])  # mappings stay valid; nothing left behind in /dev/shm
        self.buf = own
        self.base = [(gid << 40) | (j << 34) for j in range(self.G)]
        for j in range(self.G):
            cpu_kernels.register_peer(self.base[j], self.bufs[j])

    def barrier(self) -> None:
        dist.barrier(group=self.group)


def install():
    import paper_2507_05753_b200.jigsaw_grid as jg
    jg.SymmTransport = ShmSymmTransport
    os.environ["JIGSAW_TRANSPORT"] = "symm"
