"""Communicator semantics over gloo process worlds (mirrors the reference's tests/test_comm.py:
point-to-point with tag matching, wait-once, reductions in deterministic order, pairwise sums),
plus the cases the round-1 version got wrong: irecv without a shape, and reductions / pairwise
sums over rank subsets that differ between ranks (no collective sub-group creation)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from spmd import run_spmd


def _send_recv(comm):
    if comm.rank == 0:
        comm.isend(1, 7, torch.tensor([1.0, 2.0, 3.0], dtype=torch.float64)).wait()
        return None
    return comm.recv(0, 7)


def test_send_recv_shape_and_dtype_come_with_the_frame():
    got = run_spmd(2, _send_recv, kernels=False)[1]
    assert got.dtype == torch.float64 and got.tolist() == [1.0, 2.0, 3.0]


def _out_of_order(comm):
    if comm.rank == 0:
        a = comm.isend(1, 1, torch.tensor([1.0]))
        b = comm.isend(1, 2, torch.tensor([[2.0, 2.5]]))
        a.wait(), b.wait()
        return None
    second = comm.recv(0, 2)
    first = comm.recv(0, 1)
    return first.tolist(), second.tolist()


def test_tag_matching_out_of_order():
    assert run_spmd(2, _out_of_order, kernels=False)[1] == ([1.0], [[2.0, 2.5]])


def _snapshot(comm):
    if comm.rank == 0:
        x = torch.tensor([5.0, 6.0])
        h = comm.isend(1, 3, x)
        x.fill_(-1)  # the payload was copied at isend (comm.py:165-177)
        h.wait()
        return None
    return comm.recv(0, 3).tolist()


def test_isend_snapshots_payload():
    assert run_spmd(2, _snapshot, kernels=False)[1] == [5.0, 6.0]


def _errors(comm):
    from paper_2507_05753_b200 import CommError
    out = []
    for bad in (lambda: comm.isend(comm.rank, 1, torch.zeros(1)), lambda: comm.isend(5, 1, torch.zeros(1))):
        try:
            bad()
            out.append(None)
        except CommError as e:
            out.append(str(e))
    if comm.rank == 0:
        comm.isend(1, 3, torch.zeros(2)).wait()
    else:
        h = comm.irecv(0, 3)
        h.wait()
        try:
            h.wait()
            out.append(None)
        except CommError as e:
            out.append(str(e))
    return out


def test_peer_and_double_wait_errors():
    res = run_spmd(2, _errors, kernels=False)
    for r in res:
        assert "itself" in r[0] and "unknown peer" in r[1]
    assert "already waited" in res[1][2]


def _reductions(comm):
    v = torch.tensor([float(comm.rank + 1)], dtype=torch.float64)
    full = comm.allreduce_mean(list(range(comm.world_size)), v)
    # disjoint subsets reduce at the same time (the round-1 version created torch sub-groups
    # lazily here, which is collective over the whole world and hangs)
    pair = [comm.rank - comm.rank % 2, comm.rank - comm.rank % 2 + 1]
    sub = comm.allreduce_sum(pair, v)
    ps = comm.pairwise_sum(comm.rank ^ 1, v)           # pairs (0,1), (2,3)
    ps2 = comm.pairwise_sum(comm.rank ^ 2, v * 10)      # pairs (0,2), (1,3)
    pm = comm.pairwise_reduce_mean(comm.rank ^ 1, v)
    comm.barrier()
    comm.barrier(pair)
    return full.item(), sub.item(), ps.item(), ps2.item(), pm.item(), comm.sent_messages > 0


def test_reductions_over_differing_subsets():
    res = run_spmd(4, _reductions, kernels=False)
    for r, (full, sub, ps, ps2, pm, counted) in enumerate(res):
        lo = r - r % 2
        assert full == 2.5                       # (1+2+3+4)/4, reference test_comm.py four-rank mean
        assert sub == (lo + 1) + (lo + 2)
        assert ps == (lo + 1) + (lo + 2)
        assert ps2 == 10 * ((r & 1) + 1) + 10 * ((r & 1) + 3)
        assert pm == ((lo + 1) + (lo + 2)) / 2
        assert counted


def _deterministic(comm, vals):
    return comm.allreduce_mean(range(4), torch.tensor(vals[comm.rank])).numpy().tobytes()


def test_mean_bitwise_identical_on_members_and_runs():
    vals = np.random.default_rng(3).normal(size=(4, 9))
    a = run_spmd(4, _deterministic, vals, kernels=False)
    b = run_spmd(4, _deterministic, vals, kernels=False)
    assert len(set(a)) == 1 and a == b


def _timeout(comm):
    from paper_2507_05753_b200 import CommTimeout
    if comm.rank == 1:
        try:
            comm.irecv(0, 42).wait(timeout=0.5)
        except CommTimeout as e:
            return str(e)
    return None


def test_wait_timeout_names_peer_and_tag():
    # (a timed-out gloo pair is closed, as a dead peer's would be: no teardown barrier)
    msg = run_spmd(2, _timeout, kernels=False, teardown=False)[1]
    assert msg is not None and "peer=0, tag=42" in msg
