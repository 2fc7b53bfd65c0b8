"""TEST HELPER: run fn(comm, *args) on every rank of a gloo world of processes (the torch
counterpart of the reference's runtime.run_spmd, runtime.py:21-47). fn must be a top-level
function of an importable module; results come back in rank order, and a worker exception is
re-raised with its rank and traceback."""
from __future__ import annotations

import os
import socket
import sys
import traceback

import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, fn, args, kernels, teardown):
    try:
        sys.path[:0] = [HERE, ROOT]
        os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                          LOCAL_RANK=str(rank))
        import torch
        torch.set_num_threads(1)
        if kernels:
            import cpu_kernels
            cpu_kernels.install()
        from paper_2507_05753_b200 import Communicator
        comm = Communicator.from_env(backend="gloo") if world > 1 else Communicator.local()
        out = fn(comm, *args)
        q.put((rank, out, None))
        if world > 1 and teardown:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
    except BaseException:  # noqa: BLE001
        q.put((rank, None, traceback.format_exc()))


def run_spmd(world: int, fn, *args, kernels: bool = True, timeout: float = 300, teardown: bool = True):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, fn, args, kernels, teardown)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, out, err = q.get(timeout=timeout)
        if err is not None:
            for p in procs:
                p.kill()
            raise AssertionError(f"rank {rank} failed:\n{err}")
        res[rank] = out
    for p in procs:
        p.join(timeout=60)
    return [res[r] for r in range(world)]
