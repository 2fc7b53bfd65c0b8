"""Jigsaw host-side schedule on CPU: gloo world of 1 / 2 / 4 / 8 processes running the real
model.py + jigsaw_grid.py orchestration (layouts, NCCL-style collectives, buffer plumbing) with
the kernel layer replaced by the tests/cpu_kernels.py double. The gathered forward output and
every gathered parameter gradient must equal the reference's own n = 1 run (golden vectors)."""
from __future__ import annotations

import json
import os
import random
import socket
import traceback

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import rel_err

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q, r):
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                          LOCAL_RANK=str(rank))
        torch.set_num_threads(1)
        import cpu_kernels
        cpu_kernels.install()
        from oracle import model as om
        from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel
        z = np.load(os.path.join(GOLD, "wm_golden.npz"))
        meta = json.load(open(os.path.join(GOLD, "comm_golden.json")))
        comm = Communicator.from_env(backend="gloo") if world > 1 else Communicator.local()
        ctx = MpContext(comm, list(range(world)))
        cfg = ModelConfig.from_dict(meta["config"])
        model = WeatherMixerModel(ctx, cfg, seed=0, dtype="f32", device="cpu")
        oc = om.Config(**{**meta["config"], "grid": tuple(meta["config"]["grid"]), "patch": tuple(meta["config"]["patch"])})
        x = z["x"][:1] if r > 1 else z["x"]
        g = z["g_out"][:1] if r > 1 else z["g_out"]
        xl = om.local_sample(oc, x, ctx.R, ctx.C, ctx.r, ctx.c)
        gl = om.local_sample(oc, g, ctx.R, ctx.C, ctx.r, ctx.c)
        model.zero_grads()
        out = model.forward(torch.tensor(xl, dtype=torch.float32), r=r)
        model.backward(torch.tensor(gl, dtype=torch.float32))
        model.grad_sync()
        res = {"pos": ctx.pos, "out": out.numpy(), "grads": {k: p.grad.numpy().copy() for k, p in model.params.items()},
               "rc": (ctx.R, ctx.C, ctx.r, ctx.c)}
        out_q.put(res)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        out_q.put({"error": traceback.format_exc(), "rank": rank})


def _run(world, r=1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, q, r)) for rk in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rr in res:
        if "error" in rr:
            raise AssertionError(f"rank {rr['rank']} failed:\n{rr['error']}")
    return sorted(res, key=lambda d: d["pos"])


def _check(world, r=1):
    from oracle import model as om
    z = np.load(os.path.join(GOLD, "wm_golden.npz"))
    meta = json.load(open(os.path.join(GOLD, "comm_golden.json")))
    oc = om.Config(**{**meta["config"], "grid": tuple(meta["config"]["grid"]), "patch": tuple(meta["config"]["patch"])})
    res = _run(world, r)
    out_key = "out_f64" if r == 1 else "rollout_out_f64"
    gpre = "grad_f64/" if r == 1 else "rollout_grad_f64/"
    ref_out = z[out_key]
    for d in res:
        R, C, rr, cc = d["rc"]
        assert rel_err(d["out"], om.local_sample(oc, ref_out, R, C, rr, cc)) < 1e-5
    for name in meta["param_names"]:
        gref = z[gpre + name]
        for d in res:
            R, C, rr, cc = d["rc"]
            tile = om.local_tile(oc, name, gref, R, C, rr, cc)
            assert rel_err(d["grads"][name], tile) < 1e-5, (world, name, d["pos"], rel_err(d["grads"][name], tile))


def test_single_rank_schedule_matches_reference():
    _check(1)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_jigsaw_grid_matches_reference(world):
    _check(world)


def test_jigsaw_rollout_4way():
    _check(4, r=2)
