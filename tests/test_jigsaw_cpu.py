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


def _worker(rank, world, port, out_q, r, mode="fwdbwd"):
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
        if mode == "train":
            from paper_2507_05753_b200.engine import TrainStep
            tl = om.local_sample(oc, z["g_out"][:1] * 0.5, ctx.R, ctx.C, ctx.r, ctx.c)  # a target
            step = TrainStep(model, batch=1, graph=False)
            losses = []
            for _ in range(2):
                step.ws.xin.copy_(torch.tensor(xl[:1], dtype=torch.float32))
                step.target.copy_(torch.tensor(tl, dtype=torch.float32))
                step._body()
                losses.append(float(step.ws.loss.item()))
            res = {"pos": ctx.pos, "rc": (ctx.R, ctx.C, ctx.r, ctx.c), "losses": losses,
                   "params": {k: p.data.numpy().copy() for k, p in model.params.items()}}
            out_q.put(res)
            if world > 1:
                import torch.distributed as dist
                dist.barrier()
                dist.destroy_process_group()
            return
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


def _run(world, r=1, mode="fwdbwd"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, q, r, mode)) for rk in range(world)]
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


@pytest.mark.parametrize("world", [1, 2, 4])
def test_train_step_fused_adam_matches_oracle(world):
    """Two full TrainStep bodies (fused Adam in the weight-gradient epilogues, vector Adam after
    the duplicated-gradient sync) reproduce the oracle's SPEC loss + Adam, tile by tile."""
    from oracle import model as om, train as ot
    z = np.load(os.path.join(GOLD, "wm_golden.npz"))
    meta = json.load(open(os.path.join(GOLD, "comm_golden.json")))
    oc = om.Config(**{**meta["config"], "grid": tuple(meta["config"]["grid"]), "patch": tuple(meta["config"]["patch"])})
    x, t = z["x"][:1], z["g_out"][:1] * 0.5
    params = om.init_params(oc, 0, np.float64)
    mom = {k: np.zeros_like(v) for k, v in params.items()}
    vel = {k: np.zeros_like(v) for k, v in params.items()}
    ref_losses = []
    for step in (1, 2):
        model = om.SerialModel(oc, params)
        loss, g = ot.weighted_mse_loss(model.forward(x), t, ot.lat_weights(oc.grid[0]), np.ones(oc.n_vars))
        grads = model.backward(g)
        ref_losses.append(loss)
        for k in params:
            lr = 2e-5 if k.split(".")[0] in ("enc", "dec") else 1e-4
            ot.adam_step(params[k], grads[k], mom[k], vel[k], step, lr)
    res = _run(world, mode="train")
    p0 = om.init_params(oc, 0, np.float64)
    for d in res:
        assert np.allclose(d["losses"], ref_losses, rtol=1e-5), (d["losses"], ref_losses)
        R, C, rr, cc = d["rc"]
        upd_got = np.concatenate([(d["params"][k] - om.local_tile(oc, k, p0[k], R, C, rr, cc)).ravel() for k in params])
        upd_ref = np.concatenate([(om.local_tile(oc, k, params[k] - p0[k], R, C, rr, cc)).ravel() for k in params])
        assert np.linalg.norm(upd_got - upd_ref) / np.linalg.norm(upd_ref) < 1e-3
