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


def _worker(rank, world, port, out_q, r, mode="fwdbwd", opts=None):
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                          LOCAL_RANK=str(rank))
        torch.set_num_threads(1)
        import cpu_kernels
        cpu_kernels.install()
        opts = opts or {}
        if "grid" in opts:
            os.environ["JIGSAW_GRID"] = opts["grid"]
        if "fused_rs" in opts:
            os.environ["JIGSAW_FUSED_RS"] = opts["fused_rs"]
        if opts.get("transport") == "shm":
            import shm_transport
            shm_transport.install()
        from oracle import model as om
        from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel
        z = np.load(os.path.join(GOLD, "wm_golden.npz"))
        meta = json.load(open(os.path.join(GOLD, "comm_golden.json")))
        comm = Communicator.from_env(backend="gloo") if world > 1 else Communicator.local()
        n_mp = opts.get("mp", world)
        k = rank // n_mp
        ctx = MpContext(comm, list(range(k * n_mp, (k + 1) * n_mp)))
        cfg = ModelConfig.from_dict(meta["config"])
        if "panel_push" in opts:
            os.environ["JIGSAW_PANEL_PUSH"] = opts["panel_push"]
        model = WeatherMixerModel(ctx, cfg, seed=0, dtype=opts.get("dtype", "f32"), device="cpu")
        oc = om.Config(**{**meta["config"], "grid": tuple(meta["config"]["grid"]), "patch": tuple(meta["config"]["patch"])})
        x = z["x"][:1] if r > 1 else z["x"]
        g = z["g_out"][:1] if r > 1 else z["g_out"]
        xl = om.local_sample(oc, x, ctx.R, ctx.C, ctx.r, ctx.c)
        gl = om.local_sample(oc, g, ctx.R, ctx.C, ctx.r, ctx.c)
        if mode == "trainer":
            from paper_2507_05753_b200.data import TileLoader
            from paper_2507_05753_b200.engine import Trainer
            src = np.random.default_rng(7).standard_normal((6, *oc.grid, oc.n_vars)).astype(np.float32)
            ld = TileLoader(src, cfg, ctx, lead=2, batch=1, seed=3)
            tr = Trainer(model, batch=1, r_max=2, seed=11, graph=False)
            st = tr.train_epoch(ld, 0, max_steps=3)
            out_q.put({"pos": ctx.pos, "rank": rank, "rc": (ctx.R, ctx.C, ctx.r, ctx.c), "losses": st["losses"],
                       "rollouts": st["rollouts"], "order": ld.order(0).tolist(),
                       "params": {k_: p.data.numpy().copy() for k_, p in model.params.items()}})
            if world > 1:
                import torch.distributed as dist
                dist.barrier()
                dist.destroy_process_group()
            return
        if mode in ("ckpt", "ckpt_load"):
            from paper_2507_05753_b200 import checkpoint as ck
            from paper_2507_05753_b200.engine import TrainStep
            from paper_2507_05753_b200.errors import ConfigError
            tl = om.local_sample(oc, z["g_out"][:1] * 0.5, ctx.R, ctx.C, ctx.r, ctx.c)
            d0 = opts["dir"]

            def run(st, k):
                ls = []
                for _ in range(k):
                    st.ws.xin.copy_(torch.tensor(xl[:1], dtype=torch.float32))
                    st.target.copy_(torch.tensor(tl, dtype=torch.float32))
                    st._body()
                    ls.append(float(st.ws.loss.item()))
                return ls
            if mode == "ckpt_load":
                st = TrainStep(model, batch=1, graph=False)
                try:
                    ck.load(st, d0)
                    err = None
                except ConfigError as e:
                    err = str(e)
                out_q.put({"pos": ctx.pos, "rank": rank, "err": err})
            else:
                st = TrainStep(model, batch=1, graph=False)
                run(st, 2)
                ck.save(st, os.path.join(d0, "a"))
                cont = run(st, 1)
                p_cont = {k_: p.data.numpy().copy() for k_, p in model.params.items()}
                model2 = WeatherMixerModel(ctx, cfg, seed=1, dtype="f32", device="cpu")  # different init
                st2 = TrainStep(model2, batch=1, graph=False)
                hdr = ck.load(st2, os.path.join(d0, "a"))
                ck.save(st2, os.path.join(d0, "b"))
                f = ck.shard_path("", ctx.pos, ctx.n)
                same = open(os.path.join(d0, "a", f), "rb").read() == open(os.path.join(d0, "b", f), "rb").read()
                resumed = run(st2, 1)
                p_res = {k_: p.data.numpy().copy() for k_, p in model2.params.items()}
                out_q.put({"pos": ctx.pos, "rank": rank, "same": same, "cont": cont, "resumed": resumed,
                           "step": hdr["step"], "params_equal": all(np.array_equal(p_cont[k_], p_res[k_]) for k_ in p_cont)})
            if world > 1:
                import torch.distributed as dist
                dist.barrier()
                dist.destroy_process_group()
            return
        if mode == "resume":
            # a fine-tuning run interrupted after 2 batches and resumed from its checkpoint by a
            # fresh Trainer (other init) reproduces the uninterrupted run: same rollout draws,
            # same samples, same losses and weights
            from paper_2507_05753_b200.data import TileLoader
            from paper_2507_05753_b200.engine import Trainer
            src = np.random.default_rng(7).standard_normal((7, *oc.grid, oc.n_vars)).astype(np.float32)
            ld = TileLoader(src, cfg, ctx, lead=2, batch=1, seed=3)
            full = Trainer(model, batch=1, r_max=2, seed=11, graph=False).train_epoch(ld, 0)
            m2 = WeatherMixerModel(ctx, cfg, seed=0, dtype="f32", device="cpu")
            t2 = Trainer(m2, batch=1, r_max=2, seed=11, graph=False)
            first = t2.train_epoch(ld, 0, max_steps=2)
            t2.save_checkpoint(opts["dir"])
            m3 = WeatherMixerModel(ctx, cfg, seed=5, dtype="f32", device="cpu")
            t3 = Trainer(m3, batch=1, r_max=2, seed=99, graph=False)
            ep, start = t3.load_checkpoint(opts["dir"])
            rest = t3.train_epoch(ld, ep, start=start)
            out_q.put({"pos": ctx.pos, "rank": rank, "full": full["losses"], "rollouts": full["rollouts"],
                       "resumed": first["losses"] + rest["losses"],
                       "resumed_rollouts": first["rollouts"] + rest["rollouts"], "start": start,
                       "same_params": all(torch.equal(model.params[k].data, m3.params[k].data) for k in model.params)})
            if world > 1:
                import torch.distributed as dist
                dist.barrier()
                dist.destroy_process_group()
            return
        if mode == "comm":
            # one step warms the panels, the second is the steady state: its transport / all-reduce
            # byte counters must equal the analytic per-step volume of the schedule
            from paper_2507_05753_b200.engine import TrainStep
            from paper_2507_05753_b200.jigsaw_grid import step_exchange_bytes
            tl = om.local_sample(oc, z["g_out"][:1] * 0.5, ctx.R, ctx.C, ctx.r, ctx.c)
            step = TrainStep(model, batch=1, graph=False)
            step.ws.xin.copy_(torch.tensor(xl[:1], dtype=torch.float32))
            step.target.copy_(torch.tensor(tl, dtype=torch.float32))

            def counters():
                gw = step.ws.grid
                return sum(t.bytes_sent for t in (gw.row, gw.col) if t is not None), ctx.allreduce_bytes
            step.run_device()
            c1 = counters()
            step.run_device()
            c2 = counters()
            out_q.put({"pos": ctx.pos, "rank": rank, "measured": (c2[0] - c1[0], c2[1] - c1[1]),
                       "analytic": step_exchange_bytes(model, 1, 1)})
            if world > 1:
                import torch.distributed as dist
                dist.barrier()
                dist.destroy_process_group()
            return
        if mode == "pushcmp":
            from paper_2507_05753_b200.engine import TrainStep
            tl = om.local_sample(oc, z["g_out"][:1] * 0.5, ctx.R, ctx.C, ctx.r, ctx.c)
            step = TrainStep(model, batch=1, graph=False)
            step.ws.xin.copy_(torch.tensor(xl[:1], dtype=torch.float32))
            step.target.copy_(torch.tensor(tl, dtype=torch.float32))
            losses = [float(step.run_device().item()) for _ in range(2)]
            model.set_param_entry("block0.ch1.w", (1, 2), 0.25)  # external edit: pushed panels go stale
            losses += [float(step.run_device().item()) for _ in range(2)]
            out_q.put({"pos": ctx.pos, "rank": rank, "losses": losses, "pushing": step._pushing(),
                       "params": {k_: p.data.float().numpy().copy() for k_, p in model.params.items()}})
            if world > 1:
                import torch.distributed as dist
                dist.barrier()
                dist.destroy_process_group()
            return
        if mode == "train":
            from paper_2507_05753_b200.engine import TrainStep
            from paper_2507_05753_b200.train import AdamConfig
            si = opts.get("sample", lambda kk: 0)(k) if callable(opts.get("sample")) else (k if opts.get("dp") else 0)
            xl = om.local_sample(oc, z["x"][si:si + 1], ctx.R, ctx.C, ctx.r, ctx.c)
            tl = om.local_sample(oc, z["g_out"][si:si + 1] * 0.5, ctx.R, ctx.C, ctx.r, ctx.c)  # a target
            step = TrainStep(model, batch=1, graph=False, adam=AdamConfig(**opts.get("adam", {})))
            losses, scales, lrs = [], [], []
            for _ in range(opts.get("steps", 2)):
                step.ws.xin.copy_(torch.tensor(xl[:1], dtype=torch.float32))
                step.target.copy_(torch.tensor(tl, dtype=torch.float32))
                step._body()
                losses.append(float(step.ws.loss.item()))
                scales.append(float(step.grad_scale.item()))
                lrs.append(step.lr_dev[:2].tolist())
            res = {"pos": ctx.pos, "rank": rank, "rc": (ctx.R, ctx.C, ctx.r, ctx.c), "losses": losses,
                   "scales": scales, "lrs": lrs,
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
        if opts.get("transport") == "shm":
            g = model._ws.grid
            assert type(g.row if g.row is not None and g.row.G > 1 else g.col).__name__ == "ShmSymmTransport"
        res = {"pos": ctx.pos, "out": out.numpy(), "grads": {k: p.grad.numpy().copy() for k, p in model.params.items()},
               "rc": (ctx.R, ctx.C, ctx.r, ctx.c), "flops": ctx.flops, "buf_peak": ctx.param_buffer_peak,
               "batch": int(xl.shape[0])}
        out_q.put(res)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        out_q.put({"error": traceback.format_exc(), "rank": rank})


def _run(world, r=1, mode="fwdbwd", opts=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, q, r, mode, opts)) for rk in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rr in res:
        if "error" in rr:
            raise AssertionError(f"rank {rr['rank']} failed:\n{rr['error']}")
    return sorted(res, key=lambda d: (d.get("rank", 0), d["pos"]))


def _check(world, r=1, opts=None, tol=1e-5):
    from oracle import model as om
    z = np.load(os.path.join(GOLD, "wm_golden.npz"))
    meta = json.load(open(os.path.join(GOLD, "comm_golden.json")))
    oc = om.Config(**{**meta["config"], "grid": tuple(meta["config"]["grid"]), "patch": tuple(meta["config"]["patch"])})
    res = _run(world, r, opts=opts)
    out_key = "out_f64" if r == 1 else "rollout_out_f64"
    gpre = "grad_f64/" if r == 1 else "rollout_grad_f64/"
    ref_out = z[out_key]
    if r == 1:
        # MpContext.flops on the fused path: the reference's count (golden, parallel.py:65-69) minus
        # the encoder input gradient it computes and discards, split evenly over the ranks
        B = res[0]["batch"]
        want = meta["flops_n1"] - 2 * B * oc.tokens * oc.patch_features * oc.d_emb
        assert sum(d["flops"] for d in res) == want
        assert len({d["flops"] for d in res}) == 1
        R = res[0]["rc"][0]
        assert all((d["buf_peak"] > 0) == (R > 1) for d in res)
    for d in res:
        R, C, rr, cc = d["rc"]
        assert rel_err(d["out"], om.local_sample(oc, ref_out, R, C, rr, cc)) < tol
    for name in meta["param_names"]:
        gref = z[gpre + name]
        for d in res:
            R, C, rr, cc = d["rc"]
            tile = om.local_tile(oc, name, gref, R, C, rr, cc)
            assert rel_err(d["grads"][name], tile) < tol, (world, name, d["pos"], rel_err(d["grads"][name], tile))


def test_single_rank_schedule_matches_reference():
    _check(1)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_jigsaw_grid_matches_reference(world):
    _check(world)


def test_jigsaw_rollout_4way():
    _check(4, r=2)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_symmetric_memory_schedule_matches_reference(world):
    """The peer-memory transport's plumbing (slots, rotating partial regions, producer pushes,
    epilogue stores into owners' planes, q-way sub-chunks at 4 x 2) on emulated peer memory."""
    _check(world, opts={"transport": "shm"})


@pytest.mark.parametrize("world,fused", [(2, "1"), (4, "1"), (8, "1"), (8, "0")])
def test_fused_reduce_scatter_schedule_matches_reference(world, fused):
    """GEMM + reduce-scatter + epilogue as one kernel (jg_gemm rs_*: raw partials to the owners,
    arrival flags, own plane summed in member order) against the GEMM -> barrier -> epilogue
    schedule's reference results, including the q = 2 owner sub-chunks of the 4 x 2 grid."""
    _check(world, opts={"transport": "shm", "fused_rs": fused})


def test_symmetric_memory_rollout_8way():
    _check(8, r=2, opts={"transport": "shm"})


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


def _oracle_train(oc, samples, steps, adam_opts=None, clip=None):
    """Serial f64 training: per step, the mean over `samples` of each sample's gradient (dp_reduce),
    global-norm clip, scheduled Adam. Returns (per-sample losses per step, params, p0)."""
    from oracle import model as om, train as ot
    z = np.load(os.path.join(GOLD, "wm_golden.npz"))
    params = om.init_params(oc, 0, np.float64)
    p0 = {k: v.copy() for k, v in params.items()}
    mom = {k: np.zeros_like(v) for k, v in params.items()}
    vel = {k: np.zeros_like(v) for k, v in params.items()}
    a = adam_opts or {}
    losses, norms = [], []
    for step in range(1, steps + 1):
        acc, ls = None, []
        for si in samples:
            model = om.SerialModel(oc, params)
            loss, g = ot.weighted_mse_loss(model.forward(z["x"][si:si + 1]), z["g_out"][si:si + 1] * 0.5,
                                           ot.lat_weights(oc.grid[0]), np.ones(oc.n_vars))
            grads = model.backward(g)
            ls.append(loss)
            acc = grads if acc is None else {k: acc[k] + grads[k] for k in acc}
        grads = {k: v / len(samples) for k, v in acc.items()}
        names = list(grads)
        clipped, norm = ot.clip_grads([grads[k] for k in names], clip) if clip else ([grads[k] for k in names], 0.0)
        grads = dict(zip(names, clipped))
        norms.append(norm)
        losses.append(ls)
        for k in params:
            enc = k.split(".")[0] in ("enc", "dec")
            base = a.get("lr_encdec", 2e-5) if enc else a.get("lr_body", 1e-4)
            if a.get("total_steps", 0) > 0:
                lr = ot.lr_at(step - 1, a["total_steps"], a["warmup_steps"], base=base, warm_start=a.get("warm_start", 1e-6),
                              final=a.get("final_lr_body", 1e-5) * base / a.get("lr_body", 1e-4))
            else:
                lr = base
            ot.adam_step(params[k], grads[k], mom[k], vel[k], step, lr)
    return losses, params, p0, norms


def _assert_updates(oc, d, params, p0, tol=1e-3):
    from oracle import model as om
    R, C, rr, cc = d["rc"]
    upd_got = np.concatenate([(d["params"][k] - om.local_tile(oc, k, p0[k], R, C, rr, cc)).ravel() for k in params])
    upd_ref = np.concatenate([(om.local_tile(oc, k, params[k] - p0[k], R, C, rr, cc)).ravel() for k in params])
    assert np.linalg.norm(upd_got - upd_ref) / np.linalg.norm(upd_ref) < tol


def _oc():
    from oracle import model as om
    meta = json.load(open(os.path.join(GOLD, "comm_golden.json")))
    return om.Config(**{**meta["config"], "grid": tuple(meta["config"]["grid"]), "patch": tuple(meta["config"]["patch"])})


@pytest.mark.parametrize("world", [1, 2, 4])
def test_train_step_schedule_and_global_clip_match_oracle(world):
    """lr_at warm-up + cosine (device schedule) and global-norm clipping over the sharded set
    (duplicated vectors counted once) reproduce the serial oracle, tile by tile."""
    from oracle import model as om, train as ot
    oc = _oc()
    z = np.load(os.path.join(GOLD, "wm_golden.npz"))
    model = om.SerialModel(oc, om.init_params(oc, 0, np.float64))
    _, g = ot.weighted_mse_loss(model.forward(z["x"][:1]), z["g_out"][:1] * 0.5, ot.lat_weights(oc.grid[0]),
                                np.ones(oc.n_vars))
    grads = model.backward(g)
    clip = 0.5 * float(np.sqrt(sum(float((v * v).sum()) for v in grads.values())))  # clipping active
    adam = {"warmup_steps": 1, "total_steps": 4}
    losses, params, p0, norms = _oracle_train(oc, [0], 3, adam, clip)
    assert norms[0] > clip
    res = _run(world, mode="train", opts={"adam": {**adam, "clip_norm": clip}, "steps": 3})
    want_scale = [min(1.0, clip / nm) for nm in norms]
    want_lr = [[ot.lr_at(s, 4, 1, base=b, final=1e-5 * b / 1e-4) for b in (2e-5, 1e-4)] for s in range(3)]
    assert want_lr[0] == [1e-6, 1e-6] and want_lr[1] == [2e-5, 1e-4]
    for d in res:
        assert np.allclose(d["losses"], [ls[0] for ls in losses], rtol=1e-5), (d["losses"], losses)
        assert np.allclose(d["scales"], want_scale, rtol=1e-5), (d["scales"], want_scale)
        assert np.allclose(d["lrs"], want_lr, rtol=1e-6), (d["lrs"], want_lr)
        _assert_updates(oc, d, params, p0)


@pytest.mark.parametrize("world,n_mp", [(2, 1), (4, 2)])
def test_dp_replicas_match_serial_batch(world, n_mp):
    """DP-equivalence: replicas of an n_mp-way model on different samples,
    gradients averaged over the r % n groups, equal a serial run on the mean gradient; shards
    stay identical across replicas."""
    oc = _oc()
    reps = world // n_mp
    losses, params, p0, _ = _oracle_train(oc, list(range(reps)), 2)
    res = _run(world, mode="train", opts={"mp": n_mp, "dp": True, "steps": 2})
    for d in res:
        k = d["rank"] // n_mp
        assert np.allclose(d["losses"], [ls[k] for ls in losses], rtol=1e-5), (d["losses"], losses)
        _assert_updates(oc, d, params, p0)
    by_pos = {}
    for d in res:
        by_pos.setdefault(d["pos"], []).append(d)
    for pos, ds in by_pos.items():
        for k in ds[0]["params"]:
            assert np.array_equal(ds[0]["params"][k], ds[-1]["params"][k]), (pos, k)


def test_train_step_symmetric_memory_8way():
    """Full step (loss, backward, grad sync, clip, scheduled Adam) on the 4 x 2 grid through the
    peer-memory transport plumbing."""
    from oracle import model as om, train as ot
    oc = _oc()
    z = np.load(os.path.join(GOLD, "wm_golden.npz"))
    model = om.SerialModel(oc, om.init_params(oc, 0, np.float64))
    _, g = ot.weighted_mse_loss(model.forward(z["x"][:1]), z["g_out"][:1] * 0.5, ot.lat_weights(oc.grid[0]),
                                np.ones(oc.n_vars))
    clip = 0.5 * float(np.sqrt(sum(float((v * v).sum()) for v in model.backward(g).values())))
    adam = {"warmup_steps": 1, "total_steps": 4}
    losses, params, p0, norms = _oracle_train(oc, [0], 2, adam, clip)
    res = _run(8, mode="train", opts={"adam": {**adam, "clip_norm": clip}, "steps": 2, "transport": "shm"})
    for d in res:
        assert np.allclose(d["losses"], [ls[0] for ls in losses], rtol=1e-5), (d["losses"], losses)
        assert np.allclose(d["scales"], [min(1.0, clip / nm) for nm in norms], rtol=1e-5)
        _assert_updates(oc, d, params, p0)


@pytest.mark.parametrize("world", [1, 4])
def test_checkpoint_roundtrip_and_resume(world, tmp_path):
    """save -> load -> save is byte-identical; a resumed run reproduces the
    uninterrupted run's next step exactly; one file per rank."""
    res = _run(world, mode="ckpt", opts={"dir": str(tmp_path)})
    assert len(os.listdir(tmp_path / "a")) == world
    for d in res:
        assert d["same"] and d["step"] == 2
        assert d["cont"] == d["resumed"] and d["params_equal"]


def test_checkpoint_world_shape_mismatch(tmp_path):
    """Loading a 4-way checkpoint into a 2-way world is an explicit error naming both shapes."""
    _run(4, mode="ckpt", opts={"dir": str(tmp_path)})
    res = _run(2, mode="ckpt_load", opts={"dir": str(tmp_path / "a")})
    for d in res:
        assert d["err"] is not None and "4-way" in d["err"] and "2-way" in d["err"], d["err"]


@pytest.mark.parametrize("world", [1, 4])
def test_trainer_rollout_finetune_matches_oracle(world):
    """finetune_rollout: tiles from the loader, r ~ U{1, 2} from a seeded generator (same on every
    rank), loss vs the target at lead r, one Adam counter across the per-r steps — equal to the
    serial oracle fed the same samples."""
    from oracle import model as om, train as ot
    oc = _oc()
    res = _run(world, mode="trainer")
    src = np.random.default_rng(7).standard_normal((6, *oc.grid, oc.n_vars))
    rs, order = res[0]["rollouts"], res[0]["order"]
    assert all(d["rollouts"] == rs and d["order"] == order for d in res) and set(rs) <= {1, 2}
    params = om.init_params(oc, 0, np.float64)
    p0 = {k: v.copy() for k, v in params.items()}
    mom = {k: np.zeros_like(v) for k, v in params.items()}
    vel = {k: np.zeros_like(v) for k, v in params.items()}
    losses = []
    for s, r in enumerate(rs):
        i = order[s]
        model = om.SerialModel(oc, params)
        loss, g = ot.weighted_mse_loss(model.forward(src[i:i + 1], r=r), src[i + r:i + r + 1],
                                       ot.lat_weights(oc.grid[0]), np.ones(oc.n_vars))
        grads = model.backward(g)
        losses.append(loss)
        for k in params:
            ot.adam_step(params[k], grads[k], mom[k], vel[k], s + 1, 2e-5 if k.split(".")[0] in ("enc", "dec") else 1e-4)
    for d in res:
        assert np.allclose(d["losses"], losses, rtol=1e-5), (d["losses"], losses)
        _assert_updates(oc, d, params, p0)


@pytest.mark.parametrize("world", [4, 8])
def test_adam_panel_push_matches_gathers(world):
    """bf16 operand copies over the peer-memory transport: Adam storing each channel-mixing
    weight's new copy into the column group's panel slots (jg_adam_push) gives bit-identical
    training to re-gathering the panels every forward — including after an external weight edit,
    which must trigger an eager re-gather."""
    base = {"transport": "shm", "dtype": "bf16"}
    push = _run(world, mode="pushcmp", opts={**base, "panel_push": "1"})
    gath = _run(world, mode="pushcmp", opts={**base, "panel_push": "0"})
    assert all(d["pushing"] for d in push) and not any(d["pushing"] for d in gath)
    for a, b in zip(push, gath):
        assert a["losses"] == b["losses"], (a["losses"], b["losses"])
        for k in a["params"]:
            assert np.array_equal(a["params"][k], b["params"][k]), k


@pytest.mark.parametrize("world,grid,transport", [(2, "2x1", "nccl"), (2, "2x1", "shm"), (4, "4x1", "nccl"),
                                                   (4, "4x1", "shm"), (8, "8x1", "shm")])
def test_grid_override_matches_reference(world, grid, transport):
    """JIGSAW_GRID: the R > C owner-sub-chunk path (q = R / C = 2, 4: the 4 x 2 grid's) and other
    factorisations on the real schedule, both transports, against the reference's n = 1 golden."""
    _check(world, opts={"grid": grid, "transport": transport})


@pytest.mark.parametrize("world,transport,dtype,grid", [(2, "nccl", "f32", None), (4, "shm", "bf16", None),
                                                        (8, "shm", "bf16", None), (8, "nccl", "f32", None),
                                                        (4, "shm", "bf16", "4x1")])
def test_comm_volume_matches_analytic(world, transport, dtype, grid):
    """Comm roofline numerator: the bytes each rank's transports and all-reduces actually issue in
    a steady-state training step equal jigsaw_grid.step_exchange_bytes (the schedule's analytic
    volume, the balanced-grid counterpart of the reference's comm_volume tables)."""
    opts = {"transport": transport, "dtype": dtype}
    if grid:
        opts["grid"] = grid
    res = _run(world, mode="comm", opts=opts)
    for d in res:
        ex, ar = d["measured"]
        assert ex == d["analytic"]["exchange"], (d["pos"], ex, d["analytic"])
        assert abs(ar - d["analytic"]["allreduce"]) <= 1e-6 * max(1.0, ar), (d["pos"], ar, d["analytic"])
        assert ex > 0


@pytest.mark.parametrize("world", [1, 2])
def test_trainer_resume_reproduces_uninterrupted_run(world, tmp_path):
    """Trainer checkpoints carry the epoch, the position in it and the rollout RNG's epoch-start
    state: resuming mid-epoch reproduces the uninterrupted fine-tuning run."""
    res = _run(world, mode="resume", opts={"dir": str(tmp_path / "ck")})
    for d in res:
        assert d["start"] == 2
        assert d["resumed_rollouts"] == d["rollouts"]
        np.testing.assert_allclose(d["resumed"], d["full"], rtol=1e-6, atol=0)
        assert d["same_params"]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_bf16_batched_token_layers_peer_memory(world):
    """bf16 operands and bf16 partial planes through the B > 1 plane-major path (batched
    reduce-scatter GEMM launches, plane_div) on emulated peer memory, against the reference."""
    _check(world, opts={"transport": "shm", "dtype": "bf16"}, tol=3e-2)
