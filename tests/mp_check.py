"""Multi-GPU Jigsaw parity check (launched by tests/test_jigsaw_gpu.py under torchrun).

Each rank runs the sharded model on its GPU (NCCL); rank 0 gathers outputs and gradients and
compares them with (a) the reference's golden vectors (G1 config) and (b) the oracle's f64 run
at C2 scale, printing one JSON line with the worst relative errors."""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

from conftest import rel_err  # noqa: E402
from oracle import model as om  # noqa: E402
from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel  # noqa: E402


def gather_np(x):
    objs = [None] * dist.get_world_size()
    dist.all_gather_object(objs, x)
    return objs


def run_case(ctx, cfg_dict, dtype, x, g, ref_out, ref_grads, r=1):
    cfg = ModelConfig.from_dict(cfg_dict)
    oc = om.Config(**{**cfg_dict, "grid": tuple(cfg_dict["grid"]), "patch": tuple(cfg_dict["patch"])})
    model = WeatherMixerModel(ctx, cfg, seed=0, dtype=dtype)
    xl = om.local_sample(oc, x, ctx.R, ctx.C, ctx.r, ctx.c)
    gl = om.local_sample(oc, g, ctx.R, ctx.C, ctx.r, ctx.c)
    model.zero_grads()
    out = model.forward(torch.tensor(xl, dtype=torch.float32), r=r)
    model.backward(torch.tensor(gl, dtype=torch.float32))
    model.grad_sync()
    torch.cuda.synchronize()
    mine = {"rc": (ctx.R, ctx.C, ctx.r, ctx.c), "out": out.cpu().numpy(),
            "grads": {k: p.grad.cpu().numpy() for k, p in model.params.items()}}
    allr = gather_np(mine)
    if ctx.comm.rank != 0:
        return None
    if ref_out is None:
        return allr
    worst_out = max(rel_err(d["out"], om.local_sample(oc, ref_out, *d["rc"])) for d in allr)
    worst_grad, worst_name = 0.0, ""
    for name, ref in ref_grads.items():
        for d in allr:
            e = rel_err(d["grads"][name], om.local_tile(oc, name, ref, *d["rc"]))
            if e > worst_grad:
                worst_grad, worst_name = e, name
    return {"out": worst_out, "grad": worst_grad, "worst_param": worst_name}


def main():
    if os.environ.get("JIGSAW_OVERSUBSCRIBE") == "1":
        # more ranks than GPUs (e.g. the 4 x 2 grid on a 4-GPU box): ranks share devices, so the
        # small collectives go over gloo (NCCL refuses two ranks per GPU); the Jigsaw exchanges
        # still run through symmetric peer memory
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
        comm = Communicator.from_env(backend="gloo")
    else:
        comm = Communicator.from_env()
    ctx = MpContext(comm, list(range(comm.world_size)))
    z = np.load(os.path.join(HERE, "golden", "wm_golden.npz"))
    meta = json.load(open(os.path.join(HERE, "golden", "comm_golden.json")))
    results = {"n": comm.world_size}
    gref = {k: z["grad_f64/" + k] for k in meta["param_names"]}
    for dtype in ("f32", "bf16"):
        results[f"G1_{dtype}"] = run_case(ctx, meta["config"], dtype, z["x"], z["g_out"], z["out_f64"], gref)
    # C2 scale against the oracle (f64), computed on every rank (cheap)
    c2 = dict(n_vars=72, grid=(32, 64), patch=(2, 2), d_emb=512, d_tok=1024, d_ch=512, n_blocks=12)
    oc = om.Config(**c2)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1, 32, 64, 72))
    g = rng.standard_normal((1, 32, 64, 72))
    ref = om.SerialModel(oc, om.init_params(oc, 0, np.float64))
    out_ref = ref.forward(x)
    grads_ref = ref.backward(g)
    for dtype in ("f32", "bf16"):
        results[f"C2_{dtype}"] = run_case(ctx, {**c2, "grid": list(c2["grid"]), "patch": list(c2["patch"])}, dtype,
                                          x, g, out_ref, grads_ref)
    if os.environ.get("MPCHECK_TRANSPORTS") == "1":
        # the same sharded step over NVLink peer memory and over NCCL: bit-identical results
        runs = {}
        for kind in ("symm", "nccl"):
            os.environ["JIGSAW_TRANSPORT"] = kind
            runs[kind] = {dt: run_case(ctx, meta["config"], dt, z["x"], z["g_out"], None, None) for dt in ("f32", "bf16")}
        os.environ.pop("JIGSAW_TRANSPORT")
        if comm.rank == 0:
            for dt in ("f32", "bf16"):
                diff = 0.0  # worst rel_err over the output and every gradient tile
                for a, b in zip(runs["symm"][dt], runs["nccl"][dt]):
                    diff = max(diff, rel_err(a["out"], b["out"]))
                    for k in a["grads"]:
                        diff = max(diff, rel_err(a["grads"][k], b["grads"][k]))
                results[f"symm_vs_nccl_{dt}"] = diff
    results["grid"] = [ctx.R, ctx.C]
    if comm.rank == 0:
        print("MPCHECK " + json.dumps(results), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
