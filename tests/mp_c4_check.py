"""Jigsaw-sharded vs single-GPU parity at the BENCHMARKED scale (launched by
tests/test_jigsaw_gpu.py under torchrun): C4 geometry (721 -> 728 x 1440, 69 -> 70 channels,
d_emb 4320, d_tok 8640, T = 16380) with one mixer block, bf16. Every rank runs the sharded
forward + backward of an upstream gradient on its tiles, and ALSO the single-GPU model on the
whole sample on its own GPU, then compares its tiles of the output and of every parameter
gradient with the matching slices of the single-GPU result (north_star: the Jigsaw-sharded run
agrees with the single-GPU run to the bf16 tolerance, 2e-2). Prints one JSON line on rank 0."""
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

C4 = dict(n_vars=70, grid=(728, 1440), patch=(8, 8), d_emb=4320, d_tok=8640, d_ch=4320, n_blocks=1)


def main():
    comm = Communicator.from_env()
    ctx = MpContext(comm, list(range(comm.world_size)))
    cfg = ModelConfig(**C4)
    oc = om.Config(**C4)
    rng = np.random.default_rng(5)
    shape = (1, 728, 1440, 70)
    x = rng.standard_normal(shape, dtype=np.float32)
    g = rng.standard_normal(shape, dtype=np.float32) * 1e-3
    for a in (x, g):
        a[:, 721:] = 0
        a[..., 69:] = 0
    # sharded run
    model = WeatherMixerModel(ctx, cfg, seed=0, dtype="bf16", lat_real=721, vars_real=69)
    xl = om.local_sample(oc, x, ctx.R, ctx.C, ctx.r, ctx.c)
    gl = om.local_sample(oc, g, ctx.R, ctx.C, ctx.r, ctx.c)
    model.zero_grads()
    out = model.forward(torch.from_numpy(xl)).cpu().numpy()
    model.backward(torch.from_numpy(gl))
    model.grad_sync()
    torch.cuda.synchronize()
    mine = {k: p.grad.float().cpu().numpy() for k, p in model.params.items()}
    del model
    torch.cuda.empty_cache()
    # the single-GPU run of the same model on this rank's GPU
    single = WeatherMixerModel(MpContext(Communicator.local(), [0]), cfg, seed=0, dtype="bf16", lat_real=721,
                               vars_real=69)
    single.zero_grads()
    out1 = single.forward(torch.from_numpy(x)).cpu().numpy()
    single.backward(torch.from_numpy(g))
    torch.cuda.synchronize()
    worst_out = rel_err(out, om.local_sample(oc, out1, ctx.R, ctx.C, ctx.r, ctx.c))
    worst_grad, worst_name = 0.0, ""
    for name, p in single.params.items():
        ref = om.local_tile(oc, name, p.grad.double().cpu().numpy(), ctx.R, ctx.C, ctx.r, ctx.c)
        e = rel_err(mine[name], ref)
        if e > worst_grad:
            worst_grad, worst_name = e, name
    res = torch.tensor([worst_out, worst_grad], dtype=torch.float64, device="cuda")
    allres = [torch.zeros_like(res) for _ in range(comm.world_size)]
    dist.all_gather(allres, res)
    if comm.rank == 0:
        vals = [r.tolist() for r in allres]
        print("MPC4 " + json.dumps({"n": comm.world_size, "grid": [ctx.R, ctx.C], "out": max(v[0] for v in vals),
                                    "grad": max(v[1] for v in vals), "worst_param_rank0": worst_name}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
