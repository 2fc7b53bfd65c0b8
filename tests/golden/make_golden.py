"""Generate golden vectors by running the UNMODIFIED reference package (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/wm_golden.npz and tests/golden/comm_golden.json. The reference lives only
in the build container; the fixtures travel with the repo so the GPU box never needs it.

Model fixture "G1": the reference's default ModelConfig (model.py:41-50) with n_blocks=2,
batch 2, seed 0, inputs x ~ N(0,1) from default_rng(1), upstream gradient g_out ~ N(0,1) from
default_rng(2). The reference has no loss function, so backward is driven with g_out directly
(model.backward(g_out), model.py:428). Runs: n=1 f64 (gold), n=1 f32, n=2 and n=4 f64 via
run_spmd (threads, runtime.py:21), and an r=2 rollout at n=1 f64.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from jigsaw.comm import InProcWorld  # noqa: E402
from jigsaw.model import ModelConfig, WeatherMixerModel  # noqa: E402
from jigsaw.parallel import MpContext, comm_volume, primitive_send_elements  # noqa: E402
from jigsaw.runtime import run_spmd  # noqa: E402
from jigsaw.tensor import MatmulMode  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CFG = dict(n_vars=8, grid=(32, 64), patch=(4, 4), d_emb=64, d_tok=128, d_ch=64, n_blocks=2)
B = 2


def digest(params: dict) -> str:
    h = hashlib.sha256()
    for name in params:
        h.update(name.encode())
        h.update(np.ascontiguousarray(params[name]).tobytes())
    return h.hexdigest()[:16]


def local_x(x, n, pos):
    if n == 1:
        return x.copy()
    if n == 2:
        c = x.shape[-1] // 2
        return np.ascontiguousarray(x[..., pos * c:(pos + 1) * c])
    lon, c = x.shape[2] // 2, x.shape[3] // 2
    return np.ascontiguousarray(x[:, :, (pos // 2) * lon:(pos // 2 + 1) * lon, (pos % 2) * c:(pos % 2 + 1) * c])


def run(n, dtype, x, g_out, r=1):
    def worker(comm):
        ctx = MpContext(comm, list(range(n)))
        model = WeatherMixerModel(ctx, ModelConfig(**CFG), seed=0, dtype=dtype)
        model.zero_grads()
        out = model.forward(local_x(x, n, ctx.pos).astype(model.dtype), r=r)
        model.backward(local_x(g_out, n, ctx.pos).astype(model.dtype))
        model.grad_sync()
        grads = {k: p.grad.copy() for k, p in model.params.items()}
        data = {k: p.data.copy() for k, p in model.params.items()}
        return ctx.pos, out, grads, data, ctx.flops, comm.sent_elements, model
    res = run_spmd(n, worker)
    res = sorted(res, key=lambda t: t[0])
    model = res[0][6]
    g_grads, g_data = {}, {}
    for name in res[0][2]:
        g_grads[name] = model.gather_global(name, {t[0]: t[2][name] for t in res})
        g_data[name] = model.gather_global(name, {t[0]: t[3][name] for t in res})
    outs = [t[1] for t in res]
    flops = sum(t[4] for t in res)
    sent = [int(t[5]) for t in res]
    return outs, g_grads, g_data, flops, sent, model


def main():
    x = np.random.default_rng(1).standard_normal((B, 32, 64, 8))
    g_out = np.random.default_rng(2).standard_normal((B, 32, 64, 8))
    out1, gr1, data1, flops1, _, m1 = run(1, "f64", x, g_out)
    out1f, gr1f, data1f, _, _, _ = run(1, "f32", x, g_out)
    out2, gr2, _, flops2, sent2, m2 = run(2, "f64", x, g_out)
    out4, gr4, _, flops4, sent4, m4 = run(4, "f64", x, g_out)
    outr, grr, _, _, _, _ = run(1, "f64", x[:1], g_out[:1], r=2)

    def maxrel(a, b):
        return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))

    arrays = {"x": x, "g_out": g_out, "out_f64": out1[0], "out_f32": out1f[0].astype(np.float32),
              "rollout_out_f64": outr[0]}
    for name in gr1:
        arrays["grad_f64/" + name] = gr1[name]
        arrays["grad_f32/" + name] = gr1f[name].astype(np.float32)
        arrays["rollout_grad_f64/" + name] = grr[name]
    for pos in range(4):
        arrays[f"n4_out_local/{pos}"] = out4[pos]
    for pos in range(2):
        arrays[f"n2_out_local/{pos}"] = out2[pos]
    np.savez_compressed(os.path.join(HERE, "wm_golden.npz"), **arrays)

    meta = {
        "config": CFG, "batch": B, "seed": 0,
        "init_digest_f64": digest(data1), "init_digest_f32": digest(data1f),
        "param_names": list(gr1.keys()),
        "flops_n1": int(flops1), "flops_n2": int(flops2), "flops_n4": int(flops4),
        "n2_vs_n1_grad_maxrel": max(maxrel(gr2[k], gr1[k]) for k in gr1 if np.any(gr1[k])),
        "n4_vs_n1_grad_maxrel": max(maxrel(gr4[k], gr1[k]) for k in gr1 if np.any(gr1[k])),
        "sent_elements_n2": sent2, "sent_elements_n4": sent4,
        "step_comm_volume": {f"n{n}_b{b}_r{r}": int(m.step_comm_volume(b, r))
                             for n, m in ((2, m2), (4, m4)) for b in (1, 2) for r in (1, 3)},
    }
    # analytic primitive tables (parallel.py:361-401) on a few shapes
    prim = {}
    for mode in ("NT", "NN", "TN"):
        for n in (1, 2, 4):
            for a_shape, b_shape in (((2, 6, 8), (4, 8)), ((6, 8), (8, 4)), ((3, 4, 6), (4, 10))):
                try:
                    prim[f"{mode}/{n}/{a_shape}/{b_shape}"] = primitive_send_elements(MatmulMode(mode), n, a_shape, b_shape)
                except Exception as e:  # noqa: BLE001
                    prim[f"{mode}/{n}/{a_shape}/{b_shape}"] = repr(e)
    meta["primitive_send_elements"] = prim
    meta["comm_volume"] = {f"{mode}/{n}/{m},{k},{no},b{b}": [rep.forward_sent, rep.backward_sent]
                           for mode in ("NT", "NN", "TN") for n in (2, 4)
                           for (m, k, no, b) in ((128, 64, 128, 1), (256, 64, 32, 2))
                           for rep in [comm_volume(m, k, no, n, MatmulMode(mode), batch=b)]}
    with open(os.path.join(HERE, "comm_golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(json.dumps({k: v for k, v in meta.items() if k not in ("primitive_send_elements", "comm_volume", "param_names")}, indent=1))


if __name__ == "__main__":
    main()
