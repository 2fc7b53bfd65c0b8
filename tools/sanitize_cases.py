"""Small-shape workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel
family of libjigsaw_sm100.so at shapes that still take the real code paths (1-CTA and 2-CTA
cta_group::2 tiles, ragged edges, K tails, MN-/K-major operands, batched and batch-reduced
GEMMs, every epilogue incl. LNB and the TMA-store path, 3xTF32), the row-wise kernels, and a
full tiny training step (forward, loss, backward, Adam) as the model runs it.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_05753_b200 import _lib, tensor as T  # noqa: E402

_lib.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device="cuda").manual_seed(0)
E = _lib


def rnd(*shape, dt=torch.bfloat16):
    return torch.randn(*shape, device=dev, generator=g).to(dt)


# GEMMs: (m, n, k) incl. 2-CTA tiles (m > 128), ragged edges and K tails; all operand majors
for dt in (torch.bfloat16, torch.float32):
    for (m, n, k) in ((128, 64, 64), (300, 264, 200), (520, 392, 328)):
        for am in (0, 1):
            for bm in (0, 1):
                a = rnd(*((m, k) if am == 0 else (k, m)), dt=dt)
                b = rnd(*((n, k) if bm == 0 else (k, n)), dt=dt)
                out = torch.empty(m, n, device=dev)
                T.gemm_into(out, a, b, am, bm, m, n, k)
    m, n, k = 264, 200, 136
    a, w = rnd(m, k, dt=dt), rnd(n, k, dt=dt)
    bias, rbias = rnd(n, dt=torch.float32), rnd(m, dt=torch.float32)
    resid, pre = rnd(m, n, dt=torch.float32), rnd(m, n, dt=torch.float32)
    d = torch.empty(m, n, device=dev)
    d2 = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    st = torch.zeros(m, 2, device=dev)
    T.gemm_into(d, a, w, 0, 0, m, n, k, epi=E.EPI_BIAS_COL | E.EPI_RESID | E.EPI_STATS | E.EPI_COPY_D2, bias=bias,
                resid=resid, stats=st, d2=d2)
    T.gemm_into(d, a, w, 0, 0, m, n, k, epi=E.EPI_BIAS_ROW | E.EPI_GELU_FWD, bias=rbias, d2=d2)
    T.gemm_into(d, a, w, 0, 0, m, n, k, epi=E.EPI_GELU_BWD, pre=pre)
    T.gemm_into(d, a, w, 0, 0, m, n, k, epi=E.EPI_ACCUM)
    x = rnd(m, n, dt=torch.float32)
    gam = rnd(n, dt=torch.float32)
    mr = torch.stack([rnd(m, dt=torch.float32), torch.rand(m, device=dev) + 0.5], 1)
    T.gemm_into(d, a, w, 0, 0, m, n, k, epi=E.EPI_LNB, stats=st, lnb=(x, gam, mr))
    # batch-reduced (weight-gradient form) and batched
    u, gh = rnd(3, 160, 136, dt=dt), rnd(3, 136, 200, dt=dt)
    dw = torch.zeros(160, 200, device=dev)
    T.gemm_into(dw, u, gh, 0, 1, 160, 200, 136, 3, 160 * 136, 136 * 200, reduce_batch=True, epi=E.EPI_ACCUM)
    T.matmul(rnd(3, 136, 96, dt=dt), rnd(200, 96, dt=dt), "NT")
# long-K 3xTF32 (chunked accumulation path)
T.matmul(rnd(128, 1100, dt=torch.float32), rnd(1100, 96, dt=torch.float32), "NN")

# row-wise kernels through the public L0 API
x = rnd(4, 96, 128, dt=torch.float32)
gam, bet = rnd(128, dt=torch.float32), rnd(128, dt=torch.float32)
T.layer_norm(x, gam, bet)
T.layer_norm_backward(x, gam, 1e-5, rnd(4, 96, 128, dt=torch.float32))
T.gelu(x)
T.gelu_backward(x, x)
tok = T.patchify(rnd(2, 32, 64, 8, dt=torch.float32), 4, 4)
T.unpatchify(tok, 32, 64, 4, 4)

# a full tiny training step (fused model path, both dtypes) and a graph-captured one
from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel  # noqa: E402
from paper_2507_05753_b200.engine import TrainStep  # noqa: E402

cfg = ModelConfig(n_vars=8, grid=(32, 64), patch=(4, 4), d_emb=64, d_tok=128, d_ch=64, n_blocks=2)
rng = np.random.default_rng(0)
xs = torch.tensor(rng.standard_normal((2, 32, 64, 8)), dtype=torch.float32)
ts = torch.tensor(rng.standard_normal((2, 32, 64, 8)), dtype=torch.float32)
for dtype in ("bf16", "f32"):
    model = WeatherMixerModel(MpContext(Communicator.local(), [0]), cfg, seed=0, dtype=dtype, lat_real=30, vars_real=7)
    step = TrainStep(model, batch=2, graph=dtype == "bf16")
    for _ in range(2):
        loss = step(xs, ts)
    assert np.isfinite(loss)
torch.cuda.synchronize()
print("SANITIZE_CASES_DONE", flush=True)
