"""3xTF32 precision diagnostics: jg_gemm f32-mode error vs fp64 as a function of K and operand
majors, and the C3 (1 block) forward activations of the fused model vs the f64 oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2507_05753_b200 import tensor as T, _lib

_lib.load()
g = torch.Generator(device="cuda").manual_seed(0)
for (am, bm) in ((0, 0), (1, 1), (0, 1)):
    for k in (64, 512, 4320, 16380):
        m, n = 512, 384
        A = torch.randn((m, k) if am == 0 else (k, m), device="cuda", generator=g)
        B = torch.randn((n, k) if bm == 0 else (k, n), device="cuda", generator=g)
        out = torch.empty(m, n, device="cuda")
        T.gemm_into(out, A, B, am, bm, m, n, k)
        At = (A if am == 0 else A.t()).double()
        Bt = (B.t() if bm == 0 else B).double()
        ref = At @ Bt
        e = ((out.double() - ref).abs().max() / ref.abs().max()).item()
        # what single TF32 and plain fp32 would give
        tf = lambda x: (x.view(torch.int32) & ~0x1FFF).view(torch.float32)  # noqa: E731
        ref_tf = (tf(At.float()).double() @ tf(Bt.float()).double())
        e_tf = ((ref_tf - ref).abs().max() / ref.abs().max()).item()
        print(f"majors {am}{bm} K={k:6d}: 3xTF32 rel {e:.2e} | 1xTF32 would be {e_tf:.2e}", flush=True)

# ---- per-layer activations, C3 geometry with 1 block, f32 mode vs the f64 oracle ----------
from oracle import model as om, ops  # noqa: E402
from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel  # noqa: E402
cfg = dict(n_vars=72, grid=(128, 256), patch=(4, 4), d_emb=1024, d_tok=2048, d_ch=1024, n_blocks=1)
oc = om.Config(**cfg)
P = {k: v.astype(np.float32).astype(np.float64) for k, v in om.init_params(oc, 0, np.float64).items()}
rng = np.random.default_rng(1)
x = rng.standard_normal((1, 128, 256, 72), dtype=np.float32)
xp = ops.patchify(x.astype(np.float64), 4, 4)
h0 = ops.matmul(xp, P["enc.w"], "NT") + P["enc.b"]
ref = om.SerialModel(oc, P)
u, (xh, inv) = ref._ln(h0, "block0.ln1.")
t1 = ops.matmul(u, P["block0.tok1.w"], "TN") + P["block0.tok1.b"]
a = ops.gelu(t1)
o = ops.matmul(P["block0.tok2.w"], a, "NT") + P["block0.tok2.b"][:, None]
x2 = h0 + o
v, _ = ref._ln(x2, "block0.ln2.")
cc = ops.matmul(v, P["block0.ch1.w"], "NT") + P["block0.ch1.b"]
ca = ops.gelu(cc)
y = x2 + ops.matmul(ca, P["block0.ch2.w"], "NT") + P["block0.ch2.b"]
dec = ops.matmul(y, P["dec.w"], "NT") + P["dec.b"]
m = WeatherMixerModel(MpContext(Communicator.local(), [0]), ModelConfig(**cfg), seed=0, dtype="f32")
m.forward(torch.from_numpy(x))
torch.cuda.synchronize()
ws = m._ws


def rel(got, exp):
    got = got.double().cpu().numpy().reshape(exp.shape)
    return float(np.abs(got - exp).max() / np.abs(exp).max())


for name, got, exp in (("xp", ws.xp, xp), ("enc out", ws.res[0], h0), ("u=LN1", ws.u[0], u), ("h (tok1)", ws.h[0], t1),
                       ("a=gelu", ws.a[0], a), ("x2", ws.x2[0], x2), ("v=LN2", ws.v[0], v), ("c (ch1)", ws.c[0], cc),
                       ("ca", ws.ca[0], ca), ("y", ws.res[1], y), ("dec", ws.dec, dec)):
    print(f"{name:10s} rel {rel(got, exp):.2e}")
