"""tcgen05 GEMM parity against an fp64 reference of the same contraction (tensor.py:59-72 semantics)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import rel_err

pytestmark = pytest.mark.gpu


def _ref(a, b, mode):
    a64, b64 = a.double().cpu(), b.double().cpu()
    if mode == "NN":
        return a64 @ b64
    if mode == "NT":
        return a64 @ b64.transpose(-1, -2)
    return a64.transpose(-1, -2) @ b64


SHAPES = [(128, 128, 64), (64, 64, 128), (200, 300, 100), (384, 520, 272), (1000, 1030, 333), (4320 // 4, 4480 // 4, 1024)]


@pytest.mark.parametrize("mode", ["NN", "NT", "TN"])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_matmul_modes(cuda, mode, shape, dtype):
    from paper_2507_05753_b200 import tensor as T
    m, n, k = shape
    g = torch.Generator(device="cpu").manual_seed(m * 7 + n * 3 + k)
    if mode == "NN":
        a, b = torch.randn(m, k, generator=g), torch.randn(k, n, generator=g)
    elif mode == "NT":
        a, b = torch.randn(m, k, generator=g), torch.randn(n, k, generator=g)
    else:
        a, b = torch.randn(k, m, generator=g), torch.randn(k, n, generator=g)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    a_d, b_d = a.to(cuda, tdt), b.to(cuda, tdt)
    out = T.matmul(a_d, b_d, mode)
    torch.cuda.synchronize()
    ref = _ref(a_d.float(), b_d.float(), mode)  # exact product of the (rounded) operands
    err = rel_err(out.float().cpu().numpy(), ref.numpy())
    tol = 5e-5 if dtype == "f32" else 1e-2
    assert err < tol, (mode, shape, dtype, err)


@pytest.mark.parametrize("mode", ["NN", "NT", "TN"])
def test_matmul_batched_broadcast(cuda, mode):
    from paper_2507_05753_b200 import tensor as T
    g = torch.Generator(device="cpu").manual_seed(5)
    m, n, k = 136, 200, 96
    if mode == "NN":
        a, b = torch.randn(3, m, k, generator=g), torch.randn(k, n, generator=g)
    elif mode == "NT":
        a, b = torch.randn(3, m, k, generator=g), torch.randn(n, k, generator=g)
    else:
        a, b = torch.randn(3, k, m, generator=g), torch.randn(k, n, generator=g)
    out = T.matmul(a.cuda(), b.cuda(), mode)
    ref = _ref(a, b, mode)
    assert out.shape == ref.shape
    assert rel_err(out.cpu().numpy(), ref.numpy()) < 2e-5


def test_fixed_nt_example(cuda):
    # reference test_tensor.py:23-28
    from paper_2507_05753_b200 import tensor as T
    a = torch.tensor([[1.0, 2.0], [3.0, 4.0]], device=cuda)
    b = torch.tensor([[5.0, 6.0], [7.0, 8.0]], device=cuda)
    out = T.matmul(a, b, "NT")
    assert out.cpu().tolist() == [[17.0, 23.0], [39.0, 53.0]]
    outb = T.matmul(a.bfloat16(), b.bfloat16(), "NT")
    assert outb.float().cpu().tolist() == [[17.0, 23.0], [39.0, 53.0]]


def test_epilogue_fusions(cuda):
    """bias / residual / GELU fwd / GELU bwd / accumulate / stats epilogues vs torch fp64."""
    from paper_2507_05753_b200 import tensor as T, _lib
    g = torch.Generator(device="cpu").manual_seed(11)
    m, n, k = 300, 264, 200
    a = torch.randn(m, k, generator=g).cuda()
    w = torch.randn(n, k, generator=g).cuda()
    bias = torch.randn(n, generator=g).cuda()
    rbias = torch.randn(m, generator=g).cuda()
    resid = torch.randn(m, n, generator=g).cuda()
    pre = torch.randn(m, n, generator=g).cuda()
    acc = (a.double() @ w.double().T)
    # bias col + resid + stats + bf16 copy
    d = torch.empty(m, n, device=cuda)
    d2 = torch.empty(m, n, device=cuda, dtype=torch.bfloat16)
    st = torch.zeros(m, 2, device=cuda)
    T.gemm_into(d, a, w, _lib.JG_KMAJOR, _lib.JG_KMAJOR, m, n, k,
                epi=_lib.EPI_BIAS_COL | _lib.EPI_RESID | _lib.EPI_STATS | _lib.EPI_COPY_D2,
                bias=bias, resid=resid, stats=st, d2=d2)
    ref = acc + bias.double() + resid.double()
    assert rel_err(d.cpu(), ref.cpu()) < 2e-5
    assert rel_err(d2.float().cpu(), ref.cpu()) < 1e-2
    assert rel_err(st[:, 0].cpu(), ref.sum(1).cpu()) < 1e-5
    assert rel_err(st[:, 1].cpu(), (ref * ref).sum(1).cpu()) < 1e-5
    # row bias + gelu fwd
    d = torch.empty(m, n, device=cuda)
    d2 = torch.empty(m, n, device=cuda)
    T.gemm_into(d, a, w, _lib.JG_KMAJOR, _lib.JG_KMAJOR, m, n, k, epi=_lib.EPI_BIAS_ROW | _lib.EPI_GELU_FWD,
                bias=rbias, d2=d2)
    ref = acc + rbias.double()[:, None]
    assert rel_err(d.cpu(), ref.cpu()) < 2e-5
    gref = ref * 0.5 * (1 + torch.erf(ref / np.sqrt(2)))
    assert rel_err(d2.cpu(), gref.cpu()) < 2e-5
    # gelu bwd
    d = torch.empty(m, n, device=cuda)
    T.gemm_into(d, a, w, _lib.JG_KMAJOR, _lib.JG_KMAJOR, m, n, k, epi=_lib.EPI_GELU_BWD, pre=pre)
    p64 = pre.double()
    dg = 0.5 * (1 + torch.erf(p64 / np.sqrt(2))) + p64 * torch.exp(-0.5 * p64 * p64) / np.sqrt(2 * np.pi)
    assert rel_err(d.cpu(), (acc * dg).cpu()) < 2e-5
    # accumulate
    d = resid.clone()
    T.gemm_into(d, a, w, _lib.JG_KMAJOR, _lib.JG_KMAJOR, m, n, k, epi=_lib.EPI_ACCUM)
    assert rel_err(d.cpu(), (acc + resid.double()).cpu()) < 2e-5


def test_reduce_batch(cuda):
    """sum_b A[b]^T B[b] with the batch folded into the K loop (weight-gradient form)."""
    from paper_2507_05753_b200 import tensor as T, _lib
    g = torch.Generator(device="cpu").manual_seed(3)
    bsz, t, e, dt = 3, 160, 136, 200
    u = torch.randn(bsz, t, e, generator=g).cuda()
    gh = torch.randn(bsz, e, dt, generator=g).cuda()
    # dW1[t, j] = sum_b sum_e u[b,t,e] gh[b,e,j] : A = u K-major (K = e), B = gh MN-major
    out = torch.zeros(t, dt, device=cuda)
    T.gemm_into(out, u, gh, _lib.JG_KMAJOR, _lib.JG_MNMAJOR, t, dt, e, bsz, t * e, e * dt,
                reduce_batch=True, epi=_lib.EPI_ACCUM)
    ref = torch.einsum("bte,bej->tj", u.double(), gh.double())
    assert rel_err(out.cpu(), ref.cpu()) < 2e-5


@pytest.mark.parametrize("batch,m,n,k", [(1, 300, 520, 256), (2, 257, 1032, 192)])
def test_lnb_epilogue_moments(cuda, batch, m, n, k):
    """JG_EPI_LNB: the GEMM result g is stored unchanged and its layer-norm-backward row moments
    (sum g*gamma, sum g*gamma*xhat) land in `stats` (ln_bwd_moments semantics, model.py:242-250),
    per batch, including ragged row / column tiles and 2-CTA tiles."""
    from paper_2507_05753_b200 import _lib, tensor as T
    gen = torch.Generator(device="cpu").manual_seed(11)
    a = torch.randn(batch, m, k, generator=gen).to(cuda, torch.bfloat16)
    b = torch.randn(n, k, generator=gen).to(cuda, torch.bfloat16)
    x = torch.randn(batch, m, n, generator=gen).to(cuda)
    gamma = torch.randn(n, generator=gen).to(cuda)
    mr = torch.stack([torch.randn(batch * m, generator=gen), torch.rand(batch * m, generator=gen) + 0.5], 1).to(cuda)
    out = torch.empty(batch, m, n, device=cuda)
    stats = torch.zeros(batch * m, 2, device=cuda)
    T.gemm_into(out, a, b, _lib.JG_KMAJOR, _lib.JG_KMAJOR, m, n, k, batch, m * k, 0, epi=_lib.EPI_LNB,
                stats=stats, lnb=(x, gamma, mr))
    torch.cuda.synchronize()
    ref = (a.double() @ b.double().t())
    assert rel_err(out.double().cpu().numpy(), ref.cpu().numpy()) < 1e-5
    g = out.double().reshape(batch * m, n)
    h = g * gamma.double()[None, :]
    xhat = (x.double().reshape(batch * m, n) - mr[:, :1].double()) * mr[:, 1:].double()
    want = torch.stack([h.sum(1), (h * xhat).sum(1)], 1)
    assert rel_err(stats.double().cpu().numpy(), want.cpu().numpy()) < 1e-5


@pytest.mark.parametrize("majors", [(0, 0), (1, 1), (0, 1)])
@pytest.mark.parametrize("k", [4320, 16380])
def test_tf32x3_long_k_accuracy(cuda, majors, k):
    """fp32 mode at the C4 contraction lengths: tcgen05's fp32 accumulation truncates, so long-K
    3xTF32 GEMMs accumulate K-chunks into planes summed round-to-nearest (tensor.TF32X3_KCHUNK);
    without the chunking K = 16380 measured 2.2e-4 (tools/f32_diag.py)."""
    from paper_2507_05753_b200 import _lib, tensor as T
    am, bm = majors
    gen = torch.Generator(device="cuda").manual_seed(k + 10 * am + bm)
    m, n = 384, 272
    a = torch.randn((m, k) if am == 0 else (k, m), device=cuda, generator=gen)
    b = torch.randn((n, k) if bm == 0 else (k, n), device=cuda, generator=gen)
    bias = torch.randn(n, device=cuda, generator=gen)
    out = torch.empty(m, n, device=cuda)
    d2 = torch.empty(m, n, device=cuda)
    st = torch.zeros(m, 2, device=cuda)
    T.gemm_into(out, a, b, am, bm, m, n, k, epi=_lib.EPI_BIAS_COL | _lib.EPI_GELU_FWD | _lib.EPI_STATS,
                bias=bias, d2=d2, stats=st)
    torch.cuda.synchronize()
    ref = (a.double() if am == 0 else a.double().t()) @ (b.double().t() if bm == 0 else b.double()) + bias.double()
    e = rel_err(out.cpu().numpy(), ref.cpu().numpy())
    print(f"3xTF32 majors {am}{bm} K={k}: rel {e:.2e}")
    assert e < 2e-5, e
    gref = ref * 0.5 * (1 + torch.erf(ref / np.sqrt(2)))
    assert rel_err(d2.cpu().numpy(), gref.cpu().numpy()) < 2e-5
    assert rel_err(st[:, 1].cpu().numpy(), (ref * ref).sum(1).cpu().numpy()) < 2e-5


def test_tf32x3_long_k_lnb_and_reduce_batch(cuda):
    """Chunked 3xTF32 with the layer-norm-backward moments (JG_EPI_LNB -> jg_ln_bwd_moments on the
    finished output) and with a batch folded into K (reduce_batch, weight gradients)."""
    from paper_2507_05753_b200 import _lib, tensor as T
    gen = torch.Generator(device="cuda").manual_seed(5)
    m, n, k = 256, 320, 8640
    a = torch.randn(m, k, device=cuda, generator=gen)
    b = torch.randn(n, k, device=cuda, generator=gen)
    x = torch.randn(m, n, device=cuda, generator=gen)
    gamma = torch.randn(n, device=cuda, generator=gen)
    mr = torch.stack([torch.randn(m, device=cuda, generator=gen), torch.rand(m, device=cuda, generator=gen) + 0.5], 1)
    out = torch.empty(m, n, device=cuda)
    stats = torch.zeros(m, 2, device=cuda)
    T.gemm_into(out, a, b, _lib.JG_KMAJOR, _lib.JG_KMAJOR, m, n, k, epi=_lib.EPI_LNB, stats=stats, lnb=(x, gamma, mr))
    ref = a.double() @ b.double().t()
    assert rel_err(out.cpu().numpy(), ref.cpu().numpy()) < 2e-5
    h = ref * gamma.double()[None, :]
    xhat = (x.double() - mr[:, :1].double()) * mr[:, 1:].double()
    want = torch.stack([h.sum(1), (h * xhat).sum(1)], 1)
    assert rel_err(stats.cpu().numpy(), want.cpu().numpy()) < 2e-5
    # reduce_batch: dW[t, j] = sum_b sum_e u[b, t, e] gh[b, e, j], K = e long
    bsz, t, e, dt = 2, 192, 4480, 160
    u = torch.randn(bsz, t, e, device=cuda, generator=gen)
    gh = torch.randn(bsz, e, dt, device=cuda, generator=gen)
    dw = torch.zeros(t, dt, device=cuda)
    T.gemm_into(dw, u, gh, _lib.JG_KMAJOR, _lib.JG_MNMAJOR, t, dt, e, bsz, t * e, e * dt, reduce_batch=True,
                epi=_lib.EPI_ACCUM)
    want = torch.einsum("bte,bej->tj", u.double(), gh.double())
    assert rel_err(dw.cpu().numpy(), want.cpu().numpy()) < 2e-5


@pytest.mark.parametrize("tile_n", [128, 256])
@pytest.mark.parametrize("majors", [(0, 0), (1, 1)])
def test_forced_tile_width_same_result(cuda, tile_n, majors):
    """jg_gemm_desc.tile_n (forced 128- / 256-wide tiles on CTA pairs) gives the per-shape
    choice's result bit for bit (the K loop order per output element does not change)."""
    from paper_2507_05753_b200 import ShapeError, tensor as T
    m, n, k = 520, 776, 384
    g = torch.Generator(device="cpu").manual_seed(11)
    am, bm = majors
    a = torch.randn((m, k) if am == 0 else (k, m), generator=g).to(cuda, torch.bfloat16)
    b = torch.randn((n, k) if bm == 0 else (k, n), generator=g).to(cuda, torch.bfloat16)
    auto = torch.empty(m, n, device=cuda)
    T.gemm_into(auto, a, b, am, bm, m, n, k)
    forced = torch.empty_like(auto)
    try:
        T.GEMM_TILE_N = tile_n
        T.gemm_into(forced, a, b, am, bm, m, n, k)
        T.GEMM_TILE_N = 64  # CTA pairs need 128- or 256-wide tiles
        with pytest.raises(ShapeError):
            T.gemm_into(forced, a, b, am, bm, m, n, k)
    finally:
        T.GEMM_TILE_N = 0
    torch.cuda.synchronize()
    assert torch.equal(forced, auto)
    ref = (a.double().cpu() if am == 0 else a.double().cpu().T) @ (b.double().cpu().T if bm == 0 else b.double().cpu())
    assert rel_err(auto.cpu().numpy(), ref.numpy()) < 1e-2
