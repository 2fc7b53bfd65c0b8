"""Memory-safety and race checks of our own (compute-sanitizer is closed on this GPU pool):

* guard bands — every output is a window inside a larger buffer pre-filled with a sentinel bit
  pattern; after the kernel, every byte outside the window (before, after, and the padding
  columns of a row stride ldd > n) must still hold the sentinel: no out-of-bounds store from
  the TMA-store epilogue, the ragged-edge paths, the 2-CTA tiles or the row-wise kernels;
* determinism — the same GEMM (2-CTA tiles, long K, every epilogue without atomics), layer-norm
  and Adam launch repeated must give bit-identical results: a race in the mbarrier / TMEM
  pipeline or the smem staging would show up as run-to-run differences.
"""
from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu

SENT = -12345.678


def _guarded(rows, cols, ld, dtype, pad=4096):
    """(whole buffer, [rows, cols] view with row stride ld) in the middle of a sentinel buffer."""
    n = pad + rows * ld + pad
    buf = torch.full((n,), SENT, dtype=dtype, device="cuda")
    view = torch.as_strided(buf, (rows, cols), (ld, 1), pad)
    return buf, view


def _check_guard(buf, rows, cols, ld, pad=4096):
    mask = torch.ones_like(buf, dtype=torch.bool)
    idx = pad + torch.arange(rows, device=buf.device)[:, None] * ld + torch.arange(cols, device=buf.device)[None, :]
    mask[idx.reshape(-1)] = False
    outside = buf[mask]
    bad = (outside != torch.tensor(SENT, dtype=buf.dtype, device=buf.device)).sum().item()
    assert bad == 0, f"{bad} elements written outside the [{rows} x {cols}] (ld {ld}) window"


@pytest.mark.parametrize("m,n,k", [(129, 72, 64), (300, 264, 200), (520, 392, 328), (1000, 1032, 136)])
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
def test_gemm_guard_bands(cuda, m, n, k, dt):
    from paper_2507_05753_b200 import _lib, tensor as T
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    a = torch.randn(m, k, device=cuda, generator=g).to(dt)
    b = torch.randn(n, k, device=cuda, generator=g).to(dt)
    bias = torch.randn(n, device=cuda, generator=g)
    ld = n + 24
    for od in ((torch.float32, torch.bfloat16) if dt == torch.bfloat16 else (torch.float32,)):
        buf, out = _guarded(m, n, ld, od)
        buf2, out2 = _guarded(m, n, n, torch.bfloat16)
        T.gemm_into(out, a, b, 0, 0, m, n, k, ldd=ld, epi=_lib.EPI_BIAS_COL | _lib.EPI_GELU_FWD, bias=bias, d2=out2)
        torch.cuda.synchronize()
        _check_guard(buf, m, n, ld)
        _check_guard(buf2, m, n, n)
        ref = a.double() @ b.double().t() + bias.double()
        assert torch.isfinite(out.float()).all()
        assert ((out.double() - ref).abs().max() / ref.abs().max()).item() < (2e-5 if dt == torch.float32 and od == torch.float32 else 1e-2)


def test_rowwise_guard_bands(cuda):
    """Layer-norm apply / backward, GELU, colsum, Adam write only their outputs."""
    from paper_2507_05753_b200 import kernels as K
    rows, cols = 1000, 264
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(rows, cols, device=cuda, generator=g)
    gam, bet = torch.randn(cols, device=cuda, generator=g), torch.randn(cols, device=cuda, generator=g)
    st = torch.zeros(rows, 2, device=cuda)
    K.ln_moments(x, st, rows, cols)
    buf, y = _guarded(rows, cols, cols, torch.bfloat16)
    mbuf, mr = _guarded(rows, 2, 2, torch.float32)
    K.ln_apply(x, st, gam, bet, y.view(-1), mr.view(-1), rows, cols, cols, 1e-5)
    torch.cuda.synchronize()
    _check_guard(buf, rows, cols, cols)
    _check_guard(mbuf, rows, 2, 2)
    bst = torch.zeros(rows, 2, device=cuda)
    gin = torch.randn(rows, cols, device=cuda, generator=g)
    K.ln_bwd_moments(x, gin, gam, mr.contiguous(), bst, rows, cols)
    obuf, o = _guarded(rows, cols, cols, torch.float32)
    K.ln_bwd_apply(x, gin, gam, mr.contiguous(), bst, None, o.view(-1), None, torch.zeros(cols, device=cuda),
                   torch.zeros(cols, device=cuda), rows, cols, cols)
    torch.cuda.synchronize()
    _check_guard(obuf, rows, cols, cols)
    cbuf, cs = _guarded(1, cols, cols, torch.float32)
    cs.zero_()
    K.colsum(x, cs.view(-1), rows, cols)
    torch.cuda.synchronize()
    _check_guard(cbuf, 1, cols, cols)
    # Adam over a ragged length inside sentinel-guarded state
    n = 100_003
    pb, p = _guarded(1, n, n, torch.float32)
    mb, m = _guarded(1, n, n, torch.float32)
    vb, v = _guarded(1, n, n, torch.float32)
    ob, op = _guarded(1, n, n, torch.bfloat16)
    p.copy_(torch.randn(1, n, device=cuda, generator=g))
    m.zero_()
    v.zero_()
    grad = torch.randn(n, device=cuda, generator=g)
    step = torch.ones(1, dtype=torch.int32, device=cuda)
    K.adam(p.view(-1), grad, m.view(-1), v.view(-1), op.view(-1), n, 1e-3, 0.9, 0.999, 1e-8, step)
    torch.cuda.synchronize()
    for b_ in (pb, mb, vb, ob):
        _check_guard(b_, 1, n, n)


def test_gemm_and_rowwise_deterministic(cuda):
    from paper_2507_05753_b200 import _lib, kernels as K, tensor as T
    g = torch.Generator(device="cuda").manual_seed(7)
    m, n, k = 2048, 1536, 4096
    a = torch.randn(m, k, device=cuda, generator=g).bfloat16()
    b = torch.randn(k, n, device=cuda, generator=g).bfloat16()
    bias = torch.randn(n, device=cuda, generator=g)
    resid = torch.randn(m, n, device=cuda, generator=g)
    outs = []
    for _ in range(5):
        d = torch.empty(m, n, device=cuda)
        d2 = torch.empty(m, n, device=cuda, dtype=torch.bfloat16)
        T.gemm_into(d, a, b, 0, 1, m, n, k, epi=_lib.EPI_BIAS_COL | _lib.EPI_RESID | _lib.EPI_COPY_D2, bias=bias,
                    resid=resid, d2=d2)
        outs.append((d, d2))
    torch.cuda.synchronize()
    for d, d2 in outs[1:]:
        assert torch.equal(d, outs[0][0]) and torch.equal(d2, outs[0][1])
    x = torch.randn(4096, 1024, device=cuda, generator=g)
    st = torch.zeros(4096, 2, device=cuda)
    K.ln_moments(x, st, 4096, 1024)
    gam, bet = torch.randn(1024, device=cuda, generator=g), torch.randn(1024, device=cuda, generator=g)
    ys = []
    for _ in range(3):
        y = torch.empty(4096, 1024, device=cuda, dtype=torch.bfloat16)
        K.ln_apply(x, st, gam, bet, y, None, 4096, 1024, 1024, 1e-5)
        ys.append(y)
    torch.cuda.synchronize()
    assert all(torch.equal(y, ys[0]) for y in ys[1:])


@pytest.mark.parametrize("nbytes,off8", [(65520, 0), (32760, 1), (8, 0), (4 << 20, 0)])
def test_push_copies_exactly(cuda, nbytes, off8):
    """jg_push (SM-driven copy to up to 4 destinations, the layer-norm moment gathers): exact
    copies, 16-byte or 8-byte aligned, nothing written outside the destinations."""
    from paper_2507_05753_b200 import kernels as K
    n = nbytes // 8
    src = torch.randn(n + 1, dtype=torch.float64, device=cuda)[off8:off8 + n]
    bufs, dsts = [], []
    for d in range(3):
        buf, view = _guarded(1, n + 1, n + 1, torch.float64)
        dst = view.reshape(-1)[off8:off8 + n]
        bufs.append((buf, dst))
        dsts.append(dst.data_ptr())
    K.push(src, dsts, nbytes)
    torch.cuda.synchronize()
    for buf, dst in bufs:
        assert torch.equal(dst, src)
        outside = torch.cat([buf[:4096 + off8], buf[4096 + off8 + n:]])
        assert bool((outside == SENT).all())
