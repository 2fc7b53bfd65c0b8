"""Tensor-level wrappers of every libjigsaw_sm100.so entry point used by the model.

The model / Jigsaw orchestration code calls only these functions (never ctypes directly), so
the whole host-side schedule — layouts, collectives, buffer plumbing — is one layer above the
C ABI. Each wrapper passes raw device pointers and the current stream (see _lib.py).
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from . import tensor as T
from ._lib import ptr


def gemm(out, a, b, am, bm, m, n, k, *batch_args, **kw):
    """jg_gemm (see tensor.gemm_into for the argument meaning)."""
    return T.gemm_into(out, a, b, am, bm, m, n, k, *batch_args, **kw)


def _bref(addrs):
    b = _lib.make_bcast(addrs)
    return None if b is None else ctypes.byref(b)


def epilogue(acc, m, n, *, batch=1, acc_ld=None, acc_bs=0, nplanes=1, epi=0, alpha=1.0, d=None, ldd=None, d_bs=0,
             d2=None, ldd2=None, d2_bs=0, bias=None, bias_bs=0, resid=None, ldr=None, r_bs=0, pre=None, ldp=None,
             p_bs=0, stats=None, stats_bs=0, d_bcast=None, d2_bcast=None):
    """jg_epilogue: the GEMM epilogue applied to an accumulator `acc` [batch][m][acc_ld], or to the
    sum of `nplanes` partial planes of `acc` (plane stride acc_bs)."""
    g = _lib.GemmDesc()
    g.m, g.n, g.batch, g.epi, g.alpha = m, n, batch, epi, alpha
    g.d, g.ldd, g.d_bstride = ptr(d), ldd if ldd is not None else n, d_bs
    g.d_type = _lib.dtype_code(d) if d is not None else 0
    if d2 is not None:
        g.d2, g.ldd2, g.d2_bstride, g.d2_type = d2.data_ptr(), ldd2 if ldd2 is not None else n, d2_bs, _lib.dtype_code(d2)
    if bias is not None:
        g.bias, g.bias_bstride = bias.data_ptr(), bias_bs
    if resid is not None:
        g.resid, g.ldr, g.r_bstride = resid.data_ptr(), ldr if ldr is not None else n, r_bs
    if pre is not None:
        g.pre, g.ldp, g.p_bstride, g.pre_type = pre.data_ptr(), ldp if ldp is not None else n, p_bs, _lib.dtype_code(pre)
    if stats is not None:
        g.stats, g.stats_bstride = stats.data_ptr(), stats_bs
    for fld, addrs in (("d_bcast", d_bcast), ("d2_bcast", d2_bcast)):
        bc = _lib.make_bcast(addrs)
        if bc is not None:
            setattr(g, fld, bc)
    _lib.call("jg_epilogue", ctypes.byref(g), acc.data_ptr(), _lib.dtype_code(acc), acc_ld if acc_ld is not None else n,
              acc_bs, nplanes)


def sum_planes(y, x, n, nplanes, plane_stride, accumulate=False):
    """y[:n] (+)= sum_p x[p * plane_stride + i] (x fp32 or bf16, y fp32)."""
    _lib.call("jg_sum_planes", y.data_ptr(), x.data_ptr(), _lib.dtype_code(x), n, nplanes, plane_stride,
              int(accumulate))


def copy_async(dst_ptr: int, src: torch.Tensor, nbytes: int | None = None):
    """Copy-engine copy of `src` to a raw device address (e.g. a peer's symmetric buffer)."""
    _lib.call("jg_copy_async", dst_ptr, src.data_ptr(), nbytes if nbytes is not None else src.numel() * src.element_size())


_TORCH_ZERO = __import__("os").environ.get("JIGSAW_TORCH_ZERO") == "1"  # A/B only


def zero(t: torch.Tensor):
    """Zero a contiguous tensor (jg_memset; accumulators at the start of a step)."""
    assert t.is_contiguous()
    if _TORCH_ZERO:
        t.zero_()
        return
    _lib.call("jg_memset", t.data_ptr(), t.numel() * t.element_size())


def push(src: torch.Tensor, addrs, nbytes: int | None = None):
    """SM-driven copy of `src` to up to 4 raw device addresses (own / NVLink peer memory)."""
    _lib.call("jg_push", src.data_ptr(), nbytes if nbytes is not None else src.numel() * src.element_size(),
              _bref(addrs))


def axpy(y, x, alpha=1.0):
    _lib.call("jg_axpy", y.data_ptr(), x.data_ptr(), float(alpha), x.numel())


def cast_bf16(x, y):
    _lib.call("jg_cast_bf16", x.data_ptr(), y.data_ptr(), x.numel())


def patchify(x, tok, batch, lat, lon, chans, pl, pw):
    _lib.call("jg_patchify", x.data_ptr(), tok.data_ptr(), _lib.dtype_code(tok), batch, lat, lon, chans, pl, pw)


def gelu_fwd(x, y):
    """y = x * Phi(x), exact erf (reference tensor.py:75-77)."""
    _lib.call("jg_gelu_fwd", x.data_ptr(), y.data_ptr(), _lib.dtype_code(x), x.numel())


def gelu_bwd(x, g, dx):
    """dx = g * (Phi(x) + x phi(x)) (reference tensor.py:80-84)."""
    _lib.call("jg_gelu_bwd", x.data_ptr(), g.data_ptr(), dx.data_ptr(), _lib.dtype_code(x), x.numel())


def ln_moments(x, stats, rows, cols):
    _lib.call("jg_ln_moments", x.data_ptr(), stats.data_ptr(), rows, cols, cols)


def ln_apply(x, stats, gamma, beta, y, mean_rstd, rows, cols, c_total, eps, bcast=None):
    _lib.call("jg_ln_apply", x.data_ptr(), stats.data_ptr(), gamma.data_ptr(), beta.data_ptr(), y.data_ptr(),
              _lib.dtype_code(y), ptr(mean_rstd), rows, cols, c_total, float(eps), _bref(bcast))


def ln_bwd_moments(x, g, gamma, mean_rstd, bstats, rows, cols):
    _lib.call("jg_ln_bwd_moments", x.data_ptr(), g.data_ptr(), gamma.data_ptr(), mean_rstd.data_ptr(),
              bstats.data_ptr(), rows, cols)


def ln_bwd_apply(x, g, gamma, mean_rstd, bstats, resid, out, out_op, dgamma, dbeta, rows, cols, c_total,
                 bcast=None, rowsum=None, rowsum_period=0, colsum=None):
    """rowsum[r % rowsum_period] += sum_c out, colsum[c] += sum_r out, in the same pass (bias grads)."""
    _lib.call("jg_ln_bwd_apply", x.data_ptr(), g.data_ptr(), gamma.data_ptr(), mean_rstd.data_ptr(),
              bstats.data_ptr(), ptr(resid), out.data_ptr(), None if out_op is None or out_op is out else out_op.data_ptr(),
              ptr(dgamma), ptr(dbeta), ptr(rowsum), int(rowsum_period), ptr(colsum), rows, cols, c_total, _bref(bcast))


def colsum(x, out, rows, cols, ld=None):
    _lib.call("jg_colsum", x.data_ptr(), _lib.dtype_code(x), out.data_ptr(), rows, cols, ld if ld is not None else cols)


def rowsum(x, out, rows, cols, ld=None):
    _lib.call("jg_rowsum", x.data_ptr(), _lib.dtype_code(x), out.data_ptr(), rows, cols, ld if ld is not None else cols)


def blend_loss(dec, xin, target, blend_w, lat_w, var_w, g_ext, out, loss, g_blend, g_dec, batch, lat, lon, chans,
               pl, pw, inv_count, loss_scale, bcast=None):
    f32 = g_dec if g_dec is not None and g_dec.dtype == torch.float32 else None
    b16 = g_dec if g_dec is not None and g_dec.dtype == torch.bfloat16 else None
    _lib.call("jg_blend_loss", dec.data_ptr(), xin.data_ptr(), ptr(target), blend_w.data_ptr(), lat_w.data_ptr(),
              var_w.data_ptr(), ptr(g_ext), ptr(out), ptr(loss), ptr(g_blend), ptr(f32), ptr(b16),
              batch, lat, lon, chans, pl, pw, float(inv_count), float(loss_scale), _bref(bcast))


def adam(p, g, m, v, p_op, n, lr, beta1, beta2, eps, step, grad_scale=None, lr_dev=None, push=None, sms=None):
    """jg_adam; lr_dev (device float, e.g. one entry of the schedule's output) overrides lr.
    push: [(start, len, [addr, ...])] — ranges whose bf16 copy is also stored at peer addresses
    (jg_adam_push: the Jigsaw weight-panel gather done by the optimiser). sms: pinned to that
    many SMs (jg_adam_sms), beside a GEMM limited to the others."""
    if sms:
        assert not push, "jg_adam_sms has no panel push"
        _lib.call("jg_adam_sms", p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), ptr(p_op), n, float(lr),
                  float(beta1), float(beta2), float(eps), step.data_ptr(), ptr(grad_scale), ptr(lr_dev), int(sms))
        return
    if push:
        t = _lib.make_push_table(push)
        _lib.call("jg_adam_push", p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), ptr(p_op), n, float(lr),
                  float(beta1), float(beta2), float(eps), step.data_ptr(), ptr(grad_scale), ptr(lr_dev),
                  ctypes.byref(t))
        return
    _lib.call("jg_adam", p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), ptr(p_op), n, float(lr),
              float(beta1), float(beta2), float(eps), step.data_ptr(), ptr(grad_scale), ptr(lr_dev))


def sqnorm(x, out, weight=1.0, n=None):
    """out[0] += weight * sum(x[:n]^2) (fp32)."""
    _lib.call("jg_sqnorm", x.data_ptr(), x.numel() if n is None else n, float(weight), out.data_ptr())


def opt_schedule(step, scheds, sqsum, clip_norm, lr_out, grad_scale):
    """jg_opt_schedule: per-class lr of this step (device) and the global-norm clip factor."""
    arr = (_lib.LrSchedule * max(1, len(scheds)))()
    for i, s in enumerate(scheds):
        arr[i] = _lib.LrSchedule(*s)
    _lib.call("jg_opt_schedule", step.data_ptr(), arr, len(scheds), ptr(sqsum), float(clip_norm or 0.0),
              ptr(lr_out), ptr(grad_scale))


def step_increment(counter):
    _lib.call("jg_step_increment", counter.data_ptr())
