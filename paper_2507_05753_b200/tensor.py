"""Dense numeric operators on B200 — the reference's L0 API (tensor.py) over sm_100a kernels.

Same names, argument meaning and error behaviour as reference `jigsaw/tensor.py`; tensors are
torch CUDA tensors (row-major, contiguous) instead of numpy arrays, and every operator runs
a kernel of libjigsaw_sm100.so:

    matmul(a, b, mode)             tensor.py:59-72   -> jg_gemm (tcgen05; bf16, or 3xTF32 for f32)
    gelu / gelu_backward           tensor.py:75-84   -> jg_gelu_fwd / jg_gelu_bwd
    layer_norm / _backward         tensor.py:87-123  -> jg_ln_moments + jg_ln_apply / jg_ln_bwd_*
    patchify / unpatchify          tensor.py:126-151 -> jg_patchify / jg_unpatchify
    dropout_mask                   tensor.py:154-160 (identity at rate 0, the model default)

dtypes: "f32" runs fp32-accurate arithmetic (tensor cores in 3xTF32 split form), "bf16" runs
bf16 operands with fp32 accumulation. The reference's f64 has no tensor-core form on B200
and is rejected with ShapeError (the oracle/ package keeps f64 for parity checking).
"""
from __future__ import annotations

import enum

import torch

from . import _lib
from .errors import ShapeError

DTYPES = {"f32": torch.float32, "bf16": torch.bfloat16}

# Optional per-launch GEMM timer (bench.py roofline leg): a list collecting
# (start_event, end_event, algorithmic_flops, algorithmic_bytes) for every jg_gemm launch while
# set; bytes = operands read once + output written once (+ read when accumulating).
GEMM_TIMER: list | None = None

# Persistent-grid SM limit for the GEMMs issued while it is set (0: all SMs) — the backward's
# GEMMs leave SMs free for the optimiser of the blocks already finished (engine.TrainStep).
GEMM_SM_CAP = 0

# Output tile width for the GEMMs issued while it is set (0: chosen per shape by jg_gemm;
# tools/tile_n_probe.py A/B-tests the choice).
GEMM_TILE_N = 0

# 3xTF32 K-chunking (fp32 mode). tcgen05's fp32 accumulation of each MMA step is not
# round-to-nearest: its error grows ~ K^1.5 (relative ~1.3e-8 * K measured on B200,
# tools/f32_diag.py: 2e-6 at K = 64, 2.2e-4 at K = 16380). fp32-mode GEMMs with K above
# TF32X3_KCHUNK therefore accumulate K-chunks into separate fp32 planes that jg_epilogue sums
# (round-to-nearest) before the real epilogue: ~7e-6 per GEMM at 512. bf16 mode is unaffected
# (its operand rounding, 2^-9, dominates).
import os as _os  # noqa: E402

TF32X3_KCHUNK = int(_os.environ.get("JG_TF32X3_KCHUNK", "512"))


class MatmulMode(str, enum.Enum):
    """The three layer multiplication layouts: X@W, X@W.T and X.T@W (tensor.py:27-33)."""

    NN = "NN"
    NT = "NT"
    TN = "TN"


def _check_device(*ts):
    for t in ts:
        if not isinstance(t, torch.Tensor):
            raise ShapeError(f"expected a torch tensor, got {type(t).__name__}")
        if not t.is_cuda:
            raise ShapeError("operands must be CUDA tensors (no CPU path exists)")
        if t.dtype not in (torch.float32, torch.bfloat16):
            raise ShapeError(f"unsupported dtype {t.dtype}: use float32 (3xTF32) or bfloat16")


def _check_operands(a: torch.Tensor, b: torch.Tensor, mode: MatmulMode) -> None:
    """Shape/dtype validation with the reference's messages (tensor.py:43-56)."""
    if a.dtype != b.dtype:
        raise ShapeError(f"matmul dtype mismatch: {a.dtype} vs {b.dtype}")
    if a.dim() < 2 or b.dim() < 2:
        raise ShapeError(f"matmul needs >=2-D operands, got {tuple(a.shape)} and {tuple(b.shape)}")
    mode = MatmulMode(mode)
    if mode is MatmulMode.NN:
        ok = a.shape[-1] == b.shape[-2]
    elif mode is MatmulMode.NT:
        ok = a.shape[-1] == b.shape[-1]
    else:
        ok = a.shape[-2] == b.shape[-2]
    if not ok:
        raise ShapeError(f"matmul {mode.value}: incompatible shapes {tuple(a.shape)} and {tuple(b.shape)}")


def _batch_view(t: torch.Tensor, lead: tuple[int, ...]):
    """Flatten leading dims to one batch axis; returns (3-D contiguous tensor, batch stride)."""
    mat = t.shape[-2:]
    if t.dim() == 2 or all(s == 1 for s in t.shape[:-2]):
        return t.reshape(1, *mat).contiguous(), 0
    t = t.expand(*lead, *mat).reshape(-1, *mat).contiguous()
    return t, mat[0] * mat[1]


def gemm_into(out: torch.Tensor, a: torch.Tensor, b: torch.Tensor, a_major: int, b_major: int,
              m: int, n: int, k: int, batch: int = 1, a_bs: int = 0, b_bs: int = 0, *,
              reduce_batch: bool = False, epi: int = 0, alpha: float = 1.0, d2: torch.Tensor | None = None,
              bias: torch.Tensor | None = None, bias_bs: int = 0, resid: torch.Tensor | None = None,
              r_bs: int = 0, pre: torch.Tensor | None = None, p_bs: int = 0, stats: torch.Tensor | None = None,
              stats_bs: int = 0, d_bs: int | None = None, d2_bs: int | None = None,
              lda: int | None = None, ldb: int | None = None, ldd: int | None = None,
              a_lo: torch.Tensor | None = None, b_lo: torch.Tensor | None = None, adam=None,
              d_planes=None, d_bcast=None, d2_bcast=None, rs: dict | None = None, lnb=None, plane_div: int = 0,
              planes_bs: int = 0) -> torch.Tensor:
    """Low-level fused GEMM: out[b] (op)= sum_k A[b](m,k) B[b](n,k) with epilogue `epi`.

    A/B majors follow include/jigsaw_sm100.h. fp32 operands run 3xTF32: the hi/lo split is
    made here unless the caller passes pre-split `a_lo`/`b_lo` (then `a`/`b` are the hi parts).
    """
    fp32 = a.dtype == torch.float32
    if a.dtype != b.dtype:
        raise ShapeError(f"matmul dtype mismatch: {a.dtype} vs {b.dtype}")
    if fp32 and (a_lo is None or b_lo is None):
        # 3xTF32 runs on K-major hi/lo operands: split (and transpose MN-major ones) here.
        a, a_lo, a_bs = split_operand(a, a_major, m, k, batch, a_bs, lda)
        b, b_lo, b_bs = split_operand(b, b_major, n, k, batch, b_bs, ldb)
        a_major = b_major = _lib.JG_KMAJOR
        lda = ldb = a.shape[-1]
    if (fp32 and TF32X3_KCHUNK > 0 and k > TF32X3_KCHUNK and adam is None and d_planes is None and rs is None
            and d_bcast is None and d2_bcast is None and a_major == _lib.JG_KMAJOR and b_major == _lib.JG_KMAJOR):
        return _gemm_tf32x3_chunked(out, a, a_lo, b, b_lo, m, n, k, batch, a_bs, b_bs, lda, ldb, reduce_batch,
                                    dict(epi=epi, alpha=alpha, d2=d2, bias=bias, bias_bs=bias_bs, resid=resid, r_bs=r_bs,
                                         pre=pre, p_bs=p_bs, stats=stats, stats_bs=stats_bs, d_bs=d_bs, d2_bs=d2_bs,
                                         ldd=ldd, lnb=lnb))
    d = _lib.GemmDesc()
    d.m, d.n, d.k, d.batch = m, n, k, batch
    d.math = _lib.JG_MATH_TF32X3 if fp32 else _lib.JG_MATH_BF16
    d.reduce_batch = int(reduce_batch)
    d.a, d.a_lo, d.a_bstride, d.a_major = a.data_ptr(), _lib.ptr(a_lo), a_bs, a_major
    d.b, d.b_lo, d.b_bstride, d.b_major = b.data_ptr(), _lib.ptr(b_lo), b_bs, b_major
    d.lda = lda if lda is not None else (k if a_major == _lib.JG_KMAJOR else m)
    d.ldb = ldb if ldb is not None else (k if b_major == _lib.JG_KMAJOR else n)
    d.epi, d.alpha = epi, alpha
    d.max_sms = GEMM_SM_CAP
    d.tile_n = GEMM_TILE_N
    d.d, d.ldd, d.d_type = _lib.ptr(out), ldd if ldd is not None else n, _lib.dtype_code(out) if out is not None else 0
    d.d_bstride = d_bs if d_bs is not None else (0 if reduce_batch else m * n)
    if d2 is not None:
        d.d2, d.ldd2, d.d2_type = d2.data_ptr(), n, _lib.dtype_code(d2)
        d.d2_bstride = d2_bs if d2_bs is not None else (0 if reduce_batch else m * n)
    if bias is not None:
        d.bias, d.bias_bstride = bias.data_ptr(), bias_bs
    if resid is not None:
        d.resid, d.ldr, d.r_bstride = resid.data_ptr(), n, r_bs if r_bs else m * n
    if pre is not None:
        d.pre, d.ldp, d.p_bstride, d.pre_type = pre.data_ptr(), n, p_bs if p_bs else m * n, _lib.dtype_code(pre)
    if stats is not None:
        d.stats, d.stats_bstride = stats.data_ptr(), stats_bs if stats_bs else 2 * m
    if lnb is not None:
        # JG_EPI_LNB: (x [batch][m][ldx] fp32, gamma [n], mean/rstd [batch][m][2]); x batch stride m*ldx
        lx, lg, lmr = lnb[:3]
        ldx = lnb[3] if len(lnb) > 3 else n
        d.lnb_x, d.lnb_ldx, d.lnb_x_bstride = lx.data_ptr(), ldx, m * ldx
        d.lnb_gamma, d.lnb_mr = lg.data_ptr(), lmr.data_ptr()
    if d_planes is not None:
        for i, addr in enumerate(d_planes):
            d.d_planes[i] = addr
        d.plane_div, d.d_planes_bstride = plane_div, planes_bs  # (batch b -> plane b / plane_div, sample b % plane_div)
    if rs is not None:
        # fused reduce-scatter (jg_gemm_desc rs_*): flags / peer flag arrays / partial-plane source
        d.rs_flags = rs.get("flags")
        for i, addr in enumerate(rs["flag_peers"]):
            d.rs_flag_peers[i] = addr
        d.rs_src, d.rs_src_stride = rs.get("src"), rs.get("src_stride", 0)
        d.rs_part_type, d.rs_nsrc, d.rs_src_idx = rs["part_type"], rs["nsrc"], rs["src_idx"]
        d.rs_own, d.rs_need, d.rs_flag_cap = rs.get("own", -1), rs["need"], rs["flag_cap"]
    for fld, addrs in (("d_bcast", d_bcast), ("d2_bcast", d2_bcast)):
        bc = _lib.make_bcast(addrs)
        if bc is not None:
            setattr(d, fld, bc)
    if adam is not None:
        # adam = (m_view, v_view, bf16_copy_view | None, step_counter, lr, beta1, beta2, eps); out = master
        am, av, apb, astep, lr, b1, b2, eps = adam
        d.adam_m, d.adam_v, d.adam_pbf16, d.adam_step = am.data_ptr(), av.data_ptr(), _lib.ptr(apb), astep.data_ptr()
        d.adam_lr, d.adam_beta1, d.adam_beta2, d.adam_eps = lr, b1, b2, eps
    if GEMM_TIMER is not None:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _lib.gemm_raw(d)
        e.record()
        ae, oe = a.element_size(), (out.element_size() if out is not None else 2)
        outs = 1 if reduce_batch else batch
        nbytes = (m * k + n * k) * ae * batch + m * n * oe * outs * (2 if epi & _lib.EPI_ACCUM else 1)
        GEMM_TIMER.append((s, e, 2 * m * n * k * batch, nbytes))
    else:
        _lib.gemm_raw(d)
    return out


def _at(t: torch.Tensor | None, off: int):
    """Flat view of `t` starting `off` elements in (a batch item of a strided operand)."""
    return None if t is None else t.reshape(-1)[off:]


def _gemm_tf32x3_chunked(out, a, a_lo, b, b_lo, m, n, k, batch, a_bs, b_bs, lda, ldb, reduce_batch, ep):
    """fp32-mode GEMM with K accumulated in TF32X3_KCHUNK-long chunks: one batched jg_gemm per
    output item writes the chunk products as fp32 planes, jg_epilogue sums the planes in order
    and applies the epilogue (bias / residual / GELU / moments / accumulate); the layer-norm
    backward moments (JG_EPI_LNB) follow from jg_ln_bwd_moments on the finished output."""
    kc = TF32X3_KCHUNK
    S, tail = k // kc, k % kc
    per = S + (1 if tail else 0)
    epi = ep["epi"]
    lnb = ep["lnb"]
    ldd = ep["ldd"] if ep["ldd"] is not None else n
    d_bs = ep["d_bs"] if ep["d_bs"] is not None else (0 if reduce_batch else m * n)
    d2_bs = ep["d2_bs"] if ep["d2_bs"] is not None else (0 if reduce_batch else m * n)
    r_bs = ep["r_bs"] if ep["r_bs"] else m * n
    p_bs = ep["p_bs"] if ep["p_bs"] else m * n
    st_bs = ep["stats_bs"] if ep["stats_bs"] else 2 * m
    outs = [None] if reduce_batch else list(range(batch))
    for o in outs:
        items = list(range(batch)) if reduce_batch else [o]
        planes = torch.empty((len(items) * per, m, n), dtype=torch.float32, device=a.device)
        for j, bi in enumerate(items):
            pl = planes[j * per:]
            gemm_into(pl, _at(a, bi * a_bs), _at(b, bi * b_bs), _lib.JG_KMAJOR, _lib.JG_KMAJOR, m, n, kc, S, kc, kc,
                      a_lo=_at(a_lo, bi * a_bs), b_lo=_at(b_lo, bi * b_bs), lda=lda, ldb=ldb, d_bs=m * n)
            if tail:
                off = S * kc
                gemm_into(pl[S], _at(a, bi * a_bs + off), _at(b, bi * b_bs + off), _lib.JG_KMAJOR, _lib.JG_KMAJOR,
                          m, n, tail, a_lo=_at(a_lo, bi * a_bs + off), b_lo=_at(b_lo, bi * b_bs + off), lda=lda, ldb=ldb)
        ob = 0 if o is None else o
        from . import kernels as K
        K.epilogue(planes, m, n, nplanes=planes.shape[0], acc_bs=m * n, epi=epi & ~_lib.EPI_LNB, alpha=ep["alpha"],
                   d=_at(out, ob * d_bs), ldd=ldd, d2=_at(ep["d2"], ob * d2_bs), ldd2=n,
                   bias=_at(ep["bias"], ob * ep["bias_bs"]), resid=_at(ep["resid"], ob * r_bs),
                   pre=_at(ep["pre"], ob * p_bs), stats=_at(ep["stats"], ob * st_bs))
        if epi & _lib.EPI_LNB:
            lx, lg, lmr = lnb[:3]
            ldx = lnb[3] if len(lnb) > 3 else n
            if ldx != n or ldd != n:
                raise ShapeError("chunked 3xTF32 GEMM: JG_EPI_LNB needs contiguous rows")
            K.ln_bwd_moments(_at(lx, ob * m * ldx), _at(out, ob * d_bs), lg, _at(lmr, ob * st_bs),
                             _at(ep["stats"], ob * st_bs), m, n)
    return out


def split_tf32(x: torch.Tensor):
    """(hi, lo) with hi = x truncated to tf32 and lo = x - hi (exact in fp32)."""
    x = x.contiguous()
    hi = torch.empty_like(x)
    lo = torch.empty_like(x)
    _lib.call("jg_split_tf32", x.data_ptr(), hi.data_ptr(), lo.data_ptr(), x.numel())
    return hi, lo


def split_operand(x: torch.Tensor, major: int, rows: int, k: int, batch: int, bs: int, ld: int | None):
    """K-major 3xTF32 (hi, lo, batch stride) of a GEMM operand with `rows` (M or N) x `k` per batch."""
    nb = batch if bs else 1
    ldk = (k + 3) // 4 * 4
    hi = torch.empty((nb, rows, ldk), dtype=torch.float32, device=x.device)
    lo = torch.empty_like(hi)
    if major == _lib.JG_KMAJOR:
        _lib.call("jg_split_tf32_2d", x.data_ptr(), rows, k, ld if ld is not None else k, nb, bs, 0,
                  hi.data_ptr(), lo.data_ptr(), ldk)
    else:
        _lib.call("jg_split_tf32_2d", x.data_ptr(), k, rows, ld if ld is not None else rows, nb, bs, 1,
                  hi.data_ptr(), lo.data_ptr(), ldk)
    return hi, lo, (rows * ldk if bs else 0)


def matmul(a: torch.Tensor, b: torch.Tensor, mode: MatmulMode = MatmulMode.NN) -> torch.Tensor:
    """Multiply under the given mode; leading batch dimensions broadcast (tensor.py:59-72).

    NN: a[..., m, k] @ b[..., k, n] -> [..., m, n]
    NT: a[..., m, k] @ b[..., n, k].T -> [..., m, n]
    TN: a[..., m, k].T @ b[..., m, n] -> [..., k, n]
    """
    _check_device(a, b)
    _check_operands(a, b, mode)
    mode = MatmulMode(mode)
    lead = torch.broadcast_shapes(a.shape[:-2], b.shape[:-2])
    a3, a_bs = _batch_view(a, lead)
    b3, b_bs = _batch_view(b, lead)
    batch = 1
    for s in lead:
        batch *= s
    if mode is MatmulMode.NN:
        m, k, n = a.shape[-2], a.shape[-1], b.shape[-1]
        am, bm = _lib.JG_KMAJOR, _lib.JG_MNMAJOR
    elif mode is MatmulMode.NT:
        m, k, n = a.shape[-2], a.shape[-1], b.shape[-2]
        am, bm = _lib.JG_KMAJOR, _lib.JG_KMAJOR
    else:
        m, k, n = a.shape[-1], a.shape[-2], b.shape[-1]
        am, bm = _lib.JG_MNMAJOR, _lib.JG_MNMAJOR
    out = torch.empty((*lead, m, n), dtype=a.dtype, device=a.device)
    if out.numel() == 0:
        return out
    if k == 0:
        return out.zero_()
    if a.dtype == torch.bfloat16 and (a3.shape[-1] % 8 or b3.shape[-1] % 8 or n % 8):
        # TMA needs 16-byte row strides: zero-pad the contiguous axes (the product is unchanged)
        a3 = _pad_last(a3, 8)
        b3 = _pad_last(b3, 8)
        np_ = (n + 7) // 8 * 8
        tmp = torch.empty((batch, m, np_), dtype=a.dtype, device=a.device)
        gemm_into(tmp, a3, b3, am, bm, m, n, k, batch, a3[0].numel() if a_bs else 0,
                  b3[0].numel() if b_bs else 0, lda=a3.shape[-1], ldb=b3.shape[-1], ldd=np_, d_bs=m * np_)
        out.copy_(tmp[..., :n].reshape(out.shape))
        return out
    if a.dtype == torch.float32 and n % 4:
        # operands are re-laid out by the 3xTF32 split; only D needs a padded row stride
        np_ = (n + 3) // 4 * 4
        tmp = torch.empty((batch, m, np_), dtype=a.dtype, device=a.device)
        gemm_into(tmp, a3, b3, am, bm, m, n, k, batch, a_bs, b_bs, ldd=np_, d_bs=m * np_)
        out.copy_(tmp[..., :n].reshape(out.shape))
        return out
    gemm_into(out, a3, b3, am, bm, m, n, k, batch, a_bs, b_bs)
    return out


def _pad_last(t: torch.Tensor, mult: int) -> torch.Tensor:
    pad = (-t.shape[-1]) % mult
    return torch.nn.functional.pad(t, (0, pad)).contiguous() if pad else t


def _ew_dtype(t: torch.Tensor) -> int:
    return _lib.dtype_code(t)


def gelu(x: torch.Tensor) -> torch.Tensor:
    """Exact-erf GELU: x * Phi(x) (tensor.py:75-77)."""
    _check_device(x)
    x = x.contiguous()
    y = torch.empty_like(x)
    _lib.call("jg_gelu_fwd", x.data_ptr(), y.data_ptr(), _ew_dtype(x), x.numel())
    return y


def gelu_backward(x: torch.Tensor, upstream: torch.Tensor) -> torch.Tensor:
    """upstream * dGELU/dx with dGELU/dx = Phi(x) + x * phi(x) (tensor.py:80-84)."""
    _check_device(x, upstream)
    if x.shape != upstream.shape or x.dtype != upstream.dtype:
        raise ShapeError(f"gelu_backward shapes {tuple(x.shape)} / {tuple(upstream.shape)} differ")
    x, upstream = x.contiguous(), upstream.contiguous()
    dx = torch.empty_like(x)
    _lib.call("jg_gelu_bwd", x.data_ptr(), upstream.data_ptr(), dx.data_ptr(), _ew_dtype(x), x.numel())
    return dx


def _rows(x: torch.Tensor) -> int:
    r = 1
    for s in x.shape[:-1]:
        r *= s
    return r


def ln_stats(x: torch.Tensor) -> torch.Tensor:
    """Row moments [rows, 2] = (sum x, sum x^2) of the last axis (fp32)."""
    rows, c = _rows(x), x.shape[-1]
    stats = torch.zeros((rows, 2), dtype=torch.float32, device=x.device)
    _lib.call("jg_ln_moments", x.data_ptr(), stats.data_ptr(), rows, c, c)
    return stats


def layer_norm(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, eps: float = 1e-5) -> torch.Tensor:
    """Normalize the last axis to zero mean / unit variance, then affine (tensor.py:97-106)."""
    if eps <= 0:
        raise ValueError(f"layer_norm eps must be > 0, got {eps}")
    _check_device(x, gamma, beta)
    if gamma.shape != (x.shape[-1],) or beta.shape != (x.shape[-1],):
        raise ShapeError(
            f"layer_norm affine shapes {tuple(gamma.shape)}/{tuple(beta.shape)} do not match last axis of {tuple(x.shape)}")
    if x.dtype != torch.float32:
        raise ShapeError("layer_norm input must be float32 (the residual stream is kept in fp32)")
    x = x.contiguous()
    rows, c = _rows(x), x.shape[-1]
    stats = ln_stats(x)
    y = torch.empty_like(x)
    _lib.call("jg_ln_apply", x.data_ptr(), stats.data_ptr(), gamma.contiguous().data_ptr(),
              beta.contiguous().data_ptr(), y.data_ptr(), _lib.JG_F32, None, rows, c, c, float(eps), None)
    return y


def layer_norm_backward(x: torch.Tensor, gamma: torch.Tensor, eps: float, upstream: torch.Tensor):
    """Gradients of layer_norm w.r.t. (x, gamma, beta) (tensor.py:109-123)."""
    if eps <= 0:
        raise ValueError(f"layer_norm eps must be > 0, got {eps}")
    _check_device(x, gamma, upstream)
    x, upstream, gamma = x.contiguous(), upstream.contiguous(), gamma.contiguous()
    rows, c = _rows(x), x.shape[-1]
    stats = ln_stats(x)
    mr = torch.empty((rows, 2), dtype=torch.float32, device=x.device)
    scratch = torch.empty_like(x)
    zeros = torch.zeros_like(gamma)
    _lib.call("jg_ln_apply", x.data_ptr(), stats.data_ptr(), gamma.data_ptr(), zeros.data_ptr(),
              scratch.data_ptr(), _lib.JG_F32, mr.data_ptr(), rows, c, c, float(eps), None)
    bstats = torch.zeros((rows, 2), dtype=torch.float32, device=x.device)
    _lib.call("jg_ln_bwd_moments", x.data_ptr(), upstream.data_ptr(), gamma.data_ptr(), mr.data_ptr(),
              bstats.data_ptr(), rows, c)
    dx = torch.empty_like(x)
    dgamma = torch.zeros_like(gamma)
    dbeta = torch.zeros_like(gamma)
    _lib.call("jg_ln_bwd_apply", x.data_ptr(), upstream.data_ptr(), gamma.data_ptr(), mr.data_ptr(),
              bstats.data_ptr(), None, dx.data_ptr(), None, dgamma.data_ptr(), dbeta.data_ptr(), None, 0, None,
              rows, c, c, None)
    return dx, dgamma, dbeta


def patchify(x: torch.Tensor, p_lat: int, p_lon: int) -> torch.Tensor:
    """[B, lat, lon, C] -> [B, tokens, C*p_lat*p_lon], channel-major features (tensor.py:126-139)."""
    _check_device(x)
    b, lat, lon, c = x.shape
    if lat % p_lat or lon % p_lon:
        raise ShapeError(f"grid {lat}x{lon} not divisible by patch {p_lat}x{p_lon}")
    if x.dtype != torch.float32:
        raise ShapeError("patchify input must be float32")
    out = torch.empty((b, (lat // p_lat) * (lon // p_lon), c * p_lat * p_lon), dtype=x.dtype, device=x.device)
    _lib.call("jg_patchify", x.contiguous().data_ptr(), out.data_ptr(), _lib.JG_F32, b, lat, lon, c, p_lat, p_lon)
    return out


def unpatchify(tokens: torch.Tensor, lat: int, lon: int, p_lat: int, p_lon: int) -> torch.Tensor:
    """Exact inverse of patchify (tensor.py:142-151)."""
    _check_device(tokens)
    b, n_tok, feat = tokens.shape
    gl, gw = lat // p_lat, lon // p_lon
    if n_tok != gl * gw or feat % (p_lat * p_lon) or lat % p_lat or lon % p_lon:
        raise ShapeError(f"token tensor {tuple(tokens.shape)} does not fit grid {lat}x{lon}")
    c = feat // (p_lat * p_lon)
    out = torch.empty((b, lat, lon, c), dtype=tokens.dtype, device=tokens.device)
    _lib.call("jg_unpatchify", tokens.contiguous().data_ptr(), out.data_ptr(), b, lat, lon, c, p_lat, p_lon)
    return out


def dropout_mask(shape, rate: float, generator: torch.Generator | None = None, device="cuda"):
    """Inverted-dropout mask (None when the layer is a no-op), tensor.py:154-160.

    The WeatherMixer default rate is 0 (model.py:50), for which this is the identity; masks
    are per-rank RNG in the reference too (model.py:313), so they are never parity-checked.
    """
    if not 0.0 <= rate < 1.0:
        raise ValueError(f"dropout rate must be in [0, 1), got {rate}")
    if rate == 0.0:
        return None
    return (torch.rand(shape, generator=generator, device=device) >= rate).float() / (1.0 - rate)
