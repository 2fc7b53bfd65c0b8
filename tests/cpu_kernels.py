"""TEST DOUBLE (tests only): torch-CPU implementations of paper_2507_05753_b200.kernels.

Lets the gloo multi-process tests run the real host-side Jigsaw schedule (layouts,
collectives, buffer plumbing in model.py / jigsaw_grid.py) on CPU, with the kernel layer
swapped for exact float64 arithmetic that follows the C ABI's documented semantics
(include/jigsaw_sm100.h). Never used by the package; install() monkeypatches it in a test.
"""
from __future__ import annotations

import math

import torch

EPI_ACCUM, EPI_BIAS_COL, EPI_BIAS_ROW, EPI_RESID = 1, 2, 4, 8
EPI_GELU_FWD, EPI_GELU_BWD, EPI_COPY_D2, EPI_STATS = 16, 32, 64, 128
EPI_ADAM = 256
EPI_LNB = 512
KM = 0


def _view(t, size, stride, extra=0):
    return torch.as_strided(t, size, stride, t.storage_offset() + extra)


# ---- emulated peer memory (tests/shm_transport.py): raw "device addresses" handed out by the
# transport are synthetic; they resolve to shared-file arenas mapped in every rank's process.
_PEERS: list = []


def register_peer(base: int, buf: torch.Tensor) -> None:
    _PEERS.append((base, buf.numel(), buf))


def _at(addr: int, dtype, size, stride):
    es = torch.empty((), dtype=dtype).element_size()
    span = 1 + sum((a - 1) * b for a, b in zip(size, stride))
    for base, n, buf in _PEERS:
        if base <= addr < base + n:
            off = addr - base
            assert off % es == 0 and off + span * es <= n, (addr, base, n, span)
            return torch.as_strided(buf[off:off + span * es].view(dtype), size, stride)
    raise AssertionError(f"address {addr:#x} is not in any emulated peer arena")


def _bcast_copy(src, addrs):
    """Store the just-written output `src` (a strided view) at every peer address too."""
    for a in addrs or []:
        _at(a, src.dtype, tuple(src.shape), tuple(src.stride())).copy_(src)


def copy_async(dst_ptr, src, nbytes=None):
    nbytes = src.numel() * src.element_size() if nbytes is None else nbytes
    if not any(base <= dst_ptr < base + n for base, n, _ in _PEERS):  # a local (host) buffer
        import ctypes
        ctypes.memmove(dst_ptr, src.contiguous().data_ptr(), nbytes)
        return
    _at(dst_ptr, torch.uint8, (nbytes,), (1,)).copy_(src.contiguous().view(-1).view(torch.uint8)[:nbytes])


def _gelu(x):
    return x * 0.5 * (1.0 + torch.erf(x / math.sqrt(2.0)))


def _gelu_grad(x):
    return 0.5 * (1.0 + torch.erf(x / math.sqrt(2.0))) + x * torch.exp(-0.5 * x * x) / math.sqrt(2 * math.pi)


def _apply_epilogue(v, ob, m, n, epi, alpha, d, ldd, d_bs, d2, ldd2, d2_bs, bias, bias_bs, resid, ldr, r_bs,
                    pre, ldp, p_bs, stats, stats_bs, lnb=None):
    v = v * alpha
    if epi & EPI_BIAS_COL:
        v = v + _view(bias, (n,), (1,), ob * bias_bs).double()[None, :]
    if epi & EPI_BIAS_ROW:
        v = v + _view(bias, (m,), (1,), ob * bias_bs).double()[:, None]
    if epi & EPI_RESID:
        v = v + _view(resid, (m, n), (ldr, 1), ob * r_bs).double()
    if epi & EPI_GELU_BWD:
        v = v * _gelu_grad(_view(pre, (m, n), (ldp, 1), ob * p_bs).double())
    if d is not None:
        dv = _view(d, (m, n), (ldd, 1), ob * d_bs)
        if epi & EPI_ACCUM:
            v = v + dv.double()
        dv.copy_(v.to(d.dtype))
    if epi & (EPI_GELU_FWD | EPI_COPY_D2):
        _view(d2, (m, n), (ldd2, 1), ob * d2_bs).copy_((_gelu(v) if epi & EPI_GELU_FWD else v).to(d2.dtype))
    if epi & EPI_STATS:
        sv = _view(stats, (m, 2), (2, 1), ob * stats_bs)
        sv[:, 0] += v.sum(1).to(sv.dtype)
        sv[:, 1] += (v * v).sum(1).to(sv.dtype)
    if epi & EPI_LNB:  # layer-norm backward row moments of the result (jg_gemm JG_EPI_LNB)
        lx, lg, lmr = lnb[:3]
        ldx = lnb[3] if len(lnb) > 3 else n
        x = _view(lx, (m, n), (ldx, 1), ob * m * ldx).double()
        mr = _view(lmr, (m, 2), (2, 1), ob * stats_bs).double()
        h = v * lg.double()[None, :n]
        sv = _view(stats, (m, 2), (2, 1), ob * stats_bs)
        sv[:, 0] += h.sum(1).to(sv.dtype)
        sv[:, 1] += (h * (x - mr[:, :1]) * mr[:, 1:]).sum(1).to(sv.dtype)


def gemm(out, a, b, am, bm, m, n, k, batch=1, a_bs=0, b_bs=0, *, reduce_batch=False, epi=0, alpha=1.0, d2=None,
         bias=None, bias_bs=0, resid=None, r_bs=0, pre=None, p_bs=0, stats=None, stats_bs=0, d_bs=None,
         d2_bs=None, lda=None, ldb=None, ldd=None, a_lo=None, b_lo=None, adam=None, d_planes=None, d_bcast=None,
         d2_bcast=None, rs=None, lnb=None, plane_div=0, planes_bs=0):
    lda = lda if lda is not None else (k if am == KM else m)
    ldb = ldb if ldb is not None else (k if bm == KM else n)
    ldd = ldd if ldd is not None else n
    d_bs = d_bs if d_bs is not None else (0 if reduce_batch else m * n)
    d2_bs = d2_bs if d2_bs is not None else (0 if reduce_batch else m * n)
    r_bs = r_bs if r_bs else m * n
    p_bs = p_bs if p_bs else m * n
    stats_bs = stats_bs if stats_bs else 2 * m
    acc = []
    for bi in range(batch):
        try:
            A = _view(a, (m, k), (lda, 1) if am == KM else (1, lda), bi * a_bs).double()
        except RuntimeError as e:
            raise RuntimeError(f"A view: shape {tuple(a.shape)} stride {a.stride()} off {a.storage_offset()} "
                               f"m={m} n={n} k={k} batch={batch} a_bs={a_bs} lda={lda} am={am}: {e}") from None
        B = _view(b, (n, k), (ldb, 1) if bm == KM else (1, ldb), bi * b_bs).double()
        acc.append(A @ B.T)
    if reduce_batch:
        acc = [sum(acc)]
    if epi & EPI_ADAM:
        am_, av_, apb, astep, lr, b1, b2, eps = adam
        t = int(astep.item())
        for ob, v in enumerate(acc):
            w = _view(out, (m, n), (ldd, 1), ob * d_bs)
            mm = _view(am_, (m, n), (ldd, 1), ob * d_bs)
            vv = _view(av_, (m, n), (ldd, 1), ob * d_bs)
            gg = (v * alpha).float()
            mm.mul_(b1).add_((1 - b1) * gg)
            vv.mul_(b2).add_((1 - b2) * gg * gg)
            w.sub_(lr * (mm / (1 - b1 ** t)) / (torch.sqrt(vv / (1 - b2 ** t)) + eps))
            if apb is not None:
                _view(apb, (m, n), (ldd, 1), ob * d_bs).copy_(w.to(apb.dtype))
        return out
    if rs is not None:
        return _gemm_rs(acc, out, m, n, ldd, d_planes, rs, epi, alpha, d2, bias, resid, pre, stats, d_bcast, d2_bcast)
    if d_planes:  # fused reduce-scatter: batch ob's partial goes straight to its owner's plane
        assert epi == 0
        es = torch.empty((), dtype=out.dtype).element_size()
        for ob, v in enumerate(acc):
            if plane_div:  # batch ob -> plane ob // plane_div, sample ob % plane_div
                addr = d_planes[ob // plane_div] + (ob % plane_div) * planes_bs * es
            else:
                assert len(d_planes) >= len(acc)
                addr = d_planes[ob]
            _at(addr, out.dtype, (m, n), (ldd, 1)).copy_((v * alpha).to(out.dtype))
        return out
    for ob, v in enumerate(acc):
        _apply_epilogue(v, ob, m, n, epi, alpha, out, ldd, d_bs, d2, n, d2_bs, bias, bias_bs, resid, n, r_bs,
                        pre, n, p_bs, stats, stats_bs, lnb=lnb)
    if d_bcast or d2_bcast:
        assert len(acc) == 1
        _bcast_copy(_view(out, (m, n), (ldd, 1)), d_bcast)
        if d2 is not None:
            _bcast_copy(_view(d2, (m, n), (n, 1)), d2_bcast)
    return out


def _flag(addr, slot):
    return _at(addr + 4 * slot, torch.int32, (1,), (1,))


def _gemm_rs(acc, out, m, n, ldd, d_planes, rs, epi, alpha, d2, bias, resid, pre, stats, d_bcast, d2_bcast):
    """jg_gemm's fused reduce-scatter (include/jigsaw_sm100.h, rs_*) at plane granularity: raw
    partials to the owners, one arrival flag per sender (slot 1 + sender, written only by that
    sender), the own plane summed in member order with the partial dtype's rounding, then the
    epilogue with batch-0 addressing."""
    import time
    pdt = torch.bfloat16 if rs["part_type"] == 1 else torch.float32
    own = rs.get("own", -1) if rs.get("flags") else -1
    me, G = rs["src_idx"], rs["nsrc"]
    for ob, v in enumerate(acc):
        if ob == own:
            continue
        _at(d_planes[ob], pdt, (m, n), (ldd, 1)).copy_(v.to(pdt))
        _flag(rs["flag_peers"][ob], 1 + me).add_(1)
    if own < 0:
        return out
    t0 = time.time()
    peers = [j for j in range(G) if j != me]
    while any(int(_flag(rs["flags"], 1 + j).item()) < 1 for j in peers):
        assert time.time() - t0 < 120, "fused reduce-scatter: a peer never arrived"
        time.sleep(0.0005)
    for j in peers:
        _flag(rs["flags"], 1 + j).sub_(1)
    es = torch.empty((), dtype=pdt).element_size()
    tot = torch.zeros(m, n, dtype=torch.float64)
    for j in range(G):
        if j == me:
            tot += acc[own].to(pdt).double()
        else:
            tot += _at(rs["src"] + j * rs["src_stride"] * es, pdt, (m, n), (ldd, 1)).double()
    _apply_epilogue(tot, 0, m, n, epi, alpha, out, ldd, 0, d2, n, 0, bias, 0, resid, n, 0, pre, n, 0, stats, 0)
    if d_bcast or d2_bcast:
        _bcast_copy(_view(out, (m, n), (ldd, 1)), d_bcast)
        if d2 is not None:
            _bcast_copy(_view(d2, (m, n), (n, 1)), d2_bcast)
    return out


def epilogue(acc, m, n, *, batch=1, acc_ld=None, acc_bs=0, nplanes=1, epi=0, alpha=1.0, d=None, ldd=None, d_bs=0,
             d2=None, ldd2=None, d2_bs=0, bias=None, bias_bs=0, resid=None, ldr=None, r_bs=0, pre=None, ldp=None,
             p_bs=0, stats=None, stats_bs=0, d_bcast=None, d2_bcast=None):
    assert batch == 1 or not (d_bcast or d2_bcast)
    acc_ld = acc_ld if acc_ld is not None else n
    for ob in range(batch):
        if nplanes > 1:
            v = sum(_view(acc, (m, n), (acc_ld, 1), p * acc_bs).double() for p in range(nplanes))
        else:
            v = _view(acc, (m, n), (acc_ld, 1), ob * acc_bs).double()
        _apply_epilogue(v, ob, m, n, epi, alpha, d, ldd if ldd is not None else n, d_bs, d2,
                        ldd2 if ldd2 is not None else n, d2_bs, bias, bias_bs, resid, ldr if ldr is not None else n,
                        r_bs, pre, ldp if ldp is not None else n, p_bs, stats, stats_bs)
    if d_bcast:
        _bcast_copy(_view(d, (m, n), (ldd if ldd is not None else n, 1)), d_bcast)
    if d2_bcast:
        _bcast_copy(_view(d2, (m, n), (ldd2 if ldd2 is not None else n, 1)), d2_bcast)


def sum_planes(y, x, n, nplanes, plane_stride, accumulate=False):
    s = sum(x.reshape(-1)[p * plane_stride:p * plane_stride + n].double() for p in range(nplanes))
    if accumulate:
        s = s + y.reshape(-1)[:n].double()
    y.reshape(-1)[:n].copy_(s.float())  # x may be bf16 (partials), y is fp32


def axpy(y, x, alpha=1.0):
    y.add_(x.reshape(y.shape), alpha=alpha)


def cast_bf16(x, y):
    y.copy_(x.to(y.dtype))


def patchify(x, tok, batch, lat, lon, chans, pl, pw):
    t = x.reshape(batch, lat // pl, pl, lon // pw, pw, chans).permute(0, 1, 3, 5, 2, 4)
    tok.copy_(t.reshape(tok.shape).to(tok.dtype))


def _unpatchify(tok, batch, lat, lon, chans, pl, pw):
    t = tok.reshape(batch, lat // pl, lon // pw, chans, pl, pw).permute(0, 1, 4, 2, 5, 3)
    return t.reshape(batch, lat, lon, chans)


def zero(t):
    t.zero_()


def push(src, addrs, nbytes=None):
    for a in addrs or []:
        copy_async(a, src, nbytes)


def gelu_fwd(x, y):
    y.copy_(_gelu(x.double()).to(y.dtype))


def gelu_bwd(x, g, dx):
    dx.copy_((g.double() * _gelu_grad(x.double())).to(dx.dtype))


def matmul(a, b, mode="NN"):
    """tensor.matmul on CPU: exact float64 product, cast to the operand dtype."""
    from paper_2507_05753_b200.tensor import MatmulMode, _check_operands
    _check_operands(a, b, mode)
    mode = MatmulMode(mode)
    A, B = a.double(), b.double()
    if mode is MatmulMode.NT:
        B = B.transpose(-1, -2)
    elif mode is MatmulMode.TN:
        A = A.transpose(-1, -2)
    return torch.matmul(A, B).to(a.dtype)


def ln_moments(x, stats, rows, cols):
    xv = x.reshape(rows, cols).double()
    stats.view(rows, 2)[:, 0] += xv.sum(1).float()
    stats.view(rows, 2)[:, 1] += (xv * xv).sum(1).float()


def ln_apply(x, stats, gamma, beta, y, mean_rstd, rows, cols, c_total, eps, bcast=None):
    st = stats.reshape(rows, 2).double()
    mean = st[:, 0] / c_total
    var = st[:, 1] / c_total - mean * mean
    rstd = 1.0 / torch.sqrt(var + eps)
    if mean_rstd is not None:
        mean_rstd.reshape(rows, 2).copy_(torch.stack([mean, rstd], 1).float())
    xv = x.reshape(rows, cols).double()
    y.reshape(rows, cols).copy_((gamma.double() * (xv - mean[:, None]) * rstd[:, None] + beta.double()).to(y.dtype))
    _bcast_copy(y.reshape(rows, cols), bcast)


def ln_bwd_moments(x, g, gamma, mean_rstd, bstats, rows, cols):
    mr = mean_rstd.reshape(rows, 2).double()
    xh = (x.reshape(rows, cols).double() - mr[:, :1]) * mr[:, 1:]
    h = g.reshape(rows, cols).double() * gamma.double()
    bs = bstats.reshape(rows, 2)
    bs[:, 0] += h.sum(1).float()
    bs[:, 1] += (h * xh).sum(1).float()


def ln_bwd_apply(x, g, gamma, mean_rstd, bstats, resid, out, out_op, dgamma, dbeta, rows, cols, c_total,
                 bcast=None, rowsum=None, rowsum_period=0, colsum=None):
    mr = mean_rstd.reshape(rows, 2).double()
    xh = (x.reshape(rows, cols).double() - mr[:, :1]) * mr[:, 1:]
    gv = g.reshape(rows, cols).double()
    h = gv * gamma.double()
    bs = bstats.reshape(rows, 2).double()
    dx = mr[:, 1:] * (h - bs[:, :1] / c_total - xh * bs[:, 1:] / c_total)
    if resid is not None:
        dx = dx + resid.reshape(rows, cols).double()
    out.reshape(rows, cols).copy_(dx.to(out.dtype))
    if out_op is not None and out_op is not out:
        out_op.reshape(rows, cols).copy_(dx.to(out_op.dtype))
    if bcast:
        _bcast_copy((out_op if out_op is not None else out).reshape(rows, cols), bcast)
    if dgamma is not None:
        dgamma += (gv * xh).sum(0).float()
    if dbeta is not None:
        dbeta += gv.sum(0).float()
    if rowsum is not None:
        rowsum += dx.sum(1).reshape(-1, rowsum_period).sum(0).float()
    if colsum is not None:
        colsum += dx.sum(0).float()


def colsum(x, out, rows, cols, ld=None):
    out += _view(x, (rows, cols), (ld or cols, 1)).double().sum(0).float()


def rowsum(x, out, rows, cols, ld=None):
    out += _view(x, (rows, cols), (ld or cols, 1)).double().sum(1).float()


def blend_loss(dec, xin, target, blend_w, lat_w, var_w, g_ext, out, loss, g_blend, g_dec, batch, lat, lon, chans,
               pl, pw, inv_count, loss_scale, bcast=None):
    decoded = _unpatchify(dec.double(), batch, lat, lon, chans, pl, pw)
    x = xin.double()
    w = blend_w.double()
    o = w * decoded + (1 - w) * x
    if out is not None:
        out.copy_(o.float())
    if g_ext is None and target is None:
        return
    if g_ext is not None:
        gout = g_ext.double()
    else:
        wt = lat_w.double()[None, :, None, None] * var_w.double()[None, None, None, :]
        e = o - target.double()
        if loss is not None:
            loss += float((wt * e * e).sum() * inv_count)
        gout = 2 * wt * e * inv_count * loss_scale
    if g_blend is not None:
        g_blend += (gout * (decoded - x)).sum((0, 1, 2)).float()
    if g_dec is not None:
        gd = gout * w
        t = gd.reshape(batch, lat // pl, pl, lon // pw, pw, chans).permute(0, 1, 3, 5, 2, 4)
        g_dec.copy_(t.reshape(g_dec.shape).to(g_dec.dtype))
        _bcast_copy(g_dec, bcast)


def sqnorm(x, out, weight=1.0, n=None):
    xv = x.reshape(-1)[: x.numel() if n is None else n].double()
    out += float(weight) * float((xv * xv).sum())


def opt_schedule(step, scheds, sqsum, clip_norm, lr_out, grad_scale):
    t = int(step.item()) - 1
    for i, (base, warm, final, wsteps, total) in enumerate(scheds):
        if total <= 0:
            lr = base
        else:
            s_ = min(max(t, 0), total - 1)
            if s_ < wsteps:
                lr = warm + (base - warm) * s_ / wsteps
            else:
                span = total - 1 - wsteps
                u = (s_ - wsteps) / span if span > 0 else 1.0
                lr = final + 0.5 * (base - final) * (1 + math.cos(math.pi * u))
        lr_out[i] = lr
    if grad_scale is not None:
        f = 1.0
        if clip_norm and clip_norm > 0:
            norm = math.sqrt(float(sqsum.item()))
            if norm > clip_norm:
                f = clip_norm / norm
        grad_scale.fill_(f)


def adam(p, g, m, v, p_op, n, lr, beta1, beta2, eps, step, grad_scale=None, lr_dev=None, push=None, sms=None):
    t = int(step.item())
    if lr_dev is not None:
        lr = float(lr_dev.item())
    pv, gv, mv, vv = p.reshape(-1)[:n], g.reshape(-1)[:n], m.reshape(-1)[:n], v.reshape(-1)[:n]
    s = float(grad_scale.item()) if grad_scale is not None else 1.0
    gg = gv * s
    mv.mul_(beta1).add_((1 - beta1) * gg)
    vv.mul_(beta2).add_((1 - beta2) * gg * gg)
    pv.sub_(lr * (mv / (1 - beta1 ** t)) / (torch.sqrt(vv / (1 - beta2 ** t)) + eps))
    if p_op is not None:
        p_op.reshape(-1)[:n].copy_(pv.to(p_op.dtype))
    for start, ln, addrs in push or []:
        _bcast_copy(p_op.reshape(-1)[start:start + ln], addrs)


def step_increment(counter):
    counter += 1


NAMES = ["gemm", "epilogue", "sum_planes", "axpy", "cast_bf16", "patchify", "ln_moments", "ln_apply", "ln_bwd_moments",
         "ln_bwd_apply", "colsum", "rowsum", "blend_loss", "adam", "step_increment", "sqnorm", "opt_schedule",
         "copy_async", "gelu_fwd", "gelu_bwd", "push", "zero"]


def install():
    """Swap the package's kernel layer for this double (call inside a test process only)."""
    import paper_2507_05753_b200.kernels as K
    mod = globals()
    for name in NAMES:
        setattr(K, name, mod[name])
    import paper_2507_05753_b200.tensor as T
    T.matmul = matmul
