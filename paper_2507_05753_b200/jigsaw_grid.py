"""Jigsaw R x C execution of the WeatherMixer step (n = 2, 4, 8 GPUs).

Rank (r, c) of the grid (r: longitude part / token set, c: channel part) holds

  activations x, u, v, x2      [B, T_r, E/C]          patch features  [B, T_r, F/C]
  tok1 output h, gelu(h)       [B, E/R, d_tok/C]      ch1 output      [B, T_r, d_ch/C]
  enc.w [E/R, F/C]  tok1.w, tok2.w [T_r, d_tok/C]  ch1.w [d_ch/R, E/C]  ch2.w [E/R, d_ch/C]
  dec.w [F/R, E/C]  column vectors [./C] (shared by the column group), tok2.b [T_r] (row group)

so no weight or activation element is stored twice (the vectors excepted, as in the
reference, model.py:168-173). With (R, C) = (1, 2) / (2, 2) these are exactly the reference's
n = 2 / n = 4 tiles (model.py:135-150); (4, 2) is the 8-way grid.

Every layer is "gather one operand along one grid axis -> one local tcgen05 GEMM (1/n of the
FLOPs) -> reduce-scatter the fp32 partials along the other axis", replacing the reference's
point-to-point schedules (parallel.py:118-353) whose 4-way version is FLOP-imbalanced 1:3:3:1:

  channel NT (enc, ch1, ch2, dec)   fwd: W panel AG(col) at step start; GEMM -> [C][M][N/C]
                                         partials; RS(row); jg_epilogue (bias/GELU/residual/
                                         LN moments)
                                    bwd: AG(row) dY; dX = sum_j dY_j W_j (batch-reduced GEMM,
                                         GELU' fused); dW partial -> RS(col)
  tok1 TN  h = u^T W1               fwd: AG(row) u; GEMM -> [E, K/C] partial; RS(col)
  tok2 NT  o = W2 a^T               fwd: AG(col) a; GEMM -> [C][T_r][E/C]; RS(row)
  layer norm over split E           row moments all-reduced over the row group (stats_peer,
                                    model.py:220-231)
  duplicated-vector gradients       one all-reduce per (lr class, vector kind) (model.py:451-460)

Exchanges run through transport.py: on B200 the reduce-scatters are fused into the GEMM
epilogues (partial planes stored straight into the owner's NVLink-mapped buffer) and gathers
are copy-engine pushes, published by a device barrier — all on the compute stream, so the
whole step stays one CUDA graph; NCCL (or gloo in the CPU tests) is the alternative transport.
"""
from __future__ import annotations

import os

import torch

from . import _lib
from . import kernels as K
from .transport import Fanout, NcclTransport, SymmTransport, fused_rs_enabled

KM, MN = _lib.JG_KMAJOR, _lib.JG_MNMAJOR
E_ACC, E_BCOL, E_BROW, E_RES = _lib.EPI_ACCUM, _lib.EPI_BIAS_COL, _lib.EPI_BIAS_ROW, _lib.EPI_RESID
E_GF, E_GB, E_CP, E_ST = _lib.EPI_GELU_FWD, _lib.EPI_GELU_BWD, _lib.EPI_COPY_D2, _lib.EPI_STATS

CHANNEL_LAYERS = ("enc.w", "ch1.w", "ch2.w", "dec.w")
F32 = torch.float32


def _base(name: str) -> str:
    return name.split(".", 1)[-1] if name.startswith("block") else name


class GridWorkspace:
    """Transports (row / column group) with their persistent gather slots for one (batch, r)."""

    def __init__(self, m, ws):
        cfg, dev, ctx = m.cfg, m.device, m.ctx
        R, C = m.R, m.C
        B, nj = ws.B, ws.r * cfg.n_blocks
        E, H, F, Kd = cfg.d_emb, cfg.d_ch, cfg.patch_features, cfg.d_tok
        Tl, El, Er, Kl, Hl, Fl = ws.Tl, ws.El, ws.Er, ws.Kl, ws.Hl, ws.Fl
        M = B * Tl
        od = m.op_dtype
        self.R, self.C = R, C
        self.q = max(1, R // C)  # column-group owner chunks per row-gathered plane
        panel_shape = {"enc.w": (E, Fl), "ch1.w": (H, El), "ch2.w": (E, Hl), "dec.w": (F, El)}
        self.panel_names = [n for n in m.params if _base(n) in CHANNEL_LAYERS] if R > 1 else []
        nmax = max(E, H, F)
        row_persist = [(f"u_row{j}", (C, B, Tl, El), od) for j in range(nj)]  # plane-major: LN writes its plane
        row_persist += [("moments", (2, C, M, 2), F32)]  # layer-norm row moments, two alternating sub-slots
        row_persist += [("g", (C, M, El), od), ("gc", (C, M, Hl), od), ("gx2", (C, M, El), od), ("gd", (C, M, Fl), od),
                        ("tmp", (C, M, nmax // C), od)]
        col_persist = [("tmp", (R, max(E * Kl, max(E * Fl, H * El, E * Hl, F * El) // R)), od)]
        if R > 1:
            col_persist += [(f"a_col{j}", (B, R, Er, Kl), od) for j in range(nj)]
            col_persist += [("gh_col", (B, R, Er, Kl), od)]
            col_persist += [(f"panel:{n}", (R, panel_shape[_base(n)][0] // R, panel_shape[_base(n)][1]), od)
                            for n in self.panel_names]
        ps = 4
        row_scratch = max(M * nmax * ps, Tl * E * ps)
        kin_max = max(E * Fl, H * El, E * Hl, F * El)
        col_scratch = max(B * E * Kl * ps, kin_max * ps)  # token layers: all B samples' partials in one region
        kind = os.environ.get("JIGSAW_TRANSPORT", "symm" if dev.type == "cuda" else "nccl")
        if kind == "symm":
            self.row = SymmTransport(ctx.row_group, C, m.c, dev, row_scratch, row_persist) if C > 1 else None
            self.col = SymmTransport(ctx.col_group, R, m.r, dev, col_scratch, col_persist) if R > 1 else None
        else:
            self.row = NcclTransport(ctx.row_group, C, m.c, dev) if C > 1 else None
            self.col = NcclTransport(ctx.col_group, R, m.r, dev) if R > 1 else None
        if C == 1:
            # R x 1 grids (JIGSAW_GRID, e.g. 2x1 / 4x1): the row group is this rank alone — a
            # one-member transport whose gathers / reduce-scatters are local copies
            self.row = NcclTransport(None, 1, 0, dev)
        for tr, spec in ((self.row, row_persist), (self.col, col_persist)):
            if tr is not None and tr.kind == "nccl":
                for name, shape, dt in spec:
                    tr.reserve(name, shape, dt)
        self.kind = kind
        # layer-norm row moments summed over the row group through peer memory (push + barrier +
        # member-order plane sum) instead of an NCCL all-reduce
        self.peer_moments = kind == "symm" and C > 1 and peer_moments_enabled()
        self._mk = 0
        # GEMM + reduce-scatter + epilogue in one kernel (symmetric-memory transport, both axes)
        self.fused = kind == "symm" and fused_rs_enabled() and C > 1
        # reduce-scatter partial planes travel in the operand dtype (bf16 mode: half the NVLink bytes
        # and half the epilogue reads; summed in fp32); JIGSAW_PARTIALS=fp32 keeps fp32 partials
        bf = od == torch.bfloat16 and os.environ.get("JIGSAW_PARTIALS", "bf16") != "fp32"
        self.pdt = torch.bfloat16 if bf else F32
        self.dgrad = torch.empty(max(kin_max, E * Kl), dtype=F32, device=dev)  # reduced weight gradients
        # per-sample token GEMMs of a B > 1 step run side by side on a few side streams
        self.fan = Fanout(dev, min(B, int(os.environ.get("JIGSAW_FANOUT", "4"))))
        self.panels = {n: self.col.persistent(f"panel:{n}").view(panel_shape[_base(n)]) for n in self.panel_names}
        # live buffers of received parameter blocks (reference MpContext.param_buffer_peak,
        # parallel.py:71-76): the peers' planes of every gathered weight panel, held for the step
        held = sum(p.numel() * (R - 1) // R for p in self.panels.values())
        ctx.param_buffer_peak = max(ctx.param_buffer_peak, held)


def peer_moments_enabled() -> bool:
    return os.environ.get("JIGSAW_PEER_MOMENTS", "1") == "1"


def row_reduce(m, g, t: torch.Tensor) -> torch.Tensor:
    """Sum of a row-moment buffer [M, 2] over the row group (the grid form of the reference's
    stats_peer exchange, model.py:220-231): every member pushes its partials into every member's
    "moments" slot (copy engine), one barrier, then the planes are summed in member order — the
    same bits on every member, no NCCL launch. NCCL all-reduce on the NCCL transport."""
    if not g.peer_moments:
        return m.ctx.all_reduce_row(t)
    sub = g._mk % 2
    g._mk += 1
    planes = g.row.ag(t.view(-1), slot="moments", sub=sub, nsub=2)
    K.sum_planes(t.view(-1), planes, t.numel(), m.C, t.numel())
    return t


def _gw(m, ws) -> GridWorkspace:
    if getattr(ws, "grid", None) is None:
        ws.grid = GridWorkspace(m, ws)
    return ws.grid


def _panel(m, g, name):
    return g.panels[name] if m.R > 1 else m.params[name].op


def gather_panels(m, g) -> None:
    """All-gather every channel-mixing weight's rows over the column group (final for the step)."""
    for name in g.panel_names:
        g.col.ag(m.params[name].op, slot=f"panel:{name}")


def panel_push_segments(m, g, lo: int, hi: int):
    """Adam-side weight-panel gather (symmetric-memory transport, R > 1): for the flat range
    [lo, hi) of one Adam call, the channel-mixing weights in it as (start - lo, numel, addrs) —
    addrs = this rank's plane of the weight's panel slot in every column-group member's arena
    (own included), where the optimiser stores the new bf16 operand copy. The next forward then
    only needs one column-group barrier instead of one copy + barrier per panel."""
    if g.kind != "symm" or g.col is None or not g.panel_names:
        return []
    f = m.flat
    es = f.op.element_size()
    base = f.op.data_ptr()
    segs = []
    for name in g.panel_names:
        op = m.params[name].op
        start = (op.data_ptr() - base) // es
        if not lo <= start < hi:
            continue
        nbytes = op.numel() * es
        off = g.col._slot_off(f"panel:{name}", 0, nbytes) + g.col.idx * nbytes
        segs.append((start - lo, op.numel(), [g.col.base[j] + off for j in range(g.col.G)]))
        g.col.bytes_sent += (g.col.G - 1) * nbytes  # the optimiser's stores into the peers' panel slots
    return segs


def panels_ready(m, g) -> None:
    """Forward prologue when the previous step's Adam pushed the panels: one barrier publishes
    every member's pushes (their Adam kernels end with a system fence)."""
    g.col.barrier()


def _wgrad_planes(m, g, wname, acc, nplanes, plane_stride, numel):
    """Weight gradient that arrived as reduce-scatter planes: sum them into the gradient sink."""
    if nplanes == 1 and acc.dtype == F32:
        m._wgrad_reduced(wname, acc)
        return
    if getattr(m, "_grad_overwrite", False) and getattr(m, "_fused_adam", None) is None:
        K.sum_planes(m.params[wname].grad, acc, numel, nplanes, plane_stride)  # straight into the gradient
        return
    red = g.dgrad[:numel]
    K.sum_planes(red, acc, numel, nplanes, plane_stride)
    m._wgrad_reduced(wname, red.view(m.params[wname].data.shape))


# --------------------------------------------------------------------------- channel layers
def chan_fwd(m, g, X, panel, M, kin_l, nout, **epi):
    """Y[M, nout/C] = X[M, kin_l] W^T (+ epilogue), W panel [nout, kin_l]; RS over the row group."""
    C = m.C
    nl = nout // C

    def fn(s, D, d_bs, dpl, **kw):
        K.gemm(D, X, panel, KM, KM, M, nl, kin_l, C, 0, nl * kin_l, d_bs=d_bs, d_planes=dpl, **kw)

    if g.fused:
        g.row.rs_gemm_fused(M, nl, g.pdt, fn, **epi)
        return
    acc, npl, ps = g.row.rs_gemm(M, nl, g.pdt, fn)
    K.epilogue(acc, M, nl, acc_bs=ps, nplanes=npl, **epi)


def chan_bwd(m, g, dY, X, panel, M, kin_l, nout, wname, bname, bias_src, dX=None, dyrow=None, **dx_epi):
    """Backward of Y = X W^T: dX (optional, fused epilogue, may push its output to peers), dW via
    RS over the column group, bias-gradient partial (summed over the column group in grad_sync).
    `dyrow`: dY already gathered over the row group by its producer ([C, M, nout/C])."""
    R, C = m.R, m.C
    nl = nout // C
    if dyrow is None:
        dyrow = g.row.ag(dY)                                    # [C, M, nl]
    if dX is not None:
        K.gemm(dX, dyrow, panel, KM, MN, M, kin_l, nl, C, M * nl, nl * kin_l, reduce_batch=True, **dx_epi)
    if R == 1:
        out, kw = m._wgrad(wname)
        K.gemm(out, dyrow, X, MN, MN, nl, kin_l, M, C, M * nl, 0, d_bs=nl * kin_l, **kw)
    else:
        q, nr = g.q, nout // R

        def fn(s, D, d_bs, dpl, **kw):  # rows sub-chunk s of every gathered plane j -> owner j*q+s
            K.gemm(D, dyrow[..., s * nr:], X, MN, MN, nr, kin_l, M, C, M * nl, 0, d_bs=d_bs, d_planes=dpl,
                   lda=nl, **kw)

        if g.fused and getattr(m, "_grad_overwrite", False) and getattr(m, "_fused_adam", None) is None:
            g.col.rs_gemm_fused(nr, kin_l, g.pdt, fn, q=q, d=m.params[wname].grad)  # straight into the gradient
        else:
            acc, npl, ps = g.col.rs_gemm(nr, kin_l, g.pdt, fn, q=q)
            _wgrad_planes(m, g, wname, acc, npl, ps, nr * kin_l)
    if bias_src is not None:  # (None: the layer-norm backward pass that produced dY summed it)
        K.colsum(bias_src, m.params[bname].grad, M, nl)


# --------------------------------------------------------------------------- token layers
def tok1_fwd(m, g, ws, j, bi, b, urow):
    """h = u^T W1 + b1, a = gelu(h): rows of h (E) gathered over the row group, split R ways.
    urow: [C, Tl, El] view of the gathered u (plane stride B*Tl*El). Returns gelu(h) columns
    gathered over the column group ([E, Kl]) when R > 1, else the local a."""
    p, R, C = m.params, m.R, m.C
    Tl, El, Er, Kl, B = ws.Tl, ws.El, ws.Er, ws.Kl, ws.B
    ps = B * Tl * El
    if R == 1:
        K.gemm(ws.h[j][bi], urow, p[b + "tok1.w"].op, MN, MN, El, Kl, Tl, C, ps, 0, d_bs=El * Kl,
               epi=E_BCOL | E_GF, bias=p[b + "tok1.b"].data, d2=ws.a[j][bi], d2_bs=El * Kl)
        return ws.a[j][bi]
    q = g.q

    def fn(s, D, d_bs, dpl, **kw):  # rows [s*Er, (s+1)*Er) of plane j -> owner j*q+s
        K.gemm(D, urow[..., s * Er:], p[b + "tok1.w"].op, MN, MN, Er, Kl, Tl, C, ps, 0, d_bs=d_bs,
               d_planes=dpl, lda=El, **kw)

    ha = g.col.dest((Er, Kl), m.op_dtype, slot=f"a_col{j}", sub=bi, nsub=B)   # gelu(h) pushed to peers
    epi = dict(epi=E_BCOL | E_GF, bias=p[b + "tok1.b"].data, d=ws.h[j][bi], d2=ha.own, d2_bcast=ha.peers)
    if g.fused:
        g.col.rs_gemm_fused(Er, Kl, g.pdt, fn, q=q, **epi)
    else:
        acc, npl, pst = g.col.rs_gemm(Er, Kl, g.pdt, fn, q=q)
        K.epilogue(acc, Er, Kl, acc_bs=pst, nplanes=npl, **epi)
    g.col.publish(ha)
    return ha.planes.view(-1, Kl)


def tok2_fwd(m, g, ws, j, bi, b, acol):
    """x2 = x + W2 a^T + b2[:, None]: a gathered over the column group; RS over the row group."""
    p, C = m.params, m.C
    Tl, El, Kl = ws.Tl, ws.El, ws.Kl

    def fn(s, D, d_bs, dpl, **kw):
        K.gemm(D, p[b + "tok2.w"].op, acol, KM, KM, Tl, El, Kl, C, 0, El * Kl, d_bs=d_bs, d_planes=dpl, **kw)

    epi = dict(epi=E_BROW | E_RES | E_ST, bias=p[b + "tok2.b"].data, resid=ws.res[j][bi], d=ws.x2[j][bi],
               stats=ws.st2[j][bi * Tl:(bi + 1) * Tl])
    if g.fused:
        g.row.rs_gemm_fused(Tl, El, g.pdt, fn, **epi)
        return
    acc, npl, ps = g.row.rs_gemm(Tl, El, g.pdt, fn)
    K.epilogue(acc, Tl, El, acc_bs=ps, nplanes=npl, **epi)


def tok2_bwd(m, g, ws, j, bi, b, grow, acol):
    """gh = (g_x2^T W2) * gelu'(h) (RS over the column group, pushed back out over it for tok1's
    backward); dW2 += g_x2 a (local). grow: gathered g_x2 [C, Tl, El] (plane stride B*Tl*El).
    Returns (gh local block, gh gathered over the column group [E, Kl])."""
    p, R, C = m.params, m.R, m.C
    Tl, El, Er, Kl, B = ws.Tl, ws.El, ws.Er, ws.Kl, ws.B
    ps = B * Tl * El
    if R == 1:
        K.gemm(ws.gh[bi], grow, p[b + "tok2.w"].op, MN, MN, El, Kl, Tl, C, ps, 0, d_bs=El * Kl,
               epi=E_GB, pre=ws.h[j][bi])
        gh_local, ghcol = ws.gh[bi], ws.gh[bi]
    else:
        q = g.q

        def fn(s, D, d_bs, dpl, **kw):
            K.gemm(D, grow[..., s * Er:], p[b + "tok2.w"].op, MN, MN, Er, Kl, Tl, C, ps, 0, d_bs=d_bs,
                   d_planes=dpl, lda=El, **kw)

        hg = g.col.dest((Er, Kl), m.op_dtype, slot="gh_col", sub=bi, nsub=B)
        epi = dict(epi=E_GB, pre=ws.h[j][bi], d=hg.own, d_bcast=hg.peers)
        if g.fused:
            g.col.rs_gemm_fused(Er, Kl, g.pdt, fn, q=q, **epi)
        else:
            acc, npl, pst = g.col.rs_gemm(Er, Kl, g.pdt, fn, q=q)
            K.epilogue(acc, Er, Kl, acc_bs=pst, nplanes=npl, **epi)
        g.col.publish(hg)
        gh_local, ghcol = hg.own, hg.planes.view(-1, Kl)
    out, kw = m._wgrad(b + "tok2.w") if bi == 0 or B == 1 else (p[b + "tok2.w"].grad, {"epi": E_ACC})
    if bi == 0 and B > 1 and kw.get("epi") == _lib.EPI_ADAM:
        out, kw = p[b + "tok2.w"].grad, {"epi": E_ACC}
    K.gemm(out, grow, acol, KM, MN, Tl, Kl, El, C, ps, El * Kl, reduce_batch=True, **kw)
    return gh_local, ghcol


def tok1_bwd(m, g, ws, j, bi, b, ghcol):
    """gu = W1 gh^T (gh gathered over the column group, RS over the row group); dW1 += u gh."""
    p, C = m.params, m.C
    Tl, El, Kl, B = ws.Tl, ws.El, ws.Kl, ws.B

    def fn(s, D, d_bs, dpl, **kw):
        K.gemm(D, p[b + "tok1.w"].op, ghcol, KM, KM, Tl, El, Kl, C, 0, El * Kl, d_bs=d_bs, d_planes=dpl, **kw)

    if g.fused:
        g.row.rs_gemm_fused(Tl, El, g.pdt, fn, d=ws.gu[bi])
    else:
        acc, npl, ps = g.row.rs_gemm(Tl, El, g.pdt, fn, out=ws.gu[bi])
        if npl > 1 or acc.data_ptr() != ws.gu[bi].data_ptr():
            K.sum_planes(ws.gu[bi], acc, Tl * El, npl, ps)
    urow = g.row.persistent(f"u_row{j}").view(C, B, Tl, El)[:, bi]
    out, kw = m._wgrad(b + "tok1.w") if bi == 0 or B == 1 else (p[b + "tok1.w"].grad, {"epi": E_ACC})
    if bi == 0 and B > 1 and kw.get("epi") == _lib.EPI_ADAM:
        out, kw = p[b + "tok1.w"].grad, {"epi": E_ACC}
    K.gemm(out, urow, ghcol, KM, MN, Tl, Kl, El, C, B * Tl * El, El * Kl, reduce_batch=True, **kw)


# ------------------------------------------------ token layers, all B samples per exchange
# The token-mixing GEMMs run per sample (weight-first / transposed products of one sample's
# tiles), but their exchanges do not need a barrier each: every sample's GEMM stores its
# partial planes into its own part of one reduce-scatter region and its gathered output into
# its own sub-slot, and ONE barrier per layer publishes all B samples (rs_gemm_multi /
# publish_all) — B times fewer device barriers than a reduce-scatter per sample.
def tok1_fwd_all(m, g, ws, j, b, uall):
    """tok1_fwd for every sample; uall [C, B, Tl, El] (the row-gathered u). Returns the gelu(h)
    operands of tok2 per sample."""
    B = ws.B
    if g.fused:
        return [tok1_fwd(m, g, ws, j, bi, b, uall[:, bi]) for bi in range(B)]
    if m.R == 1:  # local GEMMs, one per sample, side by side
        g.fan([lambda bi=bi: tok1_fwd(m, g, ws, j, bi, b, uall[:, bi]) for bi in range(B)])
        return [ws.a[j][bi] for bi in range(B)]
    p = m.params
    Tl, El, Er, Kl = ws.Tl, ws.El, ws.Er, ws.Kl
    C, q, ps = m.C, g.q, B * Tl * El
    fns, has = [], []
    for bi in range(B):
        urow = uall[:, bi]

        def fn(s, D, d_bs, dpl, urow=urow, **kw):
            K.gemm(D, urow[..., s * Er:], p[b + "tok1.w"].op, MN, MN, Er, Kl, Tl, C, ps, 0, d_bs=d_bs,
                   d_planes=dpl, lda=El, **kw)
        fns.append(fn)
        has.append(g.col.dest((Er, Kl), m.op_dtype, slot=f"a_col{j}", sub=bi, nsub=B))
    res = g.col.rs_gemm_multi(Er, Kl, g.pdt, fns, q=q, run=g.fan)
    g.fan([lambda bi=bi, r=r: K.epilogue(r[0], Er, Kl, acc_bs=r[2], nplanes=r[1], epi=E_BCOL | E_GF,
                                         bias=p[b + "tok1.b"].data, d=ws.h[j][bi], d2=has[bi].own,
                                         d2_bcast=has[bi].peers) for bi, r in enumerate(res)])
    g.col.publish_all(has)
    return [ha.planes.view(-1, Kl) for ha in has]


def tok2_fwd_all(m, g, ws, j, b, acols):
    B = ws.B
    if g.fused or B == 1:
        for bi in range(B):
            tok2_fwd(m, g, ws, j, bi, b, acols[bi])
        return
    p, C = m.params, m.C
    Tl, El, Kl = ws.Tl, ws.El, ws.Kl
    fns = []
    for bi in range(B):
        def fn(s, D, d_bs, dpl, acol=acols[bi], **kw):
            K.gemm(D, p[b + "tok2.w"].op, acol, KM, KM, Tl, El, Kl, C, 0, El * Kl, d_bs=d_bs, d_planes=dpl, **kw)
        fns.append(fn)
    res = g.row.rs_gemm_multi(Tl, El, g.pdt, fns, run=g.fan)
    g.fan([lambda bi=bi, r=r: K.epilogue(r[0], Tl, El, acc_bs=r[2], nplanes=r[1], epi=E_BROW | E_RES | E_ST,
                                         bias=p[b + "tok2.b"].data, resid=ws.res[j][bi], d=ws.x2[j][bi],
                                         stats=ws.st2[j][bi * Tl:(bi + 1) * Tl]) for bi, r in enumerate(res)])


def tok2_bwd_all(m, g, ws, j, b, xall, acols):
    """tok2_bwd for every sample: gh reduce-scatters over the column group (one barrier), gh
    pushed back out over it (one barrier), then the dW2 GEMMs. Returns (gh local, gh gathered)
    per sample."""
    B = ws.B
    if g.fused or B == 1:
        return [tok2_bwd(m, g, ws, j, bi, b, xall[:, bi], acols[bi]) for bi in range(B)]
    p = m.params
    Tl, El, Er, Kl = ws.Tl, ws.El, ws.Er, ws.Kl
    C, q, ps = m.C, g.q, B * Tl * El
    if m.R == 1:
        # gh = (g_x2^T W2) * gelu'(h), local, one GEMM per sample side by side
        g.fan([lambda bi=bi: K.gemm(ws.gh[bi], xall[:, bi], p[b + "tok2.w"].op, MN, MN, El, Kl, Tl, C, ps, 0,
                                    d_bs=El * Kl, epi=E_GB, pre=ws.h[j][bi]) for bi in range(B)])
        _dw_tok2(m, ws, b, xall, acols)
        return [(ws.gh[bi], ws.gh[bi]) for bi in range(B)]
    fns, hgs = [], []
    for bi in range(B):
        grow = xall[:, bi]

        def fn(s, D, d_bs, dpl, grow=grow, **kw):
            K.gemm(D, grow[..., s * Er:], p[b + "tok2.w"].op, MN, MN, Er, Kl, Tl, C, ps, 0, d_bs=d_bs,
                   d_planes=dpl, lda=El, **kw)
        fns.append(fn)
        hgs.append(g.col.dest((Er, Kl), m.op_dtype, slot="gh_col", sub=bi, nsub=B))
    res = g.col.rs_gemm_multi(Er, Kl, g.pdt, fns, q=q, run=g.fan)
    g.fan([lambda bi=bi, r=r: K.epilogue(r[0], Er, Kl, acc_bs=r[2], nplanes=r[1], epi=E_GB, pre=ws.h[j][bi],
                                         d=hgs[bi].own, d_bcast=hgs[bi].peers) for bi, r in enumerate(res)])
    g.col.publish_all(hgs)
    _dw_tok2(m, ws, b, xall, acols)
    return [(hg.own, hg.planes.view(-1, Kl)) for hg in hgs]


def _dw_tok2(m, ws, b, xall, acols):
    """dW2 = sum_b g_x2[b] a[b]: the samples accumulate into one gradient, so in order."""
    p, C, B = m.params, m.C, ws.B
    Tl, El, Kl = ws.Tl, ws.El, ws.Kl
    for bi in range(B):
        out, kw = m._wgrad(b + "tok2.w") if bi == 0 else (p[b + "tok2.w"].grad, {"epi": E_ACC})
        if bi == 0 and kw.get("epi") == _lib.EPI_ADAM:
            out, kw = p[b + "tok2.w"].grad, {"epi": E_ACC}
        K.gemm(out, xall[:, bi], acols[bi], KM, MN, Tl, Kl, El, C, B * Tl * El, El * Kl, reduce_batch=True, **kw)


def tok1_bwd_all(m, g, ws, j, b, ghcols):
    B = ws.B
    if g.fused or B == 1:
        for bi in range(B):
            tok1_bwd(m, g, ws, j, bi, b, ghcols[bi])
        return
    p, C = m.params, m.C
    Tl, El, Kl = ws.Tl, ws.El, ws.Kl
    fns = []
    for bi in range(B):
        def fn(s, D, d_bs, dpl, ghcol=ghcols[bi], **kw):
            K.gemm(D, p[b + "tok1.w"].op, ghcol, KM, KM, Tl, El, Kl, C, 0, El * Kl, d_bs=d_bs, d_planes=dpl, **kw)
        fns.append(fn)
    res = g.row.rs_gemm_multi(Tl, El, g.pdt, fns, outs=[ws.gu[bi] for bi in range(B)], run=g.fan)
    g.fan([lambda bi=bi, r=r: K.sum_planes(ws.gu[bi], r[0], Tl * El, r[1], r[2]) for bi, r in enumerate(res)
           if r[1] > 1 or r[0].data_ptr() != ws.gu[bi].data_ptr()])
    for bi in range(B):
        urow = g.row.persistent(f"u_row{j}").view(C, B, Tl, El)[:, bi]
        out, kw = m._wgrad(b + "tok1.w") if bi == 0 else (p[b + "tok1.w"].grad, {"epi": E_ACC})
        if bi == 0 and kw.get("epi") == _lib.EPI_ADAM:
            out, kw = p[b + "tok1.w"].grad, {"epi": E_ACC}
        K.gemm(out, urow, ghcols[bi], KM, MN, Tl, Kl, El, C, B * Tl * El, El * Kl, reduce_batch=True, **kw)


# ------------------------------------- token layers, B > 1: plane-major, batched over samples
# For B > 1 the token-mixing tensors of the grid step are kept PLANE-MAJOR: chunk j (El rows of
# the E axis) of every sample next to each other, [C][B][El][Kl] — the gathered u and g_x2 (row
# group slots, [C][B][Tl][El]), the tok1 output h / gelu(h) and the gradient gh (at R = 1 the
# local buffers reinterpreted; at R > 1 the column-group gather slots, filled through dest_pm).
# Then every per-(chunk, sample) product has ONE uniform stride, so the local token GEMMs (tok1
# forward and the gh GEMM at R = 1) and both weight-gradient GEMMs (dW1, dW2: a reduction over
# chunks AND samples) are one launch per layer instead of one per sample; the reduce-scatter
# GEMMs stay per sample (their owner planes are per sample) and run side by side (g.fan).
def _pm_path(m, g, ws) -> bool:
    return ws.B > 1 and not g.fused


def _pm_view(t: torch.Tensor, C: int, B: int, El: int, Kl: int) -> torch.Tensor:
    return t.reshape(-1)[:C * B * El * Kl].view(C, B, El, Kl)


def tok1_fwd_pm(m, g, ws, j, b, uall):
    """h = u^T W1 + b1, a = gelu(h) for all samples; uall [C, B, Tl, El] (row-gathered u).
    Returns a plane-major [C, B, El, Kl] (tok2's operand, dW2's B operand)."""
    p, R, C, B = m.params, m.R, m.C, ws.B
    Tl, El, Er, Kl = ws.Tl, ws.El, ws.Er, ws.Kl
    if R == 1:
        hv, av = _pm_view(ws.h[j], C, B, El, Kl), _pm_view(ws.a[j], C, B, El, Kl)
        K.gemm(hv, uall, p[b + "tok1.w"].op, MN, MN, El, Kl, Tl, C * B, Tl * El, 0, d_bs=El * Kl,
               epi=E_BCOL | E_GF, bias=p[b + "tok1.b"].data, d2=av, d2_bs=El * Kl)
        return av
    q, ps = g.q, B * Tl * El
    fns, has = [], []
    for bi in range(B):
        urow = uall[:, bi]

        def fn(s, D, d_bs, dpl, urow=urow, **kw):
            K.gemm(D, urow[..., s * Er:], p[b + "tok1.w"].op, MN, MN, Er, Kl, Tl, C, ps, 0, d_bs=d_bs,
                   d_planes=dpl, lda=El, **kw)
        fns.append(fn)
        has.append(g.col.dest_pm((Er, Kl), m.op_dtype, f"a_col{j}", bi, B, q))

    def fnb(s, D, dpl, pdiv, pbs):  # every (plane, sample) item in one launch: plane-major uall
        K.gemm(D, uall[..., s * Er:], p[b + "tok1.w"].op, MN, MN, Er, Kl, Tl, C * B, Tl * El, 0,
               d_planes=dpl, plane_div=pdiv, planes_bs=pbs, lda=El)
    res = g.col.rs_gemm_batched(Er, Kl, g.pdt, B, fns, fnb, q=q, run=g.fan)
    g.fan([lambda bi=bi, r=r: K.epilogue(r[0], Er, Kl, acc_bs=r[2], nplanes=r[1], epi=E_BCOL | E_GF,
                                         bias=p[b + "tok1.b"].data, d=ws.h[j][bi], d2=has[bi].own,
                                         d2_bcast=has[bi].peers) for bi, r in enumerate(res)])
    g.col.publish_all(has)
    return _pm_view(g.col.persistent(f"a_col{j}"), C, B, El, Kl)


def tok2_fwd_pm(m, g, ws, j, b, av):
    """x2 = x + W2 a^T + b2[:, None] per sample (RS over the row group), side by side."""
    p, C, B = m.params, m.C, ws.B
    Tl, El, Kl = ws.Tl, ws.El, ws.Kl
    fns = []
    for bi in range(B):
        def fn(s, D, d_bs, dpl, a0=av[0, bi], **kw):
            K.gemm(D, p[b + "tok2.w"].op, a0, KM, KM, Tl, El, Kl, C, 0, B * El * Kl, d_bs=d_bs, d_planes=dpl, **kw)
        fns.append(fn)

    def fnb(s, D, dpl, pdiv, pbs):  # every (plane, sample) item in one launch: plane-major a
        K.gemm(D, p[b + "tok2.w"].op, av, KM, KM, Tl, El, Kl, C * B, 0, El * Kl, d_planes=dpl,
               plane_div=pdiv, planes_bs=pbs)
    res = g.row.rs_gemm_batched(Tl, El, g.pdt, B, fns, fnb, run=g.fan)
    g.fan([lambda bi=bi, r=r: K.epilogue(r[0], Tl, El, acc_bs=r[2], nplanes=r[1], epi=E_BROW | E_RES | E_ST,
                                         bias=p[b + "tok2.b"].data, resid=ws.res[j][bi], d=ws.x2[j][bi],
                                         stats=ws.st2[j][bi * Tl:(bi + 1) * Tl]) for bi, r in enumerate(res)])


def tok2_bwd_pm(m, g, ws, j, b, xall, av):
    """gh = (g_x2^T W2) * gelu'(h) for all samples (plane-major), the tok1 bias gradient, and
    dW2 = sum over chunks and samples of g_x2 a — one GEMM. xall [C, B, Tl, El]."""
    p, R, C, B = m.params, m.R, m.C, ws.B
    Tl, El, Er, Kl = ws.Tl, ws.El, ws.Er, ws.Kl
    if R == 1:
        ghv = _pm_view(ws.gh, C, B, El, Kl)
        K.gemm(ghv, xall, p[b + "tok2.w"].op, MN, MN, El, Kl, Tl, C * B, Tl * El, 0, d_bs=El * Kl, epi=E_GB,
               pre=_pm_view(ws.h[j], C, B, El, Kl), p_bs=El * Kl)
        K.colsum(ghv, p[b + "tok1.b"].grad, C * B * El, Kl)
    else:
        q, ps = g.q, B * Tl * El
        fns, hgs = [], []
        for bi in range(B):
            grow = xall[:, bi]

            def fn(s, D, d_bs, dpl, grow=grow, **kw):
                K.gemm(D, grow[..., s * Er:], p[b + "tok2.w"].op, MN, MN, Er, Kl, Tl, C, ps, 0, d_bs=d_bs,
                       d_planes=dpl, lda=El, **kw)
            fns.append(fn)
            hgs.append(g.col.dest_pm((Er, Kl), m.op_dtype, "gh_col", bi, B, q))

        def fnb(s, D, dpl, pdiv, pbs):  # every (plane, sample) item in one launch: plane-major g_x2
            K.gemm(D, xall[..., s * Er:], p[b + "tok2.w"].op, MN, MN, Er, Kl, Tl, C * B, Tl * El, 0,
                   d_planes=dpl, plane_div=pdiv, planes_bs=pbs, lda=El)
        res = g.col.rs_gemm_batched(Er, Kl, g.pdt, B, fns, fnb, q=q, run=g.fan)
        g.fan([lambda bi=bi, r=r: K.epilogue(r[0], Er, Kl, acc_bs=r[2], nplanes=r[1], epi=E_GB, pre=ws.h[j][bi],
                                             d=hgs[bi].own, d_bcast=hgs[bi].peers) for bi, r in enumerate(res)])
        for hg in hgs:  # (into one bias gradient: in order)
            K.colsum(hg.own, p[b + "tok1.b"].grad, Er, Kl)
        g.col.publish_all(hgs)
        ghv = _pm_view(g.col.persistent("gh_col"), C, B, El, Kl)
    out, kw = m._wgrad(b + "tok2.w")
    K.gemm(out, xall, av, KM, MN, Tl, Kl, El, C * B, Tl * El, El * Kl, reduce_batch=True, **kw)
    return ghv


def tok1_bwd_pm(m, g, ws, j, b, uall, ghv):
    """gu = W1 gh^T per sample (RS over the row group, side by side); dW1 = sum over chunks and
    samples of u gh — one GEMM."""
    p, C, B = m.params, m.C, ws.B
    Tl, El, Kl = ws.Tl, ws.El, ws.Kl
    fns = []
    for bi in range(B):
        def fn(s, D, d_bs, dpl, g0=ghv[0, bi], **kw):
            K.gemm(D, p[b + "tok1.w"].op, g0, KM, KM, Tl, El, Kl, C, 0, B * El * Kl, d_bs=d_bs, d_planes=dpl, **kw)
        fns.append(fn)

    def fnb(s, D, dpl, pdiv, pbs):  # every (plane, sample) item in one launch: plane-major gh
        K.gemm(D, p[b + "tok1.w"].op, ghv, KM, KM, Tl, El, Kl, C * B, 0, El * Kl, d_planes=dpl,
               plane_div=pdiv, planes_bs=pbs)
    res = g.row.rs_gemm_batched(Tl, El, g.pdt, B, fns, fnb, outs=[ws.gu[bi] for bi in range(B)], run=g.fan)
    g.fan([lambda bi=bi, r=r: K.sum_planes(ws.gu[bi], r[0], Tl * El, r[1], r[2]) for bi, r in enumerate(res)
           if r[1] > 1 or r[0].data_ptr() != ws.gu[bi].data_ptr()])
    out, kw = m._wgrad(b + "tok1.w")
    K.gemm(out, uall, ghv, KM, MN, Tl, Kl, El, C * B, Tl * El, El * Kl, reduce_batch=True, **kw)


# --------------------------------------------------------------------------- forward / backward
def forward_grid(m, ws) -> None:
    g = _gw(m, ws)
    cfg, p, ctx = m.cfg, m.params, m.ctx
    R, C = m.R, m.C
    B = ws.B
    E, H, F = cfg.d_emb, cfg.d_ch, cfg.patch_features
    Tl, El, Kl, Hl, Fl = ws.Tl, ws.El, ws.Kl, ws.Hl, ws.Fl
    M = B * Tl
    lat, lon = m.local_grid
    od = m.op_dtype
    K.zero(ws.stats)
    if getattr(m, "_panels_pushed", False) and g.kind == "symm" and g.panel_names:
        panels_ready(m, g)
    else:
        gather_panels(m, g)
    K.patchify(ws.xin, ws.xp, B, lat, lon, m.local_vars, cfg.patch[0], cfg.patch[1])
    chan_fwd(m, g, ws.xp, _panel(m, g, "enc.w"), M, Fl, E, epi=E_BCOL | E_ST, bias=p["enc.b"].data,
             d=ws.res[0], stats=ws.st1[0])
    nj = ws.r * cfg.n_blocks
    for j in range(nj):
        b = f"block{j % cfg.n_blocks}."
        row_reduce(m, g, ws.st1[j])
        hu = g.row.dest((M, El), od, slot=f"u_row{j}")          # LN1 output pushed to the row group
        K.ln_apply(ws.res[j], ws.st1[j], p[b + "ln1.gamma"].data, p[b + "ln1.beta"].data, hu.own, ws.mr1[j],
                   M, El, E, m.eps, bcast=hu.peers)
        g.row.publish(hu)
        uall = hu.planes.view(C, B, Tl, El)
        if _pm_path(m, g, ws):
            tok2_fwd_pm(m, g, ws, j, b, tok1_fwd_pm(m, g, ws, j, b, uall))
        else:
            acols = tok1_fwd_all(m, g, ws, j, b, uall)
            tok2_fwd_all(m, g, ws, j, b, acols)
        row_reduce(m, g, ws.st2[j])
        K.ln_apply(ws.x2[j], ws.st2[j], p[b + "ln2.gamma"].data, p[b + "ln2.beta"].data, ws.v[j], ws.mr2[j],
                   M, El, E, m.eps)
        chan_fwd(m, g, ws.v[j], _panel(m, g, b + "ch1.w"), M, El, H, epi=E_BCOL | E_GF,
                 bias=p[b + "ch1.b"].data, d=ws.c[j], d2=ws.ca[j])
        last = j == nj - 1
        copy_y = last and ws.y_op is not ws.res[nj]
        chan_fwd(m, g, ws.ca[j], _panel(m, g, b + "ch2.w"), M, Hl, E,
                 epi=E_BCOL | E_RES | (E_CP if copy_y else 0) | (0 if last else E_ST), bias=p[b + "ch2.b"].data,
                 resid=ws.x2[j], d=ws.res[j + 1], d2=ws.y_op if copy_y else None,
                 stats=None if last else ws.st1[j + 1])
    chan_fwd(m, g, ws.y_op, _panel(m, g, "dec.w"), M, El, F, epi=E_BCOL, bias=p["dec.b"].data, d=ws.dec)


def backward_grid(m, ws) -> None:
    g = _gw(m, ws)
    cfg, p, ctx = m.cfg, m.params, m.ctx
    B = ws.B
    E, H, F = cfg.d_emb, cfg.d_ch, cfg.patch_features
    Tl, El, Er, Kl, Hl, Fl = ws.Tl, ws.El, ws.Er, ws.Kl, ws.Hl, ws.Fl
    M = B * Tl
    od = m.op_dtype
    K.zero(ws.bstats)
    gf = ws.g
    # decoder: g = gd Wdec, its operand copy pushed to the row group for ch2's backward
    hg = g.row.dest((M, El), od, slot="g")
    hd = getattr(ws, "gd_row", None)  # the loss kernel already pushed gd to the row group
    gd, gdrow, gsrc = (None, hd.planes, hd.own) if hd is not None else (ws.gd, None, ws.gd)
    chan_bwd(m, g, gd, ws.y_op, _panel(m, g, "dec.w"), M, El, F, "dec.w", "dec.b", gsrc, dX=gf, dyrow=gdrow,
             epi=E_CP, d2=hg.own, d2_bcast=hg.peers)
    g.row.publish(hg)
    nj = ws.r * cfg.n_blocks
    for j in reversed(range(nj)):
        b = f"block{j % cfg.n_blocks}."
        # ch2: gc = (g Wc2) * gelu'(c), pushed to the row group for ch1's backward
        hc = g.row.dest((M, Hl), od, slot="gc")
        chan_bwd(m, g, None, ws.ca[j], _panel(m, g, b + "ch2.w"), M, Hl, E, b + "ch2.w", b + "ch2.b",
                 gf if j == nj - 1 else None,
                 dX=hc.own, dyrow=hg.planes, epi=E_GB, pre=ws.c[j], d_bcast=hc.peers)
        g.row.publish(hc)
        # (dX epilogue: this rank's partial LN2-backward row moments of gv, all-reduced in _ln_bwd)
        chan_bwd(m, g, None, ws.v[j], _panel(m, g, b + "ch1.w"), M, El, H, b + "ch1.w", b + "ch1.b", hc.own,
                 dX=ws.gv, dyrow=hc.planes, epi=_lib.EPI_LNB, stats=ws.bst2[j],
                 lnb=(ws.x2[j], p[b + "ln2.gamma"].data, ws.mr2[j]))
        hx = g.row.dest((M, El), od, slot="gx2")                # g_x2 operand copy -> row group
        # (same pass: tok2's row-bias gradient partial = row sums of this rank's g_x2 columns)
        m._ln_bwd(ws.x2[j], ws.gv, b + "ln2.", ws.mr2[j], ws.bst2[j], gf, ws.gx2, hx.own, M, El, E,
                  row_reduce=lambda t: row_reduce(m, g, t), bcast=hx.peers, moments=False,
                  sums=dict(rowsum=p[b + "tok2.b"].grad, rowsum_period=Tl))
        g.row.publish(hx)
        xall = hx.planes.view(m.C, B, Tl, El)
        if _pm_path(m, g, ws):
            av = _pm_view(g.col.persistent(f"a_col{j}") if m.R > 1 else ws.a[j], m.C, B, El, Kl)
            ghv = tok2_bwd_pm(m, g, ws, j, b, xall, av)
            tok1_bwd_pm(m, g, ws, j, b, g.row.persistent(f"u_row{j}").view(m.C, B, Tl, El), ghv)
        else:
            acol_all = g.col.persistent(f"a_col{j}").view(B, -1, Kl) if m.R > 1 else None
            acols = [acol_all[bi] if m.R > 1 else ws.a[j][bi] for bi in range(B)]
            ghs = tok2_bwd_all(m, g, ws, j, b, xall, acols)
            for gh_local, _ in ghs:
                K.colsum(gh_local, p[b + "tok1.b"].grad, Er, Kl)
            tok1_bwd_all(m, g, ws, j, b, [ghcol for _, ghcol in ghs])
        hg = g.row.dest((M, El), od, slot="g")                  # g operand copy -> row group
        # (same pass: column sums of g = the bias gradient of the previous block's ch2 / the encoder)
        nxt = f"block{(j - 1) % cfg.n_blocks}.ch2.b" if j > 0 else "enc.b"
        m._ln_bwd(ws.res[j], ws.gu, b + "ln1.", ws.mr1[j], ws.bst1[j], ws.gx2, gf, hg.own, M, El, E,
                  row_reduce=lambda t: row_reduce(m, g, t), bcast=hg.peers, sums=dict(colsum=p[nxt].grad))
        g.row.publish(hg)
    chan_bwd(m, g, None, ws.xp, _panel(m, g, "enc.w"), M, Fl, E, "enc.w", "enc.b", None, dyrow=hg.planes)


def grad_sync(m) -> None:
    """Sum duplicated-vector gradients over their sharing group: column vectors over the column
    group, the tok2 row bias over the row group (model.py:451-460) — one all-reduce per range."""
    f, ctx = m.flat, m.ctx
    for cls in f.CLASSES:
        lo, hi = f.kind_range[(cls, "vec_col")]
        if hi > lo and m.R > 1:
            ctx.all_reduce_col(f.grad[lo:hi])
        lo, hi = f.kind_range[(cls, "vec_row")]
        if hi > lo and m.C > 1:
            ctx.all_reduce_row(f.grad[lo:hi])


# --------------------------------------------------------------------------- comm roofline
def step_exchange_bytes(m, batch: int, r: int = 1, op_bytes: int | None = None, part_bytes: int | None = None) -> dict:
    """Bytes ONE rank sends to its peers over NVLink in one training step of this schedule
    (forward_grid, the loss's decoder-gradient push, backward_grid, grad_sync, the weight-panel
    gathers / Adam pushes) — the balanced-grid counterpart of the reference's analytic tables
    (parallel.py:361-466, model.py:483-529), in bytes rather than elements because the operands
    (bf16) and partials (bf16 or fp32) have different widths. Every rank of the grid sends the
    same amount. Returns {"exchange": gathers + reduce-scatters (transport payload),
    "allreduce": the small NCCL all-reduces (ring: 2 (G-1)/G of the buffer), "total"}.
    Checked against the transports' own byte counters in tests/test_jigsaw_cpu.py."""
    cfg = m.cfg
    R, C = m.R, m.C
    if m.ctx.n == 1:
        return {"exchange": 0, "allreduce": 0, "total": 0}
    sop = op_bytes if op_bytes is not None else torch.empty((), dtype=m.op_dtype).element_size()
    if part_bytes is None:
        bf = m.op_dtype == torch.bfloat16 and os.environ.get("JIGSAW_PARTIALS", "bf16") != "fp32"
        part_bytes = 2 if bf else 4
    sp = part_bytes
    E, H, F, Kd, T = cfg.d_emb, cfg.d_ch, cfg.patch_features, cfg.d_tok, cfg.tokens
    Tl, El, Er, Kl, Hl, Fl = T // R, E // C, E // R, Kd // C, H // C, F // C
    B, nj = batch, r * cfg.n_blocks
    M = B * Tl
    ex = 0
    # weight panels of the channel layers, gathered (or Adam-pushed) over the column group
    if R > 1:
        ex += (R - 1) * (E * Fl + F * El + cfg.n_blocks * (H * El + E * Hl)) // R * sop
    rs_row = lambda cols: (C - 1) * M * cols * sp  # noqa: E731  channel-layer / token RS over the row group
    push_row = lambda cols: (C - 1) * M * cols * sop  # noqa: E731
    # forward: enc, dec, and per pass ch1 / ch2 reduce-scatters; LN1 output pushes; token layers
    ex += rs_row(E // C) + rs_row(F // C)
    ex += nj * (rs_row(H // C) + rs_row(E // C) + push_row(El))
    ex += nj * B * ((R - 1) * Er * Kl * (sp + sop) + (C - 1) * Tl * El * sp)
    # loss: the decoder-output gradient pushed to the row group
    ex += push_row(Fl)
    # backward: dec dX copy push, per block gc / g_x2 / g pushes, token RS + gh push, dW RS (column)
    ex += push_row(El)
    ex += nj * (push_row(Hl) + push_row(El) + push_row(El))
    ex += nj * B * ((R - 1) * Er * Kl * (sp + sop) + (C - 1) * Tl * El * sp)
    if R > 1:
        dw = F * El + nj * (E * Hl + H * El) + E * Fl  # dec, per pass ch2 / ch1, enc weight-gradient planes
        ex += (R - 1) * dw // R * sp
    # small all-reduces: LN moments (fwd 2 per pass, bwd 2 per pass, [M, 2] fp32) over the row
    # group, the loss over the grid, duplicated-vector gradients over their sharing groups
    ar = 0.0
    ring = lambda G, nbytes: 2.0 * (G - 1) / G * nbytes  # noqa: E731
    gw = getattr(getattr(m, "_ws", None), "grid", None)
    if C > 1 and gw is not None and gw.peer_moments:
        ex += 4 * nj * (C - 1) * M * 2 * 4  # pushed to the row group's moment slots
    elif C > 1:
        ar += 4 * nj * ring(C, M * 2 * 4)
    ar += ring(m.ctx.n, 4)
    f = m.flat
    for cls in f.CLASSES:
        lo, hi = f.kind_range[(cls, "vec_col")]
        if hi > lo and R > 1:
            ar += ring(R, (hi - lo) * 4)
        lo, hi = f.kind_range[(cls, "vec_row")]
        if hi > lo and C > 1:
            ar += ring(C, (hi - lo) * 4)
    return {"exchange": int(ex), "allreduce": int(ar), "total": int(ex + ar)}
