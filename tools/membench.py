"""HBM roofline of the memory-bound kernels at C4 shapes (1 GPU, random data, inputs >> L2).

Each kernel is launched `reps` times back to back between CUDA events on the launching
stream; achieved GB/s = algorithmic bytes per launch / mean launch time (bytes as DESIGN.md §4
counts them). Prints a JSON line per kernel and a markdown table.

    python tools/membench.py [--tile 1x1|2x2] [--reps 20]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_05753_b200 import kernels as K, _lib

ap = argparse.ArgumentParser()
ap.add_argument("--tile", default="1x1")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--only", default="")
args = ap.parse_args()
R, C = map(int, args.tile.split("x"))
dev = torch.device("cuda")
f32, bf = torch.float32, torch.bfloat16
LAT, LON, NV, PL, PW = 728, 1440, 70, 8, 8
E, KT, H = 4320, 8640, 4320
T = (LAT // PL) * (LON // PW)
Tl, El, Kl, Er = T // R, E // C, KT // C, E // R
lon_l, nv_l = LON // R, NV // C
Fl = nv_l * PL * PW
M = Tl
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))) \
    if os.path.exists("MEASURED_PEAKS.json") else {}


def rnd(*shape, dtype=f32):
    return torch.randn(*shape, device=dev, dtype=f32).to(dtype)


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


rows = []


def run(name, fn, nbytes):
    if args.only and args.only not in name:
        return
    ms = timeit(fn, args.reps)
    gbs = nbytes / ms / 1e6
    rows.append((name, ms, nbytes, gbs))
    print(json.dumps({"kernel": name, "ms": round(ms, 4), "bytes": nbytes, "GB/s": round(gbs, 1)}), flush=True)


# patchify: fp32 grid -> bf16 tokens
x = rnd(1, LAT, lon_l, nv_l)
tok = torch.empty(1, Tl, Fl, device=dev, dtype=bf)
run("patchify", lambda: K.patchify(x, tok, 1, LAT, lon_l, nv_l, PL, PW), x.numel() * 6)

# blend + loss + dL/d(dec tokens) (bf16 operand), training form
dec = rnd(1, Tl, Fl)
tgt = rnd(1, LAT, lon_l, nv_l)
bw = torch.rand(nv_l, device=dev)
latw = torch.rand(LAT, device=dev)
varw = torch.rand(nv_l, device=dev)
loss = torch.zeros(1, device=dev)
gblend = torch.zeros(nv_l, device=dev)
gd = torch.empty(1, Tl, Fl, device=dev, dtype=bf)
run("blend_loss", lambda: K.blend_loss(dec, x, tgt, bw, latw, varw, None, None, loss, gblend, gd, 1, LAT, lon_l, nv_l,
                                        PL, PW, 1.0 / x.numel(), 1.0), x.numel() * (4 + 4 + 4 + 2))

# layer norm apply: fp32 in, bf16 out (+ mean/rstd)
res = rnd(M, El)
st = torch.stack([res.sum(1), (res * res).sum(1)], 1).contiguous()
gam, bet = rnd(El), rnd(El)
u = torch.empty(M, El, device=dev, dtype=bf)
mr = torch.empty(M, 2, device=dev)
run("ln_apply", lambda: K.ln_apply(res, st, gam, bet, u, mr, M, El, E, 1e-5), M * El * 6)

gin = rnd(M, El)
bst = torch.zeros(M, 2, device=dev)
run("ln_bwd_moments", lambda: K.ln_bwd_moments(res, gin, gam, mr, bst, M, El), M * El * 8)
out = torch.empty(M, El, device=dev)
out_op = torch.empty(M, El, device=dev, dtype=bf)
resid = rnd(M, El)
dg, db = torch.zeros(El, device=dev), torch.zeros(El, device=dev)
run("ln_bwd_apply", lambda: K.ln_bwd_apply(res, gin, gam, mr, bst, resid, out, out_op, dg, db, M, El, E),
    M * El * (4 + 4 + 4 + 4 + 2))
rsb, csb = torch.zeros(Tl, device=dev), torch.zeros(El, device=dev)
run("ln_bwd_apply_rowsum", lambda: K.ln_bwd_apply(res, gin, gam, mr, bst, resid, out, out_op, dg, db, M, El, E,
                                                  rowsum=rsb, rowsum_period=Tl), M * El * (4 + 4 + 4 + 4 + 2))
run("ln_bwd_apply_colsum", lambda: K.ln_bwd_apply(res, gin, gam, mr, bst, resid, out, out_op, dg, db, M, El, E,
                                                  colsum=csb), M * El * (4 + 4 + 4 + 4 + 2))

# bias gradients
gc = rnd(M, H // C, dtype=bf)
ob = torch.zeros(H // C, device=dev)
run("colsum_bf16", lambda: K.colsum(gc, ob, M, H // C), gc.numel() * 2)
g32 = rnd(M, El)
run("colsum_f32", lambda: K.colsum(g32, torch.zeros(El, device=dev), M, El), g32.numel() * 4)
orow = torch.zeros(M, device=dev)
run("rowsum_f32", lambda: K.rowsum(g32, orow, M, El), g32.numel() * 4)

# Jigsaw epilogue (tok2 form): sum 2 bf16 planes + row bias + residual -> x2 fp32, LN moments
if R * C > 1:
    G = C
    planes = rnd(G, M, El, dtype=bf)
    bias = rnd(M)
    x2 = torch.empty(M, El, device=dev)
    stt = torch.zeros(M, 2, device=dev)
    run("epilogue_tok2", lambda: K.epilogue(planes, M, El, acc_bs=M * El, nplanes=G,
                                             epi=_lib.EPI_BIAS_ROW | _lib.EPI_RESID | _lib.EPI_STATS, bias=bias,
                                             resid=resid, d=x2, stats=stt), M * El * (2 * G + 4 + 4))
    hp = rnd(R, Er, Kl, dtype=bf)
    h = torch.empty(Er, Kl, device=dev)
    a = torch.empty(Er, Kl, device=dev, dtype=bf)
    b1 = rnd(Kl)
    run("epilogue_tok1", lambda: K.epilogue(hp, Er, Kl, acc_bs=Er * Kl, nplanes=R,
                                             epi=_lib.EPI_BIAS_COL | _lib.EPI_GELU_FWD, bias=b1, d=h, d2=a),
        Er * Kl * (2 * R + 4 + 2))
    # channel layers: ch1 (col bias + GELU: bf16 pre-activation and activation), ch2 (col bias +
    # residual + next LN moments, fp32 out)
    Hl = H // C
    cp = rnd(G, M, Hl, dtype=bf)
    cpre = torch.empty(M, Hl, device=dev, dtype=bf)
    cact = torch.empty(M, Hl, device=dev, dtype=bf)
    bh = rnd(Hl)
    run("epilogue_ch1", lambda: K.epilogue(cp, M, Hl, acc_bs=M * Hl, nplanes=G, epi=_lib.EPI_BIAS_COL | _lib.EPI_GELU_FWD,
                                            bias=bh, d=cpre, d2=cact), M * Hl * (2 * G + 2 + 2))
    # backward GELU' epilogue (ch2 dX form): sum of planes * gelu'(pre) -> bf16 gradient
    gco = torch.empty(M, Hl, device=dev, dtype=bf)
    run("epilogue_gb", lambda: K.epilogue(cp, M, Hl, acc_bs=M * Hl, nplanes=G, epi=_lib.EPI_GELU_BWD, pre=cpre, d=gco),
        M * Hl * (2 * G + 2 + 2))
    yo = torch.empty(M, El, device=dev)
    be = rnd(El)
    run("epilogue_ch2", lambda: K.epilogue(planes, M, El, acc_bs=M * El, nplanes=G,
                                            epi=_lib.EPI_BIAS_COL | _lib.EPI_RESID | _lib.EPI_STATS, bias=be,
                                            resid=resid, d=yo, stats=stt), M * El * (2 * G + 4 + 4))
    red = torch.empty(M * El, device=dev)
    run("sum_planes", lambda: K.sum_planes(red, planes, M * El, G, M * El), M * El * (2 * G + 4))

# Adam over the 1-GPU parameter count / n (fp32 p, g, m, v; bf16 copy)
n = 1_000_000_000 // (R * C)
p, g, m, v = (torch.randn(n, device=dev) for _ in range(4))
v.abs_()
pb = torch.empty(n, device=dev, dtype=bf)
step = torch.ones(1, device=dev, dtype=torch.int32)
run("adam", lambda: K.adam(p, g, m, v, pb, n, 1e-4, 0.9, 0.999, 1e-8, step), n * 30)

hbm = peak.get("hbm_gbs") or peak.get("hbm_copy_gbs")
print(f"\n| kernel ({args.tile}) | ms | MB | GB/s | frac of {hbm} GB/s |\n|---|---|---|---|---|")
for name, ms, nb, gbs in rows:
    frac = f"{gbs / hbm:.2f}" if hbm else "-"
    print(f"| {name} | {ms:.4f} | {nb / 1e6:.1f} | {gbs:.0f} | {frac} |")
