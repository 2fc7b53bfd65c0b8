import torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2507_05753_b200 import tensor as T, _lib
def ref(a, b, mode):
    a, b = a.double().cpu(), b.double().cpu()
    return a @ b if mode == "NN" else (a @ b.T if mode == "NT" else a.T @ b)
def mk(mode, m, n, k, g):
    if mode == "NN": return torch.randn(m, k, generator=g), torch.randn(k, n, generator=g)
    if mode == "NT": return torch.randn(m, k, generator=g), torch.randn(n, k, generator=g)
    return torch.randn(k, m, generator=g), torch.randn(k, n, generator=g)
g = torch.Generator().manual_seed(0)
for (m, n, k) in [(128,128,64),(64,64,128),(128,128,32),(128,128,128),(256,256,256)]:
    for mode in ["NN","NT","TN"]:
        a, b = mk(mode, m, n, k, g)
        a, b = a.cuda(), b.cuda()
        ah, al = T.split_tf32(a); bh, bl = T.split_tf32(b)
        z_a, z_b = torch.zeros_like(a), torch.zeros_like(b)
        am = _lib.JG_KMAJOR if mode != "TN" else _lib.JG_MNMAJOR
        bm = _lib.JG_MNMAJOR if mode != "NT" else _lib.JG_KMAJOR
        out = torch.empty(m, n, device='cuda')
        T.gemm_into(out, ah, bh, am, bm, m, n, k, a_lo=z_a, b_lo=z_b)
        torch.cuda.synchronize()
        r = ref(ah, bh, mode)
        d = (out.double().cpu() - r).abs()
        e1 = float(d.max() / r.abs().max())
        # which elements are wrong
        bad = (d > 1e-3 * r.abs().max()).nonzero()
        out3 = T.matmul(a, b, mode); torch.cuda.synchronize()
        r3 = ref(a, b, mode)
        e3 = float((out3.double().cpu() - r3).abs().max() / r3.abs().max())
        print(f"{m}x{n}x{k} {mode}: tf32-hi-only err {e1:.2e} nbad {len(bad)} first {bad[:3].tolist()}  | 3xtf32 err {e3:.2e}")
        # bf16 of same
        ob = T.matmul(a.bfloat16(), b.bfloat16(), mode); torch.cuda.synchronize()
        rb = ref(a.bfloat16(), b.bfloat16(), mode)
        print("    bf16 err", float((ob.double().cpu()-rb).abs().max()/rb.abs().max()))
