"""jg_gemm at one shape with all four operand-major combinations, interleaved (best of rounds)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2507_05753_b200 import tensor as T, _lib  # noqa: E402

_lib.load()
shapes = [(4320, 8640, 16384), (4480, 4320, 16384), (16384, 4320, 8640), (8192, 8192, 8192)]
g = torch.Generator(device="cuda").manual_seed(0)
for (m, n, k) in shapes:
    res = {}
    bufs = {}
    for am in (0, 1):
        for bm in (0, 1):
            A = torch.randn((m, k) if am == 0 else (k, m), device="cuda", generator=g).bfloat16()
            B = torch.randn((n, k) if bm == 0 else (k, n), device="cuda", generator=g).bfloat16()
            bufs[(am, bm)] = (A, B)
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for rnd in range(3):
        for (am, bm), (A, B) in bufs.items():
            for _ in range(2):
                T.gemm_into(out, A, B, am, bm, m, n, k)
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            for _ in range(5):
                T.gemm_into(out, A, B, am, bm, m, n, k)
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / 5
            res[(am, bm)] = min(res.get((am, bm), 1e9), ms)
    print(f"{m}x{n}x{k}: " + "  ".join(f"{am}{bm} {2*m*n*k/ms/1e9:.0f} TF/s" for (am, bm), ms in res.items()), flush=True)
    del bufs
    torch.cuda.empty_cache()
