"""Micro-benchmark of jg_gemm (bf16) on the C4 mixing-GEMM shapes vs torch.matmul (cuBLAS)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2507_05753_b200 import tensor as T, _lib
T_, E, F, DT, DC = 16380, 4320, 4480, 8640, 4320
cases = [  # name, m, n, k, a_major, b_major
    ("ch1_fwd NT", T_, DC, E, 0, 0),
    ("tok1_fwd TN", E, DT, T_, 1, 1),
    ("tok2_fwd NT", T_, E, DT, 0, 0),
    ("ch_dX NN", T_, E, DC, 0, 1),
    ("ch_dW TN", DC, E, T_, 1, 1),
    ("sq8192 NT", 8192, 8192, 8192, 0, 0),
]
def timeit(fn, it=10):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it
for name, m, n, k, am, bm in cases:
    a = torch.randn((m, k) if am == 0 else (k, m), device='cuda').bfloat16()
    b = torch.randn((n, k) if bm == 0 else (k, n), device='cuda').bfloat16()
    out = torch.empty(m, n, device='cuda', dtype=torch.bfloat16)
    ms = timeit(lambda: T.gemm_into(out, a, b, am, bm, m, n, k))
    at = a if am == 0 else a.t()
    bt = b.t() if bm == 0 else b
    ms_t = timeit(lambda: torch.matmul(at, bt))
    ref = torch.matmul(at.float(), bt.float())
    err = ((out.float() - ref).abs().max() / ref.abs().max()).item()
    fl = 2.0 * m * n * k
    print(f"{name:12s} {m}x{n}x{k}: jg {ms:.3f} ms {fl/ms/1e9:.0f} TF/s | cuBLAS {ms_t:.3f} ms {fl/ms_t/1e9:.0f} TF/s | err {err:.1e}", flush=True)
