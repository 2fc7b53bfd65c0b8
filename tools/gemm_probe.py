"""One jg_gemm shape launched repeatedly (for ncu --set full comparisons of operand majors):
    python tools/gemm_probe.py M N K A_MAJOR B_MAJOR [reps]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2507_05753_b200 import tensor as T, _lib  # noqa: E402

m, n, k, am, bm = (int(v) for v in sys.argv[1:6])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
_lib.load()
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn((m, k) if am == 0 else (k, m), device="cuda", generator=g).bfloat16()
B = torch.randn((n, k) if bm == 0 else (k, n), device="cuda", generator=g).bfloat16()
out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    T.gemm_into(out, A, B, am, bm, m, n, k)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(10):
    T.gemm_into(out, A, B, am, bm, m, n, k)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"{m}x{n}x{k} majors {am}{bm}: {ms:.3f} ms {2 * m * n * k / ms / 1e9:.0f} TF/s")
