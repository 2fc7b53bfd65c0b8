"""Per-kernel cost of dependent launches inside a CUDA graph: 200 back-to-back tiny kernels
(jg_memset of 256 B) and 200 layer-norm applies of a 2x2-rank tile, captured and replayed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_05753_b200 import _lib, kernels as K

_lib.load()
dev = torch.device("cuda")
buf = torch.zeros(64, device=dev)
M, E = 8190, 2160
x = torch.randn(M, E, device=dev)
st = torch.zeros(M, 2, device=dev)
st[:, 1] = E
gam, bet = torch.ones(E, device=dev), torch.zeros(E, device=dev)
y = torch.empty(M, E, device=dev, dtype=torch.bfloat16)
mr = torch.empty(M, 2, device=dev)


def tiny():
    for _ in range(200):
        K.zero(buf)


def lnap():
    for _ in range(200):
        K.ln_apply(x, st, gam, bet, y, mr, M, E, E, 1e-5)


for name, fn in (("memset 256 B", tiny), ("ln_apply 8190x2160", lnap)):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) / 5 / 200 * 1e3:.2f} us per kernel in a graph", flush=True)
