"""Jigsaw-shaped GEMMs (2x2 and 4x2 channel / token layers) with local outputs vs one output
plane stored into a peer GPU over NVLink (the reduce-scatter epilogue). torchrun, 2 ranks.

    torchrun --nproc-per-node 2 tools/gemm_shape_probe.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2507_05753_b200 import Communicator
from paper_2507_05753_b200 import kernels as K
from paper_2507_05753_b200.transport import SymmTransport

comm = Communicator.from_env()
dev = torch.device("cuda", torch.cuda.current_device())
G, idx = comm.world_size, comm.rank
grp = dist.new_group(list(range(G)))
CASES = [  # name, M, N, K (per plane; 2 planes)
    ("2x2 chan K=2160", 8190, 2160, 2160), ("2x2 chan K=4320", 8190, 2160, 4320),
    ("4x2 chan K=2160", 4095, 2160, 2160), ("4x2 chan K=2240", 4095, 2240, 2160),
    ("1x2 chan K=2160", 16380, 2160, 2160),
]
mx = max(M * N for _, M, N, _ in CASES)
st = SymmTransport(grp, G, idx, dev, 2 * mx * 2, [("tmp", (G, 16), torch.bfloat16)])


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


for name, M, N, Kd in CASES:
    A = torch.randn(M, Kd, device=dev).bfloat16()
    W = torch.randn(2 * N, Kd, device=dev).bfloat16()
    D = torch.empty(2, M, N, device=dev).bfloat16()
    off = st.scratch_off
    pbytes = M * N * 2
    local = lambda: K.gemm(D, A, W, 0, 0, M, N, Kd, 2, 0, N * Kd)  # noqa: E731
    peer = 1 - idx
    planes = [st.base[idx] + off, st.base[peer] + off + pbytes]  # plane 0 own, plane 1 -> peer
    remote = lambda: K.gemm(D[0], A, W, 0, 0, M, N, Kd, 2, 0, N * Kd, d_bs=0, d_planes=planes)  # noqa: E731
    tl, tr = timeit(local), timeit(remote)
    fl = 2 * M * N * Kd * 2
    if idx == 0:
        print(f"{name:18s} M={M:5d} N={N} K={Kd}: local {tl:7.1f} us {fl / tl / 1e6:6.0f} TF/s | "
              f"1 of 2 planes to peer {tr:7.1f} us {fl / tr / 1e6:6.0f} TF/s", flush=True)
dist.barrier()
os._exit(0)
