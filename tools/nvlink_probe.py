"""NVLink evidence for the fused GEMM + reduce-scatter store (single process, two GPUs, so it may
run under ncu — multi-rank commands may not): a Jigsaw channel-layer GEMM on GPU 0 whose output
planes go to their owners — plane 0 local, plane 1 into GPU 1's memory through the epilogue's TMA
bulk stores over NVLink (peer access) — against the same GEMM with both planes local.

    python tools/nvlink_probe.py [--reps 20]           # timing + bytes
    ncu --metrics <nvlink metrics> -k regex:gemm_kernel python tools/nvlink_probe.py --reps 2

Shape: the 2x2 C4 channel layer per rank: M = 8190 rows (B T / R), 2 planes of 2160 columns
(E / C), K = 2160 (E / C), bf16 operands, bf16 partial planes (as the bench runs them).
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_05753_b200 import _lib, tensor as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--m", type=int, default=8190)
ap.add_argument("--n", type=int, default=2160)
ap.add_argument("--k", type=int, default=2160)
a = ap.parse_args()
assert torch.cuda.device_count() >= 2, "needs two GPUs in one process"
from cuda import cudart  # noqa: E402

torch.cuda.set_device(0)
_lib.load()
err, = cudart.cudaDeviceEnablePeerAccess(1, 0)
assert err in (cudart.cudaError_t.cudaSuccess, cudart.cudaError_t.cudaErrorPeerAccessAlreadyEnabled), err
torch.cuda.set_device(1)
err, = cudart.cudaDeviceEnablePeerAccess(0, 0)
torch.cuda.set_device(0)
m, n, k = a.m, a.n, a.k
g = torch.Generator(device="cuda:0").manual_seed(0)
X = torch.randn(m, k, device="cuda:0", generator=g).bfloat16()
W = torch.randn(2 * n, k, device="cuda:0", generator=g).bfloat16()  # the gathered weight panel [N, K]
local = torch.empty(2, m, n, device="cuda:0", dtype=torch.bfloat16)
remote = torch.empty(m, n, device="cuda:1", dtype=torch.bfloat16)


def gemm(planes):
    # batch b = output plane b: X W[b-th n chunk]^T, stored at planes[b]
    T.gemm_into(local[0], X, W, 0, 0, m, n, k, 2, 0, n * k, d_bs=m * n, d_planes=planes)


both_local = [local[0].data_ptr(), local[1].data_ptr()]
one_remote = [local[0].data_ptr(), remote.data_ptr()]
for planes in (both_local, one_remote):
    gemm(planes)
torch.cuda.synchronize()
# the remote plane equals the local computation
gemm(both_local)
gemm(one_remote)
torch.cuda.synchronize()
same = torch.equal(remote.to("cuda:0"), local[1])
res = {}
for name, planes in (("local", both_local), ("remote", one_remote), ("local2", both_local), ("remote2", one_remote)):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(a.reps):
        gemm(planes)
    e.record()
    torch.cuda.synchronize()
    res[name] = s.elapsed_time(e) / a.reps
fl = 2.0 * m * 2 * n * k
nb = m * n * 2
for name in ("local", "remote"):
    ms = min(res[name], res[name + "2"])
    extra = f", NVLink {nb / ms / 1e6:.0f} GB/s average over the kernel for the peer plane ({nb / 1e6:.1f} MB)" \
        if name == "remote" else ""
    print(f"{name:7s} {ms * 1e3:8.1f} us  {fl / ms / 1e9:6.0f} TFLOP/s{extra}")
print(f"remote plane bit-identical to the local computation: {same}")
