"""Timing probe of the Jigsaw reduce-scatter variants on one channel-mixing layer shape (timing
only; JG_RS_DBG ablations give wrong results). Run under torchrun, n = 2 or 4 (one group of
all ranks):

    torchrun --nproc-per-node 2 tools/rs_probe.py [M N K]

  gemm      : the plane-batched GEMM storing partial planes into the owners' buffers
  gemm+bar  : + the publishing barrier
  unfused   : + jg_epilogue (sum planes, bias, residual, moments, fp32 + bf16 outputs)
  fused     : one kernel (jg_gemm rs_*)
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2507_05753_b200 import Communicator, _lib
from paper_2507_05753_b200 import kernels as K
from paper_2507_05753_b200.transport import SymmTransport

comm = Communicator.from_env()
dev = torch.device("cuda", torch.cuda.current_device())
G, idx = comm.world_size, comm.rank
M, N, Kd = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (8190, 2160, 2160)
grp = dist.new_group(list(range(G)))
st = SymmTransport(grp, G, idx, dev, G * M * N * 4, [("tmp", (G, 16), torch.bfloat16)])
torch.manual_seed(idx)
A = torch.randn(M, Kd, device=dev).bfloat16()
W = torch.randn(G * N, Kd, device=dev).bfloat16()
bias = torch.randn(N, device=dev)
resid = torch.randn(M, N, device=dev)
d = torch.empty(M, N, device=dev)
d2 = torch.empty(M, N, device=dev).bfloat16()
stats = torch.zeros(M, 2, device=dev)
E = _lib.EPI_BIAS_COL | _lib.EPI_RESID | _lib.EPI_COPY_D2 | _lib.EPI_STATS
epi = dict(epi=E, bias=bias, resid=resid, d=d, d2=d2, stats=stats)


def fn(s, D, d_bs, dpl, **kw):
    K.gemm(D, A, W, 0, 0, M, N, Kd, G, 0, N * Kd, d_bs=d_bs, d_planes=dpl, **kw)


def v_gemm():
    st.rs_gemm(M, N, torch.bfloat16, fn)


def v_unfused():
    acc, npl, ps = st.rs_gemm(M, N, torch.bfloat16, fn)
    K.epilogue(acc, M, N, acc_bs=ps, nplanes=npl, **epi)


def v_fused():
    st.rs_gemm_fused(M, N, torch.bfloat16, fn, **dict(epi))


def timed(f, n=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n):
        f()
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) / n * 1e3], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


res = [("gemm+bar", timed(v_gemm)), ("unfused", timed(v_unfused)), ("fused", timed(v_fused))]
if idx == 0:
    fl = 2 * M * N * Kd * G
    print(f"G={G} M={M} N={N} K={Kd} JG_RS_DBG={os.environ.get('JG_RS_DBG', '0')}")
    for k, us in res:
        print(f"  {k:10s} {us:8.1f} us  {fl / us / 1e6:6.0f} TFLOP/s")
dist.barrier()
os._exit(0)
