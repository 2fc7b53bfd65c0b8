"""Compare SymmTransport with NcclTransport on random data (run under torchrun, n = 2 or 4)."""
import os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2507_05753_b200 import Communicator, MpContext, _lib
from paper_2507_05753_b200 import kernels as K
from paper_2507_05753_b200.transport import NcclTransport, SymmTransport

comm = Communicator.from_env()
ctx = MpContext(comm, list(range(comm.world_size)))
dev = torch.device("cuda", torch.cuda.current_device())
rank = comm.rank
torch.manual_seed(rank)
res = []
for axis in ("row", "col"):
    G = ctx.C if axis == "row" else ctx.R
    if G == 1:
        continue
    grp = ctx.row_group if axis == "row" else ctx.col_group
    idx = ctx.c if axis == "row" else ctx.r
    st = SymmTransport(grp, G, idx, dev, 64 << 20, [("keep", (3, G, 128, 64), torch.bfloat16),
                                                    ("tmp", (G, 128, 64), torch.bfloat16)])
    nt = NcclTransport(grp, G, idx, dev)
    x = torch.randn(128, 64, device=dev).bfloat16()
    a = st.ag(x)
    b = nt.ag(x)
    res.append((axis, "ag", (a.float() - b.float()).abs().max().item()))
    a2 = st.ag(x * 2, slot="keep", sub=1, nsub=3)
    res.append((axis, "ag_slot", (a2.float() - 2 * b.float()).abs().max().item()))
    # rs_gemm: partial P[G*64, 48] = A[G*64, 96] B[48, 96]^T, planes over output rows
    A = torch.randn(G * 64, 96, device=dev).bfloat16()
    Bm = torch.randn(48, 96, device=dev).bfloat16()

    def fn(s, D, d_bs, dpl):
        K.gemm(D, A, Bm, 0, 0, 64, 48, 96, G, 64 * 96, 0, d_bs=d_bs, d_planes=dpl)

    sa, sn, sp = st.rs_gemm(64, 48, torch.float32, fn)
    ssum = sum(sa.reshape(-1)[i * sp:(i + 1) * sp] for i in range(sn)).view(64, 48) if sn > 1 else sa
    na, nn, np_ = nt.rs_gemm(64, 48, torch.float32, fn)
    # (G > 2: NCCL's ring adds the members' partials in another order than the peer-memory
    # epilogue's member order, so equality is to fp32 rounding, not bitwise)
    tol = 0.0 if G <= 2 else 1e-6
    res.append((axis, "rs", (ssum - na).abs().max().item(), na.abs().max().item(), tol))
    # q-sub-chunked reduce-scatter (R > C grids: G / q gathered planes, each split into q owner
    # chunks): batch j of sub-GEMM s goes to owner j*q + s
    for q in sorted({v for v in (2, G) if G % v == 0 and v > 1}):
        Aq = torch.randn((G // q) * 32 * q, 96, device=dev).bfloat16()

        def fnq(s, D, d_bs, dpl, q=q, Aq=Aq):
            K.gemm(D, Aq[s * 32:], Bm, 0, 0, 32, 48, 96, G // q, q * 32 * 96, 0, d_bs=d_bs, d_planes=dpl)

        sa, sn, sp = st.rs_gemm(32, 48, torch.float32, fnq, q=q)
        ssum = sum(sa.reshape(-1)[i * sp:(i + 1) * sp] for i in range(sn)).view(32, 48) if sn > 1 else sa
        na, nn, np_ = nt.rs_gemm(32, 48, torch.float32, fnq, q=q)
        res.append((axis, f"rs_q{q}", (ssum - na).abs().max().item(), na.abs().max().item(), tol))
    # GEMM + reduce-scatter + epilogue in one kernel (rs_gemm_fused) == GEMM -> barrier -> jg_epilogue,
    # bit for bit: multi-tile 2-CTA shapes, fp32 and bf16 partials, plain sum and bias + GELU epilogue
    rows, cols, kk = 512, 384, 256
    A2 = torch.randn(G * rows, kk, device=dev).bfloat16()
    B2 = torch.randn(cols, kk, device=dev).bfloat16()
    bias = torch.randn(cols, device=dev)

    def fn2(s, D, d_bs, dpl, **kw):
        K.gemm(D, A2, B2, 0, 0, rows, cols, kk, G, rows * kk, 0, d_bs=d_bs, d_planes=dpl, **kw)

    for pdt in (torch.float32, torch.bfloat16):
        for epi in (0, _lib.EPI_BIAS_COL | _lib.EPI_GELU_FWD):
            kw = dict(epi=epi, bias=bias) if epi else {}
            ref_d, ref_d2 = torch.empty(rows, cols, device=dev), torch.empty(rows, cols, device=dev).bfloat16()
            sa, sn, sp = st.rs_gemm(rows, cols, pdt, fn2)
            K.epilogue(sa, rows, cols, acc_bs=sp, nplanes=sn, d=ref_d, d2=ref_d2 if epi else None, **kw)
            for rep in range(3):  # repeated calls exercise both regions and the flag re-arming
                got_d, got_d2 = torch.zeros(rows, cols, device=dev), torch.zeros(rows, cols, device=dev).bfloat16()
                st.rs_gemm_fused(rows, cols, pdt, fn2, d=got_d, d2=got_d2 if epi else None, **kw)
                err = (got_d - ref_d).abs().max().item()
                if epi:
                    err = max(err, (got_d2.float() - ref_d2.float()).abs().max().item())
                res.append((axis, f"rs_fused_{str(pdt)[6:]}_{epi}_{rep}", err, ref_d.abs().max().item()))
    torch.cuda.synchronize()
print(rank, res, flush=True)
bad = [r for r in res if r[2] > (r[4] * max(1.0, r[3]) if len(r) > 4 else 0.0)]
if rank == 0:
    print("TRANSPORT_OK" if not bad else f"TRANSPORT_BAD {bad}", flush=True)
dist.barrier()
os._exit(0)
