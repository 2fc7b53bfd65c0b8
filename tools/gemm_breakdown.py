"""Per-launch GEMM shapes and rates of one eager training step (rank 0 prints), random inputs.

    python tools/gemm_breakdown.py                      # 1 GPU
    torchrun --nproc-per-node 4 tools/gemm_breakdown.py # Jigsaw 2x2
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import bench
from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel
from paper_2507_05753_b200 import tensor as T
from paper_2507_05753_b200.engine import TrainStep

comm = Communicator.from_env()
ctx = MpContext(comm, list(range(comm.world_size)))
cfg_kw, lat_real, vars_real, _ = bench.CONFIGS[os.environ.get("CFG", "C4")]
model = WeatherMixerModel(ctx, ModelConfig(**cfg_kw), init="fast", lat_real=lat_real, vars_real=vars_real)
step = TrainStep(model, graph=False)
bench.fill_random_inputs(step, lat_real, 1234 + ctx.pos)
shapes = []
orig = T.gemm_into


def rec(out, a, b, am, bm, m, n, k, batch=1, *args, **kw):
    if T.GEMM_TIMER is not None:
        pe = 2 if kw.get("rs") is not None else int(kw.get("d_planes") is not None)  # 2: fused reduce-scatter
        shapes.append((m, n, k, batch, bool(kw.get("reduce_batch")), am, bm, pe))
    return orig(out, a, b, am, bm, m, n, k, batch, *args, **kw)


T.gemm_into = rec
for _ in range(3):
    step.run_device()
torch.cuda.synchronize()
T.GEMM_TIMER = []
step._body()
torch.cuda.synchronize()
recs, T.GEMM_TIMER = T.GEMM_TIMER, None
if comm.rank == int(os.environ.get("PRINT_RANK", "0")):
    tot = sum(a.elapsed_time(b) for a, b, _, _ in recs)
    fl = sum(f for _, _, f, _ in recs)
    print(f"{len(recs)} GEMMs {tot:.3f} ms {fl / tot / 1e9:.0f} TFLOP/s")
    print("   m      n      k  batch rb am bm peer   ms   TFLOP/s")
    for (s, e, f, _), (m, n, k, bt, rb, am, bm, pe) in zip(recs, shapes):
        ms = s.elapsed_time(e)
        print(f"{m:6d} {n:6d} {k:6d} {bt:3d} {int(rb)} {am} {bm} {int(pe)} {ms:7.3f} {f / ms / 1e9:7.0f}")
if comm.world_size > 1:
    dist.barrier()
os._exit(0)
