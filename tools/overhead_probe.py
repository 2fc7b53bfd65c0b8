"""Upper bounds on the exchange overheads of the captured Jigsaw step (timing only — results
of the ablated variants are WRONG): each variant disables one class of operations before the
CUDA graph is captured and reports the graph step time (CUDA events, max over ranks).

    torchrun --nproc-per-node 4 tools/overhead_probe.py [variant ...]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import bench
from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel
from paper_2507_05753_b200 import kernels as K, transport as TR
from paper_2507_05753_b200.engine import TrainStep

comm = Communicator.from_env()
ctx = MpContext(comm, list(range(comm.world_size)))
cfg_kw, lat_real, vars_real, _ = bench.CONFIGS[os.environ.get("CFG", "C4")]
model = WeatherMixerModel(ctx, ModelConfig(**cfg_kw), init="fast", lat_real=lat_real, vars_real=vars_real)
noop = lambda *a, **k: None  # noqa: E731
from paper_2507_05753_b200 import jigsaw_grid as JG
orig = {"barrier": TR.SymmTransport.barrier, "ar_row": MpContext.all_reduce_row, "ar_col": MpContext.all_reduce_col,
        "copy": K.copy_async, "epilogue": K.epilogue, "moments": JG.row_reduce}


def restore():
    TR.SymmTransport.barrier = orig["barrier"]
    MpContext.all_reduce_row, MpContext.all_reduce_col = orig["ar_row"], orig["ar_col"]
    K.copy_async, K.epilogue = orig["copy"], orig["epilogue"]
    JG.row_reduce = orig["moments"]


def apply(v):
    if v in ("nobarrier", "nocomm"):
        TR.SymmTransport.barrier = noop
    if v in ("noar", "nocomm"):
        MpContext.all_reduce_row = MpContext.all_reduce_col = noop
    if v in ("nocopy", "nocomm"):
        K.copy_async = noop
    if v == "noepilogue":
        K.epilogue = noop
    if v in ("nomoments", "nocomm"):
        JG.row_reduce = noop


def timed(step, n=10):
    for _ in range(3):
        step.run_device()
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n):
        step.run_device()
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) / n], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


variants = sys.argv[1:] or ["base", "nobarrier", "noar", "nomoments", "nocopy", "noepilogue", "nocomm"]
for v in variants:
    apply(v)
    step = TrainStep(model, batch=int(os.environ.get("B", "1")))
    bench.fill_random_inputs(step, lat_real, 1234 + ctx.pos)
    step.capture()
    restore()
    ms = timed(step)
    if comm.rank == 0:
        print(f"{v:12s} {ms:8.3f} ms/step", flush=True)
    del step
    torch.cuda.synchronize()
dist.barrier()
os._exit(0)
