"""Per-call CUDA-event breakdown of one eager training step (rank 0 prints), under torchrun or alone.
COPY_SITES=1 also lists the call sites of copy-engine copies (none in a steady-state step)."""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel
from paper_2507_05753_b200 import kernels as K, transport as TR
from paper_2507_05753_b200.engine import TrainStep

comm = Communicator.from_env()
ctx = MpContext(comm, list(range(comm.world_size)))
cfg_kw, lat_real, vars_real, _ = bench.CONFIGS[os.environ.get("CFG", "C4")]
model = WeatherMixerModel(ctx, ModelConfig(**cfg_kw), init="fast", lat_real=lat_real, vars_real=vars_real)
step = TrainStep(model, batch=int(os.environ.get("B", "1")), graph=False)
bench.fill_random_inputs(step, lat_real, 1234 + ctx.pos)
recs = collections.defaultdict(list)

def wrap(obj, name, label):
    fn = getattr(obj, name)
    def w(*a, **k):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); r = fn(*a, **k); e.record()
        recs[label].append((s, e))
        return r
    setattr(obj, name, w)

for n in ["gemm", "epilogue", "ln_apply", "ln_bwd_moments", "ln_bwd_apply", "colsum", "rowsum", "blend_loss",
          "adam", "patchify", "sum_planes", "copy_async", "axpy"]:
    wrap(K, n, n)
for cls in (TR.SymmTransport, TR.NcclTransport):
    wrap(cls, "barrier", "barrier") if hasattr(cls, "barrier") else None
import torch.distributed as dist
for n in ["all_reduce", "all_gather_into_tensor", "reduce_scatter_tensor"]:
    wrap(dist, n, "nccl." + n)
sites = collections.Counter()
if os.environ.get("COPY_SITES"):  # where the copy-engine copies of the step come from
    import traceback
    _ca = K.copy_async
    def _ca_site(*a, **k):
        st = traceback.extract_stack(limit=6)[:-1]
        sites[" <- ".join(f"{os.path.basename(f.filename)}:{f.lineno}" for f in reversed(st[-4:]))] += 1
        return _ca(*a, **k)
    K.copy_async = _ca_site
for _ in range(3):
    step._body()
torch.cuda.synchronize()
for v in recs.values():
    v.clear()
s0, s1 = torch.cuda.Event(True), torch.cuda.Event(True)
s0.record(); step._body(); s1.record(); torch.cuda.synchronize()
tot = s0.elapsed_time(s1)
if comm.rank == 0:
    print(f"eager step {tot:.2f} ms")
    rows = [(sum(a.elapsed_time(b) for a, b in v), len(v), k) for k, v in recs.items() if v]
    for ms, cnt, k in sorted(rows, reverse=True):
        print(f"  {k:28s} {cnt:4d} calls {ms:8.3f} ms {100 * ms / tot:5.1f}%")
    for site, cnt in sites.most_common(8):
        print(f"  copy_async x{cnt // 4}/step: {site}")
if comm.world_size > 1:
    dist.barrier()
os._exit(0)
