"""Where does the public call's time go? Host-side cost of each part of TrainStep.__call__ and
the device time of the call vs the back-to-back graph replays (rank 0 prints).

    torchrun --nproc-per-node 4 tools/launch_probe.py
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import bench
from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel
from paper_2507_05753_b200.engine import TrainStep

comm = Communicator.from_env()
ctx = MpContext(comm, list(range(comm.world_size)))
cfg_kw, lat_real, vars_real, _ = bench.CONFIGS[os.environ.get("CFG", "C4")]
model = WeatherMixerModel(ctx, ModelConfig(**cfg_kw), init="fast", lat_real=lat_real, vars_real=vars_real)
step = TrainStep(model)
xd, td = bench.fill_random_inputs(step, lat_real, 1234 + ctx.pos)
for _ in range(3):
    step.run_device()
torch.cuda.synchronize()
xh, th = xd.cpu().pin_memory(), td.cpu().pin_memory()
step.warm_prefetch()
step(xh, th)
cur = torch.cuda.current_stream()
res = {}


def timed_host(label, fn, n=5):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        if comm.world_size > 1:
            dist.barrier()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
    res[label] = 1e3 * sorted(ts)[len(ts) // 2]


timed_host("graph0 replay (host ms)", lambda: step.graph[0].replay())
timed_host("graph1 replay (host ms)", lambda: step.graph[1].replay())
timed_host("run_device (host ms)", lambda: step.run_device())
timed_host("call, no prefetch (wall ms)", lambda: step(xh, th))


def dev(fn, n=5):
    torch.cuda.synchronize()
    if comm.world_size > 1:
        dist.barrier()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(cur)
    for _ in range(n):
        fn()
    b.record(cur)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


res["run_device back-to-back (device ms)"] = dev(lambda: step.run_device())
res["run_device + sync each (device ms)"] = dev(lambda: (step.run_device(), torch.cuda.synchronize()))
res["call, no prefetch (device ms)"] = dev(lambda: step(xh, th))
if comm.rank == 0:
    for k, v in res.items():
        print(f"{k:40s} {v:8.3f}", flush=True)
if comm.world_size > 1:
    dist.barrier()
os._exit(0)
