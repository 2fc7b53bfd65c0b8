"""Where the end-to-end call loses time against the device-resident step (C4, bench inputs):
    graph      run_device() back to back (the bench `value` loop)
    graph+sync run_device() + loss read each step (host turnaround)
    call       TrainStep.__call__ with pinned host inputs and the next step's prefetch (bench e2e)
    call_d2d   the same with device-resident "host" tensors (copy engines without PCIe)
    push+graph the call's two staging pushes (SM copies) + graph + loss read, no copies
    h2d||graph the prefetch's host->device copies beside graph + loss read, no pushes
    d2d||graph the same with device-resident sources
Prints ms per step, max over ranks (rank 0).

    torchrun --nproc-per-node 4 tools/e2e_probe.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import bench
from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel
from paper_2507_05753_b200 import kernels as K
from paper_2507_05753_b200.engine import TrainStep

comm = Communicator.from_env()
ctx = MpContext(comm, list(range(comm.world_size)))
cfg_kw, lat_real, vars_real, _ = bench.CONFIGS[os.environ.get("CFG", "C4")]
model = WeatherMixerModel(ctx, ModelConfig(**cfg_kw), init="fast", lat_real=lat_real, vars_real=vars_real)
step = TrainStep(model, batch=1)
bench.fill_random_inputs(step, lat_real, 1234 + ctx.pos)
xd, td = step.ws.xin.clone(), step.target.clone()
xh, th = xd.cpu().pin_memory(), td.cpu().pin_memory()
N = int(os.environ.get("STEPS", "10"))
stream = torch.cuda.current_stream()


def timed(body):
    torch.cuda.synchronize()
    if comm.world_size > 1:
        dist.barrier()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(stream)
    body()
    b.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / N], device="cuda")
    if comm.world_size > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def graph():
    for _ in range(N):
        step.run_device()


def graph_sync():
    for _ in range(N):
        step.run_device()
        step.ws.loss.item()


def call(xs, ts):
    def body():
        step.prefetch(xs, ts)
        for i in range(N):
            step(xs, ts, prefetch_next=(xs, ts) if i + 1 < N else None)
    return body


def push_graph():
    for _ in range(N):
        K.push(step._stage[0], [step.ws.xin.data_ptr()])
        K.push(step._stage[1], [step.target.data_ptr()])
        step.run_device()
        step.ws.loss.item()


copy_ms = {}


def copy_graph(xs, ts, name, run=True):
    def body():
        cs = step._streams()
        evs = []
        for _ in range(N):
            cs.wait_stream(stream)
            with torch.cuda.stream(cs):
                a, b = torch.cuda.Event(True), torch.cuda.Event(True)
                a.record(cs)
                step._stage[0].copy_(xs, non_blocking=True)
                step._stage[1].copy_(ts, non_blocking=True)
                b.record(cs)
                evs.append((a, b))
            if run:
                step.run_device()
                step.ws.loss.item()
            else:
                cs.synchronize()
        stream.wait_stream(cs)
        torch.cuda.synchronize()
        copy_ms[name] = sum(a.elapsed_time(b) for a, b in evs) / N
    return body


for _ in range(3):
    step.run_device()
step.warm_prefetch()
step(xh, th)
res = {}
for rnd in range(2):
    for name, body in (("graph", graph), ("graph+sync", graph_sync), ("push+graph", push_graph),
                       ("h2d||graph", copy_graph(xh, th, "h2d||graph")),
                       ("d2d||graph", copy_graph(xd, td, "d2d||graph")), ("h2d alone", copy_graph(xh, th, "h2d alone", False)),
                       ("call", call(xh, th)), ("call_d2d", call(xd, td))):
        t = timed(body)
        res[name] = min(res.get(name, 1e9), t)
if comm.rank == 0:
    print(f"n={comm.world_size} " + "  ".join(f"{k} {v:.3f} ms" for k, v in res.items()), flush=True)
    print("rank-0 copy durations: " + "  ".join(f"{k} {v:.3f} ms" for k, v in copy_ms.items()), flush=True)
if comm.world_size > 1:
    dist.barrier()
os._exit(0)
