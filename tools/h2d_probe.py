"""Host->device copy bandwidth per rank with every rank copying at once (pinned host memory),
under torchrun: is the e2e input feed limited per GPU link or by the host in aggregate?"""
import os
import sys
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rank = int(os.environ.get("RANK", "0"))
world = int(os.environ.get("WORLD_SIZE", "1"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
if world > 1:
    dist.init_process_group("nccl")
nbytes = int(os.environ.get("H2D_BYTES", str(512 << 20)))
h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
h.fill_(1.0)
d = torch.empty_like(h, device="cuda")
for mode in ("alone", "together"):
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if mode == "alone" and world > 1:
        # one rank at a time
        res = None
        for r in range(world):
            if r == rank:
                s, e = torch.cuda.Event(True), torch.cuda.Event(True)
                s.record()
                for _ in range(5):
                    d.copy_(h, non_blocking=True)
                e.record()
                torch.cuda.synchronize()
                res = 5 * nbytes / (s.elapsed_time(e) / 1e3) / 1e9
            dist.barrier()
    else:
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(5):
            d.copy_(h, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        res = 5 * nbytes / (s.elapsed_time(e) / 1e3) / 1e9
    if world > 1:
        t = torch.tensor([res], device="cuda")
        allv = [torch.zeros(1, device="cuda") for _ in range(world)]
        dist.all_gather(allv, t)
        vals = [round(float(v), 1) for v in allv]
    else:
        vals = [round(res, 1)]
    if rank == 0:
        print(f"H2D {mode}: per-rank GB/s {vals}, sum {sum(vals):.1f}", flush=True)
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
