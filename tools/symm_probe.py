import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
g = dist.group.WORLD
print(rank, "backend", symm.get_backend(torch.device("cuda")) if hasattr(symm, "get_backend") else None, flush=True)
try:
    symm.enable_symm_mem_for_group(g.group_name)
except Exception as e:
    print("enable err", e)
t = symm.empty(1 << 20, dtype=torch.float32, device="cuda")
hdl = symm.rendezvous(t, g.group_name)
print(rank, "ptrs", [hex(p) for p in hdl.buffer_ptrs], "mc", hdl.multicast_ptr, flush=True)
peer = (rank + 1) % world
pb = hdl.get_buffer(peer, (1024,), torch.float32, 0)
pb.fill_(float(rank + 1))            # write into the peer's buffer
hdl.barrier(channel=0)
torch.cuda.synchronize()
print(rank, "got", t[:2].tolist(), "expect", float((rank - 1) % world + 1), flush=True)
# graph capture of barrier + peer write
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph, stream=s):
        pb.add_(1.0)
        hdl.barrier(channel=1)
gph.replay(); torch.cuda.synchronize()
hdl.barrier(channel=0); torch.cuda.synchronize()
print(rank, "after graph", t[:2].tolist(), flush=True)
# timing of the barrier
ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
ev0.record()
for i in range(100):
    hdl.barrier(channel=i % 2)
ev1.record(); torch.cuda.synchronize()
print(rank, "barrier us", ev0.elapsed_time(ev1) * 10, flush=True)
# peer copy bandwidth (copy engine) 256 MB
src = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
big = symm.empty(64 << 20, dtype=torch.float32, device="cuda")
h2 = symm.rendezvous(big, g.group_name)
dst = h2.get_buffer(peer, (64 << 20,), torch.float32, 0)
for _ in range(3): dst.copy_(src)
ev0.record()
for _ in range(10): dst.copy_(src)
ev1.record(); torch.cuda.synchronize()
print(rank, "peer copy GB/s", 10 * 256e6 / (ev0.elapsed_time(ev1) * 1e-3) / 1e9, flush=True)
dist.barrier()
os._exit(0)
