"""CUPTI timeline (torch.profiler) of replayed ring allreduce calls at small sizes:
every kernel / memset / memcpy of the graph with its start and duration on rank 0.
torchrun --nproc-per-node 2 tools/exp/small_timeline.py [MiB]"""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import torch
import torch.distributed as dist
from oracle import oracle as O
from paper_2308_05199_b200 import comm

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
mib = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = mib << 18
x = torch.from_numpy(O.smooth_field(n, 0.37 * rank)).to(dev)
out = torch.empty_like(x)
c = comm.Communicator(dist.group.WORLD, dev)
for _ in range(4):
    c.ring_allreduce(x, 1e-4, "sum", out, check=False)
torch.cuda.synchronize()
c.check()
from torch.profiler import profile, ProfilerActivity
dist.barrier(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        dist.barrier()
        torch.cuda.synchronize()
        c.ring_allreduce(x, 1e-4, "sum", out, check=False)
        torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
if rank == 0:
    t0 = None
    for e in evs:
        if t0 is None or e.time_range.start - last_end > 200:
            t0 = e.time_range.start
            print("--- call")
        last_end = e.time_range.end
        print("%8.1f %7.1f  %s" % (e.time_range.start - t0, e.time_range.elapsed_us(), e.name[:90]))
c.close()
dist.destroy_process_group()
