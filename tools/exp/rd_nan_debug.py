"""Debug: rd_allreduce with a NaN on rank 1 at N=3 (absorber), statuses per rank."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch, torch.distributed as dist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank % torch.cuda.device_count())
dev = torch.device("cuda", torch.cuda.current_device())
dist.init_process_group("gloo")
from paper_2308_05199_b200 import comm
from oracle import oracle as O
c = comm.Communicator(dist.group.WORLD, dev)
n = 100_003
xs = [O.smooth_field(n, 0.5 * r) for r in range(world)]
xs[1][54_321] = np.nan
xs[2][3] = np.inf
xt = torch.from_numpy(xs[rank]).to(dev)
try:
    c.rd_allreduce(xt, 1e-4, check=False)
    torch.cuda.synchronize()
    st = c.ws.status[:4].cpu().numpy().view(np.uint64)
    print(f"rank {rank} status {[hex(int(v)) for v in st]}", flush=True)
    c.check()
except Exception as e:
    print(f"rank {rank} raised {e!r}", flush=True)
c.close()
dist.destroy_process_group()
