"""Per-phase timeline of Communicator.ring_allreduce (CUDA events after every
wait and launch), per rank.  torchrun --nproc-per-node N tools/prof_allreduce.py [MiB]"""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import torch.distributed as dist

from oracle import oracle as O
from paper_2308_05199_b200 import comm


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    mib = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    n = mib * (1 << 18)
    x = torch.from_numpy(O.smooth_field(n, 0.37 * rank)).to(dev)
    c = comm.Communicator(dist.group.WORLD, dev)
    if len(sys.argv) > 2:
        c.ag_mode = sys.argv[2]
    out = torch.empty_like(x)
    for _ in range(3):
        c.ring_allreduce(x, 1e-4, "sum", out)
    torch.cuda.synchronize()
    for rep in range(2):
        dist.barrier()
        c.events = []
        c.ring_allreduce(x, 1e-4, "sum", out)
        torch.cuda.synchronize()
        ev = c.events
        c.events = None
        t0 = ev[0][1]
        line = " ".join(f"{lab}:{t0.elapsed_time(e) * 1e3:.0f}" for lab, e in ev[1:])
        for r in range(world):
            if r == rank:
                print(f"rank{rank} rep{rep} {line}", flush=True)
            dist.barrier()
    c.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
