"""Device-side timeline of a REPLAYED (CUDA-graph) ring allreduce: %globaltimer
stamps at every mark of Communicator._ring, captured into the graph.
torchrun --nproc-per-node N tools/prof_ring_stamps.py [MiB ...]   (default 1 16 64)"""
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
    for mib in [int(a) for a in sys.argv[1:]] or [1, 16, 64]:
        n = mib * (1 << 18)
        x = torch.from_numpy(O.smooth_field(n, 0.37 * rank)).to(dev)
        c = comm.Communicator(dist.group.WORLD, dev)
        c.stamps = torch.zeros(128, dtype=torch.int64, device=dev)
        if os.environ.get("GZ_AG_MODE"):
            c.ag_mode = os.environ["GZ_AG_MODE"]
        if os.environ.get("GZ_EARLY_PULL"):
            c.early_pull = os.environ["GZ_EARLY_PULL"] == "1"
        if os.environ.get("GZ_NO_STAMPS"):
            c.stamps = None
        out = torch.empty_like(x)
        for _ in range(4):  # eager, capture, replays
            c.ring_allreduce(x, 1e-4, "sum", out)
        torch.cuda.synchronize()
        res = []
        for rep in range(5):
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            c.ring_allreduce(x, 1e-4, "sum", out)
            b.record()
            torch.cuda.synchronize()
            st = c.stamps[: len(c.stamp_labels)].tolist() if c.stamps is not None else [0]
            res.append((a.elapsed_time(b) * 1e3, st))
        tot, st = sorted(res)[len(res) // 2]
        line = " ".join(f"{lab}:{(t - st[0]) / 1e3:.1f}" for lab, t in zip(c.stamp_labels[1:], st[1:]))
        for r in range(world):
            if r == rank:
                print(f"{mib} MiB rank{rank} total {tot:.1f} us | {line}", flush=True)
            dist.barrier()
        c.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
