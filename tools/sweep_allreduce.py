"""cfg4: allreduce message-size sweep (1 MiB .. 2 GiB per rank) x eb, gZ ring vs NCCL.

torchrun --nproc-per-node N tools/sweep_allreduce.py [max_mib]
Prints one markdown table (rank 0).  Inputs: the cfg2 smooth field per rank
(phase 0.37 r), generated on the device in f64 and rounded to f32."""
import math
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
import torch.distributed as dist

from paper_2308_05199_b200 import comm


def field(n, phase, dev):
    i = torch.arange(n, dtype=torch.float64, device=dev)
    return (0.5 * torch.sin(2 * math.pi * i / 65536 + phase) + 0.25 * torch.sin(2 * math.pi * i / 4099 + phase)).float()


def timed(fn, stream, reps):
    ts = []
    for _ in range(reps):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    t = torch.tensor([ts[len(ts) // 2]], device=stream.device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    max_mib = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    c = comm.Communicator(dist.group.WORLD, dev)
    s = torch.cuda.current_stream()
    rows = []
    mib = 1
    while mib <= max_mib:
        n = mib << 18
        x = field(n, 0.37 * rank, dev)
        out = torch.empty_like(x)
        y = x.clone()
        for _ in range(2):
            dist.all_reduce(y)
        tn = timed(lambda: dist.all_reduce(y), s, 7)
        for eb in (1e-2, 1e-3, 1e-4):
            for _ in range(2):
                c.ring_allreduce(x, eb, out=out)
            t = timed(lambda: c.ring_allreduce(x, eb, out=out), s, 7)
            cr = c.compression_ratio()
            rows.append((mib, eb, 4 * n / t / 1e9, cr, 4 * n / tn / 1e9))
        del x, out, y
        torch.cuda.empty_cache()
        mib *= 4 if mib < 1024 else 2
    if rank == 0:
        print(f"| MiB/rank | eb | gZ-Allreduce GB/s | CR (owned chunk) | NCCL all_reduce GB/s | ratio |  (N={world})")
        print("|---|---|---|---|---|---|")
        for mib, eb, g, cr, nc in rows:
            print(f"| {mib} | {eb:g} | {g:.1f} | {cr} | {nc:.1f} | {g / nc:.2f} |")
    c.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
