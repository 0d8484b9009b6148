"""Pinned H2D + D2H (512 MiB each, both directions at once) on every rank at the same time:
the PCIe bound of the N>1 e2e leg.  torchrun --nproc-per-node N tools/exp/pcie_ranks.py"""
import os, time
import torch
import torch.distributed as dist
rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
n = 512 << 20
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); dist.barrier()
    t = time.perf_counter()
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    if rep == 2:
        print(f"rank {rank}: both directions at once, {n / dt / 1e9:.1f} GB/s per direction", flush=True)
dist.destroy_process_group()
