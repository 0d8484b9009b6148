"""PCIe bound of the N=1 e2e leg: pinned H2D alone, D2H alone and both directions at once
(64 MiB + 7 MiB per direction, like one codec round trip).  python tools/exp/pcie_bw.py"""
import torch, time
n = 64 << 20
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=20):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    return n / dt / 1e9
run(True, True, 3)
print("h2d GB/s %.1f" % run(True, False))
print("d2h GB/s %.1f" % run(False, True))
print("both, per direction GB/s %.1f" % run(True, True))
