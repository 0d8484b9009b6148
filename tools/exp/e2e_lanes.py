"""e2e codec throughput through the public API with 1..4 steps in flight."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2308_05199_b200 as gz
import bench
from oracle import oracle as O
n = 1 << 24
xh = O.smooth_field(n)
ref = O.compress(xh, 1e-4, threads=8)
xp = torch.from_numpy(xh).pin_memory()
for lanes in (1, 2, 3, 4):
    ws = [gz.Workspace("cuda:0") for _ in range(lanes)]
    st = [torch.cuda.Stream() for _ in range(lanes)]
    bench.e2e_codec(gz, xp, ws, st, 2 * lanes, ref)
    steps = 24
    wall, _ = bench.e2e_codec(gz, xp, ws, st, steps, ref)
    print(f"lanes={lanes}: {steps * 2 * (4 * n + len(ref)) / wall / 1e9:.1f} GB/s  ({wall / steps * 1e3:.3f} ms/step)")
