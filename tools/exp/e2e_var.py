"""e2e codec throughput variance: repeated runs at 2..4 steps in flight."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2308_05199_b200 as gz
import bench
from oracle import oracle as O
n = 1 << 24
xh = O.smooth_field(n)
ref = O.compress(xh, 1e-4, threads=8)
xp = torch.from_numpy(xh).pin_memory()
for lanes in (2, 3, 4):
    ws = [gz.Workspace("cuda:0") for _ in range(lanes)]
    st = [torch.cuda.Stream() for _ in range(lanes)]
    bench.e2e_codec(gz, xp, ws, st, 2 * lanes, ref)
    res = []
    for rep in range(6):
        steps = 24
        wall, _ = bench.e2e_codec(gz, xp, ws, st, steps, ref)
        res.append(steps * 2 * (4 * n + len(ref)) / wall / 1e9)
    print(f"lanes={lanes}: " + " ".join("%.1f" % v for v in res), flush=True)
