"""Minimal driver for ncu: a few compress + decompress launches on the cfg1 field."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2308_05199_b200 as gz
from oracle import oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
x = torch.from_numpy(O.smooth_field(n)).cuda()
ws = gz.Workspace()
only = sys.argv[2] if len(sys.argv) > 2 else "both"
for _ in range(3):
    blob = gz.compress(x, 1e-4, ws)
    if only == "both":
        y = gz.decompress(blob, ws)
torch.cuda.synchronize()
print("ok", len(blob))
