"""Minimal driver for ncu: a few codec launches on the cfg1 field.
python tools/prof_codec.py [n] [both|compress|step]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2308_05199_b200 as gz
from paper_2308_05199_b200 import collectives as C
from oracle import oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
x = torch.from_numpy(O.smooth_field(n)).cuda()
ws = gz.Workspace()
only = sys.argv[2] if len(sys.argv) > 2 else "both"
blob = gz.compress(x, 1e-4, ws)
if only == "step":
    y = torch.from_numpy(O.smooth_field(n, 0.37)).cuda()
    for _ in range(3):
        out = C.reduce_step(blob, y, 1e-4, "sum", ws)
else:
    for _ in range(3):
        blob = gz.compress(x, 1e-4, ws)
        if only == "both":
            y = gz.decompress(blob, ws)
torch.cuda.synchronize()
print("ok", len(blob))
