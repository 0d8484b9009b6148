"""Per-warp K1 timestamps (experiment hook gz_debug_set_timestamps)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2308_05199_b200 as gz
from paper_2308_05199_b200 import _lib as L
from oracle import oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
lib = L.lib()
lib.gz_debug_set_timestamps.argtypes = [ctypes.c_void_p]
x = torch.from_numpy(O.smooth_field(n)).cuda()
ws = gz.Workspace()
dbg = torch.zeros(4096 * 24 * 12, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(4):
    flush.zero_()
    lib.gz_debug_set_timestamps(dbg.data_ptr() if it == 3 else None)
    b = gz.compress(x, 1e-4, ws)
torch.cuda.synchronize()
lib.gz_debug_set_timestamps(None)
k1 = dbg.cpu().numpy().reshape(-1, 12); k1 = k1[k1[:, 0] > 0]
t0 = k1[:, 0].min()
print(f"n={n} K1 warps {len(k1)}: per-warp busy p50 {np.median(k1[:,1]-k1[:,0])/1e3:.1f} us max {(k1[:,1]-k1[:,0]).max()/1e3:.1f}; span {(k1[:,1].max()-t0)/1e3:.1f} us; tiles/warp {k1[:,2].min()}..{k1[:,2].max()}")
