"""Compress timing: full, empty gather (launch + retire only), no gather."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2308_05199_b200 as gz
from paper_2308_05199_b200 import _lib as L
from oracle import oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
lib = L.lib()
lib.gz_debug_set_flags.argtypes = [ctypes.c_int]
x = torch.from_numpy(O.smooth_field(n)).cuda()
ws = gz.Workspace()
cap = int(lib.gz_compress_bound(n)); out = torch.empty(cap, dtype=torch.uint8, device="cuda")
sc = torch.empty(int(lib.gz_sidecar_bytes(n)), dtype=torch.uint8, device="cuda")
tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def comp():
    lib.gz_compress(x.data_ptr(), n, 1e-4, 32, out.data_ptr(), cap, ws.len_ptr(), sc.data_ptr(), None, tws.data_ptr(), tws.numel(), ws.status_ptr(), s)
res = {}
for flags in (0, 2, 0, 2):
    lib.gz_debug_set_flags(flags)
    ts = []
    for it in range(23):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); comp(); b.record(); torch.cuda.synchronize()
        if it >= 3: ts.append(a.elapsed_time(b) * 1e3)
    res[flags] = float(np.median(ts))
lib.gz_debug_set_flags(0)
print(f"n={n}: full {res[0]:.1f} us, empty gather {res[2]:.1f} us -> gather work {res[0]-res[2]:.1f} us")
