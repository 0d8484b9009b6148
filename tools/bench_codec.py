"""Quick codec throughput probe (CUDA events, L2 flushed between iterations)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2308_05199_b200 as gz
from paper_2308_05199_b200 import _lib as L
from oracle import oracle as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
eb = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
x = torch.from_numpy(O.smooth_field(n)).cuda()
ws = gz.Workspace()
blob = gz.compress(x, eb, ws)
lib = L.lib()
cap = int(lib.gz_compress_bound(n)); out = torch.empty(cap, dtype=torch.uint8, device="cuda")
sc = torch.empty(int(lib.gz_sidecar_bytes(n)), dtype=torch.uint8, device="cuda")
tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))
y = torch.empty(n, dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def comp():
    lib.gz_compress(x.data_ptr(), n, eb, 32, out.data_ptr(), cap, ws.len_ptr(), sc.data_ptr(), None, tws.data_ptr(), tws.numel(), ws.status_ptr(), s)
def dec():
    lib.gz_decompress_sidecar(out.data_ptr(), sc.data_ptr(), n, eb, y.data_ptr(), ws.status_ptr(), s)
only = sys.argv[3] if len(sys.argv) > 3 else "both"
for name, fn in (("compress", comp), ("decompress", dec)):
    if only != "both" and name != only: continue
    ts = []
    for it in range(23):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if it >= 3: ts.append(a.elapsed_time(b) * 1e-3)
    t = float(np.median(ts))
    L_ = len(blob)
    gbs = (4 * n + L_) / t / 1e9
    print(f"{name:10s} n={n} eb={eb} blob={L_} CR={4*n/L_:.3f} median {t*1e6:8.2f} us  min {min(ts)*1e6:8.2f} us  {gbs:8.1f} GB/s  ({gbs/6555.5*100:.1f}% of 6555.5)")
if only == "both": assert bytes(gz.decompress(blob, ws).cpu().numpy()) is not None
