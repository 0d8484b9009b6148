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
noflush = len(sys.argv) > 2
ws = gz.Workspace()
dbg = torch.zeros(4096 * 24 * 12 + 16384 * 12, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(4):
    if not noflush: flush.zero_()
    lib.gz_debug_set_timestamps(dbg.data_ptr() if it == 3 else None)
    b = gz.compress(x, 1e-4, ws)
torch.cuda.synchronize()
lib.gz_debug_set_timestamps(None)
d = dbg.cpu().numpy()
k1 = d[:4096 * 24 * 12].reshape(-1, 12); k1 = k1[k1[:, 0] > 0]
k2 = d[4096 * 24 * 12:4096 * 24 * 12 + 16384 * 8].reshape(-1, 8); k2 = k2[k2[:, 0] > 0]
k3 = d[4096 * 24 * 12 + 16384 * 8:].reshape(-1, 4); k3 = k3[k3[:, 3] > 0]
clk = 1.965e3  # cycles per us
print(f"n={n} K1 warps {len(k1)} K2 ctas {len(k2)}")
print(f"K1 end (globaltimer) p50 {np.median(k1[:,1]) / 1e3:.1f} max {k1[:,1].max() / 1e3:.1f} (us, abs)")
t0 = k1[:, 0].min()
print(f"K1 start->end per warp us: p50 {np.median((k1[:,1]-k1[:,0]))/1e3:.1f} max {((k1[:,1]-k1[:,0])).max()/1e3:.1f}; K1 span {(k1[:,1].max()-t0)/1e3:.1f}")
print(f"K2 start after K1 start: min {(k2[:,0].min()-t0)/1e3:.1f} p50 {(np.median(k2[:,0])-t0)/1e3:.1f} max {(k2[:,0].max()-t0)/1e3:.1f}; K2 end max {(k2[:,7].max()-t0)/1e3:.1f}")
for name, i in (("griddep wait", 1), ("loads+scan", 2), ("copy", 3), ("retire", 4)):
    v = k2[:, i] / clk
    print(f"  K2 {name:12s} us: p10 {np.percentile(v,10):7.2f} p50 {np.median(v):7.2f} p90 {np.percentile(v,90):7.2f} max {v.max():7.2f}")
for name, i in (("batch0 first tile (loads+shfl+stores)", 0), ("batch0 other 3 tiles", 1), ("remaining batches", 2)):
    v = k3[:, i] / clk
    print(f"  K2 copy {name:36s} us: p10 {np.percentile(v,10):7.2f} p50 {np.median(v):7.2f} p90 {np.percentile(v,90):7.2f} max {v.max():7.2f}")
