import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2308_05199_b200._lib as L
L.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgzccl_dbg.so")
import paper_2308_05199_b200 as gz
from oracle import oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
lib = L.lib()
lib.gz_debug_set_timestamps.argtypes = [ctypes.c_void_p]
x = torch.from_numpy(O.smooth_field(n)).cuda()
ws = gz.Workspace()
dbg = torch.zeros(4096 * 4 * 12, dtype=torch.int64, device="cuda")
for it in range(4):
    lib.gz_debug_set_timestamps(dbg.data_ptr() if it == 3 else None)
    b = gz.compress(x, 1e-4, ws)
torch.cuda.synchronize()
d = dbg.cpu().numpy().reshape(-1, 12)
d = d[d[:, 0] > 0]
print(f"n={n} warps {len(d)} tiles/warp min {d[:,4].min()} max {d[:,4].max()} mean {d[:,4].mean():.2f}")
for name, i, j in (("phase A", 0, 1), ("prefix wait", 1, 2), ("copy_run", 2, 7), ("offsets+discard", 7, 3), ("total", 0, 3)):
    v = (d[:, j] - d[:, i]) / 1e3
    print(f"  {name:16s} us: p10 {np.percentile(v,10):8.2f} p50 {np.median(v):8.2f} p90 {np.percentile(v,90):8.2f} max {v.max():8.2f}")

durA = (d[:, 1] - d[:, 0]) / 1e3
wait = d[:, 5] / 1e3
sm = d[:, 10]
cta = d[:, 6]
print(f"  load-wait us: p10 {np.percentile(wait,10):.2f} p50 {np.median(wait):.2f} p90 {np.percentile(wait,90):.2f} max {wait.max():.2f}")
print(f"  corr(durA, wait) = {np.corrcoef(durA, wait)[0,1]:.3f}")
sms = np.unique(sm)
m = np.array([durA[sm == x].mean() for x in sms])
print(f"  per-SM mean durA: min {m.min():.1f} p50 {np.median(m):.1f} max {m.max():.1f}; slowest SMs {sms[np.argsort(-m)[:8]]}; fastest {sms[np.argsort(m)[:8]]}")
sd = np.array([durA[sm == x].std() for x in sms])
print(f"  within-SM std of durA: p50 {np.median(sd):.1f}")
print(f"  corr(durA, cta ticket) = {np.corrcoef(durA, cta)[0,1]:.3f}")
