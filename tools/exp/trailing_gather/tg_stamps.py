"""EXPERIMENT: trailing-gather timeline at cfg1 (per-group / per-tile %globaltimer stamps)."""
import ctypes, os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..", "..")))
import numpy as np
import torch
from oracle import oracle as O
from paper_2308_05199_b200 import _lib
L = _lib.lib()
s = torch.cuda.current_stream()
n = 1 << 24
x = torch.from_numpy(O.smooth_field(n)).cuda()
cap = L.gz_compress_bound(n)
blob = torch.zeros(cap, dtype=torch.uint8, device="cuda")
sc = torch.zeros(L.gz_sidecar_bytes(n), dtype=torch.uint8, device="cuda")
wsb = L.gz_workspace_bytes(n)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
L.gz_workspace_init(ws.data_ptr(), wsb, s.cuda_stream)
st = torch.full((8,), -1, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(5):
    flush.zero_()
    torch.cuda.synchronize()
    L.gz_compress(x.data_ptr(), n, 1e-4, 32, blob.data_ptr(), cap, st.data_ptr() + 32, sc.data_ptr(), None,
                  ws.data_ptr(), wsb, st.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
gs = np.zeros((4, 16384), np.uint64)
ts = np.zeros((2, 16384), np.uint64)
L.gz_dbg_read.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
L.gz_dbg_read(gs.ctypes.data, ts.ctypes.data)
ng = 2048
g = gs[:, :ng].astype(np.int64)
t = ts.astype(np.int64)
t0 = min(g[0].min(), t[0][t[0] > 0].min())
g -= t0
t -= t0
print("tiles: packed (min/med/max)", t[0].min(), np.median(t[0]), t[0].max(), " published", t[1].min(), np.median(t[1]), t[1].max())
pub_g = t[1].reshape(ng, 8).max(1)
print("group: claim  own_ready  prefix_ready  done   (ns, percentiles 0/10/50/90/100)")
for i, name in enumerate(["claim", "own", "prefix", "done"]):
    print(f"{name:8s}", np.percentile(g[i], [0, 10, 50, 90, 100]).astype(int))
print("own_ready - last tile published", np.percentile(g[1] - pub_g, [0, 10, 50, 90, 100]).astype(int))
print("prefix - own", np.percentile(g[2] - g[1], [0, 10, 50, 90, 100]).astype(int))
print("done - prefix", np.percentile(g[3] - g[2], [0, 10, 50, 90, 100]).astype(int))
print("publish - pack", np.percentile(t[1] - t[0], [0, 10, 50, 90, 100]).astype(int))
# timeline: every 4 us, tiles published and groups done
for T in range(0, int(max(g[3].max(), t[1].max())) + 4000, 4000):
    print(f"t={T/1000:5.1f}us  tiles published {int((t[1] <= T).sum()):6d}  groups own-ready {int((g[1] <= T).sum()):5d}  done {int((g[3] <= T).sum()):5d}")
