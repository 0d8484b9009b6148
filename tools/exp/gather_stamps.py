"""%globaltimer timeline of one cfg1 compress with a GZ_DIAG_STAMPS build:
encoder warps' loop ends, gather groups' start / base-known / copied times.
python tools/exp/gather_stamps.py abso/diag.so"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from oracle import oracle as O

u64, u32, p, dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_double
L = ctypes.CDLL(sys.argv[1])
L.gz_compress.argtypes = [p, u64, dbl, u32, p, u64, p, p, p, p, u64, p, p]
L.gz_compress_bound.restype = L.gz_workspace_bytes.restype = L.gz_sidecar_bytes.restype = u64
L.gz_compress_bound.argtypes = L.gz_workspace_bytes.argtypes = L.gz_sidecar_bytes.argtypes = [u64]
L.gz_workspace_init.argtypes = [p, u64, p]
L.gz_diag_stamps.argtypes = [p, p]
L.gz_debug_stamp.argtypes = [p, p]
n = 1 << 24
s = torch.cuda.current_stream()
x = torch.from_numpy(O.smooth_field(n)).cuda()
cap = L.gz_compress_bound(n)
blob = torch.empty(cap, dtype=torch.uint8, device="cuda")
sc = torch.empty(L.gz_sidecar_bytes(n), dtype=torch.uint8, device="cuda")
wsb = L.gz_workspace_bytes(n)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
L.gz_workspace_init(ws.data_ptr(), wsb, s.cuda_stream)
st = torch.full((8,), -1, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(4):
    flush.zero_(); flush.sum()
    stamp = torch.zeros(2, dtype=torch.int64, device="cuda")
    L.gz_debug_stamp(stamp.data_ptr(), s.cuda_stream)
    L.gz_compress(x.data_ptr(), n, 1e-4, 32, blob.data_ptr(), cap, st.data_ptr() + 32, sc.data_ptr(), None,
                  ws.data_ptr(), wsb, st.data_ptr(), s.cuda_stream)
    L.gz_debug_stamp(stamp.data_ptr() + 8, s.cuda_stream)
    torch.cuda.synchronize()
    gst = np.zeros(3 * 8192, dtype=np.uint64)
    est = np.zeros(256 * 32, dtype=np.uint64)
    L.gz_diag_stamps(gst.ctypes.data, est.ctypes.data)
    t0, t1 = [int(v) for v in stamp.cpu()]
    e = est.reshape(256, 32)[:148, :24].astype(np.int64) - t0
    g = gst.reshape(8192, 3)[:2048].astype(np.int64) - t0
    cta_end = e.max(axis=1)
    pct = lambda a: " ".join("%.1f" % (v / 1e3) for v in np.percentile(a, [0, 10, 50, 90, 100]))
    print(f"rep {rep}: stamp-to-stamp {(t1 - t0) / 1e3:.1f} us")
    print(f"  encoder warp loop end (us, p0 p10 p50 p90 p100): {pct(e.ravel())}")
    print(f"  encoder CTA end: {pct(cta_end)}")
    print(f"  gather group start: {pct(g[:, 0])}  base known: {pct(g[:, 1])}  copied: {pct(g[:, 2])}")
    print(f"  gather per group: base latency {pct(g[:, 1] - g[:, 0])}  copy {pct(g[:, 2] - g[:, 1])}")
