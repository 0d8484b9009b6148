"""Per-CTA phase timeline of the single-kernel compressor (experimental build with
-DGZ_PHASE_STAMPS).  python tools/exp/phases.py lib.so [n]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from oracle import oracle as O

L = ctypes.CDLL(sys.argv[1])
u64, u32, p, dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_double
L.gz_compress.argtypes = [p, u64, dbl, u32, p, u64, p, p, p, p, u64, p, p]
L.gz_compress_bound.restype = L.gz_workspace_bytes.restype = L.gz_sidecar_bytes.restype = u64
L.gz_compress_bound.argtypes = L.gz_workspace_bytes.argtypes = L.gz_sidecar_bytes.argtypes = [u64]
L.gz_workspace_init.argtypes = [p, u64, p]
L.gz_exp_phase_stamps.argtypes = [p, u64]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 24
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
for it in range(5):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    L.gz_compress(x.data_ptr(), n, 1e-4, 32, blob.data_ptr(), cap, st.data_ptr() + 32, sc.data_ptr(), None,
                  ws.data_ptr(), wsb, st.data_ptr(), s.cuda_stream)
    b.record(s)
    torch.cuda.synchronize()
    h = np.zeros(1024 * 8, np.uint64)
    L.gz_exp_phase_stamps(h.ctypes.data, h.nbytes)
    h = h.reshape(1024, 8)[:148].astype(np.int64)
    t0 = h[:, 0].min()
    r = (h[:, :8] - t0) / 1e3
    print(f"n=2^{n.bit_length()-1} event {a.elapsed_time(b)*1e3:7.1f} us | start min/max {r[:,0].min():6.1f}/{r[:,0].max():6.1f}"
          f" | encoded min/med/max {r[:,1].min():6.1f}/{np.median(r[:,1]):6.1f}/{r[:,1].max():6.1f}"
          f" | barrier {r[:,2].max():6.1f} | scan1 {r[:,5].max():6.1f} scan2 {r[:,6].max():6.1f} | range copied max {r[:,3].max():6.1f} | tail copied max {r[:,4].max():6.1f}")
