"""Does a CUDA graph shorten the encoder -> gather boundary?  cfg1 compress (L2 flushed)
as direct launches vs one graph replay.  python tools/exp/graph_codec.py [lib.so]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from oracle import oracle as O

u64, u32, p, dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_double
L = ctypes.CDLL(sys.argv[1] if len(sys.argv) > 1 else "paper_2308_05199_b200/libgzccl.so")
L.gz_compress.argtypes = [p, u64, dbl, u32, p, u64, p, p, p, p, u64, p, p]
L.gz_decompress_sidecar.argtypes = [p, p, u64, dbl, p, p, p]
L.gz_compress_bound.restype = L.gz_workspace_bytes.restype = L.gz_sidecar_bytes.restype = u64
L.gz_compress_bound.argtypes = L.gz_workspace_bytes.argtypes = L.gz_sidecar_bytes.argtypes = [u64]
L.gz_workspace_init.argtypes = [p, u64, p]
n = 1 << 24
torch.cuda.init()
cs = torch.cuda.Stream()
x = torch.from_numpy(O.smooth_field(n)).cuda()
cap = L.gz_compress_bound(n)
blob = torch.empty(cap, dtype=torch.uint8, device="cuda")
sc = torch.empty(L.gz_sidecar_bytes(n), dtype=torch.uint8, device="cuda")
wsb = L.gz_workspace_bytes(n)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
L.gz_workspace_init(ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream)
st = torch.full((8,), -1, dtype=torch.int64, device="cuda")
y = torch.empty(n, dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_r = torch.ones(256 << 20, dtype=torch.uint8, device="cuda").view(torch.int64)


def comp(s):
    assert L.gz_compress(x.data_ptr(), n, 1e-4, 32, blob.data_ptr(), cap, st.data_ptr() + 32, sc.data_ptr(), None,
                         ws.data_ptr(), wsb, st.data_ptr(), s) == 0


def dec(s):
    assert L.gz_decompress_sidecar(blob.data_ptr(), sc.data_ptr(), n, 1e-4, y.data_ptr(), st.data_ptr(), s) == 0


torch.cuda.synchronize()
with torch.cuda.stream(cs):
    comp(cs.cuda_stream)
    dec(cs.cuda_stream)
cs.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=cs):
    comp(cs.cuda_stream)
gd = torch.cuda.CUDAGraph()
with torch.cuda.graph(gd, stream=cs):
    dec(cs.cuda_stream)
torch.cuda.synchronize()
s = torch.cuda.current_stream()
res = {"direct": [], "graph": [], "dec_direct": [], "dec_graph": []}
for it in range(40):
    for mode in ("direct", "graph"):
        flush.zero_(); flush_r.sum()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(s)
        if mode == "direct":
            comp(s.cuda_stream)
        else:
            g.replay()
        b.record(s)
        if mode == "direct":
            dec(s.cuda_stream)
        else:
            gd.replay()
        c.record(s)
        torch.cuda.synchronize()
        if it >= 5:
            res[mode].append(a.elapsed_time(b) * 1e3)
            res["dec_" + mode].append(b.elapsed_time(c) * 1e3)
for k, v in res.items():
    v.sort()
    print(f"{k:12s} median {v[len(v)//2]:.1f} min {v[0]:.1f} us")
