"""A/B: compress time of two builds of libgzccl.so (same C ABI) on the cfg1 field
(2^24, L2 flushed) and on 2^27.  python tools/exp/ab_codec.py new.so old.so"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from oracle import oracle as O

u64, u32, p, dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_double
libs = {}
persist = int(os.environ.get("PERSIST_MB", "0"))
if persist:
    import glob
    import nvidia.cuda_runtime as _cr
    cands = glob.glob(os.path.join(os.path.dirname(_cr.__file__), "lib", "libcudart*.so*")) + ["libcudart.so"]
    for c in cands:
        try:
            rt = ctypes.CDLL(c)
            break
        except OSError:
            rt = None
    torch.cuda.init()
    rc = rt.cudaDeviceSetLimit(ctypes.c_int(6), ctypes.c_size_t(persist << 20)) if rt else -1
    v = ctypes.c_size_t(0)
    rt.cudaDeviceGetLimit(ctypes.byref(v), ctypes.c_int(6))
    print("persisting L2 limit rc", rc, "now", v.value >> 20, "MB")
for path in sys.argv[1:]:
    L = ctypes.CDLL(path)
    L.gz_compress.argtypes = [p, u64, dbl, u32, p, u64, p, p, p, p, u64, p, p]
    L.gz_compress_bound.restype = L.gz_workspace_bytes.restype = L.gz_sidecar_bytes.restype = u64
    L.gz_compress_bound.argtypes = L.gz_workspace_bytes.argtypes = L.gz_sidecar_bytes.argtypes = [u64]
    L.gz_workspace_init.argtypes = [p, u64, p]
    L.gz_decompress_sidecar.argtypes = [p, p, u64, dbl, p, p, p]
    libs[os.path.basename(path)] = L
s = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n in (1 << 24, 1 << 27):
    x = torch.from_numpy(O.smooth_field(n)).cuda()
    for name, L in libs.items():
        cap = L.gz_compress_bound(n)
        blob = torch.empty(cap, dtype=torch.uint8, device="cuda")
        sc = torch.empty(L.gz_sidecar_bytes(n), dtype=torch.uint8, device="cuda")
        wsb = L.gz_workspace_bytes(n)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        L.gz_workspace_init(ws.data_ptr(), wsb, s.cuda_stream)
        st = torch.full((8,), -1, dtype=torch.int64, device="cuda")
        ts = []
        for it in range(12):
            if n == 1 << 24:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            rc = L.gz_compress(x.data_ptr(), n, 1e-4, 32, blob.data_ptr(), cap, st.data_ptr() + 32, sc.data_ptr(), None,
                               ws.data_ptr(), wsb, st.data_ptr(), s.cuda_stream)
            b.record(s)
            torch.cuda.synchronize()
            assert rc == 0, rc
            if it >= 2:
                ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        y = torch.empty(n, dtype=torch.float32, device="cuda")
        td = []
        for it in range(12):
            if n == 1 << 24:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            rc = L.gz_decompress_sidecar(blob.data_ptr(), sc.data_ptr(), n, 1e-4, y.data_ptr(), st.data_ptr(), s.cuda_stream)
            b.record(s)
            torch.cuda.synchronize()
            assert rc == 0, rc
            if it >= 2:
                td.append(a.elapsed_time(b) * 1e3)
        td.sort()
        print(f"n=2^{n.bit_length()-1} {name:24s} compress median {ts[len(ts)//2]:8.1f} us  min {ts[0]:8.1f}  len {int(st[4].item())}"
              f" | decompress median {td[len(td)//2]:8.1f} min {td[0]:8.1f}")
