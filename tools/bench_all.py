"""One-GPU regression set: compress / decompress / fused step (CUDA events, L2 flushed).
python tools/bench_all.py [log2 sizes...]   (default 24 27)
GZ_DATA=noise: uniform noise in [-1, 1) instead of the smooth field; GZ_EB: error bound (default 1e-4)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2308_05199_b200._lib as L
if os.environ.get("GZ_LIB"):
    L.LIB_PATH = os.environ["GZ_LIB"]
import paper_2308_05199_b200 as gz
from oracle import oracle as O

lib = L.lib()
EB = float(os.environ.get("GZ_EB", "1e-4"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def timeit(fn, reps=20):
    ts = []
    for it in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


for lg in [int(v) for v in sys.argv[1:]] or [24, 27]:
    n = 1 << lg
    if os.environ.get("GZ_DATA") == "noise":
        g = torch.Generator(device="cuda").manual_seed(lg)
        x = torch.rand(n, device="cuda", generator=g) * 2 - 1
        y = torch.rand(n, device="cuda", generator=g) * 2 - 1
    else:
        x = torch.from_numpy(O.smooth_field(n)).cuda()
        y = torch.from_numpy(O.smooth_field(n, 0.37)).cuda()
    ws = gz.Workspace()
    cap = int(lib.gz_compress_bound(n))
    scb = int(lib.gz_sidecar_bytes(n))
    tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))
    b1, s1 = torch.empty(cap, dtype=torch.uint8, device="cuda"), torch.empty(scb, dtype=torch.uint8, device="cuda")
    b2, s2 = torch.empty(cap, dtype=torch.uint8, device="cuda"), torch.empty(scb, dtype=torch.uint8, device="cuda")
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    l1 = torch.zeros(2, dtype=torch.int64, device="cuda")
    comp = lambda: lib.gz_compress(x.data_ptr(), n, EB, 32, b1.data_ptr(), cap, l1.data_ptr(), s1.data_ptr(), None,
                                   tws.data_ptr(), tws.numel(), ws.status_ptr(), s)
    dec = lambda: lib.gz_decompress_sidecar(b1.data_ptr(), s1.data_ptr(), n, EB, out.data_ptr(), ws.status_ptr(), s)
    step = lambda: lib.gz_reduce_step(b1.data_ptr(), s1.data_ptr(), y.data_ptr(), n, EB, 0, None, b2.data_ptr(), cap,
                                      l1.data_ptr() + 8, s2.data_ptr(), tws.data_ptr(), tws.numel(), ws.status_ptr(), s)
    comp()
    torch.cuda.synchronize()
    Lb = int(l1[0].item())
    tc, td, tst = timeit(comp), timeit(dec), timeit(step)
    gb = lambda t, by: by / t / 1e3
    print(f"2^{lg}: compress {tc:7.1f} us ({gb(tc, 4*n+Lb):6.0f} GB/s)  decompress {td:7.1f} us ({gb(td, 4*n+Lb):6.0f} GB/s)"
          f"  step {tst:7.1f} us ({gb(tst, 4*n+2*Lb):6.0f} GB/s)  CR {4*n/Lb:.3f}", flush=True)
