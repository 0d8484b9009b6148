"""Per-call device time of small codec calls without host cost: 20 calls captured
in one CUDA graph, replayed (no L2 flush).  python tools/exp/small.py [log2 sizes]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2308_05199_b200._lib as L
if os.environ.get("GZ_LIB"):
    L.LIB_PATH = os.environ["GZ_LIB"]
import paper_2308_05199_b200 as gz
from oracle import oracle as O

lib = L.lib()
R = 20
for lg in [int(v) for v in sys.argv[1:]] or [16, 18, 20]:
    n = 1 << lg
    x = torch.from_numpy(O.smooth_field(n)).cuda()
    y = torch.from_numpy(O.smooth_field(n, 0.37)).cuda()
    ws = gz.Workspace()
    cap, scb = int(lib.gz_compress_bound(n)), int(lib.gz_sidecar_bytes(n))
    tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))
    b1, s1 = torch.empty(cap, dtype=torch.uint8, device="cuda"), torch.empty(scb, dtype=torch.uint8, device="cuda")
    b2, s2 = torch.empty(cap, dtype=torch.uint8, device="cuda"), torch.empty(scb, dtype=torch.uint8, device="cuda")
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    l1 = torch.zeros(2, dtype=torch.int64, device="cuda")
    st = torch.cuda.Stream()
    res = {}
    for name in ("compress", "decompress", "step", "stamp"):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            s = st.cuda_stream
            for _ in range(R):
                if name == "compress":
                    lib.gz_compress(x.data_ptr(), n, 1e-4, 32, b1.data_ptr(), cap, l1.data_ptr(), s1.data_ptr(), None,
                                    tws.data_ptr(), tws.numel(), ws.status_ptr(), s)
                elif name == "decompress":
                    lib.gz_decompress_sidecar(b1.data_ptr(), s1.data_ptr(), n, 1e-4, out.data_ptr(), ws.status_ptr(), s)
                elif name == "step":
                    lib.gz_reduce_step(b1.data_ptr(), s1.data_ptr(), y.data_ptr(), n, 1e-4, 0, None, b2.data_ptr(), cap,
                                       l1.data_ptr() + 8, s2.data_ptr(), tws.data_ptr(), tws.numel(), ws.status_ptr(), s)
                else:
                    lib.gz_debug_stamp(l1.data_ptr(), s)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        res[name] = a.elapsed_time(b) * 1e3 / R
    print(f"2^{lg}: " + "  ".join(f"{k} {v:.1f} us" for k, v in res.items()), flush=True)
