"""Encoder claiming: fraction of tiles claimed from the global counter (1/2^s,
debug flag bits 4-6 = s; default 3) vs compress / fused-step time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import paper_2308_05199_b200 as gz
from paper_2308_05199_b200 import _lib as L
from oracle import oracle as O

lib = L.lib()
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_r = torch.ones(256 << 20, dtype=torch.uint8, device=dev).view(torch.int64)
for n in (1 << 24, 1 << 27):
    x = torch.from_numpy(O.smooth_field(n)).to(dev)
    ws = gz.Workspace(dev)
    ws.reset_status()
    cap = int(lib.gz_compress_bound(n))
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    sc = torch.empty(int(lib.gz_sidecar_bytes(n)), dtype=torch.uint8, device=dev)
    tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))
    s = torch.cuda.current_stream().cuda_stream

    def comp():
        L.check(lib.gz_compress(x.data_ptr(), n, 1e-4, 32, out.data_ptr(), cap, ws.len_ptr(), sc.data_ptr(), None,
                                tws.data_ptr(), tws.numel(), ws.status_ptr(), s), "gz_compress")

    res = []
    for sh in (1, 2, 3, 4, 5, 7):
        lib.gz_debug_set_flags(sh << 4)
        for _ in range(3):
            comp()
        ts = []
        for _ in range(30):
            flush.zero_()
            flush_r.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            comp()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        res.append(f"1/{1 << sh}: {ts[len(ts) // 2]:.1f}")
    lib.gz_debug_set_flags(0)
    print(f"n=2^{n.bit_length() - 1} compress us (median of 30):", ", ".join(res))

# fused reduce-scatter step (k_tile_encode<STEP> + gather) on the N = 4 chunk size
from paper_2308_05199_b200 import collectives as C

n = 1 << 25
ws = gz.Workspace(dev)
blob = gz.compress(torch.from_numpy(O.smooth_field(n)).to(dev), 1e-4, ws)
y = torch.from_numpy(O.smooth_field(n, 0.37)).to(dev)
res = []
for sh in (1, 2, 3, 4, 5, 7):
    lib.gz_debug_set_flags(sh << 4)
    for _ in range(3):
        C.reduce_step(blob, y, 1e-4, "sum", ws)
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        C.reduce_step(blob, y, 1e-4, "sum", ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    res.append(f"1/{1 << sh}: {ts[len(ts) // 2]:.1f}")
lib.gz_debug_set_flags(0)
print("n=2^25 fused step us (median of 20):", ", ".join(res))
