"""Where the live compress time goes at 2^24 (bench.py's N=1 leg): events around
the call, the encoder alone (debug flag 1 = skip the gather), a CUDA graph of
the call, k back-to-back calls between one pair of events, and %globaltimer
stamps around the kernels."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import paper_2308_05199_b200 as gz
from paper_2308_05199_b200 import _lib as L
from oracle import oracle as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
lib = L.lib()
dev = torch.device("cuda", 0)
x = torch.from_numpy(O.smooth_field(n)).to(dev)
ws = gz.Workspace(dev)
ws.reset_status()
cap = int(lib.gz_compress_bound(n))
out = torch.empty(cap, dtype=torch.uint8, device=dev)
sc = torch.empty(int(lib.gz_sidecar_bytes(n)), dtype=torch.uint8, device=dev)
tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_r = torch.ones(256 << 20, dtype=torch.uint8, device=dev).view(torch.int64)
st = torch.cuda.Stream()
stamps = torch.zeros(8, dtype=torch.int64, device=dev)


def comp(s):
    L.check(lib.gz_compress(x.data_ptr(), n, 1e-4, 32, out.data_ptr(), cap, ws.len_ptr(), sc.data_ptr(), None,
                            tws.data_ptr(), tws.numel(), ws.status_ptr(), s), "gz_compress")


def fl():
    flush.zero_()
    flush_r.sum()


def timeit(fn, reps=20, k=1, do_flush=True, pre=None):
    ts = []
    with torch.cuda.stream(st):
        s = st.cuda_stream
        for _ in range(3):
            fn(s)
        for _ in range(reps):
            if pre:
                pre(s)
            if do_flush:
                fl()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(k):
                fn(s)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / k)
    ts.sort()
    return ts[len(ts) // 2]


print(f"n={n}")
print(f"compress (events, flushed): {timeit(comp):.1f} us")
print(f"compress (events, no flush): {timeit(comp, do_flush=False):.1f} us")
print(f"compress x10 back-to-back (no flush): {timeit(comp, k=10, do_flush=False):.1f} us per call")
def wsinit(s):  # the skipped gather does not re-zero the workspace counters
    L.check(lib.gz_workspace_init(tws.data_ptr(), tws.numel(), s), "gz_workspace_init")


lib.gz_debug_set_flags(1)
print(f"encoder only (flushed): {timeit(comp, pre=wsinit):.1f} us")
lib.gz_debug_set_flags(0)
with torch.cuda.stream(st):
    wsinit(st.cuda_stream)

# graph of one call
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    comp(st.cuda_stream)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=st):
        comp(st.cuda_stream)
print(f"graph replay (flushed): {timeit(lambda s: g.replay()):.1f} us")


def stamped(s):
    lib.gz_debug_stamp(ctypes.c_void_p(stamps.data_ptr()), ctypes.c_void_p(s))
    comp(s)
    lib.gz_debug_stamp(ctypes.c_void_p(stamps.data_ptr() + 8), ctypes.c_void_p(s))


print(f"stamped call (flushed): {timeit(stamped):.1f} us events; globaltimer span "
      f"{(int(stamps[1]) - int(stamps[0])) / 1e3:.1f} us")
