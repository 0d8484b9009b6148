"""Allgather overlap: decode of a 2^25-value blob alone vs beside a peer-copy kernel
(the allgather's pull of the next owner).  python tools/exp/ag_overlap.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2308_05199_b200 as gz
from paper_2308_05199_b200 import _lib as L
from oracle import oracle as O

lib = L.lib()
torch.cuda.set_device(0)
L.check(lib.gz_enable_peer_access(1), "peer")
n = 1 << 25
x = torch.from_numpy(O.smooth_field(n, 0.3)).cuda()
ws = gz.Workspace()
cap, scb = int(lib.gz_compress_bound(n)), int(lib.gz_sidecar_bytes(n))
tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))
blob = torch.empty(cap, dtype=torch.uint8, device="cuda")
sc = torch.empty(scb, dtype=torch.uint8, device="cuda")
ln = torch.zeros(1, dtype=torch.int64, device="cuda")
cur = torch.cuda.current_stream()
L.check(lib.gz_compress(x.data_ptr(), n, 1e-4, 32, blob.data_ptr(), cap, ln.data_ptr(), sc.data_ptr(), None,
                        tws.data_ptr(), tws.numel(), ws.status_ptr(), cur.cuda_stream), "c")
torch.cuda.synchronize()
LB = int(ln.item())
out = torch.empty(n, dtype=torch.float32, device="cuda")
peer = torch.ones(LB, dtype=torch.uint8, device="cuda:1")
land = torch.empty(LB, dtype=torch.uint8, device="cuda:0")
cs = torch.cuda.Stream()


class CI(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("d_len", ctypes.c_void_p), ("max_bytes", ctypes.c_uint64)]


def dec(reserve):
    P = ctypes.c_void_p * 1
    L.check(lib.gz_decompress_multi(P(blob.data_ptr()), P(sc.data_ptr()), (ctypes.c_uint64 * 1)(n), 1, 1e-4,
                                    P(out.data_ptr()), reserve, ws.status_ptr(), cur.cuda_stream), "d")


def copy(budget):
    it = (CI * 1)(CI(peer.data_ptr(), land.data_ptr(), None, LB))
    L.check(lib.gz_copy_items_sms(it, 1, budget, cs.cuda_stream), "copy")


def timeit(fn, reps=10):
    ts = []
    for i in range(reps + 2):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        fn()
        b.record(cur)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


print(f"blob {LB / 1e6:.1f} MB")
for r in (0, 24):
    print(f"decode alone, reserve {r}: {timeit(lambda: dec(r)):.1f} us")


def both(r, budget):
    ev = torch.cuda.Event()
    ev.record(cur)
    cs.wait_event(ev)
    copy(budget)
    dec(r)
    cur.wait_stream(cs)


for r, b in ((24, 24), (48, 48), (0, 24), (24, 8), (12, 12)):
    print(f"decode reserve {r} + copy budget {b} concurrently: {timeit(lambda: both(r, b)):.1f} us")
print(f"copy alone budget 24: {timeit(lambda: (copy(24), cur.wait_stream(cs))):.1f} us")


def ce(n_bytes=LB):
    with torch.cuda.stream(cs):
        land[:n_bytes].copy_(peer[:n_bytes], non_blocking=True)


def both_ce(r):
    ev = torch.cuda.Event()
    ev.record(cur)
    cs.wait_event(ev)
    ce()
    dec(r)
    cur.wait_stream(cs)


print(f"CE copy alone: {timeit(lambda: (ce(), cur.wait_stream(cs))):.1f} us")
for r in (0, 8):
    print(f"decode reserve {r} + CE copy concurrently: {timeit(lambda: both_ce(r)):.1f} us")
